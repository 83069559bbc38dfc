"""The north_star multi-GPU path (efem_dist_*, dist2d.cu): element slabs,
row-owned CSR slices, off-rank contributions and column ids exchanged inside
libefem.  On one device: a LOCAL GROUP of P ranks (exchanges = device
copies, the same phases and buffers as over NCCL) and a one-rank NCCL
communicator.  The ranks' slices concatenated in rank order must be the
1-GPU matrices: pattern byte for byte, values bitwise (the ghost triangles'
local matrices come from the same closed-form code, summed in the same
ascending element order)."""
import numpy as np
import pytest
import torch

from parity import assert_row_close
from workloads import CONFIGS, NED0, RT0

pytestmark = pytest.mark.gpu


def _single(api, coords, elems, element):
    out = api.Assembler(coords, elems, element).assemble()
    return [t.cpu().numpy() for t in (out.row_ptr, out.col_idx, out.vals_M, out.vals_K)]


def _compare(got, want, bitwise=True):
    rp, ci, vm, vk = got
    assert np.array_equal(rp, want[0])
    assert np.array_equal(ci, want[1])
    if bitwise:
        assert vm.tobytes() == want[2].tobytes()
        assert vk.tobytes() == want[3].tobytes()
    else:
        assert_row_close(vm, want[2], want[0], what="M")
        assert_row_close(vk, want[3], want[0], what="K")


@pytest.mark.parametrize("element", [RT0, NED0], ids=["rt0", "ne0"])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_group_equals_single(element, P):
    from paper_1409_4618_b200 import api, dist

    coords, elems = api.build_mesh(2, 24, 0.2, 17)
    want = _single(api, coords, elems, element)
    g = dist.DistGroup(coords, elems, element, dist.slab_bounds(elems.shape[0], P))
    g.assemble()
    _compare(g.concat(), want)
    g.assemble()  # a second step into the same slices: identical
    _compare(g.concat(), want)
    # every node owned once, slabs' rows tile [0, R)
    infos = [g.info(r) for r in range(P)]
    assert infos[0][0] == 0 and infos[-1][1] == coords.shape[0]
    assert all(infos[r][1] == infos[r + 1][0] for r in range(P - 1))
    assert sum(w[1] for w in g.last) == want[0].size - 1


def test_group_unstructured_scattered_slabs():
    """A Delaunay mesh with shuffled element order and node labels: slabs are
    scattered, so ghosts, requests and owners are all over the mesh."""
    from scipy.spatial import Delaunay

    from paper_1409_4618_b200 import api, dist

    rng = np.random.default_rng(5)
    pts = np.concatenate([[[0, 0], [1, 0], [0, 1], [1, 1]], rng.random((1500, 2))])
    el = Delaunay(pts).simplices.astype(np.int32)
    perm = rng.permutation(pts.shape[0])
    pts = np.ascontiguousarray(pts[perm])
    el = np.ascontiguousarray(np.argsort(perm)[el][rng.permutation(el.shape[0])].astype(np.int32))
    coords, elems = torch.from_numpy(pts).cuda(), torch.from_numpy(el).cuda()
    for element in (RT0, NED0):
        want = _single(api, coords, elems, element)
        for P in (2, 5):
            g = dist.DistGroup(coords, elems, element, dist.slab_bounds(el.shape[0], P))
            g.assemble()
            _compare(g.concat(), want)


def test_group_config5_eight_ranks():
    """BASELINE config 5 (the 1/2/4/8-GPU sweep) as 8 ranks: the whole
    concatenated CSR against the 1-GPU one, and the per-step exchange volume
    O(interface): <= 1 MB per rank."""
    from paper_1409_4618_b200 import api, dist

    C = CONFIGS[5]
    coords, elems = api.build_mesh(2, C["n"], C["alpha"], C["seed"])
    want = _single(api, coords, elems, C["element"])
    torch.cuda.empty_cache()
    g = dist.DistGroup(coords, elems, C["element"], dist.slab_bounds(elems.shape[0], 8))
    g.assemble()
    _compare(g.concat(), want)
    sent = [g.info(r)[7] for r in range(8)]
    assert max(sent) <= 1 << 20, sent


def test_nccl_one_rank_equals_single():
    """The NCCL transport itself (efem_comm over one rank, in-process)."""
    import ctypes

    from paper_1409_4618_b200 import _lib, api, dist

    L = _lib.load()
    uid = (ctypes.c_ubyte * 128)()
    _lib.check("efem_comm_unique_id", L.efem_comm_unique_id(uid))
    comm = ctypes.c_void_p()
    _lib.check("efem_comm_init", L.efem_comm_init(ctypes.byref(comm), uid, 1, 0))
    try:
        C = CONFIGS[2]
        coords, elems = api.build_mesh(2, C["n"], C["alpha"], C["seed"])
        want = _single(api, coords, elems, C["element"])
        d = dist.DistAssembler(coords, elems, C["element"], 0, elems.shape[0], comm)
        s = d.assemble()
        w = d.window
        assert w[0] == 0 and w[2] == 0
        got = [t.cpu().numpy() for t in (s.row_ptr, s.col_idx, s.vals_M, s.vals_K)]
        _compare(got, want)
        d.close()
    finally:
        L.efem_comm_destroy(comm)


def test_group_degenerate_in_other_slab_reported():
    from paper_1409_4618_b200 import api, dist

    coords, elems = api.build_mesh(2, 8, 0.0, 0)
    c = coords.clone()
    v = elems[100].tolist()
    c[v[2]] = 0.5 * (c[v[0]] + c[v[1]])  # element 100 collapses (rank 1 of 2 holds it)
    g = dist.DistGroup(c, elems, RT0, dist.slab_bounds(elems.shape[0], 2))
    with pytest.raises(api._lib.EfemError) as ei:
        g.assemble()
    assert ei.value.status == -2


@pytest.mark.parametrize("element", [RT0, NED0], ids=["rt0", "ne0"])
def test_group_fan_overflow_off_rank0(element):
    """A 200-triangle disc whose centre has a middle node id: its fan overflows
    the fixed fan slots on a rank whose owned node range starts above 0, so
    the one-launch fallback (k_fan_fallback: scan, grid barriers, counting
    fill) runs with a node offset.  Slices concatenated = the 1-GPU CSR,
    bitwise, on the first and a replayed step."""
    from paper_1409_4618_b200 import api, dist
    from test_unstructured_gpu import fan_mesh

    pts, el = fan_mesh(200, 3)
    n = pts.shape[0]
    rng = np.random.default_rng(4)
    perm = rng.permutation(n)  # new id of node i
    perm[[0, int(np.where(perm == n // 2)[0][0])]] = perm[[int(np.where(perm == n // 2)[0][0]), 0]]
    assert perm[0] == n // 2
    c2 = np.empty_like(pts)
    c2[perm] = pts
    e2 = perm[el].astype(np.int32)
    coords, elems = torch.from_numpy(c2).cuda(), torch.from_numpy(e2).cuda()
    want = _single(api, coords, elems, element)
    offset_seen = False
    for P in (2, 3, 4):
        g = dist.DistGroup(coords, elems, element, dist.slab_bounds(elems.shape[0], P))
        infos = [g.info(r) for r in range(P)]
        owner = [r for r in range(P) if infos[r][0] <= n // 2 < infos[r][1]][0]
        offset_seen |= infos[owner][0] > 0  # the overflowing fan above the rank's first node
        for _ in range(2):
            g.assemble()
            _compare(g.concat(), want)
    assert offset_seen
