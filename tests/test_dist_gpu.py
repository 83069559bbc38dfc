"""Partitioned (multi-GPU) path on ONE GPU: the P ranks run one after another
in this process (no rank waits on another -- the collectives are replaced by
in-process concatenation, which is what all_gather returns).  The ranks'
slices must concatenate to the 1-GPU CSR byte for byte (same DOF numbering,
same per-row summation order)."""
import numpy as np

from parity import assert_row_close
import pytest
import torch

from oracle import oracle as ora
from workloads import NED0, RT0

pytestmark = pytest.mark.gpu

KINDS = [(2, RT0), (2, NED0), (3, RT0), (3, NED0)]
KIND_IDS = ["rt0_2d", "ne0_2d", "rt0_3d", "ne0_3d"]


def _exchange(parts, owned):
    """The O(interface) exchange of the owner-computes partition for P ranks
    in this process: every rank's total (== all_gather), the first-id answers
    (== all_to_all_single), placed into each rank's sub-mesh first ids."""
    from paper_1409_4618_b200 import dist

    P = len(parts)
    totals = torch.cat([dist._part_local_prefix(p, o) for p, o in zip(parts, owned)])
    sends = [dist._part_first_ids(p, totals, r) for r, p in enumerate(parts)]
    for r, p in enumerate(parts):
        segs = []
        for o, q in enumerate(parts):
            off = sum(q.send_splits[:r])
            segs.append(sends[o][off:off + q.send_splits[r]])
        recv = torch.cat(segs) if segs else torch.zeros(0, dtype=torch.int32, device="cuda")
        assert recv.numel() == sum(p.recv_splits)
        dist._part_place(p, recv)
        p.first_row = int(p.sub_first[p.l0].item()) if (not p.empty and p.l1 > p.l0) else 0
    # per rank and step: one total, its answers, its entry count
    return [dist.exchange_bytes(p) for p in parts]


def _parts(coords, elems, element, P):
    from paper_1409_4618_b200 import dist

    ranges = dist.node_ranges(coords.shape[0], P)
    parts = [dist.PartAssembler(coords, elems, element, lo, hi) for lo, hi in ranges]
    for p in parts:
        dist._exchange_plan(p, ranges)
    for r, p in enumerate(parts):
        dist._answer_plan(p, [parts[s].requests[r] for s in range(P)])
    return ranges, parts


def _emulate(coords, elems, element, P):
    from paper_1409_4618_b200 import dist

    ranges, parts = _parts(coords, elems, element, P)
    owned = [p.symbolic() for p in parts]
    _exchange(parts, owned)
    offs, total = dist.offsets_from_counts([p.owned_nnz for p in parts])
    slices = []
    for p in parts:
        s = p.alloc_slice()
        p.numeric(s)
        p.check()
        slices.append(s)
    return parts, slices, offs, total


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
@pytest.mark.parametrize("P", [2, 3, 8])
def test_partitioned_equals_single(dim, element, P):
    from paper_1409_4618_b200 import api, dist

    n = 24 if dim == 2 else 6
    coords, elems = api.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 17)
    one = api.Assembler(coords, elems, element).assemble()
    parts, slices, offs, total = _emulate(coords, elems, element, P)
    assert total == one.nnz
    rp, ci, vm, vk = dist.concat_slices(slices, offs)
    assert np.array_equal(rp, one.row_ptr.cpu().numpy())
    assert np.array_equal(ci, one.col_idx.cpu().numpy())
    # values: the partitioned path (bucket pipeline) and the 1-GPU 2D path
    # (node fans) evaluate the same closed forms in different orders
    assert_row_close(vm, one.vals_M.cpu().numpy(), rp, what="M")
    assert_row_close(vk, one.vals_K.cpu().numpy(), rp, what="K")
    # the ranks' first rows tile [0, R)
    firsts = [p.first_row for p in parts]
    assert firsts[0] == 0 and sorted(firsts) == firsts
    assert sum(p.owned_rows for p in parts) == one.n_rows


def test_partitioned_config5_against_oracle_rows():
    """BASELINE config 5 (the scaling sweep) split 8 ways; sampled rows of
    the concatenation against the oracle."""
    from paper_1409_4618_b200 import api, dist
    from workloads import CONFIGS

    C = CONFIGS[5]
    coords, elems = api.build_mesh(C["dim"], C["n"], C["alpha"], C["seed"])
    parts, slices, offs, total = _emulate(coords, elems, C["element"], 8)
    one = api.Assembler(coords, elems, C["element"])
    d2n, _, _ = one.enumerate_dofs()
    rp, ci, vm, vk = dist.concat_slices(slices, offs)
    full = one.assemble()
    assert np.array_equal(rp, full.row_ptr.cpu().numpy())
    assert np.array_equal(ci, full.col_idx.cpu().numpy())
    assert np.array_equal(vm, full.vals_M.cpu().numpy()) and np.array_equal(vk, full.vals_K.cpu().numpy())
    # a few rows at the rank boundaries against the oracle
    rows = []
    for p in parts:
        rows += [p.first_row, max(p.first_row - 1, 0), p.first_row + 1]
    rows = np.unique(np.array(rows))
    d2n_h = d2n.cpu().numpy()
    res = ora.rows_by_entity(2, C["element"], coords.cpu().numpy(), elems.cpu().numpy(), d2n_h[rows])
    for r, (cols, m, k) in zip(rows, res):
        lo, hi = rp[r], rp[r + 1]
        assert np.array_equal(d2n_h[ci[lo:hi]], cols[:, :2])
        scale = np.abs(m).max()
        assert np.abs(vm[lo:hi] - m).max() <= 1e-12 * scale
        assert np.abs(vk[lo:hi] - k).max() <= 1e-12 * np.abs(k).max()


def _emulate_async(coords, elems, element, P, caps):
    """The asynchronous rank step for P ranks in this process: every rank's
    enumeration first, then the exchange, then each rank's numeric into
    `caps` (slices with capacities)."""
    ranges, parts = _parts(coords, elems, element, P)
    W = max(hi - lo for lo, hi in ranges)
    for p in parts:
        p.bind(W, P)
    owned = [p.enumerate_async() for p in parts]
    _exchange(parts, owned)
    for p, s in zip(parts, caps):
        p.numeric_async(s)
    return parts


def test_exchange_is_interface_sized():
    """The owner-computes exchange no longer scales with N: config 5 split 8
    ways sends at most ~one node row of first ids per interface."""
    from paper_1409_4618_b200 import api, dist
    from workloads import CONFIGS

    C = CONFIGS[5]
    coords, elems = api.build_mesh(2, C["n"], C["alpha"], C["seed"])
    ranges, parts = _parts(coords, elems, C["element"], 8)
    owned = [p.symbolic() for p in parts]
    sent = _exchange(parts, owned)
    assert max(sent) <= 4 * (4 * (C["n"] + 1) + 8) + 12, sent  # (two ghost node rows on each side)
    assert max(sent) < 1 << 20


@pytest.mark.parametrize("dim,element", KINDS, ids=KIND_IDS)
@pytest.mark.parametrize("P", [2, 3, 8])
def test_partitioned_async_equals_sync(dim, element, P):
    from paper_1409_4618_b200 import api, dist

    n = 24 if dim == 2 else 6
    coords, elems = api.build_mesh(dim, n, 0.2 if dim == 2 else 0.15, 23)
    one = api.Assembler(coords, elems, element).assemble()
    sparts, sslices, offs, total = _emulate(coords, elems, element, P)
    # capacities from the synchronous pass, one spare row / entry (windows are read on the device)
    caps = [dist.CSR(torch.full((p.owned_rows + 2,), -1, dtype=torch.int32, device="cuda"),
                     torch.full((p.owned_nnz + 1,), -1, dtype=torch.int32, device="cuda"),
                     torch.zeros(p.owned_nnz + 1, dtype=torch.float64, device="cuda"),
                     torch.zeros(p.owned_nnz + 1, dtype=torch.float64, device="cuda")) for p in sparts]
    aparts = _emulate_async(coords, elems, element, P, caps)
    for sp, ap, ss, c in zip(sparts, aparts, sslices, caps):
        ap.check()  # flags: no capacity overflow, conforming
        w = ap.window.cpu().numpy()
        assert (w[1], w[3], w[4]) == (sp.owned_rows, sp.owned_nnz, sp.first_row)
        r, z = sp.owned_rows, sp.owned_nnz
        assert torch.equal(c.row_ptr[: r + 1], ss.row_ptr)
        assert torch.equal(c.col_idx[:z], ss.col_idx)
        assert torch.equal(c.vals_M[:z], ss.vals_M) and torch.equal(c.vals_K[:z], ss.vals_K)
    rp, ci, vm, vk = dist.concat_slices(sslices, offs)
    assert np.array_equal(vm, one.vals_M.cpu().numpy()) and np.array_equal(ci, one.col_idx.cpu().numpy())


def test_partitioned_async_capacity_flagged():
    from paper_1409_4618_b200 import api, dist

    coords, elems = api.build_mesh(2, 16, 0.2, 5)
    sparts, _, _, _ = _emulate(coords, elems, NED0, 2)
    p = sparts[0]
    small = dist.CSR(torch.zeros(p.owned_rows + 1, dtype=torch.int32, device="cuda"),
                     torch.zeros(p.owned_nnz - 1, dtype=torch.int32, device="cuda"),
                     torch.zeros(p.owned_nnz - 1, dtype=torch.float64, device="cuda"),
                     torch.zeros(p.owned_nnz - 1, dtype=torch.float64, device="cuda"))
    big = [small, sparts[1].alloc_slice()]
    aparts = _emulate_async(coords, elems, NED0, 2, big)
    with pytest.raises(RuntimeError, match="ECAPACITY|capacity"):
        aparts[0].check()
    aparts[1].check()


@pytest.mark.parametrize("backend", ["nccl", "gloo"])
def test_async_step_world1_equals_single(backend):
    """bench.py's timed multi-GPU step (dist.AsyncStep) in a real process group
    of size 1: the slice equals the 1-GPU CSR, the window its sizes."""
    import os
    import socket

    import torch.distributed as dist

    from paper_1409_4618_b200 import api
    from paper_1409_4618_b200 import dist as pdist

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=0, world_size=1, **kw)
    try:
        coords, elems = api.build_mesh(2, 20, 0.2, 9, device="cuda:0")
        one = api.Assembler(coords, elems, NED0).assemble()
        ranges = pdist.node_ranges(coords.shape[0], 1)
        part = pdist.PartAssembler(coords, elems, NED0, *ranges[0])
        out, _, _ = pdist.assemble_rank(part, ranges, None)
        out.vals_M.zero_()
        out.col_idx.zero_()
        step = pdist.AsyncStep(part, ranges, out)
        for _ in range(2):
            o, win, nnz_all = step()
        assert torch.equal(o.row_ptr, one.row_ptr) and torch.equal(o.col_idx, one.col_idx)
        assert torch.equal(o.vals_M, one.vals_M) and torch.equal(o.vals_K, one.vals_K)
        w = win.cpu().tolist()
        assert w[:5] == [0, one.n_rows, 0, one.nnz, 0] and nnz_all.cpu().tolist() == [one.nnz]
    finally:
        dist.destroy_process_group()


def test_partitioned_async_more_ranks_than_needed():
    """P larger than useful: trailing ranks own empty node ranges (ceil-width
    ranges); their windows are empty and the slices still tile the matrix."""
    from paper_1409_4618_b200 import api, dist

    coords, elems = api.build_mesh(2, 3, 0.1, 2)  # 16 nodes
    one = api.Assembler(coords, elems, NED0).assemble()
    P = 12  # W = 2: ranks 8..11 own nothing
    sparts, sslices, offs, total = _emulate(coords, elems, NED0, P)
    assert total == one.nnz
    caps = [dist.CSR(torch.zeros(p.owned_rows + 1, dtype=torch.int32, device="cuda"),
                     torch.zeros(max(p.owned_nnz, 1), dtype=torch.int32, device="cuda"),
                     torch.zeros(max(p.owned_nnz, 1), dtype=torch.float64, device="cuda"),
                     torch.zeros(max(p.owned_nnz, 1), dtype=torch.float64, device="cuda")) for p in sparts]
    aparts = _emulate_async(coords, elems, NED0, P, caps)
    rows = 0
    for sp, ap, c in zip(sparts, aparts, caps):
        ap.check()
        w = ap.window.cpu().tolist()
        assert w[1] == sp.owned_rows and w[3] == sp.owned_nnz
        rows += w[1]
        if sp.owned_rows:
            assert torch.equal(c.col_idx[: sp.owned_nnz], torch.from_numpy(
                dist.concat_slices(sslices, offs)[1][offs[sparts.index(sp)]:][: sp.owned_nnz]).cuda())
    assert rows == one.n_rows
