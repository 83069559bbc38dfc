"""The multi-rank host logic over a real torch.distributed (gloo) group of
2 processes on CPU: node ranges, the two all_gathers and the offsets they
produce, checked against the oracle's global numbering.  The per-node entity
counts each rank contributes (on GPU: efem_part_counts) are taken from the
oracle's dofs2nodes here, so this test needs no GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as ora
from workloads import NED0, RT0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dim, element, q):
    import torch.distributed as dist

    from paper_1409_4618_b200.dist import (_allgather_dev, allgather_counts, allgather_nnz, node_ranges,
                                           offsets_from_counts)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 9 if dim == 2 else 4
        coords, elems = ora.build_mesh(dim, n, 0.15, 3)
        A = ora.assemble(dim, element, coords, elems)
        N = coords.shape[0]
        ranges = node_ranges(N, world)
        lo, hi = ranges[rank]
        mins = A.dofs2nodes[:, 0]
        owned = torch.from_numpy(np.bincount(mins[(mins >= lo) & (mins < hi)] - lo, minlength=hi - lo)
                                 .astype(np.int32))
        global_cnt = allgather_counts(owned, ranges)
        ent_ptr = np.concatenate([[0], np.cumsum(global_cnt.numpy())])
        # global DOF id of node g's first entity == rank of its first entity in the oracle numbering
        first = np.searchsorted(mins, np.arange(N))
        ok1 = bool(np.array_equal(ent_ptr[:N], first)) and int(ent_ptr[N]) == A.n_dofs
        rows = np.nonzero((mins >= lo) & (mins < hi))[0]
        my_nnz = int(A.row_ptr[rows[-1] + 1] - A.row_ptr[rows[0]]) if len(rows) else 0
        nnzs = allgather_nnz(my_nnz, torch.device("cpu"))
        offs, total = offsets_from_counts(nnzs)
        ok2 = total == A.col_idx.shape[0] and (len(rows) == 0 or offs[rank] == A.row_ptr[rows[0]])
        # the asynchronous step's exchange (dist.assemble_rank_async): W-wide
        # buffers gathered in rank order ARE the global counts (+ zero tail)
        W = max(h - l for l, h in ranges)
        pad = torch.zeros(W, dtype=torch.int32)
        pad[: hi - lo] = owned
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        flat = torch.cat(parts).numpy()
        ok3 = bool(np.array_equal(flat[:N], global_cnt.numpy())) and not flat[N:].any()
        nz = _allgather_dev(torch.tensor([my_nnz], dtype=torch.int64))
        ok3 = ok3 and [int(v) for v in nz] == nnzs
        q.put((rank, ok1, ok2 and ok3))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim,element", [(2, NED0), (3, RT0), (3, NED0)], ids=["ne0_2d", "rt0_3d", "ne0_3d"])
def test_two_rank_gloo_offsets(dim, element):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dim, element, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] and r[2] for r in res), res


def test_node_ranges_tile():
    from paper_1409_4618_b200.dist import node_ranges

    for N in (1, 7, 100, 16785409):
        for P in (1, 2, 3, 8):
            rs = node_ranges(N, P)
            assert rs[0][0] == 0 and rs[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            # all ranges W = ceil(N / P) wide but the last (shorter, maybe empty):
            # the gathered W-wide buffers are the global counts without repacking
            W = -(-N // P)
            assert all(h - l == W for l, h in rs[:-1] if h < N) and 0 <= rs[-1][1] - rs[-1][0] <= W
            assert all(l == min(N, r * W) for r, (l, h) in enumerate(rs))
