"""The multi-rank host logic of the owner-computes partition over a real
torch.distributed (gloo) group of 2 processes on CPU: node ranges, the
O(interface) exchange (one total per rank, the ghost nodes' first DOF ids)
and the entry offsets, checked against the oracle's global numbering.  The
per-node entity counts each rank contributes (on GPU: efem_part_counts) are
taken from the oracle's dofs2nodes here, so this test needs no GPU."""
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


def _two_hop(elems, lo, hi):
    """Ascending global ids of the two-hop sub-mesh of the node range [lo, hi)
    (elements touching the nodes of the elements touching the range), as
    efem_partition builds it -- here in numpy, for the host-logic test."""
    touch = ((elems >= lo) & (elems < hi)).any(1)
    nodes1 = np.unique(elems[touch])
    mark = np.zeros(elems.max() + 1, bool)
    mark[nodes1] = True
    touch2 = mark[elems].any(1)
    return np.unique(elems[touch2])


def _worker(rank, world, port, dim, element, q):
    """The owner-computes partition's O(interface) exchange over gloo: each
    rank all-gathers one total, requests the first DOF ids of its ghost
    nodes from their owners (setup: all_gather_object of the request lists;
    step: all_to_all_single of the answers) and must obtain, for every node
    of its sub-mesh, the oracle's global first DOF id."""
    import torch.distributed as dist

    from paper_1409_4618_b200.dist import (_allgather_dev, allgather_nnz, answer_plan_host, exchange_plan_host,
                                           node_ranges, offsets_from_counts)

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
        first_true = np.searchsorted(mins, np.arange(N + 1))  # global first DOF id of every node
        # this rank's owned counts (on GPU: efem_part_counts) from the oracle's numbering
        owned = np.bincount(mins[(mins >= lo) & (mins < hi)] - lo, minlength=hi - lo).astype(np.int64)
        local = np.concatenate([[0], np.cumsum(owned)])
        totals = _allgather_dev(torch.tensor([local[-1]], dtype=torch.int64))
        first = local + int(totals[:rank].sum())  # efem_part_add_offset
        s2g = _two_hop(elems, lo, hi)
        l0, l1, own_idx, ghost_pos, recv_splits, requests = exchange_plan_host(s2g, lo, hi, ranges)
        everyone = [None] * world
        dist.all_gather_object(everyone, [r.tolist() for r in requests])
        send_splits, answer_idx = answer_plan_host([everyone[s][rank] for s in range(world)], lo)
        send = torch.from_numpy(first[answer_idx].astype(np.int32))
        recv = torch.zeros(sum(recv_splits), dtype=torch.int32)
        dist.all_to_all_single(recv, send, recv_splits, send_splits)
        sub_first = np.zeros(s2g.size, np.int64)
        sub_first[l0:l1] = first[own_idx]
        sub_first[ghost_pos] = recv.numpy()
        ok1 = bool(np.array_equal(sub_first, first_true[s2g]))
        # the interface bound: answers are only ghost nodes, a small part of the sub-mesh
        ok1 = ok1 and len(answer_idx) <= s2g.size
        rows = np.nonzero((mins >= lo) & (mins < hi))[0]
        my_nnz = int(A.row_ptr[rows[-1] + 1] - A.row_ptr[rows[0]]) if len(rows) else 0
        nnzs = allgather_nnz(my_nnz, torch.device("cpu"))
        offs, total = offsets_from_counts(nnzs)
        ok2 = total == A.col_idx.shape[0] and (len(rows) == 0 or offs[rank] == A.row_ptr[rows[0]])
        q.put((rank, ok1, ok2))
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
