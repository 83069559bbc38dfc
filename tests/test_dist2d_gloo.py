"""CPU test of the multi-rank partition logic of efem_dist_* (dist2d.cu) over a
real torch.distributed gloo group of two processes: every rank computes its
layout with efem_dist_layout (host only), the ranks all-gather them, and the
result is checked against an independent numpy statement of the rules
(node ranges from the slabs' smallest vertices; a triangle stays where its
smallest or middle vertex is owned and goes to the owners of those vertices)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _mesh():
    from oracle import oracle as ora  # (input generator only)

    c, e = ora.build_mesh(2, 13, 0.2, 3)
    rng = np.random.default_rng(1)
    e = np.ascontiguousarray(e[rng.permutation(e.shape[0])])  # scattered slabs
    return c, e


def _worker(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1409_4618_b200 import dist as pdist

    c, e = _mesh()
    bounds = pdist.slab_bounds(e.shape[0], world)
    mine = pdist.layout(e, c.shape[0], bounds, rank)
    t = torch.tensor([mine[0], mine[1], mine[2]] + mine[3], dtype=torch.int64)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    if rank == 0:
        out.put([g.tolist() for g in gathered])
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_layout_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    c, e = _mesh()
    N, T = c.shape[0], e.shape[0]
    bounds = [T * r // world for r in range(world + 1)]
    mins = [int(e[bounds[r]:bounds[r + 1]].min()) if bounds[r + 1] > bounds[r] else N for r in range(world)]
    lo = [0]
    for r in range(1, world):
        lo.append(max(lo[-1], min(mins[r], N)))
    lo.append(N)
    owner = np.searchsorted(np.array(lo[1:]), np.arange(N), side="right")
    s = np.sort(e, axis=1)
    op, oq = owner[s[:, 0]], owner[s[:, 1]]
    for r in range(world):
        got = res[r]
        assert got[0] == lo[r] and got[1] == lo[r + 1]
        sl = slice(bounds[r], bounds[r + 1])
        assert got[2] == int(((op[sl] == r) | (oq[sl] == r)).sum())
        for d in range(world):
            want = int(((op[sl] == d) & (d != r)).sum() + ((oq[sl] == d) & (d != r) & (oq[sl] != op[sl])).sum())
            assert got[3 + d] == want
    # every triangle reaches (or stays with) the owners of its smallest and middle vertex
    assert sum(res[r][2] for r in range(world)) + sum(sum(res[r][3:]) for r in range(world)) == \
        int(((op == op) * 1).sum() + (oq != op).sum())
