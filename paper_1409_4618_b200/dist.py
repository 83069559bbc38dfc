"""Row-owned partitioned assembly over several GPUs (SURVEY.md §8(e),
DESIGN.md §9).  Argument marshalling around the efem_part_* C-ABI calls plus
the two torch.distributed collectives of the method:

  1. all_gather of the per-node entity counts of every rank's node range
     (-> global DOF offsets), and
  2. all_gather of every rank's CSR entry count (-> its row-block offset).

No matrix values cross ranks (owner computes): rank r assembles the rows of
the entities whose minimum node lies in its node range from a two-hop
sub-mesh.  Concatenating the ranks' slices in rank order gives the 1-GPU CSR
byte for byte.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .api import ALL, CSR, Assembler, _ptr, _stream


def node_ranges(n_nodes: int, world: int):
    """Contiguous node ranges [lo, hi) per rank, all of width W = ceil(N / P)
    except the last (shorter, possibly empty): the ranks' W-wide count
    buffers, gathered in rank order, are then the global per-node counts
    followed by zeros -- no repacking after the all_gather."""
    w = -(-n_nodes // world) if world > 0 else 0
    cuts = [min(n_nodes, r * w) for r in range(world + 1)]
    cuts[-1] = n_nodes
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def offsets_from_counts(counts):
    """Exclusive prefix of per-rank counts (host ints)."""
    out, run = [], 0
    for c in counts:
        out.append(run)
        run += int(c)
    return out, run


class PartAssembler:
    """One rank's share: sub-mesh plan + globalisation + owned-row numeric."""

    def __init__(self, coords: torch.Tensor, elems: torch.Tensor, element: int, lo: int, hi: int, stream=None):
        L = _lib.load()
        self.lo, self.hi = int(lo), int(hi)
        self.n_global_nodes = int(coords.shape[0])
        dim = int(coords.shape[1])
        self.device = coords.device
        self.first_row = 0
        # a rank with an empty node range (more ranks than ceil-width ranges
        # need) owns nothing: no sub-mesh, no plan, an empty slice
        self.empty = self.hi <= self.lo
        self.scan_ws = torch.empty(256, dtype=torch.uint8, device=self.device)
        if self.empty:
            self.owned_cnt = torch.zeros(1, dtype=torch.int32, device=self.device)
            self.info = (ctypes.c_int64 * 4)()
            self.sub2global = self.e2d_global = None
            return
        full = _lib.efem_mesh(dim, coords.shape[0], elems.shape[0], coords.data_ptr(), elems.data_ptr())
        ws_bytes = ctypes.c_size_t()
        nn, ne = ctypes.c_int64(), ctypes.c_int64()
        with torch.cuda.device(self.device):
            _lib.check("efem_partition", L.efem_partition(ctypes.byref(full), self.lo, self.hi, None,
                                                          ctypes.byref(ws_bytes), None, None, None, None, None,
                                                          _stream(stream)))
            ws = torch.empty(max(ws_bytes.value, 256), dtype=torch.uint8, device=self.device)
            _lib.check("efem_partition", L.efem_partition(ctypes.byref(full), self.lo, self.hi, _ptr(ws),
                                                          ctypes.byref(ws_bytes), ctypes.byref(nn),
                                                          ctypes.byref(ne), None, None, None, _stream(stream)))
            self.sub_coords = torch.empty((nn.value, dim), dtype=torch.float64, device=self.device)
            self.sub_elems = torch.empty((ne.value, dim + 1), dtype=torch.int32, device=self.device)
            self.sub2global = torch.empty(nn.value, dtype=torch.int32, device=self.device)
            _lib.check("efem_partition", L.efem_partition(ctypes.byref(full), self.lo, self.hi, _ptr(ws),
                                                          ctypes.byref(ws_bytes), ctypes.byref(nn),
                                                          ctypes.byref(ne), _ptr(self.sub_coords),
                                                          _ptr(self.sub_elems), _ptr(self.sub2global),
                                                          _stream(stream)))
        del ws
        self.asm = Assembler(self.sub_coords, self.sub_elems, element)
        self.owned_cnt = torch.empty(max(self.hi - self.lo, 1), dtype=torch.int32, device=self.device)
        self.info = (ctypes.c_int64 * 4)()
        self.e2d_global = torch.empty(max(self.sub_elems.shape[0] * self.asm.m, 1), dtype=torch.int32,
                                      device=self.device)
        scan_bytes = ctypes.c_size_t()
        _lib.check("efem_part_scan", L.efem_part_scan(None, max(self.hi - self.lo, 1), None, None,
                                                      ctypes.byref(scan_bytes), None))
        self.scan_ws = torch.empty(max(scan_bytes.value, 256), dtype=torch.uint8, device=self.device)
        self.first_row = 0

    def _empty_slice_rows(self, out: CSR):
        out.row_ptr[:1].zero_()
        return out

    @property
    def owned_rows(self):
        return int(self.info[1])

    @property
    def owned_nnz(self):
        return int(self.info[3])

    def symbolic(self, stream=None):
        """Local enumeration; returns this rank's per-node entity counts."""
        if self.empty:
            return self.owned_cnt[:0]
        L = _lib.load()
        self.asm.symbolic(stream=stream)
        with torch.cuda.device(self.device):
            _lib.check("efem_part_counts", L.efem_part_counts(self.asm._plan, _ptr(self.sub2global), self.lo,
                                                              self.hi, _ptr(self.owned_cnt), self.info,
                                                              _stream(stream)))
        return self.owned_cnt[: self.hi - self.lo]

    def alloc_slice(self) -> CSR:
        dev = self.device
        return CSR(torch.empty(self.owned_rows + 1, dtype=torch.int32, device=dev),
                   torch.empty(self.owned_nnz, dtype=torch.int32, device=dev),
                   torch.empty(self.owned_nnz, dtype=torch.float64, device=dev),
                   torch.empty(self.owned_nnz, dtype=torch.float64, device=dev))

    def numeric(self, out: CSR, forms: int = ALL, stream=None):
        if self.empty:
            return self._empty_slice_rows(out)
        L = _lib.load()
        c = _lib.efem_csr(self.owned_rows, self.owned_nnz, out.row_ptr.data_ptr(), out.col_idx.data_ptr(),
                          out.vals_M.data_ptr(), out.vals_K.data_ptr())
        with torch.cuda.device(self.device):
            _lib.check("efem_part_numeric", L.efem_part_numeric(self.asm._plan, forms, self.info, self.first_row,
                                                                _ptr(self.e2d_global), ctypes.byref(c),
                                                                _stream(stream)))
        return out

    def check(self, stream=None):
        if not self.empty:
            self.asm.check(stream=stream)

    # ---- asynchronous step (no host round trip before check) ---------------
    def bind(self, width: int, world: int, stream=None):
        """Binds the sub-mesh plan to the node range (efem_part_bind, once) and
        allocates the W-wide send buffer and the P*W gathered counts."""
        L = _lib.load()
        if not self.empty:
            with torch.cuda.device(self.device):
                _lib.check("efem_part_bind", L.efem_part_bind(self.asm._plan, _ptr(self.sub2global), self.lo,
                                                              self.hi, _stream(stream)))
        self.width = int(width)
        self.owned_pad = torch.zeros(max(self.width, 1), dtype=torch.int32, device=self.device)
        self.window = torch.zeros(5, dtype=torch.int64, device=self.device)
        self.bound = True

    def enumerate_async(self, stream=None):
        if self.empty:
            return self.owned_pad  # zeros
        L = _lib.load()
        with torch.cuda.device(self.device):
            _lib.check("efem_part_enumerate_async",
                       L.efem_part_enumerate_async(self.asm._plan, _ptr(self.owned_pad), _stream(stream)))
        return self.owned_pad

    def numeric_async(self, out: CSR, forms: int = ALL, stream=None):
        """out: a slice with capacities (e.g. from alloc_slice after one
        synchronous step); the window's sizes are read on the device."""
        if self.empty:
            self.window.zero_()
            return self._empty_slice_rows(out)
        L = _lib.load()
        c = _lib.efem_csr(out.row_ptr.numel() - 1, out.col_idx.numel(), out.row_ptr.data_ptr(),
                          out.col_idx.data_ptr(), out.vals_M.data_ptr(), out.vals_K.data_ptr())
        with torch.cuda.device(self.device):
            _lib.check("efem_part_numeric_async", L.efem_part_numeric_async(self.asm._plan, forms,
                                                                            _ptr(self.e2d_global), ctypes.byref(c),
                                                                            _stream(stream)))
            _lib.check("efem_part_window", L.efem_part_window(self.asm._plan, _ptr(self.window), _stream(stream)))
        return out


# ---- O(interface) exchange (efem_part_add_offset / efem_index_* /
# efem_part_globalize_sub): the ranks all-gather one total each and answer
# only the first DOF ids of the ghost nodes other ranks' sub-meshes hold.
def exchange_plan_host(s2g, lo: int, hi: int, ranges):
    """Host arrays: (l0, l1, owned_idx, ghost_pos, recv_splits, requests) of
    a rank owning [lo, hi) whose sub-mesh holds the ascending global node ids
    s2g: the owned sub-mesh nodes [l0, l1) and their index into the owned
    range, the ghost positions grouped by owner rank, how many first ids it
    receives from each rank, and the global ids it asks each rank for."""
    s2g = np.asarray(s2g, np.int64)
    P = len(ranges)
    owned = (s2g >= lo) & (s2g < hi)
    idx = np.nonzero(owned)[0]
    l0 = int(idx[0]) if idx.size else 0
    l1 = l0 + int(idx.size)
    his = np.array([h for _, h in ranges], np.int64)
    ghost = np.nonzero(~owned)[0]
    own_of = np.searchsorted(his, s2g[ghost], side="right")
    order = np.argsort(own_of, kind="stable")
    ghost, own_of = ghost[order], own_of[order]
    recv_splits = [int((own_of == r).sum()) for r in range(P)]
    requests = [s2g[ghost[own_of == r]] for r in range(P)]
    return l0, l1, (s2g[l0:l1] - lo).astype(np.int32), ghost.astype(np.int32), recv_splits, requests


def answer_plan_host(requests_to_me, lo: int):
    """(send_splits, answer_idx): what this rank answers each rank, as indices
    into its owned range."""
    send_splits = [len(q) for q in requests_to_me]
    flat = np.concatenate([np.asarray(q, np.int64) for q in requests_to_me]) if requests_to_me else np.zeros(0)
    return send_splits, (flat - lo).astype(np.int32)


def _exchange_plan(part: "PartAssembler", ranges):
    """Host, once per partition: the owned sub-mesh nodes [l0, l1) and their
    index into the owned range, the ghost sub-mesh nodes grouped by owner
    rank (their positions and global ids: this rank's requests)."""
    P = len(ranges)
    part.P = P
    if part.empty:
        part.l0 = part.l1 = 0
        part.requests = [np.zeros(0, np.int64) for _ in range(P)]
        part.recv_splits = [0] * P
        part.recv_buf = torch.zeros(1, dtype=torch.int32, device=part.device)
        return
    s2g = part.sub2global.cpu().numpy().astype(np.int64)
    dev = part.device
    part.l0, part.l1, own_idx, ghost, part.recv_splits, part.requests = exchange_plan_host(s2g, part.lo, part.hi,
                                                                                         ranges)
    part.owned_idx = torch.from_numpy(own_idx).to(dev)
    part.ghost_pos = torch.from_numpy(ghost).to(dev)
    part.sub_first = torch.zeros(max(s2g.size, 1), dtype=torch.int32, device=dev)
    part.recv_buf = torch.zeros(max(ghost.size, 1), dtype=torch.int32, device=dev)


def _answer_plan(part: "PartAssembler", requests_to_me):
    """requests_to_me[s]: the global ids rank s asks this rank for."""
    part.send_splits, idx = answer_plan_host(requests_to_me, part.lo)
    part.answer_idx = torch.from_numpy(idx).to(part.device)
    part.send_buf = torch.zeros(max(idx.size, 1), dtype=torch.int32, device=part.device)
    part.first_buf = torch.zeros(max(part.hi - part.lo, 0) + 1, dtype=torch.int32, device=part.device)


def setup_exchange(part: "PartAssembler", ranges, group=None):
    """The request lists to their owners (torch.distributed all_gather_object,
    setup only)."""
    import torch.distributed as dist

    _exchange_plan(part, ranges)
    everyone = [None] * len(ranges)
    dist.all_gather_object(everyone, [q.tolist() for q in part.requests], group=group)
    me = dist.get_rank(group)
    _answer_plan(part, [everyone[s][me] for s in range(len(ranges))])


def _part_local_prefix(part: "PartAssembler", owned: torch.Tensor, stream=None):
    """Exclusive scan of the owned counts into first_buf; returns the device
    view of this rank's total (first_buf[width])."""
    L = _lib.load()
    w = part.hi - part.lo
    if w > 0:
        b = ctypes.c_size_t(part.scan_ws.numel())
        _lib.check("efem_part_scan", L.efem_part_scan(_ptr(owned), w, _ptr(part.first_buf), _ptr(part.scan_ws),
                                                      ctypes.byref(b), _stream(stream)))
    else:
        part.first_buf.zero_()
    return part.first_buf[w:w + 1]


def _part_first_ids(part: "PartAssembler", totals: torch.Tensor, rank: int, stream=None):
    """first_buf += the totals of the ranks before; the answers to send."""
    L = _lib.load()
    _lib.check("efem_part_add_offset", L.efem_part_add_offset(_ptr(part.first_buf), part.first_buf.numel(),
                                                              _ptr(totals), rank, _stream(stream)))
    n = part.answer_idx.numel()
    _lib.check("efem_index_gather", L.efem_index_gather(_ptr(part.send_buf), _ptr(part.first_buf),
                                                        _ptr(part.answer_idx), n, 0, _stream(stream)))
    return part.send_buf[:n]


def _part_place(part: "PartAssembler", recv: torch.Tensor, stream=None):
    """sub_first: owned nodes from first_buf, ghosts from the answers; then
    elems2dofs in global ids and the window's global first row."""
    if part.empty:
        return
    L = _lib.load()
    n_own = part.l1 - part.l0
    sub_view = part.sub_first[part.l0:]
    _lib.check("efem_index_gather", L.efem_index_gather(_ptr(sub_view), _ptr(part.first_buf), _ptr(part.owned_idx),
                                                        n_own, 0, _stream(stream)))
    _lib.check("efem_index_scatter", L.efem_index_scatter(_ptr(part.sub_first), _ptr(part.ghost_pos), _ptr(recv),
                                                          part.ghost_pos.numel(), _stream(stream)))
    _lib.check("efem_part_globalize_sub", L.efem_part_globalize_sub(part.asm._plan, _ptr(part.sub_first), part.l0,
                                                                    part.l1, _ptr(part.e2d_global), _stream(stream)))


def exchange_bytes(part: "PartAssembler") -> int:
    """Bytes this rank sends per step: its total (all-gather), its answers,
    its entry count (all-gather)."""
    return 4 + 4 * int(part.answer_idx.numel()) + 8


def _comm_device(t: torch.Tensor, group=None):
    """NCCL gathers device tensors directly; gloo (CPU tests, or several
    ranks sharing one GPU) goes through host copies."""
    import torch.distributed as dist

    return t.device if dist.get_backend(group) == "nccl" else torch.device("cpu")


def allgather_nnz(nnz: int, device, group=None):
    """Collective 2: every rank's CSR entry count."""
    import torch.distributed as dist

    t = torch.tensor([nnz], dtype=torch.int64, device=device)
    dev = _comm_device(t, group)
    t = t.to(dev)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return [int(p.item()) for p in parts]


def assemble_rank(part: PartAssembler, ranges, out: CSR | None = None, group=None, stream=None):
    """One rank's full step: local symbolic, the O(interface) exchange (the
    ranks' totals, the ghost nodes' first ids), numeric.  Returns (slice
    CSR, first global row, first global CSR entry)."""
    import torch.distributed as dist

    if not hasattr(part, "answer_idx"):
        setup_exchange(part, ranges, group=group)
    rank = dist.get_rank(group)
    owned = part.symbolic(stream=stream)
    total = _part_local_prefix(part, owned, stream=stream)
    totals = _allgather_dev(total.contiguous(), group).to(part.device)
    send = _part_first_ids(part, totals, rank, stream=stream)
    recv = _alltoall_dev(send, part.send_splits, part.recv_buf, part.recv_splits, group)
    _part_place(part, recv, stream=stream)
    part.first_row = int(part.sub_first[part.l0].item()) if part.l1 > part.l0 else 0
    nnzs = allgather_nnz(part.owned_nnz, owned.device, group=group)
    offs, _ = offsets_from_counts(nnzs)
    if out is None or out.nnz != part.owned_nnz or out.n_rows != part.owned_rows:
        out = part.alloc_slice()
    part.numeric(out, stream=stream)
    part.check(stream=stream)
    return out, part.first_row, offs[rank]


def _alltoall_dev(send: torch.Tensor, send_splits, recv: torch.Tensor, recv_splits, group=None):
    """all_to_all of the ghost answers (NCCL on the device, gloo via host)."""
    import torch.distributed as dist

    n_recv = sum(recv_splits)
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(recv[:n_recv], send[:sum(send_splits)], recv_splits, send_splits, group=group)
        return recv[:n_recv]
    r = torch.zeros(n_recv, dtype=recv.dtype)
    dist.all_to_all_single(r, send[:sum(send_splits)].cpu(), recv_splits, send_splits, group=group)
    recv[:n_recv].copy_(r.to(recv.device))
    return recv[:n_recv]


class AsyncStep:
    """dist.assemble_rank_async with its call arguments marshalled once: per
    step four library calls, two collectives and the check, no per-step
    allocation (the host enqueue stays well under the device time)."""

    def __init__(self, part: PartAssembler, ranges, out: CSR, group=None, stream=None, forms: int = ALL):
        import torch.distributed as dist

        self.part, self.out, self.group = part, out, group
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        if not getattr(part, "bound", False):
            part.bind(max(hi - lo for lo, hi in ranges), self.world, stream=stream)
        if not hasattr(part, "answer_idx"):
            setup_exchange(part, ranges, group=group)
        self.rank = dist.get_rank(group)
        self.L = _lib.load()
        self.stream = stream
        self.s = _stream(stream)
        # the collectives are issued on torch's current stream: make it the
        # stream the library calls are enqueued on, so they stay ordered
        self.tstream = stream if stream is not None else torch.cuda.current_stream(part.device)
        self.empty = part.empty
        self.plan = None if part.empty else part.asm._plan
        self.p_owned = _ptr(part.owned_pad)
        self.p_sws = _ptr(part.scan_ws)
        self.p_s2g = _ptr(part.sub2global)
        self.p_e2dg = _ptr(part.e2d_global)
        self.p_win = _ptr(part.window)
        self.sws_bytes = ctypes.c_size_t(part.scan_ws.numel())
        self.n_global = part.n_global_nodes
        self.forms = forms
        self.csr = _lib.efem_csr(out.row_ptr.numel() - 1, out.col_idx.numel(), out.row_ptr.data_ptr(),
                                 out.col_idx.data_ptr(), out.vals_M.data_ptr(), out.vals_K.data_ptr())
        self.csr_ref = ctypes.byref(self.csr)
        self.nnz_mine = part.window[3:4]
        self.nnz_all = torch.empty(self.world, dtype=torch.int64, device=part.device)

    def __call__(self, check=True):
        with torch.cuda.stream(self.tstream):
            return self._call(check)

    def _call(self, check):
        import torch.distributed as dist

        L, ck = self.L, _lib.check
        if not self.empty:
            ck("efem_part_enumerate_async", L.efem_part_enumerate_async(self.plan, self.p_owned, self.s))
        part = self.part
        # O(interface): one total per rank, the ghost nodes' first ids
        total = _part_local_prefix(part, part.owned_pad, stream=self.stream)
        totals = _allgather_dev(total.contiguous(), self.group).to(part.device)
        send = _part_first_ids(part, totals, self.rank, stream=self.stream)
        recv = _alltoall_dev(send, part.send_splits, part.recv_buf, part.recv_splits, self.group)
        if not self.empty:
            _part_place(part, recv, stream=self.stream)
            ck("efem_part_numeric_async", L.efem_part_numeric_async(self.plan, self.forms, self.p_e2dg,
                                                                    self.csr_ref, self.s))
            ck("efem_part_window", L.efem_part_window(self.plan, self.p_win, self.s))
        if self.nccl:
            dist.all_gather_into_tensor(self.nnz_all, self.nnz_mine, group=self.group)
        else:
            self.nnz_all = _allgather_dev(self.nnz_mine.contiguous(), self.group)
        if check == "async":  # only the device half (flag read-back); finish with check()
            self.check_async()
        elif check:
            self.check()
        return self.out, self.part.window, self.nnz_all

    def check_async(self):
        if not self.empty:
            _lib.check("efem_plan_check_async", self.L.efem_plan_check_async(self.plan, self.s))

    def check(self):
        if not self.empty:
            _lib.check("efem_plan_check", self.L.efem_plan_check(self.plan, self.s))


def assemble_rank_async(part: PartAssembler, ranges, out: CSR, group=None, stream=None, check=True):
    """One rank's step with every size on the device (dist.AsyncStep once):
    enumeration + owned counts, the O(interface) exchange, globalisation,
    owned-row numeric, the entry-count all_gather; one host round trip (the
    flags check) at the end.  Returns (out, window, every rank's entries)."""
    return AsyncStep(part, ranges, out, group=group, stream=stream)(check=check)


def _allgather_dev(t: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * t.numel(), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out
    parts = [torch.empty_like(t, device="cpu") for _ in range(world)]
    dist.all_gather(parts, t.cpu(), group=group)
    return torch.cat(parts)


def concat_slices(slices, entry_offsets):
    """Host-side concatenation of rank slices (row_ptr shifted by the entry
    offsets) -> numpy CSR arrays, for checking against the 1-GPU result."""
    rp = [np.zeros(1, np.int64)]
    ci, vm, vk = [], [], []
    for s, off in zip(slices, entry_offsets):
        r = s.row_ptr.cpu().numpy().astype(np.int64)
        rp.append(r[1:] + off)
        ci.append(s.col_idx.cpu().numpy())
        vm.append(s.vals_M.cpu().numpy())
        vk.append(s.vals_K.cpu().numpy())
    return (np.concatenate(rp), np.concatenate(ci), np.concatenate(vm), np.concatenate(vk))


# --------------------------------------------------------------------------- element slabs over NCCL (2D)
# efem_dist_* (dist2d.cu): the north_star multi-GPU path -- contiguous element
# slabs, row-owned CSR slices, the off-rank contributions (ghost triangles'
# local matrices) and column ids exchanged by NCCL inside libefem.  This
# module only moves the 128-byte NCCL unique id between processes (through
# torch.distributed) and marshals arguments.
def slab_bounds(n_elems: int, world: int):
    """Contiguous element slabs [b_r, b_{r+1}) of (nearly) equal size."""
    return [n_elems * r // world for r in range(world + 1)]


def _empty_csr(device):
    z32 = torch.zeros(1, dtype=torch.int32, device=device)
    z64 = torch.zeros(1, dtype=torch.float64, device=device)
    return CSR(z32, z32.clone(), z64, z64.clone())


def _slice_struct(c: CSR, n_rows: int, nnz: int):
    return _lib.efem_csr(n_rows, nnz, c.row_ptr.data_ptr(), c.col_idx.data_ptr(), c.vals_M.data_ptr(),
                         c.vals_K.data_ptr())


def _alloc_slice(rows: int, nnz: int, device):
    return CSR(torch.empty(rows + 1, dtype=torch.int32, device=device),
               torch.empty(max(nnz, 1), dtype=torch.int32, device=device),
               torch.empty(max(nnz, 1), dtype=torch.float64, device=device),
               torch.empty(max(nnz, 1), dtype=torch.float64, device=device))


def layout(elems_host, n_nodes: int, bounds, rank: int):
    """efem_dist_layout: (lo, hi, kept, sent-to-rank list) of one rank (host only)."""
    import numpy as _np

    e = _np.ascontiguousarray(elems_host, dtype=_np.int32)
    b = (ctypes.c_int64 * len(bounds))(*bounds)
    P = len(bounds) - 1
    out = (ctypes.c_int64 * (3 + P))()
    _lib.check("efem_dist_layout", _lib.load().efem_dist_layout(e.ctypes.data_as(ctypes.c_void_p), n_nodes,
                                                                  e.shape[0], b, P, rank, out))
    return out[0], out[1], out[2], list(out[3:3 + P])


class DistGroup:
    """All ranks of one distributed 2D assembly inside this process on one
    device (efem_dist_group_create): the exchanges are device copies.  For
    testing the multi-rank path where one GPU exists."""

    def __init__(self, coords: torch.Tensor, elems: torch.Tensor, element: int, bounds, stream=None):
        L = _lib.load()
        self.device = coords.device
        self.P = len(bounds) - 1
        self._mesh = _lib.efem_mesh(2, coords.shape[0], elems.shape[0], coords.data_ptr(), elems.data_ptr())
        self._keep = (coords, elems)
        self.plans = (ctypes.c_void_p * self.P)()
        b = (ctypes.c_int64 * len(bounds))(*bounds)
        with torch.cuda.device(self.device):
            _lib.check("efem_dist_group_create", L.efem_dist_group_create(self.plans, self.P, ctypes.byref(self._mesh),
                                                                          element, b, _stream(stream)))
        self.slices = None

    def close(self):
        if self.plans is not None:
            for p in self.plans:
                _lib.load().efem_dist_plan_destroy(p)
            self.plans = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self, r):
        out = (ctypes.c_int64 * 8)()
        _lib.check("efem_dist_info", _lib.load().efem_dist_info(self.plans[r], out))
        return list(out)

    def _step(self, slices, caps, forms, stream):
        arr = (_lib.efem_csr * self.P)(*[_slice_struct(s, r, z) for s, (r, z) in zip(slices, caps)])
        with torch.cuda.device(self.device):
            _lib.check("efem_dist_assemble_group", _lib.load().efem_dist_assemble_group(self.plans, self.P, forms, arr,
                                                                                        _stream(stream)))

    def windows(self, stream=None, check=True):
        out = []
        for r in range(self.P):
            w = (ctypes.c_int64 * 4)()
            st = _lib.load().efem_dist_check(self.plans[r], w, _stream(stream))
            if check:
                _lib.check("efem_dist_check", st)
            out.append((list(w), st))
        return out

    def assemble(self, forms: int = ALL, stream=None):
        """One step of every rank; slices sized by a first size-query step."""
        if self.slices is None:
            empty = [_empty_csr(self.device) for _ in range(self.P)]
            self._step(empty, [(0, 0)] * self.P, forms, stream)
            wins = self.windows(stream, check=False)
            self.slices = [_alloc_slice(w[1], w[3], self.device) for w, _ in wins]
        caps = [(s.row_ptr.numel() - 1, s.col_idx.numel()) for s in self.slices]
        self._step(self.slices, caps, forms, stream)
        self.last = [w for w, _ in self.windows(stream)]
        return self.slices

    def concat(self):
        """The global CSR (host numpy) from the ranks' slices, rank order."""
        rps, cis, vms, vks = [], [], [], []
        for s, w in zip(self.slices, self.last):
            rows, nnz, zoff = w[1], w[3], w[2]
            rps.append(s.row_ptr[:rows].cpu().numpy().astype(np.int64) + zoff)
            cis.append(s.col_idx[:nnz].cpu().numpy())
            vms.append(s.vals_M[:nnz].cpu().numpy())
            vks.append(s.vals_K[:nnz].cpu().numpy())
        total = self.last[-1][2] + self.last[-1][3]
        rp = np.concatenate(rps + [np.array([total], np.int64)]).astype(np.int32)
        return rp, np.concatenate(cis), np.concatenate(vms), np.concatenate(vks)


def nccl_comm(rank: int, world: int, group=None):
    """An efem_comm over the processes of a torch.distributed group: rank 0
    draws the NCCL unique id, torch.distributed broadcasts its 128 bytes."""
    import torch.distributed as tdist

    L = _lib.load()
    uid = (ctypes.c_ubyte * 128)()
    if rank == 0:
        _lib.check("efem_comm_unique_id", L.efem_comm_unique_id(uid))
    dev = "cuda" if tdist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
    tdist.broadcast(t, src=0, group=group)
    raw = bytes(t.cpu().tolist())
    uid = (ctypes.c_ubyte * 128).from_buffer_copy(raw)
    comm = ctypes.c_void_p()
    _lib.check("efem_comm_init", L.efem_comm_init(ctypes.byref(comm), uid, world, rank))
    return comm


class DistAssembler:
    """This process's rank of a distributed 2D assembly over NCCL
    (efem_dist_plan_create / efem_dist_assemble)."""

    def __init__(self, coords: torch.Tensor, elems: torch.Tensor, element: int, elem_lo: int, elem_hi: int, comm,
                 stream=None):
        L = _lib.load()
        self.device = coords.device
        self.comm = comm
        self._mesh = _lib.efem_mesh(2, coords.shape[0], elems.shape[0], coords.data_ptr(), elems.data_ptr())
        self._keep = (coords, elems)
        self.plan = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check("efem_dist_plan_create", L.efem_dist_plan_create(ctypes.byref(self.plan), ctypes.byref(self._mesh),
                                                                        element, elem_lo, elem_hi, comm,
                                                                        _stream(stream)))
        self.slice = None
        self.window = None

    def info(self):
        out = (ctypes.c_int64 * 8)()
        _lib.check("efem_dist_info", _lib.load().efem_dist_info(self.plan, out))
        return list(out)

    def step(self, forms: int = ALL, stream=None):
        """Enqueue one step into the current slice (asynchronous)."""
        s = self.slice
        c = _slice_struct(s, s.row_ptr.numel() - 1, s.col_idx.numel())
        with torch.cuda.device(self.device):
            _lib.check("efem_dist_assemble", _lib.load().efem_dist_assemble(self.plan, forms, ctypes.byref(c),
                                                                            _stream(stream)))

    def check(self, stream=None):
        w = (ctypes.c_int64 * 4)()
        with torch.cuda.device(self.device):
            _lib.check("efem_dist_check", _lib.load().efem_dist_check(self.plan, w, _stream(stream)))
        self.window = list(w)
        return self.window

    def assemble(self, forms: int = ALL, stream=None):
        """One step with a synchronising check; the first call sizes the slice."""
        if self.slice is None:
            self.slice = _empty_csr(self.device)
            c = _slice_struct(self.slice, 0, 0)
            with torch.cuda.device(self.device):
                _lib.check("efem_dist_assemble", _lib.load().efem_dist_assemble(self.plan, forms, ctypes.byref(c),
                                                                                _stream(stream)))
            w = (ctypes.c_int64 * 4)()
            _lib.load().efem_dist_check(self.plan, w, _stream(stream))
            self.slice = _alloc_slice(w[1], w[3], self.device)
        self.step(forms, stream)
        self.check(stream)
        return self.slice

    def close(self):
        if self.plan:
            _lib.load().efem_dist_plan_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
