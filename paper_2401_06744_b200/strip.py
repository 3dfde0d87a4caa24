"""Single-frame strip decomposition over several GPUs (BASELINE config 4b).

The finest level is cut into horizontal strips, one per rank (one process per GPU); all coarser
levels are replicated.  A rank owns the pixel rows ``[own_lo, own_hi)`` (block-row starts), solves
the block rows that cover them (boundary block rows redundantly on both sides, so the ordered
combine needs no foreign tiles) and keeps the one-block-deep halo ``[ext_lo, ext_hi)`` of the
iterate valid.  Per ORAS sweep the ranks exchange

* the strip's partial ``||r||^2`` (all-reduce of P doubles: target = eta * rs and the convergence
  test use the GLOBAL norm, solvers.py:416-422),
* the halo rows of the updated iterate (send/recv between neighbouring strips),

and per V-cycle the restricted residual of the finest level (all-gather of the rows each rank
restricted; the coarse levels are then solved identically on every rank).  Prolongation needs no
exchange: the coarse correction is replicated, every rank prolongates onto its strip plus halo.

The data movement is behind a small ``Transport``: ``TorchDistTransport`` (torch.distributed:
NCCL over NVLink on GPUs, gloo in the CPU tests) and ``LocalTransport`` (virtual ranks as threads
of one process on one device, used to check the decomposition against the single-GPU solve).
The library side is ``b200p_plan_set_strip`` + the exchange callback (include/b200paint.h).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _dev, _lib
from .multigrid import MultigridConfig, Plan

XCHG_SUM_RS, XCHG_MAX_FLAGS, XCHG_HALO_U, XCHG_GATHER_RC, XCHG_HALO_RC = 1, 2, 3, 4, 5
_EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p)


class _DeviceArray:
    """Raw device pointer -> torch tensor view (no copy) through __cuda_array_interface__."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}


def device_view(ptr, shape, dtype):
    typestr = {torch.float64: "<f8", torch.int32: "<i4"}[dtype]
    return torch.as_tensor(_DeviceArray(ptr, shape, typestr), device=_dev.device())


def halo_plan(ranges, rank):
    """Row intervals to move for a halo exchange: [(peer, y0, y1)] to receive into `rank`'s halo and
    to send from `rank`'s strip.  ranges[q] = (own_lo, own_hi, ext_lo, ext_hi, iy_lo, iy_hi)."""
    def cut(ext, own_me, own_q):
        out = []
        for lo, hi in ((ext[0], own_me[0]), (own_me[1], ext[1])):  # halo above, halo below
            a, b = max(lo, own_q[0]), min(hi, own_q[1])
            if a < b:
                out.append((a, b))
        return out
    me = ranges[rank]
    recv, send = [], []
    for q, r in enumerate(ranges):
        if q == rank:
            continue
        recv += [(q, a, b) for a, b in cut((me[2], me[3]), (me[0], me[1]), (r[0], r[1]))]
        send += [(q, a, b) for a, b in cut((r[2], r[3]), (r[0], r[1]), (me[0], me[1]))]
    return recv, send


def native_halo_plan(ranges_by_level, level, rank):
    """The library's own halo plan (b200p_strip_halo_plan, what the NCCL exchange walks): (recv, send) lists of
    (peer, y0, y1), for comparison with `halo_plan`."""
    levels, nranks = len(ranges_by_level), len(ranges_by_level[0])
    flat = [v for q in range(nranks) for l in range(levels) for v in ranges_by_level[l][q]]
    every = (C.c_int * len(flat))(*flat)
    cap = 4 * nranks
    r, s = (C.c_int * (3 * cap))(), (C.c_int * (3 * cap))()
    n = _lib.lib().b200p_strip_halo_plan(C.cast(every, C.c_void_p), levels, level, rank, nranks,
                                         C.cast(r, C.c_void_p), C.cast(s, C.c_void_p), cap)
    if n < 0:
        _lib.check(n)
    unpack = lambda a: [(a[3 * i], a[3 * i + 1], a[3 * i + 2]) for i in range(n) if a[3 * i] >= 0]
    return unpack(r), unpack(s)


def strip_ranges(height, block_size, overlap, nranks, levels=1):
    """ranges[l][q] = (own_lo, own_hi, ext_lo, ext_hi, iy_lo, iy_hi) of rank q on striped level l
    (host-only geometry).  With levels == 1 the list of level 0 is returned directly."""
    per_rank = []
    for q in range(nranks):
        r = (C.c_int * (6 * levels))()
        _lib.check(_lib.lib().b200p_strip_ranges(int(height), int(block_size), int(overlap), int(levels), q,
                                                 nranks, C.cast(r, C.c_void_p)))
        per_rank.append([tuple(r[6 * l:6 * l + 6]) for l in range(levels)])
    by_level = [[per_rank[q][l] for q in range(nranks)] for l in range(levels)]
    return by_level[0] if levels == 1 else by_level


def coarse_rows(ranges, h1):
    """Coarse (level-1) rows every rank restricted: own rows halved; the last strip runs to the end."""
    out = []
    for i, r in enumerate(ranges):
        out.append((r[0] // 2, h1 if i == len(ranges) - 1 else r[1] // 2))
    return out


class Transport:
    rank = 0
    nranks = 1

    def zeros_f64(self, shape):
        """Device buffer for the solution (a transport may need a particular allocation)."""
        return torch.zeros(tuple(shape), dtype=torch.float64, device=_dev.device())

    def sum_(self, t): raise NotImplementedError
    def max_(self, t): raise NotImplementedError
    def halo(self, u, ranges): raise NotImplementedError
    def gather_rows(self, field, rows): raise NotImplementedError


class TorchDistTransport(Transport):
    """torch.distributed (NCCL on CUDA tensors, gloo on CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)

    def sum_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def max_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)

    def halo(self, u, ranges):
        recv, send = halo_plan(ranges, self.rank)
        ops, landing = [], []
        for q, a, b in send:
            ops.append(self.dist.P2POp(self.dist.isend, u[:, a:b].contiguous(), q, self.group))
        for q, a, b in recv:
            buf = torch.empty_like(u[:, a:b])
            landing.append((buf, a, b))
            ops.append(self.dist.P2POp(self.dist.irecv, buf, q, self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        for buf, a, b in landing:
            u[:, a:b].copy_(buf)

    def gather_rows(self, field, rows):
        for q, (a, b) in enumerate(rows):
            chunk = field[:, a:b].contiguous()
            self.dist.broadcast(chunk, src=q, group=self.group)
            if q != self.rank:
                field[:, a:b].copy_(chunk)


class NcclNative(Transport):
    """The library's own exchange (b200p_plan_set_strip_nccl): an NCCL communicator created through the C-ABI
    helpers, the unique id broadcast over `group` (any torch.distributed backend; none needed for one rank).
    There are no per-exchange methods: halo send / recv, the norm all-reduces and the residual all-gather are
    issued by libb200paint on the solve's stream, so a strip solve runs as captured CUDA graphs."""

    def __init__(self, group=None):
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.nranks = 0, 1
        uid = (C.c_ubyte * 128)()
        if self.rank == 0:
            _lib.check(_lib.lib().b200p_nccl_unique_id(C.cast(uid, C.c_void_p)))
        if self.nranks > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
        comm = C.c_void_p()
        _lib.check(_lib.lib().b200p_nccl_comm_create(C.cast(uid, C.c_void_p), self.rank, self.nranks, C.byref(comm)))
        self.comm = comm

    def close(self):
        if getattr(self, "comm", None):
            _lib.lib().b200p_nccl_comm_destroy(self.comm)
            self.comm = None


class IpcTransport(Transport):
    """Peer-memory transport for one process per GPU (or several processes on one GPU): every rank
    maps its peers' buffers with CUDA IPC and PULLS the halo rows / gathered rows it needs with
    device-to-device copies over NVLink; no NCCL.  Control (handle exchange, barriers, the P-element
    reductions) goes through a host process group (gloo).  Buffers must be cudaMalloc bases:
    `zeros_f64` for the solution, the plan-owned level fields otherwise."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
        self._peers = {}     # local base pointer -> [peer tensor views]
        self._owned = []

    def zeros_f64(self, shape):
        n = int(np.prod(shape)) * 8
        p = C.c_void_p()
        _lib.check(_lib.lib().b200p_malloc(C.byref(p), n))
        _lib.check(_lib.lib().b200p_memset(p, 0, n))
        self._owned.append(p)
        return device_view(p.value, shape, torch.float64)

    def _peer_views(self, t):
        key = t.data_ptr()
        if key not in self._peers:
            h = (C.c_ubyte * 64)()
            _lib.check(_lib.lib().b200p_ipc_export(C.c_void_p(key), C.cast(h, C.c_void_p)))
            handles = [None] * self.nranks
            self.dist.all_gather_object(handles, bytes(h), group=self.group)
            views = []
            for q, hb in enumerate(handles):
                if q == self.rank:
                    views.append(t)
                    continue
                buf = (C.c_ubyte * 64).from_buffer_copy(hb)
                pp = C.c_void_p()
                _lib.check(_lib.lib().b200p_ipc_open(C.cast(buf, C.c_void_p), C.byref(pp)))
                views.append(device_view(pp.value, tuple(t.shape), t.dtype))
            self._peers[key] = views
        return self._peers[key]

    def _fence(self):
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)

    def _reduce(self, t, op):
        h = t.detach().cpu()
        self.dist.all_reduce(h, op=op, group=self.group)
        t.copy_(h)

    def sum_(self, t): self._reduce(t, self.dist.ReduceOp.SUM)
    def max_(self, t): self._reduce(t, self.dist.ReduceOp.MAX)

    def halo(self, u, ranges):
        peers = self._peer_views(u)
        self._fence()                       # everybody's strip is written
        for q, a, b in halo_plan(ranges, self.rank)[0]:
            u[:, a:b].copy_(peers[q][:, a:b])
        self._fence()                       # nobody overwrites rows that are still being pulled

    def gather_rows(self, field, rows):
        peers = self._peer_views(field)
        self._fence()
        for q, (a, b) in enumerate(rows):
            if q != self.rank:
                field[:, a:b].copy_(peers[q][:, a:b])
        self._fence()

    def close(self):
        for views in self._peers.values():
            for q, v in enumerate(views):
                if q != self.rank:
                    _lib.lib().b200p_ipc_close(C.c_void_p(v.data_ptr()))
        self._peers = {}
        for p in self._owned:
            _lib.lib().b200p_free(p)
        self._owned = []


class LocalGroup:
    """Virtual ranks inside one process (threads) on one device: the test double of a node."""

    def __init__(self, nranks):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.slots = [None] * nranks

    def transport(self, rank):
        return LocalTransport(self, rank)


class LocalTransport(Transport):
    def __init__(self, group: LocalGroup, rank: int):
        self.g, self.rank, self.nranks = group, rank, group.nranks

    def _publish(self, t):
        torch.cuda.synchronize() if t.is_cuda else None
        self.g.slots[self.rank] = t
        self.g.barrier.wait()

    def _done(self):
        torch.cuda.synchronize() if torch.cuda.is_available() else None
        self.g.barrier.wait()

    def _reduce(self, t, op):
        self._publish(t.clone())
        acc = self.g.slots[0].clone()
        for q in range(1, self.nranks):  # rank order: every virtual rank forms the same value
            acc = op(acc, self.g.slots[q])
        self.g.barrier.wait()
        t.copy_(acc)
        self._done()

    def sum_(self, t): self._reduce(t, torch.add)
    def max_(self, t): self._reduce(t, torch.maximum)

    def halo(self, u, ranges):
        self._publish(u)
        recv, _ = halo_plan(ranges, self.rank)
        for q, a, b in recv:
            u[:, a:b].copy_(self.g.slots[q][:, a:b])
        self._done()

    def gather_rows(self, field, rows):
        self._publish(field)
        for q, (a, b) in enumerate(rows):
            if q != self.rank:
                field[:, a:b].copy_(self.g.slots[q][:, a:b])
        self._done()


class StripSolver:
    """One rank of a strip-decomposed mg-oras solve of a single frame.

    Every rank passes the FULL mask and known values; `solve` returns this rank's rows of the
    solution (device tensor (C, own_hi - own_lo, W)), and the reports, identical on all ranks."""

    def __init__(self, width, height, channels, cfg: MultigridConfig | None, transport: Transport,
                 spacing: float = 1.0, levels: int = 1):
        """levels: how many of the finest levels are striped (the rest is replicated); 1 keeps 25 % of the
        work replicated, 2 about 6 %."""
        self.t = transport
        self.cfg = cfg or MultigridConfig()
        native = isinstance(transport, NcclNative)
        # a host callback between the kernels forces eager launches; the native exchange is captured with them
        self.plan = Plan(width, height, channels, 1, self.cfg, spacing, use_graphs=native)
        self.levels = int(levels)
        if not 1 <= self.levels < self.plan.num_levels:
            raise ValueError(f"need 1 <= striped levels < {self.plan.num_levels}")
        self.shapes = []
        for l in range(self.levels + 1):
            info = self.plan.level_info(l)
            self.shapes.append((int(channels), info.height, info.width))
        self.shape = self.shapes[0]
        rg = strip_ranges(height, self.cfg.block_size, self.cfg.overlap, transport.nranks, self.levels)
        self.ranges_by_level = [rg] if self.levels == 1 else rg
        self.ranges = self.ranges_by_level[0]
        # rows of the first replicated level that every rank restricted from the last striped level
        self.gather_rows = coarse_rows(self.ranges_by_level[-1], self.shapes[self.levels][1])
        self.error = None
        if native:
            flat = [v for q in range(transport.nranks) for l in range(self.levels) for v in self.ranges_by_level[l][q]]
            every = (C.c_int * len(flat))(*flat)
            _lib.check(_lib.lib().b200p_plan_set_strip_nccl(self.plan.handle, self.levels, C.cast(every, C.c_void_p),
                                                            transport.rank, transport.nranks, transport.comm))
            return
        self._cb = _EXCHANGE_FN(self._exchange)  # keep the callback object alive
        flat = [v for l in range(self.levels) for v in self.ranges_by_level[l][transport.rank]]
        mine = (C.c_int * len(flat))(*flat)
        _lib.check(_lib.lib().b200p_plan_set_strip(self.plan.handle, self.levels, C.cast(mine, C.c_void_p),
                                                   C.cast(self._cb, C.c_void_p), None))

    @property
    def own(self):
        r = self.ranges[self.t.rank]
        return r[0], r[1]

    def _exchange(self, user, kind, d_ptr, stream):
        try:
            P = self.shape[0]
            base, lvl = kind & 15, kind >> 4
            ext = torch.cuda.ExternalStream(int(stream or 0)) if stream else torch.cuda.default_stream()
            with torch.cuda.stream(ext):
                if base == XCHG_SUM_RS:
                    self.t.sum_(device_view(d_ptr, (P,), torch.float64))
                elif base == XCHG_MAX_FLAGS:
                    self.t.max_(device_view(d_ptr, (P,), torch.int32))
                elif base in (XCHG_HALO_U, XCHG_HALO_RC):
                    self.t.halo(device_view(d_ptr, self.shapes[lvl], torch.float64), self.ranges_by_level[lvl])
                elif base == XCHG_GATHER_RC:
                    self.t.gather_rows(device_view(d_ptr, self.shapes[lvl], torch.float64), self.gather_rows)
                else:
                    return 1
            return 0
        except BaseException as e:  # never let an exception cross the C boundary
            self.error = e
            return 2

    def solve(self, mask, known):
        c, h, w = self.shape
        d_mask = _dev.to_device_u8(np.ascontiguousarray(mask).view(np.uint8).reshape(1, h, w))
        d_known = _dev.to_device_f64(np.ascontiguousarray(known, dtype=np.float64).reshape(1, c, h, w))
        # one output buffer per solver (a transport may hand out cudaMalloc'ed memory that peers map: allocating
        # per solve would leak it and grow the peer-mapping cache); the caller gets a copy of the owned rows
        if getattr(self, "_d_out", None) is None:
            self._d_out = self.t.zeros_f64((1, c, h, w))
        else:
            self._d_out.zero_()
        d_out = self._d_out
        try:
            _, reports = self.plan.solve_device(d_mask, d_known, d_out)
        except Exception:
            if self.error is not None:
                raise self.error
            raise
        lo, hi = self.own
        return d_out[0, :, lo:hi].clone(), reports

    def close(self):
        self._d_out = None
        self.plan.close()
        if hasattr(self.t, "close"):
            self.t.close()
