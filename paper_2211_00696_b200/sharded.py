"""Multi-GPU phi actions, one process per GPU: the Python face of the C ABI's distributed path
(include/pq_b200.h `pq_*_dist`, paper_2211_00696_b200/csrc/dist.cpp).

The reference parallelises only its node loop over threads (phiaction.hpp:85, util.hpp:24-39)
and squares serially (phiaction.hpp:255-272, 293-301).  Here, across the ranks of a communicator:

* quadrature nodes are dealt round-robin (i % world == rank; each adaptive-CC level's fresh
  nodes likewise) and each rank sweeps only its nodes;
* ONE all-to-all moves every node vector's x-slab to the slab's owner, which forms the weighted
  sums in ascending node order (no cross-rank floating-point reduction in the node phase);
* the adaptive-CC error is an exact all-reduce(max) of 2 nb p scalars per level;
* the l modified-squaring steps and phi_0 run on slabs: modes 1..d-1 inside the slab, slab <->
  pencil all-to-alls around mode 0 (hand-written pack / unpack kernels for the flips);
* the slabs are all-gathered into full vectors on every rank (or kept as slabs, gather=False).

Transports: NCCL over NVLink (`Communicator.nccl`, the production path: the C++ engine issues
grouped ncclSend/ncclRecv on its own stream) or torch.distributed on host buffers
(`Communicator.host`, e.g. gloo -- what lets two processes share one GPU in the tests).  Right-hand
side sharding needs no communicator at all (every rank calls phiquadmv on its own b's).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib as L
from .phiquad import Context, KroneckerSum, PhiInfo, PhiRequest, QuadKind, _info, default_context


def node_partition(q: int, rank: int, world: int) -> list:
    """The nodes rank `rank` evaluates (dist.cpp owned(): slot i -> rank i % world)."""
    if not (0 <= rank < world):
        raise ValueError("node_partition: bad rank/world")
    return list(range(rank, q, world))


def slab_range(shape, world: int, rank: int) -> tuple:
    """[begin, end) of rank's x-slab in a vector of the given shape (pq_dist_slab)."""
    sh = (C.c_int * len(shape))(*[int(n) for n in shape])
    b, e = C.c_int64(), C.c_int64()
    L.check(L.lib.pq_dist_slab(len(shape), sh, world, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


class Communicator:
    """pq_comm: the ranks a distributed call spans and how their data moves."""

    def __init__(self, handle, world: int, rank: int, keep=()):
        self.handle, self.world, self.rank = handle, world, rank
        self._keep = keep  # ctypes callbacks must outlive the handle

    @classmethod
    def nccl(cls, ctx: Context, group=None) -> "Communicator":
        """NCCL communicator over the ranks of a torch.distributed group (rank 0's unique id is
        broadcast through the group); collectives run on the context's stream."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        idb = C.create_string_buffer(128)
        if rank == 0:
            L.check(L.lib.pq_nccl_unique_id(idb))
        box = [bytes(idb.raw) if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        idb = C.create_string_buffer(box[0], 128)
        h = C.c_void_p()
        L.check(L.lib.pq_comm_create_nccl(ctx.handle, world, rank, idb, C.byref(h)))
        return cls(h, world, rank)

    @classmethod
    def host(cls, group=None) -> "Communicator":
        """Collectives through torch.distributed on host buffers (gloo): all_to_all_single for the
        exchanges, all_reduce(MAX) for the adaptive-CC statistics."""
        return cls._with_host_transport(group, None)

    @classmethod
    def peer(cls, ctx: Context, group=None) -> "Communicator":
        """Peer transport: the squaring's slab <-> pencil flips fused into the mode products, whose
        epilogues store straight into the owning rank's CUDA-IPC-mapped buffer (NVLink between GPUs;
        processes sharing one GPU in the tests); torch.distributed (gloo) carries the handle
        exchange and the per-flip barrier."""
        return cls._with_host_transport(group, ctx)

    @classmethod
    def _with_host_transport(cls, group, peer_ctx) -> "Communicator":
        import torch
        import torch.distributed as dist
        if group is None and dist.get_backend() != "gloo":
            group = dist.new_group(backend="gloo")  # the host transport moves CPU tensors
        world, rank = dist.get_world_size(group), dist.get_rank(group)

        def view(ptr, n):
            if n == 0:
                return torch.empty(0, dtype=torch.float64)
            return torch.from_numpy(np.ctypeslib.as_array(ptr, (n,)))

        def a2a(user, send, scounts, recv, rcounts):
            try:
                sc = [int(scounts[h]) for h in range(world)]
                rc = [int(rcounts[h]) for h in range(world)]
                dist.all_to_all_single(view(recv, sum(rc)), view(send, sum(sc)), output_split_sizes=rc,
                                       input_split_sizes=sc, group=group)
                return 0
            except Exception:  # surfaced as PQ_ERUNTIME by the engine
                return 1

        def amax(user, buf, n):
            try:
                dist.all_reduce(view(buf, int(n)), op=dist.ReduceOp.MAX, group=group)
                return 0
            except Exception:
                return 1

        cb_a2a, cb_max = L.ALLTOALLV_CB(a2a), L.ALLREDUCE_CB(amax)
        t = L.HostTransportC(None, cb_a2a, cb_max)
        h = C.c_void_p()
        if peer_ctx is None:
            L.check(L.lib.pq_comm_create_host(world, rank, C.byref(t), C.byref(h)))
        else:
            L.check(L.lib.pq_comm_create_peer(peer_ctx.handle, world, rank, C.byref(t), C.byref(h)))
        return cls(h, world, rank, keep=(cb_a2a, cb_max, t))

    @classmethod
    def single(cls) -> "Communicator":
        h = C.c_void_p()
        L.check(L.lib.pq_comm_create_host(1, 0, None, C.byref(h)))
        return cls(h, 1, 0)

    def stats(self, reset: bool = False) -> tuple:
        """(bytes this rank sent to other ranks, exchanges issued) since the last reset."""
        b, n = C.c_double(), C.c_uint64()
        L.check(L.lib.pq_comm_stats(self.handle, 1 if reset else 0, C.byref(b), C.byref(n)))
        return b.value, int(n.value)

    def close(self) -> None:
        if self.handle:
            L.lib.pq_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _prep(a: KroneckerSum, bs):
    """Device float64 [nb, N] tensor or host numpy [nb, N] -> (pointer, space, nb, is_device)."""
    dim = a.dim()
    if hasattr(bs, "is_cuda") and bs.is_cuda:
        bs = bs.reshape(-1, dim).contiguous()
        return bs, C.c_void_p(bs.data_ptr()), L.PQ_DEVICE, bs.shape[0], True
    bs = np.ascontiguousarray(np.asarray(bs, dtype=np.float64).reshape(-1, dim))
    return bs, C.c_void_p(bs.ctypes.data), L.PQ_HOST, bs.shape[0], False


class _StreamOrder:
    """Device tensors produced on torch's current stream, consumed on the context's stream: unless
    the context runs ON torch's current stream (default_context() does), drain torch's stream before
    the call and the context's stream after it, so neither side reads before the other wrote."""

    def __init__(self, ctx: Context, dev: bool):
        self.ctx, self.dev = ctx, dev

    def __enter__(self):
        if self.dev:
            import torch
            self.bound = getattr(self.ctx, "_bound", None) == torch.cuda.current_stream().cuda_stream
            if not self.bound:
                torch.cuda.current_stream().synchronize()
        return self

    def __exit__(self, *exc):
        if self.dev and not self.bound:
            self.ctx.synchronize()


def _empty(like_device: bool, shape, device=None):
    if like_device:
        import torch
        return torch.empty(shape, dtype=torch.float64, device=device)
    return np.empty(shape)


def _ptr(x):
    return C.c_void_p(x.data_ptr() if hasattr(x, "data_ptr") else x.ctypes.data)


def phiquadmv_dist(a: KroneckerSum, bs, req: PhiRequest, comm: Communicator, ctx: Optional[Context] = None,
                   gather: bool = True, phi0: bool = False, info: Optional[PhiInfo] = None):
    """phiquadmv_multi (phiaction.hpp:307-346) across `comm`; every rank passes the same a, bs, req.
    Returns cols [nb, p, N] (gather) or this rank's slabs [nb, p, end - begin]; with phi0=True,
    (phi0, cols).  Device tensors in -> device tensors out (stream-ordered on ctx's stream)."""
    ctx = ctx or default_context()
    keep, bp, space, nb, dev = _prep(a, bs)
    n_out = a.dim() if gather else (lambda r: r[1] - r[0])(slab_range(a.shape(), comm.world, comm.rank))
    out = _empty(dev, (nb, req.p, n_out), device=getattr(keep, "device", None))
    out0 = _empty(dev, (nb, n_out), device=getattr(keep, "device", None)) if phi0 else None
    ci = L.PhiInfoC()
    d, sh, fac = a._abi()
    rc = req._c()
    with _StreamOrder(ctx, dev):
        L.check(L.lib.pq_phiquadmv_dist(ctx.handle, comm.handle, d, sh, fac, nb, bp, C.byref(rc),
                                        _ptr(out0) if phi0 else None, _ptr(out), C.byref(ci), space, 1 if gather else 0))
    if info is not None:
        info.__dict__.update(_info(ci).__dict__)
    return (out0, out) if phi0 else out


def phi_with_plan_dist(a: KroneckerSum, bs, p: int, l: int, n: int, mode: QuadKind, eps: float, comm: Communicator,
                       ctx: Optional[Context] = None, gather: bool = True, info: Optional[dict] = None):
    """phi_with_plan (phiaction.hpp:277-303) across `comm` at an explicit (l, n)."""
    ctx = ctx or default_context()
    keep, bp, space, nb, dev = _prep(a, bs)
    n_out = a.dim() if gather else (lambda r: r[1] - r[0])(slab_range(a.shape(), comm.world, comm.rank))
    out = _empty(dev, (nb, p, n_out), device=getattr(keep, "device", None))
    pts = C.c_int()
    d, sh, fac = a._abi()
    with _StreamOrder(ctx, dev):
        L.check(L.lib.pq_phi_with_plan_dist(ctx.handle, comm.handle, d, sh, fac, nb, bp, p, l, n, int(mode), float(eps),
                                            _ptr(out), C.byref(pts), space, 1 if gather else 0))
    if info is not None:
        info["points_used"] = pts.value
    return out
