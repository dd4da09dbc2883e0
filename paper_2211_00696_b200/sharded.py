"""Multi-GPU phi actions, one process per GPU (torch.distributed for the plumbing).

Two independent ways the path shards:

* right-hand sides: every rank evaluates its own b's end to end -- no data-path collective
  (bench.py's default N-GPU mode, weak scaling);
* quadrature nodes (Gauss rule): rank r sweeps nodes i with i % world == r on its GPU
  (pq_phi_nodes_partial: node exponentials, mode products, weighted partial sums in ascending
  node order), the partial sums are combined with ONE all-reduce (NCCL over NVLink on B200s),
  then either every rank runs the l modified-squaring steps (phi_with_plan_sharded: replicated)
  or the squaring itself is sharded over x-slabs with two all-to-all layout flips per step
  (phi_with_plan_distributed, dist_squaring.py: SURVEY 8(e)'s recommended design).

Parity: summing the partials changes only the association of the node sum, so results match
phi_with_plan to rounding (tests/test_sharded.py pins the host logic with world size 2 on gloo).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

import numpy as np

from . import _lib as L
from .phiquad import Context, KroneckerSum, QuadKind, cached_rule, default_context


def node_partition(q: int, rank: int, world: int) -> list:
    """Round-robin split of the q rule nodes (the C ABI's pq_phi_nodes_partial uses the same)."""
    if not (0 <= rank < world):
        raise ValueError("node_partition: bad rank/world")
    return list(range(rank, q, world))


def combine_partials(partials: list):
    """Host-side statement of the reduction: the full accumulator is the sum of the ranks'."""
    total = partials[0].copy()
    for p in partials[1:]:
        total = total + p
    return total


def phi_with_plan_sharded(a: KroneckerSum, bs, p: int, l: int, n: int, group=None, ctx: Optional[Context] = None,
                          all_reduce: Optional[Callable] = None):
    """Gauss-rule phi_1..phi_p of `a` on device-resident bs ([nb, N] float64 CUDA tensor), nodes
    sharded over the ranks of `group`.  Returns [nb, p, N] on every rank."""
    import torch
    import torch.distributed as dist

    ctx = ctx or default_context()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bs = bs.reshape(-1, a.dim()).contiguous()
    nb, N = bs.shape
    rule = cached_rule(QuadKind.gauss_legendre, n + 1)
    x = np.ascontiguousarray(rule.nodes)
    w = np.ascontiguousarray(rule.weights)
    acc = torch.empty((nb, p, N), dtype=torch.float64, device=bs.device)
    d, sh, fac = a._abi()
    L.check(L.lib.pq_phi_nodes_partial(ctx.handle, d, sh, fac, nb, C.c_void_p(bs.data_ptr()), p, l, rule.points(),
                                       x.ctypes.data_as(L.dp), w.ctypes.data_as(L.dp), rank, world, 1,
                                       C.c_void_p(acc.data_ptr())))
    if world > 1:
        # the default context runs on torch's current stream, which NCCL orders against
        if getattr(ctx, "_bound", None) is None:
            L.check(L.lib.pq_ctx_synchronize(ctx.handle))
        (all_reduce or dist.all_reduce)(acc, group=group)
        if getattr(ctx, "_bound", None) is None:
            torch.cuda.current_stream().synchronize()
    L.check(L.lib.pq_squaring_chain(ctx.handle, d, sh, fac, nb, p, l, C.c_void_p(acc.data_ptr())))
    return acc


def phi_with_plan_distributed(a: KroneckerSum, bs, p: int, l: int, n: int, group=None, ctx: Optional[Context] = None):
    """Like phi_with_plan_sharded, but the l squaring steps are sharded too: after the node
    all-reduce each rank keeps its x-slab, runs dist_squaring.squaring_distributed (local modes
    1..d-1, all-to-all to pencils, local mode 0, all-to-all back, elementwise combination), and
    the slabs are all-gathered at the end.  Returns [nb, p, N] on every rank."""
    import torch
    import torch.distributed as dist

    from .dist_squaring import DeviceBackend, SlabLayout, TorchComm, squaring_distributed
    from .phiquad import expm

    ctx = ctx or default_context()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bs = bs.reshape(-1, a.dim()).contiguous()
    nb, N = bs.shape
    rule = cached_rule(QuadKind.gauss_legendre, n + 1)
    x = np.ascontiguousarray(rule.nodes)
    w = np.ascontiguousarray(rule.weights)
    acc = torch.empty((nb, p, N), dtype=torch.float64, device=bs.device)
    d, sh, fac = a._abi()
    L.check(L.lib.pq_phi_nodes_partial(ctx.handle, d, sh, fac, nb, C.c_void_p(bs.data_ptr()), p, l, rule.points(),
                                       x.ctypes.data_as(L.dp), w.ctypes.data_as(L.dp), rank, world, 1,
                                       C.c_void_p(acc.data_ptr())))
    if world > 1:
        if getattr(ctx, "_bound", None) is None:
            L.check(L.lib.pq_ctx_synchronize(ctx.handle))
        dist.all_reduce(acc, group=group)
    shape = a.shape()
    lay = SlabLayout(shape, world)
    b0, b1 = lay.slab_range(rank)
    y = acc.reshape(nb * p, N)[:, b0:b1].contiguous()
    if l > 0:
        # E_j = expm(2^(j-l) A_k), j < l: the squaring chain (phiaction.hpp:294-301), replicated
        exps = [[None] * d for _ in range(l)]
        for k in range(d):
            f = torch.from_numpy(np.ascontiguousarray(a.factor(k))).to(bs.device)
            ek = expm(f, scale=[2.0 ** (j - l) for j in range(l)], ctx=ctx)
            for j in range(l):
                exps[j][k] = ek[j].contiguous()
        comm = TorchComm(rank, world, group) if world > 1 else None
        if comm is None:
            class _One:
                rank, world = 0, 1
            comm = _One()
        y = squaring_distributed(y, exps, lay, comm, DeviceBackend(ctx), p, nb)
    if world > 1:
        parts = [torch.empty((nb * p, lay.slab_len(r)), dtype=y.dtype, device=y.device) for r in range(world)]
        dist.all_gather(parts, y.contiguous(), group=group)
        return torch.cat(parts, dim=1).reshape(nb, p, N)
    return y.reshape(nb, p, N)
