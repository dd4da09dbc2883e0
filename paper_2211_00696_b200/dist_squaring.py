"""Distributed modified squaring (recommended design): the l doubling steps of
phiaction.hpp:255-272 sharded over the ranks of one node instead of replicated.

Layouts of a vector of shape (n0, n1, ..., n_{d-1}) in the reference's vec order (x slowest):

* slab:   rank r owns the x-indices i0 in [s[r], s[r+1])  -- a contiguous range of the vector;
* pencil: rank r owns the flattened trailing indices c = (i1, ..., i_{d-1}) in [c[r], c[r+1]) for
          every i0 -- an n0 x (c[r+1] - c[r]) block.

A squaring step E y_i for the p columns (E = E_0 (x) ... (x) E_{d-1}): modes 1..d-1 act inside
each x-slab (local); one all-to-all flips slab -> pencil; mode 0 acts on the pencil (local); a
second all-to-all flips back; the combination T_i <- 2^-i (T_i + sum_j y_j/(i-j)!) is elementwise
(local).  Per step and column every rank moves (N/G) doubles twice over NVLink (NCCL all-to-all)
and does 1/G of the DMMA work, so the squaring no longer caps node-sharded scaling.

The algorithm is written once against two small interfaces:

* a backend (`DeviceBackend`: the B200 engine's pq_mode_product / pq_squaring_combine on CUDA
  tensors; `NumpyBackend`: numpy, for the CPU tests), and
* a communicator (`TorchComm`: torch.distributed all_to_all_single -- NCCL on GPUs, gloo on CPU;
  `ThreadComm`: ranks emulated by threads in one process, for the single-GPU test).

Each output element goes through the same mode products and the same elementwise combination as
in the unsharded chain; only tile shapes (and hence DMMA summation order) differ, so the result
matches the single-GPU squaring to rounding (tests/test_dist_squaring.py: gloo world sizes 2 and 3
on CPU with the numpy backend; 2 and 4 thread-emulated ranks on one B200 with the device backend).
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import List, Sequence

import numpy as np

from . import _lib as L


class SlabLayout:
    """Slab and pencil ownership for `world` ranks of a vector of the given shape."""

    def __init__(self, shape: Sequence[int], world: int):
        if world < 1:
            raise ValueError("SlabLayout: world must be >= 1")
        self.shape = [int(n) for n in shape]
        self.world = world
        self.n0 = self.shape[0]
        self.rest = int(np.prod(self.shape[1:])) if len(self.shape) > 1 else 1
        if self.n0 < world:
            raise ValueError("SlabLayout: fewer x-slabs than ranks")
        self.s = [self.n0 * r // world for r in range(world + 1)]       # slab i0 bounds
        self.c = [self.rest * r // world for r in range(world + 1)]     # pencil column bounds

    def slab_rows(self, r: int) -> int:
        return self.s[r + 1] - self.s[r]

    def pencil_cols(self, r: int) -> int:
        return self.c[r + 1] - self.c[r]

    def slab_len(self, r: int) -> int:
        return self.slab_rows(r) * self.rest

    def slab_range(self, r: int) -> tuple:
        """[begin, end) of rank r's slab inside a full vector."""
        return self.s[r] * self.rest, self.s[r + 1] * self.rest


# ------------------------------------------------------------------------------ backends ----

class NumpyBackend:
    """CPU stand-in (tests): arrays are numpy [ncols, len]."""

    @staticmethod
    def mode_product(shape, mode, E, x):
        ncols = x.shape[0]
        t = x.reshape(ncols, *shape)
        y = np.moveaxis(np.tensordot(E, np.moveaxis(t, mode + 1, 0), axes=([1], [0])), 0, mode + 1)
        return np.ascontiguousarray(y).reshape(ncols, -1)

    @staticmethod
    def combine(t, y_old, p, nb):
        inv = [1.0]
        for k in range(1, p):
            inv.append(inv[-1] / k)
        T = t.reshape(nb, p, -1)
        Y = y_old.reshape(nb, p, -1)
        out = np.empty_like(T)
        for i in range(p):
            v = np.ldexp(1.0, -(i + 1)) * T[:, i]
            for j in range(i + 1):
                v = v + (np.ldexp(1.0, -(i + 1)) * inv[i - j]) * Y[:, j]
            out[:, i] = v
        t[...] = out.reshape(t.shape)

    @staticmethod
    def empty_like(x):
        return np.empty_like(x)

    @staticmethod
    def concat(blocks, axis):
        return np.concatenate(blocks, axis=axis)

    @staticmethod
    def contiguous(x):
        return np.ascontiguousarray(x)


class DeviceBackend:
    """The B200 engine through the C ABI; arrays are CUDA float64 tensors [ncols, len] on the
    stream the context runs on (a Context bound to torch's current stream)."""

    def __init__(self, ctx):
        self.ctx = ctx

    def mode_product(self, shape, mode, E, x):
        import torch
        ncols = x.shape[0]
        y = torch.empty_like(x)
        sh = (C.c_int * len(shape))(*shape)
        L.check(L.lib.pq_mode_product(self.ctx.handle, len(shape), sh, mode, C.c_void_p(E.data_ptr()), ncols,
                                      C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr())))
        return y

    def combine(self, t, y_old, p, nb):
        L.check(L.lib.pq_squaring_combine(self.ctx.handle, t.shape[1], p, nb, C.c_void_p(t.data_ptr()),
                                          C.c_void_p(y_old.data_ptr())))

    @staticmethod
    def empty_like(x):
        import torch
        return torch.empty_like(x)

    @staticmethod
    def concat(blocks, axis):
        import torch
        return torch.cat(blocks, dim=axis)

    @staticmethod
    def contiguous(x):
        return x.contiguous()


# ------------------------------------------------------------------------- communicators ----

class TorchComm:
    """torch.distributed all-to-all with uneven splits (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def alltoallv(self, blocks: List, recv_sizes: List[int]) -> List:
        import torch
        import torch.distributed as dist
        sizes = [int(b.numel()) for b in blocks]
        send = torch.cat([b.reshape(-1) for b in blocks])
        recv = torch.empty(sum(recv_sizes), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(recv, send, output_split_sizes=recv_sizes, input_split_sizes=sizes, group=self.group)
        return list(torch.split(recv, recv_sizes))


class ThreadComm:
    """In-process emulation: ranks are threads; `alltoallv(rank, blocks)` exchanges through a
    mailbox between two barriers (device data is handed over after the sender's stream drained)."""

    def __init__(self, world: int):
        self.world = world
        self.box = [[None] * world for _ in range(world)]
        self.bar = threading.Barrier(world)

    def bind(self, rank: int, sync=None):
        comm = self

        class _Rank:
            def __init__(self):
                self.rank, self.world = rank, comm.world

            def alltoallv(self, blocks, recv_sizes=None):
                if sync is not None:
                    sync()
                for s in range(comm.world):
                    comm.box[rank][s] = blocks[s]
                comm.bar.wait()
                got = [comm.box[s][rank] for s in range(comm.world)]
                comm.bar.wait()
                return got

        return _Rank()


# ---------------------------------------------------------------------------- algorithm -----

def _slab_to_pencil(t, lay: SlabLayout, comm, be, ncols: int):
    r = comm.rank
    m = lay.slab_rows(r)
    t3 = t.reshape(ncols, m, lay.rest)
    send = [be.contiguous(t3[:, :, lay.c[s]:lay.c[s + 1]]) for s in range(lay.world)]
    q = lay.pencil_cols(r)
    got = comm.alltoallv(send, [ncols * lay.slab_rows(s) * q for s in range(lay.world)])
    blocks = [g.reshape(ncols, lay.slab_rows(s), q) for s, g in enumerate(got)]
    return be.contiguous(be.concat(blocks, 1)).reshape(ncols, lay.n0 * q)


def _pencil_to_slab(u, lay: SlabLayout, comm, be, ncols: int):
    r = comm.rank
    q = lay.pencil_cols(r)
    u3 = u.reshape(ncols, lay.n0, q)
    send = [be.contiguous(u3[:, lay.s[s]:lay.s[s + 1], :]) for s in range(lay.world)]
    m = lay.slab_rows(r)
    got = comm.alltoallv(send, [ncols * m * lay.pencil_cols(s) for s in range(lay.world)])
    blocks = [g.reshape(ncols, m, lay.pencil_cols(s)) for s, g in enumerate(got)]
    return be.contiguous(be.concat(blocks, 2)).reshape(ncols, m * lay.rest)


def squaring_distributed(y_slab, exps: Sequence[Sequence], lay: SlabLayout, comm, be, p: int, nb: int):
    """l modified-squaring steps on this rank's slab of the [nb][p] columns (y_slab: [nb*p, slab]).
    exps[step][k] = expm(2^(step-l) A_k) (n_k x n_k, replicated on every rank).  Returns the slab
    of phi_j(A) b after the last step."""
    ncols = nb * p
    r = comm.rank
    slab_shape = [lay.slab_rows(r)] + lay.shape[1:]
    pencil_shape = [lay.n0, lay.pencil_cols(r)]
    y = y_slab
    for E in exps:
        t = y
        for k in range(1, len(lay.shape)):          # modes 1..d-1 inside the slab
            t = be.mode_product(slab_shape, k, E[k], t)
        if lay.world == 1:
            t = be.mode_product(lay.shape, 0, E[0], t)
        else:
            u = _slab_to_pencil(t, lay, comm, be, ncols)
            u = be.mode_product(pencil_shape, 0, E[0], u)   # mode 0 on the pencil
            t = _pencil_to_slab(u, lay, comm, be, ncols)
        be.combine(t, y, p, nb)                     # T_i <- 2^-i (T_i + sum_j y_j/(i-j)!)
        y = t
    return y
