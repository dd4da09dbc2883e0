"""pq_phi_0p with PAGEABLE host buffers (numpy, pre-touched) vs pinned, config 2: what a drop-in
user's std::vector buffers cost in the engine itself (the header's own allocations excluded)."""
import ctypes as C
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2211_00696_b200 as pq
from paper_2211_00696_b200.workloads import config

w = config(2)
a = pq.KroneckerSum(w.factors)
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
d, sh, fac = a._abi()
rc = req._c()
ctx = pq.Context(0)
N = w.N


def run(b, o0, o, reps=8):
    inf = pq._lib.PhiInfoC()

    def call():
        pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, 1, C.c_void_p(b.ctypes.data), C.byref(rc),
                                            C.c_void_p(o0.ctypes.data), C.c_void_p(o.ctypes.data), C.byref(inf),
                                            pq._lib.PQ_HOST))
    call()
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    return (time.perf_counter() - t0) / reps * 1e3


b = w.rhs(0)
pag = run(b.copy(), np.zeros((1, N)), np.zeros((1, w.p, N)))
bp = torch.from_numpy(b.copy()).pin_memory()
o0p = torch.zeros((1, N), dtype=torch.float64).pin_memory()
op = torch.zeros((1, w.p, N), dtype=torch.float64).pin_memory()
pin = run(bp.numpy(), o0p.numpy(), op.numpy())
t0 = time.perf_counter()
for _ in range(8):
    x = np.zeros((w.p, N))
    x[:] = 1.0
t_alloc = (time.perf_counter() - t0) / 8 * 1e3
print(json.dumps({"pageable_ms": pag, "pinned_ms": pin, "host_fresh_67MB_alloc_and_write_ms": t_alloc}))


def run_mv(b, o, reps=8):
    inf = pq._lib.PhiInfoC()

    def call():
        pq._lib.check(pq._lib.lib.pq_phiquadmv(ctx.handle, d, sh, fac, 1, C.c_void_p(b.ctypes.data), C.byref(rc),
                                               C.c_void_p(o.ctypes.data), C.byref(inf), pq._lib.PQ_HOST))
    call()
    t0 = time.perf_counter()
    for _ in range(reps):
        call()
    return (time.perf_counter() - t0) / reps * 1e3


print(json.dumps({"phiquadmv_pageable_ms": run_mv(b.copy(), np.zeros((1, w.p, N))),
                  "phiquadmv_pinned_ms": run_mv(bp.numpy(), op.numpy())}))
