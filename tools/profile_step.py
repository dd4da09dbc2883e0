#!/usr/bin/env python
"""One warm phi_0..phi_p call, then one call inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and `--set full` captures of a single step.

usage: python tools/profile_step.py [--config 2] [--n N]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import torch
    import paper_2211_00696_b200 as pq
    from paper_2211_00696_b200 import _lib as L
    from paper_2211_00696_b200.workloads import config

    w = config(args.config, args.n)
    a = pq.KroneckerSum(w.factors)
    ctx = pq.Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    b = torch.from_numpy(w.rhs(0)).cuda()
    out0 = torch.empty(w.N, dtype=torch.float64, device="cuda")
    out = torch.empty((w.p, w.N), dtype=torch.float64, device="cuda")
    d, sh, fac = a._abi()
    rc = req._c()
    info = L.PhiInfoC()

    def step():
        L.check(L.lib.pq_phi_0p(ctx.handle, d, sh, fac, 1, C.c_void_p(b.data_ptr()), C.byref(rc),
                                C.c_void_p(out0.data_ptr()), C.c_void_p(out.data_ptr()), C.byref(info), L.PQ_DEVICE))

    step()
    torch.cuda.synchronize()
    l0 = ctx.launches
    torch.cuda.profiler.start()
    for _ in range(args.reps):
        step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"launches per step: {(ctx.launches - l0) / args.reps:.0f}  plan l={info.l} n={info.n} points={info.points}")


if __name__ == "__main__":
    main()
