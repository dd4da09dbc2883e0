#!/usr/bin/env python
"""Device/host timeline of one phi_0..phi_p call (engine marks, pq_ctx_timeline).

usage: python tools/timeline.py [config] [--trace]
  default: marks under profiling mode (every GEMM bracketed by events, side streams serialised);
  --trace: PQ_TRACE=1 marks only, normal scheduling (the production overlap is kept).
  --host: the end-to-end call (pinned host b in, phi_0..phi_p to pinned host memory, PQ_HOST)."""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import paper_2211_00696_b200 as pq
    from paper_2211_00696_b200 import _lib as L
    from paper_2211_00696_b200.workloads import config
    args = [x for x in sys.argv[1:] if not x.startswith("--")]
    trace = "--trace" in sys.argv
    if trace:
        os.environ["PQ_TRACE"] = "1"
    cfg = int(args[0]) if args else 2
    w = config(cfg)
    a = pq.KroneckerSum(w.factors)
    ctx = pq.Context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx.set_stream(s.cuda_stream)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    b = torch.from_numpy(w.rhs(0)).cuda()
    out0 = torch.empty(w.N, dtype=torch.float64, device="cuda")
    out = torch.empty((w.p, w.N), dtype=torch.float64, device="cuda")
    d, sh, fac = a._abi()
    rc = req._c()
    info = L.PhiInfoC()

    space = L.PQ_DEVICE
    if "--host" in sys.argv:
        b, out0, out = b.cpu().pin_memory(), out0.cpu().pin_memory(), out.cpu().pin_memory()
        space = L.PQ_HOST

    def step():
        L.check(L.lib.pq_phi_0p(ctx.handle, d, sh, fac, 1, C.c_void_p(b.data_ptr()), C.byref(rc),
                                C.c_void_p(out0.data_ptr()), C.c_void_p(out.data_ptr()), C.byref(info), space))

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    if not trace:
        ctx.set_profiling(True)
    for it in range(2):
        step()
        js = C.c_char_p()
        L.check(L.lib.pq_ctx_timeline(ctx.handle, C.byref(js)))
        marks = json.loads(js.value.decode())
        print(f"call {it}:")
        prev = None
        for m in marks:
            dg = m["gpu_us"] - (prev["gpu_us"] if prev else 0)
            dh = m["host_us"] - (prev["host_us"] if prev else 0)
            print(f"  {m['mark']:20s} gpu {m['gpu_us']:9.1f} (+{dg:8.1f})   host {m['host_us']:9.1f} (+{dh:8.1f})")
            prev = m
        ctx.gemm_stats(reset=True)


if __name__ == "__main__":
    main()
