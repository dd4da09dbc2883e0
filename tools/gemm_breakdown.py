"""Per-call-site breakdown of the DMMA GEMM launches of one phi_0..phi_p call (profiling mode:
each launch bracketed by CUDA events; executed flops counted on the device), for a BASELINE
config.  Usage: python tools/gemm_breakdown.py [config] [steps]"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2211_00696_b200 as pq  # noqa: E402
from paper_2211_00696_b200.workloads import config  # noqa: E402

PEAK = 37.15
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = config(cfg)
nb = w.nb if cfg == 3 else 1
a = pq.KroneckerSum(w.factors)
ctx = pq.Context(0)
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
bs = torch.from_numpy(np.stack([w.rhs(k) for k in range(nb)])).cuda()
out0 = torch.empty((nb, w.N), dtype=torch.float64, device="cuda")
out = torch.empty((nb, w.p, w.N), dtype=torch.float64, device="cuda")
d, sh, fac = a._abi()
rc = req._c()
info = pq._lib.PhiInfoC()
if cfg == 4:
    from paper_2211_00696_b200.workloads import allen_cahn_u0
    u0 = torch.from_numpy(allen_cahn_u0(w.N)).cuda()


def call():
    if cfg == 4:
        pq.integrate(pq.KroneckerSum(w.A), ("cubic", 1.0, -1.0), u0, 0.0, 10 * w.tau, 10, pq.etdrk4_tableau(),
                     pq.PhiRequest(eps=w.eps), ctx=ctx)
        return
    pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, nb, C.c_void_p(bs.data_ptr()), C.byref(rc),
                                        C.c_void_p(out0.data_ptr()), C.c_void_p(out.data_ptr()), C.byref(info),
                                        pq._lib.PQ_DEVICE))


torch.cuda.synchronize()
for _ in range(3):
    call()
ctx.synchronize()
ctx.set_profiling(True)
ctx.gemm_breakdown(reset=True)
ctx.gemm_stats(reset=True)
for _ in range(steps):
    call()
bd = ctx.gemm_breakdown(reset=True)
ks = ctx.kernel_stats(reset=True)
ctx.set_profiling(False)
tot_ms = sum(v["ms"] for v in bd.values())
tot_fl = sum(v["flops"] for v in bd.values())
print(f"config {cfg}: {steps} calls, GEMM {tot_ms / steps * 1e3:.1f} us/call, executed "
      f"{tot_fl / (tot_ms / 1e3) / 1e12:.2f} TF/s = {tot_fl / (tot_ms / 1e3) / 1e12 / PEAK:.3f} of peak")
print(f"{'site / shape':58s} {'launch':>6s} {'us/call':>8s} {'share':>6s} {'exec TF/s':>9s} {'frac':>6s} {'skip':>5s}")
for k, v in sorted(bd.items(), key=lambda kv: -kv[1]["ms"]):
    tf = v["flops"] / (v["ms"] / 1e3) / 1e12 if v["ms"] > 0 else 0
    print(f"{k:58s} {v['launches'] / steps:6.1f} {v['ms'] / steps * 1e3:8.1f} {v['ms'] / tot_ms:6.1%} {tf:9.2f} "
          f"{tf / PEAK:6.3f} {1 - v['flops'] / max(v['dense'], 1):5.2f}")
print(json.dumps({"kernel_stats": ks}))
