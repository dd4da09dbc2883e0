"""One phi_0..phi_p call of a BASELINE config bracketed by cudaProfilerStart/Stop (after 3 warm-up
calls), for `ncu --profile-from-start off ...`.  Usage: python tools/profile_call.py [config]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2211_00696_b200 as pq  # noqa: E402
from paper_2211_00696_b200.workloads import config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = config(cfg)
nb = w.nb if cfg == 3 else 1
a = pq.KroneckerSum(w.factors)
ctx = pq.Context(0)
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
d, sh, fac = a._abi()
rc = req._c()
out0 = torch.empty((nb, w.N), dtype=torch.float64, device="cuda")
out = torch.empty((nb, w.p, w.N), dtype=torch.float64, device="cuda")
info = pq._lib.PhiInfoC()
for i in range(4):
    b = torch.from_numpy(np.stack([w.rhs(200 + 10 * i + k) for k in range(nb)])).cuda()
    torch.cuda.synchronize()
    if i == 3:
        torch.cuda.cudart().cudaProfilerStart()
    pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, nb, C.c_void_p(b.data_ptr()), C.byref(rc),
                                        C.c_void_p(out0.data_ptr()), C.c_void_p(out.data_ptr()), C.byref(info),
                                        pq._lib.PQ_DEVICE))
    ctx.synchronize()
    if i == 3:
        torch.cuda.cudart().cudaProfilerStop()
print(f"config {cfg}: plan (l, n, points) = ({info.l}, {info.n}, {info.points})")
