"""Phase marks of device-resident phi_0..phi_p calls (PQ_TRACE-style: a CUDA event + the host clock at
every engine mark, no stream serialisation): for each of the last `calls` calls, the GPU time and
the host time of every mark relative to the call's first mark.  Shows where the host is on the
critical path (host time ahead of / behind the GPU).  Usage: python tools/trace_call.py [config] [calls]"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

os.environ["PQ_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2211_00696_b200 as pq  # noqa: E402
from paper_2211_00696_b200.workloads import config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = config(cfg)
nb = w.nb if cfg == 3 else 1
a = pq.KroneckerSum(w.factors)
ctx = pq.Context(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
d, sh, fac = a._abi()
rc = req._c()
bs = [torch.from_numpy(np.stack([w.rhs(300 + 10 * i + k) for k in range(nb)])).cuda() for i in range(calls + 4)]
out0 = torch.empty((nb, w.N), dtype=torch.float64, device="cuda")
out = torch.empty((nb, w.p, w.N), dtype=torch.float64, device="cuda")
info = pq._lib.PhiInfoC()
lib = pq._lib.lib
lib.pq_ctx_timeline.argtypes = [C.c_void_p, C.POINTER(C.c_char_p)]
for i in range(calls + 4):
    torch.cuda.synchronize()
    js = C.c_char_p()
    lib.pq_ctx_timeline(ctx.handle, C.byref(js))  # clears the marks
    pq._lib.check(lib.pq_phi_0p(ctx.handle, d, sh, fac, nb, C.c_void_p(bs[i].data_ptr()), C.byref(rc),
                                C.c_void_p(out0.data_ptr()), C.c_void_p(out.data_ptr()), C.byref(info),
                                pq._lib.PQ_DEVICE))
    torch.cuda.synchronize()
    if i >= 4:
        lib.pq_ctx_timeline(ctx.handle, C.byref(js))
        marks = json.loads(js.value.decode())
        print(f"call {i - 4}: " + "  ".join(f"{m['mark']}@gpu{m['gpu_us']:.0f}/host{m['host_us']:.0f}" for m in marks))
