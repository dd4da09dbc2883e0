"""Device timeline of phi_0..phi_p calls from CUPTI (torch.profiler's kineto collects every kernel
and memcpy of the process, the engine's own kernels included): span per call, busy time (union
of kernel intervals over all streams), the largest idle gaps and the kernels around them.
Usage: python tools/timeline.py [config] [calls] [--host] [--dump=file.csv]   (--host: pinned host buffers,
PQ_HOST; --dump: every op of the last call, start offset / duration / stream)"""
import ctypes as C
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2211_00696_b200 as pq  # noqa: E402
from paper_2211_00696_b200.workloads import config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2
calls = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 3
host = "--host" in sys.argv
w = config(cfg)
nb = w.nb if cfg == 3 else 1
a = pq.KroneckerSum(w.factors)
ctx = pq.Context(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
bsh = [np.stack([w.rhs(100 + 10 * i + k) for k in range(nb)]) for i in range(calls + 3)]
if host:
    bs = [torch.from_numpy(b).pin_memory() for b in bsh]
    out0 = torch.empty((nb, w.N), dtype=torch.float64).pin_memory()
    out = torch.empty((nb, w.p, w.N), dtype=torch.float64).pin_memory()
else:
    bs = [torch.from_numpy(b).cuda() for b in bsh]
    out0 = torch.empty((nb, w.N), dtype=torch.float64, device="cuda")
    out = torch.empty((nb, w.p, w.N), dtype=torch.float64, device="cuda")
d, sh, fac = a._abi()
rc = req._c()
if cfg == 4:
    from paper_2211_00696_b200.workloads import allen_cahn_u0
    u_etd = torch.from_numpy(allen_cahn_u0(w.N)).cuda()
info = pq._lib.PhiInfoC()
space = pq._lib.PQ_HOST if host else pq._lib.PQ_DEVICE


def call(i):
    if cfg == 4:
        pq.integrate(pq.KroneckerSum(w.A), ("cubic", 1.0, -1.0), u_etd, 0.0, 20 * w.tau, 20, pq.etdrk4_tableau(),
                     pq.PhiRequest(eps=w.eps), ctx=ctx)
        return
    pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, nb, C.c_void_p(bs[i].data_ptr()), C.byref(rc),
                                        C.c_void_p(out0.data_ptr()), C.c_void_p(out.data_ptr()), C.byref(info), space))


for i in range(3):
    call(i)
torch.cuda.synchronize()
marks = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for i in range(calls):
        e = torch.cuda.Event(enable_timing=False)
        call(3 + i)
        torch.cuda.synchronize()
tmp = tempfile.NamedTemporaryFile(suffix=".json", delete=False).name
prof.export_chrome_trace(tmp)
ev = json.load(open(tmp))["traceEvents"]
ker = sorted([(e["ts"], e["ts"] + e["dur"], e["name"], e.get("args", {}).get("stream")) for e in ev
              if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda x: x[0])
# split into calls at idle gaps > 100 us
groups, cur = [], [ker[0]]
for k in ker[1:]:
    if k[0] - max(x[1] for x in cur) > 150:
        groups.append(cur)
        cur = [k]
    else:
        cur.append(k)
groups.append(cur)
for gi, g in enumerate(groups):
    t0, t1 = g[0][0], max(x[1] for x in g)
    busy, end = 0.0, t0
    gaps = []
    for s, e, n, strm in g:
        if s > end:
            gaps.append((s - end, end - t0, n))
        busy += max(0.0, e - max(s, end))
        end = max(end, e)
    gaps.sort(reverse=True)
    names = {}
    for s, e, n, strm in g:
        names[n] = names.get(n, 0) + (e - s)
    print(f"call {gi}: span {t1 - t0:.1f} us, busy (union) {busy:.1f} us = {busy / (t1 - t0):.1%}, "
          f"{len(g)} device ops, streams {len(set(x[3] for x in g))}")
    for gap, at, n in gaps[:8]:
        print(f"   idle {gap:7.1f} us at +{at:8.1f} us before {n[:70]}")
top = sorted(names.items(), key=lambda kv: -kv[1])[:12]
print("last call, device time by op (summed over streams):")
for n, t in top:
    print(f"   {t:8.1f} us  {n[:100]}")
dump = [a for a in sys.argv if a.startswith("--dump=")]
if dump:
    g = groups[-1]
    t0 = g[0][0]
    with open(dump[0].split("=", 1)[1], "w") as f:
        f.write("start_us,dur_us,stream,name\n")
        for s, e, n, strm in g:
            f.write(f"{s - t0:.1f},{e - s:.1f},{strm},\"{n[:90]}\"\n")
