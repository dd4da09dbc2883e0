"""Device timeline of the e2e leg (bench.py): K host callers, each with its own context, stream and
pinned buffers, calling pq_phi_0p with PQ_HOST concurrently.  Reports kernel-busy (union of
kernel intervals), D2H/H2D-busy, and their overlap over the whole region (CUPTI via torch.profiler).
Usage: python tools/timeline_e2e.py [callers] [calls_per_caller]"""
import ctypes as C
import json
import sys
import tempfile
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2211_00696_b200 as pq  # noqa: E402
from paper_2211_00696_b200.workloads import config  # noqa: E402

ncall = int(sys.argv[1]) if len(sys.argv) > 1 else 4
per = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = config(2)
a = pq.KroneckerSum(w.factors)
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
d, sh, fac = a._abi()
rc = req._c()
pr = torch.cuda.Stream.priority_range()
lo, hi = max(pr), min(pr)
callers = []
for k in range(ncall):
    st = torch.cuda.Stream(priority=hi + (lo - hi) * k // max(1, ncall - 1))
    cx = pq.Context(0)
    cx.set_stream(st.cuda_stream)
    bs = [torch.from_numpy(w.rhs(500 + 10 * k + i)[None, :].copy()).pin_memory() for i in range(per + 1)]
    o0 = torch.empty((1, w.N), dtype=torch.float64).pin_memory()
    o = torch.empty((1, w.p, w.N), dtype=torch.float64).pin_memory()
    callers.append((cx, bs, o0, o))


def call(cx, b, o0, o):
    inf = pq._lib.PhiInfoC()
    pq._lib.check(pq._lib.lib.pq_phi_0p(cx.handle, d, sh, fac, 1, C.c_void_p(b.data_ptr()), C.byref(rc),
                                        C.c_void_p(o0.data_ptr()), C.c_void_p(o.data_ptr()), C.byref(inf),
                                        pq._lib.PQ_HOST))


for cx, bs, o0, o in callers:
    call(cx, bs[-1], o0, o)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    def worker(i):
        cx, bs, o0, o = callers[i]
        for j in range(per):
            call(cx, bs[j], o0, o)
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(ncall)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
tmp = tempfile.NamedTemporaryFile(suffix=".json", delete=False).name
prof.export_chrome_trace(tmp)
ev = json.load(open(tmp))["traceEvents"]


def union(iv):
    iv = sorted(iv)
    tot, end = 0.0, None
    out = []
    for s, e in iv:
        if end is None or s > end:
            out.append([s, e])
            end = e
        else:
            out[-1][1] = max(out[-1][1], e)
            end = out[-1][1]
    return out


ker = [(e["ts"], e["ts"] + e["dur"]) for e in ev if e.get("cat") == "kernel"]
d2h = [(e["ts"], e["ts"] + e["dur"]) for e in ev if e.get("cat") == "gpu_memcpy" and "DtoH" in e["name"]]
h2d = [(e["ts"], e["ts"] + e["dur"]) for e in ev if e.get("cat") == "gpu_memcpy" and "HtoD" in e["name"]]
t0 = min(s for s, _ in ker + d2h + h2d)
t1 = max(e for _, e in ker + d2h + h2d)
span = t1 - t0
uk, ud, uh = union(ker), union(d2h), union(h2d)
kb = sum(e - s for s, e in uk)
db = sum(e - s for s, e in ud)
hb = sum(e - s for s, e in uh)
# time when NO kernel runs but a D2H does
idle_k = []
end = t0
for s, e in uk:
    if s > end:
        idle_k.append((end, s))
    end = max(end, e)
if t1 > end:
    idle_k.append((end, t1))
d2h_in_idle = sum(max(0.0, min(e, ie) - max(s, is_)) for is_, ie in idle_k for s, e in ud)
print(f"{ncall} callers x {per} calls: span {span / 1e3:.2f} ms = {span / (ncall * per) / 1e3:.3f} ms per call "
      f"({ncall * per / (span / 1e6):.1f} calls/s)")
print(f"kernel-busy {kb / span:.1%}, D2H-busy {db / span:.1%}, H2D-busy {hb / span:.1%}; no-kernel time "
      f"{(span - kb) / 1e3:.2f} ms, of which a D2H runs {d2h_in_idle / 1e3:.2f} ms")
gaps = sorted(((e - s), s - t0) for s, e in idle_k)[::-1][:10]
for g, at in gaps:
    print(f"   no kernel for {g:8.1f} us at +{at / 1e3:8.3f} ms")
print("D2H bytes/s while active: ", end="")
tot_bytes = sum(e.get("args", {}).get("bytes", 0) for e in ev if e.get("cat") == "gpu_memcpy" and "DtoH" in e["name"])
print(f"{tot_bytes / (db / 1e6) / 1e9:.1f} GB/s over {tot_bytes / 1e6:.0f} MB")

if "--streams" in sys.argv:  # per stream: kernel busy windows and copies, in ms from the start
    by = {}
    for e in ev:
        if e.get("cat") in ("kernel", "gpu_memcpy"):
            by.setdefault(e["args"].get("stream"), []).append(e)
    rows = []
    for sid, es in by.items():
        es.sort(key=lambda e: e["ts"])
        seg = None
        for e in es:
            kind = "K" if e["cat"] == "kernel" else ("D2H" if "DtoH" in e["name"] else "H2D" if "HtoD" in e["name"] else "D2D")
            if kind != "K" and e["args"].get("bytes", 1 << 30) < (1 << 20):
                kind += "(%s %dB)" % ("pageable" if "Pageable" in e["name"] else "pinned", e["args"]["bytes"])
            s, f = (e["ts"] - t0) / 1e3, (e["ts"] + e["dur"] - t0) / 1e3
            if seg and seg[0] == kind and s - seg[2] < 0.05:
                seg[2] = f
            else:
                if seg:
                    rows.append((seg[1], sid, *seg))
                seg = [kind, s, f]
        rows.append((seg[1], sid, *seg))
    for _, sid, kind, s, f in sorted(rows):
        if kind != "K" or f - s > 0.05:
            print(f"  stream {sid:>4} {kind:>24} {s:8.3f} .. {f:8.3f}")
