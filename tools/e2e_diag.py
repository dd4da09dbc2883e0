import ctypes as C, threading, time, json, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2211_00696_b200 as pq
from paper_2211_00696_b200.workloads import config
w = config(2); a = pq.KroneckerSum(w.factors); req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
d, sh, fac = a._abi(); rc = req._c(); N = w.N
pr = torch.cuda.Stream.priority_range(); lo, hi = max(pr), min(pr)
print("priority range", pr)
def make(prio):
    cx = pq.Context(0); st = torch.cuda.Stream(priority=prio); cx.set_stream(st.cuda_stream)
    bufs = (torch.from_numpy(w.rhs(1)).pin_memory(), torch.empty((1, N), dtype=torch.float64).pin_memory(),
            torch.empty((1, w.p, N), dtype=torch.float64).pin_memory())
    return cx, st, bufs
def call(cx, bufs):
    inf = pq._lib.PhiInfoC()
    pq._lib.check(pq._lib.lib.pq_phi_0p(cx.handle, d, sh, fac, 1, C.c_void_p(bufs[0].data_ptr()), C.byref(rc),
        C.c_void_p(bufs[1].data_ptr()), C.c_void_p(bufs[2].data_ptr()), C.byref(inf), pq._lib.PQ_HOST))
NC = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prios = [hi + (lo - hi) * k // max(1, NC - 1) for k in range(NC)] if sys.argv[2:3] != ['same'] else [0] * NC
callers = [make(pp) for pp in prios]
print('callers', NC, 'priorities', prios)
for cx, st, b in callers: call(cx, b); call(cx, b)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(6): call(*[callers[0][0], callers[0][2]])
print("single caller ms/call", (time.perf_counter() - t0) / 6 * 1e3)
log = [[] for _ in range(NC)]
def worker(i):
    cx, st, b = callers[i]
    for _ in range(6):
        s = time.perf_counter(); call(cx, b); log[i].append((s - T0, time.perf_counter() - T0))
T0 = time.perf_counter()
ths = [threading.Thread(target=worker, args=(i,)) for i in range(NC)]
[t.start() for t in ths]; [t.join() for t in ths]
tot = time.perf_counter() - T0
print(NC, "callers: total ms", tot * 1e3, "per action", tot / (6 * NC) * 1e3)
for i in range(NC): print(i, " ".join(f"[{s*1e3:.1f},{e*1e3:.1f}]" for s, e in log[i]))

# device-resident calls from the same callers (no PCIe): does concurrency cost device throughput?
def make_dev():
    return (torch.from_numpy(w.rhs(1)).cuda(), torch.empty((1, N), dtype=torch.float64, device="cuda"),
            torch.empty((1, w.p, N), dtype=torch.float64, device="cuda"))
dbufs = [make_dev() for _ in range(NC)]
def call_dev(cx, bufs):
    inf = pq._lib.PhiInfoC()
    pq._lib.check(pq._lib.lib.pq_phi_0p(cx.handle, d, sh, fac, 1, C.c_void_p(bufs[0].data_ptr()), C.byref(rc),
        C.c_void_p(bufs[1].data_ptr()), C.c_void_p(bufs[2].data_ptr()), C.byref(inf), pq._lib.PQ_DEVICE))
def dworker(i):
    cx, st, _ = callers[i]
    for _ in range(6):
        call_dev(cx, dbufs[i])
    cx.synchronize()
torch.cuda.synchronize()
T0 = time.perf_counter()
for _ in range(6): call_dev(callers[0][0], dbufs[0])
callers[0][0].synchronize()
print("device-resident single caller ms/call", (time.perf_counter() - T0) / 6 * 1e3)
T0 = time.perf_counter()
ths = [threading.Thread(target=dworker, args=(i,)) for i in range(NC)]
[t.start() for t in ths]; [t.join() for t in ths]
print(NC, "device-resident callers: per action ms", (time.perf_counter() - T0) / (6 * NC) * 1e3)
