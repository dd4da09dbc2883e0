"""Do PCIe copies slow the device-resident phi calls? NC device-resident config-2 callers run while a
copier thread streams the transfers of one call (17 MB H2D + 84 MB D2H, pinned) back to back on its
own stream; prints both rates next to the rates each reaches alone."""
import ctypes as C
import json
import sys
import threading
import time

import torch

sys.path.insert(0, "/root/repo")
import paper_2211_00696_b200 as pq
from paper_2211_00696_b200.workloads import config

w = config(2)
a = pq.KroneckerSum(w.factors)
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
d, sh, fac = a._abi()
rc = req._c()
N = w.N
NC = int(sys.argv[1]) if len(sys.argv) > 1 else 4
DIR = sys.argv[2] if len(sys.argv) > 2 else "both"  # both | h2d | d2h
REPS = 8


def make():
    cx = pq.Context(0)
    st = torch.cuda.Stream()
    cx.set_stream(st.cuda_stream)
    return cx, (torch.from_numpy(w.rhs(1)).cuda(), torch.empty((1, N), dtype=torch.float64, device="cuda"),
                torch.empty((1, w.p, N), dtype=torch.float64, device="cuda"))


def call_dev(cx, bufs):
    inf = pq._lib.PhiInfoC()
    pq._lib.check(pq._lib.lib.pq_phi_0p(cx.handle, d, sh, fac, 1, C.c_void_p(bufs[0].data_ptr()), C.byref(rc),
                                        C.c_void_p(bufs[1].data_ptr()), C.c_void_p(bufs[2].data_ptr()),
                                        C.byref(inf), pq._lib.PQ_DEVICE))


callers = [make() for _ in range(NC)]
for cx, b in callers:
    call_dev(cx, b)
    cx.synchronize()
cst = torch.cuda.Stream()
hb = torch.empty(N, dtype=torch.float64).pin_memory()
ho = torch.empty(5 * N, dtype=torch.float64).pin_memory()
db = torch.empty_like(hb, device="cuda")
do = torch.empty_like(ho, device="cuda")
stop = threading.Event()
ncopy = [0]


def copier():
    while not stop.is_set():
        with torch.cuda.stream(cst):
            if DIR in ("both", "h2d"):
                db.copy_(hb, non_blocking=True)
                if DIR == "h2d":
                    do.copy_(ho, non_blocking=True)
            if DIR in ("both", "d2h"):
                ho.copy_(do, non_blocking=True)
        cst.synchronize()
        ncopy[0] += 1


def worker(i):
    cx, b = callers[i]
    for _ in range(REPS):
        call_dev(cx, b)
    cx.synchronize()


def run_compute():
    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(NC)]
    [t.start() for t in ths]
    [t.join() for t in ths]
    return NC * REPS / (time.perf_counter() - t0)


alone = run_compute()
t0 = time.perf_counter()
th = threading.Thread(target=copier)
th.start()
time.sleep(0.05)
n0 = ncopy[0]
t1 = time.perf_counter()
with_copies = run_compute()
t2 = time.perf_counter()
n1 = ncopy[0]
stop.set()
th.join()
print(json.dumps({"callers": NC, "copies": DIR, "device_actions_per_s_alone": alone, "device_actions_per_s_with_copier": with_copies,
                  "copier_actions_per_s_during": (n1 - n0) / (t2 - t1)}))
