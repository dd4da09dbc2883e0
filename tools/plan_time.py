import sys, time, ctypes as C
sys.path.insert(0,'/root/repo')
import paper_2211_00696_b200 as pq
from paper_2211_00696_b200 import _lib as L
from paper_2211_00696_b200.workloads import config
for cfg in (1,2,3,5):
    w = config(cfg)
    alpha = pq.infnorm_bound(pq.KroneckerSum(w.factors))
    l, n, cost = C.c_int(), C.c_int(), C.c_double()
    t0=time.perf_counter()
    for k in range(30):
        beta = 4.0 + 0.0137*k
        L.check(L.lib.pq_setup_quadrature(w.eps, w.p, alpha, beta, w.mode, 0.0, 1.0, w.d, C.byref(l), C.byref(n), C.byref(cost)))
    print("cfg", cfg, "alpha %.1f" % alpha, "fresh beta: %.1f us" % ((time.perf_counter()-t0)/30*1e6), l.value, n.value)
