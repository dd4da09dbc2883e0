import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2211_00696_b200 as pq
from paper_2211_00696_b200.workloads import allen_cahn_u0, config
w = config(4)
a = pq.KroneckerSum(w.A)
u0 = allen_cahn_u0(w.N)
tab = pq.etdrk4_tableau()
req = pq.PhiRequest(eps=w.eps)
res = pq.integrate(a, ("cubic", 1.0, -1.0), u0, 0.0, 2 * w.tau, 2, tab, req)  # warm
t0 = time.perf_counter()
res = pq.integrate(a, ("cubic", 1.0, -1.0), u0, 0.0, 20 * w.tau, 20, tab, req)
dt = time.perf_counter() - t0
print(f"config 4 ETDRK4 n={w.n}: 20 steps in {dt*1e3:.1f} ms = {dt/20*1e3:.2f} ms/step, phi calls {res.phi_calls}, |u|={np.linalg.norm(res.u):.12e}")
