import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2211_00696_b200 as pq
from paper_2211_00696_b200.workloads import allen_cahn_u0, config
w = config(4)
a = pq.KroneckerSum(w.A)
u0 = allen_cahn_u0(w.N)
ctx = pq.default_context()
l0 = ctx.launches
res = pq.integrate(a, ("cubic", 1.0, -1.0), u0, 0.0, 20 * w.tau, 20, pq.etdrk4_tableau(), pq.PhiRequest(eps=w.eps))
print("launches counted for 20 steps:", ctx.launches - l0)
