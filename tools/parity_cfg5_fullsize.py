#!/usr/bin/env python
"""Config 5 at FULL size (n = 512, N = 134 M DOF, 1.07 GB per vector) against the compiled
reference, node phase only: phi_with_plan at pinned (l, n) = (0, 12), Gauss (13 nodes, p = 6) --
the reference needs one ~9-minute wave of 13 exp-actions on 16 threads; adding even one squaring
step would add 6 serial exp-actions (~50 min).  SURVEY 8(d) parity plan, config 5.  One JSON line."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import paper_2211_00696_b200 as pq
    from conftest import rel2
    from oracle.ref import Ref
    from paper_2211_00696_b200.workloads import config
    ref = Ref()
    threads = os.cpu_count() or 1
    w = config(5)
    b = w.rhs(0)
    t0 = time.perf_counter()
    got = pq.phi_with_plan(pq.KroneckerSum(w.factors), [b], w.p, 0, 12, pq.QuadKind.gauss_legendre, w.eps)
    cols = [np.asarray(got[0].col(j + 1)) for j in range(w.p)]
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    want, _ = ref.phi_with_plan(w.factors, b[None, :], w.p, 0, 12, 0, w.eps, threads=threads)
    t_cpu = time.perf_counter() - t0
    errs = [rel2(cols[j], want[0][j]) for j in range(w.p)]
    print(json.dumps({"workload": w.name + " (node phase: phi_with_plan l=0 n=12, 13 GL nodes)", "N": int(w.N),
                      "rel2_per_phi_j": errs, "max_rel2_phi_j": max(errs), "gpu_call_s_incl_first_call": t_gpu,
                      "reference_s": t_cpu, "reference_threads": threads}), flush=True)


if __name__ == "__main__":
    main()
