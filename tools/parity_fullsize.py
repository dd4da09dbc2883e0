#!/usr/bin/env python
"""Full-size parity margins against the compiled reference (oracle/_ref) on this box's cores:
configs 1 and 2 at full size and config 5 at n = 96 through phiquadmv, and config 3 at full size
(one RHS) through phi_with_plan at pinned (l, n) = (1, 9); prints one JSON object per case (plan
equality, max relative 2-norm error over phi_1..phi_p, phi_0 error, GPU and CPU times)."""
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
    for cfg, n in [(1, None), (2, None), (5, 96)]:
        w = config(cfg, n=n)
        a = pq.KroneckerSum(w.factors)
        b = w.rhs(0)
        info = pq.PhiInfo()
        t0 = time.perf_counter()
        phi0, cols = pq.phi_0p(a, [b], pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode)), info)
        t_gpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        want, rinfo = ref.phiquadmv(w.factors, b[None, :], w.p, w.eps, w.mode, threads=threads)
        want0 = ref.exp_action(w.factors, b)
        t_cpu = time.perf_counter() - t0
        print(json.dumps({
            "workload": w.name, "N": int(w.N), "plan_gpu": [info.l, info.n, info.points],
            "plan_ref": [rinfo["l"], rinfo["n"], rinfo["points"]],
            "max_rel2_phi_j": max(rel2(cols[0, j], want[0][j]) for j in range(w.p)),
            "rel2_phi0": rel2(phi0[0], want0), "gpu_call_s_incl_first_call": t_gpu,
            "reference_s": t_cpu, "reference_threads": threads}), flush=True)
    w = config(3)
    b = w.rhs(0)
    t0 = time.perf_counter()
    got = pq.phi_with_plan(pq.KroneckerSum(w.factors), [b], w.p, 1, 9, pq.QuadKind.gauss_legendre, w.eps)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    want, _ = ref.phi_with_plan(w.factors, b[None, :], w.p, 1, 9, 0, w.eps, threads=threads)
    t_cpu = time.perf_counter() - t0
    print(json.dumps({
        "workload": w.name + " (1 RHS, phi_with_plan l=1 n=9)", "N": int(w.N),
        "max_rel2_phi_j": max(rel2(np.asarray(got[0].col(j + 1)), want[0][j]) for j in range(w.p)),
        "gpu_call_s_incl_first_call": t_gpu, "reference_s": t_cpu, "reference_threads": threads}), flush=True)


if __name__ == "__main__":
    main()
