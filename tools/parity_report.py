#!/usr/bin/env python
"""Parity margins against the committed reference fixtures (tests/golden/ref_phi_cases.npz):
max relative 2-norm error per case, one JSON object on stdout.  Run it twice to compare the
exponential paths:  PQ_EXPM=pade python tools/parity_report.py   (Pade-13 + LU, dense.hpp)
                    python tools/parity_report.py                (shared-power Taylor, default)
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def rel2(a, b):
    a, b = np.asarray(a, dtype=np.float64).ravel(), np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def split(flat, shape):
    fs, off = [], 0
    for s in shape:
        fs.append(flat[off:off + s * s].reshape(s, s))
        off += s * s
    return fs


def main():
    import paper_2211_00696_b200 as pq
    from paper_2211_00696_b200.workloads import config, fd_laplacian

    C = np.load(ROOT / "tests" / "golden" / "ref_phi_cases.npz")
    out = {"expm_path": os.environ.get("PQ_EXPM", "taylor")}
    fs = split(C["lap3_factors"], [int(s) for s in C["lap3_shape"]])
    for kind, l, n in [(0, 0, 12), (0, 3, 9), (1, 0, 0), (1, 2, 0)]:
        got = pq.phi_with_plan(pq.KroneckerSum(fs), [C["lap3_b"]], 4, l, n, pq.QuadKind(kind), 1e-12)[0]
        want = C[f"plan_k{kind}_l{l}_n{n}"]
        out[f"plan_k{kind}_l{l}_n{n}"] = max(rel2(got.col(j + 1), want[j]) for j in range(4))
    w = config(2, n=12)
    phi0, cols = pq.phi_0p(pq.KroneckerSum(w.factors), [w.rhs(0)],
                           pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode)))
    out["cfg2n12_phi0"] = rel2(phi0[0], C["cfg2n12_phi0"])
    out["cfg2n12_phi"] = max(rel2(cols[0, j], C["cfg2n12_phi"][j]) for j in range(w.p))
    a = pq.KroneckerSum(split(C["asym_factors"], [2, 3, 4]))
    out["asym_exp_action"] = rel2(pq.exp_action(a, C["asym_x"]), C["asym_exp_action"])
    lap = [0.01 * fd_laplacian(6, 1.0 / 7.0)] * 3
    tabs = [pq.exp_euler_tableau(), pq.exp_rk2_tableau(), pq.exp_rk3_tableau(), pq.etdrk4_tableau()]
    for t, tab in enumerate(tabs):
        res = pq.integrate(pq.KroneckerSum(lap), ("cubic", 1.0, -1.0), C["etd_u0"], 0.0, 0.01, 5, tab,
                           pq.PhiRequest(eps=1e-14))
        out[f"etd_tab{t}"] = rel2(res.u, C[f"etd_tab{t}_u"])
    # a mid-size headline-family case: phi columns of config 2 at n = 32 (device result only)
    w = config(2, n=32)
    _, cols = pq.phi_0p(pq.KroneckerSum(w.factors), [w.rhs(1)],
                        pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode)))
    if os.environ.get("PQ_PARITY_DUMP"):
        np.save(os.environ["PQ_PARITY_DUMP"], cols[0])
    out["max"] = max(v for k, v in out.items() if isinstance(v, float))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
