#!/usr/bin/env python
"""Regenerates tests/golden/ref_golden.json and ref_phi_cases.npz from the COMPILED REFERENCE
(oracle/_ref/libpqref.so = the unmodified reference headers behind our flat shim).  Run in the dev
container, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Floats are stored as float.hex strings (bit-exact).  The fixtures let the CPU test suite pin the
numpy oracle and the product's host estimator, and let the GPU tests check parity, on machines
where the reference itself is absent (the GPU box).
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle.ref import Ref  # noqa: E402
from paper_2211_00696_b200.workloads import config, fd_laplacian  # noqa: E402


def hx(v):
    return [float(x).hex() for x in np.asarray(v, dtype=np.float64).reshape(-1)]


def main():
    ref = Ref()
    out = {"source": "oracle/_ref/libpqref.so (reference headers proj/include/phiquad, compiled -O3)"}

    # quadrature.hpp:31-86
    out["rules"] = []
    for kind, ms in ((0, [1, 2, 3, 4, 5, 8, 9, 10, 13, 16, 37, 40]), (1, [2, 3, 5, 7, 13, 25, 49, 97])):
        for m in ms:
            x, w = ref.rule(kind, m)
            out["rules"].append({"kind": kind, "m": m, "nodes": hx(x), "weights": hx(w)})

    # bounds.hpp / roots.hpp: a seeded grid of estimator queries
    rng = np.random.default_rng(2211)
    q = []
    for _ in range(60):
        kind = int(rng.integers(0, 2))
        p = int(rng.integers(1, 21))
        alpha = float(10 ** rng.uniform(-1, 3.5))
        beta = float(10 ** rng.uniform(-1, 1))
        eps = float(10 ** rng.uniform(-14, -6))
        n = float(rng.integers(2, 60))
        rec = {"kind": kind, "p": p, "alpha": alpha.hex(), "beta": beta.hex(), "eps": eps.hex(), "n": n.hex(),
               "quaderr": ref.quaderr(n, p, alpha, beta, kind).hex(),
               "quadnodes": ref.quadnodes(eps, p, alpha, beta, kind)}
        for d in (1, 3):
            l, nn, c = ref.setup_quadrature(eps, p, alpha, beta, kind, 0.0, 1.0, d)
            rec[f"plan_d{d}"] = [l, nn, c.hex()]
        q.append(rec)
    out["estimator"] = q

    # the BASELINE configurations' plans (alpha = infnorm_bound of -tau A, beta = ||b||_inf)
    plans = []
    for idx in (1, 2, 3, 5):
        w = config(idx)
        alpha = ref.infnorm_bound(w.factors)
        beta = float(np.max(np.abs(w.rhs(0))))
        l, n, c = ref.setup_quadrature(w.eps, w.p, alpha, beta, w.mode, 0.0, 1.0, w.d)
        plans.append({"config": idx, "alpha": alpha.hex(), "beta": beta.hex(), "l": l, "n": n, "cost": c.hex()})
    out["baseline_plans"] = plans

    # quartic_roots / real_roots_greater_one on seeded stationarity quartics
    qs = []
    for _ in range(40):
        kind = int(rng.integers(0, 2))
        c4 = ref.bound_quartic(float(rng.integers(2, 80)), int(rng.integers(0, 20)), float(10 ** rng.uniform(-1, 4)),
                               1.0, kind)
        qs.append({"coeffs": hx(c4), "real_gt1": hx(ref.real_roots_greater_one(*c4))})
    out["quartics"] = qs

    # dense.hpp:194 expm on seeded matrices
    ex = []
    for n, sc in ((1, 3.0), (4, 0.3), (7, 2.0), (12, 9.0), (16, 40.0)):
        a = np.random.default_rng(100 + n).uniform(-sc, sc, (n, n))
        ex.append({"n": n, "a": hx(a), "expm": hx(ref.expm(a))})
    out["expm"] = ex
    (HERE / "ref_golden.json").write_text(json.dumps(out, indent=1))

    # phi pipeline cases (phi_with_plan / phiquadmv / exp_action / lincomb / integrate)
    cases = {}
    rng = np.random.default_rng(7)
    lap = [-2e-3 * fd_laplacian(n, 1.0 / (n + 1)) for n in (12, 10, 9)]
    b3 = rng.standard_normal(12 * 10 * 9)
    for kind, l, n in ((0, 0, 12), (0, 3, 9), (1, 0, 0), (1, 2, 0)):
        y, pts = ref.phi_with_plan(lap, b3, 4, l, n, kind, 1e-12)
        cases[f"plan_k{kind}_l{l}_n{n}"] = y[0]
        cases[f"plan_k{kind}_l{l}_n{n}_points"] = np.array([pts])
    cases["lap3_factors"] = np.concatenate([f.reshape(-1) for f in lap])
    cases["lap3_shape"] = np.array([12, 10, 9])
    cases["lap3_b"] = b3
    w = config(2, n=12)
    b2 = w.rhs(0)
    y, info = ref.phiquadmv(w.factors, b2, w.p, w.eps, w.mode)
    cases["cfg2n12_phi"] = y[0]
    cases["cfg2n12_phi0"] = ref.exp_action(w.factors, b2)
    cases["cfg2n12_plan"] = np.array([info["l"], info["n"], info["points"]])
    asym = [rng.uniform(-0.5, 0.5, (n, n)) for n in (2, 3, 4)]
    xa = rng.standard_normal(24)
    cases["asym_factors"] = np.concatenate([f.reshape(-1) for f in asym])
    cases["asym_x"] = xa
    cases["asym_mode_apply"] = ref.mode_apply(asym, xa)
    cases["asym_kron_matvec"] = ref.kron_matvec(asym, xa)
    cases["asym_exp_action"] = ref.exp_action(asym, xa)
    cases["asym_dense_phi3"] = ref.phi_dense_oracle(asym, xa, 3)
    ac = [0.01 * fd_laplacian(6, 1.0 / 7.0)] * 3
    u0 = np.random.default_rng(2024).uniform(-0.9, 0.9, 216)
    for tab in (0, 1, 2, 3):
        u, calls = ref.integrate(ac, 1, u0, 0.0, 0.01, 5, tab, eps=1e-14)
        cases[f"etd_tab{tab}_u"] = u
        cases[f"etd_tab{tab}_calls"] = np.array([calls])
    cases["etd_u0"] = u0
    np.savez_compressed(HERE / "ref_phi_cases.npz", **cases)
    print("wrote", HERE / "ref_golden.json", HERE / "ref_phi_cases.npz")


if __name__ == "__main__":
    main()
