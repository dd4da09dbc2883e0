#!/usr/bin/env python
"""Full-size parity fixtures from the COMPILED REFERENCE (oracle/_ref/libpqref.so, the unmodified
reference headers): runs the reference's own CPU path once, here, on BASELINE-size inputs and
stores size-independent fingerprints of its outputs (tests/sketch.py) under tests/golden/.
tests/test_gpu_fullsize_sketch.py compares the B200 engine against them on the same seeded
inputs and the same (l, n).  Usage (dev container, /root/reference present; ~1 h on 8 cores):

    make -C oracle && python tests/golden/make_fullsize_sketches.py [case ...]

Cases (SURVEY 8(d) parity plan / VERDICT r01 "next round" item 1):
  cfg3_full      config 3 at n = 256 (16.8 M DOF), RHS seed 0, phiquadmv with the reference's own
                 plan (expected (l, n) = (7, 9)) + exp_action (phi_0)
  cfg5_l1n12     config 5 at n = 512 (134 M DOF), RHS seed 0, phi_with_plan at pinned (l, n) =
                 (1, 12): the 13-node Gauss phase plus ONE modified-squaring step, p = 6
  cfg4_2steps    config 4 (Allen-Cahn, n = 128) ETDRK4, 2 steps of dt = 1e-3 (reference integrate
                 with the ETDRK4 ExpRKTableau)
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.ref import Ref  # noqa: E402
from sketch import fingerprint  # noqa: E402
from paper_2211_00696_b200.workloads import allen_cahn_u0, config  # noqa: E402

THREADS = os.cpu_count() or 1


def save(name, meta, fps):
    arr = {}
    for k, fp in fps.items():
        arr[f"{k}.norm"] = np.array([fp["norm"]])
        arr[f"{k}.sketch"] = fp["sketch"]
        arr[f"{k}.samples"] = fp["samples"]
    np.savez_compressed(HERE / f"fullsize_{name}.npz", **arr)
    (HERE / f"fullsize_{name}.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(name, json.dumps(meta), flush=True)


def cfg3_full(ref):
    w = config(3)
    b = w.rhs(0)
    t0 = time.time()
    out, info = ref.phiquadmv(w.factors, b[None, :], w.p, w.eps, w.mode, threads=THREADS)
    phi0 = ref.exp_action(w.factors, b)
    fps = {f"phi{j + 1}": fingerprint(out[0, j]) for j in range(w.p)}
    fps["phi0"] = fingerprint(phi0)
    save("cfg3_full", {"config": 3, "n": w.n, "rhs_seed_index": 0, "p": w.p, "eps": w.eps, "rule": "gauss",
                       "plan": [info["l"], info["n"], info["points"]], "ref_seconds": time.time() - t0,
                       "threads": THREADS, "call": "phiquadmv + exp_action"}, fps)


def cfg5_l1n12(ref):
    w = config(5)
    b = w.rhs(0)
    t0 = time.time()
    out, pts = ref.phi_with_plan(w.factors, b[None, :], w.p, 1, 12, 0, w.eps, threads=THREADS)
    fps = {f"phi{j + 1}": fingerprint(out[0, j]) for j in range(w.p)}
    save("cfg5_l1n12", {"config": 5, "n": w.n, "rhs_seed_index": 0, "p": w.p, "eps": w.eps, "rule": "gauss",
                        "l": 1, "n_param": 12, "points": pts, "ref_seconds": time.time() - t0, "threads": THREADS,
                        "call": "phi_with_plan(l=1, n=12)"}, fps)


def cfg4_2steps(ref):
    w = config(4)
    u0 = allen_cahn_u0(w.N)
    t0 = time.time()
    u, calls = ref.integrate(w.A, 1, u0, 0.0, 2 * w.tau, 2, 3, eps=w.eps, threads=THREADS)
    save("cfg4_2steps", {"config": 4, "n": w.n, "u0_seed": 2024, "steps": 2, "dt": w.tau, "eps": w.eps,
                         "phi_calls": calls, "ref_seconds": time.time() - t0, "threads": THREADS,
                         "call": "integrate(ETDRK4, f = u - u^3)"}, {"u": fingerprint(u)})


CASES = {"cfg4_2steps": cfg4_2steps, "cfg3_full": cfg3_full, "cfg5_l1n12": cfg5_l1n12}

if __name__ == "__main__":
    ref = Ref()
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name](ref)
