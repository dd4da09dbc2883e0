"""Parity at the shapes the BASELINE configs actually run (VERDICT r01 "next round" item 1),
against the compiled reference (oracle/_ref) on identical seeded inputs and identical (l, n):

* config 3's batch of 8 right-hand sides at n = 64 with the reference's own plan (live reference);
* config 3 at full size (n = 256, 16.8 M DOF, one RHS) at its real plan (7, 9), phi_0..phi_3;
* config 5 at full size (n = 512, 134 M DOF): the 13-node Gauss phase plus ONE squaring step at
  pinned (l, n) = (1, 12), p = 6;
* config 4 (Allen-Cahn ETDRK4) at full n = 128 for 2 steps.

The full-size reference outputs were computed once on CPU by tests/golden/make_fullsize_sketches.py
(minutes to an hour of reference time each) and are stored as fingerprints (tests/sketch.py): the
norm, a 16-row sign sketch and 4096 seeded samples per column.  Bar: 1e-11 relative (north_star) on
the sketch estimate of ||ours - ref|| / ||ref|| and on the sampled entries.  Margins are appended to
$PQ_MARGINS_OUT (jsonl) when set (profiles/r02_parity_margins.jsonl).
"""
import json
import os
from pathlib import Path

import numpy as np
import pytest

from conftest import rel2

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
BAR = 1e-11


def _fixture(name):
    meta_p, arr_p = GOLD / f"fullsize_{name}.json", GOLD / f"fullsize_{name}.npz"
    if not meta_p.exists():
        pytest.skip(f"fixture {arr_p.name} not generated (tests/golden/make_fullsize_sketches.py {name})")
    meta = json.loads(meta_p.read_text())
    z = np.load(arr_p)
    keys = sorted({k.split(".")[0] for k in z.files})
    fps = {k: {"norm": float(z[f"{k}.norm"][0]), "sketch": z[f"{k}.sketch"], "samples": z[f"{k}.samples"]}
           for k in keys}
    return meta, fps


def _record(case, margins):
    out = os.environ.get("PQ_MARGINS_OUT")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps({"case": case, **margins}) + "\n")


def _check(case, got_cols, fps, extra=None):
    from sketch import compare, fingerprint
    worst = {}
    for name, vec in got_cols.items():
        m = compare(fingerprint(vec), fps[name])
        worst[name] = m
        assert m["sketch_rel"] <= BAR, (name, m)
        assert m["samples_relinf"] <= BAR, (name, m)
        assert m["norm_rel"] <= BAR, (name, m)
    _record(case, {"columns": worst, **(extra or {})})


def test_config3_eight_rhs_n64_reference_plan(pq, ref):
    """All 8 RHS of config 3 (seeds 1000..1007) at n = 64 through phiquadmv_multi with the plan the
    reference chooses for the batch (beta = max over the 8 ||b||_inf, phiaction.hpp:312-313)."""
    from paper_2211_00696_b200.workloads import config
    w = config(3, n=64)
    bs = np.stack([w.rhs(k) for k in range(8)])
    want, rinfo = ref.phiquadmv(w.factors, bs, w.p, w.eps, w.mode, threads=os.cpu_count() or 1)
    info = pq.PhiInfo()
    got = pq.phiquadmv_multi(pq.KroneckerSum(w.factors), list(bs), pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(0)),
                             info)
    assert (info.l, info.n, info.points) == (rinfo["l"], rinfo["n"], rinfo["points"])
    errs = [rel2(got[m].col(j + 1), want[m, j]) for m in range(8) for j in range(w.p)]
    _record("cfg3_n64_8rhs", {"plan": [info.l, info.n, info.points], "max_rel2": max(errs)})
    assert max(errs) <= BAR, max(errs)


def test_config3_full_size_real_plan(pq):
    """Config 3 at n = 256 (16.8 M DOF), RHS seed 0, phi_0..phi_3 at the reference's own plan."""
    import torch
    from paper_2211_00696_b200.workloads import config
    meta, fps = _fixture("cfg3_full")
    w = config(3)
    b = torch.from_numpy(w.rhs(meta["rhs_seed_index"])).cuda()
    info = pq.PhiInfo()
    phi0, cols = pq.phi_0p(pq.KroneckerSum(w.factors), b.reshape(1, -1),
                           pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(0)), info)
    torch.cuda.synchronize()
    assert [info.l, info.n, info.points] == meta["plan"] == [7, 9, 10]
    got = {f"phi{j + 1}": cols[0, j].cpu().numpy() for j in range(w.p)}
    got["phi0"] = phi0[0].cpu().numpy()
    _check("cfg3_full_plan_7_9", got, fps, {"plan": meta["plan"], "ref_seconds": meta["ref_seconds"]})


def test_config5_full_size_nodes_plus_one_squaring(pq):
    """Config 5 at n = 512 (134 M DOF, 1.07 GB per vector): phi_with_plan at pinned (l, n) = (1, 12)
    -- the 13 Gauss nodes and ONE modified-squaring step -- for phi_1..phi_6."""
    import torch
    from paper_2211_00696_b200.workloads import config
    meta, fps = _fixture("cfg5_l1n12")
    w = config(5)
    b = torch.from_numpy(w.rhs(meta["rhs_seed_index"])).cuda()
    out = pq.phi_with_plan(pq.KroneckerSum(w.factors), b.reshape(1, -1), w.p, 1, 12, pq.QuadKind(0), w.eps)
    torch.cuda.synchronize()
    got = {f"phi{j + 1}": out[0].col(j + 1).cpu().numpy() for j in range(w.p)}
    del out
    _check("cfg5_full_l1_n12", got, fps, {"ref_seconds": meta["ref_seconds"]})


def test_config4_etdrk4_full_size_two_steps(pq):
    """Config 4 at n = 128: two ETDRK4 steps (dt = 1e-3) of Allen-Cahn from the seeded u0."""
    from paper_2211_00696_b200.workloads import allen_cahn_u0, config
    meta, fps = _fixture("cfg4_2steps")
    w = config(4)
    u0 = allen_cahn_u0(w.N)
    res = pq.integrate(pq.KroneckerSum(w.A), ("cubic", 1.0, -1.0), u0, 0.0, 2 * w.tau, 2, pq.etdrk4_tableau(),
                       pq.PhiRequest(eps=w.eps))
    assert res.phi_calls == meta["phi_calls"]
    _check("cfg4_etdrk4_n128_2steps", {"u": np.asarray(res.u)}, fps, {"phi_calls": res.phi_calls})
