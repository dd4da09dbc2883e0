"""TEST INFRASTRUCTURE (run by tests/test_gpu_guards.py with PQ_WS_GUARD=1): every engine path at
small, odd shapes with canary-guarded workspace buffers (4 KB before and after each).  After every
call the canaries are checked (an out-of-bounds write into or out of any workspace buffer shows up
as a damaged guard) and each call runs three times with bitwise-equal results required (a shared-
memory or cross-stream race shows up as run-to-run differences).  The substitute for
compute-sanitizer memcheck / racecheck, which is closed on this GPU pool.  Prints one JSON line."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import paper_2211_00696_b200 as pq
    from paper_2211_00696_b200 import sharded as S
    from paper_2211_00696_b200.workloads import allen_cahn_u0, config

    ctx = pq.Context(0)
    rng = np.random.default_rng(11)

    def adv(shape, scale):
        fs = []
        for k, n in enumerate(shape):
            h = 1.0 / (n + 1)
            lap = (2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)) / h**2
            advm = (np.eye(n, k=1) - np.eye(n, k=-1)) / (2 * h)
            fs.append(-scale * ((1.0, 0.5, 0.2)[k % 3] * lap + (8.0, -3.0, 1.0)[k % 3] * advm))
        return pq.KroneckerSum(fs)

    cases = []
    w2 = config(2, n=24)
    a2 = pq.KroneckerSum(w2.factors)
    b2 = w2.rhs(0)
    cases.append(("cc_phi0p_n24", lambda: pq.phi_0p(a2, [b2], pq.PhiRequest(p=4, eps=1e-10, mode=pq.QuadKind(1)),
                                                      ctx=ctx)))
    w3 = config(3, n=20)
    a3 = pq.KroneckerSum(w3.factors)
    b3 = np.stack([w3.rhs(k) for k in range(3)])
    cases.append(("gauss_3rhs_n20", lambda: pq.phi_0p(a3, list(b3), pq.PhiRequest(p=3, eps=1e-10), ctx=ctx)))
    a_odd = adv((17, 23, 9), 3e-3)
    b_odd = rng.standard_normal(a_odd.dim())
    cases.append(("odd_shape_cc_p9", lambda: pq.phiquadmv(a_odd, b_odd, pq.PhiRequest(p=9, eps=1e-10,
                                                                                         mode=pq.QuadKind(1)), ctx=ctx)))
    a_big = adv((72, 65, 64), 2e-3)  # N >= 2^18: band tiles, two-stream squaring, side-stream exponentials
    b_big = rng.standard_normal(a_big.dim())
    cases.append(("band_two_stream_cc", lambda: pq.phi_0p(a_big, [b_big], pq.PhiRequest(p=4, eps=1e-10,
                                                                                            mode=pq.QuadKind(1)),
                                                            ctx=ctx)))
    cases.append(("band_gauss_pinned_l", lambda: pq.phi_with_plan(a_big, [b_big], 3, 4, 9, pq.QuadKind(0), 1e-10,
                                                                   ctx=ctx)))
    m = rng.uniform(-0.3, 0.3, (37, 37))
    cases.append(("expm_pade_batch", lambda: pq.expm(m, scale=[0.5, 2.0, 7.0], ctx=ctx)))
    cases.append(("kron_matvec", lambda: pq.kron_matvec(a_odd, b_odd, ctx=ctx)))
    cases.append(("phi_lincomb", lambda: pq.phi_lincomb(a_odd, [b_odd, 2 * b_odd, -b_odd],
                                                        pq.cached_rule(pq.QuadKind(0), 9), ctx=ctx)))
    w4 = config(4, n=16)
    u0 = allen_cahn_u0(w4.N)
    cases.append(("etdrk4_n16", lambda: pq.integrate(pq.KroneckerSum(w4.A), ("cubic", 1.0, -1.0), u0, 0.0,
                                                     3 * w4.tau, 3, pq.etdrk4_tableau(), pq.PhiRequest(eps=1e-14),
                                                     ctx=ctx).u))
    comm = S.Communicator.single()
    cases.append(("dist_world1_cc", lambda: S.phiquadmv_dist(a2, b2[None, :], pq.PhiRequest(p=4, eps=1e-10,
                                                                                             mode=pq.QuadKind(1)),
                                                             comm, ctx=ctx, phi0=True)))
    cases.append(("dist_world1_gauss", lambda: S.phi_with_plan_dist(a3, b3, 3, 2, 7, pq.QuadKind(0), 1e-10, comm,
                                                                    ctx=ctx)))

    def flat(r):
        if isinstance(r, tuple):
            return np.concatenate([flat(x) for x in r])
        if isinstance(r, list):
            return np.concatenate([flat(x) for x in r]) if r else np.zeros(0)
        if hasattr(r, "cols"):
            return np.concatenate([np.asarray(c).reshape(-1) for c in r.cols])
        if hasattr(r, "cpu"):
            return r.cpu().numpy().reshape(-1)
        return np.asarray(r, dtype=np.float64).reshape(-1)

    report = {}
    for name, fn in cases:
        runs = [flat(fn()) for _ in range(3)]
        ctx.synchronize()
        damaged, names = ctx.check_guards()
        report[name] = {"damaged": damaged, "names": names, "bitwise_repeat": all(np.array_equal(runs[0], r)
                                                                                  for r in runs[1:]),
                        "finite": bool(np.all(np.isfinite(runs[0])))}
    comm.close()
    print(json.dumps(report))


if __name__ == "__main__":
    main()
