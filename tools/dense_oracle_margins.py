#!/usr/bin/env python
"""Margins of the engine against the GPU dense phi oracle (tests/test_gpu_dense_oracle.py)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import paper_2211_00696_b200 as pq
    from conftest import rel2
    from test_gpu_dense_oracle import dense_phi
    from paper_2211_00696_b200.workloads import config
    for cfg, n in [(1, None), (2, 16)]:
        w = config(cfg, n=n)
        b = w.rhs(0)
        want = dense_phi(pq, w.factors, b, w.p)
        got = pq.phiquadmv(pq.KroneckerSum(w.factors), b, pq.PhiRequest(p=w.p, eps=1e-14,
                                                                       mode=pq.QuadKind.gauss_legendre))
        print(json.dumps({"workload": w.name, "N": int(w.N), "p": w.p, "eps": 1e-14,
                          "rel2_per_column": [rel2(got.col(j + 1), want[j]) for j in range(w.p)]}))


if __name__ == "__main__":
    main()
