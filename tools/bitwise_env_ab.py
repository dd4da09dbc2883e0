"""Run a few phi calls and save their results (to compare two builds / env settings bitwise).
Usage: python tools/bitwise_env_ab.py OUT.npz   (then compare two files with --compare A B)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print({"arrays": len(a.files), "bitwise_equal": len(a.files) - len(bad), "differ": bad})
    sys.exit(1 if bad else 0)

import torch  # noqa: E402,F401

import paper_2211_00696_b200 as pq  # noqa: E402
from paper_2211_00696_b200.workloads import config  # noqa: E402

out = {}
for cfg, n, nb in [(2, 48, 1), (2, 64, 2), (3, 40, 3), (5, 24, 1), (1, 64, 1), (2, 128, 1), (3, 96, 2)]:
    w = config(cfg, n=n)
    a = pq.KroneckerSum(w.factors)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    bs = np.stack([w.rhs(77 + m) for m in range(nb)])
    for dev in (False, True):
        x = torch.from_numpy(bs).cuda() if dev else bs
        r0, r = pq.phi_0p(a, x, req)
        tag = f"cfg{cfg}_n{n}_nb{nb}_{'dev' if dev else 'host'}"
        for name, v in (("phi0", r0), ("cols", r)):
            out[f"{tag}_{name}"] = v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)
np.savez(sys.argv[1], **out)
print("saved", len(out))
