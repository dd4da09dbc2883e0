"""Worker for tests/test_gpu_env_variants.py: three host callers (own contexts, streams, pinned
buffers) call pq_phi_0p concurrently, three rounds each, on config 2 at n = 64 (10 MB of results:
the compute gate's and the bounce's size class); every result must equal the same call made
alone, bitwise.  The sequential results are saved to argv[1] for cross-variant comparison.
Runtime switches (PQ_COMPUTE_GATE, PQ_SQ_FUSE, PQ_PLAN_SPEC, ...) come from the environment."""
import ctypes as C
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2211_00696_b200 as pq  # noqa: E402
from paper_2211_00696_b200.workloads import config  # noqa: E402

w = config(2, n=64)
a = pq.KroneckerSum(w.factors)
req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
d, sh, fac = a._abi()
rc = req._c()
K = 3


def call(ctx, b, o0, o):
    info = pq._lib.PhiInfoC()
    pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, 1, C.c_void_p(b.data_ptr()), C.byref(rc),
                                        C.c_void_p(o0.data_ptr()), C.c_void_p(o.data_ptr()), C.byref(info),
                                        pq._lib.PQ_HOST))


callers = []
for k in range(K):
    ctx = pq.Context(0)
    st = torch.cuda.Stream()
    ctx.set_stream(st.cuda_stream)
    callers.append((ctx, torch.from_numpy(w.rhs(40 + k).copy()).pin_memory(),
                    torch.empty((1, w.N), dtype=torch.float64).pin_memory(),
                    torch.empty((1, w.p, w.N), dtype=torch.float64).pin_memory()))
want = []
for ctx, b, o0, o in callers:
    call(ctx, b, o0, o)
    want.append((o0.numpy().copy(), o.numpy().copy()))
errors = []


def worker(k):
    ctx, b, o0, o = callers[k]
    try:
        for _ in range(3):
            o0.fill_(float("nan"))
            o.fill_(float("nan"))
            call(ctx, b, o0, o)
            if not (np.array_equal(o0.numpy(), want[k][0]) and np.array_equal(o.numpy(), want[k][1])):
                errors.append(f"caller {k}: concurrent result differs from its sequential call")
    except Exception as e:  # pragma: no cover
        errors.append(repr(e))


ths = [threading.Thread(target=worker, args=(k,)) for k in range(K)]
for t in ths:
    t.start()
for t in ths:
    t.join()
np.savez(sys.argv[1], **{f"phi0_{k}": want[k][0] for k in range(K)}, **{f"cols_{k}": want[k][1] for k in range(K)})
for ctx, *_ in callers:
    ctx.close()
if errors:
    print("FAIL", errors)
    sys.exit(1)
print("OK")
