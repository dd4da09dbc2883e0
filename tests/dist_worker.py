"""TEST INFRASTRUCTURE: one rank of a distributed phi call (paper_2211_00696_b200/sharded.py ->
the C ABI's pq_*_dist), launched by tests/test_sharded.py with torch.distributed.run.  Every rank
shares GPU 0 and talks through the host transport (gloo), so no kernel waits on another process.
Rank r writes <out>.r<r>.npz with its gathered result, its slab result and its bytes sent."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def case_inputs(case):
    from paper_2211_00696_b200.workloads import config
    if case == "cfg3_gauss":      # config 3 family, Gauss, 2 RHS, planned (l > 0), phi_0
        w = config(3, n=32)
        return w, np.stack([w.rhs(k) for k in range(2)]), "plan"
    if case == "cfg2_cc":         # headline family, adaptive CC ladder, planned, phi_0
        w = config(2, n=24)
        return w, w.rhs(3)[None, :], "plan"
    if case == "cfg5_pinned":     # config 5 family, p = 6, pinned (l, n) = (2, 8), uneven slabs at world 3
        w = config(5, n=40)
        return w, w.rhs(1)[None, :], (2, 8)
    if case == "cfg1_2d":         # d = 2 (config 1 family), planned
        w = config(1, n=48)
        return w, w.rhs(0)[None, :], "plan"
    if case == "cc_pinned_l0":    # CC at l = 0 (no squaring), 3 RHS
        w = config(2, n=20)
        return w, np.stack([w.rhs(k) for k in range(3)]), (0, 0)
    if case == "d1_gauss":        # one factor: slabs of a single dimension, one rank owns the pencil
        w = config(1, n=48)
        w.d, w.factors = 1, [w.factors[0]]
        w.n = 48
        rng = np.random.default_rng(3)
        return w, rng.standard_normal((1, 48)), (3, 6)
    if case == "cc_2rhs_planned":  # adaptive CC with 2 RHS and l > 0 (squaring on 2 x p columns)
        w = config(2, n=20)
        return w, np.stack([w.rhs(k) for k in range(2)]), "plan"
    raise ValueError(case)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--device-inputs", action="store_true")
    ap.add_argument("--transport", default="host", choices=["host", "nccl", "peer"])
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    import paper_2211_00696_b200 as pq
    from paper_2211_00696_b200 import sharded as S
    w, bs, plan = case_inputs(args.case)
    a = pq.KroneckerSum(w.factors)
    ctx = pq.Context(0)
    comm = (S.Communicator.nccl(ctx) if args.transport == "nccl" else
            S.Communicator.peer(ctx) if args.transport == "peer" else S.Communicator.host())
    inp = torch.from_numpy(bs).cuda() if args.device_inputs else bs
    res = {}
    if plan == "plan":
        req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
        info = pq.PhiInfo()
        phi0, cols = S.phiquadmv_dist(a, inp, req, comm, ctx=ctx, phi0=True, info=info)
        comm.stats(reset=True)
        phi0_s, cols_s = S.phiquadmv_dist(a, inp, req, comm, ctx=ctx, phi0=True, gather=False)
        res["bytes_slab_call"] = comm.stats(reset=True)[0]
        res.update(phi0=phi0, cols=cols, phi0_slab=phi0_s, cols_slab=cols_s,
                   plan=np.array([info.l, info.n, info.points]))
    else:
        l, n = plan
        kind = pq.QuadKind(w.mode)
        inf = {}
        cols = S.phi_with_plan_dist(a, inp, w.p, l, n, kind, w.eps, comm, ctx=ctx, info=inf)
        cols_s = S.phi_with_plan_dist(a, inp, w.p, l, n, kind, w.eps, comm, ctx=ctx, gather=False)
        res.update(cols=cols, cols_slab=cols_s, plan=np.array([l, n, inf["points_used"]]))
    res = {k: (v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)) for k, v in res.items()}
    res["slab"] = np.array(S.slab_range(a.shape(), world, rank))
    np.savez(f"{args.out}.r{rank}.npz", **res)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
