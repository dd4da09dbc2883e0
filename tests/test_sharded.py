"""Node-sharded phi (paper_2211_00696_b200/sharded.py): the host-side partition and reduction
logic with world size 2 over gloo on CPU (the per-node device work is stood in for by the numpy
oracle), and on one B200 the sharded path against the unsharded one (world size 1, plus an
emulated 2-way split reduced on the host)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import pq_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _partial_oracle(factors, b, p, rule, nodes):
    x, w = rule
    return O.phi_fixed(factors, b, p, (x[nodes], w[nodes]))[0]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2211_00696_b200.sharded import node_partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    fs = [rng.uniform(-0.4, 0.4, (3, 3)), rng.uniform(-0.4, 0.4, (4, 4))]
    b = rng.standard_normal(12)
    rule = O.cached_rule(0, 9)
    mine = node_partition(len(rule[0]), rank, world)
    part = torch.from_numpy(_partial_oracle(fs, b, 3, rule, mine))
    dist.all_reduce(part)
    full = O.phi_fixed(fs, b, 3, rule)[0]
    q.put((rank, mine, float(np.max(np.abs(part.numpy() - full)))))
    dist.destroy_process_group()


def test_node_partition_covers_each_node_once():
    from paper_2211_00696_b200.sharded import node_partition
    for q in (1, 7, 13, 25):
        for world in (1, 2, 3, 8):
            got = sorted(i for r in range(world) for i in node_partition(q, r, world))
            assert got == list(range(q))


def test_sharded_reduction_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nodes = sorted(i for _, mine, _ in res for i in mine)
    assert nodes == list(range(9))
    for _, _, err in res:
        assert err <= 1e-14


@pytest.mark.gpu
def test_sharded_single_gpu_matches_unsharded(pq):
    import ctypes as C
    import torch
    from paper_2211_00696_b200 import _lib as L
    from paper_2211_00696_b200.sharded import phi_with_plan_sharded
    from paper_2211_00696_b200.workloads import config
    w = config(3, n=24)
    a = pq.KroneckerSum(w.factors)
    bs = torch.from_numpy(np.stack([w.rhs(k) for k in range(2)])).cuda()
    l, n = 4, 9
    got = phi_with_plan_sharded(a, bs, w.p, l, n).cpu().numpy()
    want = np.stack([c.cols for c in pq.phi_with_plan(a, list(bs.cpu().numpy()), w.p, l, n,
                                                      pq.QuadKind.gauss_legendre, w.eps)])
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
    # emulated 2-rank split on one GPU: partial sums over disjoint node sets, summed on the host
    ctx = pq.default_context()
    rule = pq.cached_rule(pq.QuadKind.gauss_legendre, n + 1)
    d, sh, fac = a._abi()
    parts = []
    for r in range(2):
        acc = torch.empty((2, w.p, w.N), dtype=torch.float64, device="cuda")
        L.check(L.lib.pq_phi_nodes_partial(ctx.handle, d, sh, fac, 2, C.c_void_p(bs.data_ptr()), w.p, l,
                                           rule.points(), rule.nodes.ctypes.data_as(L.dp),
                                           rule.weights.ctypes.data_as(L.dp), r, 2, 1, C.c_void_p(acc.data_ptr())))
        ctx.synchronize()
        parts.append(acc)
    tot = parts[0] + parts[1]
    L.check(L.lib.pq_squaring_chain(ctx.handle, d, sh, fac, 2, w.p, l, C.c_void_p(tot.data_ptr())))
    ctx.synchronize()
    assert np.max(np.abs(tot.cpu().numpy() - want)) <= 1e-12 * np.max(np.abs(want))
