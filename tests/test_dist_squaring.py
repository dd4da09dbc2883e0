"""Distributed modified squaring (paper_2211_00696_b200/dist_squaring.py).

CPU: world sizes 2 and 3 over gloo (3 gives uneven slabs and pencils), numpy backend, against the
same steps on the whole vector in one process.  GPU: the device backend (pq_mode_product /
pq_squaring_combine) with 2 and 4 ranks emulated by threads on one B200, against the engine's own
squaring chain, and phi_with_plan_distributed at world size 1 against phi_with_plan."""
import os
import socket
import threading

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(seed=3, shape=(7, 5, 4), p=3, nb=2, l=3):
    from scipy.linalg import expm
    rng = np.random.default_rng(seed)
    fs = [rng.uniform(-0.5, 0.5, (n, n)) for n in shape]
    y0 = rng.standard_normal((nb * p, int(np.prod(shape))))
    exps = [[expm(2.0 ** (j - l) * f) for f in fs] for j in range(l)]
    return shape, p, nb, exps, y0


def _whole(shape, p, nb, exps, y0):
    from paper_2211_00696_b200.dist_squaring import NumpyBackend, SlabLayout, squaring_distributed

    class One:
        rank, world = 0, 1
    return squaring_distributed(y0.copy(), exps, SlabLayout(shape, 1), One(), NumpyBackend(), p, nb)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2211_00696_b200.dist_squaring import NumpyBackend, SlabLayout, squaring_distributed

    class NumpyComm:  # gloo all_to_all on CPU tensors, numpy in and out
        def alltoallv(self, blocks, recv_sizes):
            import torch
            send = torch.cat([torch.from_numpy(np.ascontiguousarray(b)).reshape(-1) for b in blocks])
            recv = torch.empty(sum(recv_sizes), dtype=torch.float64)
            dist.all_to_all_single(recv, send, output_split_sizes=recv_sizes,
                                   input_split_sizes=[int(b.size) for b in blocks])
            return [t.numpy() for t in torch.split(recv, recv_sizes)]

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape, p, nb, exps, y0 = _problem()
    lay = SlabLayout(shape, world)
    comm = NumpyComm()
    comm.rank, comm.world = rank, world
    b0, b1 = lay.slab_range(rank)
    got = squaring_distributed(np.ascontiguousarray(y0[:, b0:b1]), exps, lay, comm, NumpyBackend(), p, nb)
    want = _whole(shape, p, nb, exps, y0)[:, b0:b1]
    q.put((rank, float(np.max(np.abs(got - want)) / np.max(np.abs(want)))))
    dist.destroy_process_group()


def test_slab_layout_covers_vector():
    from paper_2211_00696_b200.dist_squaring import SlabLayout
    for shape in [(7, 5, 4), (8, 3), (16, 16, 16)]:
        for world in (1, 2, 3, 4, 7):
            if shape[0] < world:
                continue
            lay = SlabLayout(shape, world)
            assert sum(lay.slab_len(r) for r in range(world)) == int(np.prod(shape))
            assert sum(lay.pencil_cols(r) for r in range(world)) == lay.rest
            assert lay.slab_range(world - 1)[1] == int(np.prod(shape))


def test_numpy_squaring_matches_reference_steps():
    """The whole-vector numpy path of the distributed code equals the oracle's squaring steps."""
    from oracle import pq_oracle as O
    shape, p, nb, exps, y0 = _problem()
    got = _whole(shape, p, nb, exps, y0)
    y = y0.reshape(nb, p, -1).copy()
    for E in exps:
        y = np.stack([O.squaring_step(y[m], E) for m in range(nb)])
    assert np.max(np.abs(got.reshape(nb, p, -1) - y)) <= 1e-13 * np.max(np.abs(y))


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_squaring_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, err in res:
        assert err <= 1e-13, (rank, err)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_distributed_squaring_device_emulated(pq, world):
    import torch
    from paper_2211_00696_b200.dist_squaring import DeviceBackend, SlabLayout, ThreadComm, squaring_distributed
    from paper_2211_00696_b200.workloads import config
    w = config(2, n=32)
    shape, p, nb, l = [f.shape[0] for f in w.factors], w.p, 1, 3
    rng = np.random.default_rng(11)
    y0 = torch.from_numpy(rng.standard_normal((nb * p, w.N))).cuda()
    fs = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in w.factors]
    exps = []
    for j in range(l):
        exps.append([pq.expm(f, scale=[2.0 ** (j - l)])[0].contiguous() for f in fs])
    torch.cuda.synchronize()
    # the engine's own chain on the whole vector (one context, squaring exponentials given)
    ref_ctx = pq.Context(0)
    want = squaring_distributed(y0.clone(), exps, SlabLayout(shape, 1),
                                type("One", (), {"rank": 0, "world": 1})(), DeviceBackend(ref_ctx), p, nb)
    torch.cuda.synchronize()
    lay = SlabLayout(shape, world)
    comm = ThreadComm(world)
    out = [None] * world
    errors = []

    def rank_main(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = pq.Context(0)
                ctx.set_stream(s.cuda_stream)
                b0, b1 = lay.slab_range(r)
                out[r] = squaring_distributed(y0[:, b0:b1].contiguous(), exps, lay, comm.bind(r, s.synchronize),
                                              DeviceBackend(ctx), p, nb)
                s.synchronize()
        except Exception as e:  # surfaced below
            errors.append(e)
            comm.bar.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    got = torch.cat(out, dim=1)
    rel = float(torch.linalg.norm(got - want) / torch.linalg.norm(want))
    assert rel <= 1e-13, rel


@pytest.mark.gpu
def test_phi_with_plan_distributed_world1_matches_engine(pq):
    import torch
    from paper_2211_00696_b200.sharded import phi_with_plan_distributed
    from paper_2211_00696_b200.workloads import config
    w = config(3, n=32)
    a = pq.KroneckerSum(w.factors)
    b = torch.from_numpy(np.stack([w.rhs(0), w.rhs(1)])).cuda()
    got = phi_with_plan_distributed(a, b, w.p, 4, 9)
    want = torch.stack([pq.phi_with_plan(a, b[m], w.p, 4, 9, pq.QuadKind.gauss_legendre, w.eps)[0].cols
                        for m in range(2)])
    rel = float(torch.linalg.norm(got - want.reshape(got.shape)) / torch.linalg.norm(want))
    assert rel <= 1e-12, rel
