"""Multi-GPU path (paper_2211_00696_b200/sharded.py -> C ABI pq_*_dist, csrc/dist.cpp).

CPU: slab geometry from the C ABI, the node partition, and the host transport's collectives
(the gloo callbacks the engine calls) with world size 2.
GPU: the REAL distributed product with 2 and 3 processes sharing the one B200 through the host
transport (gloo), against the compiled reference (oracle/_ref) at identical plans, and the
gathered result against the slabs.  Collectives go through the host, so no kernel ever waits on
another process (one GPU is all this environment has)."""
import ctypes as C
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import rel2

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_node_partition_covers_each_node_once():
    from paper_2211_00696_b200.sharded import node_partition
    for q in (1, 7, 13, 25):
        for world in (1, 2, 3, 8):
            got = sorted(i for r in range(world) for i in node_partition(q, r, world))
            assert got == list(range(q))


@pytest.mark.parametrize("shape,world", [([10, 4, 4], 3), ([256, 256, 256], 8), ([64, 64], 2), ([7], 7),
                                         ([13, 5], 4)])
def test_slab_ranges_tile_the_vector(shape, world):
    from paper_2211_00696_b200.sharded import slab_range
    N = int(np.prod(shape))
    rest = N // shape[0]
    spans = [slab_range(shape, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == N
    for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
        assert e0 == b1
    for b, e in spans:
        assert b % rest == 0 and e % rest == 0 and e > b  # whole x-slabs, none empty


def test_slab_ranges_reject_more_ranks_than_slabs():
    from paper_2211_00696_b200.sharded import slab_range
    with pytest.raises(ValueError):
        slab_range([3, 8, 8], 4, 0)


def _transport_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2211_00696_b200 import _lib as L
    from paper_2211_00696_b200.sharded import Communicator
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Communicator.host()
    cb_a2a, cb_max, t = comm._keep
    # rank r sends (r + 1) * (h + 1) doubles of value 100 r + h to rank h != r (self excluded, as the engine does)
    sc = np.array([0 if h == rank else (rank + 1) * (h + 1) for h in range(world)], dtype=np.int64)
    rc = np.array([0 if h == rank else (h + 1) * (rank + 1) for h in range(world)], dtype=np.int64)
    send = np.concatenate([np.full(sc[h], 100.0 * rank + h) for h in range(world)])
    recv = np.full(int(rc.sum()), np.nan)
    dp = C.POINTER(C.c_double)
    i64 = C.POINTER(C.c_int64)
    rcode = cb_a2a(None, send.ctypes.data_as(dp) if send.size else dp(), sc.ctypes.data_as(i64),
                   recv.ctypes.data_as(dp) if recv.size else dp(), rc.ctypes.data_as(i64))
    want = np.concatenate([np.full(rc[h], 100.0 * h + rank) for h in range(world)])
    buf = np.array([rank, -rank, 0.5 * rank], dtype=np.float64)
    rmax = cb_max(None, buf.ctypes.data_as(dp), 3)
    q.put((rank, rcode, bool(np.array_equal(recv, want)), rmax, buf.tolist()))
    comm.close()
    dist.destroy_process_group()


def test_host_transport_gloo_world2():
    """The alltoallv / allreduce-max callbacks the engine's host transport calls, over gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, rcode, ok, rmax, buf in got:
        assert rcode == 0 and ok and rmax == 0
        assert buf == [1.0, 0.0, 0.5]


# ------------------------------------------------------------------ GPU: the real product ----

def _launch(case, world, tmp_path, device_inputs=False, transport="host"):
    out = str(tmp_path / case)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "tests" / "dist_worker.py"),
           "--case", case, "--out", out, "--transport", transport] + (["--device-inputs"] if device_inputs else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-5000:]
    return [dict(np.load(f"{out}.r{k}.npz")) for k in range(world)]


def _reference(ref, case):
    sys.path.insert(0, str(ROOT / "tests"))
    from dist_worker import case_inputs
    w, bs, plan = case_inputs(case)
    if plan == "plan":
        want, info = ref.phiquadmv(w.factors, bs, w.p, w.eps, w.mode, threads=os.cpu_count() or 1)
        want0 = np.stack([ref.exp_action(w.factors, b) for b in bs])
        return w, want, want0, [info["l"], info["n"], info["points"]]
    l, n = plan
    want, pts = ref.phi_with_plan(w.factors, bs, w.p, l, n, w.mode, w.eps, threads=os.cpu_count() or 1)
    return w, want, None, [l, n, pts]


@pytest.mark.gpu
@pytest.mark.parametrize("case,world", [("cfg3_gauss", 2), ("cfg2_cc", 2), ("cfg5_pinned", 3), ("cfg1_2d", 2),
                                        ("cc_pinned_l0", 3), ("cfg2_cc", 3), ("d1_gauss", 2),
                                        ("cc_2rhs_planned", 2)])
def test_distributed_vs_reference(ref, tmp_path, case, world):
    """world processes on the one GPU; every rank's gathered phi_0..phi_p equals the reference's
    (1e-11 relative 2-norm per column, identical plan), and the slabs tile the gathered result."""
    ranks = _launch(case, world, tmp_path)
    w, want, want0, plan = _reference(ref, case)
    nb, p, N = want.shape
    for k, res in enumerate(ranks):
        assert list(res["plan"]) == plan, (k, res["plan"], plan)
        errs = [rel2(res["cols"][m, j], want[m, j]) for m in range(nb) for j in range(p)]
        assert max(errs) <= 1e-11, (k, max(errs))
        if want0 is not None:
            assert max(rel2(res["phi0"][m], want0[m]) for m in range(nb)) <= 1e-11
        b, e = res["slab"]
        assert np.array_equal(res["cols_slab"], res["cols"][:, :, b:e])  # slabs are the gathered result's pieces
        if want0 is not None:
            assert np.array_equal(res["phi0_slab"], res["phi0"][:, b:e])
    # every rank gathers the same bits
    for res in ranks[1:]:
        assert np.array_equal(res["cols"], ranks[0]["cols"])


@pytest.mark.gpu
def test_distributed_device_inputs_world2(ref, tmp_path):
    """Device-resident b (torch CUDA tensors) through the same path."""
    ranks = _launch("cfg3_gauss", 2, tmp_path, device_inputs=True)
    w, want, want0, plan = _reference(ref, "cfg3_gauss")
    for res in ranks:
        assert list(res["plan"]) == plan
        assert max(rel2(res["cols"][m, j], want[m, j]) for m in range(want.shape[0]) for j in range(w.p)) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("case,world", [("cfg3_gauss", 2), ("cfg2_cc", 3), ("cfg5_pinned", 2), ("cfg5_pinned", 3)])
def test_distributed_peer_transport(ref, tmp_path, case, world):
    """The peer transport: the squaring's and phi_0's slab <-> pencil flips fused into the mode
    products (remote-store epilogues into CUDA-IPC-mapped buffers of the other processes on this
    GPU; host barriers between the flips, so no kernel waits on another process).  cfg5_pinned at
    world 3 (n1 = 40 not divisible by 3) exercises the fallback to packed exchanges."""
    ranks = _launch(case, world, tmp_path, transport="peer")
    w, want, want0, plan = _reference(ref, case)
    nb, p, N = want.shape
    for k, res in enumerate(ranks):
        assert list(res["plan"]) == plan, (k, res["plan"], plan)
        assert max(rel2(res["cols"][m, j], want[m, j]) for m in range(nb) for j in range(p)) <= 1e-11
        if want0 is not None:
            assert max(rel2(res["phi0"][m], want0[m]) for m in range(nb)) <= 1e-11
        b, e = res["slab"]
        assert np.array_equal(res["cols_slab"], res["cols"][:, :, b:e])
    for res in ranks[1:]:
        assert np.array_equal(res["cols"], ranks[0]["cols"])


@pytest.mark.gpu
def test_distributed_nccl_transport_world1(ref, tmp_path):
    """The NCCL transport end to end on the one GPU this environment has: libnccl.so.2 loaded by
    dlopen, the unique id broadcast through torch.distributed, ncclCommInitRank, the distributed
    call (its exchanges are local copies at world 1) and ncclCommDestroy; results against the
    reference."""
    ranks = _launch("cfg3_gauss", 1, tmp_path, device_inputs=True, transport="nccl")
    w, want, want0, plan = _reference(ref, "cfg3_gauss")
    res = ranks[0]
    assert list(res["plan"]) == plan
    assert max(rel2(res["cols"][m, j], want[m, j]) for m in range(want.shape[0]) for j in range(w.p)) <= 1e-11
    assert max(rel2(res["phi0"][m], want0[m]) for m in range(want.shape[0])) <= 1e-11


@pytest.mark.gpu
def test_distributed_bytes_per_call(tmp_path):
    """Bytes a rank sends in a slab-output call (gather=False), against the DESIGN.md count for
    Gauss: node transpose (own nodes) or reduce-scatter (p partial sums, when ceil(q/G) > p) times
    nb (N - S_r), plus the slab <-> pencil flips of the l squaring steps and phi_0."""
    ranks = _launch("cfg3_gauss", 2, tmp_path)
    sys.path.insert(0, str(ROOT / "tests"))
    from dist_worker import case_inputs
    w, bs, _ = case_inputs("cfg3_gauss")
    nb, N = bs.shape
    n0, rest = w.n, N // w.n
    for r, res in enumerate(ranks):
        l, n, q = (int(x) for x in res["plan"])
        b, e = (int(x) for x in res["slab"])
        S = e - b
        own = len(range(r, q, 2))
        # node transpose (own nodes' slabs) or, when ceil(q/G) > p, the reduce-scatter of p partial sums
        node = (w.p if (q + 1) // 2 > w.p else own) * nb * (N - S)
        # a flip sends this rank's slab except its own pencil columns, twice per Kronecker apply
        c_lo, c_hi = rest * r // 2, rest * (r + 1) // 2
        flip = 2 * (S // rest) * (rest - (c_hi - c_lo))
        want = 8.0 * (node + (l * nb * w.p + nb) * flip)
        assert res["bytes_slab_call"] == want, (r, res["bytes_slab_call"], want)
