"""bench.py's JSON line keeps the driver's contract: one line, the required keys with the right
types, K timed steps / W >= 3 warm-up, e2e byte counts, roofline and clock records."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_bench_line_contract():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "2", "--warmup", "3", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k, t in [("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int), ("warmup", int),
                 ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str), ("dtype", str), ("data", str),
                 ("config", dict), ("gpu_launches", int), ("clocks", dict), ("e2e", dict), ("roofline", dict)]:
        assert isinstance(d[k], t), (k, d[k])
    assert "vs_baseline" in d and "cpu_baseline" in d
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["workload"] and "l2" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    ro = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in ro
    assert ro["achieved"] > 0 and ro["peak"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["gpu_launches"] > 0


@pytest.mark.parametrize("shard", ["rhs", "nodes", "nodes-peer"])
def test_bench_two_ranks_plumbing(shard):
    """The N > 1 launch the driver uses (torch.distributed.run, one process per rank), with gloo
    carrying the barrier / max-over-ranks so both ranks can share the one GPU of this box.  rhs: the
    RHS shards have no data-path collective (weak scaling); nodes: one action across both ranks
    through the distributed engine path with the host transport (strong scaling)."""
    import os
    env = dict(os.environ, PQ_BENCH_BACKEND="gloo")
    port = {"rhs": 29517, "nodes": 29519, "nodes-peer": 29521}[shard]
    extra = ["--transport", "peer", "--config", "2"] if shard == "nodes-peer" else ["--config", "1"]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                        "--gpus", "2", "--steps", "2", "--warmup", "3", "--e2e-callers", "1",
                        "--shard", shard.split("-")[0]] + extra,
                       capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["scaling"] == ("weak" if shard == "rhs" else "strong")
    assert f"{shard.split('-')[0]}-sharded x2" in d["config"]["parallelism"]
    assert d["e2e"]["value"] > 0
    if shard != "rhs":
        assert d["distributed"]["bytes_sent_per_step_rank0"] > 0
