"""bench.py's arms agree on what they measure (CPU checks, no GPU): the reference arm loads the
workload definitions WITHOUT importing the package (so libpq_b200.so is never mapped there), both
arms print the identical `config` dict, and every step draws a fresh right-hand-side seed."""
import argparse
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _args(**kw):
    a = argparse.Namespace(config=2, shard="rhs", steps=20, warmup=5, etd_steps=100, gpus=1)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_reference_arm_does_not_load_the_engine():
    code = ("import sys; sys.argv=['bench.py']; sys.path.insert(0, %r); import bench; W = bench.load_workloads(); "
            "W.config(2); print('paper_2211_00696_b200' in sys.modules, 'paper_2211_00696_b200._lib' in sys.modules)"
            % str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=str(ROOT), timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split() == ["False", "False"]


def test_both_arms_print_the_same_config():
    sys.path.insert(0, str(ROOT))
    import bench
    W = bench.load_workloads()
    for cfg in (1, 2, 3, 4, 5):
        w = W.config(cfg)
        a = _args(config=cfg)
        # the reference arm and the GPU arm both build their `config` with bench_config(w, args, world)
        assert bench.bench_config(w, a, 1) == bench.bench_config(w, _args(config=cfg), 1)
        assert bench.bench_config(w, a, 1)["workload"] == w.name


def test_fresh_seed_every_step_and_rank():
    sys.path.insert(0, str(ROOT))
    import bench
    a = _args(steps=4, warmup=3)
    s0 = bench.step_seeds(a, 0, 1)
    s1 = bench.step_seeds(a, 1, 1)
    flat0 = [x for st in s0 for x in st]
    flat1 = [x for st in s1 for x in st]
    assert len(s0) == 7 and len(set(flat0)) == 7          # one distinct seed per step (warm-up included)
    assert not set(flat0) & set(flat1)                    # ranks never share a right-hand side
    s8 = bench.step_seeds(a, 0, 8)
    assert len({x for st in s8 for x in st}) == 7 * 8      # config 3: 8 fresh RHS per step
