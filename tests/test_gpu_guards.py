"""Kernel hygiene without compute-sanitizer (closed on this GPU pool): tests/guard_worker.py runs
every engine path with canary-guarded workspace buffers (PQ_WS_GUARD=1) -- no out-of-bounds write
may touch a canary -- and repeats every call three times: results must be bitwise equal (races in
shared memory or across the engine's streams would show as run-to-run differences)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_workspace_guards_and_bitwise_repeatability():
    env = dict(os.environ, PQ_WS_GUARD="1")
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "guard_worker.py")], capture_output=True, text=True,
                       timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    out = os.environ.get("PQ_MARGINS_OUT")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps({"case": "workspace_guards", "report": rep}) + "\n")
    for name, v in rep.items():
        assert v["damaged"] == 0, (name, v)
        assert v["bitwise_repeat"], name
        assert v["finite"], name
