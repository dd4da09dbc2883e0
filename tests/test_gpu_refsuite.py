"""The reference's own test suite on the B200 engine.

tests/cpp/Makefile (`make refsuite`) compiles the reference's unit tests and its acceptance gate
(proj/tests/test_*.cpp, acceptance.cpp) in place -- unmodified, not copied -- against this repo's
drop-in headers (include/phiquad -> libpq_b200.so), with a minimal Catch2-compatible harness
(tests/cpp/catch_shim; Catch2 is not in the image).  __graft_entry__.build() builds them where the
reference is mounted; the binaries travel with the repo snapshot, so running them needs neither
/root/reference nor Catch2.  test_cli drives this repo's CLI (PHIQUAD_CLI).

Every test case and assertion of the reference's suite must pass, and the acceptance gate must
report all seven criteria (planner table, CC point counts 49/97, full pipeline vs the dense
oracle at p = 20 both rules, a-priori bound never undercut, algebraic identities on 100 random
systems, ETD convergence orders, speed vs the dense reference) as PASS."""
import os
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "tests" / "cpp" / "_bin" / "refsuite"
HOST_ONLY = ["test_bounds", "test_quadrature", "test_roots"]  # planner / rules / roots: no device calls
DEVICE = ["test_dense", "test_kron", "test_oracle", "test_phiaction", "test_integrators", "test_problems", "test_cli"]


def _run(name, timeout=900, env=None):
    exe = BIN / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs /root/reference at build time: make -C tests/cpp refsuite)")
    env = dict(os.environ, PHIQUAD_CLI=str(ROOT / "paper_2211_00696_b200" / "phiquad_cli"), **(env or {}))
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=timeout, env=env)
    return r


@pytest.mark.parametrize("name", HOST_ONLY)
def test_reference_unit_suite_host(name):
    r = _run(name)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert ", 0 failed," in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", DEVICE)
def test_reference_unit_suite_on_b200(name):
    r = _run(name)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert ", 0 failed," in r.stdout


@pytest.mark.gpu
def test_reference_acceptance_gate_on_b200():
    # Criterion 7 times ONE phiquadmv call at r = 4 (~3.5 ms) against the dense oracle and needs
    # >= 10x.  Round 1 saw that call take 20-60 ms in most runs: the PQ_SLOWLOG timeline put the
    # time in the workspace regrowth (cudaFree of the previous, larger chain buffers is a
    # device-wide sync).  Replaced buffers are now retired without a free inside the call
    # (engine.cpp ws_bytes / pq_ctx::graveyard), so the gate runs ONCE, no retry; a slow call prints
    # its phase timeline to stderr (PQ_SLOWLOG) for the failure message.
    r = _run("acceptance", env={"PQ_SLOWLOG": "10"})
    c7 = [ln for ln in r.stdout.splitlines() if ln.startswith("criterion 7:")]
    print(c7, r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    verdicts = [ln for ln in r.stdout.splitlines() if ln.startswith("criterion ") and ": " in ln and "note" not in ln]
    assert len(verdicts) == 7 and all(": PASS" in ln for ln in verdicts), r.stdout + r.stderr
    assert "acceptance: all 7 criteria passed" in r.stdout


def _numbers(line):
    return [float(x) for x in re.findall(r"[-+]?\d+\.?\d*(?:[eE][-+]?\d+)?", line)]


@pytest.mark.gpu
@pytest.mark.parametrize("demo", ["demo_heat3d", "demo_phi_action"])
def test_reference_demos_on_b200(demo):
    """The reference's demos (proj/demos), built against the drop-in headers: every line matches the
    reference build's output (tests/golden/<demo>_ref_output.txt, `make -C tests/cpp demos_golden`)
    exactly, except the reported error figures, which must stay <= max(1e-11, 2x the reference's)."""
    r = _run(demo, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    got = r.stdout.splitlines()
    want = (ROOT / "tests" / "golden" / f"{demo}_ref_output.txt").read_text().splitlines()
    assert len(got) == len(want)
    for g, w in zip(got, want):
        if re.search(r"=\s*[-+]?[\d.]+e[-+]\d+\s*$", w):  # an error figure (scientific notation)
            gv, wv = _numbers(g)[-1], _numbers(w)[-1]
            assert g.rsplit("=", 1)[0] == w.rsplit("=", 1)[0]
            assert gv <= max(1e-11, 2 * wv), (g, w)
        else:
            assert g == w
