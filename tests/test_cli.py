"""phiquad_cli (paper_2211_00696_b200/cli/phiquad_cli.cpp): the reference CLI's wire format on the
B200 engine.  Expectations are the reference's own CLI tests
(proj/tests/test_cli.cpp): exact plan rows and trailers, bench/converge layouts, the phi
subcommand reproducing the in-process result bit for bit, exit codes 0 / 2 / 3.  `plan` and the
argument errors are host-only (CPU suite); bench / converge / phi run on the GPU."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2211_00696_b200" / "phiquad_cli"


def run(*args, timeout=600):
    if not CLI.exists():
        import paper_2211_00696_b200.build as b
        b.build()
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout


# ---- host-only --------------------------------------------------------------------------------

def test_plan_rows_and_trailer():
    code, out = run("plan", "--eps", "1e-14", "--p", "20", "--alpha", "384", "--rule", "gauss")
    assert code == 0
    assert out.splitlines() == ["alpha,rule,l,n,C", "384,gauss,3,36,96", "# plan: l=3,n=36,rule=gauss,eps=1e-14"]


def test_plan_shortest_round_trip_norm():
    code, out = run("plan", "--eps", "1e-14", "--p", "20", "--alpha", "332.8", "--rule", "gauss")
    assert code == 0 and out.splitlines()[1] == "332.8,gauss,3,33,93"


def test_plan_small_norm_unscaled_and_nested_rule():
    assert run("plan", "--alpha", "0.5", "--p", "20")[1].splitlines()[1].startswith("0.5,gauss,0,")
    assert run("plan", "--alpha", "384", "--p", "20", "--rule", "cc")[1].splitlines()[1].startswith("384,cc,4,")


def test_plan_several_norms():
    code, out = run("plan", "--alpha", "384", "1536", "6144", "--p", "20")
    lines = out.splitlines()
    assert code == 0 and len(lines) == 5
    assert [l.split(",")[0] for l in lines[1:4]] == ["384", "1536", "6144"]


def test_plan_output_file(tmp_path):
    path = tmp_path / "plan.csv"
    code, out = run("plan", "--alpha", "384", "--p", "20", "--out", path)
    assert code == 0 and out == ""
    assert path.read_text().splitlines()[0] == "alpha,rule,l,n,C"


@pytest.mark.parametrize("args,code", [
    (["plan", "--alpha", "1", "--bogus"], 2),          # unknown flag
    (["plan"], 2),                                       # missing required flag
    (["plan", "--alpha", "1", "--rule", "simpson"], 2),  # unknown rule
    (["bench", "--problem", "7"], 2),                    # out of range
    (["bench", "--problem", "1", "--r", "4", "--p", "20", "--verify"], 2),  # oversized dense check
    (["converge", "--problem", "1", "--r", "2", "--tau", "0.5"], 2),
])
def test_exit_codes(args, code):
    assert run(*args)[0] == code


def test_help_lists_subcommands():
    code, out = run("--help")
    assert code == 0 and "plan" in out and "bench" in out


# ---- GPU --------------------------------------------------------------------------------------

@pytest.mark.gpu
def test_bench_verified_within_tolerance():
    code, out = run("bench", "--problem", "1", "--r", "2", "--p", "20", "--verify")
    lines = out.splitlines()
    assert code == 0 and len(lines) == 22 and lines[0] == "p,rel_err"
    for p in range(1, 21):
        pc, ec = lines[p].split(",")
        assert pc == str(p) and float(ec) <= 1e-11
    assert lines[21].startswith("# plan:") and "dim=27" in lines[21]


@pytest.mark.gpu
def test_bench_full_scale_plan():
    code, out = run("bench", "--problem", "1", "--r", "4", "--p", "20")
    lines = out.splitlines()
    assert code == 0
    assert "l=3,n=36,rule=gauss" in lines[-1] and "alpha=384" in lines[-1] and "dim=3375" in lines[-1]
    assert lines[1] == "1,nan"


@pytest.mark.gpu
def test_bench_boundary_layer_dimension_and_reruns():
    code, out = run("bench", "--problem", "2", "--r", "5", "--p", "4")
    assert code == 0 and "dim=992" in out.splitlines()[-1]
    args = ["bench", "--problem", "2", "--r", "3", "--p", "8", "--rule", "cc", "--verify"]
    a, b = run(*args), run(*args)
    assert a[0] == 0 and a[1] == b[1] and a[1]


@pytest.mark.gpu
def test_converge_ladder_and_single_step():
    code, out = run("converge", "--r", "2")
    lines = out.splitlines()
    assert code == 0 and len(lines) == 8 and lines[0] == "tau,err_euler,err_rk2,err_rk3"
    assert lines[1].startswith("0.5,") and lines[6].startswith("0.015625,") and lines[7].startswith("# plan:")
    err3 = [float(lines[i].rsplit(",", 1)[1]) for i in (1, 3, 6)]
    assert err3[0] > err3[1] > err3[2]
    code, out = run("converge", "--r", "2", "--tau", "0.5")
    assert code == 0 and len(out.splitlines()) == 3 and out.splitlines()[1].startswith("0.5,")
    assert run("converge", "--problem", "3", "--r", "2", "--tau", "0.5")[0] == 0


@pytest.mark.gpu
def test_phi_subcommand_bit_for_bit(pq, tmp_path):
    rng = np.random.default_rng(1234)
    ax, ay = rng.uniform(-0.5, 0.5, (3, 3)), rng.uniform(-0.5, 0.5, (2, 2))
    b = rng.uniform(-0.5, 0.5, 6)

    def write(path, m):
        m = np.atleast_2d(m)
        path.write_text(f"{m.shape[0]} {m.shape[1]}\n" + "\n".join(" ".join(f"{v:.17g}" for v in row) for row in m) + "\n")

    write(tmp_path / "ax.txt", ax)
    write(tmp_path / "ay.txt", ay)
    write(tmp_path / "b.txt", b[:, None])
    code, out = run("phi", "--matrix-file", tmp_path / "ax.txt", "--matrix-file", tmp_path / "ay.txt",
                    "--b-file", tmp_path / "b.txt", "--p", "3", "--threads", "1")
    assert code == 0
    tok = out.split()
    rows, cols = int(tok[0]), int(tok[1])
    got = np.array([float(t) for t in tok[2:]]).reshape(rows, cols)
    want = pq.phiquadmv(pq.KroneckerSum([ax, ay]), b, pq.PhiRequest(p=3, eps=1e-14, mode=pq.QuadKind.gauss_legendre))
    for j in range(3):
        assert np.array_equal(got[:, j], np.asarray(want.col(j + 1)))


@pytest.mark.gpu
def test_unreachable_tolerance_exit_code_3():
    assert run("bench", "--problem", "1", "--r", "2", "--p", "2", "--rule", "cc", "--eps", "1e-300")[0] == 3
