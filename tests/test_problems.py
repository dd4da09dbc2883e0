"""Drop-in problems.hpp (FE/Shishkin benchmark assembly): tests/cpp/
problems_dump.cpp, written against the reference API, compiled against include/phiquad must print
exactly the golden output the same source printed when compiled against the reference headers
(tests/golden/problems_ref_output.txt: meshes, operators, data, sources, error norms; %.17g, so
equality is bitwise).  Host-only: runs in the CPU suite."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_problem_assembly_bitwise_equals_reference():
    r = subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp"), "_bin/problems_b200"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(ROOT / "tests" / "cpp" / "_bin" / "problems_b200")], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stderr
    want = (ROOT / "tests" / "golden" / "problems_ref_output.txt").read_text()
    got_lines, want_lines = out.stdout.splitlines(), want.splitlines()
    assert len(got_lines) == len(want_lines) == 507
    for g, w in zip(got_lines, want_lines):
        assert g == w
