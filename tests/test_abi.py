"""The C-ABI library: loads, exports every entry point include/pq_b200.h declares, maps errors to
the reference's exception types, and has no CPU fallback (no device -> PQ_ERUNTIME)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from conftest import has_gpu

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "pq_b200.h").read_text()
    return sorted(set(re.findall(r"PQ_API\s+[\w\s\*]+?\b(pq_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("pq_phiquadmv", "pq_phi_with_plan", "pq_phi_fixed", "pq_phi_adaptive", "pq_squaring_step",
                 "pq_mode_apply", "pq_exp_action", "pq_kron_matvec", "pq_expm", "pq_setup_quadrature",
                 "pq_quadnodes", "pq_integrate", "pq_erk_step", "pq_phi_lincomb", "pq_phi_nodes_partial"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2211_00696_b200 import LIB_PATH
    lib = C.CDLL(str(LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2211_00696_b200._lib import SIGNATURES
    assert set(declared_symbols()) <= set(SIGNATURES)


def test_error_mapping(pq):
    with pytest.raises(ValueError):
        pq.gauss_legendre(0)
    with pytest.raises(ValueError):
        pq.clenshaw_curtis(1)
    with pytest.raises(ValueError):
        pq.quadnodes(2.0, 3, 10.0, 1.0, pq.QuadKind.gauss_legendre)
    with pytest.raises(ValueError):
        pq.setup_quadrature(1e-10, 3, -1.0, 1.0, pq.QuadKind.gauss_legendre)
    with pytest.raises(ValueError):
        pq.KroneckerSum([])
    with pytest.raises(ValueError):
        pq.KroneckerSum([[[1.0, float("nan")], [0.0, 1.0]]])


@pytest.mark.skipif(has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback_without_a_device(pq):
    with pytest.raises(RuntimeError, match="no CUDA device"):
        pq.Context(0)
