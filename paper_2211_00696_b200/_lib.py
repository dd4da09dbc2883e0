"""ctypes binding of libpq_b200.so (include/pq_b200.h).

Loading is strict: if the shared library is missing or a symbol is absent, import fails loudly —
there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PQ_B200_LIB", _HERE / "libpq_b200.so"))

PQ_OK, PQ_EINVAL, PQ_ECONVERGENCE, PQ_ERUNTIME, PQ_ERANGE, PQ_EINTERNAL = range(6)
PQ_GAUSS_LEGENDRE, PQ_CLENSHAW_CURTIS = 0, 1
PQ_HOST, PQ_DEVICE = 0, 1
PQ_SOURCE_ZERO, PQ_SOURCE_CUBIC, PQ_SOURCE_CONSTANT, PQ_SOURCE_CALLBACK = range(4)

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
vp = C.c_void_p


class PhiRequestC(C.Structure):
    _fields_ = [("p", C.c_int), ("eps", C.c_double), ("mode", C.c_int), ("has_l", C.c_int), ("l", C.c_int),
                ("c1", C.c_double), ("c2", C.c_double), ("threads", C.c_int)]


class PhiInfoC(C.Structure):
    _fields_ = [("l", C.c_int), ("n", C.c_int), ("points", C.c_int), ("mode", C.c_int), ("planned", C.c_int),
                ("alpha", C.c_double), ("beta", C.c_double), ("plan_cost", C.c_double)]


class TableauC(C.Structure):
    _fields_ = [("stages", C.c_int), ("order", C.c_int), ("c", dp), ("nterms", C.c_int), ("row", ip), ("col", ip),
                ("k", ip), ("coef", dp)]


SOURCE_CB = C.CFUNCTYPE(C.c_int, C.c_double, dp, dp, C.c_int64, vp)


class SourceC(C.Structure):
    _fields_ = [("kind", C.c_int), ("s1", C.c_double), ("s3", C.c_double), ("vec", dp), ("cb", SOURCE_CB),
                ("user", vp)]


ALLTOALLV_CB = C.CFUNCTYPE(C.c_int, vp, dp, C.POINTER(C.c_int64), dp, C.POINTER(C.c_int64))
ALLREDUCE_CB = C.CFUNCTYPE(C.c_int, vp, dp, C.c_int64)


class HostTransportC(C.Structure):
    _fields_ = [("user", vp), ("alltoallv", ALLTOALLV_CB), ("allreduce_max", ALLREDUCE_CB)]


# name -> (restype, argtypes)
SIGNATURES = {
    "pq_version": (C.c_char_p, []),
    "pq_last_error": (C.c_char_p, []),
    "pq_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "pq_ctx_destroy": (C.c_int, [vp]),
    "pq_ctx_set_stream": (C.c_int, [vp, vp]),
    "pq_ctx_stream": (vp, [vp]),
    "pq_ctx_synchronize": (C.c_int, [vp]),
    "pq_ctx_launches": (C.c_uint64, [vp]),
    "pq_ctx_set_workspace_limit": (C.c_int, [vp, C.c_uint64]),
    "pq_ctx_release_workspace": (C.c_int, [vp]),
    "pq_ctx_set_profiling": (C.c_int, [vp, C.c_int]),
    "pq_ctx_phase_times": (C.c_int, [vp, dp]),
    "pq_ctx_gemm_stats": (C.c_int, [vp, C.c_int, C.POINTER(C.c_uint64), dp, dp]),
    "pq_ctx_gemm_dense_flops": (C.c_int, [vp, C.c_int, dp]),
    "pq_mode_product": (C.c_int, [vp, C.c_int, ip, C.c_int, vp, C.c_int, vp, vp]),
    "pq_squaring_combine": (C.c_int, [vp, C.c_longlong, C.c_int, C.c_int, vp, vp]),
    "pq_ctx_timeline": (C.c_int, [vp, C.POINTER(C.c_char_p)]),
    "pq_ctx_kernel_stats": (C.c_int, [vp, C.c_int, C.POINTER(C.c_char_p)]),
    "pq_ctx_gemm_breakdown": (C.c_int, [vp, C.c_int, C.POINTER(C.c_char_p)]),
    "pq_ctx_check_guards": (C.c_int, [vp, ip]),
    "pq_gauss_legendre": (C.c_int, [C.c_int, dp, dp]),
    "pq_clenshaw_curtis": (C.c_int, [C.c_int, dp, dp]),
    "pq_cached_rule": (C.c_int, [C.c_int, C.c_int, C.POINTER(dp), C.POINTER(dp)]),
    "pq_quartic_roots": (C.c_int, [dp, dp]),
    "pq_real_roots_greater_one": (C.c_int, [dp, dp, ip]),
    "pq_log_bound_at_rho": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, dp]),
    "pq_bound_quartic": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, dp]),
    "pq_theorem_bound": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, dp]),
    "pq_corollary_bound": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, dp]),
    "pq_quaderr": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, dp]),
    "pq_quadnodes": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, ip]),
    "pq_setup_quadrature": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, C.c_double,
                                      C.c_double, C.c_int, ip, ip, dp]),
    "pq_infnorm_bound": (C.c_int, [C.c_int, ip, dp, dp]),
    "pq_expm": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp, C.c_int]),
    "pq_mode_apply": (C.c_int, [vp, C.c_int, ip, dp, vp, vp, C.c_int]),
    "pq_kron_matvec": (C.c_int, [vp, C.c_int, ip, dp, vp, vp, C.c_int]),
    "pq_exp_action": (C.c_int, [vp, C.c_int, ip, dp, vp, vp, C.c_int]),
    "pq_phi_fixed": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, vp, C.c_int, C.c_int, dp, dp, vp, C.c_int]),
    "pq_phi_adaptive": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, vp, C.c_int, C.c_double, vp, ip, C.c_int]),
    "pq_squaring_step": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, vp, C.c_int]),
    "pq_phi_fixed_cols": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, C.POINTER(vp), C.c_int, C.c_int, dp, dp,
                                    C.POINTER(vp), C.c_int]),
    "pq_phi_adaptive_cols": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, C.POINTER(vp), C.c_int, C.c_double,
                                       C.POINTER(vp), ip, C.c_int]),
    "pq_squaring_step_cols": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, C.POINTER(vp), C.c_int]),
    "pq_phi_with_plan": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_double, vp, ip, C.c_int]),
    "pq_phiquadmv": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, vp, C.POINTER(PhiRequestC), vp,
                               C.POINTER(PhiInfoC), C.c_int]),
    "pq_phi_with_plan_cols": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, C.POINTER(vp), C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_double, C.POINTER(vp), ip, C.c_int]),
    "pq_phiquadmv_cols": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, C.POINTER(vp), C.POINTER(PhiRequestC),
                                    C.POINTER(vp), C.POINTER(PhiInfoC), C.c_int]),
    "pq_phi_0p": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, vp, C.POINTER(PhiRequestC), vp, vp,
                            C.POINTER(PhiInfoC), C.c_int]),
    "pq_phi_lincomb": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, vp, C.c_int, dp, dp, vp, C.c_int]),
    "pq_phi_nodes_partial": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, vp, C.c_int, C.c_int, C.c_int, dp, dp,
                                       C.c_int, C.c_int, C.c_int, vp]),
    "pq_squaring_chain": (C.c_int, [vp, C.c_int, ip, dp, C.c_int, C.c_int, C.c_int, vp]),
    "pq_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "pq_comm_create_nccl": (C.c_int, [vp, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)]),
    "pq_comm_create_host": (C.c_int, [C.c_int, C.c_int, C.POINTER(HostTransportC), C.POINTER(vp)]),
    "pq_comm_create_peer": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(HostTransportC), C.POINTER(vp)]),
    "pq_comm_destroy": (C.c_int, [vp]),
    "pq_comm_stats": (C.c_int, [vp, C.c_int, dp, C.POINTER(C.c_uint64)]),
    "pq_dist_slab": (C.c_int, [C.c_int, ip, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pq_phiquadmv_dist": (C.c_int, [vp, vp, C.c_int, ip, dp, C.c_int, vp, C.POINTER(PhiRequestC), vp, vp,
                                    C.POINTER(PhiInfoC), C.c_int, C.c_int]),
    "pq_phi_with_plan_dist": (C.c_int, [vp, vp, C.c_int, ip, dp, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_double, vp, ip, C.c_int, C.c_int]),
    "pq_builtin_tableau": (C.c_int, [C.c_int, C.c_double, C.POINTER(TableauC)]),
    "pq_integrate": (C.c_int, [vp, C.c_int, ip, dp, C.POINTER(SourceC), vp, C.c_double, C.c_double, C.c_int,
                               C.POINTER(TableauC), C.POINTER(PhiRequestC), vp, ip, C.c_int]),
    "pq_erk_step": (C.c_int, [vp, C.c_int, ip, dp, C.POINTER(SourceC), C.c_double, C.c_double, vp,
                              C.POINTER(TableauC), C.POINTER(PhiRequestC), vp, ip, C.c_int]),
}


def load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built (run __graft_entry__.build()); the engine has no CPU fallback")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError = missing export = broken build
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


class ConvergenceError(RuntimeError):
    """phiquad::ConvergenceError (util.hpp:11-14)."""


def check(rc: int) -> None:
    if rc == PQ_OK:
        return
    msg = (lib.pq_last_error() or b"").decode()
    if rc == PQ_EINVAL:
        raise ValueError(msg)
    if rc == PQ_ECONVERGENCE:
        raise ConvergenceError(msg)
    if rc == PQ_ERANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)
