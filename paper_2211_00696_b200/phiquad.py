"""Python mirror of the reference's phiquad C++ API (proj/include/phiquad/*.hpp), backed by the
sm_100a engine through the C ABI (include/pq_b200.h).

Names, argument meaning and error behaviour follow the reference: ValueError for
std::invalid_argument, ConvergenceError for phiquad::ConvergenceError, IndexError for
std::out_of_range, RuntimeError for std::runtime_error.  Vectors may be numpy float64 arrays
(host; copied in and out) or torch.float64 CUDA tensors (device-resident; stream-ordered on the
context stream, which defaults to torch's current stream when torch is in use).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import ConvergenceError, check, lib

__all__ = [
    "QuadKind", "QuadratureRule", "gauss_legendre", "clenshaw_curtis", "cached_rule", "quartic_roots",
    "real_roots_greater_one", "BoundQuery", "CostModel", "QuadraturePlan", "log_bound_at_rho", "bound_quartic",
    "theorem_bound", "corollary_bound", "quaderr", "quadnodes", "setup_quadrature", "KroneckerSum", "expm",
    "mode_apply", "kron_matvec", "exp_action", "infnorm_bound", "PhiRequest", "PhiInfo", "PhiColumns",
    "phi_fixed", "phi_fixed_multi", "phi_adaptive", "phi_adaptive_multi", "squaring_step", "phi_with_plan",
    "phiquadmv", "phiquadmv_multi", "phi_0p", "phi_lincomb", "ExpRKTableau", "PhiTerm", "exp_euler_tableau",
    "exp_rk2_tableau", "exp_rk3_tableau", "etdrk4_tableau", "erk_step", "integrate", "IntegrationResult",
    "Context", "default_context", "ConvergenceError",
]


class QuadKind(enum.IntEnum):
    gauss_legendre = L.PQ_GAUSS_LEGENDRE
    clenshaw_curtis = L.PQ_CLENSHAW_CURTIS


def _dp(a: np.ndarray):
    return a.ctypes.data_as(L.dp)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(L.ip)


# ---------------------------------------------------------------- context ------------------

class Context:
    """One device, one stream, a device workspace (pq_ctx)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        check(lib.pq_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        if stream is not None:
            check(lib.pq_ctx_set_stream(h, C.c_void_p(stream)))

    def set_stream(self, stream: Optional[int]) -> None:
        """Run on an external CUDA stream handle (e.g. torch.cuda.current_stream().cuda_stream).
        Handle 0 is the legacy default stream (passed as cudaStreamLegacy); None = own stream."""
        if stream is None:
            check(lib.pq_ctx_set_stream(self.handle, None))
        else:
            check(lib.pq_ctx_set_stream(self.handle, C.c_void_p(stream if stream != 0 else 1)))

    @property
    def launches(self) -> int:
        return int(lib.pq_ctx_launches(self.handle))

    def synchronize(self) -> None:
        check(lib.pq_ctx_synchronize(self.handle))

    def set_profiling(self, on: bool) -> None:
        check(lib.pq_ctx_set_profiling(self.handle, 1 if on else 0))

    def gemm_stats(self, reset: bool = True) -> tuple:
        """(launches, device ms, executed FLOPs, dense FLOPs) of the DMMA GEMM launches recorded while
        profiling; executed < dense when negligible exponential blocks were skipped."""
        n, ms, fl, dense = C.c_uint64(), C.c_double(), C.c_double(), C.c_double()
        check(lib.pq_ctx_gemm_dense_flops(self.handle, 0, C.byref(dense)))
        check(lib.pq_ctx_gemm_stats(self.handle, 1 if reset else 0, C.byref(n), C.byref(ms), C.byref(fl)))
        if reset:
            check(lib.pq_ctx_gemm_dense_flops(self.handle, 1, None))
        return int(n.value), ms.value, fl.value, dense.value

    def kernel_stats(self, reset: bool = True) -> dict:
        """{kernel: {"launches", "ms", "bytes"}} of the streaming kernels recorded while profiling
        (device time from events on the launching stream, algorithmic bytes)."""
        import json
        js = C.c_char_p()
        check(lib.pq_ctx_kernel_stats(self.handle, 1 if reset else 0, C.byref(js)))
        return json.loads(js.value.decode())

    def check_guards(self) -> tuple:
        """(damaged buffer count, names) of the canary-guarded workspace (PQ_WS_GUARD=1)."""
        n = C.c_int()
        check(lib.pq_ctx_check_guards(self.handle, C.byref(n)))
        return n.value, (lib.pq_last_error() or b"").decode() if n.value else ""

    def gemm_breakdown(self, reset: bool = True) -> dict:
        """{"<call site> M N K Z layout": {"launches", "ms", "flops", "dense"}} of the profiled GEMMs."""
        import json
        js = C.c_char_p()
        check(lib.pq_ctx_gemm_breakdown(self.handle, 1 if reset else 0, C.byref(js)))
        return json.loads(js.value.decode())

    def set_workspace_limit(self, nbytes: int) -> None:
        check(lib.pq_ctx_set_workspace_limit(self.handle, nbytes))

    def close(self) -> None:
        if self.handle:
            lib.pq_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


_default: Optional[Context] = None


def default_context() -> Context:
    """Process-wide context on device 0.  When torch has initialised CUDA, the context follows
    torch's current stream, so device tensors produced by torch are consumed in stream order (an
    explicitly created Context keeps its own stream; order it with synchronize() or set_stream())."""
    global _default
    if _default is None:
        _default = Context(0)
        _default._bound = None
    import sys
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        s = torch.cuda.current_stream().cuda_stream
        if _default._bound != s:
            _default.set_stream(s)
            _default._bound = s
    return _default


# ---------------------------------------------------------------- vectors --------------------

def _is_device(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


class _Vec:
    """A caller vector batch viewed through the C ABI: (pointer, space)."""

    def __init__(self, xs, n: int, what: str):
        if isinstance(xs, (list, tuple)):
            if len(xs) and _is_device(xs[0]):
                import torch
                self.t = torch.stack([x.reshape(-1) for x in xs]).contiguous()
                self.device = True
            else:
                self.a = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float64).reshape(-1) for x in xs])
                                              if len(xs) else np.zeros((0, n)))
                self.device = False
        elif _is_device(xs):
            self.t = xs.contiguous()
            self.device = True
        else:
            self.a = np.ascontiguousarray(np.asarray(xs, dtype=np.float64))
            self.device = False
        if self.device:
            import torch
            if self.t.dtype != torch.float64:
                raise ValueError(f"{what}: device vectors must be float64")
            self.count = self.t.numel() // n if n else 0
            if self.t.numel() != self.count * n:
                raise ValueError(f"{what}: vector length mismatch")
        else:
            self.count = self.a.size // n if n else 0
            if self.a.size != self.count * n:
                raise ValueError(f"{what}: vector length mismatch")

    @property
    def ptr(self):
        return C.c_void_p(self.t.data_ptr() if self.device else self.a.ctypes.data)

    @property
    def space(self) -> int:
        return L.PQ_DEVICE if self.device else L.PQ_HOST

    def empty(self, count: int, n: int):
        if self.device:
            import torch
            return torch.empty((count, n), dtype=torch.float64, device=self.t.device)
        return np.empty((count, n), dtype=np.float64)


def _out_ptr(o):
    return C.c_void_p(o.data_ptr() if _is_device(o) else o.ctypes.data)


# ---------------------------------------------------------------- rules & estimator -----------

@dataclass
class QuadratureRule:
    """quadrature.hpp:21-27"""
    kind: QuadKind
    nodes: np.ndarray
    weights: np.ndarray

    def points(self) -> int:
        return int(self.nodes.size)


def gauss_legendre(m: int) -> QuadratureRule:
    x, w = np.empty(max(m, 0)), np.empty(max(m, 0))
    check(lib.pq_gauss_legendre(m, _dp(x), _dp(w)))
    return QuadratureRule(QuadKind.gauss_legendre, x, w)


def clenshaw_curtis(m: int) -> QuadratureRule:
    x, w = np.empty(max(m, 0)), np.empty(max(m, 0))
    check(lib.pq_clenshaw_curtis(m, _dp(x), _dp(w)))
    return QuadratureRule(QuadKind.clenshaw_curtis, x, w)


_rule_cache: dict = {}


def cached_rule(kind: QuadKind, m: int) -> QuadratureRule:
    key = (int(kind), m)
    if key not in _rule_cache:
        px, pw = L.dp(), L.dp()
        check(lib.pq_cached_rule(int(kind), m, C.byref(px), C.byref(pw)))
        _rule_cache[key] = QuadratureRule(QuadKind(kind), np.ctypeslib.as_array(px, (m,)).copy(),
                                          np.ctypeslib.as_array(pw, (m,)).copy())
    return _rule_cache[key]


def quartic_roots(a3: float, a2: float, a1: float, a0: float = 1.0) -> np.ndarray:
    c = np.array([a3, a2, a1, a0], dtype=np.float64)
    out = np.empty(8)
    check(lib.pq_quartic_roots(_dp(c), _dp(out)))
    return out[0::2] + 1j * out[1::2]


def real_roots_greater_one(a3: float, a2: float, a1: float, a0: float = 1.0) -> list:
    c = np.array([a3, a2, a1, a0], dtype=np.float64)
    out = np.empty(4)
    cnt = C.c_int()
    check(lib.pq_real_roots_greater_one(_dp(c), _dp(out), C.byref(cnt)))
    return [float(v) for v in out[: cnt.value]]


@dataclass
class BoundQuery:
    """bounds.hpp:20-26"""
    n: float = 0.0
    p: int = 0
    alpha: float = 0.0
    beta: float = 1.0
    kind: QuadKind = QuadKind.gauss_legendre


@dataclass
class CostModel:
    """bounds.hpp:30-38"""
    c1: float = 0.0
    c2: float = 1.0
    d: int = 1

    def cost(self, n: float, l: int, p: int) -> float:
        return self.c1 * self.d * n + self.c2 * (n + float(l) * p)


@dataclass
class QuadraturePlan:
    l: int = 0
    n: int = 0
    cost: float = 0.0


def _scalar(fn, q: BoundQuery, *extra) -> float:
    out = C.c_double()
    check(fn(float(q.n), int(q.p), float(q.alpha), float(q.beta), int(q.kind), *extra, C.byref(out)))
    return out.value


def log_bound_at_rho(q: BoundQuery, rho: float) -> float:
    out = C.c_double()
    check(lib.pq_log_bound_at_rho(float(q.n), int(q.p), float(q.alpha), float(q.beta), int(q.kind), float(rho),
                                  C.byref(out)))
    return out.value


def bound_quartic(q: BoundQuery) -> np.ndarray:
    out = np.empty(4)
    check(lib.pq_bound_quartic(float(q.n), int(q.p), float(q.alpha), float(q.beta), int(q.kind), _dp(out)))
    return out


def theorem_bound(q: BoundQuery) -> float:
    return _scalar(lib.pq_theorem_bound, q)


def corollary_bound(q: BoundQuery) -> float:
    return _scalar(lib.pq_corollary_bound, q)


def quaderr(n: float, p: int, alpha: float, beta: float, kind: QuadKind) -> float:
    out = C.c_double()
    check(lib.pq_quaderr(float(n), p, float(alpha), float(beta), int(kind), C.byref(out)))
    return out.value


def quadnodes(eps: float, p: int, alpha: float, beta: float, kind: QuadKind) -> int:
    n = C.c_int()
    check(lib.pq_quadnodes(float(eps), p, float(alpha), float(beta), int(kind), C.byref(n)))
    return n.value


def setup_quadrature(eps: float, p: int, alpha: float, beta: float, kind: QuadKind,
                     cost: CostModel = CostModel()) -> QuadraturePlan:
    l, n, c = C.c_int(), C.c_int(), C.c_double()
    check(lib.pq_setup_quadrature(float(eps), p, float(alpha), float(beta), int(kind), cost.c1, cost.c2, cost.d,
                                  C.byref(l), C.byref(n), C.byref(c)))
    return QuadraturePlan(l.value, n.value, c.value)


# ---------------------------------------------------------------- Kronecker sums --------------

class KroneckerSum:
    """kron.hpp:16-53 — one to three square factors, vec order = row-major, leftmost slowest."""

    def __init__(self, factors: Sequence[np.ndarray]):
        fs = [np.ascontiguousarray(np.asarray(f, dtype=np.float64)) for f in factors]
        if not (1 <= len(fs) <= 3):
            raise ValueError("KroneckerSum: need one to three factors")
        for f in fs:
            if f.ndim != 2 or f.shape[0] != f.shape[1] or f.shape[0] == 0:
                raise ValueError("KroneckerSum: factors must be square and nonempty")
            if not np.all(np.isfinite(f)):
                raise ValueError("DenseMatrix: non-finite entry")
        self.factors = fs
        self._shape = np.array([f.shape[0] for f in fs], dtype=np.int32)
        self._flat = np.ascontiguousarray(np.concatenate([f.reshape(-1) for f in fs]))

    def order(self) -> int:
        return len(self.factors)

    def dim(self) -> int:
        return int(np.prod(self._shape.astype(np.int64)))

    def shape(self) -> list:
        return [int(s) for s in self._shape]

    def factor(self, d: int) -> np.ndarray:
        return self.factors[d]

    def scaled(self, s: float) -> "KroneckerSum":
        return KroneckerSum([s * f for f in self.factors])

    # C-ABI triple
    def _abi(self):
        return self.order(), _ip(self._shape), _dp(self._flat)


def infnorm_bound(a: KroneckerSum) -> float:
    out = C.c_double()
    d, sh, f = a._abi()
    check(lib.pq_infnorm_bound(d, sh, f, C.byref(out)))
    return out.value


def expm(a, scale: Optional[Sequence[float]] = None, ctx: Optional[Context] = None):
    """dense.hpp:194 — one matrix, or a batch expm(scale[i] * a) when `scale` is given."""
    ctx = ctx or default_context()
    if _is_device(a):
        import torch
        n = a.shape[0]
        batch = 1 if scale is None else len(scale)
        out = torch.empty((batch, n, n), dtype=torch.float64, device=a.device)
        sc = None if scale is None else torch.as_tensor(scale, dtype=torch.float64, device=a.device)
        check(lib.pq_expm(ctx.handle, n, batch, C.c_void_p(a.contiguous().data_ptr()),
                          C.c_void_p(sc.data_ptr()) if sc is not None else None, C.c_void_p(out.data_ptr()),
                          L.PQ_DEVICE))
        return out[0] if scale is None else out
    m = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ValueError("expm: matrix not square")
    n = m.shape[0]
    batch = 1 if scale is None else len(scale)
    out = np.empty((batch, n, n))
    sc = None if scale is None else np.ascontiguousarray(np.asarray(scale, dtype=np.float64))
    check(lib.pq_expm(ctx.handle, n, batch, C.c_void_p(m.ctypes.data), C.c_void_p(sc.ctypes.data) if sc is not None
                      else None, C.c_void_p(out.ctypes.data), L.PQ_HOST))
    return out[0] if scale is None else out


def _apply(fn, a: KroneckerSum, x, ctx: Optional[Context], what: str):
    ctx = ctx or default_context()
    n = a.dim()
    v = _Vec(x, n, what)
    if v.count != 1:
        raise ValueError(f"{what}: vector length mismatch")
    out = v.empty(1, n)
    d, sh, f = a._abi()
    check(fn(ctx.handle, d, sh, f, v.ptr, _out_ptr(out), v.space))
    return out.reshape(-1)


def mode_apply(ms: Sequence[np.ndarray], shape: Sequence[int], x, ctx: Optional[Context] = None):
    """kron.hpp:92-108 — (M_0 (x) ... (x) M_{d-1}) x."""
    if len(ms) != len(shape):
        raise ValueError("mode_apply: rank mismatch")
    for m, s in zip(ms, shape):
        if np.asarray(m).shape[0] != s:
            raise ValueError("mode_apply: factor extent mismatch")
    return _apply(lib.pq_mode_apply, KroneckerSum(ms), x, ctx, "mode_apply")


def kron_matvec(a: KroneckerSum, x, ctx: Optional[Context] = None):
    """kron.hpp:111-119"""
    return _apply(lib.pq_kron_matvec, a, x, ctx, "kron_matvec")


def exp_action(a: KroneckerSum, b, ctx: Optional[Context] = None):
    """kron.hpp:123-128 (phi_0)"""
    return _apply(lib.pq_exp_action, a, b, ctx, "exp_action")


# ---------------------------------------------------------------- phi engine ------------------

@dataclass
class PhiRequest:
    """phiaction.hpp:35-42"""
    p: int = 1
    eps: float = 1e-14
    mode: QuadKind = QuadKind.gauss_legendre
    l: Optional[int] = None
    cost: CostModel = field(default_factory=CostModel)
    threads: int = 1

    def _c(self) -> L.PhiRequestC:
        return L.PhiRequestC(self.p, self.eps, int(self.mode), 0 if self.l is None else 1,
                             0 if self.l is None else int(self.l), self.cost.c1, self.cost.c2, self.threads)


@dataclass
class PhiInfo:
    """phiaction.hpp:45-54"""
    l: int = 0
    n: int = 0
    points: int = 0
    mode: QuadKind = QuadKind.gauss_legendre
    alpha: float = 0.0
    beta: float = 0.0
    planned: bool = False
    plan_cost: float = 0.0


class PhiColumns:
    """phiaction.hpp:20-30 — cols[j-1] approximates phi_j(A) b, j = 1..p."""

    def __init__(self, dim: int, cols):
        self.dim = dim
        self.cols = cols  # (p, N) array or tensor

    def p(self) -> int:
        return int(self.cols.shape[0])

    def col(self, j: int):
        if j < 1 or j > self.p():
            raise IndexError("PhiColumns::col: index out of range")
        return self.cols[j - 1]


def _wrap(out, nb: int, p: int, n: int) -> list:
    out = out.reshape(nb, p, n)
    return [PhiColumns(n, out[m]) for m in range(nb)]


def phi_fixed_multi(a: KroneckerSum, bs, p: int, rule: QuadratureRule, threads: int = 1,
                    ctx: Optional[Context] = None) -> list:
    if p < 1:
        raise ValueError("phi_fixed: need p >= 1")
    ctx = ctx or default_context()
    n = a.dim()
    v = _Vec(bs, n, "phi_fixed")
    out = v.empty(v.count * p, n)
    d, sh, f = a._abi()
    x = np.ascontiguousarray(rule.nodes, dtype=np.float64)
    w = np.ascontiguousarray(rule.weights, dtype=np.float64)
    check(lib.pq_phi_fixed(ctx.handle, d, sh, f, v.count, v.ptr, p, rule.points(), _dp(x), _dp(w), _out_ptr(out),
                           v.space))
    return _wrap(out, v.count, p, n)


def phi_fixed(a: KroneckerSum, b, p: int, rule: QuadratureRule, threads: int = 1, ctx=None) -> PhiColumns:
    return phi_fixed_multi(a, [b], p, rule, threads, ctx)[0]


def phi_adaptive_multi(a: KroneckerSum, bs, p: int, eps: float, threads: int = 1, ctx=None, info: Optional[dict] = None):
    ctx = ctx or default_context()
    n = a.dim()
    v = _Vec(bs, n, "phi_adaptive")
    out = v.empty(v.count * p, n)
    pts = C.c_int()
    d, sh, f = a._abi()
    check(lib.pq_phi_adaptive(ctx.handle, d, sh, f, v.count, v.ptr, p, float(eps), _out_ptr(out), C.byref(pts),
                              v.space))
    if info is not None:
        info["points_used"] = pts.value
    return _wrap(out, v.count, p, n)


def phi_adaptive(a: KroneckerSum, b, p: int, eps: float, threads: int = 1, ctx=None, info=None) -> PhiColumns:
    return phi_adaptive_multi(a, [b], p, eps, threads, ctx, info)[0]


def squaring_step(y: PhiColumns, exps: Sequence[np.ndarray], shape: Sequence[int], ctx=None) -> None:
    """phiaction.hpp:255-272 — rewrites y's columns in place to phi_j(2A) b."""
    ctx = ctx or default_context()
    ex = KroneckerSum(exps)
    if ex.shape() != list(shape):
        raise ValueError("squaring_step: shape mismatch")
    p = y.p()
    d, sh, f = ex._abi()
    if _is_device(y.cols):
        cols = y.cols.contiguous()
        check(lib.pq_squaring_step(ctx.handle, d, sh, f, p, C.c_void_p(cols.data_ptr()), L.PQ_DEVICE))
        y.cols = cols
    else:
        cols = np.ascontiguousarray(np.asarray(y.cols, dtype=np.float64)).copy()
        check(lib.pq_squaring_step(ctx.handle, d, sh, f, p, C.c_void_p(cols.ctypes.data), L.PQ_HOST))
        y.cols = cols


def phi_with_plan(a: KroneckerSum, bs, p: int, l: int, n: int, mode: QuadKind, eps: float, threads: int = 1,
                  ctx=None, info: Optional[dict] = None) -> list:
    ctx = ctx or default_context()
    dim = a.dim()
    v = _Vec(bs, dim, "phi_with_plan")
    out = v.empty(v.count * p, dim)
    pts = C.c_int()
    d, sh, f = a._abi()
    check(lib.pq_phi_with_plan(ctx.handle, d, sh, f, v.count, v.ptr, p, l, n, int(mode), float(eps), _out_ptr(out),
                               C.byref(pts), v.space))
    if info is not None:
        info["points_used"] = pts.value
    return _wrap(out, v.count, p, dim)


def _info(ci: L.PhiInfoC) -> PhiInfo:
    return PhiInfo(ci.l, ci.n, ci.points, QuadKind(ci.mode), ci.alpha, ci.beta, bool(ci.planned), ci.plan_cost)


def phiquadmv_multi(a: KroneckerSum, bs, req: PhiRequest, info: Optional[PhiInfo] = None, ctx=None) -> list:
    ctx = ctx or default_context()
    dim = a.dim()
    v = _Vec(bs, dim, "phiquadmv")
    out = v.empty(v.count * req.p, dim)
    ci = L.PhiInfoC()
    d, sh, f = a._abi()
    rc = req._c()
    check(lib.pq_phiquadmv(ctx.handle, d, sh, f, v.count, v.ptr, C.byref(rc), _out_ptr(out), C.byref(ci), v.space))
    if info is not None:
        info.__dict__.update(_info(ci).__dict__)
    return _wrap(out, v.count, req.p, dim)


def phiquadmv(a: KroneckerSum, b, req: PhiRequest, info: Optional[PhiInfo] = None, ctx=None) -> PhiColumns:
    return phiquadmv_multi(a, [b], req, info, ctx)[0]


def phi_0p(a: KroneckerSum, bs, req: PhiRequest, info: Optional[PhiInfo] = None, ctx=None):
    """phi_0 (exp_action) and phi_1..phi_p (phiquadmv) of every RHS in one call -> (phi0 [nb,N], cols [nb,p,N])."""
    ctx = ctx or default_context()
    dim = a.dim()
    v = _Vec(bs, dim, "phi_0p")
    out0 = v.empty(v.count, dim)
    out = v.empty(v.count * req.p, dim)
    ci = L.PhiInfoC()
    d, sh, f = a._abi()
    rc = req._c()
    check(lib.pq_phi_0p(ctx.handle, d, sh, f, v.count, v.ptr, C.byref(rc), _out_ptr(out0), _out_ptr(out), C.byref(ci),
                        v.space))
    if info is not None:
        info.__dict__.update(_info(ci).__dict__)
    return out0, out.reshape(v.count, req.p, dim)


def phi_lincomb(a: KroneckerSum, bs, rule: QuadratureRule, threads: int = 1, ctx=None):
    """phiaction.hpp:355-389 — sum_j phi_j(A) b_j, one quadrature sweep, no squaring."""
    ctx = ctx or default_context()
    dim = a.dim()
    v = _Vec(bs, dim, "phi_lincomb")
    if v.count < 1:
        raise ValueError("phi_lincomb: need at least one vector")
    out = v.empty(1, dim)
    d, sh, f = a._abi()
    x = np.ascontiguousarray(rule.nodes, dtype=np.float64)
    w = np.ascontiguousarray(rule.weights, dtype=np.float64)
    check(lib.pq_phi_lincomb(ctx.handle, d, sh, f, v.count, v.ptr, rule.points(), _dp(x), _dp(w), _out_ptr(out),
                             v.space))
    return out.reshape(-1)


# ---------------------------------------------------------------- integrators -----------------

@dataclass
class PhiTerm:
    """integrators.hpp:20-23"""
    k: int = 1
    c: float = 0.0


@dataclass
class ExpRKTableau:
    """integrators.hpp:32-38 (increment form)."""
    stages: int = 1
    order: int = 1
    c: list = field(default_factory=list)
    a: list = field(default_factory=list)   # a[i][j] -> list[PhiTerm]
    b: list = field(default_factory=list)   # b[j] -> list[PhiTerm]

    def _c(self):
        rows, cols, ks, coefs = [], [], [], []
        for i, row in enumerate(self.a):
            for j, terms in enumerate(row):
                for t in terms:
                    rows.append(i); cols.append(j); ks.append(t.k); coefs.append(t.c)
        for j, terms in enumerate(self.b):
            for t in terms:
                rows.append(-1); cols.append(j); ks.append(t.k); coefs.append(t.c)
        keep = [np.ascontiguousarray(np.asarray(self.c, dtype=np.float64)), np.asarray(rows, np.int32),
                np.asarray(cols, np.int32), np.asarray(ks, np.int32), np.asarray(coefs, np.float64)]
        tc = L.TableauC(self.stages, self.order, _dp(keep[0]), len(rows), _ip(keep[1]), _ip(keep[2]), _ip(keep[3]),
                        _dp(keep[4]))
        return tc, keep


def _builtin(id_: int, c2: float) -> ExpRKTableau:
    t = L.TableauC()
    check(lib.pq_builtin_tableau(id_, c2, C.byref(t)))
    st = t.stages
    tab = ExpRKTableau(st, t.order, [t.c[i] for i in range(st)], [[[] for _ in range(st)] for _ in range(st)],
                       [[] for _ in range(st)])
    for e in range(t.nterms):
        term = PhiTerm(t.k[e], t.coef[e])
        if t.row[e] == -1:
            tab.b[t.col[e]].append(term)
        else:
            tab.a[t.row[e]][t.col[e]].append(term)
    return tab


def exp_euler_tableau() -> ExpRKTableau:
    return _builtin(0, 0.0)


def exp_rk2_tableau(c2: float = 0.5) -> ExpRKTableau:
    if not (0.0 < c2 <= 1.0):
        raise ValueError("exp_rk2_tableau: need c2 in (0,1]")
    return _builtin(1, c2)


def exp_rk3_tableau(c2: float = 1.0 / 3.0) -> ExpRKTableau:
    if not (0.0 < c2 <= 1.0):
        raise ValueError("exp_rk3_tableau: need c2 in (0,1]")
    return _builtin(2, c2)


def etdrk4_tableau() -> ExpRKTableau:
    """Krogstad's fourth-order ETDRK4 in the reference's increment form (config 4)."""
    return _builtin(3, 0.0)


@dataclass
class IntegrationResult:
    u: object
    steps: int
    phi_calls: int


def _source(f) -> tuple:
    """f: None (zero), ('cubic', s1, s3), ('constant', vec) or a Python callable f(t, u) -> array."""
    keep = []
    if f is None:
        return L.SourceC(L.PQ_SOURCE_ZERO, 0.0, 0.0, None, L.SOURCE_CB(0), None), keep
    if isinstance(f, tuple) and f[0] == "cubic":
        return L.SourceC(L.PQ_SOURCE_CUBIC, float(f[1]), float(f[2]), None, L.SOURCE_CB(0), None), keep
    if isinstance(f, tuple) and f[0] == "constant":
        vec = f[1]
        if _is_device(vec):
            ptr = C.cast(C.c_void_p(vec.data_ptr()), L.dp)
        else:
            vec = np.ascontiguousarray(np.asarray(vec, dtype=np.float64))
            ptr = _dp(vec)
        keep.append(vec)
        return L.SourceC(L.PQ_SOURCE_CONSTANT, 0.0, 0.0, ptr, L.SOURCE_CB(0), None), keep

    def cb(t, u, out, n, user):
        try:
            uu = np.ctypeslib.as_array(u, (n,))
            r = np.asarray(f(t, uu.copy()), dtype=np.float64).reshape(-1)
            if r.size != n:
                return 1
            np.ctypeslib.as_array(out, (n,))[:] = r
            return 0
        except Exception:
            return 1

    c = L.SOURCE_CB(cb)
    keep.append(c)
    return L.SourceC(L.PQ_SOURCE_CALLBACK, 0.0, 0.0, None, c, None), keep


def integrate(a: KroneckerSum, f, u0, t0: float, t_end: float, m: int, tab: ExpRKTableau,
              base: PhiRequest = PhiRequest(), ctx=None) -> IntegrationResult:
    """integrators.hpp:193-202 — m steps of erk_step; f is a source spec (see _source)."""
    ctx = ctx or default_context()
    dim = a.dim()
    v = _Vec(u0, dim, "integrate")
    out = v.empty(1, dim)
    src, keep = _source(f)
    tc, tkeep = tab._c()
    rc = base._c()
    calls = C.c_int()
    d, sh, fac = a._abi()
    check(lib.pq_integrate(ctx.handle, d, sh, fac, C.byref(src), v.ptr, float(t0), float(t_end), int(m), C.byref(tc),
                           C.byref(rc), _out_ptr(out), C.byref(calls), v.space))
    return IntegrationResult(out.reshape(-1), m, calls.value)


def erk_step(a: KroneckerSum, f, tau: float, t: float, u, tab: ExpRKTableau, base: PhiRequest = PhiRequest(),
             ctx=None):
    """integrators.hpp:160-184 with a fresh PhiEngine(a, tau, base); returns (u_next, phi_calls)."""
    ctx = ctx or default_context()
    dim = a.dim()
    v = _Vec(u, dim, "erk_step")
    out = v.empty(1, dim)
    src, keep = _source(f)
    tc, tkeep = tab._c()
    rc = base._c()
    calls = C.c_int()
    d, sh, fac = a._abi()
    check(lib.pq_erk_step(ctx.handle, d, sh, fac, C.byref(src), float(tau), float(t), v.ptr, C.byref(tc), C.byref(rc),
                          _out_ptr(out), C.byref(calls), v.space))
    return out.reshape(-1), calls.value
