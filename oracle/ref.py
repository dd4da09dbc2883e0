"""TEST INFRASTRUCTURE ONLY — ctypes handle on the compiled reference (oracle/_ref/libpqref.so,
built by oracle/Makefile from the unmodified reference headers).  Used by tests/ as the parity
checker and by bench.py's `--impl reference` / cpu_baseline legs; never by the product.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

REF_SO = Path(__file__).resolve().parent / "_ref" / "libpqref.so"
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


def available() -> bool:
    return REF_SO.exists()


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Ref:
    """Thin wrapper: factors are a list of square numpy arrays; vectors numpy float64."""

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle` where /root/reference exists")
        self.lib = C.CDLL(str(REF_SO))
        self.lib.pqref_last_error.restype = C.c_char_p

    def _chk(self, rc: int) -> None:
        if rc:
            raise RefError(rc, self.lib.pqref_last_error().decode())

    @staticmethod
    def _kron(factors):
        fs = [np.ascontiguousarray(np.asarray(f, dtype=np.float64)) for f in factors]
        shape = np.array([f.shape[0] for f in fs], dtype=np.int32)
        flat = np.ascontiguousarray(np.concatenate([f.reshape(-1) for f in fs]))
        return len(fs), shape, flat, int(np.prod(shape.astype(np.int64)))

    @staticmethod
    def _p(a, t=dp):
        return a.ctypes.data_as(t)

    def rule(self, kind: int, m: int):
        x, w = np.empty(m), np.empty(m)
        self._chk(self.lib.pqref_rule(kind, m, self._p(x), self._p(w)))
        return x, w

    def quartic_roots(self, a3, a2, a1, a0=1.0):
        out = np.empty(8)
        self._chk(self.lib.pqref_quartic_roots(C.c_double(a3), C.c_double(a2), C.c_double(a1), C.c_double(a0),
                                               self._p(out)))
        return out[0::2] + 1j * out[1::2]

    def real_roots_greater_one(self, a3, a2, a1, a0=1.0):
        out, cnt = np.empty(4), C.c_int()
        self._chk(self.lib.pqref_real_roots_greater_one(C.c_double(a3), C.c_double(a2), C.c_double(a1),
                                                        C.c_double(a0), self._p(out), C.byref(cnt)))
        return list(out[: cnt.value])

    def _bound(self, name, n, p, alpha, beta, kind, *extra):
        out = C.c_double()
        fn = getattr(self.lib, name)
        self._chk(fn(C.c_double(n), C.c_int(p), C.c_double(alpha), C.c_double(beta), C.c_int(kind),
                     *[C.c_double(e) for e in extra], C.byref(out)))
        return out.value

    def log_bound_at_rho(self, n, p, alpha, beta, kind, rho):
        return self._bound("pqref_log_bound_at_rho", n, p, alpha, beta, kind, rho)

    def theorem_bound(self, n, p, alpha, beta, kind):
        return self._bound("pqref_theorem_bound", n, p, alpha, beta, kind)

    def corollary_bound(self, n, p, alpha, beta, kind):
        return self._bound("pqref_corollary_bound", n, p, alpha, beta, kind)

    def quaderr(self, n, p, alpha, beta, kind):
        return self._bound("pqref_quaderr", n, p, alpha, beta, kind)

    def bound_quartic(self, n, p, alpha, beta, kind):
        out = np.empty(4)
        self._chk(self.lib.pqref_bound_quartic(C.c_double(n), C.c_int(p), C.c_double(alpha), C.c_double(beta),
                                               C.c_int(kind), self._p(out)))
        return out

    def quadnodes(self, eps, p, alpha, beta, kind):
        n = C.c_int()
        self._chk(self.lib.pqref_quadnodes(C.c_double(eps), C.c_int(p), C.c_double(alpha), C.c_double(beta),
                                           C.c_int(kind), C.byref(n)))
        return n.value

    def setup_quadrature(self, eps, p, alpha, beta, kind, c1=0.0, c2=1.0, d=1):
        l, n, c = C.c_int(), C.c_int(), C.c_double()
        self._chk(self.lib.pqref_setup_quadrature(C.c_double(eps), C.c_int(p), C.c_double(alpha), C.c_double(beta),
                                                  C.c_int(kind), C.c_double(c1), C.c_double(c2), C.c_int(d),
                                                  C.byref(l), C.byref(n), C.byref(c)))
        return l.value, n.value, c.value

    def expm(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.empty_like(a)
        self._chk(self.lib.pqref_expm(C.c_int(a.shape[0]), self._p(a), self._p(out)))
        return out

    def _vec_op(self, name, factors, x):
        d, sh, fl, n = self._kron(factors)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        y = np.empty(n)
        self._chk(getattr(self.lib, name)(C.c_int(d), self._p(sh, ip), self._p(fl), self._p(x), self._p(y)))
        return y

    def mode_apply(self, mats, x):
        return self._vec_op("pqref_mode_apply", mats, x)

    def kron_matvec(self, factors, x):
        return self._vec_op("pqref_kron_matvec", factors, x)

    def exp_action(self, factors, b):
        return self._vec_op("pqref_exp_action", factors, b)

    def infnorm_bound(self, factors):
        d, sh, fl, n = self._kron(factors)
        out = C.c_double()
        self._chk(self.lib.pqref_infnorm_bound(C.c_int(d), self._p(sh, ip), self._p(fl), C.byref(out)))
        return out.value

    def phi_fixed(self, factors, bs, p, kind, points, threads=1):
        d, sh, fl, n = self._kron(factors)
        bs = np.ascontiguousarray(np.asarray(bs, dtype=np.float64).reshape(-1, n))
        out = np.empty((bs.shape[0], p, n))
        self._chk(self.lib.pqref_phi_fixed(C.c_int(d), self._p(sh, ip), self._p(fl), C.c_int(bs.shape[0]),
                                           self._p(bs), C.c_int(p), C.c_int(kind), C.c_int(points),
                                           C.c_int(threads), self._p(out)))
        return out

    def phi_adaptive(self, factors, bs, p, eps, threads=1):
        d, sh, fl, n = self._kron(factors)
        bs = np.ascontiguousarray(np.asarray(bs, dtype=np.float64).reshape(-1, n))
        out = np.empty((bs.shape[0], p, n))
        pts = C.c_int()
        self._chk(self.lib.pqref_phi_adaptive(C.c_int(d), self._p(sh, ip), self._p(fl), C.c_int(bs.shape[0]),
                                              self._p(bs), C.c_int(p), C.c_double(eps), C.c_int(threads),
                                              self._p(out), C.byref(pts)))
        return out, pts.value

    def squaring_step(self, exps, y):
        d, sh, fl, n = self._kron(exps)
        y = np.ascontiguousarray(np.asarray(y, dtype=np.float64)).copy()
        p = y.size // n
        self._chk(self.lib.pqref_squaring_step(C.c_int(d), self._p(sh, ip), self._p(fl), C.c_int(p), self._p(y)))
        return y.reshape(p, n)

    def phi_with_plan(self, factors, bs, p, l, n_param, kind, eps, threads=1):
        d, sh, fl, n = self._kron(factors)
        bs = np.ascontiguousarray(np.asarray(bs, dtype=np.float64).reshape(-1, n))
        out = np.empty((bs.shape[0], p, n))
        pts = C.c_int()
        self._chk(self.lib.pqref_phi_with_plan(C.c_int(d), self._p(sh, ip), self._p(fl), C.c_int(bs.shape[0]),
                                               self._p(bs), C.c_int(p), C.c_int(l), C.c_int(n_param), C.c_int(kind),
                                               C.c_double(eps), C.c_int(threads), self._p(out), C.byref(pts)))
        return out, pts.value

    def phiquadmv(self, factors, bs, p, eps, kind, fixed_l=-1, c1=0.0, c2=1.0, threads=1):
        d, sh, fl, n = self._kron(factors)
        bs = np.ascontiguousarray(np.asarray(bs, dtype=np.float64).reshape(-1, n))
        out = np.empty((bs.shape[0], p, n))
        ii, dd = np.zeros(4, np.int32), np.zeros(3)
        self._chk(self.lib.pqref_phiquadmv(C.c_int(d), self._p(sh, ip), self._p(fl), C.c_int(bs.shape[0]),
                                           self._p(bs), C.c_int(p), C.c_double(eps), C.c_int(kind), C.c_int(fixed_l),
                                           C.c_double(c1), C.c_double(c2), C.c_int(threads), self._p(out),
                                           self._p(ii, ip), self._p(dd)))
        info = dict(l=int(ii[0]), n=int(ii[1]), points=int(ii[2]), planned=bool(ii[3]), alpha=dd[0], beta=dd[1],
                    plan_cost=dd[2])
        return out, info

    def phi_lincomb(self, factors, bs, kind, points, threads=1):
        d, sh, fl, n = self._kron(factors)
        bs = np.ascontiguousarray(np.asarray(bs, dtype=np.float64).reshape(-1, n))
        out = np.empty(n)
        self._chk(self.lib.pqref_phi_lincomb(C.c_int(d), self._p(sh, ip), self._p(fl), C.c_int(bs.shape[0]),
                                             self._p(bs), C.c_int(kind), C.c_int(points), C.c_int(threads),
                                             self._p(out)))
        return out

    def phi_dense_oracle(self, factors, b, p, guard=1000):
        d, sh, fl, n = self._kron(factors)
        b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
        out = np.empty((p, n))
        self._chk(self.lib.pqref_phi_dense_oracle(C.c_int(d), self._p(sh, ip), self._p(fl), self._p(b), C.c_int(p),
                                                  C.c_int(guard), self._p(out)))
        return out

    def integrate(self, factors, source, u0, t0, t_end, m, tableau, c2=0.0, eps=1e-14, kind=0, threads=1,
                  src_vec=None):
        d, sh, fl, n = self._kron(factors)
        u0 = np.ascontiguousarray(u0, dtype=np.float64).reshape(-1)
        sv = np.ascontiguousarray(src_vec if src_vec is not None else np.zeros(1), dtype=np.float64)
        out = np.empty(n)
        calls = C.c_int()
        self._chk(self.lib.pqref_integrate(C.c_int(d), self._p(sh, ip), self._p(fl), C.c_int(source), self._p(sv),
                                           self._p(u0), C.c_double(t0), C.c_double(t_end), C.c_int(m),
                                           C.c_int(tableau), C.c_double(c2), C.c_double(eps), C.c_int(kind),
                                           C.c_int(threads), self._p(out), C.byref(calls)))
        return out, calls.value

    def fe_laplacian_1d(self, n_elem):
        out = np.empty((n_elem - 1, n_elem - 1))
        self._chk(self.lib.pqref_fe_laplacian_1d(C.c_int(n_elem), self._p(out)))
        return out
