"""BASELINE.json configurations as seeded synthetic operators (no dataset exists for this path).

Every builder returns the phi ARGUMENT's factors, i.e. the Kronecker factors of -tau*A, exactly as
the reference CLI passes `prob.a.scaled(-tau)` (phiquad_cli.cpp:110), plus the request parameters.
Right-hand sides are iid N(0,1) from numpy's PCG64 with seed 1000 + k (RHS k); the same bytes feed
the GPU engine and the CPU reference.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def tridiag(n: int, lo: float, di: float, up: float) -> np.ndarray:
    t = np.zeros((n, n))
    i = np.arange(n)
    t[i, i] = di
    t[i[1:], i[1:] - 1] = lo
    t[i[:-1], i[:-1] + 1] = up
    return t


def fd_laplacian(n: int, h: float) -> np.ndarray:
    """(1/h^2) tridiag(-1, 2, -1) with Dirichlet ends (the reference fe_laplacian_1d, problems.hpp:63-75)."""
    return tridiag(n, -1.0, 2.0, -1.0) / (h * h)


def advection_diffusion(n: int, h: float, d: float, b: float) -> np.ndarray:
    """d/h^2 tridiag(-1,2,-1) + b/(2h) tridiag(-1,0,1) (sub -1, sup +1): BASELINE config 2."""
    return d * fd_laplacian(n, h) + (b / (2.0 * h)) * tridiag(n, -1.0, 0.0, 1.0)


def variable_diffusion(n: int, h: float) -> np.ndarray:
    """(1/h^2) D^T diag(a(x_{i+1/2})) D, a(x) = 1 + sin(2 pi x)/2, D the Dirichlet difference
    matrix on the n interior nodes of [0, 1] (BASELINE config 5)."""
    xh = (np.arange(n + 1) + 0.5) * h        # x_{i+1/2}, i = 0..n (faces)
    a = 1.0 + 0.5 * np.sin(2.0 * np.pi * xh)
    A = np.zeros((n, n))
    i = np.arange(n)
    A[i, i] = a[:-1] + a[1:]
    A[i[:-1], i[:-1] + 1] = -a[1:-1]
    A[i[1:], i[1:] - 1] = -a[1:-1]
    return A / (h * h)


@dataclass
class Workload:
    name: str
    d: int
    n: int
    tau: float
    p: int
    eps: float
    mode: int                     # 0 Gauss-Legendre, 1 Clenshaw-Curtis
    nb: int = 1
    factors: list = field(default_factory=list)   # factors of -tau*A
    A: list = field(default_factory=list)         # factors of A
    note: str = ""

    @property
    def N(self) -> int:
        return self.n ** self.d

    def rhs(self, k: int = 0) -> np.ndarray:
        return np.random.default_rng(1000 + k).standard_normal(self.N)

    def flops_per_exp_action(self) -> float:
        """F_exp = 2 N sum_k n_k (dense)."""
        return 2.0 * self.N * self.d * self.n


def config(idx: int, n: int | None = None) -> Workload:
    """BASELINE.json configs[idx-1]; `n` overrides the grid size (reduced parity cases)."""
    if idx == 1:
        n = n or 64
        A = [fd_laplacian(n, 1.0 / (n + 1))] * 2
        w = Workload("cfg1_lap2d_n64_gl_p3", 2, n, 1e-2, 3, 1e-8, 0, 1, A=A)
    elif idx == 2:
        n = n or 128
        h = 1.0 / (n + 1)
        A = [advection_diffusion(n, h, d, b) for d, b in ((1.0, 10.0), (0.5, 0.0), (0.1, -5.0))]
        w = Workload("cfg2_advdiff3d_n128_cc_p4", 3, n, 5e-3, 4, 1e-10, 1, 1, A=A)
    elif idx == 3:
        n = n or 256
        A = [fd_laplacian(n, 1.0 / (n + 1))] * 3
        w = Workload("cfg3_lap3d_n256_gl_p3_8rhs", 3, n, 1e-3, 3, 1e-10, 0, 8, A=A)
    elif idx == 4:
        n = n or 128
        A = [0.01 * fd_laplacian(n, 1.0 / (n + 1))] * 3
        w = Workload("cfg4_allen_cahn3d_n128_etdrk4", 3, n, 1e-3, 3, 1e-14, 0, 1, A=A,
                     note="ETDRK4 dt=1e-3, 100 steps, f(u) = u - u^3")
    elif idx == 5:
        n = n or 512
        A = [variable_diffusion(n, 1.0 / (n + 1))] * 3
        w = Workload("cfg5_vardiff3d_n512_gl_p6", 3, n, 1e-3, 6, 1e-12, 0, 1, A=A)
    else:
        raise ValueError(f"unknown config {idx}")
    w.factors = [np.ascontiguousarray(-w.tau * a) for a in w.A]
    return w


def allen_cahn_u0(N: int, seed: int = 2024) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-0.9, 0.9, N)
