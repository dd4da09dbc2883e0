"""GPU dense phi oracle for mid-size operators: phi_1..phi_p(A) b from ONE
exponential of the augmented matrix [[A, b e1^T], [0, J]] (reference oracle.hpp:15-45), assembled
on the host and exponentiated on the B200 -- beyond the reference's CPU guard N + p <= 1000.  An
algorithmically independent check of the quadrature + scaling-and-squaring pipeline at config 1's
full size (N = 4096; the augmented matrix is 4099 x 4099)."""
import numpy as np
import pytest

from conftest import rel2

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def dense_phi(pq, factors, b, p):
    n = len(b)
    dense = np.zeros((n, n))
    # Kronecker sum, leftmost factor slowest (kron.hpp:139-164)
    shape = [f.shape[0] for f in factors]
    for k, f in enumerate(factors):
        left = int(np.prod(shape[:k])) if k else 1
        right = int(np.prod(shape[k + 1:])) if k + 1 < len(shape) else 1
        dense += np.kron(np.kron(np.eye(left), f), np.eye(right))
    m = n + p
    aug = np.zeros((m, m))
    aug[:n, :n] = dense
    aug[:n, n] = b
    for j in range(1, p):
        aug[n + j - 1, n + j] = 1.0
    e = np.asarray(pq.expm(aug)).reshape(m, m)
    return [e[:n, n + j] for j in range(p)]


@pytest.mark.parametrize("cfg,n", [(1, None), (2, 16)])
def test_midsize_against_dense_augmented_exponential(pq, cfg, n):
    """config 1 at full size (2D Laplacian, N = 4096) and the headline advection-diffusion family at
    n = 16 (N = 4096, p = 4), at eps = 1e-14 so the comparison measures the engine, not the plan."""
    from paper_2211_00696_b200.workloads import config
    w = config(cfg, n=n)
    b = w.rhs(0)
    want = dense_phi(pq, w.factors, b, w.p)
    got = pq.phiquadmv(pq.KroneckerSum(w.factors), b, pq.PhiRequest(p=w.p, eps=1e-14,
                                                                   mode=pq.QuadKind.gauss_legendre))
    for j in range(w.p):
        assert rel2(got.col(j + 1), want[j]) <= 1e-11, j
