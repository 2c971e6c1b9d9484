"""Pins of the oracle's ADMM solver (readings R21-R26 in DESIGN.md).

Pins: the z-update against the periodic operator applied by rolls (not the
FFT), finite-difference gradient and exact GN Hessian of the column objective,
an exact one-Newton-step b-update on a quadratic column objective (dense
solve), the residual-balancing rule, and solver properties (proximal-point
monotonicity with alpha = 0, objective decrease on a synthetic pair).
"""
import numpy as np
import pytest

from oracle import hysco_oracle as O
from synth import phantom

H = (1.1, 0.9, 1.25)


def _pair(shape, seed):
    rng = np.random.default_rng(seed)
    n1, n2, n3 = shape
    Ip = np.zeros(shape)
    Im = np.zeros(shape)
    Ip[..., 2:n3 - 2] = rng.uniform(0.5, 2.0, (n1, n2, n3 - 4))
    Im[..., 2:n3 - 2] = rng.uniform(0.5, 2.0, (n1, n2, n3 - 4))
    return Ip, Im


def _rand_b(shape, seed, amp=0.3, h3=H[2]):
    n1, n2, n3 = shape
    b = np.random.default_rng(seed).standard_normal((n1, n2, n3 + 1))
    return b * (amp * h3 / np.abs(np.diff(b, axis=2)).max())


def test_z_update_solves_periodic_system():
    rng = np.random.default_rng(0)
    b = rng.standard_normal((6, 5, 9))
    u = rng.standard_normal((6, 5, 9))
    for alpha, rho in ((300.0, 40.0), (1.0, 1e-3), (0.0, 2.0)):
        z = O.admm_z_update(b, u, H, alpha, rho)
        lhs = alpha * O.periodic_laplacian_xy(z, H) + rho * z
        assert np.linalg.norm(lhs - rho * (b + u)) <= 1e-11 * np.linalg.norm(rho * (b + u))


def test_periodic_laplacian_is_symmetric_psd_with_constant_nullspace():
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal((2, 4, 5, 3))
    Lx, Ly = O.periodic_laplacian_xy(x, H), O.periodic_laplacian_xy(y, H)
    assert abs(np.sum(Lx * y) - np.sum(x * Ly)) <= 1e-12 * np.abs(np.sum(Lx * y))
    assert np.sum(Lx * x) >= 0
    assert np.abs(O.periodic_laplacian_xy(np.ones((4, 5, 3)), H)).max() == 0


@pytest.mark.parametrize("seed", [3, 4])
def test_column_objective_gradient_matches_fd(seed):
    shape = (3, 2, 10)
    Ip, Im = _pair(shape, seed)
    b = _rand_b(shape, seed + 10)
    v = _rand_b(shape, seed + 20)
    rho = 37.0
    cs = O.admm_b_objective(Ip, Im, b, v, H, rho=rho)
    q = np.random.default_rng(seed).standard_normal(b.shape)
    e = 1e-6
    Fp = np.sum(O.admm_b_objective(Ip, Im, b + e * q, v, H, rho=rho, derivs=False).F)
    Fm = np.sum(O.admm_b_objective(Ip, Im, b - e * q, v, H, rho=rho, derivs=False).F)
    fd = (Fp - Fm) / (2 * e)
    assert abs(fd - np.sum(cs.grad * q)) <= 1e-6 * abs(fd)


def test_column_hessian_exact_at_zero_residual():
    """At r = 0 (I-_j = I+_{j+1}, b = h3/2, interior support) the GN column
    Hessian tridiag(d, e) is the exact Hessian: FD of the gradient."""
    n1, n2, n3 = 2, 2, 10
    rng = np.random.default_rng(7)
    Ip = np.zeros((n1, n2, n3))
    Ip[..., 3:7] = rng.uniform(0.5, 1.5, (n1, n2, 4))
    Im = np.zeros_like(Ip)
    Im[..., :-1] = Ip[..., 1:]
    b = np.full((n1, n2, n3 + 1), H[2] / 2)
    v = b + 0.1 * rng.standard_normal(b.shape)
    cs = O.admm_b_objective(Ip, Im, b, v, H, rho=5.0)
    q = rng.standard_normal(b.shape) * 1e-3
    e = 1e-4
    fd = (O.admm_b_objective(Ip, Im, b + e * q, v, H, rho=5.0).grad
          - O.admm_b_objective(Ip, Im, b - e * q, v, H, rho=5.0).grad) / (2 * e)
    Hq = cs.d * q
    Hq[..., :-1] += cs.e * q[..., 1:]
    Hq[..., 1:] += cs.e * q[..., :-1]
    assert np.linalg.norm(fd - Hq) <= 1e-6 * np.linalg.norm(Hq)


def test_b_update_exact_newton_on_quadratic_column_objective():
    """No data (zero images) and beta = 0: Fc = alpha S3 + rho hd/2 ||b - v||^2 is
    quadratic, so one GN step with gamma = 1 is the exact minimiser
    (alpha hd D3^T D3 / h3^2 + rho hd I) b = rho hd v (dense solve per column)."""
    shape = (2, 3, 7)
    Ip = np.zeros(shape)
    Im = np.zeros(shape)
    v = _rand_b(shape, 5, amp=0.2)
    alpha, rho = 300.0, 50.0
    b = O.admm_b_update(Ip, Im, np.zeros_like(v), v, H, alpha=alpha, beta=0.0, rho=rho, inner=1)
    hd = H[0] * H[1] * H[2]
    n = shape[2] + 1
    D = (np.eye(n, k=1)[:-1] - np.eye(n)[:-1]) / H[2]
    A = alpha * hd * D.T @ D + rho * hd * np.eye(n)
    for i in range(shape[0]):
        for j in range(shape[1]):
            ref = np.linalg.solve(A, rho * hd * v[i, j])
            assert np.allclose(b[i, j], ref, rtol=1e-10, atol=1e-12)


def test_rho_residual_balancing_rule():
    assert O.admm_rho_update(8.0, 100.0, 1.0) == (16.0, 0.5)     # primal residual large: rho up, u down
    assert O.admm_rho_update(8.0, 1.0, 100.0) == (4.0, 2.0)      # dual residual large: rho down, u up
    assert O.admm_rho_update(8.0, 3.0, 1.0) == (8.0, 1.0)


def test_admm_alpha_zero_is_monotone_proximal_point():
    """alpha = 0: z = b + u, so u stays 0 and each b-update is a proximal step on
    F: F(b_k) is non-increasing (Armijo descent on F + rho hd/2 ||b - b_prev||^2)."""
    p = phantom.make_pair((6, 5, 20), (1.25, 1.25, 1.25), 12)
    Ip, Im = p.Ip.astype(np.float64), p.Im.astype(np.float64)
    b0, _ = O.ot_init(Ip, Im, 1.25)
    Fs = []
    b, u = b0.copy(), np.zeros_like(b0)
    rho = 20.0
    for _ in range(6):
        b = O.admm_b_update(Ip, Im, b, b - u, p.h, alpha=0.0, rho=rho)
        z = O.admm_z_update(b, u, p.h, alpha=0.0, rho=rho)
        assert np.allclose(z, b + u)
        u = u + b - z
        assert np.abs(u).max() <= 1e-12 * max(np.abs(b).max(), 1.0)
        Fs.append(np.sum(O.admm_b_objective(Ip, Im, b, b, p.h, alpha=0.0, rho=0.0, derivs=False).F))
    assert all(Fs[k + 1] <= Fs[k] * (1 + 1e-12) for k in range(len(Fs) - 1))


def test_admm_reduces_objective_on_synthetic_pair():
    p = phantom.make_pair((10, 9, 24), (1.25, 1.25, 1.25), 3)
    Ip, Im = p.Ip.astype(np.float64), p.Im.astype(np.float64)
    b0, _ = O.ot_init(Ip, Im, 1.25)
    J0 = O.evaluate(Ip, Im, b0, p.h).J
    b, z, rep = O.admm(Ip, Im, b0, p.h, max_iter=15, fixed=True)
    st = O.evaluate(Ip, Im, b, p.h)
    assert np.isfinite(st.J) and st.J < 0.2 * J0
    assert rep["iters"] == 15 and rep["r_norm"][-1] < rep["r_norm"][0]


def test_b_update_column_stop_rule_col_tol():
    """R23 column stop ("different step sizes and stopping criteria for each
    image column"): a column takes no step when its GN step predicts a decrease
    -grad.q <= col_tol |Fc|.  On the quadratic column objective of the test
    above (zero images, beta = 0) from b = 0 the GN step is exact, q = A^{-1}
    rho hd v, so the ratio -grad.q / Fc(0) = 2 v^T (rho hd A^{-1}) v / ||v||^2
    has a dense-algebra closed form: 2 for a constant column (D3 v = 0) and
    small for an oscillating one.  With col_tol between the two ratios the
    oscillating columns stay exactly 0 and the constant columns reach the
    minimiser; col_tol = 0 moves every column, col_tol = inf none."""
    shape = (1, 4, 9)
    n = shape[2] + 1
    v = np.zeros((1, 4, n))
    v[0, 0] = 0.7                                   # constant
    v[0, 1] = -0.3
    v[0, 2] = 0.2 * (-1.0) ** np.arange(n)          # oscillating
    v[0, 3] = 0.1 * np.cos(np.pi * np.arange(n) * 0.9)
    alpha, rho = 300.0, 50.0
    hd = H[0] * H[1] * H[2]
    D = (np.eye(n, k=1)[:-1] - np.eye(n)[:-1]) / H[2]
    A = alpha * hd * D.T @ D + rho * hd * np.eye(n)
    ratio = [2.0 * v[0, j] @ np.linalg.solve(A, rho * hd * v[0, j]) / (v[0, j] @ v[0, j]) for j in range(4)]
    assert ratio[0] > 1.999 and ratio[1] > 1.999 and ratio[2] < 0.5 and ratio[3] < 0.5, ratio
    Z = np.zeros(shape)
    kw = dict(alpha=alpha, beta=0.0, rho=rho, inner=1)
    b = O.admm_b_update(Z, Z, np.zeros_like(v), v, H, col_tol=1.0, **kw)
    for j in range(4):
        if ratio[j] <= 1.0:
            assert np.array_equal(b[0, j], np.zeros(n)), j
        else:
            assert np.allclose(b[0, j], np.linalg.solve(A, rho * hd * v[0, j]), rtol=1e-10, atol=1e-13), j
    b = O.admm_b_update(Z, Z, np.zeros_like(v), v, H, col_tol=0.0, **kw)
    assert all(np.abs(b[0, j]).max() > 0 for j in range(4))
    b = O.admm_b_update(Z, Z, np.zeros_like(v), v, H, col_tol=np.inf, **kw)
    assert np.array_equal(b, np.zeros_like(v))
