"""Pins of the oracle's push-forward matrices, distortion simulator and
least-squares correction (readings R27-R29 in DESIGN.md).

Pins: closed forms (b = 0 -> identity, integer-voxel b -> shift matrix,
half-voxel b -> two-point average), mass conservation, consistency with the
separately pinned Jacobian-modulation transform of Eq.(1) (push forward, then
pull back, recovers the true image in local means), the exact
normal-equation solution against a least-squares solve of the stacked system
by a different algorithm (LAPACK lstsq on [A+; A-; sqrt(lambda) D1]), the
b = 0 / lambda = 0 mean, exact recovery of a simulated true image as
lambda -> 0, the sign symmetry of the pair, and monotone smoothing in lambda.
"""
import numpy as np
import pytest

from oracle import hysco_oracle as O
from synth import phantom


def test_push_forward_identity_at_zero():
    for s in (+1.0, -1.0):
        A = O.push_forward_matrix(np.zeros(10), 1.3, s)
        assert np.array_equal(A, np.eye(9))


@pytest.mark.parametrize("m", [1, 2, -3])
def test_push_forward_integer_shift(m):
    h3, n3 = 1.7, 12
    for s in (+1.0, -1.0):
        A = O.push_forward_matrix(np.full(n3 + 1, m * h3), h3, s)
        E = np.zeros((n3, n3))
        for k in range(n3):
            j = k + int(s) * m
            if 0 <= j < n3:
                E[j, k] = 1.0                    # mass shifted out of [0, n3) is dropped
        assert np.allclose(A, E, atol=1e-12, rtol=0)


def test_push_forward_half_voxel():
    h3, n3 = 2.0, 7
    A = O.push_forward_matrix(np.full(n3 + 1, 0.5 * h3), h3, +1.0)
    for k in range(n3):
        assert A[k, k] == pytest.approx(0.5, abs=1e-15)
        if k + 1 < n3:
            assert A[k + 1, k] == pytest.approx(0.5, abs=1e-15)
    assert np.count_nonzero(A) == 2 * n3 - 1


def test_push_forward_mass_and_band():
    h3 = 1.25
    b = phantom.random_feasible_b((3, 4, 40), h3, seed=7, amp=0.8).astype(np.float64)
    for idx in np.ndindex(3, 4):
        for s in (+1.0, -1.0):
            A = O.push_forward_matrix(b[idx], h3, s)
            assert (A >= 0).all()
            u = np.arange(40) + s * 0.5 * (b[idx][:-1] + b[idx][1:]) / h3
            assert (np.diff(u) > 0).all()         # feasible b: the map is monotone
            for k in range(40):
                nz = np.nonzero(A[:, k])[0]
                assert set(nz) <= {int(np.floor(u[k])), int(np.floor(u[k])) + 1}
                if 0.0 <= u[k] <= 39.0:
                    assert A[:, k].sum() == pytest.approx(1.0, abs=1e-12)


def _smooth_case(n3, L=60.0, amp=2.0):
    """Smooth true image and field map on one column of length L mm."""
    h3 = L / n3
    xc = (np.arange(n3) + 0.5) * h3
    xn = np.arange(n3 + 1) * h3
    T = np.exp(-((xc - 0.5 * L) / (0.15 * L)) ** 2) + 0.5 * np.exp(-((xc - 0.35 * L) / (0.05 * L)) ** 2)
    b = amp * np.sin(2 * np.pi * xn / L) * np.exp(-((xn - 0.5 * L) / (0.3 * L)) ** 2)
    return T, b, h3


def test_push_forward_mass_conservation():
    T, b, h3 = _smooth_case(96)
    T[:10] = 0.0
    T[-10:] = 0.0                                  # no mass near the ends: none is truncated
    for s in (+1.0, -1.0):
        I = O.push_forward(T[None], b[None], h3, s)[0]
        assert I.sum() == pytest.approx(T.sum(), rel=1e-12)


@pytest.mark.parametrize("n3", [128, 512])
def test_push_forward_then_jacobian_modulation(n3):
    """T[A t, b, +-v] ~ t (Eq.(1) mass preservation).  Hat splitting
    onto a stretched lattice leaves an aliasing ripple of a few per cent that
    does not shrink with h (sum_k hat(j - k delta) != 1/delta unless 1/delta is
    an integer), so pointwise agreement is pinned loosely and local means
    (16 windows) tightly; the wrong sign is far off."""
    T, b, h3 = _smooth_case(n3)
    for s in (+1.0, -1.0):
        I = O.push_forward(T[None], b[None], h3, s)
        back = O.mp_transform(I, b[None], h3, s)[0]
        wrong = O.mp_transform(I, b[None], h3, -s)[0]
        rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
        assert rel(back, T) < 0.07
        assert rel(back.reshape(16, -1).mean(1), T.reshape(16, -1).mean(1)) < 0.01
        assert rel(wrong, T) > 0.3


def test_simulated_pair_differs_and_correction_aligns():
    T, b, h3 = _smooth_case(200)
    Ip, Im = O.simulate_pair(T[None], b[None], h3)
    Tp, Tm = O.apply_correction(Ip, Im, b[None], h3)
    assert np.linalg.norm(Ip - Im) > 0.1 * np.linalg.norm(T)
    assert O.relative_improvement(Ip, Im, Tp, Tm) > 95.0


def test_lsq_zero_b_zero_lambda_is_mean():
    rng = np.random.default_rng(1)
    Ip, Im = rng.uniform(0, 2, (2, 3, 17)), rng.uniform(0, 2, (2, 3, 17))
    x = O.lsq_correct(Ip, Im, np.zeros((2, 3, 18)), 1.1, lam=0.0)
    assert np.allclose(x, 0.5 * (Ip + Im), atol=1e-12, rtol=0)


@pytest.mark.parametrize("lam", [0.0, 0.05, 2.0])
def test_lsq_matches_stacked_lstsq(lam):
    h3, n3 = 1.3, 23
    rng = np.random.default_rng(3)
    b = phantom.random_feasible_b((2, 2, n3), h3, seed=5, amp=0.7).astype(np.float64)
    Ip, Im = rng.uniform(0, 2, (2, 2, n3)), rng.uniform(0, 2, (2, 2, n3))
    x = O.lsq_correct(Ip, Im, b, h3, lam=lam)
    D1 = np.diff(np.eye(n3), axis=0)
    for idx in np.ndindex(2, 2):
        M = np.vstack([O.push_forward_matrix(b[idx], h3, 1.0), O.push_forward_matrix(b[idx], h3, -1.0),
                       np.sqrt(lam) * D1])
        rhs = np.concatenate([Ip[idx], Im[idx], np.zeros(n3 - 1)])
        ref = np.linalg.lstsq(M, rhs, rcond=None)[0]
        assert np.allclose(x[idx], ref, atol=1e-9, rtol=0)


def test_lsq_recovers_simulated_truth():
    T, b, h3 = _smooth_case(120)
    Ip, Im = O.simulate_pair(T[None], b[None], h3)
    x0 = O.lsq_correct(Ip, Im, b[None], h3, lam=1e-10)[0]
    assert np.linalg.norm(x0 - T) / np.linalg.norm(T) < 1e-6
    x = O.lsq_correct(Ip, Im, b[None], h3, lam=0.05)[0]
    assert np.linalg.norm(x - T) / np.linalg.norm(T) < 0.05


def test_lsq_sign_symmetry():
    h3, n3 = 0.9, 19
    rng = np.random.default_rng(4)
    b = phantom.random_feasible_b((2, 3, n3), h3, seed=9, amp=0.6).astype(np.float64)
    Ip, Im = rng.uniform(0, 2, (2, 3, n3)), rng.uniform(0, 2, (2, 3, n3))
    assert np.allclose(O.lsq_correct(Ip, Im, b, h3), O.lsq_correct(Im, Ip, -b, h3), atol=1e-12, rtol=0)


def test_lsq_smoothing_monotone_in_lambda():
    h3, n3 = 1.0, 30
    rng = np.random.default_rng(6)
    b = phantom.random_feasible_b((1, 1, n3), h3, seed=2, amp=0.5).astype(np.float64)
    Ip, Im = rng.uniform(0, 2, (1, 1, n3)), rng.uniform(0, 2, (1, 1, n3))
    norms = [np.linalg.norm(np.diff(O.lsq_correct(Ip, Im, b, h3, lam=l)[0, 0])) for l in (0.01, 0.1, 1.0)]
    assert norms[0] > norms[1] > norms[2]
