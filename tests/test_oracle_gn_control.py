"""Pins of the oracle's Gauss-Newton control flow (R14-R16).

`oracle.gn_armijo` is the GN / Armijo / stop-rule iteration that
`oracle.gauss_newton` runs on the field-map objective.  Here it runs on
quadratic objectives J(b) = 1/2 b^T A b - c^T b + J0 whose every decision has
a closed form:

* exact model H = A and an exact PCG solve: q = -A^{-1} grad, the full step
  lands on the minimiser, J(b + q) - J(b) = 1/2 grad.q, so gamma = 1 passes
  Armijo and the gradient vanishes;
* a model H = s A with s < 1 (too little curvature): q = -(1/s) A^{-1} grad and
  J(b + gamma q) - J(b) = gamma grad.q (1 - gamma / (2 s)), so the Armijo test
  J_t <= J + c1 gamma grad.q holds exactly when gamma <= 2 s (1 - c1): the
  number of halvings is the smallest k with 2^-k <= 2 s (1 - c1), and more than
  ls_max - 1 of them is a line-search failure;
* a feasible set max|b| < 1 (the barrier's role, Eq.(3)) that the full step
  leaves: the trial is rejected as infeasible and halved (R15);
* the three stop tests of P:284 (R16), each triggered by a constructed case
  where the other two cannot fire.
"""
import math

import numpy as np
import pytest

from oracle import hysco_oracle as O

C1 = 1e-4


class Quad:
    """J(b) = 1/2 b^T A b - c^T b + J0 on vectors b, feasible iff max|b| < bound."""

    def __init__(self, A, c, J0=0.0, bound=np.inf):
        self.A, self.c, self.J0, self.bound = np.asarray(A, float), np.asarray(c, float), J0, bound

    def __call__(self, b):
        st = type("St", (), {})()
        st.infeasible = bool(np.max(np.abs(b)) >= self.bound)
        if st.infeasible:
            st.J, st.grad = np.inf, None
            return st
        st.J = 0.5 * b @ self.A @ b - self.c @ b + self.J0
        st.grad = self.A @ b - self.c
        return st


def spd(n, seed, cond=10.0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return Q @ np.diag(np.geomspace(1.0, cond, n)) @ Q.T


def run(f, b0, s=1.0, max_gn=1, max_pcg=None, **kw):
    A = f.A
    n = len(b0)
    return O.gn_armijo(f, lambda st: (lambda v: s * (A @ v)), lambda st: s * np.diag(A), np.asarray(b0, float),
                       kw.pop("h3", 1.0), max_gn=max_gn, max_pcg=max_pcg or n, pcg_tol=0.0, **kw)


def halvings_expected(s, c1=C1):
    """smallest k >= 0 with 2^-k <= 2 s (1 - c1)."""
    k = 0
    while 2.0 ** -k > 2.0 * s * (1.0 - c1):
        k += 1
    return k


def test_full_newton_step_accepted_on_quadratic():
    A, c = spd(6, 1), np.random.default_rng(2).standard_normal(6)
    f = Quad(A, c)
    b, st, rep = run(f, np.zeros(6))
    assert rep["history"][0]["gamma"] == 1.0 and rep["ls_halvings"] == 0 and rep["f_evals"] == 2
    np.testing.assert_allclose(b, np.linalg.solve(A, c), rtol=1e-9, atol=1e-12)
    assert np.linalg.norm(st.grad) <= 1e-9 * np.linalg.norm(c)


@pytest.mark.parametrize("s", [0.7, 0.5, 0.3, 0.125, 0.04])
def test_armijo_halves_exactly_the_closed_form_count(s):
    A, c = spd(5, 3), np.random.default_rng(4).standard_normal(5)
    b0 = np.random.default_rng(5).standard_normal(5)
    f = Quad(A, c)
    k = halvings_expected(s)
    assert abs(2.0 ** -k - 2 * s * (1 - C1)) > 1e-3          # no decision sits on the threshold
    b, st, rep = run(f, b0, s=s)
    gam = 2.0 ** -k
    assert rep["ls_halvings"] == k and rep["f_evals"] == 2 + k and rep["gn_iters"] == 1
    assert rep["history"][0]["gamma"] == gam
    q = -np.linalg.solve(A, f(b0).grad) / s
    np.testing.assert_allclose(b, b0 + gam * q, rtol=1e-9, atol=1e-12)
    # the accepted J obeys the closed form J(b + gamma q) - J(b) = gamma g.q (1 - gamma/(2 s))
    gq = float(f(b0).grad @ q)
    assert math.isclose(st.J - f(b0).J, gam * gq * (1 - gam / (2 * s)), rel_tol=1e-9)


def test_parity_mode_accepts_full_step_even_if_J_rises():
    """armijo=False (R15 parity mode): the first feasible trial is taken."""
    A, c = spd(5, 3), np.random.default_rng(4).standard_normal(5)
    b0 = np.random.default_rng(5).standard_normal(5)
    f = Quad(A, c)
    b, st, rep = run(f, b0, s=0.125, armijo=False)
    assert rep["ls_halvings"] == 0 and rep["history"][0]["gamma"] == 1.0
    assert st.J > f(b0).J                                      # 1 - 1/(2 s) = -3 < 0: J went up


def test_infeasible_trial_is_halved():
    """Full step to the minimiser b* with max|b*| = 1.5 >= bound 1: rejected as
    infeasible, gamma = 1/2 lands at 0.75 b* (feasible; Armijo: 1/2 (1 - 1/4) >= c1)."""
    A = spd(4, 6)
    bstar = np.array([1.5, -0.3, 0.2, 0.9])
    f = Quad(A, A @ bstar, bound=1.0)
    for armijo in (True, False):
        b, st, rep = run(f, np.zeros(4), armijo=armijo)
        assert rep["ls_halvings"] == 1 and rep["f_evals"] == 3 and rep["history"][0]["gamma"] == 0.5
        np.testing.assert_allclose(b, 0.5 * bstar, rtol=1e-9)


def test_line_search_failure_after_ls_max_trials():
    """s = 1e-5 needs 16 halvings > ls_max - 1 = 9: LS_FAIL, b unchanged, GN stops."""
    A, c = spd(5, 7), np.random.default_rng(8).standard_normal(5)
    b0 = np.random.default_rng(9).standard_normal(5)
    f = Quad(A, c)
    assert halvings_expected(1e-5) == 16
    b, st, rep = run(f, b0, s=1e-5, max_gn=5)
    assert rep["stop_reason"] == O.STOP_LSFAIL and rep["gn_iters"] == 0
    assert rep["f_evals"] == 1 + 10 and rep["ls_halvings"] == 9
    assert np.array_equal(b, b0)
    # ls_max = 17 leaves room for the 16 halvings: accepted at gamma = 2^-16
    b, st, rep = run(f, b0, s=1e-5, ls_max=17)
    assert rep["stop_reason"] == O.STOP_MAXITER and rep["history"][0]["gamma"] == 2.0 ** -16


def test_stop_on_gradient():
    """Exact solve: grad(b1) ~ 0 <= 1e-2 ||grad(b0)|| -> STOP_GRAD after one step."""
    A, c = spd(6, 10), np.random.default_rng(11).standard_normal(6)
    b, st, rep = run(Quad(A, c), np.zeros(6), max_gn=10, fixed=False)
    assert rep["stop_reason"] == O.STOP_GRAD and rep["gn_iters"] == 1


def _one_cg_step_case(J0, h3):
    """A 2x2 coupled quadratic where ONE Jacobi-PCG iteration (a line search
    along grad) leaves ||grad|| well above 1e-2 ||grad0|| (so STOP_GRAD cannot
    fire in the first step)."""
    A = np.array([[1.0, 0.9], [0.9, 1.0]])
    c = np.array([1.0, 0.2])
    f = Quad(A, c, J0=J0)
    return f, dict(max_gn=10, max_pcg=1, fixed=False, h3=h3)


def test_stop_on_objective_change():
    """J0 = 1e12: |J_old - J| / |J_old| ~ 1e-12 <= 1e-4 -> STOP_DJ (grad test first fails)."""
    f, kw = _one_cg_step_case(1e12, 1.0)
    b, st, rep = run(f, np.zeros(2), **kw)
    assert np.linalg.norm(st.grad) > 1e-2 * np.linalg.norm(f(np.zeros(2)).grad)
    assert rep["stop_reason"] == O.STOP_DJ and rep["gn_iters"] == 1


def test_stop_on_field_map_change():
    """J(b0) = 0 (so |dJ| <= 1e-4 |J_old| = 0 is false) and h3 = 1e6: every step
    is below 1e-3 h3 -> STOP_DB (grad and dJ tests first fail)."""
    f, kw = _one_cg_step_case(0.0, 1e6)
    b, st, rep = run(f, np.zeros(2), **kw)
    assert rep["stop_reason"] == O.STOP_DB and rep["gn_iters"] == 1
    # with h3 = 1 the same step (max|q| ~ 0.6) is not small: no stop, 10 steps
    f, kw = _one_cg_step_case(0.0, 1.0)
    kw.update(tol_grad_rel=0.0)
    b, st, rep = run(f, np.zeros(2), **kw)
    assert rep["stop_reason"] == O.STOP_MAXITER and rep["gn_iters"] == 10


def test_fixed_mode_ignores_stop_rules_and_infeasible_start():
    """fixed: exactly max_gn steps although the DJ rule would stop after one
    (one CG iteration = exact line search along grad, so gamma = 1 passes)."""
    f, kw = _one_cg_step_case(1e12, 1.0)
    kw.update(fixed=True, max_gn=4)
    b, st, rep = run(f, np.zeros(2), **kw)
    assert rep["stop_reason"] == O.STOP_MAXITER and rep["gn_iters"] == 4 and rep["f_evals"] == 5
    A, c = spd(6, 10), np.random.default_rng(11).standard_normal(6)
    b, st, rep = run(Quad(A, c, bound=1.0), np.full(6, 2.0), max_gn=4)
    assert rep["stop_reason"] == O.STOP_INFEASIBLE and rep["gn_iters"] == 0 and rep["f_evals"] == 1


def test_gauss_newton_is_gn_armijo_on_the_field_map_objective():
    """gauss_newton() = gn_armijo(evaluate, hessvec, make_precond) (no other logic)."""
    rng = np.random.default_rng(12)
    Ip = np.zeros((3, 3, 10))
    Im = np.zeros((3, 3, 10))
    Ip[..., 2:8] = rng.uniform(0.5, 2, (3, 3, 6))
    Im[..., 2:8] = rng.uniform(0.5, 2, (3, 3, 6))
    h = (1.0, 1.1, 1.2)
    b0 = np.zeros((3, 3, 11))
    b1, _, r1 = O.gauss_newton(Ip, Im, b0, h, max_gn=3)
    b2, _, r2 = O.gn_armijo(lambda b: O.evaluate(Ip, Im, b, h), lambda st: (lambda v: O.hessvec(st, v)),
                            lambda st: O.hess_diag(st), b0, h[2], max_gn=3)
    assert np.array_equal(b1, b2) and r1["f_evals"] == r2["f_evals"] and r1["J"] == r2["J"]
