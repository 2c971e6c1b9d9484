"""Pins of the oracle's objective, GN Hessian, PCG, OT init, blur, GN and apply (CPU).

Pins: finite differences, brute force (dense assembly, unit-vector probing,
north-west-corner coupling), textbook properties of CG, exact special cases.
"""
import numpy as np
import pytest

from oracle import hysco_oracle as O
from synth import phantom

H = (1.1, 0.9, 1.25)


def _smooth_pair(shape, seed):
    """Small positive test images with zero margins (no method arithmetic)."""
    rng = np.random.default_rng(seed)
    n1, n2, n3 = shape
    Ip = np.zeros(shape)
    Im = np.zeros(shape)
    Ip[..., 2:n3 - 2] = rng.uniform(0.5, 2.0, (n1, n2, n3 - 4))
    Im[..., 2:n3 - 2] = rng.uniform(0.5, 2.0, (n1, n2, n3 - 4))
    return Ip, Im


def _rand_b(shape, seed, amp=0.3, h3=H[2]):
    n1, n2, n3 = shape
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((n1, n2, n3 + 1))
    return b * (amp * h3 / np.abs(np.diff(b, axis=2)).max())


# ---------------------------------------------------------------- objective

def test_identical_images_zero_field():
    I = np.random.default_rng(1).uniform(0, 1, (3, 4, 6))
    st = O.evaluate(I, I, np.zeros((3, 4, 7)), H)
    assert st.D == 0 and st.S == 0 and st.P == 0 and st.J == 0
    assert np.array_equal(st.grad, np.zeros((3, 4, 7)))


def test_infeasible_is_infinite():
    I = np.ones((2, 2, 4))
    b = np.zeros((2, 2, 5))
    b[0, 1, 2] = H[2] * 1.0          # Db = +1 and -1 on the adjacent cells
    st = O.evaluate(I, I, b, H)
    assert st.infeasible and np.isinf(st.J) and st.grad is None


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gradient_matches_central_fd(seed):
    shape = (3, 4, 7)
    Ip, Im = _smooth_pair(shape, seed)
    b = _rand_b(shape, seed + 10)
    st = O.evaluate(Ip, Im, b, H)
    rng = np.random.default_rng(seed + 20)
    for _ in range(5):
        v = rng.standard_normal(b.shape)
        e = 1e-6
        fd = (O.evaluate(Ip, Im, b + e * v, H).J - O.evaluate(Ip, Im, b - e * v, H).J) / (2 * e)
        an = float(np.sum(st.grad * v))
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(an))


# ---------------------------------------------------------------- GN Hessian

def _dense_H(st, shape):
    N = shape[0] * shape[1] * (shape[2] + 1)
    return np.stack([O.hessvec(st, np.eye(N)[k].reshape(shape[0], shape[1], shape[2] + 1)).ravel()
                     for k in range(N)], 1)


def test_hessian_symmetric_spd_and_diag_by_probing():
    shape = (4, 4, 4)                 # 4x4x5 nodes
    Ip, Im = _smooth_pair((4, 4, 8), 3)
    Ip, Im = Ip[..., 2:6], Im[..., 2:6]
    b = _rand_b(shape, 4)
    st = O.evaluate(Ip, Im, b, H)
    Hd = _dense_H(st, shape)
    assert np.abs(Hd - Hd.T).max() <= 1e-12 * np.abs(Hd).max()
    assert np.linalg.eigvalsh(0.5 * (Hd + Hd.T)).min() > 0
    assert np.allclose(O.hess_diag(st).ravel(), np.diag(Hd), rtol=1e-13, atol=0)
    # data+barrier part (H - alpha hd L) is tridiagonal along PE: zero across columns
    Lm = np.stack([O.laplacian(np.eye(Hd.shape[0])[k].reshape(4, 4, 5), H).ravel()
                   for k in range(Hd.shape[0])], 1)
    T = (Hd - st.alpha * st.hd * Lm).reshape(4, 4, 5, 4, 4, 5)
    for i in range(4):
        for j in range(4):
            for i2 in range(4):
                for j2 in range(4):
                    if (i, j) != (i2, j2):
                        assert np.all(T[i, j, :, i2, j2, :] == 0)
            blk = T[i, j, :, i, j, :]
            assert np.all(np.triu(blk, 2) == 0) and np.all(np.tril(blk, -2) == 0)


def test_hessian_equals_fd_of_gradient_at_zero_residual():
    """At r = 0 the GN Hessian is the exact Hessian: I-_j = I+_{j+1}, b = h3/2,
    interior support (queries at half-integers, away from interpolation kinks)."""
    n1, n2, n3 = 3, 3, 10
    rng = np.random.default_rng(7)
    Ip = np.zeros((n1, n2, n3))
    Ip[..., 3:7] = rng.uniform(0.5, 1.5, (n1, n2, 4))
    Im = np.zeros_like(Ip)
    Im[..., :-1] = Ip[..., 1:]
    b = np.full((n1, n2, n3 + 1), H[2] / 2)
    st = O.evaluate(Ip, Im, b, H)
    assert np.abs(st.r).max() < 1e-15
    q = rng.standard_normal(b.shape) * 1e-3
    e = 1e-4
    fd = (O.evaluate(Ip, Im, b + e * q, H).grad - O.evaluate(Ip, Im, b - e * q, H).grad) / (2 * e)
    Hq = O.hessvec(st, q)
    assert np.linalg.norm(fd - Hq) <= 1e-6 * np.linalg.norm(Hq)


# ---------------------------------------------------------------- PCG

def test_pcg_identity_and_exact_jacobi_one_iteration():
    rng = np.random.default_rng(0)
    rhs = rng.standard_normal(20)
    x, it, _, rel = O.pcg(lambda v: v, rhs, np.ones(20), maxit=10, tol=0.1)
    assert it == 1 and np.allclose(x, rhs) and rel < 1e-14
    dg = rng.uniform(1, 5, 20)
    x, it, _, rel = O.pcg(lambda v: dg * v, rhs, dg, maxit=10, tol=0.1)
    assert it == 1 and np.allclose(x, rhs / dg)


def test_pcg_dense_solve_and_krylov_minimality():
    rng = np.random.default_rng(1)
    n = 8
    B = rng.standard_normal((n, n))
    A = B.T @ B + np.eye(n)
    rhs = rng.standard_normal(n)
    Md = np.diag(A).copy()
    x, it, _, _ = O.pcg(lambda v: A @ v, rhs, Md, maxit=50, tol=1e-14)
    assert np.allclose(x, np.linalg.solve(A, rhs), rtol=1e-8, atol=1e-10)
    # k-th PCG iterate minimises the A-norm error over K_k(M^-1 A, M^-1 rhs)
    xs = np.linalg.solve(A, rhs)
    for k in (1, 2, 3, 5):
        xk, _, _, _ = O.pcg(lambda v: A @ v, rhs, Md, maxit=k, tol=0.0, fixed=True)
        K = [rhs / Md]
        for _ in range(k - 1):
            K.append((A @ K[-1]) / Md)
        V = np.linalg.qr(np.stack(K, 1))[0]
        y = np.linalg.solve(V.T @ A @ V, V.T @ rhs)     # Galerkin = A-norm minimiser
        assert np.allclose(xk, V @ y, rtol=1e-8, atol=1e-10)
        assert (xk - xs) @ A @ (xk - xs) <= (V @ y - xs) @ A @ (V @ y - xs) * (1 + 1e-9)


def test_pcg_early_stop_relative_residual():
    rng = np.random.default_rng(2)
    n = 30
    B = rng.standard_normal((n, n))
    A = B.T @ B + 0.1 * np.eye(n)
    rhs = rng.standard_normal(n)
    x, it, _, rel = O.pcg(lambda v: A @ v, rhs, np.diag(A).copy(), maxit=10, tol=0.1)
    assert rel < 0.1 or it == 10
    if it < 10:
        _, _, _, rel_prev = O.pcg(lambda v: A @ v, rhs, np.diag(A).copy(), maxit=it - 1, tol=0.0, fixed=True)
        assert rel_prev >= 0.1


# ---------------------------------------------------------------- block preconditioner (R20)

def test_block_pe_equals_column_blocks_of_probed_hessian():
    """hess_block_pe = the per-PE-column tridiagonal blocks of H_J, read off the
    dense H assembled by unit-vector probing of hessvec (brute force)."""
    shape = (3, 4, 5)                 # 3x4x6 nodes
    Ip, Im = _smooth_pair((3, 4, 9), 11)
    Ip, Im = Ip[..., 2:7], Im[..., 2:7]
    st = O.evaluate(Ip, Im, _rand_b(shape, 12), H)
    Hd = _dense_H(st, shape).reshape(3, 4, 6, 3, 4, 6)
    d, e = O.hess_block_pe(st)
    for i in range(3):
        for j in range(4):
            blk = Hd[i, j, :, i, j, :]
            assert np.allclose(np.diag(blk), d[i, j], rtol=1e-13, atol=0)
            assert np.allclose(np.diag(blk, 1), e[i, j], rtol=1e-12, atol=1e-12 * np.abs(blk).max())
            assert np.all(np.triu(blk, 2) == 0)


def test_thomas_equals_dense_solve():
    rng = np.random.default_rng(5)
    n1, n2, P = 3, 2, 9
    e = rng.uniform(-1, 1, (n1, n2, P - 1))
    d = np.abs(np.concatenate([e, np.zeros((n1, n2, 1))], -1)) + np.abs(
        np.concatenate([np.zeros((n1, n2, 1)), e], -1)) + rng.uniform(0.1, 1, (n1, n2, P))
    r = rng.standard_normal((n1, n2, P))
    z = O.solve_tridiag_pe(d, e, r)
    for i in range(n1):
        for j in range(n2):
            T = np.diag(d[i, j]) + np.diag(e[i, j], 1) + np.diag(e[i, j], -1)
            assert np.allclose(z[i, j], np.linalg.solve(T, r[i, j]), rtol=1e-12, atol=1e-12)


def test_block_pcg_exact_in_one_iteration_without_inplane_coupling():
    """With no in-plane coupling of H_J the column blocks ARE H_J, so
    block-preconditioned CG solves H q = -grad exactly in one iteration:
    (a) a single PE column (n1 = n2 = 1), (b) alpha = 0 (no regulariser)."""
    for shape, alpha in (((1, 1, 12), 300.0), ((3, 4, 8), 0.0)):
        n1, n2, n3 = shape
        Ip, Im = _smooth_pair((n1, n2, n3 + 4), 21)
        Ip, Im = Ip[..., 2:n3 + 2], Im[..., 2:n3 + 2]
        st = O.evaluate(Ip, Im, _rand_b(shape, 22), H, alpha=alpha)
        rhs = -st.grad
        x, it, _, rel = O.pcg(lambda v: O.hessvec(st, v), rhs, O.make_precond(st, "block"), maxit=10, tol=1e-12)
        Hd = _dense_H(st, shape)
        xs = np.linalg.solve(Hd, rhs.ravel()).reshape(rhs.shape)
        assert it == 1 and rel < 1e-10
        assert np.linalg.norm(x - xs) <= 1e-8 * np.linalg.norm(xs)


def test_block_pcg_is_galerkin_over_block_krylov_space():
    """k-th block-PCG iterate minimises the H-norm error over K_k(M^-1 H, M^-1 rhs)
    with M the column-block preconditioner (textbook CG property, brute force)."""
    shape = (3, 3, 5)
    Ip, Im = _smooth_pair((3, 3, 9), 31)
    Ip, Im = Ip[..., 2:7], Im[..., 2:7]
    st = O.evaluate(Ip, Im, _rand_b(shape, 32), H)
    Hd = _dense_H(st, shape)
    Minv = O.make_precond(st, "block")
    rhs = -st.grad
    xs = np.linalg.solve(Hd, rhs.ravel())
    for k in (1, 2, 3):
        xk, _, _, _ = O.pcg(lambda v: O.hessvec(st, v), rhs, Minv, maxit=k, tol=0.0, fixed=True)
        K = [Minv(rhs).ravel()]
        for _ in range(k - 1):
            K.append(Minv((Hd @ K[-1]).reshape(rhs.shape)).ravel())
        V = np.linalg.qr(np.stack(K, 1))[0]
        y = np.linalg.solve(V.T @ Hd @ V, V.T @ rhs.ravel())
        assert np.allclose(xk.ravel(), V @ y, rtol=1e-7, atol=1e-9 * np.abs(V @ y).max())


def test_block_pcg_needs_fewer_iterations_than_jacobi():
    """On a synthetic pair the block preconditioner reaches the paper's 0.1
    relative residual in fewer PCG iterations than Jacobi."""
    p = phantom.make_pair((10, 9, 24), (1.25, 1.25, 1.25), 3)
    b0, _ = O.ot_init(p.Ip.astype(np.float64), p.Im.astype(np.float64), 1.25)
    st = O.evaluate(p.Ip.astype(np.float64), p.Im.astype(np.float64), b0, (1.25, 1.25, 1.25))
    its = {}
    for kind in ("jacobi", "block"):
        _, it, _, rel = O.pcg(lambda v: O.hessvec(st, v), -st.grad, O.make_precond(st, kind), maxit=50, tol=0.1)
        assert rel < 0.1
        its[kind] = it
    assert its["block"] < its["jacobi"]


# ---------------------------------------------------------------- OT initialisation

def test_ot_identical_is_zero_and_swap_negates():
    rng = np.random.default_rng(3)
    Ip = rng.uniform(0, 100, (3, 4, 12))
    Im = rng.uniform(0, 100, (3, 4, 12))
    b0, _ = O.ot_init(Ip, Ip, 1.25, blur=False)
    assert np.array_equal(b0, np.zeros_like(b0))
    b1, _ = O.ot_init(Ip, Im, 1.25, blur=False)
    b2, _ = O.ot_init(Im, Ip, 1.25, blur=False)
    assert np.array_equal(b1, -b2)
    assert np.all(b1[..., 0] == 0) and np.all(b1[..., -1] == 0)


def test_ot_constant_images_degenerate():
    b0, _ = O.ot_init(np.full((2, 2, 5), 3.0), np.full((2, 2, 5), 3.0), 1.0)
    assert np.array_equal(b0, np.zeros((2, 2, 6)))


@pytest.mark.parametrize("c", [1, 2, 3])
def test_ot_recovers_integer_constant_shift_exactly(c):
    """I+ = i shifted by +c cells, I- by -c: with eps = 0, b0 = c*h3 on nodes with 0 < C < 1."""
    rng = np.random.default_rng(c)
    m = 32
    base = np.zeros(m)
    base[9:23] = rng.uniform(0.5, 2.0, 14)
    ip = np.roll(base, c)
    im = np.roll(base, -c)
    h3 = 1.25
    b = O.ot_column(ip, im, h3)
    Cp, Cm = O.cdf(ip), O.cdf(im)
    t = 1e-12                       # cumsum may end at 1 - ulp before the last node
    inside = (Cp > t) & (Cp < 1 - t) & (Cm > t) & (Cm < 1 - t)
    assert inside.sum() >= 3
    assert np.allclose(b[inside], c * h3, rtol=0, atol=1e-13)


def test_ot_shift_recovered_on_volume_with_small_eps():
    n3 = 32
    base = np.zeros(n3)
    base[10:22] = np.hanning(14)[1:13] + 0.2
    Ip = np.broadcast_to(np.roll(base, 2), (2, 2, n3))
    Im = np.broadcast_to(np.roll(base, -2), (2, 2, n3))
    b0, _ = O.ot_init(Ip, Im, 1.0, eps=1e-3, blur=False, feas_cap=np.inf)
    mid = b0[..., 12:20]
    assert np.abs(mid - 2.0).max() < 0.02        # error ~ eps-proportional


def _nw_corner_map(wp, wm, K):
    """Brute force: split each cell's (uniform) mass into K sub-atoms at the sub-cell
    centres, couple + to - with the north-west-corner rule (the monotone coupling),
    and return a function mapping a cumulative mass level r to the - position
    whose atom receives the + mass at level r."""
    posp = (np.repeat(np.arange(len(wp)), K) + (np.tile(np.arange(K), len(wp)) + 0.5) / K)
    posm = (np.repeat(np.arange(len(wm)), K) + (np.tile(np.arange(K), len(wm)) + 0.5) / K)
    mp = np.repeat(wp / K, K)
    mm = np.repeat(wm / K, K)
    plan = []                                   # (cum_start, cum_end, x+, x-)
    i = j = 0
    cum = 0.0
    rp, rm = mp[0], mm[0]
    while i < len(mp) and j < len(mm):
        t = min(rp, rm)
        plan.append((cum, cum + t, posp[i], posm[j]))
        cum += t
        rp -= t
        rm -= t
        if rp <= 1e-15:
            i += 1
            rp = mp[i] if i < len(mp) else 0
        if rm <= 1e-15:
            j += 1
            rm = mm[j] if j < len(mm) else 0

    def to_minus(r):
        for (a, b_, _, xm) in plan:
            if a <= r <= b_:
                return xm
        return plan[-1][3]
    return to_minus


def test_ot_matches_brute_force_monotone_coupling():
    rng = np.random.default_rng(11)
    m = 6
    ip = rng.uniform(0.2, 1.0, m)
    im = rng.uniform(0.2, 1.0, m)
    wp, wm = ip / ip.sum(), im / im.sum()
    Cp, Cm = O.cdf(ip), O.cdf(im)
    for K, tol in ((10, 0.1), (100, 0.01), (1000, 0.001)):
        f = _nw_corner_map(wp, wm, K)
        for l in range(1, m):
            # + mass below node l is Cp(l); where it lands in - is Q-(Cp(l))
            assert abs(f(Cp[l]) - O.quantile(Cm, Cp[l])) <= tol
    # the field map is then h3 (T- - T+)/2 with T+(l) = (l + Q-(Cp(l)))/2 etc.
    h3 = 1.3
    b = O.ot_column(ip, im, h3)
    for l in range(m + 1):
        Tp = 0.5 * (O.quantile(Cp, Cp[l]) + O.quantile(Cm, Cp[l]))
        Tm = 0.5 * (O.quantile(Cp, Cm[l]) + O.quantile(Cm, Cm[l]))
        assert abs(Tp - 0.5 * (l + O.quantile(Cm, Cp[l]))) < 1e-12
        assert abs(b[l] - h3 * (Tm - Tp) / 2) < 1e-12


def test_quantile_definition_and_vectorised_agree():
    rng = np.random.default_rng(5)
    C = O.cdf(rng.uniform(0.01, 1.0, 9))
    r = np.concatenate([rng.uniform(0, 1, 50), C, [0.0, 1.0, -0.1]])
    assert np.allclose(O.quantile(C, r), O.quantile_vec(C, r), rtol=0, atol=1e-14)
    # right-inverse on the CDF's own knots: Q(C(x)) = x
    assert np.allclose(O.quantile(C, C), np.arange(10), atol=1e-12)
    q = O.quantile(C, np.sort(rng.uniform(0, 1, 40)))
    assert np.all(np.diff(q) >= 0)


def test_ot_maps_monotone():
    rng = np.random.default_rng(8)
    ip, im = rng.uniform(0, 5, 30) + 0.1, rng.uniform(0, 5, 30) + 0.1
    Cp, Cm = O.cdf(ip), O.cdf(im)
    Tp = 0.5 * (O.quantile_vec(Cp, Cp) + O.quantile_vec(Cm, Cp))
    Tm = 0.5 * (O.quantile_vec(Cp, Cm) + O.quantile_vec(Cm, Cm))
    assert np.all(np.diff(Tp) >= 0) and np.all(np.diff(Tm) >= 0)


# ---------------------------------------------------------------- blur

def test_blur_constant_delta_and_smoothing():
    c = np.full((5, 6, 7), 2.5)
    assert np.allclose(O.blur3(c), 2.5, atol=1e-14)
    w = np.exp(-0.5)
    w1 = np.array([w, 1.0, w]) / (1 + 2 * w)          # [0.27406862, 0.45186276, 0.27406862]
    assert abs(w1[0] - 0.27406862) < 1e-8 and abs(w1[1] - 0.45186276) < 1e-8
    d = np.zeros((6, 6, 6))
    d[2, 3, 4] = 1.0
    out = O.blur3(d)
    ref = np.zeros_like(d)
    ref[1:4, 2:5, 3:6] = w1[:, None, None] * w1[None, :, None] * w1[None, None, :]
    assert np.allclose(out, ref, atol=1e-15)
    # periodic wrap at the corner
    d = np.zeros((4, 4, 4))
    d[0, 0, 0] = 1.0
    out = O.blur3(d)
    assert abs(out[3, 3, 3] - w1[0] ** 3) < 1e-15
    # S decreases for a zero-margin field (periodic = Neumann there)
    rng = np.random.default_rng(2)
    b = np.zeros((10, 10, 11))
    b[2:-2, 2:-2, 2:-2] = rng.standard_normal((6, 6, 7))
    assert O.smoothness_quadform(O.blur3(b), H) < O.smoothness_quadform(b, H)


def test_feasibility_guard():
    Ip = np.zeros((1, 1, 12))
    Im = np.zeros((1, 1, 12))
    Ip[0, 0, 1] = 100.0
    Im[0, 0, 10] = 100.0                # far apart narrow bumps: a steep OT map
    b0, info = O.ot_init(Ip, Im, 1.0, blur=False)
    assert info["max_Db_raw"] >= 0.95 and info["scaled"]
    assert abs(np.abs(O.diff_pe(b0, 1.0)).max() - 0.95) < 1e-12


# ---------------------------------------------------------------- GN and apply

def test_gn_identical_images_stays_zero():
    I = np.random.default_rng(4).uniform(0, 1, (3, 3, 6))
    b, st, rep = O.gauss_newton(I, I, np.zeros((3, 3, 7)), H, max_gn=3)
    assert np.array_equal(b, np.zeros_like(b)) and rep["J"] == 0


def test_gn_monotone_and_recovers_synthetic_pair():
    pair = phantom.make_config("C1_16x16x8")
    h = pair.h
    b0, _ = O.ot_init(pair.Ip, pair.Im, h[2])
    st0 = O.evaluate(pair.Ip, pair.Im, b0, h)
    b, st, rep = O.gauss_newton(pair.Ip, pair.Im, b0, h, max_gn=10, max_pcg=10, fixed=True)
    Js = [st0.J] + [r["J"] for r in rep["history"]]
    assert all(Js[k + 1] <= Js[k] for k in range(len(Js) - 1))
    assert rep["gn_iters"] == 10 and rep["pcg_iters"] == 100
    Tp, Tm = O.apply_correction(pair.Ip, pair.Im, b, h[2])
    ri = O.relative_improvement(pair.Ip, pair.Im, Tp, Tm)
    Tp0, Tm0 = O.apply_correction(pair.Ip, pair.Im, b0, h[2])
    assert ri > 90.0 and ri >= O.relative_improvement(pair.Ip, pair.Im, Tp0, Tm0)


def test_apply_special_cases_and_true_field():
    rng = np.random.default_rng(9)
    Ip, Im = rng.uniform(0, 1, (2, 3, 8)), rng.uniform(0, 1, (2, 3, 8))
    Tp, Tm = O.apply_correction(Ip, Im, np.zeros((2, 3, 9)), 1.25)
    assert np.array_equal(Tp, Ip) and np.array_equal(Tm, Im)
    b = _rand_b((2, 3, 8), 5)
    Tp, Tm = O.apply_correction(Ip, Im, b, 1.25)
    Sp, Sm = O.apply_correction(Im, Ip, -b, 1.25)
    assert np.array_equal(Tp, Sm) and np.array_equal(Tm, Sp)
    # the analytic field corrects the generated pair (continuum-exact generator)
    pair = phantom.make_pair((12, 10, 32), (1.25, 1.25, 1.25), seed=3)
    Tp, Tm = O.apply_correction(pair.Ip, pair.Im, pair.b_true, 1.25)
    assert O.relative_improvement(pair.Ip, pair.Im, Tp, Tm) >= 95.0
