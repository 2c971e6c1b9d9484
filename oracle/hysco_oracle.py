"""CPU fp64 oracle for the PyHySCO GN-PCG hot path (arXiv 2403.10706).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module.  The product path
(paper_2403_10706_b200, libhysco.so) never imports, links or calls it, and it
shares no code with the CUDA path.

Plain, slow, obviously-correct NumPy float64, written from PAPER.md (cited as
P:<line>) in the paper's order and notation.  Where the paper is silent or
garbled the reading taken is named R<n>; every reading is listed in DESIGN.md
§"Readings of the paper".

Conventions: the phase-encoding (PE) axis is the last axis.  Images
live on cells (n1, n2, n3); the field map b lives on the e3-staggered grid
(n1, n2, n3+1): cell centres in dims 1-2, nodes in dim 3.  b is in mm (R2).
Node l sits at l*h3, cell k is centred at (k+1/2)*h3.

Pins: every function here is checked in tests/test_oracle_*.py against closed
forms, invariants, brute force and the hand-derived worked example in
tests/golden/.  The one result with no independent pin is the field map after
a fixed number of GN-PCG iterations on a synthetic pair (parity unpinned as a
whole; pinned only through its pinned pieces), see DESIGN.md.  Push-forward /
least-squares pins: tests/test_oracle_lsq.py.
"""
from __future__ import annotations

import numpy as np

ALPHA_DEFAULT = 300.0   # P:100 "we fix alpha=300"
BETA_DEFAULT = 1e-4     # P:100 "and beta=1e-4"

# ---------------------------------------------------------------------------
# Linear operators of the discretization
# ---------------------------------------------------------------------------


def avg_pe(b):
    """Averaging operator A: nodes -> cell centres along PE."""
    return 0.5 * (b[..., :-1] + b[..., 1:])


def avg_pe_T(y):
    """A^T: cells -> nodes."""
    out = np.zeros(y.shape[:-1] + (y.shape[-1] + 1,))
    out[..., :-1] += 0.5 * y
    out[..., 1:] += 0.5 * y
    return out


def diff_pe(b, h3):
    """Finite-difference operator D: (Db)_k = (b_{k+1} - b_k)/h3, dimensionless (R2)."""
    return (b[..., 1:] - b[..., :-1]) / h3


def diff_pe_T(y, h3):
    """D^T: cells -> nodes."""
    out = np.zeros(y.shape[:-1] + (y.shape[-1] + 1,))
    out[..., :-1] -= y / h3
    out[..., 1:] += y / h3
    return out


def short_diff(b, axis):
    """Short forward difference along `axis` (n-1 differences), no scaling."""
    return np.diff(b, axis=axis)


def short_diff_T(y, axis):
    """Adjoint of short_diff along `axis`."""
    shp = list(y.shape)
    shp[axis] += 1
    out = np.zeros(shp)
    lo = [slice(None)] * y.ndim
    hi = [slice(None)] * y.ndim
    lo[axis] = slice(0, -1)
    hi[axis] = slice(1, None)
    out[tuple(lo)] -= y
    out[tuple(hi)] += y
    return out


def laplacian(b, h):
    """H b: negative Laplacian on the node array, L = sum_d D_d^T D_d / h_d^2 (Eq.(5), R3).

    Homogeneous Neumann (short differences), symmetric positive semi-definite,
    constants in the null space.
    """
    out = np.zeros(b.shape)
    for ax in range(3):
        out += short_diff_T(short_diff(b, ax), ax) / h[ax] ** 2
    return out


def smoothness_quadform(b, h):
    """b^T L b = sum_d ||D_d b||^2 / h_d^2."""
    return sum(float(np.sum(short_diff(b, ax) ** 2)) / h[ax] ** 2 for ax in range(3))


# ---------------------------------------------------------------------------
# Image model: 1D piecewise-linear interpolation along PE (R5)
# ---------------------------------------------------------------------------


def interp_pe(f, u):
    """Evaluate the piecewise-linear (hat-function) model of each column of f.

    f : (..., n3) samples at index positions 0..n3-1 (cell centres).
    u : (..., n3) query positions in index units (centre k at u = k).
    Model (R5): f(u) = sum_k f_k max(0, 1 - |u - k|), i.e. zero beyond one cell
    past the outer centres.  Returns (value, slope per index unit), the slope
    being the right-hand one at breakpoints.
    """
    n3 = f.shape[-1]
    fl = np.floor(u).astype(np.int64)
    t = u - fl

    def take(idx):
        ok = (idx >= 0) & (idx < n3)
        v = np.take_along_axis(f, np.clip(idx, 0, n3 - 1), axis=-1)
        return np.where(ok, v, 0.0)

    f0 = take(fl)
    f1 = take(fl + 1)
    return (1.0 - t) * f0 + t * f1, f1 - f0


# ---------------------------------------------------------------------------
# Barrier phi (Eq.(3))
# ---------------------------------------------------------------------------


def phi(z):
    """phi(z) = z^4/(1 - z^2) on (-1,1), +inf otherwise."""
    z = np.asarray(z, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(np.abs(z) < 1.0, z ** 4 / (1.0 - z ** 2), np.inf)


def dphi(z):
    """phi'(z) = 2 z^3 (2 - z^2)/(1 - z^2)^2."""
    z = np.asarray(z, dtype=np.float64)
    return 2.0 * z ** 3 * (2.0 - z ** 2) / (1.0 - z ** 2) ** 2


def d2phi(z):
    """phi''(z) = 2 z^2 (6 - 3 z^2 + z^4)/(1 - z^2)^3  (>= 0 on (-1,1))."""
    z = np.asarray(z, dtype=np.float64)
    return 2.0 * z ** 2 * (6.0 - 3.0 * z ** 2 + z ** 4) / (1.0 - z ** 2) ** 3


# ---------------------------------------------------------------------------
# Mass-preserving transform (Eq.(1))
# ---------------------------------------------------------------------------


def mp_transform(I, b, h3, sign):
    """T[I, b, sign*v] at the cell centres: I(x + sign*b(x) v) * (1 + sign*d_v b)(x).

    Geometric term via the averaging operator, modulation via the finite
    difference operator, both at cell centres.
    """
    n3 = I.shape[-1]
    k = np.arange(n3, dtype=np.float64)
    u = k + sign * avg_pe(b) / h3
    val, _ = interp_pe(np.asarray(I, np.float64), u)
    return val * (1.0 + sign * diff_pe(b, h3))


def apply_correction(Ip, Im, b, h3):
    """Jacobian-modulation correction: the two corrected images."""
    return mp_transform(Ip, b, h3, +1.0), mp_transform(Im, b, h3, -1.0)


# ---------------------------------------------------------------------------
# Objective J = D + alpha S + beta P, gradient, GN Hessian
# ---------------------------------------------------------------------------


class EvalState:
    """Everything evaluate() produces; the GN Hessian is applied from it."""
    pass


def evaluate(Ip, Im, b, h, alpha=ALPHA_DEFAULT, beta=BETA_DEFAULT):
    """Discrete objective (Eq.(6)) with gradient and GN-Hessian parts.

    D = hd/2 sum_k r_k^2, r = T[I+,b,v] - T[I-,b,-v]      (Eq.(2), midpoint rule P:105)
    S = hd/2 b^T L b                                       (Eq.(5))
    P = hd/2 sum_k phi((Db)_k)                             (Eq.(3), midpoint rule, R4)
    J = D + alpha S + beta P                               (Eq.(4)/(6))
    Infeasible (some |Db| >= 1): J = +inf, no gradient (R4, Eq.(3) "infinity else").
    """
    Ip = np.asarray(Ip, np.float64)
    Im = np.asarray(Im, np.float64)
    b = np.asarray(b, np.float64)
    h1, h2, h3 = (float(v) for v in h)
    hd = h1 * h2 * h3
    n3 = Ip.shape[-1]
    k = np.arange(n3, dtype=np.float64)

    st = EvalState()
    st.h, st.hd, st.alpha, st.beta = (h1, h2, h3), hd, alpha, beta
    Ab = avg_pe(b)
    Db = diff_pe(b, h3)
    st.Db = Db
    st.infeasible = bool(np.any(np.abs(Db) >= 1.0))

    up, um = k + Ab / h3, k - Ab / h3
    vp, sp = interp_pe(Ip, up)          # value, slope per index unit
    vm, sm = interp_pe(Im, um)
    Tp = vp * (1.0 + Db)
    Tm = vm * (1.0 - Db)
    r = Tp - Tm
    st.r = r

    st.D = 0.5 * hd * float(np.sum(r * r))
    st.S = 0.5 * hd * smoothness_quadform(b, (h1, h2, h3))
    if st.infeasible:
        st.P = np.inf
        st.J = np.inf
        st.grad = None
        return st
    st.P = 0.5 * hd * float(np.sum(phi(Db)))
    st.J = st.D + alpha * st.S + beta * st.P

    # Residual Jacobian J_r q = g*(A q) + s*(D q)  (product rule on Eq.(1))
    st.g = (sp / h3) * (1.0 + Db) + (sm / h3) * (1.0 - Db)
    st.s = vp + vm
    st.d2phi = d2phi(Db)
    st.b = b
    # grad J = hd J_r^T r + alpha hd L b + beta (hd/2) D^T phi'(Db)
    st.grad = (hd * (avg_pe_T(st.g * r) + diff_pe_T(st.s * r, h3))
               + alpha * hd * laplacian(b, (h1, h2, h3))
               + beta * 0.5 * hd * diff_pe_T(dphi(Db), h3))
    return st


def residual_jac(st, q):
    """J_r q."""
    return st.g * avg_pe(q) + st.s * diff_pe(q, st.h[2])


def residual_jac_T(st, y):
    """J_r^T y."""
    return avg_pe_T(st.g * y) + diff_pe_T(st.s * y, st.h[2])


def hessvec(st, q):
    """GN Hessian matvec (R12):

    H_J q = hd J_r^T J_r q + alpha hd L q + beta (hd/2) D^T diag(phi''(Db)) D q.
    """
    h3 = st.h[2]
    q = np.asarray(q, np.float64)
    return (st.hd * residual_jac_T(st, residual_jac(st, q))
            + st.alpha * st.hd * laplacian(q, st.h)
            + st.beta * 0.5 * st.hd * diff_pe_T(st.d2phi * diff_pe(q, h3), h3))


def hess_diag(st):
    """diag(H_J): the Jacobi preconditioner (R13).

    diag(J_r^T J_r)_l = sum_k (J_r)_{k,l}^2 = a_l^2 + c_{l-1}^2 with
    a_k = dr_k/db_k = g_k/2 - s_k/h3, c_k = dr_k/db_{k+1} = g_k/2 + s_k/h3;
    diag(L)_l = sum_d (#neighbours of l along d)/h_d^2;
    diag(D^T Phi D)_l = (phi''_{l-1} + phi''_l)/h3^2.
    """
    h1, h2, h3 = st.h
    a = st.g / 2.0 - st.s / h3
    c = st.g / 2.0 + st.s / h3
    shp = st.b.shape
    dJ = np.zeros(shp)
    dJ[..., :-1] += a ** 2
    dJ[..., 1:] += c ** 2
    dB = np.zeros(shp)
    dB[..., :-1] += st.d2phi / h3 ** 2
    dB[..., 1:] += st.d2phi / h3 ** 2
    dL = np.zeros(shp)
    for ax, hh in enumerate((h1, h2, h3)):
        n = shp[ax]
        cnt = np.full(n, 2.0)
        if n == 1:
            cnt[:] = 0.0
        else:
            cnt[0] = cnt[-1] = 1.0
        sh = [1, 1, 1]
        sh[ax] = n
        dL = dL + cnt.reshape(sh) / hh ** 2
    return st.hd * dJ + st.alpha * st.hd * dL + st.beta * 0.5 * st.hd * dB


def hess_block_pe(st):
    """Per-PE-column tridiagonal block of H_J: the block-diagonal preconditioner
    "more accurate (yet also more expensive)" than Jacobi (SURVEY §8(f)
    NEXT-1, reading R20 in DESIGN.md).

    Column block of H_J = its entries between nodes of one PE column.  The
    in-plane Laplacian couples different columns only, so inside a column it
    contributes its diagonal alone.  Returns (d, e):
      d = diag(H_J) (hess_diag, the Jacobi diagonal);
      e[..., l] = H_J[l, l+1] within the column, l = 0..n3-1:
        hd (J_r^T J_r)[l, l+1] = hd a_l c_l   (cell l holds a_l at l, c_l at l+1)
        alpha hd (D3^T D3 / h3^2)[l, l+1] = -alpha hd / h3^2
        beta hd/2 (D^T diag(phi'') D)[l, l+1] = -beta hd/2 phi''_l / h3^2.
    """
    h3 = st.h[2]
    a = st.g / 2.0 - st.s / h3
    c = st.g / 2.0 + st.s / h3
    e = st.hd * a * c - st.alpha * st.hd / h3 ** 2 - st.beta * 0.5 * st.hd * st.d2phi / h3 ** 2
    return hess_diag(st), e


def solve_tridiag_pe(d, e, r):
    """Solve T z = r for every PE column, T = tridiag(e, d, e) (symmetric,
    positive definite), by the Thomas algorithm (textbook LU without pivoting):
    forward  m_0 = d_0, m_l = d_l - e_{l-1}^2 / m_{l-1},
             y_0 = r_0 / m_0, y_l = (r_l - e_{l-1} y_{l-1}) / m_l;
    backward z_{n} = y_{n}, z_l = y_l - (e_l / m_l) z_{l+1}."""
    n = d.shape[-1]
    m = np.empty_like(d)
    y = np.empty_like(r)
    m[..., 0] = d[..., 0]
    y[..., 0] = r[..., 0] / m[..., 0]
    for l in range(1, n):
        m[..., l] = d[..., l] - e[..., l - 1] ** 2 / m[..., l - 1]
        y[..., l] = (r[..., l] - e[..., l - 1] * y[..., l - 1]) / m[..., l]
    z = np.empty_like(r)
    z[..., n - 1] = y[..., n - 1]
    for l in range(n - 2, -1, -1):
        z[..., l] = y[..., l] - (e[..., l] / m[..., l]) * z[..., l + 1]
    return z


def make_precond(st, kind="jacobi"):
    """The PCG preconditioner solve r -> z = M^{-1} r: "jacobi" (P:198-199,
    R13) or "block" (the per-PE-column tridiagonal block, R20)."""
    if kind == "jacobi":
        Md = hess_diag(st)
        return lambda r: r / Md
    if kind == "block":
        d, e = hess_block_pe(st)
        return lambda r: solve_tridiag_pe(d, e, r)
    raise ValueError(kind)


# ---------------------------------------------------------------------------
# PCG: up to maxit iterations, stop if relative residual < tol
# ---------------------------------------------------------------------------


def pcg(Hmul, rhs, Mdiag, maxit=10, tol=0.1, fixed=False):
    """Preconditioned CG (Hestenes-Stiefel / Saad Alg. 9.1), x0 = 0 (R14).

    Mdiag: the Jacobi diagonal (z = r / Mdiag), or a callable z = M^{-1}(r)
    (make_precond).  Returns (x, iterations, matvecs, final relative residual
    ||r||/||r0||).  In fixed mode all maxit iterations run (parity / timing
    mode, R14).
    """
    Minv = Mdiag if callable(Mdiag) else (lambda v: v / Mdiag)
    x = np.zeros_like(rhs)
    r = rhs.copy()
    r0 = float(np.linalg.norm(r))
    if r0 == 0.0:
        return x, 0, 0, 0.0
    z = Minv(r)
    p = z.copy()
    rz = float(np.sum(r * z))
    it = 0
    rel = 1.0
    for it in range(1, maxit + 1):
        Hp = Hmul(p)
        pHp = float(np.sum(p * Hp))
        if pHp <= 0.0:
            it -= 1
            break
        a = rz / pHp
        x = x + a * p
        r = r - a * Hp
        rel = float(np.linalg.norm(r)) / r0
        if not fixed and rel < tol:
            break
        z = Minv(r)
        rz_new = float(np.sum(r * z))
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it, it, rel


# ---------------------------------------------------------------------------
# Optimal-transport initialisation
# ---------------------------------------------------------------------------


def ot_shift(Ip, Im, eps=1e-3):
    """Positivity shift (R6): one global shift common to both images,
    min -> eps * (max - min).  Returns None when both images are constant."""
    m0 = min(float(np.min(Ip)), float(np.min(Im)))
    M0 = max(float(np.max(Ip)), float(np.max(Im)))
    if M0 == m0:
        return None
    return -m0 + eps * (M0 - m0)


def cdf(col):
    """C(x) = sum_{j<x} w(j), x = 0..m, of the unit-mass measure w (R7); C(m) = 1 exactly."""
    w = col / np.sum(col)
    C = np.concatenate([[0.0], np.cumsum(w)])
    C[-1] = 1.0
    return C


def quantile(C, r):
    """Pseudo-inverse C^{-1}(r) = min{x : C(x) >= r} made piecewise linear (R8).

    Q(r) = 0 for r <= 0; otherwise x* = min{x in 1..m : C(x) >= r} and
    Q(r) = x* - 1 + (r - C(x*-1)) / (C(x*) - C(x*-1)).
    """
    r = np.asarray(r, np.float64)
    m = len(C) - 1
    out = np.zeros(r.shape)
    for idx in np.ndindex(r.shape):
        rv = r[idx]
        if rv <= 0.0:
            out[idx] = 0.0
            continue
        xs = m
        for x in range(1, m + 1):           # the min-definition, literally
            if C[x] >= rv:
                xs = x
                break
        out[idx] = xs - 1 + (rv - C[xs - 1]) / (C[xs] - C[xs - 1])
    return out


def quantile_vec(C, r):
    """Vectorised quantile(): identical definition via searchsorted (left = min{x: C(x) >= r})."""
    r = np.asarray(r, np.float64)
    m = len(C) - 1
    xs = np.searchsorted(C[1:], r, side="left") + 1
    xs = np.clip(xs, 1, m)
    with np.errstate(divide="ignore", invalid="ignore"):   # 0/0 only where r <= 0 (masked)
        q = xs - 1 + (r - C[xs - 1]) / (C[xs] - C[xs - 1])
    return np.where(r <= 0.0, 0.0, q)


def ot_column(ip, im, h3, vec=True):
    """b0 on the nodes of one column (R9).

    T+ = Q_half o C+, T- = Q_half o C-, Q_half = (Q+ + Q-)/2, and the field map
    is the average of the displacements of T+ and -T-: b0 = h3 (T- - T+)/2.
    """
    Cp, Cm = cdf(ip), cdf(im)
    Q = quantile_vec if vec else quantile

    def Qh(r):
        return 0.5 * (Q(Cp, r) + Q(Cm, r))

    Tp = Qh(Cp)
    Tm = Qh(Cm)
    return h3 * (Tm - Tp) / 2.0


def gaussian_weights_1d(sigma=1.0):
    """Normalised 3-tap Gaussian (3x3x3 kernel, standard deviation 1.0)."""
    w = np.exp(-np.array([-1.0, 0.0, 1.0]) ** 2 / (2.0 * sigma ** 2))
    return w / w.sum()


def blur3(b, sigma=1.0):
    """3x3x3 Gaussian blur applied with an FFT (periodic) convolution, as the
    paper's FFT3D operator does (R11)."""
    w = gaussian_weights_1d(sigma)
    K3 = w[:, None, None] * w[None, :, None] * w[None, None, :]
    Kp = np.zeros(b.shape)
    for a in range(3):
        for c in range(3):
            for e in range(3):
                Kp[(a - 1) % b.shape[0], (c - 1) % b.shape[1], (e - 1) % b.shape[2]] += K3[a, c, e]
    return np.real(np.fft.ifftn(np.fft.fftn(b) * np.fft.fftn(Kp)))


def ot_init(Ip, Im, h3, eps=1e-3, blur=True, feas_cap=0.95, vec=True):
    """Parallelised OT initialisation, steps (c2).1-6 of DESIGN.md.

    Returns (b0, info) with info = {"max_Db_raw": ..., "scaled": bool}.
    """
    Ip = np.asarray(Ip, np.float64)
    Im = np.asarray(Im, np.float64)
    n1, n2, n3 = Ip.shape
    b0 = np.zeros((n1, n2, n3 + 1))
    info = {"max_Db_raw": 0.0, "scaled": False}
    shift = ot_shift(Ip, Im, eps)
    if shift is None:
        return b0, info
    ip, im = Ip + shift, Im + shift
    for i in range(n1):
        for j in range(n2):
            b0[i, j] = ot_column(ip[i, j], im[i, j], h3, vec=vec)
    if blur:
        b0 = blur3(b0)
    mx = float(np.max(np.abs(diff_pe(b0, h3)))) if n3 > 0 else 0.0
    info["max_Db_raw"] = mx
    if mx >= feas_cap:                           # R10 feasibility guard
        b0 = b0 * (feas_cap / mx)
        info["scaled"] = True
    return b0, info


# ---------------------------------------------------------------------------
# Gauss-Newton with Armijo line search (R14-R16)
# ---------------------------------------------------------------------------

STOP_MAXITER, STOP_GRAD, STOP_DJ, STOP_DB, STOP_LSFAIL, STOP_INFEASIBLE = 0, 1, 2, 3, 4, 5


def gn_armijo(objective, hess_of, precond_of, b0, h3, max_gn=10, max_pcg=10, pcg_tol=0.1,
              fixed=True, c1=1e-4, ls_max=10, tol_grad_rel=1e-2, tol_dJ_rel=1e-4,
              tol_db_rel=1e-3, log=None, armijo=True):
    """The Gauss-Newton iteration with Armijo line search of P:183-199, written
    for any objective (so its control flow is pinned on objectives with closed
    forms, tests/test_oracle_gn_control.py).

    objective(b) -> state with .J, .grad (None if infeasible), .infeasible
    (and optionally .D, .S, .P); hess_of(state) -> v -> H v (the GN Hessian,
    P:186); precond_of(state) -> the PCG preconditioner (diagonal or callable).

    Per GN step (Eq.(7)): q from PCG on H q = -grad (x0 = 0, R14),
    then Armijo (R15): gamma = 1, 1/2, ... (at most ls_max trials)
    until b + gamma q is feasible and J(b + gamma q) <= J(b) + c1 gamma grad.q;
    no acceptable trial -> stop with LS_FAIL (b unchanged).  Stop rules (P:284,
    "norm of the gradient, change in loss function or field map", tolerances
    R16), tested in this order after each accepted step unless `fixed`:
    ||grad|| <= tol_grad_rel ||grad(b0)||, |J_old - J| <= tol_dJ_rel |J_old|,
    max|gamma q| <= tol_db_rel h3.  armijo=False accepts the first feasible
    trial (the parity mode of R15).  An infeasible b0 stops before any step.
    """
    b = np.asarray(b0, np.float64).copy()
    st = objective(b)
    rep = {"gn_iters": 0, "f_evals": 1, "h_evals": 0, "pcg_iters": 0, "ls_halvings": 0,
           "stop_reason": STOP_MAXITER, "history": []}

    def parts(s):
        return {k: getattr(s, k, np.nan) for k in ("J", "D", "S", "P")}

    if st.infeasible:
        rep["stop_reason"] = STOP_INFEASIBLE
        rep.update(grad_norm=np.nan, **parts(st))
        return b, st, rep
    g0 = float(np.linalg.norm(st.grad))
    for it in range(max_gn):
        q, npcg, nmv, rel = pcg(hess_of(st), -st.grad, precond_of(st), max_pcg, pcg_tol, fixed)
        rep["h_evals"] += nmv
        rep["pcg_iters"] += npcg
        gq = float(np.sum(st.grad * q))
        gamma = 1.0
        accepted = False
        for t in range(ls_max):                     # Armijo (R15)
            bt = b + gamma * q
            stt = objective(bt)
            rep["f_evals"] += 1
            if (not stt.infeasible) and (not armijo or stt.J <= st.J + c1 * gamma * gq):
                accepted = True
                break
            if t + 1 < ls_max:
                rep["ls_halvings"] += 1
            gamma *= 0.5
        if not accepted:
            rep["stop_reason"] = STOP_LSFAIL
            break
        J_old = st.J
        b, st = bt, stt
        rep["gn_iters"] += 1
        rep["history"].append(dict(parts(st), gamma=gamma, pcg_iters=npcg, relres=rel))
        if log is not None:
            log(rep["history"][-1])
        if not fixed:
            if float(np.linalg.norm(st.grad)) <= tol_grad_rel * g0:
                rep["stop_reason"] = STOP_GRAD
                break
            if abs(J_old - st.J) <= tol_dJ_rel * abs(J_old):
                rep["stop_reason"] = STOP_DJ
                break
            if float(np.max(np.abs(gamma * q))) <= tol_db_rel * h3:
                rep["stop_reason"] = STOP_DB
                break
    rep.update(grad_norm=float(np.linalg.norm(st.grad)), **parts(st))
    return b, st, rep


def gauss_newton(Ip, Im, b0, h, alpha=ALPHA_DEFAULT, beta=BETA_DEFAULT, max_gn=10,
                 max_pcg=10, pcg_tol=0.1, fixed=True, c1=1e-4, ls_max=10,
                 tol_grad_rel=1e-2, tol_dJ_rel=1e-4, tol_db_rel=1e-3, log=None, armijo=True,
                 precond="jacobi"):
    """b_{k+1} = b_k + gamma_k q_k with H_J q_k = -grad J (Eq.(7)) on
    the field-map objective J = D + alpha S + beta P (evaluate()), GN
    Hessian hessvec() and its preconditioner (make_precond()).

    fixed=True: exactly max_gn GN steps of exactly max_pcg PCG iterations
    (parity / timing mode, R14, R16); fixed=False: the paper's stopping rules
    with DESIGN.md's tolerances (R16).  armijo=False accepts the full step
    unless infeasible (halving only for feasibility): the parity mode of R15.
    precond: "jacobi" (the paper's default) or "block" (R20).
    """
    return gn_armijo(lambda b: evaluate(Ip, Im, b, h, alpha, beta),
                     lambda st: (lambda v: hessvec(st, v)),
                     lambda st: make_precond(st, precond),
                     b0, h[2], max_gn=max_gn, max_pcg=max_pcg, pcg_tol=pcg_tol, fixed=fixed, c1=c1,
                     ls_max=ls_max, tol_grad_rel=tol_grad_rel, tol_dJ_rel=tol_dJ_rel,
                     tol_db_rel=tol_db_rel, log=log, armijo=armijo)


def correct_pair(Ip, Im, h, alpha=ALPHA_DEFAULT, beta=BETA_DEFAULT, max_gn=10, max_pcg=10,
                 fixed=True, blur=True, eps=1e-3, armijo=True, precond="jacobi"):
    """The whole path: OT init (+blur, guard) -> GN-PCG -> Jacobian-modulation apply."""
    b0, _ = ot_init(Ip, Im, h[2], eps=eps, blur=blur)
    b, st, rep = gauss_newton(Ip, Im, b0, h, alpha, beta, max_gn=max_gn, max_pcg=max_pcg,
                              fixed=fixed, armijo=armijo, precond=precond)
    Tp, Tm = apply_correction(Ip, Im, b, h[2])
    return b0, b, Tp, Tm, rep


def relative_improvement(Ip, Im, Tp, Tm):
    """100 (1 - SSD(T+ - T-)/SSD(I+ - I-))."""
    Ip = np.asarray(Ip, np.float64)
    Im = np.asarray(Im, np.float64)
    return 100.0 * (1.0 - float(np.sum((Tp - Tm) ** 2)) / float(np.sum((Ip - Im) ** 2)))


# ---------------------------------------------------------------------------
# ADMM.  Readings R21-R26 in DESIGN.md.
#   F(b) = D(b) + alpha S3(b) + beta P(b)        (column-separable)
#   G(z) = alpha (S1(z) + S2(z))                 (in-plane smoothness)
#   b <- argmin_b F(b) + rho hd/2 ||b - z + u||^2   (Eq. x_update)
#   z <- argmin_z G(z) + rho hd/2 ||b - z + u||^2   (Eq. z_update)
#   u <- u + b - z                                  (Eq. u_update)
# rho adapted as in Boyd et al. 2011 §3.4.1; stop when b, z and u all
# change by less than a tolerance.
# ---------------------------------------------------------------------------


class ColState:
    """Per-PE-column objective of the ADMM b-update and its derivatives."""


def admm_b_objective(Ip, Im, b, v, h, alpha=ALPHA_DEFAULT, beta=BETA_DEFAULT, rho=1.0, derivs=True):
    """Fc(b) = D + alpha S3 + beta P + rho hd/2 ||b - v||^2 per PE column (R21):
    D, P as in `evaluate` (Eq.(2), Eq.(3)), S3 = hd/2 sum ||D3 b||^2 / h3^2 (the PE
    part of Eq.(5)).  Returns ColState with F (per column, +inf if infeasible),
    and with derivs: grad (nodes) and the column-tridiagonal GN Hessian
    d (diagonal), e (H[l, l+1]) -- data (Gauss-Newton) + alpha hd D3^T D3 / h3^2
    + beta hd/2 D^T phi'' D + rho hd I."""
    Ip = np.asarray(Ip, np.float64)
    Im = np.asarray(Im, np.float64)
    b = np.asarray(b, np.float64)
    h1, h2, h3 = (float(x) for x in h)
    hd = h1 * h2 * h3
    n3 = Ip.shape[-1]
    k = np.arange(n3, dtype=np.float64)
    cs = ColState()
    Ab = avg_pe(b)
    Db = diff_pe(b, h3)
    infeas = np.any(np.abs(Db) >= 1.0, axis=-1)
    vp, sp = interp_pe(Ip, k + Ab / h3)
    vm, sm = interp_pe(Im, k - Ab / h3)
    r = vp * (1.0 + Db) - vm * (1.0 - Db)
    with np.errstate(divide="ignore", invalid="ignore"):
        ph = np.where(np.abs(Db) < 1.0, phi(np.where(np.abs(Db) < 1.0, Db, 0.0)), np.inf)
    Dc = 0.5 * hd * np.sum(r * r, axis=-1)
    S3c = 0.5 * hd * np.sum(((b[..., 1:] - b[..., :-1]) / h3) ** 2, axis=-1)
    Pc = 0.5 * hd * np.sum(np.where(np.abs(Db) < 1.0, ph, 0.0), axis=-1)
    Xc = 0.5 * hd * np.sum((b - v) ** 2, axis=-1)
    cs.F = np.where(infeas, np.inf, Dc + alpha * S3c + beta * Pc + rho * Xc)
    cs.infeasible = infeas
    if not derivs:
        return cs
    Dbs = np.where(np.abs(Db) < 1.0, Db, 0.0)
    g = (sp / h3) * (1.0 + Db) + (sm / h3) * (1.0 - Db)
    s = vp + vm
    LPE = diff_pe_T(diff_pe(b, h3), h3)            # D3^T D3 b / h3^2
    cs.grad = (hd * (avg_pe_T(g * r) + diff_pe_T(s * r, h3)) + alpha * hd * LPE
               + beta * 0.5 * hd * diff_pe_T(dphi(Dbs), h3) + rho * hd * (b - v))
    a = g / 2.0 - s / h3
    c = g / 2.0 + s / h3
    p2 = d2phi(Dbs)
    d = np.zeros(b.shape)
    d[..., :-1] += hd * a ** 2 + beta * 0.5 * hd * p2 / h3 ** 2 + alpha * hd / h3 ** 2
    d[..., 1:] += hd * c ** 2 + beta * 0.5 * hd * p2 / h3 ** 2 + alpha * hd / h3 ** 2
    cs.d = d + rho * hd
    cs.e = hd * a * c - beta * 0.5 * hd * p2 / h3 ** 2 - alpha * hd / h3 ** 2
    return cs


ADMM_COL_TOL = 1e-6   # R23: a column stops when the GN step predicts < 1e-6 |Fc| decrease


def admm_b_update(Ip, Im, b, v, h, alpha=ALPHA_DEFAULT, beta=BETA_DEFAULT, rho=1.0, inner=2,
                  c1=1e-4, ls_max=10, col_tol=ADMM_COL_TOL):
    """b-update: `inner` Gauss-Newton steps on every PE column
    independently.  The column system H_col q = -grad_col is tridiagonal, so the
    per-column ("BlockPCG") solve is exact (Thomas, R23); each column takes its
    own Armijo step gamma in {1, 1/2, ...} on its own Fc ("different step
    sizes and stopping criteria for each image column"): a column stops when
    the step predicts a decrease -grad.q <= col_tol |Fc| (R23); a column
    without an acceptable step keeps b."""
    b = np.asarray(b, np.float64).copy()
    for _ in range(inner):
        cs = admm_b_objective(Ip, Im, b, v, h, alpha, beta, rho)
        if np.all(cs.infeasible):
            break
        q = -solve_tridiag_pe(cs.d, cs.e, np.where(cs.infeasible[..., None], 0.0, cs.grad))
        gq = np.sum(cs.grad * q, axis=-1)
        gamma = np.ones(b.shape[:-1])
        with np.errstate(invalid="ignore"):
            done = cs.infeasible | (-gq <= col_tol * np.abs(np.where(cs.infeasible, 0.0, cs.F)))
        bn = b.copy()
        for _t in range(ls_max):
            cand = b + gamma[..., None] * q
            ct = admm_b_objective(Ip, Im, cand, v, h, alpha, beta, rho, derivs=False)
            ok = (~done) & (~ct.infeasible) & (ct.F <= cs.F + c1 * gamma * gq)
            bn[ok] = cand[ok]
            done |= ok
            gamma = np.where(done, gamma, 0.5 * gamma)
        b = bn
    return b


def periodic_laplacian_xy(z, h):
    """alpha-free in-plane operator of G: sum_{d=1,2} D_d^T D_d z / h_d^2 with
    periodic differences (the BCCB structure P:236-237 assumes), by rolls."""
    out = np.zeros(z.shape)
    for ax in (0, 1):
        dz = np.roll(z, -1, axis=ax) - z                 # forward difference, periodic
        out += (np.roll(dz, 1, axis=ax) - dz) / h[ax] ** 2
    return out


def admm_z_update(b, u, h, alpha=ALPHA_DEFAULT, rho=1.0):
    """z-update: (alpha hd L_xy^per + rho hd I) z = rho hd (b + u)
    on every PE node slice, solved by the 2-D FFT that diagonalises the periodic
    (BCCB) operator: eigenvalues 4 sin^2(pi k / n) / h^2 per axis."""
    n1, n2 = b.shape[0], b.shape[1]
    lam = (4.0 * np.sin(np.pi * np.arange(n1) / n1) ** 2 / h[0] ** 2)[:, None] + \
          (4.0 * np.sin(np.pi * np.arange(n2) / n2) ** 2 / h[1] ** 2)[None, :]
    F = np.fft.fft2(rho * (b + u), axes=(0, 1))
    return np.real(np.fft.ifft2(F / (alpha * lam + rho)[..., None], axes=(0, 1)))


def admm_rho_update(rho, r_norm, s_norm, mu=10.0, tau=2.0):
    """Residual balancing (Boyd et al. 2011 §3.4.1): returns (rho', factor)
    where the scaled multiplier u must be multiplied by `factor` = rho/rho'."""
    if r_norm > mu * s_norm:
        return rho * tau, 1.0 / tau
    if s_norm > mu * r_norm:
        return rho / tau, tau
    return rho, 1.0


def admm_rho0(h, alpha=ALPHA_DEFAULT):
    """Initial augmentation (unspecified in the paper, R24): alpha (1/h1^2 + 1/h2^2),
    the diagonal scale of the in-plane regulariser it splits off."""
    return alpha * (1.0 / h[0] ** 2 + 1.0 / h[1] ** 2)


def admm(Ip, Im, b0, h, alpha=ALPHA_DEFAULT, beta=BETA_DEFAULT, rho0=None, max_iter=20, inner=2,
         tol=1e-3, fixed=False, mu=10.0, tau=2.0):
    """ADMM field-map solve.  z0 = b0, u0 = 0, rho0 (R24).  Per
    iteration: b-update, z-update, u-update, residual balancing of rho (R25).
    Stop (not fixed): ||b - b_prev||, ||z - z_prev|| and ||u - u_prev|| all
    <= tol * max(||b||, tiny) (R26).  Returns (b, z, report)."""
    b = np.asarray(b0, np.float64).copy()
    z = b.copy()
    u = np.zeros_like(b)
    rho = admm_rho0(h, alpha) if rho0 is None else float(rho0)
    rep = {"iters": 0, "rho": [], "r_norm": [], "s_norm": [], "stop": "maxiter"}
    for _k in range(max_iter):
        b_prev, z_prev, u_prev = b, z, u
        b = admm_b_update(Ip, Im, b, z - u, h, alpha, beta, rho, inner)
        z = admm_z_update(b, u, h, alpha, rho)
        u = u + b - z
        r_norm = float(np.linalg.norm(b - z))
        s_norm = rho * float(np.linalg.norm(z - z_prev))
        rep["iters"] += 1
        rep["rho"].append(rho)
        rep["r_norm"].append(r_norm)
        rep["s_norm"].append(s_norm)
        db = float(np.linalg.norm(b - b_prev))
        dz = float(np.linalg.norm(z - z_prev))
        du = float(np.linalg.norm(u - u_prev))
        rho, f = admm_rho_update(rho, r_norm, s_norm, mu, tau)
        u = u * f
        if not fixed and max(db, dz, du) <= tol * max(float(np.linalg.norm(b)), 1e-300):
            rep["stop"] = "converged"
            break
    rep["rho_final"] = rho
    return b, z, rep


# ---------------------------------------------------------------------------
# Push-forward matrices, distortion simulation and least-squares correction
# (SURVEY §8(f) NEXT-3).  Readings R27-R29 in DESIGN.md.
#   True cell k (centre at index position k) is carried by the distortion to
#   u_k = k + sign (A b)_k / h3 (the map x -> x + sign b(x) v of Eq.(1),
#   P:72-76, in index units); its unit mass is split between the distorted
#   cells next to u_k with hat weights (R27):
#       A[j, k] = max(0, 1 - |u_k - j|),   j, k = 0..n3-1,
#   mass landing outside [0, n3) is dropped.  The distorted image is I = A t.
#   Least squares (R28, R29): t = argmin ||A+ t - i+||^2 + ||A- t - i-||^2
#   + lambda ||D1 t||^2 per PE column, D1 the forward difference in index
#   units, i.e. the normal equations
#       (A+^T A+ + A-^T A- + lambda L1) t = A+^T i+ + A-^T i-,
#   L1 = D1^T D1 (1-D Neumann Laplacian).
# ---------------------------------------------------------------------------

LSQ_LAMBDA_DEFAULT = 0.05   # R29


def push_forward_matrix(bcol, h3, sign):
    """Dense n3 x n3 push-forward matrix of one PE column (R27).
    bcol: nodes (n3+1,) in mm."""
    bcol = np.asarray(bcol, np.float64)
    n3 = bcol.shape[0] - 1
    u = np.arange(n3, dtype=np.float64) + sign * avg_pe(bcol) / h3
    j = np.arange(n3, dtype=np.float64)
    return np.maximum(0.0, 1.0 - np.abs(u[None, :] - j[:, None]))


def push_forward(T, b, h3, sign):
    """Distorted image I = A t per PE column of the true image T:
    T cells (..., n3), b nodes (..., n3+1)."""
    T = np.asarray(T, np.float64)
    b = np.asarray(b, np.float64)
    out = np.zeros_like(T)
    for idx in np.ndindex(T.shape[:-1]):
        out[idx] = push_forward_matrix(b[idx], h3, sign) @ T[idx]
    return out


def simulate_pair(T, b, h3):
    """The distorted pair (I+, I-) of a true image under field map b."""
    return push_forward(T, b, h3, +1.0), push_forward(T, b, h3, -1.0)


def neumann_laplacian_1d(n):
    """L1 = D1^T D1 for the (n-1) x n forward difference D1 (index units):
    tridiagonal [1 -1; -1 2 -1; ...; -1 1] (R28)."""
    L = np.zeros((n, n))
    for k in range(n):
        if k > 0:
            L[k, k] += 1.0
            L[k, k - 1] -= 1.0
        if k < n - 1:
            L[k, k] += 1.0
            L[k, k + 1] -= 1.0
    return L


def lsq_correct(Ip, Im, b, h3, lam=LSQ_LAMBDA_DEFAULT):
    """Least-squares correction (R28): per PE column the exact solution
    of the normal equations above (dense direct solve)."""
    Ip = np.asarray(Ip, np.float64)
    Im = np.asarray(Im, np.float64)
    b = np.asarray(b, np.float64)
    n3 = Ip.shape[-1]
    L1 = neumann_laplacian_1d(n3)
    out = np.zeros_like(Ip)
    for idx in np.ndindex(Ip.shape[:-1]):
        Ap = push_forward_matrix(b[idx], h3, +1.0)
        Am = push_forward_matrix(b[idx], h3, -1.0)
        N = Ap.T @ Ap + Am.T @ Am + lam * L1
        out[idx] = np.linalg.solve(N, Ap.T @ Ip[idx] + Am.T @ Im[idx])
    return out
