"""Pins of the oracle's building blocks (CPU, -m "not gpu").

Each test checks the oracle against something other than itself: closed forms,
exact rationals, invariants, a second independent construction (dense stencil
assembly, unit-vector probing) or finite differences.
"""
import re
from fractions import Fraction

import numpy as np
import pytest

from oracle import hysco_oracle as O

RNG = np.random.default_rng(12345)


# ---------------------------------------------------------------- barrier phi (Eq.(3))

def test_phi_closed_forms():
    assert O.phi(0.0) == 0 and O.dphi(0.0) == 0 and O.d2phi(0.0) == 0
    assert abs(O.phi(0.5) - 1.0 / 12.0) < 1e-15                # 0.0625/0.75
    assert abs(O.dphi(0.5) - 7.0 / 9.0) < 1e-15                # 2(1/8)(7/4)/(9/16)
    assert abs(O.d2phi(0.5) - 170.0 / 27.0) < 1e-13            # 2(1/4)(85/16)/(27/64)
    assert np.isinf(O.phi(1.0)) and np.isinf(O.phi(-1.3))
    # phi is even, phi' odd, phi'' even
    z = np.linspace(0.0, 0.95, 20)
    assert np.allclose(O.phi(z), O.phi(-z), rtol=1e-15, atol=0)
    assert np.allclose(O.dphi(z), -O.dphi(-z), rtol=1e-15, atol=0)
    assert np.all(O.d2phi(z) >= 0)


@pytest.mark.parametrize("z", [-0.9, -0.5, 0.1, 0.5, 0.9])
def test_phi_derivatives_fd(z):
    e = 1e-6
    fd1 = (O.phi(z + e) - O.phi(z - e)) / (2 * e)
    fd2 = (O.dphi(z + e) - O.dphi(z - e)) / (2 * e)
    assert abs(fd1 - O.dphi(z)) <= 1e-8 * max(1.0, abs(O.dphi(z)))
    assert abs(fd2 - O.d2phi(z)) <= 1e-7 * max(1.0, abs(O.d2phi(z)))


# ---------------------------------------------------------------- interpolation (R5)

def test_interp_nodes_midpoints_worked_example():
    f = RNG.standard_normal((3, 4, 7))
    k = np.broadcast_to(np.arange(7.0), f.shape)
    v, _ = O.interp_pe(f, k)
    assert np.array_equal(v, f)
    v, _ = O.interp_pe(f[..., :6], np.broadcast_to(np.arange(6.0) + 0.5, f[..., :6].shape))
    assert np.allclose(v[..., :5], 0.5 * (f[..., :5] + f[..., 1:6]), atol=1e-15)
    # SPEC S:115 worked example: column [0, 6, 0] at centre 0 + 0.25 -> 1.5, slope 6 (per index)
    v, s = O.interp_pe(np.array([0.0, 6.0, 0.0]), np.array([0.25, 0.0, 0.0]))
    assert v[0] == 1.5 and s[0] == 6.0


def test_interp_affine_reproduced_and_zero_padding():
    c0, c1 = 2.5, -0.75
    f = c0 + c1 * np.arange(9.0)
    u = RNG.uniform(0, 8, 9)
    v, s = O.interp_pe(f, u)
    assert np.allclose(v, c0 + c1 * u, atol=1e-13)
    assert np.allclose(s[u < 8], c1, atol=1e-13)
    # hat model: zero one cell past the outer centres, linear ramp in between
    f = np.array([3.0, 1.0, 2.0])
    v, _ = O.interp_pe(f, np.array([-1.0, -0.5, 2.5]))
    assert np.allclose(v, [0.0, 1.5, 1.0])
    v, _ = O.interp_pe(f, np.array([-1.5, 3.0, 7.2]))
    assert np.array_equal(v, [0.0, 0.0, 0.0])


# ---------------------------------------------------------------- A, D, L

def test_avg_diff_identities_and_adjoints():
    h3 = 1.7
    c = np.full((2, 3, 6), 4.2)
    assert np.allclose(O.avg_pe(c), 4.2) and np.allclose(O.diff_pe(c, h3), 0.0)
    ramp = np.broadcast_to(np.arange(6.0) * h3, (2, 3, 6))
    assert np.allclose(O.diff_pe(ramp, h3), 1.0, atol=1e-14)
    b = RNG.standard_normal((2, 3, 6))
    y = RNG.standard_normal((2, 3, 5))
    assert abs(np.sum(O.diff_pe(b, h3) * y) - np.sum(b * O.diff_pe_T(y, h3))) < 1e-12
    assert abs(np.sum(O.avg_pe(b) * y) - np.sum(b * O.avg_pe_T(y))) < 1e-12


def _dense_laplacian_stencil(shape, h):
    """Independent construction: the 7-point Neumann stencil written neighbour by neighbour."""
    N = int(np.prod(shape))
    L = np.zeros((N, N))
    idx = np.arange(N).reshape(shape)
    for p in np.ndindex(shape):
        for ax in range(3):
            for dlt in (-1, 1):
                q = list(p)
                q[ax] += dlt
                if 0 <= q[ax] < shape[ax]:
                    L[idx[p], idx[p]] += 1.0 / h[ax] ** 2
                    L[idx[p], idx[tuple(q)]] -= 1.0 / h[ax] ** 2
    return L


@pytest.mark.parametrize("shape", [(3, 3, 4), (4, 2, 5), (1, 1, 6), (5, 5, 5)])
def test_laplacian_equals_dense_stencil(shape):
    h = (1.1, 0.9, 1.3)
    Ld = _dense_laplacian_stencil(shape, h)
    N = Ld.shape[0]
    Lo = np.stack([O.laplacian(np.eye(N)[k].reshape(shape), h).ravel() for k in range(N)], 1)
    assert np.allclose(Lo, Ld, atol=1e-12)
    assert np.allclose(Ld, Ld.T)
    assert np.linalg.eigvalsh(Ld).min() > -1e-10
    assert np.allclose(O.laplacian(np.full(shape, 3.3), h), 0.0, atol=1e-12)
    b = RNG.standard_normal(shape)
    assert abs(O.smoothness_quadform(b, h) - b.ravel() @ Ld @ b.ravel()) < 1e-10


# ---------------------------------------------------------------- mp_transform (Eq.(1))

def test_mp_transform_special_cases():
    h3 = 1.25
    I = RNG.uniform(0, 1, (3, 4, 10))
    assert np.allclose(O.mp_transform(I, np.zeros((3, 4, 11)), h3, +1), I, atol=0)
    # integer constant shift c voxels = pure shift of the samples
    c = 2
    Tp = O.mp_transform(I, np.full((3, 4, 11), c * h3), h3, +1)
    assert np.allclose(Tp[..., :-c], I[..., c:], atol=1e-14)
    assert np.allclose(Tp[..., -c:], 0.0)
    Tm = O.mp_transform(I, np.full((3, 4, 11), c * h3), h3, -1)
    assert np.allclose(Tm[..., c:], I[..., :-c], atol=1e-14)
    # linear b (slope s) on a constant image -> 1 +- s where the query stays inside
    s = 0.1
    b = np.broadcast_to(np.arange(11) * h3 * s, (3, 4, 11))
    Ic = np.full((3, 4, 10), 2.0)
    Tp = O.mp_transform(Ic, b, h3, +1)
    up = np.arange(10) + s * (np.arange(10) + 0.5)
    assert np.allclose(Tp[..., up <= 9], 2.0 * (1 + s), atol=1e-13)
    Tm = O.mp_transform(Ic, b, h3, -1)
    um = np.arange(10) - s * (np.arange(10) + 0.5)
    assert np.allclose(Tm[..., um >= 0], 2.0 * (1 - s), atol=1e-13)


@pytest.mark.parametrize("c", [0.3, 1.0, 2.75, -1.6])
def test_mp_transform_conserves_mass_constant_b(c):
    """Partition of unity of the hat basis: any constant b conserves column mass
    exactly when the support stays interior."""
    h3 = 0.8
    I = np.zeros((2, 3, 20))
    I[..., 5:15] = RNG.uniform(0.5, 1.5, (2, 3, 10))
    b = np.full((2, 3, 21), c * h3)
    for sgn in (+1, -1):
        T = O.mp_transform(I, b, h3, sgn)
        assert np.allclose(T.sum(-1), I.sum(-1), rtol=1e-12, atol=0)


def test_mp_transform_mass_refinement_rate():
    """Varying b: mass error is a discretisation error, O(h^2) under refinement."""
    errs = []
    for n in (256, 512, 1024):
        h3 = 16.0 / n
        xc = (np.arange(n) + 0.5) * h3
        xn = np.arange(n + 1) * h3
        I = np.exp(-((xc - 8) / 2.0) ** 2)[None, None, :]
        b = (0.8 * np.exp(-((xn - 7.5) / 3.0) ** 2))[None, None, :]
        T = O.mp_transform(I, b, h3, +1)
        errs.append(abs(T.sum() * h3 - I.sum() * h3))
    rate = np.log2(errs[0] / errs[1]), np.log2(errs[1] / errs[2])
    assert 1.7 < rate[0] < 2.3 and 1.7 < rate[1] < 2.3


# ---------------------------------------------------------------- golden worked example

def _frac(expr):
    toks = re.findall(r"[+-]?[^+-]+", expr.replace(" ", ""))
    return float(sum(Fraction(t) for t in toks))


def _golden():
    vals = {}
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", "micro_eval.txt")
    for line in open(p):
        line = line.strip()
        if line and not line.startswith("#"):
            k, v = line.split()
            vals[k] = _frac(v)
    return vals


def test_golden_micro_eval():
    g = _golden()
    Ip = np.array([[[4.0, 8.0]]])
    Im = np.array([[[2.0, 6.0]]])
    b = np.array([[[0.0, 0.25, 0.0]]])
    st = O.evaluate(Ip, Im, b, (1.0, 1.0, 1.0), 300.0, 1e-4)
    for key in ("D", "S", "P", "J"):
        assert abs(getattr(st, key) - g[key]) <= 1e-15 * abs(g[key]), key
    for l in range(3):
        assert abs(st.grad[0, 0, l] - g["grad%d" % l]) <= 1e-13 * abs(g["grad%d" % l])
    # tridiagonal data+barrier part by unit-vector probing of H_J minus alpha hd L
    H = np.stack([O.hessvec(st, np.eye(3)[k].reshape(1, 1, 3)).ravel() for k in range(3)], 1)
    Lm = np.stack([O.laplacian(np.eye(3)[k].reshape(1, 1, 3), (1, 1, 1)).ravel() for k in range(3)], 1)
    T = H - 300.0 * Lm
    for l in range(3):
        assert abs(T[l, l] - g["d%d" % l]) <= 1e-13 * abs(g["d%d" % l])
    for l in range(2):
        assert abs(T[l, l + 1] - g["e%d" % l]) <= 1e-13 * abs(g["e%d" % l])
        assert abs(T[l + 1, l] - g["e%d" % l]) <= 1e-13 * abs(g["e%d" % l])
    assert T[0, 2] == 0 and T[2, 0] == 0
