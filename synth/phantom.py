"""Seeded synthetic reversed-gradient-polarity EPI pairs (input generator only).

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NONE of the method's arithmetic (no interpolation model, no objective,
no OT, no solver): it samples an analytic continuum object and an analytic
field map and distorts the object with the exact continuum inverse of the
forward model, Eq. (1) of PAPER.md:

    T[I, b, v](x) = I(x + b(x) v) * (1 + d_v b)(x)

so that I_plus(y) = I_true(x) / (1 + d_3 b(x)) where y = x + b(x), and
I_minus(y) = I_true(x) / (1 - d_3 b(x)) where y = x - b(x).  The pair is then
exactly corrected by the continuum b_true.

Recipe: HCP-b0-like ellipsoidal
object of peak ~1000 with smooth texture, a field map made of three signed
Gaussian bumps scaled so that max |d_3 b| = 0.4 (a few voxels of
displacement), PE = last axis, fp64 generation rounded once to fp32.

Workload shapes follow BASELINE.json `configs` and PAPER.md Table 1.
"""
from __future__ import annotations

import dataclasses
import numpy as np

# name -> (shape with PE last, voxel size in mm, seed)
CONFIGS = {
    # BASELINE.json configs[0]: 16x16x8, "PE along dim 2" (0-based: the size-8 last axis)
    "C1_16x16x8": ((16, 16, 8), (1.25, 1.25, 1.25), 0),
    # configs[1]: HCP 3T 168x144x111 @1.25 mm, PE on the 144 axis -> kernels see (168,111,144)
    "C2_hcp3t": ((168, 111, 144), (1.25, 1.25, 1.25), 1),
    # configs[2]: HCP 7T 200x200x132 @1.05 mm -> (200,132,200)
    "C3_hcp7t": ((200, 132, 200), (1.05, 1.05, 1.05), 2),
    # configs[4]: C2's FOV (210 x 138.75 x 180 mm) resampled at 512x512x384
    "C5_512": ((512, 512, 384), (210.0 / 512, 138.75 / 512, 180.0 / 384), 1),
}


@dataclasses.dataclass
class Pair:
    Ip: np.ndarray          # float32 (n1, n2, n3)   distorted along +PE
    Im: np.ndarray          # float32 (n1, n2, n3)   distorted along -PE
    b_true: np.ndarray      # float64 (n1, n2, n3+1) analytic field map (mm) at the staggered nodes
    I_true: np.ndarray      # float64 (n1, n2, n3)   undistorted object at the cell centres
    h: tuple                # (h1, h2, h3) mm
    seed: int


def _draw(rng, L):
    """Geometry draws, in a fixed order (DESIGN.md input recipe)."""
    Lmin = float(min(L))
    g = {}
    g["w"] = rng.uniform(-1.0, 1.0, 8)
    g["mu"] = rng.uniform(0.25, 0.75, (8, 3)) * L
    g["s"] = rng.uniform(0.05, 0.15, 8) * Lmin
    g["a"] = rng.uniform(0.5, 1.0, 3)
    g["sign"] = np.where(rng.uniform(0.0, 1.0, 3) < 0.5, -1.0, 1.0)
    g["nu"] = rng.uniform(0.3, 0.7, (3, 3)) * L
    g["tau"] = rng.uniform(0.08, 0.2, 3) * Lmin
    return g


def _image(x1, x2, x3, L, g):
    """Continuum object at points (broadcastable coordinate arrays, mm)."""
    c = L / 2.0
    rho = np.sqrt(((x1 - c[0]) / (0.4 * L[0])) ** 2 + ((x2 - c[1]) / (0.4 * L[1])) ** 2
                  + ((x3 - c[2]) / (0.4 * L[2])) ** 2)
    mask = 1.0 / (1.0 + np.exp(-(1.0 - rho) / 0.05))
    tex = 0.0
    for m in range(8):
        d2 = (x1 - g["mu"][m, 0]) ** 2 + (x2 - g["mu"][m, 1]) ** 2 + (x3 - g["mu"][m, 2]) ** 2
        tex = tex + g["w"][m] * np.exp(-d2 / (2.0 * g["s"][m] ** 2))
    return 1000.0 * mask * (1.0 + 0.3 * np.tanh(tex))


class _Field:
    """b(x) = kappa * sum_m sign_m a_m exp(-|x-nu_m|^2/(2 tau_m^2)), separable per bump."""

    def __init__(self, g, kappa=1.0):
        self.g = g
        self.kappa = kappa

    def inplane(self, x1, x2):
        g = self.g
        return [g["sign"][m] * g["a"][m]
                * np.exp(-((x1 - g["nu"][m, 0]) ** 2 + (x2 - g["nu"][m, 1]) ** 2) / (2 * g["tau"][m] ** 2))
                for m in range(3)]

    def eval(self, amp, x3):
        """b and d b/d x3 given the in-plane amplitudes `amp` (list of arrays)."""
        g = self.g
        b = 0.0
        db = 0.0
        for m in range(3):
            e = np.exp(-(x3 - g["nu"][m, 2]) ** 2 / (2 * g["tau"][m] ** 2))
            b = b + amp[m] * e
            db = db + amp[m] * e * (-(x3 - g["nu"][m, 2]) / g["tau"][m] ** 2)
        return self.kappa * b, self.kappa * db


def make_pair(shape, h, seed, max_dv=0.4, noise=0.0, chunk=32, planes=None) -> Pair:
    """Generate one seeded pair.  shape = (n1, n2, n3) with PE last; h in mm.
    planes = (i0, i1): only those planes of dim 1 (a slab of the same volume;
    equal to the corresponding planes of the full generation up to the Newton
    stopping tolerance, 1e-12 mm)."""
    n1, n2, n3 = (int(v) for v in shape)
    h = tuple(float(v) for v in h)
    L = np.array([n1 * h[0], n2 * h[1], n3 * h[2]])
    rng = np.random.default_rng(seed)
    g = _draw(rng, L)
    fld = _Field(g)

    # kappa: max |d3 b| = max_dv on a 4x oversampled PE grid (analytic derivative)
    x1c = (np.arange(n1) + 0.5) * h[0]
    x2c = (np.arange(n2) + 0.5) * h[1]
    x3f = (np.arange(4 * n3) + 0.5) * (h[2] / 4)
    mx = 0.0
    for i0 in range(0, n1, chunk):
        X1, X2 = np.meshgrid(x1c[i0:i0 + chunk], x2c, indexing="ij")
        amp = [a[..., None] for a in fld.inplane(X1, X2)]
        _, db = fld.eval(amp, x3f[None, None, :])
        mx = max(mx, float(np.abs(db).max()))
    fld.kappa = max_dv / mx

    x3c = (np.arange(n3) + 0.5) * h[2]
    x3n = np.arange(n3 + 1) * h[2]
    p0, p1 = (0, n1) if planes is None else (int(planes[0]), int(planes[1]))
    m1 = p1 - p0
    Ip = np.empty((m1, n2, n3), np.float64)
    Im = np.empty((m1, n2, n3), np.float64)
    It = np.empty((m1, n2, n3), np.float64)
    bt = np.empty((m1, n2, n3 + 1), np.float64)
    for a0 in range(0, m1, chunk):
        i0 = p0 + a0
        X1, X2 = np.meshgrid(x1c[i0:min(i0 + chunk, p1)], x2c, indexing="ij")
        X1e, X2e = X1[..., None], X2[..., None]
        amp = [a[..., None] for a in fld.inplane(X1, X2)]
        It[a0:a0 + chunk] = _image(X1e, X2e, x3c[None, None, :], L, g)
        bt[a0:a0 + chunk] = fld.eval(amp, x3n[None, None, :])[0]
        y = np.broadcast_to(x3c[None, None, :], X1.shape + (n3,))
        for sgn, out in ((1.0, Ip), (-1.0, Im)):
            # Newton on x + sgn*b(x) = y (monotone since |d3 b| <= 0.4 < 1)
            x = y.copy()
            for _ in range(30):
                b, db = fld.eval(amp, x)
                res = x + sgn * b - y
                x = x - res / (1.0 + sgn * db)
                if float(np.abs(res).max()) < 1e-12:
                    break
            b, db = fld.eval(amp, x)
            out[a0:a0 + chunk] = _image(X1e, X2e, x, L, g) / (1.0 + sgn * db)
    if noise > 0.0:
        assert planes is None, "noise is drawn for the whole volume"
        nrng = np.random.default_rng(seed + 7919)
        Ip += nrng.normal(0.0, noise * 1000.0, Ip.shape)
        Im += nrng.normal(0.0, noise * 1000.0, Im.shape)
    return Pair(Ip.astype(np.float32), Im.astype(np.float32), bt, It, h, seed)


def make_config(name, **kw) -> Pair:
    shape, h, seed = CONFIGS[name]
    return make_pair(shape, h, seed, **kw)


def random_feasible_b(shape, h3, seed, amp=0.3):
    """A random smooth field map on the staggered node grid with max|Db| < amp (mm).

    Used for parity at non-stationary points.  Smoothness comes
    from summing a few random separable cosines; no method arithmetic.
    """
    n1, n2, n3 = shape
    rng = np.random.default_rng(seed)
    i = np.arange(n1)[:, None, None]
    j = np.arange(n2)[None, :, None]
    l = np.arange(n3 + 1)[None, None, :]
    b = np.zeros((n1, n2, n3 + 1))
    for _ in range(4):
        f = rng.uniform(0.2, 1.2, 3)
        ph = rng.uniform(0, 2 * np.pi, 3)
        b += rng.uniform(-1, 1) * np.cos(f[0] * i / max(n1, 2) * 3 + ph[0]) \
            * np.cos(f[1] * j / max(n2, 2) * 3 + ph[1]) * np.cos(f[2] * l / max(n3, 2) * 3 + ph[2])
    b += 0.05 * rng.standard_normal(b.shape)
    dv = np.abs(np.diff(b, axis=2)).max()
    return (b * (amp * h3 / dv)).astype(np.float32) if dv > 0 else b.astype(np.float32)
