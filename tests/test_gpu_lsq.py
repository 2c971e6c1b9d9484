"""GPU parity of the push-forward simulator and the least-squares correction
(NEXT-3, readings R27-R29) against the CPU fp64 oracle.

push_forward is a fixed gather per column: fp32 <= 1e-5, fp64 <= 1e-12
(relative L2).  lsq_correct solves the normal equations by Jacobi-PCG to a
relative residual rtol (1e-6 fp32, 1e-12 fp64), the oracle by a dense direct
solve: the gap is bounded by cond(N) * rtol, with cond(N) <= ~1e2 for these
maps and lambda = 0.05 (lambda = 0.005: ~1e3): fp32 <= 2e-4, fp64 <= 1e-9.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import hysco_oracle as O          # noqa: E402
from paper_2403_10706_b200 import hysco as H  # noqa: E402
from synth import phantom                      # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
TD = {H.HYSCO_F32: torch.float32, H.HYSCO_F64: torch.float64}
ND = {H.HYSCO_F32: np.float32, H.HYSCO_F64: np.float64}
TOL_PF = {H.HYSCO_F32: 1e-5, H.HYSCO_F64: 1e-12}
TOL_LSQ = {H.HYSCO_F32: 2e-4, H.HYSCO_F64: 1e-9}
DTYPES = pytest.mark.parametrize("dtype", [H.HYSCO_F32, H.HYSCO_F64], ids=["f32", "f64"])
# several warps' worth of columns, ragged n3 (not a multiple of 32), HCP-length
# columns (144), long columns (300), and the smallest n3 the library takes (2)
SHAPES = [(6, 5, 37), (4, 4, 8), (3, 5, 144), (2, 3, 300), (2, 4, 2)]
H3 = 1.25


def rel(a, ref):
    a, ref = np.asarray(a, np.float64), np.asarray(ref, np.float64)
    n = np.linalg.norm(ref)
    return np.linalg.norm(a - ref) / (n if n > 0 else 1.0)


def dev(a, dtype):
    t = torch.from_numpy(np.ascontiguousarray(a).astype(ND[dtype])).to(DEV)
    torch.cuda.synchronize()
    return t


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def rnd(a, dtype):
    return np.asarray(a).astype(ND[dtype]).astype(np.float64)


def _inputs(shape, seed, dtype, amp=0.8):
    rng = np.random.default_rng(seed)
    T = rnd(rng.uniform(0.0, 2.0, (1,) + shape), dtype)
    b = rnd(phantom.random_feasible_b(shape, H3, seed=seed + 1, amp=amp)[None], dtype)
    return T, b


def _ctx(shape, dtype, Ip=None, Im=None, batch=1):
    c = H.hysco_create(shape, (1.1, 0.9, H3), batch, dtype=dtype)
    if Ip is not None:
        H.hysco_bind_images(c, Ip, Im)
    return c


@DTYPES
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_push_forward_parity(shape, dtype):
    T, b = _inputs(shape, 11, dtype)
    c = _ctx(shape, dtype)
    Tt, bt = dev(T, dtype), dev(b, dtype)
    Ip = torch.zeros_like(Tt)
    Im = torch.zeros_like(Tt)
    torch.cuda.synchronize()
    assert not H.hysco_push_forward(c, bt, Tt, Ip, Im)
    rp, rm = O.simulate_pair(T, b, H3)
    assert rel(host(Ip), rp) <= TOL_PF[dtype]
    assert rel(host(Im), rm) <= TOL_PF[dtype]
    H.hysco_destroy(c)


@DTYPES
def test_push_forward_closed_forms(dtype):
    shape = (3, 4, 40)
    T, _ = _inputs(shape, 2, dtype)
    c = _ctx(shape, dtype)
    Tt = dev(T, dtype)
    Ip, Im = torch.zeros_like(Tt), torch.zeros_like(Tt)
    torch.cuda.synchronize()
    H.hysco_push_forward(c, dev(np.zeros((1, 3, 4, 41)), dtype), Tt, Ip, Im)
    assert np.array_equal(host(Ip), T) and np.array_equal(host(Im), T)       # b = 0: identity, exactly
    H.hysco_push_forward(c, dev(np.full((1, 3, 4, 41), 2 * H3), dtype), Tt, Ip, Im)
    sh = np.zeros_like(T)
    sh[..., 2:] = T[..., :-2]                                                 # two-voxel shift, mass dropped
    assert rel(host(Ip), sh) <= 1e-6
    H.hysco_destroy(c)


@DTYPES
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("lam", [0.05, 0.005])
def test_lsq_parity(shape, dtype, lam):
    rng = np.random.default_rng(5)
    Ipn = rnd(rng.uniform(0.0, 2.0, (1,) + shape), dtype)
    Imn = rnd(rng.uniform(0.0, 2.0, (1,) + shape), dtype)
    b = rnd(phantom.random_feasible_b(shape, H3, seed=8, amp=0.6)[None], dtype)
    Ip, Im = dev(Ipn, dtype), dev(Imn, dtype)
    c = _ctx(shape, dtype, Ip, Im)
    out = torch.zeros_like(Ip)
    torch.cuda.synchronize()
    reps, infeas = H.hysco_lsq_correct(c, dev(b, dtype), out, H.default_lsq_opts(lam=lam))
    assert not infeas
    assert reps[0]["unconverged"] == 0 and reps[0]["infeasible"] == 0, reps
    ref = O.lsq_correct(Ipn, Imn, b, H3, lam=lam)
    assert rel(host(out), ref) <= TOL_LSQ[dtype], reps
    H.hysco_destroy(c)


def test_lsq_zero_field_lambda0_is_mean():
    shape = (4, 3, 50)
    rng = np.random.default_rng(1)
    Ipn, Imn = rng.uniform(0, 2, (1,) + shape), rng.uniform(0, 2, (1,) + shape)
    Ip, Im = dev(Ipn, H.HYSCO_F64), dev(Imn, H.HYSCO_F64)
    c = _ctx(shape, H.HYSCO_F64, Ip, Im)
    out = torch.zeros_like(Ip)
    torch.cuda.synchronize()
    reps, _ = H.hysco_lsq_correct(c, dev(np.zeros((1, 4, 3, 51)), H.HYSCO_F64), out, H.default_lsq_opts(lam=0.0))
    assert np.allclose(host(out), 0.5 * (Ipn + Imn), atol=1e-13, rtol=0)
    assert reps[0]["max_iters"] <= 1                    # N = 2 I: one Jacobi-PCG step is exact
    H.hysco_destroy(c)


def test_simulate_then_lsq_recovers_truth_on_gpu():
    """GPU pipeline: push_forward(T) -> lsq_correct with the same b ~ T."""
    shape = (8, 6, 96)
    dtype = H.HYSCO_F64
    n = shape[2]
    xc = (np.arange(n) + 0.5) / n
    T = np.exp(-((xc - 0.5) / 0.2) ** 2)[None, None, None, :] * np.ones((1,) + shape)
    b = phantom.random_feasible_b(shape, H3, seed=3, amp=0.5).astype(np.float64)[None]
    c = _ctx(shape, dtype)
    Tt, bt = dev(T, dtype), dev(b, dtype)
    Ip, Im = torch.zeros_like(Tt), torch.zeros_like(Tt)
    torch.cuda.synchronize()
    H.hysco_push_forward(c, bt, Tt, Ip, Im)
    H.hysco_bind_images(c, Ip, Im)
    out = torch.zeros_like(Tt)
    torch.cuda.synchronize()
    reps, _ = H.hysco_lsq_correct(c, bt, out, H.default_lsq_opts(lam=1e-9, max_iter=2000))
    assert rel(host(out), T) < 1e-4, reps
    H.hysco_destroy(c)


@DTYPES
def test_lsq_and_push_forward_infeasible_column(dtype):
    shape = (3, 4, 20)
    T, b = _inputs(shape, 4, dtype, amp=0.5)
    b[0, 1, 2, 7] += 1.5 * H3                            # |Db| > 1 in column (1, 2)
    Tt, bt = dev(T, dtype), dev(b, dtype)
    c = _ctx(shape, dtype, Tt, Tt)
    Ip, Im, out = torch.zeros_like(Tt), torch.zeros_like(Tt), torch.zeros_like(Tt)
    torch.cuda.synchronize()
    assert H.hysco_push_forward(c, bt, Tt, Ip, Im)
    reps, infeas = H.hysco_lsq_correct(c, bt, out, None)
    assert infeas and reps[0]["infeasible"] == 1
    o = host(out)
    assert np.all(o[0, 1, 2] == 0.0)
    ok = np.ones(shape[:2], bool)
    ok[1, 2] = False
    ref = O.lsq_correct(T, T, b, H3)
    assert rel(o[0][ok], ref[0][ok]) <= TOL_LSQ[dtype]
    H.hysco_destroy(c)


def test_lsq_batch_pairs_independent():
    shape = (3, 4, 33)
    dtype = H.HYSCO_F32
    rng = np.random.default_rng(9)
    Ipn = rnd(rng.uniform(0, 2, (2,) + shape), dtype)
    Imn = rnd(rng.uniform(0, 2, (2,) + shape), dtype)
    b = rnd(np.stack([phantom.random_feasible_b(shape, H3, seed=s, amp=0.6) for s in (1, 2)]), dtype)
    Ip, Im = dev(Ipn, dtype), dev(Imn, dtype)
    c = _ctx(shape, dtype, Ip, Im, batch=2)
    out = torch.zeros_like(Ip)
    torch.cuda.synchronize()
    reps, _ = H.hysco_lsq_correct(c, dev(b, dtype), out, None, batch=2)
    assert len(reps) == 2
    o = host(out)
    for p in range(2):
        assert rel(o[p], O.lsq_correct(Ipn[p], Imn[p], b[p], H3)) <= TOL_LSQ[dtype]
    H.hysco_destroy(c)


def test_lsq_argument_and_state_errors():
    shape = (2, 2, 8)
    c = _ctx(shape, H.HYSCO_F32)
    x = torch.zeros((1,) + shape, device=DEV)
    bn = torch.zeros((1, 2, 2, 9), device=DEV)
    torch.cuda.synchronize()
    with pytest.raises(H.HyscoError) as e:
        H.hysco_lsq_correct(c, bn, x)                    # no images bound
    assert e.value.status == H.HYSCO_ERR_STATE
    H.hysco_bind_images(c, x, x)
    with pytest.raises(H.HyscoError) as e:
        H.hysco_lsq_correct(c, bn, x, H.default_lsq_opts(lam=-1.0))
    assert e.value.status == H.HYSCO_ERR_ARG
    with pytest.raises(H.HyscoError) as e:
        H.hysco_push_forward(c, None, x, x, x)
    assert e.value.status == H.HYSCO_ERR_ARG
    H.hysco_destroy(c)


# ------------------------------------------------ full size (BASELINE configs[1])

def test_hcp3t_lsq_and_push_forward_sampled_columns():
    """HCP 3T shape in the production launch configuration; the oracle checks
    64 sampled columns one by one (push forward of the synthetic pair's I+,
    least squares of the pair under a smooth feasible field map)."""
    pair = phantom.make_config("C2_hcp3t")
    shape = pair.Ip.shape
    dtype = H.HYSCO_F32
    Ipn, Imn = rnd(pair.Ip[None], dtype), rnd(pair.Im[None], dtype)
    b = rnd(phantom.random_feasible_b(shape, pair.h[2], seed=21, amp=0.6)[None], dtype)
    Ip, Im, bt = dev(Ipn, dtype), dev(Imn, dtype), dev(b, dtype)
    c = H.hysco_create(shape, pair.h, 1, dtype=dtype)
    H.hysco_bind_images(c, Ip, Im)
    Pp, Pm, out = torch.zeros_like(Ip), torch.zeros_like(Ip), torch.zeros_like(Ip)
    torch.cuda.synchronize()
    assert not H.hysco_push_forward(c, bt, Ip, Pp, Pm)
    assert H.hysco_last_launch_count(c) == 1
    reps, infeas = H.hysco_lsq_correct(c, bt, out, None)
    assert H.hysco_last_launch_count(c) == 1
    assert not infeas and reps[0]["unconverged"] == 0, reps
    rng = np.random.default_rng(0)
    cols = [(int(rng.integers(shape[0])), int(rng.integers(shape[1]))) for _ in range(64)]
    ii = np.array([a for a, _ in cols])
    jj = np.array([bb for _, bb in cols])
    bs = b[0, ii, jj][:, None]
    ref_p = O.push_forward(Ipn[0, ii, jj][:, None], bs, pair.h[2], +1.0)[:, 0]
    ref_m = O.push_forward(Ipn[0, ii, jj][:, None], bs, pair.h[2], -1.0)[:, 0]
    ref_t = O.lsq_correct(Ipn[0, ii, jj][:, None], Imn[0, ii, jj][:, None], bs, pair.h[2])[:, 0]
    assert rel(host(Pp)[0, ii, jj], ref_p) <= TOL_PF[dtype]
    assert rel(host(Pm)[0, ii, jj], ref_m) <= TOL_PF[dtype]
    assert rel(host(out)[0, ii, jj], ref_t) <= TOL_LSQ[dtype]
    H.hysco_destroy(c)
