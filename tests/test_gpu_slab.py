"""Slab decomposition along dim 1 on one GPU.

A loopback group (hysco_create_loopback: nranks contexts, one stream, halo
planes exchanged by device copies, pair totals allreduced by a fixed-order
device sum) runs the same kernels, halo exchanges and deferred decisions as
an NCCL group.  Its result must equal the single-context solve up to
reduction order, and the oracle within the parity tolerances.
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


def rel(a, ref):
    a, ref = np.asarray(a, np.float64), np.asarray(ref, np.float64)
    return np.linalg.norm(a - ref) / max(np.linalg.norm(ref), 1e-300)


def single(Ip, Im, h, dtype, so, batch):
    n1, n2, n3 = Ip.shape[1:]
    ctx = H.hysco_create((n1, n2, n3), h, batch, dtype=dtype)
    tIp = torch.from_numpy(Ip.astype(ND[dtype])).to(DEV)
    tIm = torch.from_numpy(Im.astype(ND[dtype])).to(DEV)
    H.hysco_bind_images(ctx, tIp, tIm)
    b = torch.zeros((batch, n1, n2, n3 + 1), dtype=TD[dtype], device=DEV)
    Tp = torch.zeros((batch, n1, n2, n3), dtype=TD[dtype], device=DEV)
    Tm = torch.zeros_like(Tp)
    torch.cuda.synchronize()          # torch fills on its stream; the context runs on its own
    reps, _ = H.hysco_correct(ctx, b, Tp, Tm, solve_opts=so, batch=batch)
    H.hysco_destroy(ctx)
    return b.cpu().numpy(), Tp.cpu().numpy(), Tm.cpu().numpy(), reps


def grouped(Ip, Im, h, dtype, so, batch, nranks):
    n1, n2, n3 = Ip.shape[1:]
    ctxs = H.hysco_create_loopback((n1, n2, n3), h, nranks, batch=batch, dtype=dtype)
    keep, bs, tps, tms = [], [], [], []
    for r, c in enumerate(ctxs):
        i0, i1 = H.slab_bounds(n1, nranks, r)
        tIp = torch.from_numpy(np.ascontiguousarray(Ip[:, i0:i1]).astype(ND[dtype])).to(DEV)
        tIm = torch.from_numpy(np.ascontiguousarray(Im[:, i0:i1]).astype(ND[dtype])).to(DEV)
        keep += [tIp, tIm]
        H.hysco_bind_images(c, tIp, tIm)
        bs.append(torch.zeros((batch, i1 - i0, n2, n3 + 1), dtype=TD[dtype], device=DEV))
        tps.append(torch.zeros((batch, i1 - i0, n2, n3), dtype=TD[dtype], device=DEV))
        tms.append(torch.zeros((batch, i1 - i0, n2, n3), dtype=TD[dtype], device=DEV))
    torch.cuda.synchronize()
    reps, _ = H.hysco_group_correct(ctxs, bs, tps, tms, solve_opts=so, batch=batch)
    n_launch = [H.hysco_last_launch_count(c) for c in ctxs]
    for c in ctxs:
        H.hysco_destroy(c)
    cat = lambda ts: np.concatenate([t.cpu().numpy() for t in ts], axis=1)  # noqa: E731
    return cat(bs), cat(tps), cat(tms), reps, n_launch


@pytest.mark.parametrize("nranks", [1, 2, 4])
def test_loopback_slabs_equal_single_f64(nranks):
    p = phantom.make_config("C1_16x16x8")
    Ip, Im = p.Ip[None].astype(np.float64), p.Im[None].astype(np.float64)
    so = H.default_solve_opts()            # real Armijo: decisions must match exactly in fp64
    b1, tp1, tm1, r1 = single(Ip, Im, p.h, H.HYSCO_F64, so, 1)
    b2, tp2, tm2, r2, nl = grouped(Ip, Im, p.h, H.HYSCO_F64, so, 1, nranks)
    assert (r2[0]["gn_iters"], r2[0]["pcg_iters"], r2[0]["f_evals"], r2[0]["ls_halvings"]) == \
        (r1[0]["gn_iters"], r1[0]["pcg_iters"], r1[0]["f_evals"], r1[0]["ls_halvings"])
    assert rel(b2, b1) <= 1e-11 and rel(tp2, tp1) <= 1e-11 and rel(tm2, tm1) <= 1e-11
    assert abs(r2[0]["J"] - r1[0]["J"]) <= 1e-11 * abs(r1[0]["J"])
    assert all(n > 0 for n in nl)


def test_loopback_slabs_ragged_batch_f32_vs_oracle():
    pairs = [phantom.make_pair((7, 6, 37), (1.1, 0.9, 1.3), 40 + k) for k in range(2)]
    Ip = np.stack([q.Ip for q in pairs])
    Im = np.stack([q.Im for q in pairs])
    h = pairs[0].h
    so = H.default_solve_opts(armijo=0)
    b1, tp1, _, _ = single(Ip, Im, h, H.HYSCO_F32, so, 2)
    b2, tp2, _, reps, _ = grouped(Ip, Im, h, H.HYSCO_F32, so, 2, 3)      # planes split 2 / 2 / 3
    assert rel(b2, b1) <= 1e-5 and rel(tp2, tp1) <= 1e-5
    for k, q in enumerate(pairs):
        _, bref, tpr, _, rep = O.correct_pair(q.Ip.astype(np.float64), q.Im.astype(np.float64), h, armijo=False)
        assert rel(b2[k], bref) <= 1e-4 and rel(tp2[k], tpr) <= 1e-4
        assert reps[k]["gn_iters"] == rep["gn_iters"]


def test_loopback_slabs_long_columns_f64():
    """P = 301 > 8 x 32 (two register segments per column, like configs[4]'s
    P = 385) through the slab path: equals the single-context solve."""
    p = phantom.make_pair((4, 3, 300), (1.25, 1.25, 1.0), 19)
    Ip, Im = p.Ip[None].astype(np.float64), p.Im[None].astype(np.float64)
    so = H.default_solve_opts(max_gn=3)
    b1, tp1, _, r1 = single(Ip, Im, p.h, H.HYSCO_F64, so, 1)
    b2, tp2, _, r2, _ = grouped(Ip, Im, p.h, H.HYSCO_F64, so, 1, 2)
    assert (r2[0]["gn_iters"], r2[0]["pcg_iters"]) == (r1[0]["gn_iters"], r1[0]["pcg_iters"])
    assert rel(b2, b1) <= 1e-11 and rel(tp2, tp1) <= 1e-11
    _, bref, _, _, rep = O.correct_pair(p.Ip.astype(np.float64), p.Im.astype(np.float64), p.h, max_gn=3)
    assert rel(b1[0], bref) <= 1e-9


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_slabs_block_precond_f64(nranks):
    """The block preconditioner (R20) is column-local, so slabs run it with no
    extra exchange: equal to the single-context block solve, fixed and with the
    paper's stop rules."""
    p = phantom.make_pair((9, 7, 30), (1.2, 1.0, 1.1), 23)
    Ip, Im = p.Ip[None].astype(np.float64), p.Im[None].astype(np.float64)
    for so in (H.default_solve_opts(armijo=0, precond=H.HYSCO_PRECOND_PE_BLOCK),
               H.default_solve_opts(fixed_iters=0, max_gn=20, precond=H.HYSCO_PRECOND_PE_BLOCK)):
        b1, tp1, _, r1 = single(Ip, Im, p.h, H.HYSCO_F64, so, 1)
        b2, tp2, _, r2, _ = grouped(Ip, Im, p.h, H.HYSCO_F64, so, 1, nranks)
        assert (r2[0]["gn_iters"], r2[0]["pcg_iters"], r2[0]["stop_reason"]) == \
            (r1[0]["gn_iters"], r1[0]["pcg_iters"], r1[0]["stop_reason"])
        assert rel(b2, b1) <= 1e-11 and rel(tp2, tp1) <= 1e-11


def test_loopback_single_plane_slabs_periodic_blur():
    """Every rank owns one plane: the periodic blur ring and the Neumann ends
    are all exchange-driven."""
    p = phantom.make_pair((4, 5, 20), (1.0, 1.2, 1.1), 77)
    Ip, Im = p.Ip[None].astype(np.float64), p.Im[None].astype(np.float64)
    so = H.default_solve_opts(max_gn=3)
    b1, tp1, _, _ = single(Ip, Im, p.h, H.HYSCO_F64, so, 1)
    b2, tp2, _, _, _ = grouped(Ip, Im, p.h, H.HYSCO_F64, so, 1, 4)
    assert rel(b2, b1) <= 1e-11 and rel(tp2, tp1) <= 1e-11


def test_nccl_slab_one_rank_equals_single():
    p = phantom.make_config("C1_16x16x8")
    n1, n2, n3 = p.Ip.shape
    so = H.default_solve_opts(armijo=0)
    b1, tp1, _, r1 = single(p.Ip[None], p.Im[None], p.h, H.HYSCO_F32, so, 1)
    ctx = H.hysco_create_slab((n1, n2, n3), p.h, 0, 1, n1, 0)
    tIp = torch.from_numpy(p.Ip[None]).to(DEV)
    tIm = torch.from_numpy(p.Im[None]).to(DEV)
    H.hysco_bind_images(ctx, tIp, tIm)
    b = torch.zeros((1, n1, n2, n3 + 1), device=DEV)
    Tp = torch.zeros((1, n1, n2, n3), device=DEV)
    reps, _ = H.hysco_correct(ctx, b, Tp, None, solve_opts=so)
    assert rel(b.cpu().numpy(), b1) <= 1e-5 and rel(Tp.cpu().numpy(), tp1) <= 1e-5
    assert reps[0]["gn_iters"] == r1[0]["gn_iters"]
    # per-kernel calls are not available on slab contexts
    with pytest.raises(H.HyscoError) as e:
        H.hysco_apply(ctx, b, Tp, None)
    assert e.value.status == H.HYSCO_ERR_STATE
    H.hysco_destroy(ctx)


def test_loopback_hcp3t_four_slabs():
    p = phantom.make_config("C2_hcp3t")
    so = H.default_solve_opts(armijo=0, max_gn=3)
    b1, tp1, _, r1 = single(p.Ip[None], p.Im[None], p.h, H.HYSCO_F32, so, 1)
    b2, tp2, _, r2, _ = grouped(p.Ip[None], p.Im[None], p.h, H.HYSCO_F32, so, 1, 4)
    assert rel(b2, b1) <= 1e-5 and rel(tp2, tp1) <= 1e-5
    assert r2[0]["pcg_iters"] == r1[0]["pcg_iters"] == 30


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_slabs_push_forward_and_lsq_equal_single(nranks):
    """NEXT-3 on slab contexts: column-local, so the concatenated slabs equal
    the single-context result bit for bit (no exchange)."""
    shape = (7, 5, 30)
    h = (1.1, 1.2, 1.25)
    rng = np.random.default_rng(3)
    T = rng.uniform(0, 2, (1,) + shape).astype(np.float32)
    b = phantom.random_feasible_b(shape, h[2], seed=6, amp=0.6)[None].astype(np.float32)
    n1 = shape[0]
    c = H.hysco_create(shape, h, 1)
    tT, tb = torch.from_numpy(T).to(DEV), torch.from_numpy(b).to(DEV)
    Ip, Im, out = torch.zeros_like(tT), torch.zeros_like(tT), torch.zeros_like(tT)
    torch.cuda.synchronize()
    H.hysco_push_forward(c, tb, tT, Ip, Im)
    H.hysco_bind_images(c, Ip, Im)
    torch.cuda.synchronize()
    H.hysco_lsq_correct(c, tb, out)
    torch.cuda.synchronize()
    ref_p, ref_m, ref_t = Ip.cpu().numpy(), Im.cpu().numpy(), out.cpu().numpy()
    H.hysco_destroy(c)
    ctxs = H.hysco_create_loopback(shape, h, nranks)
    got_p, got_m, got_t, keep = [], [], [], []
    for r, cx in enumerate(ctxs):
        i0, i1 = H.slab_bounds(n1, nranks, r)
        sT = torch.from_numpy(np.ascontiguousarray(T[:, i0:i1])).to(DEV)
        sb = torch.from_numpy(np.ascontiguousarray(b[:, i0:i1])).to(DEV)
        sp, sm, so_ = torch.zeros_like(sT), torch.zeros_like(sT), torch.zeros_like(sT)
        torch.cuda.synchronize()
        H.hysco_push_forward(cx, sb, sT, sp, sm)
        H.hysco_bind_images(cx, sp, sm)
        torch.cuda.synchronize()
        H.hysco_lsq_correct(cx, sb, so_)
        torch.cuda.synchronize()
        keep += [sT, sb, sp, sm, so_]
        got_p.append(sp.cpu().numpy())
        got_m.append(sm.cpu().numpy())
        got_t.append(so_.cpu().numpy())
    for cx in ctxs:
        H.hysco_destroy(cx)
    assert np.array_equal(np.concatenate(got_p, axis=1), ref_p)
    assert np.array_equal(np.concatenate(got_m, axis=1), ref_m)
    assert np.array_equal(np.concatenate(got_t, axis=1), ref_t)


def admm_single(Ip, Im, b0, h, dtype, ao, batch):
    n1, n2, n3 = Ip.shape[1:]
    ctx = H.hysco_create((n1, n2, n3), h, batch, dtype=dtype)
    tIp = torch.from_numpy(Ip.astype(ND[dtype])).to(DEV)
    tIm = torch.from_numpy(Im.astype(ND[dtype])).to(DEV)
    H.hysco_bind_images(ctx, tIp, tIm)
    b = torch.from_numpy(np.ascontiguousarray(b0).astype(ND[dtype])).to(DEV)
    torch.cuda.synchronize()
    reps = H.hysco_admm(ctx, b, ao, batch=batch)
    torch.cuda.synchronize()
    H.hysco_destroy(ctx)
    return b.cpu().numpy(), reps


def admm_grouped(Ip, Im, b0, h, dtype, ao, batch, nranks):
    n1, n2, n3 = Ip.shape[1:]
    ctxs = H.hysco_create_loopback((n1, n2, n3), h, nranks, batch=batch, dtype=dtype)
    keep, bs = [], []
    for r, c in enumerate(ctxs):
        i0, i1 = H.slab_bounds(n1, nranks, r)
        tIp = torch.from_numpy(np.ascontiguousarray(Ip[:, i0:i1]).astype(ND[dtype])).to(DEV)
        tIm = torch.from_numpy(np.ascontiguousarray(Im[:, i0:i1]).astype(ND[dtype])).to(DEV)
        keep += [tIp, tIm]
        H.hysco_bind_images(c, tIp, tIm)
        bs.append(torch.from_numpy(np.ascontiguousarray(b0[:, i0:i1]).astype(ND[dtype])).to(DEV))
    torch.cuda.synchronize()
    reps = H.hysco_group_admm(ctxs, bs, ao, batch=batch)
    torch.cuda.synchronize()
    for c in ctxs:
        H.hysco_destroy(c)
    return np.concatenate([t.cpu().numpy() for t in bs], axis=1), reps


ADMM_SLAB = [(1, (8, 6, 20), 2), (2, (8, 6, 20), 2), (3, (7, 5, 24), 1), (4, (12, 10, 24), 1)]


@pytest.mark.parametrize("stop", ["fixed", "paper"])
@pytest.mark.parametrize("dtype", [H.HYSCO_F64, H.HYSCO_F32], ids=["f64", "f32"])
@pytest.mark.parametrize("nranks,shape,batch", ADMM_SLAB, ids=[f"r{c[0]}-{c[1]}" for c in ADMM_SLAB])
def test_loopback_admm_equals_single(nranks, shape, batch, dtype, stop):
    """ADMM on slabs (hysco_group_admm): the column-local b-update on every
    slab, the transposed z-update (every rank transforms all n1 planes of its
    range of PE nodes), allreduced residual norms -- equal to the
    single-context ADMM (same iterations, rho and stop decisions; b to fp64
    summation order / the fp32 gate) and, in fp64, to the oracle."""
    h = (1.25, 1.1, 1.2)
    pairs = [phantom.make_pair(shape, h, 60 + k) for k in range(batch)]
    Ip = np.stack([q.Ip for q in pairs]).astype(ND[dtype]).astype(np.float64)
    Im = np.stack([q.Im for q in pairs]).astype(ND[dtype]).astype(np.float64)
    b0 = np.stack([O.ot_init(Ip[k], Im[k], h[2])[0] for k in range(batch)]).astype(ND[dtype]).astype(np.float64)
    ao = H.default_admm_opts(max_iter=12, fixed_iters=1) if stop == "fixed" else H.default_admm_opts(max_iter=50)
    b1, r1 = admm_single(Ip, Im, b0, h, dtype, ao, batch)
    b2, r2 = admm_grouped(Ip, Im, b0, h, dtype, ao, batch, nranks)
    tol = 1e-11 if dtype == H.HYSCO_F64 else 1e-4
    for k in range(batch):
        assert (r2[k]["iters"], r2[k]["converged"]) == (r1[k]["iters"], r1[k]["converged"])
        assert abs(r2[k]["rho"] - r1[k]["rho"]) <= 1e-12 * r1[k]["rho"]
        assert rel(b2[k], b1[k]) <= tol
        assert abs(r2[k]["J"] - r1[k]["J"]) <= tol * abs(r1[k]["J"])
        if dtype == H.HYSCO_F64 and stop == "fixed":
            bref, _, rep = O.admm(Ip[k], Im[k], b0[k], h, max_iter=12, fixed=True)
            assert rel(b2[k], bref) <= 1e-12


def test_nccl_slab_one_rank_admm_equals_single():
    """hysco_admm on an NCCL slab context (one rank: the transposes are NCCL
    self send / receive) equals the single-context ADMM."""
    p = phantom.make_pair((8, 6, 20), (1.25, 1.1, 1.2), 61)
    Ip, Im = p.Ip[None].astype(np.float64), p.Im[None].astype(np.float64)
    b0 = O.ot_init(Ip[0], Im[0], p.h[2])[0][None]
    ao = H.default_admm_opts(max_iter=10, fixed_iters=1)
    b1, r1 = admm_single(Ip, Im, b0, p.h, H.HYSCO_F64, ao, 1)
    n1, n2, n3 = Ip.shape[1:]
    ctx = H.hysco_create_slab((n1, n2, n3), p.h, 0, 1, n1, 0, dtype=H.HYSCO_F64)
    tIp, tIm = torch.from_numpy(Ip).to(DEV), torch.from_numpy(Im).to(DEV)
    H.hysco_bind_images(ctx, tIp, tIm)
    b = torch.from_numpy(np.ascontiguousarray(b0)).to(DEV)
    torch.cuda.synchronize()
    r2 = H.hysco_admm(ctx, b, ao)
    torch.cuda.synchronize()
    H.hysco_destroy(ctx)
    assert r2[0]["iters"] == r1[0]["iters"] and rel(b.cpu().numpy(), b1) <= 1e-11
