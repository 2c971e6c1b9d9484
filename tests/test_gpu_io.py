"""GPU side of the front-end (NEXT-4, R30-R31): the PE-last permutation kernel
(bit-exact against numpy transposes), the cell-centred field map (against the
oracle's averaging operator A), and the command line run end to end
(NIfTI in -> permute -> OT + GN + corrections -> permute back -> NIfTI out),
which must reproduce the direct C-ABI run on numpy-permuted arrays bit for
bit, with corrected images matching the oracle's Eq.(1) transform."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import hysco_oracle as O          # noqa: E402
from paper_2403_10706_b200 import hysco as H  # noqa: E402
from synth import phantom                      # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TO_KERNEL = {1: (0, 1, 2), 2: (0, 2, 1), 3: (1, 2, 0)}   # file [nz][ny][nx] -> kernel layout (R30)


def _dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    torch.cuda.synchronize()
    return t


@pytest.mark.parametrize("dims", [(37, 5, 70), (33, 65, 17), (1, 40, 3)], ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("pe", [1, 2, 3])
@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
def test_permute_pe_bitwise(dims, pe, dt):
    nx, ny, nz = dims
    rng = np.random.default_rng(pe)
    a = rng.standard_normal((2, nz, ny, nx)).astype(dt)
    dtype = H.HYSCO_F64 if dt == np.float64 else H.HYSCO_F32
    src = _dev(a)
    fwd = torch.empty_like(src)
    H.hysco_permute_pe(src, fwd, dims, pe, False, dtype, batch=2)
    torch.cuda.synchronize()
    perm = TO_KERNEL[pe]
    expect = np.stack([x.transpose(perm) for x in a])
    n, _ = H.hysco_pe_shape(dims, (1, 1, 1), pe)
    assert expect.shape[1:] == tuple(n)
    assert np.array_equal(fwd.cpu().numpy().reshape(expect.shape), expect)
    back = torch.empty_like(src)
    H.hysco_permute_pe(fwd, back, dims, pe, True, dtype, batch=2)
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), a)


@pytest.mark.parametrize("dtype", [H.HYSCO_F32, H.HYSCO_F64], ids=["f32", "f64"])
def test_fieldmap_cells(dtype):
    shape = (5, 7, 37)
    nd = np.float64 if dtype == H.HYSCO_F64 else np.float32
    b = np.stack([phantom.random_feasible_b(shape, 1.25, seed=s, amp=0.7) for s in (1, 2)]).astype(nd)
    c = H.hysco_create(shape, (1.1, 1.2, 1.25), 2, dtype=dtype)
    out = torch.zeros((2,) + shape, dtype=torch.float64 if dtype == H.HYSCO_F64 else torch.float32, device=DEV)
    torch.cuda.synchronize()
    H.hysco_fieldmap_cells(c, _dev(b), out)
    torch.cuda.synchronize()
    ref = O.avg_pe(b.astype(np.float64))
    tol = 1e-15 if dtype == H.HYSCO_F64 else 1e-7
    assert np.max(np.abs(out.cpu().numpy() - ref)) <= tol * np.max(np.abs(ref))
    mm = out.cpu().numpy().copy()
    H.hysco_fieldmap_cells(c, _dev(b), out, H.HYSCO_FIELDMAP_MM)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), mm)
    H.hysco_fieldmap_cells(c, _dev(b), out, H.HYSCO_FIELDMAP_VOXEL)     # R31: voxels along +PE
    torch.cuda.synchronize()
    assert np.max(np.abs(out.cpu().numpy() - ref / 1.25)) <= tol * np.max(np.abs(ref / 1.25))
    with pytest.raises(H.HyscoError) as e:
        H.hysco_fieldmap_cells(c, _dev(b), out, 7)
    assert e.value.status == H.HYSCO_ERR_ARG
    H.hysco_destroy(c)


def _info(dims, pix):
    i = H.hysco_nifti_info()
    for k in range(3):
        i.dim[k] = dims[k]
        i.pixdim[k] = pix[k]
    i.qfac = 1.0
    i.sform_code = 1
    i.srow[:] = [pix[0], 0, 0, 0, 0, pix[1], 0, 0, 0, 0, pix[2], 0]
    return i


@pytest.mark.parametrize("pe", [2, 3])
def test_cli_end_to_end_matches_direct_api(tmp_path, pe):
    kshape = (10, 12, 24)                            # kernel layout (n1, n2, n3), PE last
    hk = (1.5, 1.4, 1.25)
    pair = phantom.make_pair(kshape, hk, seed=3)
    inv = np.argsort(TO_KERNEL[pe])                  # kernel -> file
    Ipf = np.ascontiguousarray(pair.Ip.transpose(inv))
    Imf = np.ascontiguousarray(pair.Im.transpose(inv))
    nz, ny, nx = Ipf.shape
    # voxel sizes of the file axes so that hysco_pe_shape gives back hk
    pix = [0.0, 0.0, 0.0]
    file_axis_of = {1: (2, 1, 0), 2: (2, 0, 1), 3: (1, 0, 2)}[pe]   # NIfTI axis (0 = x) of n1, n2, n3
    for k in range(3):
        pix[file_axis_of[k]] = hk[k]
    info = _info((nx, ny, nz), pix)
    H.hysco_nifti_write(str(tmp_path / "p.nii.gz"), Ipf, info)
    H.hysco_nifti_write(str(tmp_path / "m.nii.gz"), Imf, info)
    out = str(tmp_path / "o")
    r = subprocess.run([sys.executable, "-m", "paper_2403_10706_b200.cli", str(tmp_path / "p.nii.gz"),
                        str(tmp_path / "m.nii.gz"), "--pe-axis", str(pe), "--out", out, "--stop", "fixed",
                        "--correction", "both"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["kernel_shape"] == list(kshape)
    got = {k: H.hysco_nifti_read(f"{out}_{k}.nii.gz")[0] for k in ("fieldmap", "plus", "minus", "lsq")}

    # direct C-ABI run on the kernel-layout arrays
    c = H.hysco_create(kshape, hk, 1)
    Ip, Im = _dev(pair.Ip[None]), _dev(pair.Im[None])
    H.hysco_bind_images(c, Ip, Im)
    b = torch.zeros((1,) + kshape[:2] + (kshape[2] + 1,), device=DEV)
    Tp, Tm, Tl, fm = (torch.zeros_like(Ip) for _ in range(4))
    torch.cuda.synchronize()
    H.hysco_correct(c, b, Tp, Tm, H.default_ot_opts(), H.default_solve_opts())
    H.hysco_lsq_correct(c, b, Tl, H.default_lsq_opts())
    H.hysco_fieldmap_cells(c, b, fm, H.HYSCO_FIELDMAP_VOXEL)     # the CLI's default unit (R31)
    torch.cuda.synchronize()
    H.hysco_destroy(c)
    for k, t in (("fieldmap", fm), ("plus", Tp), ("minus", Tm), ("lsq", Tl)):
        assert np.array_equal(got[k], t.cpu().numpy()[0].transpose(inv)), k
    bn = b.cpu().numpy()[0].astype(np.float64)
    rp, rm = O.apply_correction(pair.Ip.astype(np.float64), pair.Im.astype(np.float64), bn, hk[2])
    assert np.linalg.norm(got["plus"].transpose(TO_KERNEL[pe]) - rp) <= 1e-5 * np.linalg.norm(rp)
    assert np.linalg.norm(got["minus"].transpose(TO_KERNEL[pe]) - rm) <= 1e-5 * np.linalg.norm(rm)


@pytest.mark.parametrize("opts", [["--solver", "admm", "--correction", "lsq", "--pe-axis", "3"],
                                  ["--precond", "block", "--dtype", "f64", "--pe-axis", "1", "--no-gzip"],
                                  ["--log-iters", "--pe-axis", "2"]],
                         ids=["admm_lsq_pe3", "block_f64_pe1_plain", "log_iters_pe2"])
def test_cli_option_paths(tmp_path, opts):
    """Other CLI paths: outputs exist with the file's shape and voxel sizes and
    are finite; the Jacobian-corrected pair (when written) agrees better than
    the input pair; every least-squares column converged."""
    kshape = (8, 10, 20)
    hk = (1.5, 1.4, 1.25)
    pair = phantom.make_pair(kshape, hk, seed=4)
    pe = int(opts[opts.index("--pe-axis") + 1])
    inv = np.argsort(TO_KERNEL[pe])
    Ipf = np.ascontiguousarray(pair.Ip.transpose(inv))
    Imf = np.ascontiguousarray(pair.Im.transpose(inv))
    nz, ny, nx = Ipf.shape
    pix = [0.0, 0.0, 0.0]
    for k in range(3):
        pix[{1: (2, 1, 0), 2: (2, 0, 1), 3: (1, 0, 2)}[pe][k]] = hk[k]
    info = _info((nx, ny, nz), pix)
    H.hysco_nifti_write(str(tmp_path / "p.nii.gz"), Ipf, info)
    H.hysco_nifti_write(str(tmp_path / "m.nii.gz"), Imf, info)
    out = str(tmp_path / "o")
    r = subprocess.run([sys.executable, "-m", "paper_2403_10706_b200.cli", str(tmp_path / "p.nii.gz"),
                        str(tmp_path / "m.nii.gz"), "--out", out] + opts,
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["kernel_shape"] == list(kshape) and not line["infeasible"]
    ext = ".nii" if "--no-gzip" in opts else ".nii.gz"
    names = ["fieldmap"] + (["lsq"] if "lsq" in opts else ["plus", "minus"])
    for k in names:
        v, i2 = H.hysco_nifti_read(f"{out}_{k}{ext}", H.HYSCO_F64)
        assert v.shape == (nz, ny, nx) and np.isfinite(v).all()
        assert np.allclose(tuple(i2.pixdim), pix, rtol=1e-6)
    if "plus" in names:
        tp = H.hysco_nifti_read(f"{out}_plus{ext}", H.HYSCO_F64)[0]
        tm = H.hysco_nifti_read(f"{out}_minus{ext}", H.HYSCO_F64)[0]
        assert O.relative_improvement(Ipf, Imf, tp, tm) > 50.0
    if "lsq" in names:
        assert line["report"]["lsq"]["unconverged"] == 0
    if "--log-iters" in opts:                    # one record per accepted GN step, descending J
        hist = line["report"]["history"]
        assert [h["k"] for h in hist] == list(range(line["report"]["gn_iters"] + 1))
        assert all(hist[k + 1]["J"] <= hist[k]["J"] for k in range(len(hist) - 1))
        assert r.stderr.count("hysco: GN ") == len(hist)


def test_cli_io_error_in_reader_thread_and_unwritable_output(tmp_path):
    """Exit 4 with the file name and libhysco's message (fetched on the reader
    thread: the message is thread-local) for a truncated input, and for an
    output prefix in a directory that does not exist."""
    a = phantom.make_pair((6, 5, 12), (1.25, 1.25, 1.25), seed=2).Ip
    info = _info((12, 5, 6), (1.25, 1.25, 1.25))
    H.hysco_nifti_write(str(tmp_path / "a.nii"), a, info)
    (tmp_path / "t.nii").write_bytes((tmp_path / "a.nii").read_bytes()[:600])
    r = subprocess.run([sys.executable, "-m", "paper_2403_10706_b200.cli", str(tmp_path / "a.nii"),
                        str(tmp_path / "t.nii"), "--pe-axis", "1", "--out", str(tmp_path / "o")],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 4 and "t.nii" in r.stderr and "trunc" in r.stderr.lower(), r.stderr[-500:]
    r = subprocess.run([sys.executable, "-m", "paper_2403_10706_b200.cli", str(tmp_path / "a.nii"),
                        str(tmp_path / "a.nii"), "--pe-axis", "1", "--out", str(tmp_path / "no" / "o")],
                       capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 4 and "fieldmap" in r.stderr, r.stderr[-500:]
