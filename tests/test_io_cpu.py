"""Front-end host functions (include/hysco_io.h, NEXT-4; readings R30-R31):
NIfTI-1 read / write through the C ABI (no GPU needed) against fixtures built
byte by byte here from the NIfTI-1 header layout (Python struct, independent
of the library's parser), and the PE-last layout table against numpy."""
import gzip
import struct

import numpy as np
import pytest

from paper_2403_10706_b200 import hysco as H


def _header(dims, datatype, bitpix, pixdim=(1.0, 1.0, 1.0), vox_offset=352.0, slope=1.0, inter=0.0, ndim=3,
            dim4=1, endian="<", magic=b"n+1\0"):
    """The 348-byte NIfTI-1 header (field offsets of nifti1.h), plus the 4-byte extension flag."""
    h = bytearray(348)
    struct.pack_into(endian + "i", h, 0, 348)
    struct.pack_into(endian + "8h", h, 40, ndim, dims[0], dims[1], dims[2], dim4, 1, 1, 1)
    struct.pack_into(endian + "h", h, 70, datatype)
    struct.pack_into(endian + "h", h, 72, bitpix)
    struct.pack_into(endian + "8f", h, 76, 1.0, pixdim[0], pixdim[1], pixdim[2], 0, 0, 0, 0)
    struct.pack_into(endian + "f", h, 108, vox_offset)
    struct.pack_into(endian + "f", h, 112, slope)
    struct.pack_into(endian + "f", h, 116, inter)
    struct.pack_into(endian + "h", h, 254, 1)                       # sform_code
    struct.pack_into(endian + "12f", h, 280, pixdim[0], 0, 0, -10.0, 0, pixdim[1], 0, -20.0, 0, 0, pixdim[2], 5.0)
    h[344:348] = magic
    return bytes(h) + b"\0" * 4


def _write(path, data_bytes, **kw):
    raw = _header(**kw) + data_bytes
    if str(path).endswith(".gz"):
        raw = gzip.compress(raw)
    open(path, "wb").write(raw)


def _info(dims, pixdim=(1.2, 1.3, 1.4)):
    i = H.hysco_nifti_info()
    for k in range(3):
        i.dim[k] = dims[k]
        i.pixdim[k] = pixdim[k]
    i.qfac = 1.0
    i.sform_code = 1
    i.srow[:] = [pixdim[0], 0, 0, -1.5, 0, pixdim[1], 0, 2.5, 0, 0, pixdim[2], 3.5]
    return i


@pytest.mark.parametrize("ext", [".nii", ".nii.gz"])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_write_read_roundtrip_bitwise(tmp_path, ext, dt):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((3, 4, 5)).astype(dt)                  # [nz][ny][nx]
    p = str(tmp_path / ("v" + ext))
    H.hysco_nifti_write(p, a, _info((5, 4, 3)))
    b, info = H.hysco_nifti_read(p, H.HYSCO_F64 if dt == np.float64 else H.HYSCO_F32)
    assert b.dtype == dt and np.array_equal(a, b)
    assert tuple(info.dim) == (5, 4, 3)
    assert np.allclose(tuple(info.pixdim), (1.2, 1.3, 1.4), rtol=1e-7)
    assert info.sform_code == 1 and np.allclose(list(info.srow), _info((5, 4, 3)).srow[:], rtol=1e-7)
    if ext == ".nii.gz":
        assert open(p, "rb").read(2) == b"\x1f\x8b"


def test_writer_byte_layout(tmp_path):
    p = str(tmp_path / "z.nii")
    H.hysco_nifti_write(p, np.zeros((2, 2, 2), np.float32), _info((2, 2, 2)))
    raw = open(p, "rb").read()
    assert len(raw) == 352 + 32 and raw[352:] == b"\0" * 32
    assert struct.unpack_from("<i", raw, 0)[0] == 348
    assert struct.unpack_from("<8h", raw, 40)[:4] == (3, 2, 2, 2)
    assert struct.unpack_from("<hh", raw, 70) == (16, 32)
    assert struct.unpack_from("<f", raw, 108)[0] == 352.0
    assert struct.unpack_from("<ff", raw, 112) == (1.0, 0.0)
    assert raw[344:348] == b"n+1\0"


def test_int16_scaled_and_vox_offset(tmp_path):
    raw = np.array([[[0, 1], [2, -3]], [[4, 5], [300, -7]]], dtype="<i2")     # [nz][ny][nx]
    p = str(tmp_path / "s.nii")
    hdr_pad = b"\0" * 48                                                       # vox_offset 400: 48 bytes of extension
    open(p, "wb").write(_header((2, 2, 2), 4, 16, slope=2.0, inter=1.0, vox_offset=400.0) + hdr_pad + raw.tobytes())
    v, info = H.hysco_nifti_read(p, H.HYSCO_F64)
    assert np.array_equal(v, 2.0 * raw.astype(np.float64) + 1.0)
    assert info.datatype == 4


def test_uint8_gzip_and_slope_zero_means_unscaled(tmp_path):
    raw = np.arange(24, dtype=np.uint8).reshape(2, 3, 4)
    p = str(tmp_path / "u.nii.gz")
    _write(p, raw.tobytes(), dims=(4, 3, 2), datatype=2, bitpix=8, slope=0.0, inter=5.0)
    v, _ = H.hysco_nifti_read(p)
    assert np.array_equal(v, raw.astype(np.float32))


def test_4d_singleton_squeezed(tmp_path):
    raw = np.arange(8, dtype="<f4").reshape(2, 2, 2)
    p = str(tmp_path / "f.nii")
    _write(p, raw.tobytes(), dims=(2, 2, 2), datatype=16, bitpix=32, ndim=4, dim4=1)
    v, _ = H.hysco_nifti_read(p)
    assert np.array_equal(v, raw)


@pytest.mark.parametrize("kind", ["sizeof", "bigendian", "magic", "4d", "datatype", "missing", "nan"])
def test_read_errors(tmp_path, kind):
    p = str(tmp_path / "e.nii")
    data = np.ones(8, "<f4").tobytes()
    kw = dict(dims=(2, 2, 2), datatype=16, bitpix=32)
    if kind == "sizeof":
        raw = bytearray(_header(**kw) + data)
        struct.pack_into("<i", raw, 0, 540)
        open(p, "wb").write(bytes(raw))
    elif kind == "bigendian":
        _write(p, np.ones(8, ">f4").tobytes(), endian=">", **kw)
    elif kind == "magic":
        _write(p, data, magic=b"ni1\0", **kw)
    elif kind == "4d":
        _write(p, data * 2, ndim=4, dim4=2, **kw)
    elif kind == "datatype":
        _write(p, data, dims=(2, 2, 2), datatype=128, bitpix=24)
    elif kind == "nan":
        _write(p, np.array([1, 2, np.nan, 4, 5, 6, 7, 8], "<f4").tobytes(), **kw)
    else:
        p = str(tmp_path / "does_not_exist.nii")
    with pytest.raises(H.HyscoError) as e:
        H.hysco_nifti_read(p)
    assert e.value.status == H.HYSCO_ERR_ARG
    if kind == "bigendian":
        assert "big-endian" in str(e.value)


def test_read_shape_mismatch_and_write_nan(tmp_path):
    p = str(tmp_path / "m.nii")
    H.hysco_nifti_write(p, np.ones((2, 2, 2), np.float32), _info((2, 2, 2)))
    out = np.empty(7, np.float32)
    L = H.lib()
    assert L.hysco_nifti_read(p.encode(), H.HYSCO_F32, out.ctypes.data, 7, None) == H.HYSCO_ERR_SHAPE
    bad = np.ones((2, 2, 2), np.float32)
    bad[1, 1, 1] = np.inf
    with pytest.raises(H.HyscoError):
        H.hysco_nifti_write(str(tmp_path / "n.nii"), bad, _info((2, 2, 2)))
    assert not (tmp_path / "n.nii").exists()


def test_pe_shape_matches_numpy_layout():
    """R30: the kernel layout moves the PE axis last and keeps the other two in file order."""
    nx, ny, nz = 5, 6, 7
    a = np.zeros((nz, ny, nx))
    expect = {1: a.shape, 2: a.transpose(0, 2, 1).shape, 3: a.transpose(1, 2, 0).shape}
    hx = (1.1, 1.2, 1.3)
    for pe in (1, 2, 3):
        n, h = H.hysco_pe_shape((nx, ny, nz), hx, pe)
        assert n == expect[pe]
        assert n[2] == (nx, ny, nz)[pe - 1] and h[2] == hx[pe - 1]
        assert sorted(h) == sorted(hx)
    with pytest.raises(H.HyscoError):
        H.hysco_pe_shape((nx, ny, nz), hx, 4)


def test_large_gzip_is_multi_member_and_standard(tmp_path):
    """> 4 MiB: several gzip members compressed in parallel; Python's gzip
    (an independent reader) must see the plain NIfTI byte stream."""
    rng = np.random.default_rng(2)
    a = rng.standard_normal((40, 100, 300)).astype(np.float32)     # 4.8 MB of voxels
    p = str(tmp_path / "big.nii.gz")
    H.hysco_nifti_write(p, a, _info((300, 100, 40)))
    raw = gzip.decompress(open(p, "rb").read())
    assert len(raw) == 352 + a.nbytes
    assert np.array_equal(np.frombuffer(raw[352:], "<f4").reshape(a.shape), a)
    assert open(p, "rb").read().count(b"\x1f\x8b\x08") >= 2         # more than one member
    b, _ = H.hysco_nifti_read(p)
    assert np.array_equal(a, b)


def test_write_non_contiguous_view_keeps_data_alive(tmp_path):
    """A transposed / strided array is copied to C order for the C call; the
    copy must outlive the call (the file holds the view's values, not freed
    memory).  Large enough that a freed buffer would be unmapped."""
    rng = np.random.default_rng(5)
    base = rng.standard_normal((60, 70, 80)).astype(np.float32)
    for view in (base.transpose(2, 1, 0), base[::2, :, ::2]):
        assert not view.flags["C_CONTIGUOUS"]
        nz, ny, nx = view.shape
        p = str(tmp_path / "v.nii.gz")
        H.hysco_nifti_write(p, view, _info((nx, ny, nz)))
        back, _ = H.hysco_nifti_read(p)
        assert np.array_equal(back, view)


def _cli(tmp_path, *argv):
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return subprocess.run([sys.executable, "-m", "paper_2403_10706_b200.cli", *argv], capture_output=True,
                          text=True, cwd=root, timeout=300)


def test_cli_exit_codes_before_the_gpu(tmp_path):
    """The CLI's documented exit status (cli.py): 4 for an unreadable input, 2
    for images of different sizes; both are decided before any GPU work."""
    a = np.ones((4, 5, 6), np.float32)
    H.hysco_nifti_write(str(tmp_path / "a.nii"), a, _info((6, 5, 4)))
    H.hysco_nifti_write(str(tmp_path / "b.nii"), np.ones((4, 5, 7), np.float32), _info((7, 5, 4)))
    r = _cli(tmp_path, str(tmp_path / "a.nii"), str(tmp_path / "missing.nii"), "--pe-axis", "2", "--out",
             str(tmp_path / "o"))
    assert r.returncode == 4 and "missing.nii" in r.stderr
    r = _cli(tmp_path, str(tmp_path / "a.nii"), str(tmp_path / "b.nii"), "--pe-axis", "2", "--out",
             str(tmp_path / "o"))
    assert r.returncode == 2 and "differ" in r.stderr
    assert not list(tmp_path.glob("o_*"))
