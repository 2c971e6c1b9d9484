"""C-ABI checks that need no GPU: the library builds, loads and exports every
symbol include/hysco.h and include/hysco_io.h declare; host-side defaults and argument validation."""
import ctypes
import os
import re

import pytest

from paper_2403_10706_b200 import build as B
from paper_2403_10706_b200 import hysco as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = "".join(open(os.path.join(ROOT, "include", f)).read() for f in ("hysco.h", "hysco_io.h"))
    return sorted(set(re.findall(r"HYSCO_API[^;(]*?\b(hysco_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    B.build()
    lib = ctypes.CDLL(B.LIB)
    decl = _declared()
    assert len(decl) >= 16
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(decl) == sorted(H.EXPORTED)


def test_only_c_abi_is_exported():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True).stdout
    syms = [l.split()[-1] for l in out.splitlines() if " T " in l]
    assert syms and all(s.startswith("hysco_") for s in syms), syms


def test_defaults_match_paper_and_readings():
    so = H.default_solve_opts()
    assert (so.max_gn, so.max_pcg, so.pcg_rtol, so.fixed_iters, so.ls_max) == (10, 10, 0.1, 1, 10)   # P:196, R14, R15
    assert so.armijo_c1 == 1e-4 and so.tol_grad_rel == 1e-2 and so.tol_dJ_rel == 1e-4 and so.tol_db_rel == 1e-3
    assert so.armijo == 1
    ot = H.default_ot_opts()
    assert (ot.eps, ot.blur, ot.feas_cap) == (1e-3, 1, 0.95)                                         # R6, R10, R11
    assert H.hysco_version() == 1


def test_struct_layouts_match_header():
    assert ctypes.sizeof(H.hysco_config) == 4 * 8 + 5 * 8 + 2 * 4
    assert ctypes.sizeof(H.hysco_report) == 6 * 4 + 6 * 8
    assert ctypes.sizeof(H.hysco_ot_opts) == 24
    assert ctypes.sizeof(H.hysco_solve_opts) == 2 * 4 + 8 + 2 * 4 + 4 * 8 + 8   # + armijo, padded


@pytest.mark.parametrize("shape", [(0, 4, 8), (4, 4, 1), (4, -1, 8)])
def test_create_rejects_bad_shapes(shape):
    with pytest.raises(H.HyscoError) as e:
        H.hysco_create(shape, (1.0, 1.0, 1.0))
    assert e.value.status == H.HYSCO_ERR_SHAPE


def test_create_rejects_bad_args_and_null_ctx():
    with pytest.raises(H.HyscoError) as e:
        H.hysco_create((4, 4, 8), (1.0, -1.0, 1.0))
    assert e.value.status == H.HYSCO_ERR_ARG
    with pytest.raises(H.HyscoError) as e:
        H.hysco_create((4, 4, 8), (1.0, 1.0, 1.0), dtype=7)
    assert e.value.status == H.HYSCO_ERR_ARG
    L = H.lib()
    assert L.hysco_hessvec(None, None, None) == H.HYSCO_ERR_ARG
    assert L.hysco_destroy(None) == H.HYSCO_ERR_ARG
    assert L.hysco_last_launch_count(None) == -1


def test_no_gpu_fails_loudly_not_silently():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.HyscoError) as e:
        H.hysco_create((4, 4, 8), (1.0, 1.0, 1.0))
    assert e.value.status in (H.HYSCO_ERR_CUDA, H.HYSCO_ERR_NOMEM)
