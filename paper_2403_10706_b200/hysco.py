"""Thin ctypes binding of libhysco.so (include/hysco.h) — argument marshalling only.

Every step of the path runs in the CUDA kernels behind the C ABI.  torch is
used only to hold device memory and streams; there is no CPU fallback: if the
extension is missing this module raises at import-use time.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libhysco.so")

HYSCO_OK, HYSCO_INFEASIBLE = 0, 1
HYSCO_ERR_ARG, HYSCO_ERR_SHAPE, HYSCO_ERR_STATE, HYSCO_ERR_CUDA, HYSCO_ERR_NCCL, HYSCO_ERR_NOMEM = -1, -2, -3, -4, -5, -6
HYSCO_F32, HYSCO_F64 = 0, 1
HYSCO_PRECOND_JACOBI, HYSCO_PRECOND_PE_BLOCK = 0, 1
STOP_NAMES = {0: "maxiter", 1: "grad", 2: "dJ", 3: "db", 4: "ls_fail", 5: "infeasible"}

EXPORTED = ["hysco_default_solve_opts", "hysco_default_ot_opts", "hysco_default_admm_opts", "hysco_admm",
            "hysco_create", "hysco_bind_images",
            "hysco_ot_init", "hysco_objective_grad", "hysco_hessvec", "hysco_hess_diag", "hysco_precond_solve",
            "hysco_solve",
            "hysco_apply", "hysco_correct", "hysco_correct_host", "hysco_correct_host_stream",
            "hysco_last_launch_count", "hysco_pcg_path", "hysco_history",
            "hysco_last_error", "hysco_destroy", "hysco_version", "hysco_profile_kernels",
            "hysco_nccl_unique_id", "hysco_create_slab", "hysco_create_loopback", "hysco_group_correct",
            "hysco_group_solve", "hysco_group_admm", "hysco_push_forward", "hysco_default_lsq_opts", "hysco_lsq_correct",
            # front-end (include/hysco_io.h)
            "hysco_nifti_info_read", "hysco_nifti_read", "hysco_nifti_write", "hysco_io_last_error", "hysco_pe_shape",
            "hysco_permute_pe", "hysco_fieldmap_cells", "hysco_fieldmap_cells_units"]
PROF_NAMES = ["matvec", "pcg_update", "pcg_dir", "eval", "pcg_resident", "trial_init", "resident_sync_floor",
              "pcg_l2", "pcg_dirmv", "pcg_upd"]


class HyscoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"hysco status {status}: {msg}")
        self.status = status


class hysco_config(ctypes.Structure):
    _fields_ = [("n1", ctypes.c_int64), ("n2", ctypes.c_int64), ("n3", ctypes.c_int64),
                ("batch", ctypes.c_int64), ("h1", ctypes.c_double), ("h2", ctypes.c_double),
                ("h3", ctypes.c_double), ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("dtype", ctypes.c_int32), ("device", ctypes.c_int32)]


class hysco_ot_opts(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("blur", ctypes.c_int32), ("feas_cap", ctypes.c_double)]


class hysco_solve_opts(ctypes.Structure):
    _fields_ = [("max_gn", ctypes.c_int32), ("max_pcg", ctypes.c_int32), ("pcg_rtol", ctypes.c_double),
                ("fixed_iters", ctypes.c_int32), ("ls_max", ctypes.c_int32), ("armijo_c1", ctypes.c_double),
                ("tol_grad_rel", ctypes.c_double), ("tol_dJ_rel", ctypes.c_double),
                ("tol_db_rel", ctypes.c_double), ("armijo", ctypes.c_int32), ("precond", ctypes.c_int32)]


class hysco_admm_opts(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int32), ("inner", ctypes.c_int32), ("ls_max", ctypes.c_int32),
                ("fixed_iters", ctypes.c_int32), ("tol", ctypes.c_double), ("rho0", ctypes.c_double),
                ("mu", ctypes.c_double), ("tau", ctypes.c_double), ("armijo_c1", ctypes.c_double),
                ("col_tol", ctypes.c_double)]


class hysco_admm_report(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32), ("rho", ctypes.c_double),
                ("r_norm", ctypes.c_double), ("s_norm", ctypes.c_double), ("J", ctypes.c_double),
                ("D", ctypes.c_double), ("S", ctypes.c_double), ("P", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class hysco_iter_record(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("pcg_iters", ctypes.c_int32), ("ls_halvings", ctypes.c_int32),
                ("f_evals", ctypes.c_int32), ("J", ctypes.c_double), ("D", ctypes.c_double), ("S", ctypes.c_double),
                ("P", ctypes.c_double), ("grad_norm", ctypes.c_double), ("gamma", ctypes.c_double),
                ("relres", ctypes.c_double), ("step_max", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class hysco_lsq_opts(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("max_iter", ctypes.c_int32), ("rtol", ctypes.c_double)]


class hysco_lsq_report(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int32), ("unconverged", ctypes.c_int64), ("infeasible", ctypes.c_int64),
                ("max_relres", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class hysco_nifti_info(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int64 * 3), ("pixdim", ctypes.c_double * 3), ("datatype", ctypes.c_int32),
                ("scl_slope", ctypes.c_double), ("scl_inter", ctypes.c_double), ("qform_code", ctypes.c_int32),
                ("sform_code", ctypes.c_int32), ("qfac", ctypes.c_double), ("quatern", ctypes.c_double * 3),
                ("qoffset", ctypes.c_double * 3), ("srow", ctypes.c_double * 12)]


class hysco_report(ctypes.Structure):
    _fields_ = [("gn_iters", ctypes.c_int32), ("f_evals", ctypes.c_int32), ("h_evals", ctypes.c_int32),
                ("pcg_iters", ctypes.c_int32), ("stop_reason", ctypes.c_int32), ("ls_halvings", ctypes.c_int32),
                ("J", ctypes.c_double), ("D", ctypes.c_double), ("S", ctypes.c_double), ("P", ctypes.c_double),
                ("grad_norm", ctypes.c_double), ("last_relres", ctypes.c_double)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["stop"] = STOP_NAMES.get(self.stop_reason, "?")
        return d


_lib = None


def lib():
    """Load the in-tree libhysco.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2403_10706_b200.build` "
                          "(there is no CPU fallback)")
    # torch first: its bundled libnccl.so.2 then satisfies libhysco's NCCL
    # dependency (one NCCL in the process; loading the system NCCL first would
    # break torch's own import)
    import torch  # noqa: F401
    L = ctypes.CDLL(LIB_PATH)
    vp, st = ctypes.c_void_p, ctypes.c_int
    L.hysco_default_solve_opts.argtypes = [ctypes.POINTER(hysco_solve_opts)]
    L.hysco_default_solve_opts.restype = None
    L.hysco_default_ot_opts.argtypes = [ctypes.POINTER(hysco_ot_opts)]
    L.hysco_default_ot_opts.restype = None
    L.hysco_create.argtypes = [ctypes.POINTER(hysco_config), vp, ctypes.POINTER(vp)]
    L.hysco_bind_images.argtypes = [vp, vp, vp]
    L.hysco_ot_init.argtypes = [vp, ctypes.POINTER(hysco_ot_opts), vp]
    L.hysco_objective_grad.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_double), vp]
    L.hysco_hessvec.argtypes = [vp, vp, vp]
    L.hysco_hess_diag.argtypes = [vp, vp]
    L.hysco_default_admm_opts.argtypes = [ctypes.POINTER(hysco_admm_opts)]
    L.hysco_default_admm_opts.restype = None
    L.hysco_admm.argtypes = [vp, vp, ctypes.POINTER(hysco_admm_opts), ctypes.POINTER(hysco_admm_report)]
    L.hysco_admm.restype = st
    L.hysco_push_forward.argtypes = [vp, vp, vp, vp, vp]
    L.hysco_push_forward.restype = st
    L.hysco_default_lsq_opts.argtypes = [ctypes.POINTER(hysco_lsq_opts)]
    L.hysco_default_lsq_opts.restype = None
    L.hysco_lsq_correct.argtypes = [vp, vp, ctypes.POINTER(hysco_lsq_opts), vp, ctypes.POINTER(hysco_lsq_report)]
    L.hysco_lsq_correct.restype = st
    L.hysco_precond_solve.argtypes = [vp, ctypes.c_int32, vp, vp]
    L.hysco_solve.argtypes = [vp, vp, ctypes.POINTER(hysco_solve_opts), ctypes.POINTER(hysco_report)]
    L.hysco_apply.argtypes = [vp, vp, vp, vp]
    L.hysco_correct.argtypes = [vp, ctypes.POINTER(hysco_ot_opts), ctypes.POINTER(hysco_solve_opts), vp, vp, vp,
                                ctypes.POINTER(hysco_report)]
    L.hysco_correct_host.argtypes = [vp, vp, vp, ctypes.POINTER(hysco_ot_opts), ctypes.POINTER(hysco_solve_opts),
                                     vp, vp, vp, ctypes.POINTER(hysco_report)]
    L.hysco_correct_host_stream.argtypes = [vp, ctypes.c_int32, ctypes.POINTER(vp), ctypes.POINTER(vp),
                                            ctypes.POINTER(hysco_ot_opts), ctypes.POINTER(hysco_solve_opts),
                                            ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                            ctypes.POINTER(hysco_report)]
    L.hysco_correct_host_stream.restype = st
    for f in ("hysco_create", "hysco_bind_images", "hysco_ot_init", "hysco_objective_grad", "hysco_hessvec",
              "hysco_hess_diag", "hysco_precond_solve", "hysco_solve", "hysco_apply", "hysco_correct",
              "hysco_correct_host",
              "hysco_destroy"):
        getattr(L, f).restype = st
    L.hysco_destroy.argtypes = [vp]
    L.hysco_last_launch_count.argtypes = [vp]
    L.hysco_last_launch_count.restype = ctypes.c_int64
    L.hysco_pcg_path.argtypes = [vp, ctypes.POINTER(ctypes.c_int32)]
    L.hysco_pcg_path.restype = ctypes.c_int32
    L.hysco_history.argtypes = [vp, ctypes.c_int32, ctypes.POINTER(hysco_iter_record), ctypes.c_int32,
                                ctypes.POINTER(ctypes.c_int32)]
    L.hysco_history.restype = st
    NI = ctypes.POINTER(hysco_nifti_info)
    L.hysco_nifti_info_read.argtypes = [ctypes.c_char_p, NI]
    L.hysco_nifti_read.argtypes = [ctypes.c_char_p, ctypes.c_int, vp, ctypes.c_int64, NI]
    L.hysco_nifti_write.argtypes = [ctypes.c_char_p, ctypes.c_int, vp, NI]
    L.hysco_io_last_error.argtypes = []
    L.hysco_io_last_error.restype = ctypes.c_char_p
    L.hysco_pe_shape.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double), ctypes.c_int32,
                                 ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)]
    L.hysco_permute_pe.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_int, ctypes.c_int64, vp]
    L.hysco_fieldmap_cells.argtypes = [vp, vp, vp]
    L.hysco_fieldmap_cells_units.argtypes = [vp, vp, vp, ctypes.c_int32]
    L.hysco_last_error.argtypes = [vp]
    L.hysco_last_error.restype = ctypes.c_char_p
    L.hysco_profile_kernels.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]
    L.hysco_profile_kernels.restype = st
    L.hysco_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.hysco_nccl_unique_id.restype = st
    L.hysco_create_slab.argtypes = [ctypes.POINTER(hysco_config), ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_char_p, vp, ctypes.POINTER(vp)]
    L.hysco_create_slab.restype = st
    L.hysco_create_loopback.argtypes = [ctypes.POINTER(hysco_config), ctypes.c_int32, vp, ctypes.POINTER(vp)]
    L.hysco_create_loopback.restype = st
    L.hysco_group_correct.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, ctypes.POINTER(hysco_ot_opts),
                                      ctypes.POINTER(hysco_solve_opts), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                      ctypes.POINTER(vp), ctypes.POINTER(hysco_report)]
    L.hysco_group_correct.restype = st
    L.hysco_group_solve.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, ctypes.POINTER(vp),
                                    ctypes.POINTER(hysco_solve_opts), ctypes.POINTER(hysco_report)]
    L.hysco_group_solve.restype = st
    L.hysco_group_admm.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, ctypes.POINTER(vp),
                                   ctypes.POINTER(hysco_admm_opts), ctypes.POINTER(hysco_admm_report)]
    L.hysco_group_admm.restype = st
    L.hysco_version.argtypes = []
    L.hysco_version.restype = ctypes.c_int32
    _lib = L
    return L


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (must be contiguous)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    assert t.is_contiguous(), "tensors must be C-contiguous"
    return t.data_ptr()


def _check(ctx, s, ok=(HYSCO_OK,)):
    if s not in ok:
        msg = lib().hysco_last_error(ctx).decode() if ctx else ""
        raise HyscoError(s, msg)
    return s


def default_solve_opts(**kw):
    o = hysco_solve_opts()
    lib().hysco_default_solve_opts(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def default_admm_opts(**kw):
    o = hysco_admm_opts()
    lib().hysco_default_admm_opts(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def hysco_admm(ctx, b_inout, opts=None, batch=1):
    """ADMM solve from b_inout (device nodes, overwritten); returns per-pair reports."""
    reps = (hysco_admm_report * batch)()
    _check(ctx, lib().hysco_admm(ctx, _ptr(b_inout), ctypes.byref(opts) if opts is not None else None, reps))
    return [r.as_dict() for r in reps]


def default_lsq_opts(**kw):
    """hysco_lsq_opts with the library defaults; `lam` is the C field `lambda`."""
    o = hysco_lsq_opts()
    lib().hysco_default_lsq_opts(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def hysco_push_forward(ctx, b, T, Ip_out, Im_out):
    """Distortion simulation I+- = A+- T (device tensors); returns True if some column was infeasible."""
    s = _check(ctx, lib().hysco_push_forward(ctx, _ptr(b), _ptr(T), _ptr(Ip_out), _ptr(Im_out)),
               (HYSCO_OK, HYSCO_INFEASIBLE))
    return s == HYSCO_INFEASIBLE


def hysco_lsq_correct(ctx, b, T_out, opts=None, batch=1):
    """Least-squares correction of the bound pair into T_out; returns (reports, infeasible)."""
    reps = (hysco_lsq_report * batch)()
    s = _check(ctx, lib().hysco_lsq_correct(ctx, _ptr(b), ctypes.byref(opts) if opts is not None else None,
                                            _ptr(T_out), reps), (HYSCO_OK, HYSCO_INFEASIBLE))
    return [r.as_dict() for r in reps], s == HYSCO_INFEASIBLE


def default_ot_opts(**kw):
    o = hysco_ot_opts()
    lib().hysco_default_ot_opts(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


# ---- C-ABI mirrors (same names) -------------------------------------------

def hysco_create(shape, h, batch=1, alpha=300.0, beta=1e-4, dtype=HYSCO_F32, device=0, stream=None):
    cfg = hysco_config(int(shape[0]), int(shape[1]), int(shape[2]), int(batch), float(h[0]), float(h[1]),
                       float(h[2]), float(alpha), float(beta), int(dtype), int(device))
    out = ctypes.c_void_p()
    s = lib().hysco_create(ctypes.byref(cfg), stream, ctypes.byref(out))
    if s != HYSCO_OK:
        raise HyscoError(s, "hysco_create failed")
    return out.value


def hysco_bind_images(ctx, Ip, Im):
    _check(ctx, lib().hysco_bind_images(ctx, _ptr(Ip), _ptr(Im)))


def hysco_ot_init(ctx, b_out, opts=None):
    _check(ctx, lib().hysco_ot_init(ctx, ctypes.byref(opts) if opts is not None else None, _ptr(b_out)))


def hysco_objective_grad(ctx, b, grad_out=None, batch=1):
    jdsp = (ctypes.c_double * (4 * batch))()
    s = _check(ctx, lib().hysco_objective_grad(ctx, _ptr(b), jdsp, _ptr(grad_out)), (HYSCO_OK, HYSCO_INFEASIBLE))
    return np.array(jdsp[:]).reshape(batch, 4), s == HYSCO_INFEASIBLE


def hysco_hessvec(ctx, q, Hq_out):
    _check(ctx, lib().hysco_hessvec(ctx, _ptr(q), _ptr(Hq_out)))


def hysco_hess_diag(ctx, diag_out):
    _check(ctx, lib().hysco_hess_diag(ctx, _ptr(diag_out)))


def hysco_precond_solve(ctx, kind, r, z_out):
    """z = M^{-1} r at the last objective_grad b (kind: HYSCO_PRECOND_*)."""
    _check(ctx, lib().hysco_precond_solve(ctx, int(kind), _ptr(r), _ptr(z_out)))


def hysco_solve(ctx, b_inout, opts=None, batch=1):
    reps = (hysco_report * batch)()
    s = _check(ctx, lib().hysco_solve(ctx, _ptr(b_inout), ctypes.byref(opts) if opts is not None else None, reps),
               (HYSCO_OK, HYSCO_INFEASIBLE))
    return [r.as_dict() for r in reps], s == HYSCO_INFEASIBLE


def hysco_apply(ctx, b, Ip_corr, Im_corr):
    _check(ctx, lib().hysco_apply(ctx, _ptr(b), _ptr(Ip_corr), _ptr(Im_corr)))


def hysco_correct(ctx, b_out=None, Ip_corr=None, Im_corr=None, ot_opts=None, solve_opts=None, batch=1):
    reps = (hysco_report * batch)()
    s = _check(ctx, lib().hysco_correct(ctx, ctypes.byref(ot_opts) if ot_opts is not None else None,
                                        ctypes.byref(solve_opts) if solve_opts is not None else None,
                                        _ptr(b_out), _ptr(Ip_corr), _ptr(Im_corr), reps),
               (HYSCO_OK, HYSCO_INFEASIBLE))
    return [r.as_dict() for r in reps], s == HYSCO_INFEASIBLE


def hysco_correct_host_stream(ctx, Ips, Ims, b_outs=None, Ip_corrs=None, Im_corrs=None, ot_opts=None,
                              solve_opts=None, batch=1):
    """Pipelined corrections of len(Ips) items on host (pinned) buffers; returns
    (reports per item, any infeasible)."""
    n = len(Ips)

    def arr(xs):
        if xs is None:
            return None
        a = (ctypes.c_void_p * n)()
        for k, x in enumerate(xs):
            a[k] = _ptr(x)
        return a
    reps = (hysco_report * (n * batch))()
    s = _check(ctx, lib().hysco_correct_host_stream(ctx, n, arr(Ips), arr(Ims),
                                                    ctypes.byref(ot_opts) if ot_opts is not None else None,
                                                    ctypes.byref(solve_opts) if solve_opts is not None else None,
                                                    arr(b_outs), arr(Ip_corrs), arr(Im_corrs), reps),
               (HYSCO_OK, HYSCO_INFEASIBLE))
    out = [r.as_dict() for r in reps]
    return [out[k * batch:(k + 1) * batch] for k in range(n)], s == HYSCO_INFEASIBLE


def hysco_correct_host(ctx, Ip, Im, b_out=None, Ip_corr=None, Im_corr=None, ot_opts=None, solve_opts=None,
                       batch=1):
    reps = (hysco_report * batch)()
    s = _check(ctx, lib().hysco_correct_host(ctx, _ptr(Ip), _ptr(Im),
                                             ctypes.byref(ot_opts) if ot_opts is not None else None,
                                             ctypes.byref(solve_opts) if solve_opts is not None else None,
                                             _ptr(b_out), _ptr(Ip_corr), _ptr(Im_corr), reps),
               (HYSCO_OK, HYSCO_INFEASIBLE))
    return [r.as_dict() for r in reps], s == HYSCO_INFEASIBLE


def hysco_last_launch_count(ctx):
    return int(lib().hysco_last_launch_count(ctx))


PCG_PATHS = {0: "streaming", 1: "resident-strips", 2: "resident-tiles", 3: "l2-resident"}


def hysco_pcg_path(ctx):
    """(path name, (TI, TJ, TH, TW)) of the context's PCG (include/hysco.h)."""
    t = (ctypes.c_int32 * 4)()
    k = int(lib().hysco_pcg_path(ctx, t))
    return PCG_PATHS.get(k, "none"), tuple(int(v) for v in t)


def hysco_history(ctx, pair=0):
    """Per-GN-step records of the last solve (include/hysco.h hysco_history):
    a list of dicts, record 0 = the GN start."""
    out = (hysco_iter_record * 64)()
    n = ctypes.c_int32(0)
    _check(ctx, lib().hysco_history(ctx, int(pair), out, 64, ctypes.byref(n)))
    return [out[k].as_dict() for k in range(n.value)]


def hysco_profile_kernels(ctx, reps=20, flush_l2=True):
    out = (ctypes.c_double * len(PROF_NAMES))()
    _check(ctx, lib().hysco_profile_kernels(ctx, int(reps), int(bool(flush_l2)), out))
    return dict(zip(PROF_NAMES, out[:]))


def _cfg(shape, h, batch, alpha, beta, dtype, device):
    return hysco_config(int(shape[0]), int(shape[1]), int(shape[2]), int(batch), float(h[0]), float(h[1]),
                        float(h[2]), float(alpha), float(beta), int(dtype), int(device))


def slab_bounds(n1, nranks, rank):
    """Planes [i0, i1) of `rank` in a split of n1 planes over nranks (as hysco_create_loopback)."""
    return n1 * rank // nranks, n1 * (rank + 1) // nranks


def hysco_nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    s = lib().hysco_nccl_unique_id(buf)
    if s != HYSCO_OK:
        raise HyscoError(s, "ncclGetUniqueId failed")
    return bytes(buf.raw)


def hysco_create_slab(shape_local, h, rank, nranks, n1_global, i0, nccl_id=None, batch=1, alpha=300.0, beta=1e-4,
                      dtype=HYSCO_F32, device=0, stream=None):
    cfg = _cfg(shape_local, h, batch, alpha, beta, dtype, device)
    out = ctypes.c_void_p()
    s = lib().hysco_create_slab(ctypes.byref(cfg), int(rank), int(nranks), int(n1_global), int(i0),
                                nccl_id, stream, ctypes.byref(out))
    if s != HYSCO_OK:
        raise HyscoError(s, "hysco_create_slab failed")
    return out.value


def hysco_create_loopback(shape, h, nranks, batch=1, alpha=300.0, beta=1e-4, dtype=HYSCO_F32, device=0,
                          stream=None):
    cfg = _cfg(shape, h, batch, alpha, beta, dtype, device)
    out = (ctypes.c_void_p * nranks)()
    s = lib().hysco_create_loopback(ctypes.byref(cfg), int(nranks), stream, out)
    if s != HYSCO_OK:
        raise HyscoError(s, "hysco_create_loopback failed")
    return [out[r] for r in range(nranks)]


def _ptrs(ts, n):
    arr = (ctypes.c_void_p * n)()
    for r in range(n):
        arr[r] = _ptr(ts[r]) if ts is not None and ts[r] is not None else None
    return arr


def hysco_group_correct(ctxs, b_out=None, Ip_corr=None, Im_corr=None, ot_opts=None, solve_opts=None, batch=1):
    n = len(ctxs)
    cs = (ctypes.c_void_p * n)(*ctxs)
    reps = (hysco_report * batch)()
    s = _check(ctxs[0], lib().hysco_group_correct(cs, n, ctypes.byref(ot_opts) if ot_opts is not None else None,
                                                  ctypes.byref(solve_opts) if solve_opts is not None else None,
                                                  _ptrs(b_out, n), _ptrs(Ip_corr, n), _ptrs(Im_corr, n), reps),
               (HYSCO_OK, HYSCO_INFEASIBLE))
    return [r.as_dict() for r in reps], s == HYSCO_INFEASIBLE


def hysco_group_admm(ctxs, b_inout, opts=None, batch=1):
    """ADMM on a loopback slab group (the transposed z-update, include/hysco.h):
    b_inout[r] = rank r's dense slab of nodes (overwritten); per-pair reports."""
    n = len(ctxs)
    cs = (ctypes.c_void_p * n)(*ctxs)
    reps = (hysco_admm_report * batch)()
    _check(ctxs[0], lib().hysco_group_admm(cs, n, _ptrs(b_inout, n), ctypes.byref(opts) if opts is not None else None,
                                           reps))
    return [r.as_dict() for r in reps]


def hysco_group_solve(ctxs, b_inout, solve_opts=None, batch=1):
    n = len(ctxs)
    cs = (ctypes.c_void_p * n)(*ctxs)
    reps = (hysco_report * batch)()
    s = _check(ctxs[0], lib().hysco_group_solve(cs, n, _ptrs(b_inout, n),
                                                ctypes.byref(solve_opts) if solve_opts is not None else None, reps),
               (HYSCO_OK, HYSCO_INFEASIBLE))
    return [r.as_dict() for r in reps], s == HYSCO_INFEASIBLE


def hysco_last_error(ctx):
    return lib().hysco_last_error(ctx).decode()


def hysco_destroy(ctx):
    if ctx:
        lib().hysco_destroy(ctx)


def hysco_version():
    return int(lib().hysco_version())


# ---- front-end (include/hysco_io.h; NEXT-4) --------------------------------

def _io_check(s):
    if s != HYSCO_OK:
        raise HyscoError(s, lib().hysco_io_last_error().decode())
    return s


def hysco_nifti_info_read(path):
    info = hysco_nifti_info()
    _io_check(lib().hysco_nifti_info_read(os.fsencode(path), ctypes.byref(info)))
    return info


def hysco_nifti_read(path, dtype=HYSCO_F32):
    """Voxel data as a C array [nz][ny][nx] of dtype (scaled), and the header."""
    info = hysco_nifti_info_read(path)
    nx, ny, nz = info.dim
    out = np.empty((nz, ny, nx), dtype=np.float64 if dtype == HYSCO_F64 else np.float32)
    _io_check(lib().hysco_nifti_read(os.fsencode(path), dtype, _ptr(out), out.size, ctypes.byref(info)))
    return out, info


def hysco_nifti_write(path, data, info):
    """data: C array [nz][ny][nx] of float32 / float64; dims, voxel sizes, geometry from info."""
    dtype = HYSCO_F64 if data.dtype == np.float64 else HYSCO_F32
    assert data.dtype in (np.float32, np.float64) and data.shape == (info.dim[2], info.dim[1], info.dim[0])
    arr = np.ascontiguousarray(data)      # a copy for non-contiguous views: keep it alive across the call
    _io_check(lib().hysco_nifti_write(os.fsencode(path), dtype, _ptr(arr), ctypes.byref(info)))


def hysco_pe_shape(dims, pixdim, pe_axis):
    """Kernel layout (n1, n2, n3) and voxel sizes of a volume with NIfTI dims whose PE axis is pe_axis."""
    d = (ctypes.c_int64 * 3)(*[int(x) for x in dims])
    p = (ctypes.c_double * 3)(*[float(x) for x in pixdim])
    n = (ctypes.c_int64 * 3)()
    h = (ctypes.c_double * 3)()
    _io_check(lib().hysco_pe_shape(d, p, int(pe_axis), n, h))
    return tuple(n), tuple(h)


def hysco_permute_pe(d_in, d_out, dims, pe_axis, inverse=False, dtype=HYSCO_F32, batch=1, stream=None):
    d = (ctypes.c_int64 * 3)(*[int(x) for x in dims])
    _io_check(lib().hysco_permute_pe(_ptr(d_in), _ptr(d_out), d, int(pe_axis), int(bool(inverse)), dtype,
                                     int(batch), stream))


HYSCO_FIELDMAP_MM, HYSCO_FIELDMAP_VOXEL = 0, 1


def hysco_fieldmap_cells(ctx, b, out, units=None):
    """Field map at the cell centres: mm along +PE (units None / HYSCO_FIELDMAP_MM)
    or voxels (HYSCO_FIELDMAP_VOXEL)."""
    if units is None:
        _check(ctx, lib().hysco_fieldmap_cells(ctx, _ptr(b), _ptr(out)))
    else:
        _check(ctx, lib().hysco_fieldmap_cells_units(ctx, _ptr(b), _ptr(out), int(units)))
