"""CPU emulation (NumPy float32) of the eval kernel's residual forming, to pick
an fp32 formula before touching the kernel: r_k = I+(u+)(1+Db) - I-(u-)(1-Db)
(Eq.(1)-(2)) formed (a) in fp64 from the fp32 inputs (the kernel today),
(b) naively in fp32, (c) rearranged in fp32 as (p0 - m0) + (tp dp - tm dm) +
Db (vp + vm), which never subtracts the ~1e3-sized interpolated values.
Reports the relative L2 error of the residual's gradient contribution and of
the whole gradient (the 1e-5 gate, R18) at the OT start and at b_true."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from synth import phantom
from oracle import hysco_oracle as O

f32 = np.float32


def forms(Ip, Im, b, h3):
    n1, n2, n3 = Ip.shape
    b32 = b.astype(f32)
    Ab = (f32(0.5) * (b32[..., :-1] + b32[..., 1:])).astype(f32)
    Db = ((b32[..., 1:] - b32[..., :-1]) * f32(1.0 / h3)).astype(f32)
    k = np.arange(n3)
    pad = lambda I: np.concatenate([np.zeros(I.shape[:-1] + (2,), f32), I, np.zeros(I.shape[:-1] + (2,), f32)], -1)
    Pp, Pm = pad(Ip), pad(Im)
    dl = (Ab * f32(1.0 / h3)).astype(f32)
    lim = f32(n3 + 2)
    dl = np.clip(dl, -lim, lim)
    flp = np.floor(dl); tp = (dl - flp).astype(f32)
    md = -dl; flm = np.floor(md); tm = (md - flm).astype(f32)
    kp = np.clip(k + flp.astype(int), -2, n3) + 2
    km = np.clip(k + flm.astype(int), -2, n3) + 2
    g = lambda A, idx: np.take_along_axis(A, idx, -1)
    p0, p1 = g(Pp, kp), g(Pp, kp + 1)
    m0, m1 = g(Pm, km), g(Pm, km + 1)
    # (a) fp64 forming (today)
    vp = tp.astype(float) * (p1.astype(float) - p0) + p0
    vm = tm.astype(float) * (m1.astype(float) - m0) + m0
    Dd = Db.astype(float)
    ra = vp * (1 + Dd) - vm * (1 - Dd)
    # (b) naive fp32
    vp32 = (tp * (p1 - p0) + p0).astype(f32)
    vm32 = (tm * (m1 - m0) + m0).astype(f32)
    rb = (vp32 * (f32(1) + Db) - vm32 * (f32(1) - Db)).astype(f32)
    # (c) rearranged fp32 (fma emulated exactly in fp64 then rounded once)
    dp = (p1 - p0).astype(f32)
    dm = (m1 - m0).astype(f32)
    tmdm = (tm * dm).astype(f32)
    inner = (tp.astype(float) * dp - tmdm).astype(f32)          # fmaf(tp, dp, -tm dm)
    dvpm = ((p0 - m0).astype(f32) + inner).astype(f32)
    s32 = (vp32 + vm32).astype(f32)
    rc = (Db.astype(float) * s32 + dvpm).astype(f32)              # fmaf(Db, s, dvpm)
    return ra, rb.astype(float), rc.astype(float)


def main():
    p = phantom.make_config(sys.argv[1] if len(sys.argv) > 1 else "C2_hcp3t")
    Ip, Im = p.Ip, p.Im
    h = p.h
    I64 = Ip.astype(float), Im.astype(float)
    b0, _ = O.ot_init(*I64, h[2])
    for name, b in (("OT b0", b0), ("b_true", p.b_true)):
        st = O.evaluate(*I64, b.astype(f32).astype(float), h)
        rex = st.r if hasattr(st, "r") else None
        ra, rb, rc = forms(Ip, Im, b, h[2])
        ref = ra if rex is None else rex
        gd = lambda r: O.residual_jac_T(st, r) * np.prod(h)
        G = np.linalg.norm(st.grad)
        for lab, r in (("fp64 forming", ra), ("naive fp32", rb), ("rearranged fp32", rc)):
            e = np.linalg.norm(gd(r) - gd(ref)) / G
            print(f"{name:7s} {lab:16s} rel L2 of r {np.linalg.norm(r - ref) / np.linalg.norm(ref):.2e}, "
                  f"of grad {e:.2e}")


if __name__ == "__main__":
    main()
