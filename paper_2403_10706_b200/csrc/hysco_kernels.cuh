// hysco_kernels.cuh — sm_100a kernels of the GN-PCG field-map solve.
//
// Paper: PAPER.md (arXiv 2403.10706), cited P:<line>; readings R<n> in DESIGN.md.
// All kernels are HBM/L2-bandwidth-bound stencil, scan and gather work: no
// dense contraction exists on this path, so there are no tensor-core kernels
// (DESIGN.md "Roofline").  Reductions are deterministic (pair_reduce).
#pragma once

#include "hysco_common.cuh"

namespace hysco {

// ---------------------------------------------------------------------------
// 1D piecewise-linear image model along PE (hat functions, R5)
// value at u = k + del (index units, centre k at integer k) and the slope per
// index unit (right-hand at breakpoints).  del is cell-relative (H3 in
// SURVEY.md): the fractional part is formed from the small displacement, not
// from an absolute coordinate, which keeps fp32 accurate.
// ---------------------------------------------------------------------------
// The interpolated VALUE is always formed in fp64: after a good OT start the
// residual r = T+ - T- is a small difference of ~1e3-sized values, and an
// fp32 value costs ~3e-5 relative error in grad J at the 3T shape (DESIGN.md
// "Precision").  Images stay fp32 in HBM; the slope is returned in T.
template <typename T>
__device__ __forceinline__ void interp_from(const T* __restrict__ s, int n3, int kk, T t, double& val, T& slope) {
    const T v0 = (kk >= 0 && kk < n3) ? s[kk] : T(0);
    const T v1 = (kk + 1 >= 0 && kk + 1 < n3) ? s[kk + 1] : T(0);
    const double td = (double)t;
    val = (1.0 - td) * (double)v0 + td * (double)v1;
    slope = v1 - v0;
}

// Query at u = k + sign * Ab / h3 (A b at the cell centre, in voxels).
// fp32: floor/fraction taken from the small cell-relative offset (accurate t).
// fp64: from the absolute index coordinate, the oracle's exact arithmetic, so
// the one-sided slope chosen at an interpolation kink (|offset| below the
// rounding of k) is the same decision on both sides (R5).
__device__ __forceinline__ void interp_col(const float* __restrict__ s, int n3, int k, float Ab, float sign,
                                           const Geom& g, double& val, float& slope) {
    float del = sign * Ab * g.f_ih3;
    del = fminf(fmaxf(del, (float)-(n3 + 2)), (float)(n3 + 2));   // infeasible b can push far out
    const float fl = floorf(del);
    interp_from(s, n3, k + (int)fl, del - fl, val, slope);
}
__device__ __forceinline__ void interp_col(const double* __restrict__ s, int n3, int k, double Ab, double sign,
                                           const Geom& g, double& val, double& slope) {
    double u = (double)k + sign * (Ab / g.h3);
    u = fmin(fmax(u, -2.0 * (n3 + 2)), 2.0 * (n3 + 2));
    const double fl = floor(u);
    interp_from(s, n3, (int)fl, u - fl, val, slope);
}

// (b_{k+1} - b_k)/h3: fp64 divides like the oracle, fp32 multiplies.
__device__ __forceinline__ float diff_h3(float b0, float b1, const Geom& g) { return (b1 - b0) * g.f_ih3; }
__device__ __forceinline__ double diff_h3(double b0, double b1, const Geom& g) { return (b1 - b0) / g.h3; }

// diag of the in-plane (dims 1,2) Neumann Laplacian at column (i, j) (R3)
__device__ __forceinline__ double diag_lxy(const Geom& g, int i, int j) {   // i: local plane
    return (double)(has_im(g, i) + has_ip(g, i)) * g.ih1sq + (double)((j > 0) + (j < g.n2 - 1)) * g.ih2sq;
}

enum { EVAL_PLAIN = 0, EVAL_GN_START = 1, EVAL_TRIAL = 2 };

// After an evaluation: objective parts (Eq.(2)-(6)), then GN start / Armijo
// acceptance (R15) and the R16 stop rules.  tot = [sum r^2, b^T L b, sum phi,
// ||grad||^2, infeasible (> 0 if any |Db| >= 1)].
__device__ inline void hist_record(HistRec* hr, const PairState& s, int k, double gamma, int pcg, double relres,
                                   double step) {
    if (!hr || k >= HIST_MAX) return;
    HistRec& r = hr[k];
    r.k = k;
    r.pcg_iters = pcg;
    r.ls_halvings = s.ls_halvings;
    r.f_evals = s.f_evals;
    r.J = s.J;
    r.D = s.D;
    r.S = s.S;
    r.P = s.P;
    r.grad_norm = sqrt(s.gnorm2);
    r.gamma = gamma;
    r.relres = relres;
    r.step_max = step;
}

// hr: this pair's history row (HIST_MAX records) or null.
__device__ inline void decide_eval(const Geom& g, const Ctl& c, const SolveParams& sp, int mode, PairState& s,
                                   const double* tot, HistRec* hr = nullptr) {
    const bool active = (mode != EVAL_TRIAL) || s.ls_active;
    if (active) {
        const bool inf = tot[4] > 0.0;
        s.D = 0.5 * g.hd * tot[0];
        s.S = 0.5 * g.hd * tot[1];
        s.P = inf ? INFINITY : 0.5 * g.hd * tot[2];
        s.infeasible = inf ? 1 : 0;
        s.J = inf ? INFINITY : s.D + g.alpha * s.S + g.beta * s.P;
        s.gnorm2 = tot[3];
    }
    if (mode == EVAL_GN_START) {
        s.f_evals = 1;
        s.h_evals = 0;
        s.pcg_iters = 0;
        s.ls_halvings = 0;
        s.gn_k = 0;
        s.J_acc = s.J;
        s.J_prev = s.J;
        s.g0norm = sqrt(s.gnorm2);
        s.relres = 0.0;
        s.stop_reason = s.infeasible ? STOP_INFEASIBLE : STOP_MAXITER;
        s.gn_active = (!s.infeasible && sp.max_gn > 0) ? 1 : 0;
        s.pcg_active = 0;
        s.ls_active = 0;
        hist_record(hr, s, 0, 0.0, 0, 0.0, 0.0);
    } else if (mode == EVAL_TRIAL && active) {
        if (s.ls_restore) {                       // line search failed: state restored at b_old
            s.ls_active = 0;
            s.gn_active = 0;
        } else {
            s.f_evals += 1;
            if (!s.infeasible && (!sp.armijo || s.J <= s.J_acc + sp.c1 * s.gamma * s.gq)) {   // Armijo (R15)
                s.J_prev = s.J_acc;
                s.J_acc = s.J;
                s.gn_k += 1;
                s.ls_active = 0;
                hist_record(hr, s, s.gn_k, s.gamma, s.pcg_k, s.relres, s.gamma * s.qmax);
                int stop = -1;
                if (!sp.fixed) {                  // R16 stopping rules
                    if (sqrt(s.gnorm2) <= sp.tol_grad_rel * s.g0norm) stop = STOP_GRAD;
                    else if (fabs(s.J_prev - s.J) <= sp.tol_dJ_rel * fabs(s.J_prev)) stop = STOP_DJ;
                    else if (s.gamma * s.qmax <= sp.tol_db_rel * g.h3) stop = STOP_DB;
                }
                if (stop >= 0) {
                    s.stop_reason = stop;
                    s.gn_active = 0;
                } else {
                    s.gn_active = s.gn_k < sp.max_gn ? 1 : 0;
                }
            } else {
                s.ls_tries += 1;
                if (s.ls_tries < sp.ls_max) {
                    s.gamma *= 0.5;
                    s.ls_halvings += 1;
                } else {
                    s.stop_reason = STOP_LSFAIL;
                    s.ls_restore = 1;             // next pass: b = b_old, re-evaluate, stop
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// A4 fused evaluation.  A CTA takes a tile of EV_CT
// consecutive columns (one per warp) and stages, with every load of the tile
// in flight, the b columns c0-1 .. c0+EV_CT (own and j-neighbours, shared
// between warps), the i-1 / i+1 b columns and the zero-padded I+, I- columns.
// Per cell: Ab, Db, both gathers with slopes, residual r, GN Jacobian row
// (a, c), phi, phi', phi''.  Per node: grad J (data + alpha hd L b +
// barrier), folded tridiagonal Hessian (dt: diagonal incl. alpha hd L_PE;
// et: super-diagonal incl. -alpha hd / h3^2) -- DESIGN.md "Folded GN Hessian".
// Scalars D, S, P and ||grad||^2 reduce per pair; TRIAL mode also takes the
// Armijo decision (R15).
// ---------------------------------------------------------------------------
#ifndef EV_CT_DEF
#define EV_CT_DEF 8
#endif
constexpr int EV_CT = EV_CT_DEF;   // columns per tile = warps per CTA

// Shared-memory elements of one eval tile (hysco_api.cu sizes the launch with this).
__host__ __device__ inline size_t eval_smem_elems(int n3) {
    const size_t P = (size_t)n3 + 1;
    return (3 * EV_CT + 2) * P + 2 * EV_CT * ((size_t)n3 + 4);
}
// apply_kernel: per warp the column's I+, I- and b
__host__ __device__ inline size_t apply_smem_elems(int n3) { return (size_t)8 * (2 * (size_t)n3 + n3 + 1); }   // 8 warps (256 threads)

// One cell's two gathers (I+ at k + Ab/h3, I- at k - Ab/h3) from columns
// padded with two zeros on each side (index kk clamped to [-2, n3] reads the
// same values as the unpadded bounds tests).  Values in fp64, slopes (per
// index unit) in T.  fp32: floor/fraction from the cell-relative offset and
// v0 + t (v1 - v0) with the difference exact in fp64; fp64: the oracle's
// arithmetic (absolute coordinate, (1-t) v0 + t v1), see R5.
__device__ __forceinline__ void gather_pm(const float* __restrict__ sIp, const float* __restrict__ sIm, int n3, int k,
                                          float Ab, const Geom& g, double& vp, double& vm, float& spl, float& sml) {
    float del = Ab * g.f_ih3;
    const float lim = (float)(n3 + 2);   // infeasible b can push far out
    del = fminf(fmaxf(del, -lim), lim);
    {
        const float fl = floorf(del);
        const int kk = min(max(k + (int)fl, -2), n3);
        const float v0 = sIp[kk], v1 = sIp[kk + 1];
        const double d = (double)v1 - (double)v0;
        vp = fma((double)(del - fl), d, (double)v0);
        spl = (float)d;
    }
    {
        const float md = -del;
        const float fl = floorf(md);
        const int kk = min(max(k + (int)fl, -2), n3);
        const float v0 = sIm[kk], v1 = sIm[kk + 1];
        const double d = (double)v1 - (double)v0;
        vm = fma((double)(md - fl), d, (double)v0);
        sml = (float)d;
    }
}
__device__ __forceinline__ void gather_one(const double* __restrict__ s, int n3, int k, double Ab, double sign,
                                           const Geom& g, double& val, double& slope) {
    double u = (double)k + sign * (Ab / g.h3);
    u = fmin(fmax(u, -2.0 * (n3 + 2)), 2.0 * (n3 + 2));
    const double fl = floor(u);
    const int kk = min(max((int)fl, -2), n3);
    const double t = u - fl, v0 = s[kk], v1 = s[kk + 1];
    val = (1.0 - t) * v0 + t * v1;
    slope = v1 - v0;
}
__device__ __forceinline__ void gather_pm(const double* __restrict__ sIp, const double* __restrict__ sIm, int n3, int k,
                                          double Ab, const Geom& g, double& vp, double& vm, double& spl, double& sml) {
    gather_one(sIp, n3, k, Ab, 1.0, g, vp, spl);
    gather_one(sIm, n3, k, Ab, -1.0, g, vm, sml);
}

// phi, phi', phi'' (Eq.(3)) for |z| < 1 with one reciprocal of (1 - z^2)
// (fp32: the hardware reciprocal, ~1 ulp; the barrier enters J scaled by beta).
__device__ __forceinline__ double recip(double x) { return 1.0 / x; }
__device__ __forceinline__ float recip(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
template <typename T>
__device__ __forceinline__ void phi3(T z, T& f0, T& f1, T& f2) {
    const T z2 = z * z, inv = recip(T(1) - z2);
    f0 = z2 * z2 * inv;
    f1 = T(2) * z * z2 * (T(2) - z2) * inv * inv;
    f2 = T(2) * z2 * (T(6) - T(3) * z2 + z2 * z2) * inv * inv * inv;
}

// Load a column (l < len) into registers NCH x 32 elements at a time, then
// store them to shared memory: all loads of a segment are in flight together
// (columns longer than NCH x 32, e.g. P = 385, take several segments).
template <typename T, int NCH>
__device__ __forceinline__ void stage_col(const T* __restrict__ src, T* dst, int len, int lane) {
    for (int base = 0; base < len; base += 32 * NCH) {
        T v[NCH];
#pragma unroll
        for (int m = 0; m < NCH; m++) {
            const int l = base + 32 * m + lane;
            v[m] = l < len ? src[l] : T(0);
        }
#pragma unroll
        for (int m = 0; m < NCH; m++) {
            const int l = base + 32 * m + lane;
            if (l < len) dst[l] = v[m];
        }
    }
}

// Armijo retry staging: b_t = b_old + gamma q (written back to b for the own
// columns); a plain b column otherwise.  Branch-free within a column so every
// load of the column stays in flight.
template <typename T, int NCH>
__device__ __forceinline__ void stage_bq(const T* __restrict__ src, const T* __restrict__ q, T gm, T* dst,
                                         T* __restrict__ gout, int len, int lane) {
    for (int base = 0; base < len; base += 32 * NCH) {
        T v[NCH], w[NCH];
#pragma unroll
        for (int m = 0; m < NCH; m++) {
            const int l = base + 32 * m + lane;
            v[m] = l < len ? src[l] : T(0);
            w[m] = l < len ? q[l] : T(0);
        }
#pragma unroll
        for (int m = 0; m < NCH; m++) {
            const int l = base + 32 * m + lane;
            const T t = fma(gm, w[m], v[m]);
            if (l < len) dst[l] = t;
            if (gout && l < len) gout[l] = t;
        }
    }
}
template <typename T, int NCH>
__device__ __forceinline__ void stage_b(const T* __restrict__ src, const T* __restrict__ q, T gm, T* dst,
                                        T* __restrict__ gout, int len, int lane) {
    if (q) stage_bq<T, NCH>(src, q, gm, dst, gout, len, lane);   // uniform branch
    else stage_col<T, NCH>(src, dst, len, lane);
}

// bb: the b to evaluate.  EVAL_TRIAL with bold / q given (single-GPU path):
// after a rejected trial (ls_tries > 0) or for the restore pass, the trial b
// = b_old + gamma q (gamma = 0 to restore, R15) is formed while staging and
// written to bb, which replaces the separate retry kernel.
template <typename T, int NCH>
__global__ void __launch_bounds__(32 * EV_CT, (NCH <= 5 ? 3 : 4) * 8 / EV_CT) eval_kernel(Geom g, Ctl c, SolveParams sp, int mode,
                                                   const T* __restrict__ Ip, const T* __restrict__ Im,
                                                   const T* bb, const T* __restrict__ bold,
                                                   const T* __restrict__ q, T* __restrict__ grad,
                                                   T* __restrict__ dt, T* __restrict__ et) {
    count_launch(c);
    if (mode == EVAL_TRIAL && !c.defer) {    // no search pending in any pair (an unrolled retry slot):
        bool any = false;                    // leave at once -- no reduction, no decision -- after
        for (int p = 0; p < (int)gridDim.y; p++) any |= c.st[p].ls_active != 0;   // setting the loop
        if (!any) {                          // conditions a completed evaluation would have set
            if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
                set_cond(c, COND_LS, 0u);
                set_cond(c, COND_GN, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->gn_active != 0; }));
            }
            return;
        }
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int pair = blockIdx.y;
    const int n3 = g.n3, P = g.P, n2 = g.n2, IS = n3 + 4;
    // tile staging: b of columns c0-1 .. c0+EV_CT, b of the i-1 and i+1 columns,
    // I+ / I- of the tile columns with two zero pads on each side
    T* sb = reinterpret_cast<T*>(smem_raw);
    T* sbim = sb + (EV_CT + 2) * P;
    T* sbip = sbim + EV_CT * P;
    T* sIp = sbip + EV_CT * P + (size_t)wid * 2 * IS + 2;
    T* sIm = sIp + IS;
    if (lane < 2) {
        sIp[-2 + lane] = T(0);
        sIp[n3 + lane] = T(0);
        sIm[-2 + lane] = T(0);
        sIm[n3 + lane] = T(0);
    }

    bool active = true;
    if (mode == EVAL_TRIAL) active = c.st[pair].ls_active != 0;
    const T* bsrc = bb;
    const T* qp = nullptr;
    T* bdst = nullptr;
    T gm = T(0);
    if (mode == EVAL_TRIAL && q && (c.st[pair].ls_tries > 0 || c.st[pair].ls_restore)) {
        bsrc = bold;
        qp = q + (size_t)pair * g.ps;
        bdst = const_cast<T*>(bb) + (size_t)pair * g.ps;
        gm = c.st[pair].ls_restore ? T(0) : (T)c.st[pair].gamma;
    }

    const T hd = gw<T>(g.hd, g.f_hd), ahd = gw<T>(g.ahd, g.f_ahd), bh2 = gw<T>(g.bh2, g.f_bh2);
    const T ih3 = gw<T>(g.ih3, g.f_ih3), ih3sq = gw<T>(g.ih3sq, g.f_ih3sq);
    const T ih1sq = gw<T>(g.ih1sq, g.f_ih1sq), ih2sq = gw<T>(g.ih2sq, g.f_ih2sq);
    const long long sI = (long long)n2 * P;   // node stride along dim 1
    const T* bp = bsrc + (size_t)pair * g.ps;
    const T* ipp = Ip + (size_t)pair * g.Nc;
    const T* imp = Im + (size_t)pair * g.Nc;

    double aD = 0, aS = 0, aP = 0, aG = 0, aInf = 0;
    if (active) {
        for (long long c0 = (long long)blockIdx.x * EV_CT; c0 < g.ncol; c0 += (long long)gridDim.x * EV_CT) {
            const long long col = c0 + wid;
            const bool valid = col < g.ncol;
            const int i = (int)(col / n2), j = (int)(col - (long long)i * n2);
            const bool him = valid && has_im(g, i), hip = valid && has_ip(g, i), hjm = j > 0, hjp = j < n2 - 1;
            if (valid) {
                const T* bc = bp + col * P;
                const T* qc = qp ? qp + col * P : nullptr;
                stage_b<T, NCH>(bc, qc, gm, sb + (wid + 1) * P, bdst ? bdst + col * P : nullptr, P, lane);
                if (him) stage_b<T, NCH>(bc - sI, qc ? qc - sI : nullptr, gm, sbim + wid * P, nullptr, P, lane);
                if (hip) stage_b<T, NCH>(bc + sI, qc ? qc + sI : nullptr, gm, sbip + wid * P, nullptr, P, lane);
                stage_col<T, NCH>(ipp + col * n3, sIp, n3, lane);
                stage_col<T, NCH>(imp + col * n3, sIm, n3, lane);
            }
            if (wid == 0 && c0 > 0)
                stage_b<T, NCH>(bp + (c0 - 1) * P, qp ? qp + (c0 - 1) * P : nullptr, gm, sb, nullptr, P, lane);
            if (wid == EV_CT - 1 && c0 + EV_CT < g.ncol)
                stage_b<T, NCH>(bp + (c0 + EV_CT) * P, qp ? qp + (c0 + EV_CT) * P : nullptr, gm, sb + (EV_CT + 1) * P,
                                nullptr, P, lane);
            __syncthreads();
            if (valid) {
                T* gc = grad + (size_t)pair * g.ps + col * P;
                T* dc = dt + (size_t)pair * g.ps + col * P;
                T* ec = et + (size_t)pair * g.ps + col * P;
                const T* sbc = sb + (wid + 1) * P;
                // a missing in-plane neighbour reads the column itself: b - b = 0
                // adds exactly nothing to L b or to the |grad b|^2 terms (R3)
                const T* sjm = hjm ? sbc - P : sbc;
                const T* sjp = hjp ? sbc + P : sbc;
                const T* sim = him ? sbim + wid * P : sbc;
                const T* sip = hip ? sbip + wid * P : sbc;
                T fS = 0, fG = 0, fP = 0;                 // per-lane partials of this column
                T cr_c = 0, c2_c = 0, p1_c = 0, p2_c = 0;   // lane 0: cell (chunk start - 1) -> node
                for (int seg = 0; seg < P; seg += 32 * NCH) {
#pragma unroll
                    for (int m = 0; m < NCH; m++) {
                        const int l = seg + 32 * m + lane;
                        // branch-free: lanes past the last cell compute on a clamped
                        // cell and mask their contributions
                        const bool cv = l < n3;
                        const int lc = cv ? l : n3 - 1;
                        const T b0 = sbc[lc], b1 = sbc[lc + 1];
                        const T Ab = T(0.5) * (b0 + b1);              // averaging operator A
                        const T Db = diff_h3(b0, b1, g);              // finite difference D
                        double vp, vm;
                        T spl, sml;
                        gather_pm(sIp, sIm, n3, lc, Ab, g, vp, vm, spl, sml);   // I+(x + b), I-(x - b)
                        const double Dbd = (double)Db;
                        const double rd = vp * (1.0 + Dbd) - vm * (1.0 - Dbd);  // Eq.(1)-(2) residual (fp64)
                        const T r = (T)rd;
                        const T gg = (spl * (T(1) + Db) + sml * (T(1) - Db)) * ih3;
                        const T s = (T)(vp + vm);
                        const T a = gg * T(0.5) - s * ih3;            // dr_k/db_k
                        const T cc = gg * T(0.5) + s * ih3;           // dr_k/db_{k+1}
                        const T dd = b1 - b0;
                        const bool infz = fabs(Db) >= T(1);           // phi = +inf (Eq.(3))
                        T f0, p1, p2;
                        phi3(infz ? T(0) : Db, f0, p1, p2);
                        if (cv) {
                            aD = fma(rd, rd, aD);
                            fS += dd * dd * ih3sq;
                            fP += f0;
                            if (infz) aInf = 1.0;
                        }
                        const T ar = cv ? a * r : T(0), a2 = cv ? a * a : T(0);
                        const T cr = cv ? cc * r : T(0), c2 = cv ? cc * cc : T(0);
                        p1 = cv ? p1 : T(0);
                        p2 = cv ? p2 : T(0);
                        const T ev = hd * a * cc - bh2 * p2 * ih3sq - ahd * ih3sq;
                        // cell l-1 -> node l: one rotation per quantity; lane 0 takes the
                        // previous chunk's lane 31 (kept from the last rotation)
                        const T rcr = __shfl_sync(FULL, cr, (lane + 31) & 31);
                        const T rc2 = __shfl_sync(FULL, c2, (lane + 31) & 31);
                        const T rp1 = __shfl_sync(FULL, p1, (lane + 31) & 31);
                        const T rp2 = __shfl_sync(FULL, p2, (lane + 31) & 31);
                        const T pcr = lane ? rcr : cr_c, pc2 = lane ? rc2 : c2_c;
                        const T pp1 = lane ? rp1 : p1_c, pp2 = lane ? rp2 : p2_c;
                        cr_c = rcr;
                        c2_c = rc2;
                        p1_c = rp1;
                        p2_c = rp2;
                        if (l < P) {
                            const T bl = sbc[l];
                            T lpe = 0, l1 = 0, l2 = 0;
                            if (l > 0) lpe += bl - sbc[l - 1];
                            if (l < n3) lpe += bl - sbc[l + 1];
                            const T vip = sip[l], vjp = sjp[l];
                            l1 = (bl - sim[l]) + (bl - vip);
                            fS += (vip - bl) * (vip - bl) * ih1sq;
                            l2 = (bl - sjm[l]) + (bl - vjp);
                            fS += (vjp - bl) * (vjp - bl) * ih2sq;
                            const T Lb = lpe * ih3sq + l1 * ih1sq + l2 * ih2sq;
                            const T gv = hd * (pcr + ar) + ahd * Lb + bh2 * (pp1 - p1) * ih3;
                            const T dv = hd * (pc2 + a2) + bh2 * (pp2 + p2) * ih3sq + ahd * T((l > 0) + (l < n3)) * ih3sq;
                            gc[l] = gv;
                            dc[l] = dv;
                            ec[l] = (l < n3) ? ev : T(0);
                            fG += gv * gv;
                        }
                    }
                }
                aS += (double)fS;
                aG += (double)fG;
                aP += (double)fP;
            }
            __syncthreads();
        }
    }
    double v[5] = {aD, aS, aP, aG, aInf}, tot[5];
    if (!pair_reduce<5, 0x10u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {                       // multi-rank: decide after the allreduce (inf flag summed)
        store_red(c, pair, gridDim.y, tot, 5, 0);
        return;
    }
    decide_eval(g, c, sp, mode, c.st[pair], tot, c.hist ? c.hist + (size_t)pair * HIST_MAX : nullptr);
    if (mode == EVAL_GN_START && last_pair(c))
        set_cond(c, COND_GN, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->gn_active != 0; }));
    if (mode == EVAL_TRIAL && last_pair(c)) {
        set_cond(c, COND_LS, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->ls_active != 0; }));
        // the GN step ends with the search; its loop condition is final once no
        // pair searches (ls_retry only moves b), so no separate tail kernel
        set_cond(c, COND_GN, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->gn_active != 0; }));
    }
}

// ---------------------------------------------------------------------------
// A9 Jacobian-modulation correction: T+ = I+(x+b)(1+Db), T- = I-(x-b)(1-Db)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) apply_kernel(Geom g, Ctl c, const T* __restrict__ Ip,
                                                    const T* __restrict__ Im, const T* __restrict__ bb,
                                                    T* __restrict__ Tp, T* __restrict__ Tm, T* __restrict__ bout) {
    count_launch(c);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int pair = blockIdx.y;
    const int n3 = g.n3, P = g.P;
    T* sIp = reinterpret_cast<T*>(smem_raw) + (size_t)wid * (2 * n3 + P);
    T* sIm = sIp + n3;
    T* sb = sIm + n3;
    const size_t pc = (size_t)pair * g.Nc, pn = (size_t)pair * g.ps;
    for (long long col = (long long)blockIdx.x * nwb + wid; col < g.ncol; col += (long long)gridDim.x * nwb) {
        const size_t oc = pc + col * n3, on = pn + col * P;
        for (int k = lane; k < n3; k += 32) {
            sIp[k] = Ip[oc + k];
            sIm[k] = Im[oc + k];
        }
        for (int l = lane; l < P; l += 32) {
            const T v = bb[on + l];
            sb[l] = v;
            if (bout) bout[on + l] = v;   // the solve's b output (replaces a device copy)
        }
        __syncwarp();
        for (int k = lane; k < n3; k += 32) {
            const T b0 = sb[k], b1 = sb[k + 1];
            const T Db = diff_h3(b0, b1, g);
            const T Ab = T(0.5) * (b0 + b1);
            double vp, vm;
            T sp, sm;
            interp_col(sIp, n3, k, Ab, T(1), g, vp, sp);
            interp_col(sIm, n3, k, Ab, T(-1), g, vm, sm);
            if (Tp) Tp[oc + k] = (T)(vp * (double)(T(1) + Db));
            if (Tm) Tm[oc + k] = (T)(vm * (double)(T(1) - Db));
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// A1 OT initialisation
// ---------------------------------------------------------------------------

// positivity shift (R6): tot = [max(-v), max(v)] over both images of the pair
__device__ inline void decide_minmax(const SolveParams& sp, PairState& s, const double* tot) {
    s.vmin = -tot[0];
    s.vmax = tot[1];
    s.degenerate = (s.vmax == s.vmin) ? 1 : 0;
    s.shift = -s.vmin + sp.ot_eps * (s.vmax - s.vmin);
}

// Positivity shift (R6): per pair, min/max over I+ and I-.
template <typename T>
__global__ void __launch_bounds__(256) ot_minmax_kernel(Geom g, Ctl c, SolveParams sp, const T* __restrict__ Ip,
                                                        const T* __restrict__ Im) {
    count_launch(c);
    const int pair = blockIdx.y;
    const size_t pc = (size_t)pair * g.Nc;
    double mn = -INFINITY, mx = -INFINITY;   // max of (-v) and max of v
    long long t0 = 0;
    if constexpr (sizeof(T) == 4) {          // 16-byte loads, max / min in fp32 (exact; widened once)
        const T* a = Ip + pc;
        const T* b = Im + pc;
        if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
            float fmn = -INFINITY, fmx = -INFINITY;
            const long long n4 = g.Nc / 4;
            for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n4;
                 v += (long long)gridDim.x * blockDim.x) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(a) + v);
                const float4 y = __ldg(reinterpret_cast<const float4*>(b) + v);
                fmx = fmaxf(fmx, fmaxf(fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)), fmaxf(fmaxf(y.x, y.y), fmaxf(y.z, y.w))));
                fmn = fmaxf(fmn, fmaxf(fmaxf(fmaxf(-x.x, -x.y), fmaxf(-x.z, -x.w)),
                                       fmaxf(fmaxf(-y.x, -y.y), fmaxf(-y.z, -y.w))));
            }
            mn = (double)fmn;
            mx = (double)fmx;
            t0 = n4 * 4;
        }
    }
    for (long long t = t0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; t < g.Nc;
         t += (long long)gridDim.x * blockDim.x) {
        const double a = (double)Ip[pc + t], b = (double)Im[pc + t];
        mn = fmax(mn, fmax(-a, -b));
        mx = fmax(mx, fmax(a, b));
    }
    double v[2] = {mn, mx}, tot[2];
    if (!pair_reduce<2, 0x3u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {
        store_red(c, pair, gridDim.y, tot, 0, 2);
        return;
    }
    decide_minmax(sp, c.st[pair], tot);
}

// Pseudo-inverse of a piecewise-linear CDF (R8):
// Q(r) = 0 for r <= 0, else x* = min{x in 1..m : C(x) >= r} and
// Q(r) = x* - 1 + (r - C(x*-1)) / (C(x*) - C(x*-1)).
__device__ __forceinline__ double ot_quantile(const double* __restrict__ C, int m, double r) {
    if (r <= 0.0) return 0.0;
    int lo = 1, hi = m;                 // C[m] = 1 >= r
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (C[mid] >= r) hi = mid;
        else lo = mid + 1;
    }
    return (double)(lo - 1) + (r - C[lo - 1]) / (C[lo] - C[lo - 1]);
}

// One warp per PE column: fp64 warp-scan CDFs of the shifted, unit-mass
// columns (R7), quantile search, b0 = h3 (T- - T+)/2 (R9).
template <typename T>
__global__ void __launch_bounds__(256) ot_column_kernel(Geom g, Ctl c, const T* __restrict__ Ip,
                                                        const T* __restrict__ Im, T* __restrict__ b0) {
    count_launch(c);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const int pair = blockIdx.y;
    const int n3 = g.n3, P = g.P;
    double* Cp = reinterpret_cast<double*>(smem_raw) + (size_t)wid * 2 * P;
    double* Cm = Cp + P;
    const size_t pc = (size_t)pair * g.Nc, pn = (size_t)pair * g.ps;
    const double shift = c.st[pair].shift;
    const bool degen = c.st[pair].degenerate != 0;
    for (long long col = (long long)blockIdx.x * nwb + wid; col < g.ncol; col += (long long)gridDim.x * nwb) {
        const T* ip = Ip + pc + col * n3;
        const T* im = Im + pc + col * n3;
        T* bo = b0 + pn + col * P;
        if (degen) {
            for (int l = lane; l < P; l += 32) bo[l] = T(0);
            continue;
        }
        double tp = 0, tm = 0;
        for (int k = lane; k < n3; k += 32) {
            tp += (double)ip[k] + shift;
            tm += (double)im[k] + shift;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            tp += __shfl_xor_sync(FULL, tp, o);
            tm += __shfl_xor_sync(FULL, tm, o);
        }
        const double itp = 1.0 / tp, itm = 1.0 / tm;   // unit mass per column
        double carp = 0, carm = 0;
        for (int base = 0; base < n3; base += 32) {
            const int k = base + lane;
            double wp = 0, wm = 0;
            if (k < n3) {
                wp = ((double)ip[k] + shift) * itp;
                wm = ((double)im[k] + shift) * itm;
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double up = __shfl_up_sync(FULL, wp, o), um = __shfl_up_sync(FULL, wm, o);
                if (lane >= o) {
                    wp += up;
                    wm += um;
                }
            }
            if (k < n3) {
                Cp[k + 1] = carp + wp;
                Cm[k + 1] = carm + wm;
            }
            carp += __shfl_sync(FULL, wp, 31);
            carm += __shfl_sync(FULL, wm, 31);
        }
        __syncwarp();
        if (lane == 0) {
            Cp[0] = 0.0;
            Cm[0] = 0.0;
            Cp[n3] = 1.0;
            Cm[n3] = 1.0;
        }
        __syncwarp();
        for (int l = lane; l < P; l += 32) {
            const double rp = Cp[l], rm = Cm[l];
            // Q+(C+(l)) = l exactly when C+(l-1) < C+(l) (the min-definition then
            // selects x* = l); likewise Q-(C-(l)); else the search decides
            const double qpp = (l > 0 && Cp[l - 1] < rp) ? (double)l : ot_quantile(Cp, n3, rp);
            const double qmm = (l > 0 && Cm[l - 1] < rm) ? (double)l : ot_quantile(Cm, n3, rm);
            const double Tpl = 0.5 * (qpp + ot_quantile(Cm, n3, rp));   // T+ = Q_half o C+
            const double Tml = 0.5 * (ot_quantile(Cp, n3, rm) + qmm);   // T- = Q_half o C-
            bo[l] = (T)(g.h3 * (Tml - Tpl) * 0.5);
        }
        __syncwarp();
    }
}

}  // namespace hysco

#include "hysco_nodes.cuh"
#include "hysco_resident.cuh"
#include "hysco_flat.cuh"
#include "hysco_l2pcg.cuh"
#include "hysco_admm.cuh"
#include "hysco_lsq.cuh"

namespace hysco {

// Multi-rank decisions (Ctl::defer): one thread per pair applies the decision
// of `op` to the allreduced totals, then the loop condition is set (host-read
// mirror `dcond`; multi-rank solves are host-orchestrated).
__global__ void decide_kernel(Geom g, Ctl c, SolveParams sp, int op, int mode, int batch) {
    count_launch(c);
    for (int p = threadIdx.x; p < batch; p += blockDim.x) {
        double tot[RED_W];
        const double* rs = c.red + (size_t)p * RED_W;
        const double* rm = c.red + (size_t)(batch + p) * RED_W;
        PairState& s = c.st[p];
        switch (op) {
            case OP_EVAL:
                for (int k = 0; k < 5; k++) tot[k] = rs[k];
                decide_eval(g, c, sp, mode, s, tot, c.hist ? c.hist + (size_t)p * HIST_MAX : nullptr);
                break;
            case OP_PCG_INIT:
                decide_pcg_init(s, rs);
                break;
            case OP_MATVEC:
                decide_matvec(s, rs);
                break;
            case OP_UPDATE:
                decide_update(sp, s, rs);
                break;
            case OP_TRIAL:
                tot[0] = rs[0];
                tot[1] = rm[0];
                decide_trial(s, tot);
                break;
            case OP_MINMAX:
                decide_minmax(sp, s, rm);
                break;
            default:
                decide_guard(sp, s, rm);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (op == OP_EVAL && mode == EVAL_GN_START)
            set_cond(c, COND_GN, any_pair(c, batch, [](volatile PairState* q) { return q->gn_active != 0; }));
        if ((op == OP_EVAL && mode == EVAL_TRIAL) || op == OP_TRIAL)
            set_cond(c, COND_LS, any_pair(c, batch, [](volatile PairState* q) { return q->ls_active != 0; }));
        if (op == OP_PCG_INIT || op == OP_UPDATE)
            set_cond(c, COND_PCG, any_pair(c, batch, [](volatile PairState* q) { return q->pcg_active != 0; }));
    }
}

}  // namespace hysco
