// hysco_nodes.cuh — node-array kernels (GN Hessian matvec, Jacobi-PCG vector
// ops, Armijo trial/retry, blur, guard) with a warp-per-PE-column mapping.
//
// One warp owns one PE column of P = n3+1 nodes at a time; lane k handles
// nodes l = seg + 32 m + k for the NCH chunks of a 32*NCH-node segment, with
// every chunk's loads issued before any use (memory-level parallelism for an
// HBM-bound kernel).  The column's (i, j) and its in-plane neighbour flags are
// warp-uniform, so there is no per-node index division and no divergence;
// PE neighbours (l-1, l+1) come from warp shuffles of registers already
// loaded.  Included from hysco_kernels.cuh.
#pragma once

namespace hysco {

#define HYSCO_FOR_COLS(g)                                                                        \
    for (long long col = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);         \
         col < (g).ncol; col += (long long)gridDim.x * (blockDim.x >> 5))

struct ColInfo {
    long long off;              // node offset of the column within its pair
    int i, j;
    bool him, hip, hjm, hjp;    // in-plane neighbours exist (Neumann, R3)
};

__device__ __forceinline__ ColInfo col_info(const Geom& g, long long col) {
    ColInfo c;
    c.off = col * g.P;
    c.i = (int)(col / g.n2);
    c.j = (int)(col - (long long)c.i * g.n2);
    c.him = has_im(g, c.i);
    c.hip = has_ip(g, c.i);
    c.hjm = c.j > 0;
    c.hjp = c.j < g.n2 - 1;
    return c;
}

// v[m] holds node l = seg + 32 m + lane (0 beyond the column).  Returns the
// values at l-1 and l+1 (0 outside [0, P)), from shuffles; only the segment
// edges touch memory.
template <int NCH, typename T>
__device__ __forceinline__ void pe_neighbours(const T (&v)[NCH], T (&vm)[NCH], T (&vp)[NCH], const T* __restrict__ colp,
                                              int seg, int P) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int m = 0; m < NCH; m++) {
        const T up = __shfl_up_sync(FULL, v[m], 1);
        const T dn = __shfl_down_sync(FULL, v[m], 1);
        const T prev31 = __shfl_sync(FULL, m > 0 ? v[m > 0 ? m - 1 : 0] : T(0), 31);
        const T next0 = __shfl_sync(FULL, m + 1 < NCH ? v[m + 1 < NCH ? m + 1 : 0] : T(0), 0);
        const int l = seg + 32 * m + lane;
        if (lane > 0) vm[m] = up;
        else if (m > 0) vm[m] = prev31;
        else vm[m] = (l > 0 && l - 1 < P) ? colp[l - 1] : T(0);
        if (lane < 31) vp[m] = dn;
        else if (m + 1 < NCH) vp[m] = next0;
        else vp[m] = (l + 1 < P) ? colp[l + 1] : T(0);
    }
}

// ---- decisions after the PCG / Armijo / guard reductions (see hysco_common.cuh)
// matvec: alpha_c = (r.z)/(p.Hp); breakdown if p.Hp <= 0 (oracle pcg(): keep x)
__device__ inline void decide_matvec(PairState& s, const double* tot) {
    if (!s.pcg_active) return;
    if (tot[0] <= 0.0) {
        s.alpha_c = 0.0;
        s.pcg_active = 0;
    } else {
        s.alpha_c = s.rz / tot[0];
        s.h_evals += 1;
    }
}
// A pair takes a PCG step when it has a GN step to take and no Armijo search
// pending: in the unrolled resident graph (gn_sequence) a rejected trial's
// retry takes the next step's slot, whose PCG kernels then do nothing.
__device__ __forceinline__ bool pcg_step_active(const PairState& s) { return s.gn_active && !s.ls_active; }
// PCG start (R14): tot = [r.z, r.r]
__device__ inline void decide_pcg_init(PairState& s, const double* tot) {
    if (pcg_step_active(s)) {
        s.rz = tot[0];
        s.rr0 = tot[1];
        s.rr = tot[1];
        s.pcg_k = 0;
        s.beta_c = 0.0;
        s.alpha_c = 0.0;   // no pending direction update (hysco_flat.cuh)
        s.relres = tot[1] > 0.0 ? 1.0 : 0.0;
        s.pcg_active = tot[1] > 0.0 ? 1 : 0;
    } else {
        s.pcg_active = 0;
    }
}
// PCG update: tot = [r.z, r.r]; beta and the relative-residual stop
__device__ inline void decide_update(const SolveParams& sp, PairState& s, const double* tot) {
    if (!s.pcg_active) return;
    s.pcg_k += 1;
    s.pcg_iters += 1;
    s.rr = tot[1];
    s.relres = sqrt(tot[1] / s.rr0);
    s.beta_c = tot[0] / s.rz;
    s.rz = tot[0];
    if (s.pcg_k >= sp.max_pcg || (!sp.fixed && s.relres < sp.pcg_rtol)) s.pcg_active = 0;
}
// Armijo start (R15): tot = [grad.q, max|q|]
__device__ inline void decide_trial(PairState& s, const double* tot) {
    if (pcg_step_active(s)) {
        s.gq = tot[0];
        s.qmax = tot[1];
        s.gamma = 1.0;
        s.ls_tries = 0;
        s.ls_restore = 0;
        s.ls_active = 1;
    } else if (!s.gn_active) {
        s.ls_active = 0;
    }                                   // (a pending search keeps its state)
}
// feasibility guard (R10): tot = [max |Db0|]
__device__ inline void decide_guard(const SolveParams& sp, PairState& s, const double* tot) {
    s.maxDb = tot[0];
    s.scale = (tot[0] >= sp.feas_cap) ? sp.feas_cap / tot[0] : 1.0;
}

// ---------------------------------------------------------------------------
// A5 GN Hessian matvec, folded form:
//   Hq = dt q + et_{l-1} q_{l-1} + et_l q_{l+1} + alpha hd L_xy q
// PCG mode also reduces p.Hp and forms alpha_c = (r.z)/(p.Hp) per pair.
// ---------------------------------------------------------------------------
template <typename T, int NCH, bool PCG>
__global__ void __launch_bounds__(256, (NCH <= 5 ? 4 : 3)) matvec_kernel(Geom g, Ctl c, const T* __restrict__ dt,
                                                     const T* __restrict__ et, const T* __restrict__ q,
                                                     T* __restrict__ Hq) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    bool active = true;
    if (PCG) active = c.st[pair].pcg_active != 0;
    const size_t po = (size_t)pair * g.ps;
    const T ahd = (T)g.ahd, ih1sq = (T)g.ih1sq, ih2sq = (T)g.ih2sq;
    const long long sI = (long long)g.n2 * g.P;
    const int P = g.P;
    double acc = 0;
    if (active) {
        HYSCO_FOR_COLS(g) {
            const ColInfo ci = col_info(g, col);
            const T* qc = q + po + ci.off;
            const T* dc = dt + po + ci.off;
            const T* ec = et + po + ci.off;
            T* hc = Hq + po + ci.off;
            for (int seg = 0; seg < P; seg += 32 * NCH) {
                T qv[NCH], dv[NCH], ev[NCH], l1[NCH], l2[NCH];
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    const bool ok = l < P;
                    qv[m] = ok ? qc[l] : T(0);
                    dv[m] = ok ? dc[l] : T(0);
                    ev[m] = ok ? ec[l] : T(0);
                    const T a = (ok && ci.him) ? qc[l - sI] : T(0);
                    const T b = (ok && ci.hip) ? qc[l + sI] : T(0);
                    const T e = (ok && ci.hjm) ? qc[l - P] : T(0);
                    const T f = (ok && ci.hjp) ? qc[l + P] : T(0);
                    l1[m] = (ci.him ? qv[m] - a : T(0)) + (ci.hip ? qv[m] - b : T(0));
                    l2[m] = (ci.hjm ? qv[m] - e : T(0)) + (ci.hjp ? qv[m] - f : T(0));
                }
                // PE neighbours inline per chunk (shuffles; chunk edges from the
                // neighbouring chunk's lane 31 / lane 0, segment edges from memory)
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    T qm = __shfl_up_sync(FULL, qv[m], 1), em = __shfl_up_sync(FULL, ev[m], 1);
                    T qp = __shfl_down_sync(FULL, qv[m], 1);
                    const T qprev = __shfl_sync(FULL, qv[m > 0 ? m - 1 : 0], 31);
                    const T eprev = __shfl_sync(FULL, ev[m > 0 ? m - 1 : 0], 31);
                    const T qnext = __shfl_sync(FULL, qv[m + 1 < NCH ? m + 1 : m], 0);
                    if (lane == 0) {
                        qm = m > 0 ? qprev : ((l > 0 && l - 1 < P) ? qc[l - 1] : T(0));
                        em = m > 0 ? eprev : ((l > 0 && l - 1 < P) ? ec[l - 1] : T(0));
                    }
                    if (lane == 31) qp = m + 1 < NCH ? qnext : ((l + 1 < P) ? qc[l + 1] : T(0));
                    if (l < P) {
                        T h = dv[m] * qv[m];
                        if (l > 0) h += em * qm;
                        if (l < g.n3) h += ev[m] * qp;
                        h += ahd * (l1[m] * ih1sq + l2[m] * ih2sq);
                        hc[l] = h;
                        if (PCG) acc += (double)qv[m] * (double)h;
                    }
                }
            }
        }
    }
    if (!PCG) return;
    double v[1] = {acc}, tot[1];
    if (!pair_reduce<1, 0u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {
        store_red(c, pair, gridDim.y, tot, 1, 0);
        return;
    }
    decide_matvec(c.st[pair], tot);
}

// Jacobi preconditioner M = diag(H_J) = dt + alpha hd diag(L_xy) (R13);
// the in-plane part is a per-column constant.
__device__ __forceinline__ double jacobi_shift(const Geom& g, const ColInfo& ci) {
    return g.ahd * diag_lxy(g, ci.i, ci.j);
}

// PCG start (R14): x = 0, r = -grad, z = r/M, p = z; r.z and r.r per pair.
template <typename T, int NCH>
__global__ void __launch_bounds__(256) pcg_init_kernel(Geom g, Ctl c, const T* __restrict__ grad,
                                                       const T* __restrict__ dt, T* __restrict__ x,
                                                       T* __restrict__ r, T* __restrict__ p) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    const bool active = pcg_step_active(c.st[pair]);
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    double arz = 0, arr = 0;
    if (active) {
        HYSCO_FOR_COLS(g) {
            const ColInfo ci = col_info(g, col);
            const size_t o = po + ci.off;
            const T cm = (T)jacobi_shift(g, ci);
            for (int seg = 0; seg < P; seg += 32 * NCH) {
                T gv[NCH], dv[NCH];
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    gv[m] = l < P ? grad[o + l] : T(0);
                    dv[m] = l < P ? dt[o + l] : T(1);
                }
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    if (l < P) {
                        const T rv = -gv[m];
                        const T z = rv / (dv[m] + cm);
                        x[o + l] = T(0);
                        r[o + l] = rv;
                        p[o + l] = z;
                        arz += (double)rv * (double)z;
                        arr += (double)rv * (double)rv;
                    }
                }
            }
        }
    }
    double v[2] = {arz, arr}, tot[2];
    if (!pair_reduce<2, 0u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {
        store_red(c, pair, gridDim.y, tot, 2, 0);
        return;
    }
    decide_pcg_init(c.st[pair], tot);
    if (last_pair(c)) set_cond(c, COND_PCG, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->pcg_active != 0; }));
}

// A6 PCG update: x += a p, r -= a Hp, z = r/M; r.z, r.r; beta; stop test.
template <typename T, int NCH>
__global__ void __launch_bounds__(256, 4) pcg_update_kernel(Geom g, Ctl c, SolveParams sp,
                                                         const T* __restrict__ dt, const T* __restrict__ p,
                                                         const T* __restrict__ Hp, T* __restrict__ x,
                                                         T* __restrict__ r) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    const bool active = c.st[pair].pcg_active != 0;
    const T a = (T)c.st[pair].alpha_c;
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    double arz = 0, arr = 0;
    if (active) {
        HYSCO_FOR_COLS(g) {
            const ColInfo ci = col_info(g, col);
            const size_t o = po + ci.off;
            const T cm = (T)jacobi_shift(g, ci);
            for (int seg = 0; seg < P; seg += 32 * NCH) {
                T xv[NCH], pv[NCH], hv[NCH], rv[NCH], dv[NCH];
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    const bool ok = l < P;
                    xv[m] = ok ? x[o + l] : T(0);
                    pv[m] = ok ? p[o + l] : T(0);
                    hv[m] = ok ? Hp[o + l] : T(0);
                    rv[m] = ok ? r[o + l] : T(0);
                    dv[m] = ok ? dt[o + l] : T(1);
                }
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    if (l < P) {
                        x[o + l] = xv[m] + a * pv[m];
                        const T rn = rv[m] - a * hv[m];
                        r[o + l] = rn;
                        const T z = rn / (dv[m] + cm);
                        arz += (double)rn * (double)z;
                        arr += (double)rn * (double)rn;
                    }
                }
            }
        }
    }
    double v[2] = {arz, arr}, tot[2];
    if (!pair_reduce<2, 0u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {
        store_red(c, pair, gridDim.y, tot, 2, 0);
        return;
    }
    decide_update(sp, c.st[pair], tot);
    if (last_pair(c)) set_cond(c, COND_PCG, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->pcg_active != 0; }));
}

// New search direction p = z + beta p (z = r/M recomputed, not stored).
template <typename T, int NCH>
__global__ void __launch_bounds__(256) pcg_dir_kernel(Geom g, Ctl c, const T* __restrict__ dt,
                                                      const T* __restrict__ r, T* __restrict__ p) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    if (!c.st[pair].pcg_active) return;
    const T be = (T)c.st[pair].beta_c;
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    HYSCO_FOR_COLS(g) {
        const ColInfo ci = col_info(g, col);
        const size_t o = po + ci.off;
        const T cm = (T)jacobi_shift(g, ci);
        for (int seg = 0; seg < P; seg += 32 * NCH) {
            T rv[NCH], dv[NCH], pv[NCH];
#pragma unroll
            for (int m = 0; m < NCH; m++) {
                const int l = seg + 32 * m + lane;
                const bool ok = l < P;
                rv[m] = ok ? r[o + l] : T(0);
                dv[m] = ok ? dt[o + l] : T(1);
                pv[m] = ok ? p[o + l] : T(0);
            }
#pragma unroll
            for (int m = 0; m < NCH; m++) {
                const int l = seg + 32 * m + lane;
                if (l < P) p[o + l] = rv[m] / (dv[m] + cm) + be * pv[m];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Block preconditioner (R20): B = the per-PE-column tridiagonal blocks
// of H_J, diag M = dt + alpha hd diag(L_xy) (the Jacobi diagonal), off-diagonal
// et (folded).  Thomas algorithm, one LANE per column (the column's loads
// walk consecutive nodes, so each lane stays inside its own cache lines):
//   factor (once per GN step): m_0 = M_0, m_l = M_l - et_{l-1} f_{l-1},
//                              w_l = 1/m_l, f_l = et_l w_l;
//   solve  (per PCG iteration): y_l = (r_l - et_{l-1} y_{l-1}) w_l,
//                               z_l = y_l - f_l z_{l+1}.
// ---------------------------------------------------------------------------
constexpr int BLK_THREADS = 64;   // columns per CTA

template <typename T>
__global__ void __launch_bounds__(BLK_THREADS) bfac_kernel(Geom g, Ctl c, const T* __restrict__ dt,
                                                          const T* __restrict__ et, T* __restrict__ w,
                                                          T* __restrict__ f, int need_active) {
    count_launch(c);
    const int pair = blockIdx.y;
    if (need_active && !pcg_step_active(c.st[pair])) return;
    const long long col = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= g.ncol) return;
    const ColInfo ci = col_info(g, col);
    const size_t o = (size_t)pair * g.ps + ci.off;
    const T cm = (T)jacobi_shift(g, ci);
    const int P = g.P;
    T fprev = T(0), eprev = T(0);
    for (int l = 0; l < P; l++) {
        const T M = __ldg(dt + o + l) + cm;
        const T e = __ldg(et + o + l);             // et at l = n3 is 0
        const T m = M - eprev * fprev;
        const T wl = T(1) / m;
        const T fl = e * wl;
        w[o + l] = wl;
        f[o + l] = fl;
        fprev = fl;
        eprev = e;
    }
}

// z = B^{-1} r per column (hysco_precond_solve; the PCG uses pcg_blk_kernel).
template <typename T>
__global__ void __launch_bounds__(BLK_THREADS) psolve_kernel(Geom g, Ctl c, const T* __restrict__ et,
                                                            const T* __restrict__ w, const T* __restrict__ f,
                                                            const T* __restrict__ r, T* __restrict__ z) {
    count_launch(c);
    const long long col = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= g.ncol) return;
    const size_t o = (size_t)blockIdx.y * g.ps + (size_t)col * g.P;
    const int P = g.P;
    T y = T(0), eprev = T(0);
    for (int l = 0; l < P; l++) {                 // forward: y into z
        y = (__ldg(r + o + l) - eprev * y) * __ldg(w + o + l);
        eprev = __ldg(et + o + l);
        z[o + l] = y;
    }
    T zn = T(0);
    for (int l = P - 1; l >= 0; l--) {            // backward
        zn = z[o + l] - __ldg(f + o + l) * zn;
        z[o + l] = zn;
    }
}

// Warp-level inclusive scans of affine maps y -> A y + B over the 32 lanes of
// a chunk (forward: lane order; backward: reverse lane order).  Composition
// (A, B) after (A', B') = (A A', A B' + B).
template <typename T>
__device__ __forceinline__ void affine_scan_up(T& A, T& B, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T Ap = __shfl_up_sync(FULL, A, o), Bp = __shfl_up_sync(FULL, B, o);
        if (lane >= o) {
            B = fma(A, Bp, B);
            A = A * Ap;
        }
    }
}
template <typename T>
__device__ __forceinline__ void affine_scan_down(T& A, T& B, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T An = __shfl_down_sync(FULL, A, o), Bn = __shfl_down_sync(FULL, B, o);
        if (lane + o < 32) {
            B = fma(A, Bn, B);
            A = A * An;
        }
    }
}

// Block-preconditioned PCG step (R20), one warp per column, fused:
//   ITER: x += a p, r -= a Hp;   INIT: x = 0, r = -grad;
//   z = B^{-1} r by the Thomas recurrences written as affine scans
//     forward  y_l = w_l r_l - (w_l et_{l-1}) y_{l-1},
//     backward z_l = y_l - f_l z_{l+1}     (w, f from bfac_kernel);
//   INIT also p = z;  per pair r.z and r.r -> the Jacobi path's decisions
//   (decide_pcg_init / decide_update: beta = (r.z)_new / (r.z)_old, stop test).
// Columns longer than one NCH x 32 segment keep y in z between the sweeps.
template <typename T, int NCH, bool INIT>
__global__ void __launch_bounds__(256) pcg_blk_kernel(Geom g, Ctl c, SolveParams sp, const T* __restrict__ grad,
                                                      T* __restrict__ p, const T* __restrict__ Hp,
                                                      T* __restrict__ x, T* __restrict__ r,
                                                      const T* __restrict__ w, const T* __restrict__ et,
                                                      const T* __restrict__ f, T* __restrict__ z) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    const bool active = INIT ? pcg_step_active(c.st[pair]) : c.st[pair].pcg_active != 0;
    const T a = INIT ? T(0) : (T)c.st[pair].alpha_c;
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    const bool multi = P > 32 * NCH;
    double arz = 0, arr = 0;
    if (active) {
        HYSCO_FOR_COLS(g) {
            const size_t o = po + (size_t)col * P;
            T rv[NCH], yv[NCH];
            T ycar = T(0), ecar = T(0);          // y and et at the node before this chunk
            for (int seg = 0; seg < P; seg += 32 * NCH) {
                T wv[NCH], ev[NCH];
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    const bool ok = l < P;
                    if (INIT) {
                        rv[m] = ok ? -grad[o + l] : T(0);
                    } else {
                        rv[m] = ok ? r[o + l] : T(0);
                    }
                    wv[m] = ok ? w[o + l] : T(0);
                    ev[m] = ok ? et[o + l] : T(0);
                }
                if (!INIT) {
                    T pv[NCH], hv[NCH], xv[NCH];
#pragma unroll
                    for (int m = 0; m < NCH; m++) {
                        const int l = seg + 32 * m + lane;
                        const bool ok = l < P;
                        pv[m] = ok ? p[o + l] : T(0);
                        hv[m] = ok ? Hp[o + l] : T(0);
                        xv[m] = ok ? x[o + l] : T(0);
                    }
#pragma unroll
                    for (int m = 0; m < NCH; m++) {
                        const int l = seg + 32 * m + lane;
                        rv[m] = rv[m] - a * hv[m];
                        if (l < P) x[o + l] = xv[m] + a * pv[m];
                    }
                }
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    if (l < P) {
                        r[o + l] = rv[m];
                        if (INIT) x[o + l] = T(0);
                    }
                    arr += (double)rv[m] * (double)rv[m];
                    // forward sweep over this chunk: et_{l-1} from the lane below
                    const T eup = __shfl_up_sync(FULL, ev[m], 1);
                    const T em = lane ? eup : ecar;
                    T A = -wv[m] * em, B = wv[m] * rv[m];
                    affine_scan_up(A, B, lane);
                    const T y = fma(A, ycar, B);
                    yv[m] = y;
                    ycar = __shfl_sync(FULL, y, 31);
                    ecar = __shfl_sync(FULL, ev[m], 31);
                    if (multi && l < P) z[o + l] = y;
                }
            }
            // backward sweep from the top segment down
            T zcar = T(0);                        // z at the node after this chunk
            const int nseg = (P + 32 * NCH - 1) / (32 * NCH);
            for (int sgi = nseg - 1; sgi >= 0; sgi--) {
                const int seg = sgi * 32 * NCH;
                T fv[NCH];
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    const bool ok = l < P;
                    fv[m] = ok ? f[o + l] : T(0);
                    if (multi) {
                        yv[m] = ok ? z[o + l] : T(0);
                        rv[m] = ok ? r[o + l] : T(0);
                    }
                }
#pragma unroll
                for (int mm = NCH - 1; mm >= 0; mm--) {
                    const int l = seg + 32 * mm + lane;
                    T A = -fv[mm], B = yv[mm];
                    affine_scan_down(A, B, lane);
                    const T zz = fma(A, zcar, B);
                    zcar = __shfl_sync(FULL, zz, 0);
                    if (l < P) {
                        z[o + l] = zz;
                        if (INIT) p[o + l] = zz;
                    }
                    arz += (double)rv[mm] * (double)zz;
                }
            }
        }
    }
    double v[2] = {arz, arr}, tot[2];
    if (!pair_reduce<2, 0u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {                       // multi-rank: OP_PCG_INIT / OP_UPDATE after the allreduce
        store_red(c, pair, gridDim.y, tot, 2, 0);
        return;
    }
    if (INIT) decide_pcg_init(c.st[pair], tot);
    else decide_update(sp, c.st[pair], tot);
    if (last_pair(c)) set_cond(c, COND_PCG, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->pcg_active != 0; }));
}

// z = r / d elementwise (hysco_precond_solve, Jacobi kind).
template <typename T>
__global__ void __launch_bounds__(256) jacobi_div_kernel(Geom g, Ctl c, const T* __restrict__ r,
                                                         const T* __restrict__ d, T* __restrict__ z) {
    count_launch(c);
    const size_t po = (size_t)blockIdx.y * g.ps;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < g.Nn; t += (long long)gridDim.x * blockDim.x) {
        z[po + t] = r[po + t] / d[po + t];
    }
}

// p = z + beta p with the stored z (block preconditioner).
template <typename T, int NCH>
__global__ void __launch_bounds__(256) pcg_dir_blk_kernel(Geom g, Ctl c, const T* __restrict__ z, T* __restrict__ p) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    if (!c.st[pair].pcg_active) return;
    const T be = (T)c.st[pair].beta_c;
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    HYSCO_FOR_COLS(g) {
        const size_t o = po + (size_t)col * P;
        for (int seg = 0; seg < P; seg += 32 * NCH) {
            T zv[NCH], pv[NCH];
#pragma unroll
            for (int m = 0; m < NCH; m++) {
                const int l = seg + 32 * m + lane;
                zv[m] = l < P ? z[o + l] : T(0);
                pv[m] = l < P ? p[o + l] : T(0);
            }
#pragma unroll
            for (int m = 0; m < NCH; m++) {
                const int l = seg + 32 * m + lane;
                if (l < P) p[o + l] = zv[m] + be * pv[m];
            }
        }
    }
}

// A7 start of the Armijo search: g.q, max|q|, b_old = b, b = b + q (gamma = 1).
template <typename T, int NCH>
__global__ void __launch_bounds__(256) trial_init_kernel(Geom g, Ctl c, const T* __restrict__ grad,
                                                         const T* __restrict__ q, T* __restrict__ b,
                                                         T* __restrict__ bold) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    const bool active = pcg_step_active(c.st[pair]);
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    double agq = 0, aqm = 0;
    if (active) {
        HYSCO_FOR_COLS(g) {
            const size_t o = po + (size_t)col * P;
            for (int seg = 0; seg < P; seg += 32 * NCH) {
                T qv[NCH], gv[NCH], bv[NCH];
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    const bool ok = l < P;
                    qv[m] = ok ? q[o + l] : T(0);
                    gv[m] = ok ? grad[o + l] : T(0);
                    bv[m] = ok ? b[o + l] : T(0);
                }
#pragma unroll
                for (int m = 0; m < NCH; m++) {
                    const int l = seg + 32 * m + lane;
                    if (l < P) {
                        agq += (double)gv[m] * (double)qv[m];
                        aqm = fmax(aqm, (double)fabs(qv[m]));
                        bold[o + l] = bv[m];
                        b[o + l] = bv[m] + qv[m];
                    }
                }
            }
        }
    }
    double v[2] = {agq, aqm}, tot[2];
    if (!pair_reduce<2, 0x2u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {
        store_red(c, pair, gridDim.y, tot, 1, 1);
        return;
    }
    decide_trial(c.st[pair], tot);
    if (last_pair(c)) set_cond(c, COND_LS, any_pair(c, gridDim.y, [](volatile PairState* q2) { return q2->ls_active != 0; }));
}

// Armijo retry / restore: b = b_old + gamma q, or b = b_old after a failed search.
template <typename T, int NCH>
__global__ void __launch_bounds__(256) ls_retry_kernel(Geom g, Ctl c, const T* __restrict__ q,
                                                       const T* __restrict__ bold, T* __restrict__ b) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    const PairState& s = c.st[pair];
    if (!s.ls_active) return;
    const bool restore = s.ls_restore != 0;
    const T gm = (T)s.gamma;
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    HYSCO_FOR_COLS(g) {
        const size_t o = po + (size_t)col * P;
        for (int seg = 0; seg < P; seg += 32 * NCH) {
#pragma unroll
            for (int m = 0; m < NCH; m++) {
                const int l = seg + 32 * m + lane;
                if (l < P) b[o + l] = restore ? bold[o + l] : bold[o + l] + gm * q[o + l];
            }
        }
    }
}

// End of a GN step: loop condition = any pair still iterating.
__global__ void gn_tail_kernel(Ctl c, int batch) {
    count_launch(c);
    if (threadIdx.x == 0)
        set_cond(c, COND_GN, any_pair(c, batch, [](volatile PairState* q) { return q->gn_active != 0; }));
}

// diag(H_J) output for hysco_hess_diag.
template <typename T, int NCH>
__global__ void __launch_bounds__(256) hess_diag_kernel(Geom g, Ctl c, const T* __restrict__ dt, T* __restrict__ out) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const size_t po = (size_t)blockIdx.y * g.ps;
    const int P = g.P;
    HYSCO_FOR_COLS(g) {
        const ColInfo ci = col_info(g, col);
        const size_t o = po + ci.off;
        const T cm = (T)jacobi_shift(g, ci);
        for (int l = lane; l < P; l += 32) out[o + l] = dt[o + l] + cm;
    }
}

// 3-tap periodic Gaussian along one axis of the node array (R11).
template <typename T, int NCH>
__global__ void __launch_bounds__(256) blur_axis_kernel(Geom g, Ctl c, int axis, double w0, double w1,
                                                        const T* __restrict__ in, T* __restrict__ out) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const size_t po = (size_t)blockIdx.y * g.ps;
    const T a = (T)w0, mid = (T)w1;
    const int P = g.P;
    HYSCO_FOR_COLS(g) {
        const ColInfo ci = col_info(g, col);
        const T* cc = in + po + ci.off;
        T* oc = out + po + ci.off;
        if (axis == 2) {
            for (int l = lane; l < P; l += 32) {
                const int lm = l == 0 ? P - 1 : l - 1, lp = l == P - 1 ? 0 : l + 1;
                oc[l] = a * cc[lm] + mid * cc[l] + a * cc[lp];
            }
        } else {
            long long cm_, cp_;
            if (axis == 0 && g.slab) {      // periodic ring across ranks: halo planes hold the wrap
                cm_ = ci.off - (long long)g.n2 * P;
                cp_ = ci.off + (long long)g.n2 * P;
            } else if (axis == 0) {
                cm_ = (long long)(((ci.i + g.n1 - 1) % g.n1) * g.n2 + ci.j) * P;
                cp_ = (long long)(((ci.i + 1) % g.n1) * g.n2 + ci.j) * P;
            } else {
                cm_ = (long long)(ci.i * g.n2 + (ci.j + g.n2 - 1) % g.n2) * P;
                cp_ = (long long)(ci.i * g.n2 + (ci.j + 1) % g.n2) * P;
            }
            const T* mc = in + po + cm_;
            const T* pc = in + po + cp_;
            for (int l = lane; l < P; l += 32) oc[l] = a * mc[l] + mid * cc[l] + a * pc[l];
        }
    }
}

// Feasibility guard (R10): max |Db| per pair; scale to feas_cap if reached.
template <typename T, int NCH>
__global__ void __launch_bounds__(256) guard_max_kernel(Geom g, Ctl c, SolveParams sp, const T* __restrict__ b) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    double mx = 0.0;
    HYSCO_FOR_COLS(g) {
        const T* bc = b + po + (size_t)col * P;
        for (int l = lane; l < g.n3; l += 32) mx = fmax(mx, fabs((double)(bc[l + 1] - bc[l])) / g.h3);
    }
    double v[1] = {mx}, tot[1];
    if (!pair_reduce<1, 0x1u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {
        store_red(c, pair, gridDim.y, tot, 0, 1);
        return;
    }
    decide_guard(sp, c.st[pair], tot);
}

// Last blur pass (along PE, periodic) fused with the guard's max |D b0|
// (R10): each lane forms the blurred node l and l + 1 of its column directly
// (the difference never needs another lane's output).  Single-GPU path.
template <typename T>
__global__ void __launch_bounds__(256) blur_pe_guard_kernel(Geom g, Ctl c, SolveParams sp, double w0, double w1,
                                                            const T* __restrict__ in, T* __restrict__ out) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    const size_t po = (size_t)pair * g.ps;
    const T a = (T)w0, mid = (T)w1;
    const int P = g.P;
    double mx = 0.0;
    HYSCO_FOR_COLS(g) {
        const T* cc = in + po + (size_t)col * P;
        T* oc = out + po + (size_t)col * P;
        for (int l = lane; l < P; l += 32) {
            const int lm = l == 0 ? P - 1 : l - 1, lp = l == P - 1 ? 0 : l + 1, lq = lp == P - 1 ? 0 : lp + 1;
            const T v = a * cc[lm] + mid * cc[l] + a * cc[lp];
            oc[l] = v;
            if (l < g.n3) {
                const T v1 = a * cc[l] + mid * cc[lp] + a * cc[lq];   // blurred node l + 1
                mx = fmax(mx, fabs((double)(v1 - v)) / g.h3);
            }
        }
    }
    double v[1] = {mx}, tot[1];
    if (!pair_reduce<1, 0x1u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    decide_guard(sp, c.st[pair], tot);
}

template <typename T, int NCH>
__global__ void __launch_bounds__(256) guard_scale_kernel(Geom g, Ctl c, T* __restrict__ b) {
    count_launch(c);
    const int lane = threadIdx.x & 31;
    const int pair = blockIdx.y;
    const double sc = c.st[pair].scale;
    if (sc == 1.0) return;
    const size_t po = (size_t)pair * g.ps;
    const int P = g.P;
    HYSCO_FOR_COLS(g) {
        T* bc = b + po + (size_t)col * P;
        for (int l = lane; l < P; l += 32) bc[l] = (T)((double)bc[l] * sc);
    }
}

// Field map at the cell centres, (A b)_k = (b_k + b_{k+1}) / 2 (output of
// the front-end, hysco_io.h), times `scale` (1: mm; 1/h3: voxels, R31).
// Grid-stride over cells of all pairs.
template <typename T>
__global__ void fieldmap_cells_kernel(Geom g, Ctl c, const T* __restrict__ b, T* __restrict__ out, long long total,
                                      T scale) {
    count_launch(c);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long col = i / g.n3, k = i - col * g.n3;    // col runs over pairs x columns
        const T* bc = b + col * g.P;
        out[i] = scale * (T(0.5) * (bc[k] + bc[k + 1]));
    }
}

}  // namespace hysco
