// hysco_l2pcg.cuh — persistent L2-resident Jacobi-PCG (A5 + A6 for a whole GN
// step in ONE cooperative launch), for volumes whose PCG state does not fit
// in shared memory and registers but whose working set (p, dt, et, r, x, Hp:
// 6 node arrays) is about the size of the 126 MB L2 -- e.g. HCP 7T (5.3 M
// nodes, 127 MB in fp32).  Included from hysco_kernels.cuh after
// hysco_resident.cuh, whose synchronisation it reuses.
//
// Each CTA (one per SM) owns the contiguous PE-column range [c0, c1) of the
// pair for the whole solve, so its node arrays stay in L2 between iterations
// and no launch boundary separates the three phases of an iteration:
//   A  p-halo acquire (the CTAs owning the i-1 / i+1 columns) ->
//      Hp = H p over the own columns (matvec body) and p.Hp -> all-reduce
//   B  x += a p, r -= a Hp, z = r/M; r.z, r.r -> all-reduce (update body)
//   C  p = z + beta p -> p-halo release (direction body)
// The per-column arithmetic is the streaming kernels' (hysco_nodes.cuh), one
// warp per column, so results equal the streaming path up to the order of the
// per-pair fp64 sums.  A thread touches the same nodes of its own columns in
// every phase (same column loop, same lane mapping), so x, r, Hp need no
// synchronisation between phases; p of other columns is read through L2
// (ld.global.cg: L1 is not coherent) after the halo flags / CTA barrier.
// Start (pcg_init: x = 0, r = -grad, p = z) and end (the Armijo start of
// trial_init: g.q, max|q|, b_old = b, b = b + q) are fused in, as in the
// shared-memory resident kernel.
#pragma once

namespace hysco {

constexpr int L2P_THREADS = 512;   // 16 warps per SM, up to 128 registers (no spills)

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

template <typename T, int NCH, bool FIXED>
__global__ void __launch_bounds__(L2P_THREADS, 1)
    pcg_l2_kernel(Geom g, Ctl c, SolveParams sp, int pair, const T* __restrict__ grad, const T* __restrict__ dt,
                  const T* __restrict__ et, T* __restrict__ x, T* __restrict__ r, T* __restrict__ p,
                  T* __restrict__ Hp, T* __restrict__ bcur, T* __restrict__ bold, double* __restrict__ gpart,
                  unsigned* __restrict__ flags, int batch) {
    count_launch(c);
    if (!pcg_step_active(c.st[pair])) {      // uniform over the grid: no step (finished, or a search pending)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (!c.st[pair].gn_active) c.st[pair].ls_active = 0;
            if (pair == batch - 1)
                set_cond(c, COND_LS, any_pair(c, batch, [](volatile PairState* q2) { return q2->ls_active != 0; }));
        }
        return;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int P = g.P, n2 = g.n2;
    const long long c0 = (long long)blockIdx.x * g.ncol / gridDim.x;
    const long long c1 = (long long)(blockIdx.x + 1) * g.ncol / gridDim.x;
    const size_t po = (size_t)pair * g.ps;
    const long long sI = (long long)n2 * P;
    const T ahd = (T)g.ahd, ih1sq = (T)g.ih1sq, ih2sq = (T)g.ih2sq;
    const unsigned launch = *reinterpret_cast<volatile unsigned*>(flags + (size_t)gridDim.x * RES_FLAG_STRIDE);
    const int blo = res_owner(c0 - n2 > 0 ? c0 - n2 : 0, g.ncol, gridDim.x);
    const int bhi = res_owner(c1 - 1 + n2 < g.ncol ? c1 - 1 + n2 : g.ncol - 1, g.ncol, gridDim.x);
    double* part0 = gpart;
    double* part1 = gpart + RES_PART_DOUBLES;
    double* part2 = gpart + 2 * RES_PART_DOUBLES;

    // ---- start (pcg_init): x = 0, r = -grad, z = r/M, p = z; r.z, r.r
    double arz = 0, arr = 0;
    for (long long col = c0 + wid; col < c1; col += nw) {
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
    halo_release(flags, res_tag(launch, 0));   // p_0 published
    double v0[2] = {arz, arr}, t0[2];
    reduce_publish<2>(v0, part0, res_tag(launch, 0));
    reduce_collect<2>(part0, res_tag(launch, 0), t0);
    double rz = t0[0];
    const double rr0 = t0[1];
    double rr = rr0;
    int k_it = 0;
    if (rr0 > 0.0) {
        for (k_it = 0; k_it < sp.max_pcg;) {
            halo_acquire(flags, blo, bhi, res_tag(launch, k_it));   // neighbours' p_k
            // ---- A: Hp = dt p + et_{l-1} p_{l-1} + et_l p_{l+1} + alpha hd L_xy p; p.Hp
            double apq = 0;
            for (long long col = c0 + wid; col < c1; col += nw) {
                const ColInfo ci = col_info(g, col);
                const T* qc = p + po + ci.off;
                const T* dc = dt + po + ci.off;
                const T* ec = et + po + ci.off;
                T* hc = Hp + po + ci.off;
                for (int seg = 0; seg < P; seg += 32 * NCH) {
                    T qv[NCH], dv[NCH], ev[NCH], l1[NCH], l2[NCH];
#pragma unroll
                    for (int m = 0; m < NCH; m++) {
                        const int l = seg + 32 * m + lane;
                        const bool ok = l < P;
                        qv[m] = ok ? ldcg(qc + l) : T(0);
                        dv[m] = ok ? dc[l] : T(0);
                        ev[m] = ok ? ec[l] : T(0);
                        const T a = (ok && ci.him) ? ldcg(qc + l - sI) : T(0);
                        const T b = (ok && ci.hip) ? ldcg(qc + l + sI) : T(0);
                        const T e = (ok && ci.hjm) ? ldcg(qc + l - P) : T(0);
                        const T f = (ok && ci.hjp) ? ldcg(qc + l + P) : T(0);
                        l1[m] = (ci.him ? qv[m] - a : T(0)) + (ci.hip ? qv[m] - b : T(0));
                        l2[m] = (ci.hjm ? qv[m] - e : T(0)) + (ci.hjp ? qv[m] - f : T(0));
                    }
#pragma unroll
                    for (int m = 0; m < NCH; m++) {
                        const int l = seg + 32 * m + lane;
                        T qm = __shfl_up_sync(FULL, qv[m], 1), em = __shfl_up_sync(FULL, ev[m], 1);
                        T qp = __shfl_down_sync(FULL, qv[m], 1);
                        const T qprev = __shfl_sync(FULL, qv[m > 0 ? m - 1 : 0], 31);
                        const T eprev = __shfl_sync(FULL, ev[m > 0 ? m - 1 : 0], 31);
                        const T qnext = __shfl_sync(FULL, qv[m + 1 < NCH ? m + 1 : m], 0);
                        if (lane == 0) {
                            qm = m > 0 ? qprev : ((l > 0 && l - 1 < P) ? ldcg(qc + l - 1) : T(0));
                            em = m > 0 ? eprev : ((l > 0 && l - 1 < P) ? ec[l - 1] : T(0));
                        }
                        if (lane == 31) qp = m + 1 < NCH ? qnext : ((l + 1 < P) ? ldcg(qc + l + 1) : T(0));
                        if (l < P) {
                            T h = dv[m] * qv[m];
                            if (l > 0) h += em * qm;
                            if (l < g.n3) h += ev[m] * qp;
                            h += ahd * (l1[m] * ih1sq + l2[m] * ih2sq);
                            hc[l] = h;
                            apq += (double)qv[m] * (double)h;
                        }
                    }
                }
            }
            double v1[1] = {apq}, t1[1];
            reduce_publish<1>(v1, part1, res_tag(launch, k_it));
            reduce_collect<1>(part1, res_tag(launch, k_it), t1);
            if (t1[0] <= 0.0) break;                  // breakdown (oracle pcg(): keep x)
            const T a = (T)(rz / t1[0]);
            // ---- B: x += a p, r -= a Hp, z = r/M; r.z, r.r (own nodes, own writes)
            double brz = 0, brr = 0;
            for (long long col = c0 + wid; col < c1; col += nw) {
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
                        pv[m] = ok ? ldcg(p + o + l) : T(0);
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
                            brz += (double)rn * (double)z;
                            brr += (double)rn * (double)rn;
                        }
                    }
                }
            }
            double v3[2] = {brz, brr}, t3[2];
            reduce_publish<2>(v3, part2, res_tag(launch, k_it));
            reduce_collect<2>(part2, res_tag(launch, k_it), t3);
            k_it += 1;
            const double beta = t3[0] / rz;
            rz = t3[0];
            rr = t3[1];
            if (k_it >= sp.max_pcg || (!FIXED && sqrt(t3[1] / rr0) < sp.pcg_rtol)) break;
            // ---- C: p = z + beta p (own columns), then publish p_{k+1}
            const T be = (T)beta;
            for (long long col = c0 + wid; col < c1; col += nw) {
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
                        pv[m] = ok ? ldcg(p + o + l) : T(0);
                    }
#pragma unroll
                    for (int m = 0; m < NCH; m++) {
                        const int l = seg + 32 * m + lane;
                        if (l < P) p[o + l] = rv[m] / (dv[m] + cm) + be * pv[m];
                    }
                }
            }
            halo_release(flags, res_tag(launch, k_it));
        }
    }
    // ---- end (trial_init): q = x, g.q, max|q|, b_old = b, b = b + q
    double agq = 0, aqm = 0;
    for (long long col = c0 + wid; col < c1; col += nw) {
        const size_t o = po + (size_t)col * P;
        for (int seg = 0; seg < P; seg += 32 * NCH) {
            T qv[NCH], gv[NCH], bv[NCH];
#pragma unroll
            for (int m = 0; m < NCH; m++) {
                const int l = seg + 32 * m + lane;
                const bool ok = l < P;
                qv[m] = ok ? (k_it > 0 ? x[o + l] : T(0)) : T(0);
                gv[m] = ok ? grad[o + l] : T(0);
                bv[m] = ok ? bcur[o + l] : T(0);
            }
#pragma unroll
            for (int m = 0; m < NCH; m++) {
                const int l = seg + 32 * m + lane;
                if (l < P) {
                    agq += (double)gv[m] * (double)qv[m];
                    aqm = fmax(aqm, (double)fabs(qv[m]));
                    bold[o + l] = bv[m];
                    bcur[o + l] = bv[m] + qv[m];
                }
            }
        }
    }
    double v4[2] = {agq, aqm}, t4[2];
    reduce_publish<2, 0x2u>(v4, part0, res_tag(launch, 31));
    reduce_collect<2, 0x2u>(part0, res_tag(launch, 31), t4);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        decide_trial(c.st[pair], t4);
        if (pair == batch - 1)
            set_cond(c, COND_LS, any_pair(c, batch, [](volatile PairState* q2) { return q2->ls_active != 0; }));
        // every CTA read `launch` before its first publish, which CTA 0 has collected
        *reinterpret_cast<volatile unsigned*>(flags + (size_t)gridDim.x * RES_FLAG_STRIDE) = launch + 1;
        PairState& s = c.st[pair];
        s.rz = rz;
        s.rr0 = rr0;
        s.rr = rr;
        s.pcg_k = k_it;
        s.pcg_iters += k_it;
        s.h_evals += k_it;
        s.relres = rr0 > 0.0 ? sqrt(rr / rr0) : 0.0;
        s.pcg_active = 0;
    }
}

}  // namespace hysco
