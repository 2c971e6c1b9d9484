// hysco_resident.cuh — on-chip-resident Jacobi-PCG (A5 + A6 for a whole GN
// step in ONE persistent launch), fp32.
//
// Why: a PCG iteration of the streaming kernels moves ~60 B/node through HBM
// and needs three launches.  For a volume whose PCG state fits the chip
// (HCP 3T: 2.70 M nodes; per SM 127 columns x 145 nodes), each CTA keeps its
// contiguous range of PE columns resident for all iterations:
//   shared memory : p (read by neighbouring threads), dt, et   (12 B/node)
//   registers     : r and Hp, K slots per thread               ( 8 B/node)
//   global / L2   : x (read-modify-write, owner only) and a copy of p that
//                   neighbouring CTAs read for the in-plane Laplacian halo.
// One CTA per SM (cooperative launch guarantees co-residency); the three
// reductions of an iteration (p.Hp, r.z, r.r) use a grid barrier and a
// deterministic fixed-order sum of per-CTA partials that every CTA performs
// identically, so all CTAs take the same alpha/beta/stop decisions.
// Arithmetic per node is the streaming kernels' (same formulas and order).
#pragma once

#include <cooperative_groups.h>

namespace hysco {

constexpr int RES_THREADS = 768;

// Opaque copy: stops ptxas from hoisting per-slot index math (and everything
// derived from it) out of the PCG iteration loop, which would keep ~15
// values live per slot across all iterations.
__device__ __forceinline__ int opaque(int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
// x += v at L2 with no return value: the owner is the only writer of x, so
// the sum is the plain fp32 x + fl(a p) and no load latency is exposed.
__device__ __forceinline__ void red_add(float* p, float v) {
    asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// Grid-wide barrier: the launch is cooperative, so cooperative_groups' grid
// sync applies (measured 1.2 us per barrier on B200 with 148 CTAs vs 2.0 us for
// a hand-written counter/generation barrier; tools/barrier_bench.cu).
__device__ __forceinline__ void grid_barrier(unsigned*, unsigned*) { cooperative_groups::this_grid().sync(); }

// Block-reduce NV doubles, publish per-CTA partials, barrier, and fold all
// partials in fixed order (identically in every CTA).  Result in out[] (all threads).
// Optional phase trace (tools/res_trace.cu): thread 0 of every CTA stamps the
// global timer at phase boundaries of the first 16 iterations.
__device__ __forceinline__ void res_stamp(unsigned long long* tr) {
    if (tr && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        *tr = t;
    }
}

template <int NV>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], double* __restrict__ part, unsigned* bar, double (&out)[NV],
                                            unsigned long long* tr = nullptr) {
    __shared__ double sred[NV][32];
    __shared__ double stot[NV];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
        if (lane == 0) sred[k][wid] = x;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double x = 0;
        for (int w = 0; w < nw; w++) x += sred[threadIdx.x][w];
        part[blockIdx.x * NV + threadIdx.x] = x;
    }
    res_stamp(tr);                         // all warps of this CTA are done with the phase
    grid_barrier(bar, bar + 1);
    if (wid < NV) {                        // warp k folds value k (fixed order)
        double x = 0;
        for (int b = lane; b < (int)gridDim.x; b += 32) x += __ldcg(&part[b * NV + wid]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
        if (lane == 0) stot[wid] = x;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++) out[k] = stot[k];
}

// Split form of grid_reduce: publish this CTA's partials and arrive (returns
// the arrival token), do independent work, then reduce_finish waits and folds
// all partials in the same fixed order.
template <int NV>
__device__ __forceinline__ unsigned reduce_arrive(double (&v)[NV], double* __restrict__ part,
                                                  const cooperative_groups::grid_group& grid) {
    __shared__ double sred2[NV][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
        if (lane == 0) sred2[k][wid] = x;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double x = 0;
        for (int w = 0; w < nw; w++) x += sred2[threadIdx.x][w];
        part[blockIdx.x * NV + threadIdx.x] = x;
    }
    return grid.barrier_arrive();
}

template <int NV>
__device__ __forceinline__ void reduce_finish(unsigned tok, const double* __restrict__ part,
                                              const cooperative_groups::grid_group& grid, double (&out)[NV]) {
    __shared__ double stot2[NV];
    grid.barrier_wait(std::move(tok));
    const int wid = threadIdx.x >> 5;
    if (wid < NV) {                        // warp k folds value k (fixed order)
        const int lane = threadIdx.x & 31;
        double x = 0;
        for (int b = lane; b < (int)gridDim.x; b += 32) x += __ldcg(&part[b * NV + wid]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
        if (lane == 0) stot2[wid] = x;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++) out[k] = stot2[k];
}


// Resident-path preconditioner application: z = r * rcp.approx(M) (~1 ulp;
// M > 0 is only the Jacobi preconditioner).
__device__ __forceinline__ float precond(float r, float M) {
    float inv;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(M));
    return r * inv;
}

// q = n / d for 0 <= n < 2^31 with a precomputed multiplier (no IDIV in the loop).
struct FastDiv {
    unsigned m, s;
    __device__ __forceinline__ void init(unsigned d) {
        unsigned l = 0;
        while ((1u << l) < d) l++;
        const unsigned p = 31 + l;
        m = (unsigned)(((1ull << p) + d - 1) / d);
        s = p - 32;
    }
    __device__ __forceinline__ int div(int n) const { return (int)(__umulhi((unsigned)n, m) >> s); }
};

// Global copy of p used for the in-plane halo: per pair (n1 + 2) x n2 x P
// floats with zero ghost planes at i = -1 and i = n1, so an i-neighbour read
// needs no existence test (a missing Neumann neighbour contributes 0 to the
// off-diagonal sum; its diagonal share is already excluded from M).
__host__ __device__ inline size_t res_ghost_pair_floats(const Geom& g) { return (size_t)(g.n1 + 2) * g.n2 * g.P; }

template <int K, bool FIXED>
__global__ void __launch_bounds__(RES_THREADS, 1)
    pcg_resident_kernel(Geom g, Ctl c, SolveParams sp, int pair, const float* __restrict__ grad,
                        const float* __restrict__ dt, const float* __restrict__ et, float* __restrict__ x,
                        float* __restrict__ pgh, double* __restrict__ gpart, unsigned* bar, int nbmax,
                        unsigned long long* trace = nullptr) {
    count_launch(c);
    if (!c.st[pair].gn_active) return;       // uniform over the grid
    unsigned long long* trk = trace ? trace + ((size_t)blockIdx.x * 16 + 15) * 8 : nullptr;   // launch-level stamps
    res_stamp(trk);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int NT = blockDim.x;
    const int KNT = K * NT;
    const int P = g.P, n2 = g.n2;
    (void)nbmax;
    // shared layout (floats): [guard][j-halo: P][own + padding: KNT][next-column halo: P][guard]
    //                         [M: KNT][guard][et: KNT][guard]
    // Slots n >= Nb are padding (M = 1, et = 0, r = 0, Hp forced to 0), so the
    // slot loops need no bounds branch; et at l = n3 is 0, so p_{l-1}/p_{l+1}
    // across a column boundary contribute nothing and need no PE test.
    float* sp_ = reinterpret_cast<float*>(smem_raw) + 1 + P;
    float* sM = sp_ + KNT + P + 1;
    float* se = sM + KNT + 1;

    const long long c0 = (long long)blockIdx.x * g.ncol / gridDim.x;
    const long long c1 = (long long)(blockIdx.x + 1) * g.ncol / gridDim.x;
    const int ncl = (int)(c1 - c0);
    const int Nb = ncl * P;
    const size_t n0 = (size_t)pair * g.ps + (size_t)c0 * P;
    const int sI = n2 * P;
    const float wi = (float)(g.ahd * g.ih1sq), wj = (float)(g.ahd * g.ih2sq);
    // this CTA's first node in the ghost-padded global copy of p
    float* __restrict__ pgc = pgh + (size_t)pair * res_ghost_pair_floats(g) + (size_t)(c0 + n2) * P;
    float* __restrict__ xl = x + n0;
    double* part2 = gpart;                 // [G][2] for r.z, r.r
    double* part1 = gpart + 2 * gridDim.x; // [G][1] for p.Hp
    FastDiv fdP, fdN2;
    fdP.init((unsigned)P);
    fdN2.init((unsigned)n2);
    bool xset = false;                     // x holds alpha_0 p_0 + ... (else still to be zeroed)

    if (threadIdx.x == 0) {
        sp_[-P - 1] = 0.f;
        se[-1] = 0.f;
        se[KNT] = 0.f;
    }
    // per-slot masks (bit k = slot k): node valid, j-1 neighbour exists, j+1 neighbour exists
    unsigned mval = 0, mjm = 0, mjp = 0;
    float r[K], hv[K];
    float frz = 0.f, frr = 0.f;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int n = threadIdx.x + k * NT;
        float rv = 0.f, M = 1.f, e = 0.f;
        if (n < Nb) {
            const int col = (int)c0 + fdP.div(n);
            const int i = fdN2.div(col), j = col - i * n2;
            M = dt[n0 + n] + (float)(g.ahd * diag_lxy(g, i, j));
            e = et[n0 + n];
            rv = -grad[n0 + n];
            mval |= 1u << k;
            if (j > 0) mjm |= 1u << k;
            if (j < n2 - 1) mjp |= 1u << k;
        }
        const float z = precond(rv, M);
        sM[n] = M;
        se[n] = e;
        sp_[n] = z;
        r[k] = rv;
        hv[k] = 0.f;
        if (n < Nb) pgc[n] = z;               // x = 0 is written by the first update (or below)
        frz = fmaf(rv, z, frz);
        frr = fmaf(rv, rv, frr);
    }
    double v2[2] = {(double)frz, (double)frr}, t2[2];
    res_stamp(trk ? trk + 1 : nullptr);
    grid_reduce<2>(v2, part2, bar, t2);       // also publishes p0 to the neighbours
    res_stamp(trk ? trk + 2 : nullptr);
    double rz = t2[0];
    const double rr0 = t2[1];
    double relres = rr0 > 0 ? 1.0 : 0.0;
    int k_it = 0, hev = 0;
    if (rr0 > 0.0) {
        cooperative_groups::grid_group grid = cooperative_groups::this_grid();
        unsigned tok3 = 0;                    // pending split barrier "new p published"
        bool pend3 = false;
        for (k_it = 0; k_it < sp.max_pcg;) {
            unsigned long long* tr = (trace && k_it < 16) ? trace + ((size_t)blockIdx.x * 16 + k_it) * 8 : nullptr;
            res_stamp(tr);
            if (pend3) grid.barrier_wait(std::move(tok3));
            // j-halo columns (c0-1 and c1) from the global copy; zeros off the ends
            for (int t = threadIdx.x; t < 2 * P; t += NT) {
                const bool nxt = t >= P;
                const int l = nxt ? t - P : t;
                const long long col = nxt ? c1 : c0 - 1;
                float v = 0.f;
                if (col >= 0 && col < g.ncol) v = __ldcg(pgc + (nxt ? Nb : -P) + l);
                sp_[(nxt ? Nb : -P) + l] = v;
            }
            __syncthreads();
            res_stamp(tr ? tr + 1 : nullptr);
            // ---- Hp = M p + et_{l-1} p_{l-1} + et_l p_{l+1} - alpha hd sum_inplane p_nb / h^2
            float fpq = 0.f;
            {
                const int tid = opaque(threadIdx.x);
                const unsigned mv = (unsigned)opaque((int)mval), mm = (unsigned)opaque((int)mjm),
                               mp = (unsigned)opaque((int)mjp);
                const float* gm = pgc + tid - sI;   // i-1 neighbours (ghost plane at i = -1)
                const float* gp = pgc + tid + sI;   // i+1 neighbours (ghost plane at i = n1)
                const float* s0 = sp_ + tid;
                const float* m0 = sM + tid;
                const float* e0 = se + tid;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int o = k * NT;
                    const float pv = s0[o];
                    float h = m0[o] * pv;
                    h = fmaf(e0[o - 1], s0[o - 1], h);
                    h = fmaf(e0[o], s0[o + 1], h);
                    const float si = __ldcg(gm + o) + __ldcg(gp + o);
                    float sj = 0.f;
                    if (mm & (1u << k)) sj = s0[o - P];
                    if (mp & (1u << k)) sj += s0[o + P];
                    h = fmaf(-wi, si, fmaf(-wj, sj, h));
                    h = (mv & (1u << k)) ? h : 0.f;
                    hv[k] = h;
                    fpq = fmaf(pv, h, fpq);
                }
            }
            double v1[1] = {(double)fpq}, t1[1];
            grid_reduce<1>(v1, part1, bar, t1, tr ? tr + 2 : nullptr);
            res_stamp(tr ? tr + 3 : nullptr);
            if (t1[0] <= 0.0) break;                  // breakdown (oracle pcg(): keep x)
            hev += 1;
            const float a = (float)(rz / t1[0]);
            // ---- r -= a Hp, z = r/M (kept in the dead Hp registers); r.z, r.r
            float frz2 = 0.f, frr2 = 0.f;
            {
                const int tid = opaque(threadIdx.x);
                const float* m0 = sM + tid;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const float rn = fmaf(-a, hv[k], r[k]);
                    r[k] = rn;
                    const float z = precond(rn, m0[k * NT]);
                    hv[k] = z;
                    frz2 = fmaf(rn, z, frz2);
                    frr2 = fmaf(rn, rn, frr2);
                }
            }
            double v3[2] = {(double)frz2, (double)frr2}, t3[2];
            const unsigned tok2 = reduce_arrive<2>(v3, part2, grid);
            res_stamp(tr ? tr + 4 : nullptr);
            // ---- x += a p while the r.z / r.r partials gather (fire-and-forget L2
            // adds; x feeds no reduction)
            {
                const int tid = opaque(threadIdx.x);
                const unsigned mv = (unsigned)opaque((int)mval);
                float* xt = xl + tid;
                const float* s0 = sp_ + tid;
                if (xset) {
#pragma unroll
                    for (int k = 0; k < K; k++)
                        if (mv & (1u << k)) red_add(xt + k * NT, a * s0[k * NT]);
                } else {                      // first update: x_1 = 0 + a p_0 (plain stores)
#pragma unroll
                    for (int k = 0; k < K; k++)
                        if (mv & (1u << k)) xt[k * NT] = 0.f + a * s0[k * NT];
                }
            }
            xset = true;
            reduce_finish<2>(tok2, part2, grid, t3);
            res_stamp(tr ? tr + 5 : nullptr);
            k_it += 1;
            relres = sqrt(t3[1] / rr0);
            const double beta = t3[0] / rz;
            rz = t3[0];
            if (k_it >= sp.max_pcg || (!sp.fixed && relres < sp.pcg_rtol)) break;
            // ---- p = z + beta p on own columns and on the global halo copy
            const float be = (float)beta;
            {
                const int tid = opaque(threadIdx.x);
                const unsigned mv = (unsigned)opaque((int)mval);
                float* s0 = sp_ + tid;
                float* gt = pgc + tid;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int o = k * NT;
                    const float pn = fmaf(be, s0[o], hv[k]);
                    s0[o] = pn;
                    if (mv & (1u << k)) gt[o] = pn;
                }
            }
            res_stamp(tr ? tr + 6 : nullptr);
            tok3 = grid.barrier_arrive();
            pend3 = true;
        }
    }
    if (!xset)                                // no update happened (r0 = 0 or breakdown): x = 0
        for (int n = threadIdx.x; n < Nb; n += NT) xl[n] = 0.f;
    res_stamp(trk ? trk + 3 : nullptr);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        PairState& s = c.st[pair];
        s.rz = rz;
        s.rr0 = rr0;
        s.pcg_k = k_it;
        s.pcg_iters += k_it;
        s.h_evals += hev;
        s.relres = relres;
        s.pcg_active = 0;
    }
}

}  // namespace hysco
