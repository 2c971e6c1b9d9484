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

namespace hysco {

constexpr int RES_THREADS = 768;

// Compiler-only memory fence between the unrolled node slots: keeps ptxas from
// hoisting every slot's loads to the top (which blows the 80-register budget
// of a 768-thread CTA and spills into an L1 that shared memory has consumed).
__device__ __forceinline__ void slot_fence() { asm volatile("" ::: "memory"); }

// Opaque copy: stops ptxas from hoisting per-slot index math (and everything
// derived from it) out of the PCG iteration loop, which would keep ~15
// values live per slot across all iterations.
__device__ __forceinline__ int opaque(int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

// Sense-free generation barrier over all CTAs of the launch (all co-resident).
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = gen;
        const unsigned g0 = *vgen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vgen == g0) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Block-reduce NV doubles, publish per-CTA partials, barrier, and fold all
// partials in fixed order (identically in every CTA).  Result in out[] (all threads).
template <int NV>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], double* __restrict__ part, unsigned* bar, double (&out)[NV]) {
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
    grid_barrier(bar, bar + 1);
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < NV; k++) {
            double x = 0;
            for (int b = lane; b < (int)gridDim.x; b += 32) x += __ldcg(&part[b * NV + k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
            if (lane == 0) stot[k] = x;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++) out[k] = stot[k];
}

// Per-column flags of the CTA's columns: bits 0-3 = in-plane neighbour exists
// (i-1, i+1, j-1, j+1; Neumann, R3), bits 4-7 = that neighbour column is in
// this CTA's shared memory (else read from the global copy of p).
enum { NB_IM = 1, NB_IP = 2, NB_JM = 4, NB_JP = 8, LOC_SHIFT = 4 };

// Resident-path preconditioner application: z = r / M with the fast
// reciprocal (<= 2 ulp; M is only a preconditioner).
__device__ __forceinline__ float precond(float r, float M) { return __fdividef(r, M); }

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

template <int K, bool FIXED>
__global__ void __launch_bounds__(RES_THREADS, 1)
    pcg_resident_kernel(Geom g, Ctl c, SolveParams sp, int pair, const float* __restrict__ grad,
                        const float* __restrict__ dt, const float* __restrict__ et, float* __restrict__ x,
                        float* __restrict__ pg, double* __restrict__ gpart, unsigned* bar, int nbmax) {
    count_launch(c);
    if (!c.st[pair].gn_active) return;       // uniform over the grid
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // Each array holds K*NT slots (+1 guard each side): nodes n >= Nb are padding
    // (p = 0, M = 1, et = 0, column flags 0), so no slot needs a bounds branch.
    // et at l = n3 is 0 (stored by eval), so p_{l+1} / p_{l-1} across a column
    // boundary contribute nothing and need no PE-boundary test either.
    const int NT = blockDim.x;
    const int KNT = K * NT;
    float* sp_ = reinterpret_cast<float*>(smem_raw) + 1;   // p
    float* sM = sp_ + KNT + 1;                             // M = diag(H) (Jacobi, R13)
    float* se = sM + KNT + 1;                              // et (PE super-diagonal)
    int* scol = reinterpret_cast<int*>(se + KNT + 1);      // per-column neighbour flags
    (void)nbmax;

    const int P = g.P, n2 = g.n2;
    const long long c0 = (long long)blockIdx.x * g.ncol / gridDim.x;
    const long long c1 = (long long)(blockIdx.x + 1) * g.ncol / gridDim.x;
    const int ncl = (int)(c1 - c0);
    const int Nb = ncl * P;
    const int nq = (KNT + P - 1) / P;                      // columns incl. padding
    const size_t n0 = (size_t)pair * g.Nn + (size_t)c0 * P;
    const int sI = n2 * P;
    const float wi = (float)(g.ahd * g.ih1sq), wj = (float)(g.ahd * g.ih2sq);
    const float* __restrict__ pgl = pg + n0;            // this CTA's columns in the global copy of p
    float* __restrict__ pgw = pg + n0;
    float* __restrict__ xl = x + n0;
    double* part2 = gpart;                 // [G][2] for r.z, r.r
    double* part5 = gpart + 2 * gridDim.x; // [G][1] for p.Hp
    FastDiv fdP;
    fdP.init((unsigned)P);

    if (threadIdx.x == 0) {
        sp_[-1] = 0.f;
        sp_[KNT] = 0.f;
        se[-1] = 0.f;
        se[KNT] = 0.f;
    }
    for (int q = threadIdx.x; q < nq; q += NT) {
        int f = 0;
        if (q < ncl) {
            const long long col = c0 + q;
            const int i = (int)(col / n2), j = (int)(col - (long long)i * n2);
            f = (i > 0 ? NB_IM : 0) | (i < g.n1 - 1 ? NB_IP : 0) | (j > 0 ? NB_JM : 0) | (j < n2 - 1 ? NB_JP : 0);
            f |= ((q - n2 >= 0) ? NB_IM : 0) << LOC_SHIFT;
            f |= ((q + n2 < ncl) ? NB_IP : 0) << LOC_SHIFT;
            f |= ((q - 1 >= 0) ? NB_JM : 0) << LOC_SHIFT;
            f |= ((q + 1 < ncl) ? NB_JP : 0) << LOC_SHIFT;
        }
        scol[q] = f;
    }
    __syncthreads();

    // prologue: M, et to shared memory; x = 0, r = -grad, p = z = r/M (R14)
    float r[K], hv[K];
    float frz = 0.f, frr = 0.f;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int n = threadIdx.x + k * NT;
        float rv = 0.f, M = 1.f, e = 0.f;
        if (n < Nb) {
            const int q = fdP.div(n);
            const long long col = c0 + q;
            const int i = (int)(col / n2), j = (int)(col - (long long)i * n2);
            M = dt[n0 + n] + (float)(g.ahd * diag_lxy(g, i, j));
            e = et[n0 + n];
            rv = -grad[n0 + n];
        }
        const float z = precond(rv, M);
        sM[n] = M;
        se[n] = e;
        sp_[n] = z;
        r[k] = rv;
        hv[k] = 0.f;
        if (n < Nb) {
            pgw[n] = z;
            xl[n] = 0.f;
        }
        frz = fmaf(rv, z, frz);
        frr = fmaf(rv, rv, frr);
    }
    double v2[2] = {(double)frz, (double)frr}, t2[2];
    grid_reduce<2>(v2, part2, bar, t2);
    double rz = t2[0];
    const double rr0 = t2[1];
    double relres = rr0 > 0 ? 1.0 : 0.0;
    int k_it = 0, hev = 0;
    volatile const float* vM = sM;
    volatile const float* ve = se;
    volatile const int* vcol = scol;
    // Three grid reductions per iteration (p.Hp; r.z and r.r; the halo barrier
    // after the new p), exactly the streaming kernels' Hestenes-Stiefel order.
    // (A single-reduction variant that expands r'.z' algebraically cancels
    // badly once the residual drops fast and was rejected.)
    if (rr0 > 0.0) {
        for (k_it = 0; k_it < sp.max_pcg;) {
            // ---- Hp = M p + et_{l-1} p_{l-1} + et_l p_{l+1} - alpha hd sum_inplane p_nb / h^2
            float fpq = 0.f;
            {
                const int tid = opaque(threadIdx.x);
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int n = tid + k * NT;
                    const int f = vcol[fdP.div(n)];
                    const float pv = sp_[n];
                    float h = vM[n] * pv;
                    h = fmaf(ve[n - 1], sp_[n - 1], h);
                    h = fmaf(ve[n], sp_[n + 1], h);
                    const int mim = n - sI, mip = n + sI, mjm = n - P, mjp = n + P;
                    const float lim = sp_[(f & (NB_IM << LOC_SHIFT)) ? mim : n];
                    const float lip = sp_[(f & (NB_IP << LOC_SHIFT)) ? mip : n];
                    const float ljm = sp_[(f & (NB_JM << LOC_SHIFT)) ? mjm : n];
                    const float ljp = sp_[(f & (NB_JP << LOC_SHIFT)) ? mjp : n];
                    const bool gim = (f & NB_IM) && !(f & (NB_IM << LOC_SHIFT));
                    const bool gip = (f & NB_IP) && !(f & (NB_IP << LOC_SHIFT));
                    const bool gjm = (f & NB_JM) && !(f & (NB_JM << LOC_SHIFT));
                    const bool gjp = (f & NB_JP) && !(f & (NB_JP << LOC_SHIFT));
                    const float xim = gim ? __ldcg(pgl + mim) : lim;
                    const float xip = gip ? __ldcg(pgl + mip) : lip;
                    const float xjm = gjm ? __ldcg(pgl + mjm) : ljm;
                    const float xjp = gjp ? __ldcg(pgl + mjp) : ljp;
                    const float si = ((f & NB_IM) ? xim : 0.f) + ((f & NB_IP) ? xip : 0.f);
                    const float sj = ((f & NB_JM) ? xjm : 0.f) + ((f & NB_JP) ? xjp : 0.f);
                    h = fmaf(-wi, si, fmaf(-wj, sj, h));
                    hv[k] = h;
                    fpq = fmaf(pv, h, fpq);
                }
            }
            double v1[1] = {(double)fpq}, t1[1];
            grid_reduce<1>(v1, part5, bar, t1);
            if (t1[0] <= 0.0) break;                  // breakdown (oracle pcg(): keep x)
            hev += 1;
            const float a = (float)(rz / t1[0]);
            // ---- x += a p, r -= a Hp, z = r/M; r.z, r.r
            float frz2 = 0.f, frr2 = 0.f;
            {
                const int tid = opaque(threadIdx.x);
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int n = tid + k * NT;
                    if (n < Nb) xl[n] = fmaf(a, sp_[n], xl[n]);
                    const float rn = fmaf(-a, hv[k], r[k]);
                    r[k] = rn;
                    const float z = precond(rn, vM[n]);
                    frz2 = fmaf(rn, z, frz2);
                    frr2 = fmaf(rn, rn, frr2);
                }
            }
            double v3[2] = {(double)frz2, (double)frr2}, t3[2];
            grid_reduce<2>(v3, part2, bar, t3);
            k_it += 1;
            relres = sqrt(t3[1] / rr0);
            const double beta = t3[0] / rz;
            rz = t3[0];
            if (k_it >= sp.max_pcg || (!sp.fixed && relres < sp.pcg_rtol)) break;
            // ---- p = z + beta p (own columns; the global copy feeds the neighbours' halo)
            const float be = (float)beta;
            {
                const int tid = opaque(threadIdx.x);
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int n = tid + k * NT;
                    const float pn = fmaf(be, sp_[n], precond(r[k], vM[n]));
                    sp_[n] = pn;
                    if (n < Nb) pgw[n] = pn;
                }
            }
            grid_barrier(bar, bar + 1);
        }
    }
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
