// hysco_lsq.cuh -- push-forward simulation and least-squares correction
// (readings R27-R29 in DESIGN.md).
//
// One warp per PE column.  The push-forward matrix A of a column (R27) is
// never formed: the map u_k = k + s (A b)_k / h3 of true cell k is kept as
// (j0_k = floor(u_k), w_k = u_k - j0_k), A[j,k] = max(0, 1 - |u_k - j|), and
//   (A t)_j   = sum_{k : j0_k = j} (1 - w_k) t_k + sum_{k : j0_k = j-1} w_k t_k
//   (A^T y)_k = (1 - w_k) y_{j0_k} + w_k y_{j0_k+1}        (y outside [0,n3) = 0)
// For a feasible b (|Db| < 1) u is strictly increasing, so the k feeding
// distorted cell j form one contiguous range [F(j-1), F(j+1)), F(m) = first k
// with j0_k >= m (a binary search per m): A t is a deterministic gather, no
// atomics.  A column whose j0 is not monotone (|Db| >= 1, or rounding at
// |Db| ~ 1) is counted infeasible.
//
// Least squares (R28): Jacobi-PCG per column on the normal equations
//   (A+^T A+ + A-^T A- + lambda L1) t = A+^T i+ + A-^T i-,
// L1 the 1-D Neumann Laplacian in index units, from t = 0, until
// ||r|| <= rtol ||rhs|| or max_iter; scalars in fp64.
#pragma once

namespace hysco {

constexpr int LSQ_WARPS = 4;

// Per-warp shared-memory layout: 2 maps (j0 int, F int, w T) + T work arrays.
__host__ __device__ inline int lsq_ts(int n3) { return (n3 + 2) & ~1; }      // T array stride
__host__ __device__ inline int lsq_is(int n3) { return (n3 + 4) & ~1; }      // int array stride (F has n3 + 3)
template <typename T>
__host__ __device__ inline size_t lsq_warp_bytes(int n3, int nT) {
    return (size_t)4 * lsq_is(n3) * sizeof(int) + (size_t)nT * lsq_ts(n3) * sizeof(T);
}

template <typename T>
struct LsqMap {
    int* j0;     // [n3]
    int* F;      // [n3 + 3]: F[m + 1] = first k with j0_k >= m, m = -1 .. n3 + 1
    T* w;        // [n3]
};

// Build the column map of sign s from b (shared, P nodes); returns true if
// the map is monotone and every |Db| < 1 (warp-uniform).
template <typename T>
__device__ bool lsq_build_map(int lane, int n3, const T* __restrict__ sb, T s, T ih3, LsqMap<T> m) {
    bool ok = true;
    for (int k = lane; k < n3; k += 32) {
        const T db = (sb[k + 1] - sb[k]) * ih3;
        ok &= fabs(db) < T(1);
        // u = k + d split as j0 = k + floor(d), w = d - floor(d): w keeps the
        // precision of the displacement d, not of u ~ n3
        const T d = s * T(0.5) * (sb[k] + sb[k + 1]) * ih3;
        const T fd = floor(d);
        const T jf = T(k) + fd;
        int j0 = (int)fmin(fmax(jf, T(-2)), T(n3));
        T w = d - fd;
        if (jf < T(-2) || jf >= T(n3)) w = T(0);    // no entry lands in [0, n3)
        m.j0[k] = j0;
        m.w[k] = w;
    }
    __syncwarp();
    for (int k = lane; k + 1 < n3; k += 32) ok &= m.j0[k] <= m.j0[k + 1];
    for (int q = lane; q < n3 + 3; q += 32) {       // lower_bound of q - 1 in j0
        const int target = q - 1;
        int lo = 0, hi = n3;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (m.j0[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        m.F[q] = lo;
    }
    __syncwarp();
    return __all_sync(FULL, ok);
}

// y = A t (distorted cells) for one map; t, y shared.
template <typename T>
__device__ __forceinline__ void lsq_apply_A(int lane, int n3, const LsqMap<T>& m, const T* __restrict__ t,
                                            T* __restrict__ y) {
    for (int j = lane; j < n3; j += 32) {
        const int k0 = m.F[j], k1 = m.F[j + 2];     // F(j - 1), F(j + 1)
        T acc = T(0);
        for (int k = k0; k < k1; k++) {
            const T wk = m.w[k];
            acc += (m.j0[k] == j ? T(1) - wk : wk) * t[k];
        }
        y[j] = acc;
    }
}

// (A^T y)_k for one map (y shared, zero outside [0, n3)).
template <typename T>
__device__ __forceinline__ T lsq_apply_AT(int k, int n3, const LsqMap<T>& m, const T* __restrict__ y) {
    const int j = m.j0[k];
    const T wk = m.w[k];
    const T a = (j >= 0 && j < n3) ? y[j] : T(0);
    const T c = (j + 1 >= 0 && j + 1 < n3) ? y[j + 1] : T(0);
    return (T(1) - wk) * a + wk * c;
}

template <typename T>
__device__ __forceinline__ T lsq_diag_AT_A(int k, int n3, const LsqMap<T>& m) {
    const int j = m.j0[k];
    const T wk = m.w[k];
    return ((j >= 0 && j < n3) ? (T(1) - wk) * (T(1) - wk) : T(0)) + ((j + 1 >= 0 && j + 1 < n3) ? wk * wk : T(0));
}

template <typename T>
__device__ __forceinline__ void lsq_carve(unsigned char* base, int n3, LsqMap<T>& mp, LsqMap<T>& mm, T*& tarr) {
    int* ib = reinterpret_cast<int*>(base);
    const int is = lsq_is(n3);
    mp.j0 = ib;
    mp.F = ib + is;
    mm.j0 = ib + 2 * is;
    mm.F = ib + 3 * is;
    tarr = reinterpret_cast<T*>(ib + 4 * is);
    mp.w = tarr;
    mm.w = tarr + lsq_ts(n3);
}

// Stats slots in c.red[pair * RED_W + ...] (memset before the launch).
enum { LSQ_ST_ITERS = 0, LSQ_ST_UNCONV = 1, LSQ_ST_RELRES = 2, LSQ_ST_INFEAS = 3 };

__device__ __forceinline__ void atomic_max_nonneg(double* a, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(a), (unsigned long long)__double_as_longlong(v));
}

// I+ = A+ t, I- = A- t per column (P:331 distortion simulation).
template <typename T>
__global__ void __launch_bounds__(32 * LSQ_WARPS) push_forward_kernel(Geom g, Ctl c, const T* __restrict__ b,
                                                                      const T* __restrict__ Tt, T* __restrict__ Ip,
                                                                      T* __restrict__ Im) {
    count_launch(c);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int pair = blockIdx.y, n3 = g.n3, P = g.P;
    LsqMap<T> mp, mm;
    T* ta;
    lsq_carve<T>(smem_raw + (size_t)wid * lsq_warp_bytes<T>(n3, 6), n3, mp, mm, ta);
    const int ts = lsq_ts(n3);
    T* sb = ta + 2 * ts;
    T* st = ta + 3 * ts;
    T* yp = ta + 4 * ts;
    T* ym = ta + 5 * ts;
    const T ih3 = gw<T>(g.ih3, g.f_ih3);
    for (long long col = (long long)blockIdx.x * LSQ_WARPS + wid; col < g.ncol;
         col += (long long)gridDim.x * LSQ_WARPS) {
        const size_t oc = (size_t)pair * g.Nc + (size_t)col * n3, on = (size_t)pair * g.Nn + (size_t)col * P;
        for (int l = lane; l < P; l += 32) sb[l] = b[on + l];
        for (int k = lane; k < n3; k += 32) st[k] = Tt[oc + k];
        __syncwarp();
        const bool okp = lsq_build_map<T>(lane, n3, sb, T(1), ih3, mp);
        const bool okm = lsq_build_map<T>(lane, n3, sb, T(-1), ih3, mm);
        if (!(okp && okm) && lane == 0) atomicAdd(&c.red[(size_t)pair * RED_W + LSQ_ST_INFEAS], 1.0);
        lsq_apply_A<T>(lane, n3, mp, st, yp);
        lsq_apply_A<T>(lane, n3, mm, st, ym);
        __syncwarp();
        for (int k = lane; k < n3; k += 32) {
            Ip[oc + k] = yp[k];
            Im[oc + k] = ym[k];
        }
        __syncwarp();
    }
}

// Least-squares correction (R28): t per column by Jacobi-PCG.
template <typename T>
__global__ void __launch_bounds__(32 * LSQ_WARPS) lsq_kernel(Geom g, Ctl c, const T* __restrict__ b,
                                                             const T* __restrict__ Ip, const T* __restrict__ Im,
                                                             T* __restrict__ Tout, double lam_d, int max_iter,
                                                             double rtol) {
    count_launch(c);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int pair = blockIdx.y, n3 = g.n3, P = g.P;
    LsqMap<T> mp, mm;
    T* ta;
    lsq_carve<T>(smem_raw + (size_t)wid * lsq_warp_bytes<T>(n3, 9), n3, mp, mm, ta);
    const int ts = lsq_ts(n3);
    T* sb = ta + 2 * ts;     // b column, then the Jacobi inverse diagonal
    T* sx = ta + 3 * ts;
    T* sr = ta + 4 * ts;
    T* sp = ta + 5 * ts;
    T* sq = ta + 6 * ts;
    T* yp = ta + 7 * ts;
    T* ym = ta + 8 * ts;
    T* minv = sb;
    const T ih3 = gw<T>(g.ih3, g.f_ih3);
    const T lam = (T)lam_d;
    double* st = c.red + (size_t)pair * RED_W;
    for (long long col = (long long)blockIdx.x * LSQ_WARPS + wid; col < g.ncol;
         col += (long long)gridDim.x * LSQ_WARPS) {
        const size_t oc = (size_t)pair * g.Nc + (size_t)col * n3, on = (size_t)pair * g.Nn + (size_t)col * P;
        for (int l = lane; l < P; l += 32) sb[l] = b[on + l];
        for (int k = lane; k < n3; k += 32) {
            yp[k] = Ip[oc + k];
            ym[k] = Im[oc + k];
        }
        __syncwarp();
        const bool okp = lsq_build_map<T>(lane, n3, sb, T(1), ih3, mp);
        const bool okm = lsq_build_map<T>(lane, n3, sb, T(-1), ih3, mm);
        if (!(okp && okm)) {
            if (lane == 0) atomicAdd(&st[LSQ_ST_INFEAS], 1.0);
            for (int k = lane; k < n3; k += 32) Tout[oc + k] = T(0);
            __syncwarp();
            continue;
        }
        // rhs = A+^T i+ + A-^T i-; M^-1; x = 0, r = rhs, p = z = M^-1 r
        double rr = 0, rz = 0;
        for (int k = lane; k < n3; k += 32) {
            const T rk = lsq_apply_AT<T>(k, n3, mp, yp) + lsq_apply_AT<T>(k, n3, mm, ym);
            const T dk = lsq_diag_AT_A<T>(k, n3, mp) + lsq_diag_AT_A<T>(k, n3, mm) +
                         lam * T((k > 0) + (k < n3 - 1));
            const T mi = dk > T(0) ? T(1) / dk : T(0);
            minv[k] = mi;
            sx[k] = T(0);
            sr[k] = rk;
            sp[k] = mi * rk;
            rr += (double)rk * (double)rk;
            rz += (double)rk * (double)(mi * rk);
        }
        rr = warp_sum_t(rr);
        rz = warp_sum_t(rz);
        const double rr0 = rr, stop = rtol * rtol * rr0;
        int it = 0;
        while (it < max_iter && rr > stop) {
            __syncwarp();
            // q = (A+^T A+ + A-^T A- + lam L1) p
            lsq_apply_A<T>(lane, n3, mp, sp, yp);
            lsq_apply_A<T>(lane, n3, mm, sp, ym);
            __syncwarp();
            double pq = 0;
            for (int k = lane; k < n3; k += 32) {
                const T pk = sp[k];
                T lp = T(0);
                if (k > 0) lp += pk - sp[k - 1];
                if (k < n3 - 1) lp += pk - sp[k + 1];
                const T qk = lsq_apply_AT<T>(k, n3, mp, yp) + lsq_apply_AT<T>(k, n3, mm, ym) + lam * lp;
                sq[k] = qk;
                pq += (double)pk * (double)qk;
            }
            pq = warp_sum_t(pq);
            if (!(pq > 0)) break;                       // p in the null space (lambda = 0 corner)
            const double alpha = rz / pq;
            double rr1 = 0, rz1 = 0;
            for (int k = lane; k < n3; k += 32) {
                sx[k] += (T)alpha * sp[k];
                const T rk = sr[k] - (T)alpha * sq[k];
                sr[k] = rk;
                const T zk = minv[k] * rk;
                rr1 += (double)rk * (double)rk;
                rz1 += (double)rk * (double)zk;
            }
            rr1 = warp_sum_t(rr1);
            rz1 = warp_sum_t(rz1);
            const T beta = (T)(rz1 / rz);
            for (int k = lane; k < n3; k += 32) sp[k] = minv[k] * sr[k] + beta * sp[k];
            rr = rr1;
            rz = rz1;
            it++;
        }
        for (int k = lane; k < n3; k += 32) Tout[oc + k] = sx[k];
        if (lane == 0) {
            atomic_max_nonneg(&st[LSQ_ST_ITERS], (double)it);
            const double rel = rr0 > 0 ? sqrt(rr / rr0) : 0.0;
            atomic_max_nonneg(&st[LSQ_ST_RELRES], rel);
            if (rr > stop) atomicAdd(&st[LSQ_ST_UNCONV], 1.0);
        }
        __syncwarp();
    }
}

}  // namespace hysco
