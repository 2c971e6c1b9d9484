// hysco_admm.cuh — ADMM field-map solve (
// readings R21-R26 in DESIGN.md), sm_100a.
//
//   b <- argmin F(b) + rho hd/2 ||b - z + u||^2,  F = D + alpha S3 + beta P
//        (column-separable: one warp per PE column runs `inner` Gauss-Newton
//        steps, each an exact tridiagonal (Thomas) solve and its own Armijo
//        search on the column objective -- no grid-wide communication)
//   z <- (alpha hd L_xy^per + rho hd I)^{-1} rho hd (b + u)
//        (periodic in-plane operator, diagonalised by 2-D FFTs over (n1, n2)
//        for every PE node slice: cuFFT R2C / C2R, batch = P, stride = P)
//   u <- u + b - z;  residual norms per pair -> rho balancing on the host.
#pragma once

namespace hysco {

constexpr int ADMM_WARPS = 4;   // columns per CTA (one warp each)
#ifndef ADMM_MINB
#define ADMM_MINB 5   // fp32 admm_b_kernel: >= 5 CTAs per SM (<= 102 registers; measured 73.7 vs 68 pairs/s at 1)
#endif

// Per-warp shared scratch (elements): I+, I- padded by two zeros per side,
// b, v = z - u, q, grad, diag, offdiag, trial b (nodes), and the cell
// quantities a, c, r, phi', phi''.
__host__ __device__ inline size_t admm_warp_elems(int n3) {
    const size_t P = (size_t)n3 + 1;
    return 2 * ((size_t)n3 + 4) + 7 * P + 5 * P;   // cell arrays sized P: PCR reuses them
}

// Solve the column system tridiag(e, d, e) q = rhs by parallel cyclic
// reduction across the warp (ceil(log2 P) steps; equation i keeps
// a_i x_{i-s} + b_i x_i + c_i x_{i+s} = r_i).  The PCR buffers alias the cell
// arrays (dead after the derivative pass).  Replaces the oracle's sequential
// Thomas recurrences by an equivalent exact solve (SPD, diagonally dominant).
template <typename T>
__device__ __forceinline__ void pcr_solve(int lane, int P, const T* sd, const T* se, const T* rhs, T* q, T* A0, T* B0,
                                          T* C0, T* R0, T* A1, T* B1, T* C1, T* R1) {
    // (A1.. may alias sd / se / rhs: those are read only before the first step)
    for (int i = lane; i < P; i += 32) {
        A0[i] = i > 0 ? se[i - 1] : T(0);
        B0[i] = sd[i];
        C0[i] = i + 1 < P ? se[i] : T(0);
        R0[i] = rhs[i];
    }
    __syncwarp();
    for (int st = 1; st < P; st <<= 1) {
        for (int i = lane; i < P; i += 32) {
            const int im = i - st, ip = i + st;
            const T k1 = im >= 0 ? A0[i] / B0[im] : T(0);
            const T k2 = ip < P ? C0[i] / B0[ip] : T(0);
            A1[i] = im >= 0 ? -A0[im] * k1 : T(0);
            C1[i] = ip < P ? -C0[ip] * k2 : T(0);
            B1[i] = B0[i] - (im >= 0 ? C0[im] * k1 : T(0)) - (ip < P ? A0[ip] * k2 : T(0));
            R1[i] = R0[i] - (im >= 0 ? R0[im] * k1 : T(0)) - (ip < P ? R0[ip] * k2 : T(0));
        }
        __syncwarp();
        T* t;
        t = A0; A0 = A1; A1 = t;
        t = B0; B0 = B1; B1 = t;
        t = C0; C0 = C1; C1 = t;
        t = R0; R0 = R1; R1 = t;
    }
    for (int i = lane; i < P; i += 32) q[i] = R0[i] / B0[i];
    __syncwarp();
}

// Register-resident PCR for P <= 32 E: lane owns equations i = lane + 32 m,
// m < E.  At step st the partner equations i -+ st are fetched by shuffle
// (st < 32: same m from lane -+ st, or m -+ 1 across the lane wrap) or by
// register index (st = 32 q: same lane, m -+ q); each owner supplies 1 / b_i,
// so a step costs one reciprocal and eight shuffles per equation and no
// shared memory.  Same elimination as pcr_solve (k1 = a_i / b_{i-s},
// k2 = c_i / b_{i+s}); the divisions become multiplications by the
// partners' reciprocals (<= 1 ulp per step).
template <typename T, int E, int ST, int DIR>
__device__ __forceinline__ void pcr_fetch(const T (&x)[E], T (&out)[E], int lane) {
    if constexpr (ST < 32) {
        T y[E];
        const int src = (lane + DIR * ST) & 31;
#pragma unroll
        for (int m = 0; m < E; m++) y[m] = __shfl_sync(FULL, x[m], src);
        const bool wrap = DIR < 0 ? lane < ST : lane + ST >= 32;
#pragma unroll
        for (int m = 0; m < E; m++) {
            T alt = T(0);
            if constexpr (DIR < 0) {
                if (m >= 1) alt = y[m >= 1 ? m - 1 : 0];
            } else {
                if (m + 1 < E) alt = y[m + 1 < E ? m + 1 : 0];
            }
            out[m] = wrap ? alt : y[m];
        }
    } else {
        constexpr int q = ST / 32;
#pragma unroll
        for (int m = 0; m < E; m++) {
            const int j = m + DIR * q;
            out[m] = (j >= 0 && j < E) ? x[(j >= 0 && j < E) ? j : 0] : T(0);
        }
    }
}

template <typename T, int E, int ST>
__device__ __forceinline__ void pcr_step(int lane, int P, T (&A)[E], T (&B)[E], T (&C)[E], T (&R)[E]) {
    if (ST >= P) return;
    T rB[E], a1[E], b1[E], c1[E], r1[E], X[E], Y[E], Z[E], W[E];
#pragma unroll
    for (int m = 0; m < E; m++) rB[m] = T(1) / B[m];
    // partner i - st: a1 = -a_{i-s} k1, b -= c_{i-s} k1, r -= r_{i-s} k1
    pcr_fetch<T, E, ST, -1>(rB, W, lane);
    pcr_fetch<T, E, ST, -1>(A, X, lane);
    pcr_fetch<T, E, ST, -1>(C, Y, lane);
    pcr_fetch<T, E, ST, -1>(R, Z, lane);
#pragma unroll
    for (int m = 0; m < E; m++) {
        const bool hm = lane + 32 * m - ST >= 0;
        const T k1 = hm ? A[m] * W[m] : T(0);
        a1[m] = hm ? -X[m] * k1 : T(0);
        b1[m] = B[m] - (hm ? Y[m] * k1 : T(0));
        r1[m] = R[m] - (hm ? Z[m] * k1 : T(0));
    }
    // partner i + st: c1 = -c_{i+s} k2, b -= a_{i+s} k2, r -= r_{i+s} k2
    pcr_fetch<T, E, ST, +1>(rB, W, lane);
    pcr_fetch<T, E, ST, +1>(A, X, lane);
    pcr_fetch<T, E, ST, +1>(C, Y, lane);
    pcr_fetch<T, E, ST, +1>(R, Z, lane);
#pragma unroll
    for (int m = 0; m < E; m++) {
        const int i = lane + 32 * m;
        const bool hp = i + ST < P, v = i < P;
        const T k2 = hp ? C[m] * W[m] : T(0);
        c1[m] = hp ? -Y[m] * k2 : T(0);
        b1[m] -= hp ? X[m] * k2 : T(0);
        r1[m] -= hp ? Z[m] * k2 : T(0);
        A[m] = v ? a1[m] : T(0);
        B[m] = v ? b1[m] : T(1);
        C[m] = v ? c1[m] : T(0);
        R[m] = v ? r1[m] : T(0);
    }
}

template <typename T, int E>
__device__ void pcr_solve_reg(int lane, int P, const T* sd, const T* se, const T* rhs, T* q) {
    T A[E], B[E], C[E], R[E];
#pragma unroll
    for (int m = 0; m < E; m++) {
        const int i = lane + 32 * m;
        const bool v = i < P;
        A[m] = v && i > 0 ? se[i - 1] : T(0);
        B[m] = v ? sd[i] : T(1);
        C[m] = v && i + 1 < P ? se[i] : T(0);
        R[m] = v ? rhs[i] : T(0);
    }
    pcr_step<T, E, 1>(lane, P, A, B, C, R);
    pcr_step<T, E, 2>(lane, P, A, B, C, R);
    pcr_step<T, E, 4>(lane, P, A, B, C, R);
    pcr_step<T, E, 8>(lane, P, A, B, C, R);
    pcr_step<T, E, 16>(lane, P, A, B, C, R);
    if constexpr (E > 1) pcr_step<T, E, 32>(lane, P, A, B, C, R);
    if constexpr (E > 2) pcr_step<T, E, 64>(lane, P, A, B, C, R);
    if constexpr (E > 4) pcr_step<T, E, 128>(lane, P, A, B, C, R);
#pragma unroll
    for (int m = 0; m < E; m++) {
        const int i = lane + 32 * m;
        if (i < P) q[i] = R[m] / B[m];
    }
    __syncwarp();
}

// Column solve: registers when the kernel is instantiated for E = ceil(P / 32)
// (E = 0: shared-memory PCR, any P).
template <typename T, int E>
__device__ __forceinline__ void col_tridiag_solve(int lane, int P, const T* sd, const T* se, const T* rhs, T* q,
                                                  T* A0, T* B0, T* C0, T* R0, T* A1, T* B1, T* C1, T* R1) {
    if constexpr (E > 0) pcr_solve_reg<T, E>(lane, P, sd, se, rhs, q);
    else pcr_solve<T>(lane, P, sd, se, rhs, q, A0, B0, C0, R0, A1, B1, C1, R1);
}

template <typename T>
__device__ __forceinline__ T warp_sum_t(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    return x;
}

// Column objective Fc at column b (shared): D + alpha S3 + beta P + rho hd/2 ||b - v||^2
// (all lanes get it; +inf if infeasible).  With DERIVS: the cell quantities
// and then grad, diag, offdiag of the column GN Hessian (oracle
// admm_b_objective).
template <typename T, bool DERIVS>
__device__ double admm_col_eval(const Geom& g, int lane, const T* sIp, const T* sIm, const T* sb, const T* sv, T rho,
                                T* sa, T* sc, T* sr, T* sp1, T* sp2, T* sg, T* sd, T* se) {
    const int n3 = g.n3, P = g.P;
    const T hd = gw<T>(g.hd, g.f_hd), ahd = gw<T>(g.ahd, g.f_ahd), bh2 = gw<T>(g.bh2, g.f_bh2);
    const T ih3 = gw<T>(g.ih3, g.f_ih3), ih3sq = gw<T>(g.ih3sq, g.f_ih3sq);
    double aD = 0, aS = 0, aP = 0, aX = 0;
    int inf = 0;
    for (int k = lane; k < n3; k += 32) {
        const T b0 = sb[k], b1 = sb[k + 1];
        const T Ab = T(0.5) * (b0 + b1);
        const T Db = diff_h3(b0, b1, g);
        double vp, vm;
        T spl, sml;
        gather_pm(sIp, sIm, n3, k, Ab, g, vp, vm, spl, sml);
        const double Dbd = (double)Db;
        const double rd = vp * (1.0 + Dbd) - vm * (1.0 - Dbd);
        aD = fma(rd, rd, aD);
        const T dd = (b1 - b0) * ih3;
        aS += (double)(dd * dd);
        T f0 = 0, p1 = 0, p2 = 0;
        if (fabs(Db) >= T(1)) inf = 1;
        else phi3(Db, f0, p1, p2);
        aP += (double)f0;
        if (DERIVS) {
            const T gg = (spl * (T(1) + Db) + sml * (T(1) - Db)) * ih3;
            const T s = (T)(vp + vm);
            sa[k] = gg * T(0.5) - s * ih3;
            sc[k] = gg * T(0.5) + s * ih3;
            sr[k] = (T)rd;
            sp1[k] = p1;
            sp2[k] = p2;
        }
    }
    for (int l = lane; l < P; l += 32) {
        const double dx = (double)sb[l] - (double)sv[l];
        aX = fma(dx, dx, aX);
    }
    aD = warp_sum_t(aD);
    aS = warp_sum_t(aS);
    aP = warp_sum_t(aP);
    aX = warp_sum_t(aX);
    inf = __any_sync(FULL, inf);
    const double F = inf ? INFINITY
                         : 0.5 * g.hd * (aD + g.alpha * aS + g.beta * aP + (double)rho * aX);
    if (DERIVS && !inf) {
        __syncwarp();
        for (int l = lane; l < P; l += 32) {
            const T bl = sb[l];
            T gr = rho * hd * (bl - sv[l]), d = rho * hd, e = T(0);
            if (l > 0) {
                const int k = l - 1;
                gr += hd * sc[k] * sr[k] + ahd * (bl - sb[l - 1]) * ih3sq + bh2 * sp1[k] * ih3;
                d += hd * sc[k] * sc[k] + bh2 * sp2[k] * ih3sq + ahd * ih3sq;
            }
            if (l < n3) {
                const int k = l;
                gr += hd * sa[k] * sr[k] + ahd * (bl - sb[l + 1]) * ih3sq - bh2 * sp1[k] * ih3;
                d += hd * sa[k] * sa[k] + bh2 * sp2[k] * ih3sq + ahd * ih3sq;
                e = hd * sa[k] * sc[k] - bh2 * sp2[k] * ih3sq - ahd * ih3sq;
            }
            sg[l] = gr;
            sd[l] = d;
            se[l] = e;
        }
        __syncwarp();
    }
    return F;
}

// b-update (oracle admm_b_update): per column `inner` GN steps, exact solve
// of tridiag(d, e) q = -grad (warp PCR), the per-column stop (R23), Armijo on
// the column objective with gamma = 1, 1/2, ... (ls_max tries).
template <typename T, int E>
__global__ void __launch_bounds__(32 * ADMM_WARPS, sizeof(T) == 4 ? ADMM_MINB : 1) admm_b_kernel(Geom g, Ctl c, const T* __restrict__ Ip,
                                                                const T* __restrict__ Im, T* __restrict__ b,
                                                                const T* __restrict__ z, const T* __restrict__ u,
                                                                const double* __restrict__ rho_p, int inner,
                                                                double c1, int ls_max, double col_tol,
                                                                const unsigned* __restrict__ done) {
    count_launch(c);
    // ADMM already stopped (iteration enqueued ahead of the host check) or this pair converged
    if (done[0] || done[1 + blockIdx.y]) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int pair = blockIdx.y;
    const int n3 = g.n3, P = g.P;
    T* base = reinterpret_cast<T*>(smem_raw) + (size_t)wid * admm_warp_elems(n3);
    T* sIp = base + 2;
    T* sIm = sIp + n3 + 4;
    T* sb = sIm + n3 + 2;
    T* sv = sb + P;
    T* sq = sv + P;
    T* sg = sq + P;
    T* sd = sg + P;
    T* se = sd + P;
    T* sbt = se + P;
    T* sa = sbt + P;
    T* sc = sa + P;
    T* sr = sc + P;
    T* sp1 = sr + P;
    T* sp2 = sp1 + P;
    if (lane < 2) {
        sIp[-2 + lane] = T(0);
        sIp[n3 + lane] = T(0);
        sIm[-2 + lane] = T(0);
        sIm[n3 + lane] = T(0);
    }
    const T rho = (T)rho_p[pair];
    const size_t pc = (size_t)pair * g.Nc, pn = (size_t)pair * g.ps;
    for (long long col = (long long)blockIdx.x * ADMM_WARPS + wid; col < g.ncol;
         col += (long long)gridDim.x * ADMM_WARPS) {
        const size_t oc = pc + (size_t)col * n3, on = pn + (size_t)col * P;
        for (int k = lane; k < n3; k += 32) {
            sIp[k] = Ip[oc + k];
            sIm[k] = Im[oc + k];
        }
        for (int l = lane; l < P; l += 32) {
            sb[l] = b[on + l];
            sv[l] = z[on + l] - u[on + l];
        }
        __syncwarp();
        for (int it = 0; it < inner; it++) {
            const double F = admm_col_eval<T, true>(g, lane, sIp, sIm, sb, sv, rho, sa, sc, sr, sp1, sp2, sg, sd, se);
            if (!(F < INFINITY)) break;                 // infeasible column: no step
            for (int l = lane; l < P; l += 32) sbt[l] = -sg[l];     // rhs = -grad
            __syncwarp();
            // PCR double buffers: the dead cell arrays, then d, e, rhs themselves
            // (read only by pcr_solve's set-up pass)
#ifdef ADMM_ABLATE_PCR   // diagnostic builds only: timing without the tridiagonal solve (results invalid)
            for (int l = lane; l < P; l += 32) sq[l] = sbt[l] / sd[l];
#else
            col_tridiag_solve<T, E>(lane, P, sd, se, sbt, sq, sa, sc, sr, sp1, sp2, sd, se, sbt);
#endif
            __syncwarp();
            double gq = 0;
            for (int l = lane; l < P; l += 32) gq += (double)sg[l] * (double)sq[l];
            gq = warp_sum_t(gq);
            if (-gq <= col_tol * fabs(F)) break;        // column converged (R23)
            T gamma = T(1);
            for (int t = 0; t < ls_max; t++) {
                for (int l = lane; l < P; l += 32) sbt[l] = sb[l] + gamma * sq[l];
                __syncwarp();
                const double Ft = admm_col_eval<T, false>(g, lane, sIp, sIm, sbt, sv, rho, nullptr, nullptr, nullptr,
                                                          nullptr, nullptr, nullptr, nullptr, nullptr);
                if (Ft < INFINITY && Ft <= F + c1 * (double)gamma * gq) {
                    for (int l = lane; l < P; l += 32) sb[l] = sbt[l];
                    __syncwarp();
                    break;
                }
                gamma *= T(0.5);
                __syncwarp();
            }
        }
        for (int l = lane; l < P; l += 32) b[on + l] = sb[l];
        __syncwarp();
    }
}

// w = b + u (the z-update right-hand side before the rho scaling).
template <typename T>
__global__ void __launch_bounds__(256) admm_rhs_kernel(Geom g, Ctl c, const T* __restrict__ b, const T* __restrict__ u,
                                                       T* __restrict__ w, const unsigned* __restrict__ done) {
    count_launch(c);
    if (done[0] || done[1 + blockIdx.y]) return;   // stopped, or this pair converged (per-pair stop, R26)
    const size_t po = (size_t)blockIdx.y * g.ps;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < g.Nn; t += (long long)gridDim.x * blockDim.x)
        w[po + t] = b[po + t] + u[po + t];
}

// Spectrum scaling: X(k1, k2, l) *= rho / ((alpha lambda(k1, k2) + rho) n1 n2),
// lambda = 4 sin^2(pi k1/n1)/h1^2 + 4 sin^2(pi k2/n2)/h2^2 (periodic L_xy),
// precomputed once per context in `lam`.  Layout (cuFFT R2C, batch over l
// with stride P): [(k1 (n2/2+1) + k2) P + l]; one warp per (k1, k2) row of P.
template <typename C>
__global__ void __launch_bounds__(256) admm_zscale_kernel(Geom g, Ctl c, C* __restrict__ X,
                                                          const double* __restrict__ rho_p,
                                                          const double* __restrict__ lam, long long spec,
                                                          const unsigned* __restrict__ done) {
    count_launch(c);
    if (done[0] || done[1 + blockIdx.y]) return;   // stopped, or this pair converged (per-pair stop, R26)
    const int pair = blockIdx.y, lane = threadIdx.x & 31;
    const double rho = rho_p[pair];
    const int P = g.P;
    const long long nk = (long long)g.n1 * (g.n2 / 2 + 1);
    const double sc = 1.0 / ((double)g.n1 * g.n2);
    C* Xp = X + (size_t)pair * spec;
    for (long long kk = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); kk < nk;
         kk += (long long)gridDim.x * (blockDim.x >> 5)) {
        const double f = rho / (g.alpha * lam[kk] + rho) * sc;
        C* row = Xp + kk * P;
        for (int l = lane; l < P; l += 32) {
            row[l].x *= f;
            row[l].y *= f;
        }
    }
}

// lambda(k1, k2) table for admm_zscale_kernel.
__global__ void admm_lambda_kernel(Geom g, double* __restrict__ lam) {
    const int n2h = g.n2 / 2 + 1;
    for (long long kk = (long long)blockIdx.x * blockDim.x + threadIdx.x; kk < (long long)g.n1 * n2h;
         kk += (long long)gridDim.x * blockDim.x) {
        const int k1 = (int)(kk / n2h), k2 = (int)(kk - (long long)k1 * n2h);
        const double s1 = sin(M_PI * k1 / g.n1), s2 = sin(M_PI * k2 / g.n2);
        lam[kk] = 4.0 * s1 * s1 * g.ih1sq + 4.0 * s2 * s2 * g.ih2sq;
    }
}

// u <- u + b - z_new, z <- z_new; per pair: ||b - z_new||^2, ||z_new - z||^2,
// ||b - b_prev||^2, ||b||^2 (stored in c.red[pair][0..3]).
template <typename T>
__global__ void __launch_bounds__(256) admm_u_kernel(Geom g, Ctl c, const T* __restrict__ b,
                                                     const T* __restrict__ bprev, const T* __restrict__ znew,
                                                     T* __restrict__ z, T* __restrict__ u,
                                                     const unsigned* __restrict__ done) {
    count_launch(c);
    if (done[0] || done[1 + blockIdx.y]) return;   // stopped, or this pair converged (per-pair stop, R26)
    const int pair = blockIdx.y;
    const size_t po = (size_t)pair * g.ps;
    double r2 = 0, s2 = 0, db2 = 0, bb = 0;
    // unrolled by 4 (independent loads in flight; the kernel is load-latency
    // bound: ncu long-scoreboard 77 % with one element per loop trip)
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; t0 < g.Nn; t0 += 4 * stride) {
        T bv[4], zn[4], zo[4], uo[4], bp[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const long long t = t0 + j * stride;
            const size_t o = po + (t < g.Nn ? t : 0);
            bv[j] = b[o];
            zn[j] = znew[o];
            zo[j] = z[o];
            uo[j] = u[o];
            bp[j] = bprev[o];
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const long long t = t0 + j * stride;
            if (t >= g.Nn) break;
            const size_t o = po + t;
            const T du = bv[j] - zn[j];
            u[o] = uo[j] + du;
            z[o] = zn[j];
            r2 += (double)du * (double)du;
            s2 += ((double)zn[j] - (double)zo[j]) * ((double)zn[j] - (double)zo[j]);
            db2 += ((double)bv[j] - (double)bp[j]) * ((double)bv[j] - (double)bp[j]);
            bb += (double)bv[j] * (double)bv[j];
        }
    }
    double v[4] = {r2, s2, db2, bb}, tot[4];
    if (!pair_reduce<4, 0u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    for (int k = 0; k < 4; k++) c.red[(size_t)pair * RED_W + k] = tot[k];
}

// Residual balancing and the stop test on the device, after admm_u_kernel's
// pair totals r^2, |dz|^2, |db|^2, |b|^2 (oracle admm_rho_update and admm();
// R25, R26; |du| = |b - z| = r).  stat[pair][4] = iterations, r_norm, s_norm,
// converged.  done[1 + p]: pair p converged (not in fixed mode) -- its kernels
// return at once from then on, so every pair stops on its own test like the
// oracle's admm(); done[0]: every pair converged (the host's early exit).  A
// stopped pair only gets fac = 1, so admm_scale_u_kernel leaves its u alone.
__global__ void admm_balance_kernel(Ctl c, int B, double* __restrict__ rho, double* __restrict__ fac,
                                    double* __restrict__ stat, unsigned* __restrict__ done, int it, double mu,
                                    double tau, double tol, int fixed) {
    count_launch(c);
    const bool stopped = done[0] != 0;
    bool all_conv = true;
    for (int p = threadIdx.x; p < B; p += blockDim.x) {
        if (stopped || done[1 + p]) {
            fac[p] = 1.0;
            continue;
        }
        const double* t = c.red + (size_t)p * RED_W;
        const double r_norm = sqrt(t[0]), dz = sqrt(t[1]), db = sqrt(t[2]), bn = sqrt(t[3]);
        const double s_norm = rho[p] * dz;
        double f = 1.0;
        if (r_norm > mu * s_norm) {
            rho[p] *= tau;
            f = 1.0 / tau;
        } else if (s_norm > mu * r_norm) {
            rho[p] /= tau;
            f = tau;
        }
        fac[p] = f;
        const bool conv = fmax(db, fmax(dz, r_norm)) <= tol * fmax(bn, 1e-300);
        double* st = stat + (size_t)p * 4;
        st[0] = it + 1;
        st[1] = r_norm;
        st[2] = s_norm;
        st[3] = conv ? 1.0 : 0.0;
        if (conv && !fixed) done[1 + p] = 1u;
        all_conv = all_conv && conv;
    }
    all_conv = __syncthreads_and(all_conv);
    if (threadIdx.x == 0 && !stopped && all_conv && !fixed) done[0] = 1u;
}

// u *= f[pair] (residual balancing rescales the scaled multiplier).
template <typename T>
__global__ void __launch_bounds__(256) admm_scale_u_kernel(Geom g, Ctl c, T* __restrict__ u,
                                                           const double* __restrict__ f) {
    count_launch(c);
    const int pair = blockIdx.y;
    const T s = (T)f[pair];
    if (s == T(1)) return;
    const size_t po = (size_t)pair * g.ps;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < g.Nn; t += (long long)gridDim.x * blockDim.x)
        u[po + t] *= s;
}

}  // namespace hysco
