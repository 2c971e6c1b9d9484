// hysco_common.cuh — shared device-side types and helpers of libhysco (sm_100a).
//
// Nothing here is shared with oracle/ (the CPU fp64 test oracle); this is the
// product path only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hysco {

constexpr unsigned FULL = 0xffffffffu;

// Per-pair geometry, passed by value (all pairs share shape and voxel size).
struct Geom {
    int n1, n2, n3;      // cells; PE = n3 (contiguous)
    int P;               // n3 + 1 nodes per column (e3-staggered grid)
    long long ncol;      // n1 * n2 PE columns per pair
    long long Nc, Nn;    // cells / nodes per pair
    double h1, h2, h3;   // mm
    double hd;           // h1 h2 h3 (midpoint-rule weight)
    double alpha, beta;  // weights
    double ahd;          // alpha * hd
    double bh2;          // beta * hd / 2
    double ih1sq, ih2sq, ih3sq, ih3;
    // slab decomposition along dim 1: this rank owns global
    // planes [i0, i0 + n1) of n1g; node arrays then carry one halo plane on
    // each side and a pair stride ps = (n1 + 2) n2 P (ps = Nn without slabs).
    long long ps;
    int i0, n1g, slab;
    // fp32 copies of the weights (set by geom_finish): kernels read them as
    // constant-bank operands instead of converting the doubles per use
    float f_hd, f_ahd, f_bh2, f_ih1sq, f_ih2sq, f_ih3sq, f_ih3;
};

// Fill the fp32 copies of Geom's weights (host).
inline void geom_finish(Geom& g) {
    g.f_hd = (float)g.hd;
    g.f_ahd = (float)g.ahd;
    g.f_bh2 = (float)g.bh2;
    g.f_ih1sq = (float)g.ih1sq;
    g.f_ih2sq = (float)g.ih2sq;
    g.f_ih3sq = (float)g.ih3sq;
    g.f_ih3 = (float)g.ih3;
}
// A weight in the kernel's arithmetic type.
template <typename T> __device__ __forceinline__ T gw(double d, float f);
template <> __device__ __forceinline__ float gw<float>(double, float f) { return f; }
template <> __device__ __forceinline__ double gw<double>(double d, float) { return d; }

// in-plane neighbours along dim 1 exist (homogeneous Neumann, R3), global index
__device__ __forceinline__ bool has_im(const Geom& g, int i) { return g.i0 + i > 0; }
__device__ __forceinline__ bool has_ip(const Geom& g, int i) { return g.i0 + i < g.n1g - 1; }

// Device-resident per-pair solver state (no host round trip during a solve).
struct PairState {
    // objective at the last evaluated b
    double J, D, S, P, gnorm2;
    int infeasible;
    // Gauss-Newton / Armijo (R15, R16)
    int gn_active, gn_k, stop_reason;
    int ls_active, ls_tries, ls_restore, ls_halvings;
    int f_evals, h_evals, pcg_iters;
    double J_acc, J_prev, g0norm, gq, qmax, gamma;
    // PCG (R14)
    int pcg_active, pcg_k;
    double rz, rr0, rr, alpha_c, beta_c, relres;
    // OT init (R6, R10)
    double vmin, vmax, shift, maxDb, scale;
    int degenerate;
};

// Options the device-side control flow needs (copied from hysco_solve_opts).
struct SolveParams {
    int max_gn, max_pcg, fixed, ls_max;
    int armijo;   // 1: Armijo sufficient decrease (R15); 0: full step unless infeasible (parity mode)
    int precond;  // 0: Jacobi; 1: per-PE-column tridiagonal blocks (R20)
    double pcg_rtol, c1, tol_grad_rel, tol_dJ_rel, tol_db_rel;
    double feas_cap, ot_eps;
};

enum { COND_GN = 0, COND_PCG = 1, COND_LS = 2, NCOND = 3 };

// Per-iteration solver history ("OptimizationLogger"; hysco_history):
// record 0 = the GN start, record k = after the k-th accepted GN step.
// Same layout as hysco_iter_record (include/hysco.h).
constexpr int HIST_MAX = 64;
struct HistRec {
    int k, pcg_iters, ls_halvings, f_evals;
    double J, D, S, P, grad_norm, gamma, relres, step_max;
};

// Control block shared by all kernels of a context.
struct Ctl {
    PairState* st;                 // [batch]
    double* part;                  // [batch][max_blocks][8] block partials
    unsigned* ctr;                 // [batch] last-block counters (self-resetting)
    unsigned* gctr;                // [1] last-pair counter (self-resetting)
    unsigned long long* launches;  // kernel launch counter
    unsigned* dcond;               // [NCOND] loop conditions (mirrors of the graph handles)
    cudaGraphConditionalHandle h[NCOND];
    int use_graph;                 // 1: set graph conditionals from device code
    unsigned live;                 // bit k: h[k] belongs to the graph being built (else only dcond is set)
    int part_stride;               // doubles per pair in `part`
    int defer;                     // 1 (multi-rank): last blocks store pair totals in `red`,
                                   //   decisions run in decide_kernel after the allreduce
    double* red;                   // [batch][RED_W] pair totals (multi-rank)
    HistRec* hist;                 // [batch][HIST_MAX] per-GN-step history (may be null)
};
constexpr int RED_W = 8;

enum { STOP_MAXITER = 0, STOP_GRAD = 1, STOP_DJ = 2, STOP_DB = 3, STOP_LSFAIL = 4, STOP_INFEASIBLE = 5 };

__device__ __forceinline__ void count_launch(const Ctl& c) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(c.launches, 1ull);
}

__device__ __forceinline__ void set_cond(const Ctl& c, int slot, unsigned v) {
    c.dcond[slot] = v;
    if (c.use_graph && ((c.live >> slot) & 1u)) cudaGraphSetConditional(c.h[slot], v);
}

template <unsigned MAXMASK>
__device__ __forceinline__ double comb(int k, double a, double b) {
    return ((MAXMASK >> k) & 1u) ? fmax(a, b) : a + b;
}

template <unsigned MAXMASK>
__device__ __forceinline__ double ident(int k) {
    return ((MAXMASK >> k) & 1u) ? -INFINITY : 0.0;
}

// Deterministic two-level reduction of NV doubles over the blocks of one pair
// (blockIdx.y): block partials are written in fixed slots, the last block to
// finish (atomic ticket) folds them in a fixed order.  Bit-reproducible for a
// fixed grid.  MAXMASK bit k set = value k is a max-reduction, else a sum.
// Returns true in every thread of the pair's last block; tot[] is then valid.
template <int NV, unsigned MAXMASK>
__device__ bool pair_reduce(const Ctl& c, double (&v)[NV], double (&tot)[NV]) {
    __shared__ double sred[NV][32];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    const int pair = blockIdx.y;
    double* part = c.part + (size_t)pair * c.part_stride;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = comb<MAXMASK>(k, x, __shfl_xor_sync(FULL, x, o));
        if (lane == 0) sred[k][wid] = x;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        const int k = threadIdx.x;
        double x = sred[k][0];
        for (int w = 1; w < nw; w++) x = comb<MAXMASK>(k, x, sred[k][w]);
        part[(size_t)blockIdx.x * NV + k] = x;
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned prev = atomicAdd(&c.ctr[pair], 1u);
        s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
#pragma unroll
    for (int k = 0; k < NV; k++) {
        double x = ident<MAXMASK>(k);
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
            x = comb<MAXMASK>(k, x, __ldcg(&part[(size_t)b * NV + k]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = comb<MAXMASK>(k, x, __shfl_xor_sync(FULL, x, o));
        v[k] = x;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++)
        if (lane == 0) sred[k][wid] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++) {
        double x = sred[k][0];
        for (int w = 1; w < nw; w++) x = comb<MAXMASK>(k, x, sred[k][w]);
        tot[k] = x;
    }
    if (threadIdx.x == 0) c.ctr[pair] = 0;
    return true;
}

// Called by ONE thread of a pair's last block after it has written that
// pair's state: returns true for the last pair to finish (all pairs done).
__device__ __forceinline__ bool last_pair(const Ctl& c) {
    __threadfence();
    unsigned prev = atomicAdd(c.gctr, 1u);
    if (prev == gridDim.y - 1) {
        __threadfence();
        *c.gctr = 0;
        return true;
    }
    return false;
}

// any(flag) over pairs, read through L2 (written by other blocks of this kernel).
template <typename F>
__device__ __forceinline__ unsigned any_pair(const Ctl& c, int batch, F flag) {
    unsigned a = 0;
    for (int p = 0; p < batch; p++) a |= flag((volatile PairState*)(c.st + p)) ? 1u : 0u;
    return a;
}

// Node index decomposition within one pair: t -> (i, j, l), t = (i n2 + j) P + l.
struct NodeIdx {
    int i, j, l;
    long long col;
};
__device__ __forceinline__ NodeIdx node_idx(const Geom& g, long long t) {
    NodeIdx r;
    r.col = t / g.P;
    r.l = (int)(t - r.col * g.P);
    r.i = (int)(r.col / g.n2);
    r.j = (int)(r.col - (long long)r.i * g.n2);
    return r;
}

}  // namespace hysco

namespace hysco {

// ---------------------------------------------------------------------------
// Device-side decisions that follow each reduction (GN / PCG / Armijo control,
// OT shift, guard).  Single rank: called by the reducing kernel's last block.
// Multi-rank (Ctl::defer): the last block stores the pair totals in `red`
// (sums in red[pair][.], maxima in red[batch + pair][.]); the host allreduces
// them and decide_kernel calls the same function on the global totals.
// ---------------------------------------------------------------------------
enum { OP_EVAL = 0, OP_PCG_INIT = 1, OP_MATVEC = 2, OP_UPDATE = 3, OP_TRIAL = 4, OP_MINMAX = 5, OP_GUARD = 6 };

// store totals for the allreduce: k < nsum -> sum part, else max part
__device__ __forceinline__ void store_red(const Ctl& c, int pair, int batch, const double* tot, int nsum, int nmax) {
    for (int k = 0; k < nsum; k++) c.red[(size_t)pair * RED_W + k] = tot[k];
    for (int k = 0; k < nmax; k++) c.red[(size_t)(batch + pair) * RED_W + k] = tot[nsum + k];
}

}  // namespace hysco
