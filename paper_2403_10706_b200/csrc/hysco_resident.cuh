// hysco_resident.cuh — on-chip-resident Jacobi-PCG (A5 + A6 for a whole GN
// step in ONE persistent launch), fp32.
//
// Why: a PCG iteration of the streaming kernels moves ~60 B/node through HBM
// and needs three launches.  For a volume whose PCG state fits the chip
// (HCP 3T: 2.70 M nodes; per SM 126 columns x 146 padded nodes), each CTA
// keeps its contiguous range of PE columns resident for all iterations:
//   shared memory : p (read by neighbouring threads), M = diag(H), et  (12 B/node)
//   registers     : r and Hp / z, K float2 pairs per thread              ( 8 B/node)
//   global / L2   : x (L2 adds, owner only, padded layout) and a copy of p
//                   that neighbouring CTAs read for the in-plane halo.
// A thread owns pairs of consecutive nodes of one column (columns padded to
// an even length), so every access is 64-bit and every per-slot offset is a
// compile-time immediate (NT is a constant).
// One CTA per SM (cooperative launch guarantees co-residency).  Per iteration:
//   local Hp part (PE tridiagonal + in-CTA j-neighbours)
//   wait for the neighbour CTAs' p flags; remote Hp part (i-neighbours and
//     CTA-boundary j-neighbours from L2); p.Hp -> all-reduce
//   r, z = r/M, r.z, r.r -> publish;  x += a p (L2 adds);  collect
//   p = z + beta p (shared + global copy) -> release this CTA's p flag
// Reductions: exact integer (fixed-point limb) all-reduces for the PCG
// scalars, a deterministic fixed-order fold of tagged per-CTA partials for
// the Armijo start (it has a max): every CTA takes the same alpha / beta /
// stop decisions, and the results are bitwise reproducible.
#pragma once


namespace hysco {

#ifndef RES_THREADS_DEF
#define RES_THREADS_DEF 512
#define RES_KMAX_DEF 18
#endif
constexpr int RES_THREADS = RES_THREADS_DEF;  // 16 warps: 128 registers per thread, 18 node-pair slots without spills
constexpr int RES_KMAX = RES_KMAX_DEF;        // slots per thread (capacity 18 x 512 node pairs per SM)
static_assert(RES_KMAX % 3 == 0 && 5 * RES_KMAX <= 128, "three slot-count variants; 5 mask fields in 128 bits");

// Opaque copy: stops ptxas from hoisting per-slot index math (and everything
// derived from it) out of the PCG iteration loop, which would keep ~15
// values live per slot across all iterations.
__device__ __forceinline__ int opaque(int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
// ---------------------------------------------------------------------------
// Synchronisation without grid barriers.  The launch is cooperative (all CTAs
// co-resident), but no cooperative_groups grid sync is used:
//  * all-reduce (the Armijo start; the PCG scalars use the limb all-reduce
//    below): every CTA publishes its fp64 partial with ONE 64-bit store
//    whose low 8 mantissa bits carry a tag (launch, iteration); readers poll
//    the slots until every tag matches and fold them in a fixed order.  The
//    data is its own flag, so an all-reduce costs one publish and one poll
//    round trip through L2 instead of arrive-atomic + poll + fold.  The tag
//    perturbs a partial by <= 2^-44 relative; every CTA folds the same tagged
//    values, so all CTAs still take identical alpha / beta / stop decisions.
//  * p halo: a CTA releases a per-CTA flag after storing its new p; a reader
//    acquires only the flags of the CTAs that own its i- / j-neighbour
//    columns (a neighbourhood wait, not a grid barrier).
// Slots are reused every iteration without a hazard: a CTA rewrites a slot of
// reduction R for iteration k+1 only after the next all-reduce of iteration k
// has completed, which every CTA enters after reading R(k).  A stale slot
// holds the previous iteration's or the previous launch's tag (the launch
// counter advances once per launch), never the awaited one.  Polls are
// bounded: a stall of ~2^26 polls traps (a kernel error, not a hang).
// ---------------------------------------------------------------------------
constexpr unsigned RES_SPIN_LIMIT = 1u << 26;
// Contention: 148 pollers reading the same few cache lines serialise at one
// L2 slice (measured: the first poll of a collect took ~4800 cycles, vs
// ~250 for an L2 hit).  So every partial is published to RES_REPL replicas
// RES_RSTRIDE doubles apart (different lines / slices) and CTA b polls replica
// b % RES_REPL; the p-halo flags sit one per 128-byte line.
constexpr int RES_REPL = 16;
constexpr int RES_RSTRIDE = 512;             // doubles per replica (>= G x NV)
constexpr int RES_PART_DOUBLES = RES_REPL * RES_RSTRIDE;   // one reduction buffer
constexpr int RES_FLAG_STRIDE = 32;          // uints between flags (128 B)
__host__ __device__ inline size_t res_flags_words(int G) { return (size_t)(G + 1) * RES_FLAG_STRIDE; }

__device__ __forceinline__ unsigned res_tag(unsigned launch, int seq) { return ((launch & 7u) << 5) | ((unsigned)seq & 31u); }
__device__ __forceinline__ double tag_value(double v, unsigned tag) {
    return __longlong_as_double((__double_as_longlong(v) & ~0xffll) | (long long)tag);
}
__device__ __forceinline__ unsigned value_tag(double v) { return (unsigned)(__double_as_longlong(v) & 0xff); }
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Optional phase trace (tools/res_trace.cu): thread 0 of every CTA stamps the
// global timer at phase boundaries of the first 16 iterations.
__device__ __forceinline__ void res_stamp(unsigned long long* tr) {
    if (tr && threadIdx.x == 0) {
        unsigned long long t;
#ifdef RES_TRACE_CLOCK   // diagnostic builds: SM cycle counter (per-CTA durations only)
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
#else
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
#endif
        *tr = t;
    }
}

// Publish this CTA's NV partials (block-reduced in fixed order) with tag.
// MAXMASK bit k set: value k is a max-reduction (of values >= 0), else a sum.
template <int NV, unsigned MAXMASK = 0>
__device__ __forceinline__ void reduce_publish(double (&v)[NV], double* __restrict__ part, unsigned tag) {
    __shared__ double sred[NV][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = comb<MAXMASK>(k, x, __shfl_xor_sync(FULL, x, o));
        if (lane == 0) sred[k][wid] = x;
    }
    __syncthreads();
    if (wid < NV) {                          // warp k folds value k over the warps (shuffle tree)
        const int k = wid;
        double x = lane < nw ? sred[k][lane] : ident<MAXMASK>(k);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = comb<MAXMASK>(k, x, __shfl_xor_sync(FULL, x, o));
        if (lane < RES_REPL)                 // all lanes hold the total: lane r writes replica r
            st_relaxed_f64(part + lane * RES_RSTRIDE + blockIdx.x * NV + k, tag_value(x, tag));
    }
}

// Wait for every CTA's tagged partials and fold them in fixed order (warp k
// folds value k, identically in every CTA).  Result in out[] (all threads).
template <int NV, unsigned MAXMASK = 0>
__device__ __forceinline__ void reduce_collect(const double* __restrict__ part, unsigned tag, double (&out)[NV],
                                               unsigned long long* dbg = nullptr) {
    constexpr int MS = 8;                    // slots per lane: up to 256 CTAs
    __shared__ double stot[NV];
    const int wid = threadIdx.x >> 5;
    if (wid < NV) {
        const int lane = threadIdx.x & 31, G = gridDim.x;
        part += (blockIdx.x % RES_REPL) * RES_RSTRIDE;
        double v[MS];
        unsigned pending = 0;
        unsigned long long c0 = 0, c1 = 0;
        if (dbg) c0 = clock64();
#pragma unroll
        for (int m = 0; m < MS; m++) {
            const int b = lane + 32 * m;
            v[m] = 0.0;
            if (b < G) {
                v[m] = ld_relaxed_f64(part + b * NV + wid);
                if (value_tag(v[m]) != tag) pending |= 1u << m;
            }
        }
        unsigned spins = 0;
        if (dbg) {
            __syncwarp();
            c1 = clock64();
        }
        while (__any_sync(FULL, pending != 0)) {
            if (++spins > RES_SPIN_LIMIT) __trap();
#pragma unroll
            for (int m = 0; m < MS; m++)
                if (pending & (1u << m)) {
                    v[m] = ld_relaxed_f64(part + (lane + 32 * m) * NV + wid);
                    if (value_tag(v[m]) == tag) pending &= ~(1u << m);
                }
        }
        const bool mx = (MAXMASK >> wid) & 1u;
        double x = v[0];
#pragma unroll
        for (int m = 1; m < MS; m++) x = mx ? fmax(x, v[m]) : x + v[m];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(FULL, x, o);
            x = mx ? fmax(x, y) : x + y;
        }
        if (lane == 0) stot[wid] = x;
        if (dbg && threadIdx.x == 0) {       // diagnostic: first-poll cycles, spin cycles, spins
            const unsigned long long c2 = clock64();
            dbg[0] = c1 - c0;
            dbg[8] = c2 - c1;
            dbg[16] = spins;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++) out[k] = stot[k];
}

// ---------------------------------------------------------------------------
// Exact fixed-point all-reduce on integer atomics (the per-iteration PCG
// reductions).  Measured on B200 (tools/sync_bench.cu, 148 x 512 threads):
// the tagged all-poll above costs ~3.4 us per all-reduce, a release/acquire
// barrier 1.2 us, this 1.0-1.4 us.  Each value v of a CTA is divided by a
// power of two 2^e that every CTA derives from the same previous value, and
// q = v 2^-e (|q| < 2^59) is split EXACTLY into four signed 40-bit limbs of
// weights 2^20, 2^-20, 2^-60, 2^-100 (floor / subtract / scale: exact fp64
// steps; the last limb rounds below 2^-100).  Limb w is added to its own
// 64-bit word as (w << 8) + 1 with one red.add: the word's low byte counts
// the arrivals, its upper bits sum the limbs (integer: exact and independent
// of the arrival order).  A fifth word per value counts non-finite or
// out-of-range partials (result NaN).  Readers poll the words until all G
// arrivals are in and evaluate the same integer sums identically, so every
// CTA takes the same decisions and the result is bitwise reproducible.
// Words are never reset: a reader takes the difference to the word's value
// after the previous use (kept in shared memory).  Two parity sets: a CTA
// adds to set s for reduction n + 2 only after reduction n + 1 completed,
// i.e. after every CTA read reduction n.  Needs G < 256 (one arrival byte).
// ---------------------------------------------------------------------------
constexpr int RES_LIMB_W = 16;               // words per parity set (5 per value, NV <= 2)
constexpr int RES_LIMB_DOUBLES = 64;         // allocation after the three poll buffers (2 sets + pad)
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Binary exponent of the scale for a value expected near `prev` (same in
// every CTA: prev is an all-reduced result).
__device__ __forceinline__ int limb_exp(double prev) {
    return (prev != 0.0 && isfinite(prev)) ? ilogb(prev) : 0;
}
// Read the words' current values (before this launch's first limb reduction;
// the caller's next __syncthreads orders the loads before any arrival).
__device__ __forceinline__ void limb_init(const unsigned long long* words, unsigned long long* s_prev) {
    if (threadIdx.x < 2 * RES_LIMB_W) s_prev[threadIdx.x] = ld_relaxed_u64(words + threadIdx.x);
}
template <int NV>
__device__ __forceinline__ void limb_publish(double (&v)[NV], const int (&ex)[NV], unsigned long long* words, int par) {
    __shared__ double sred[NV][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
        if (lane == 0) sred[k][wid] = x;
    }
    __syncthreads();
    if (wid < NV) {
        const int k = wid;
        double x = lane < nw ? sred[k][lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
        if (lane < 5) {
            const double q = ldexp(x, -ex[k]);
            const bool bad = !(fabs(q) < 0x1p59);          // also NaN
            long long limb = 0;
            if (!bad) {
                const double t3 = q * 0x1p-20, l3 = floor(t3);
                const double t2 = (t3 - l3) * 0x1p40, l2 = floor(t2);
                const double t1 = (t2 - l2) * 0x1p40, l1 = floor(t1);
                const double l0 = rint((t1 - l1) * 0x1p40);
                const double lv = lane == 3 ? l3 : lane == 2 ? l2 : lane == 1 ? l1 : l0;
                limb = (long long)lv;
            }
            const long long add = lane < 4 ? limb * 256 + 1 : (long long)bad * 256 + 1;
            red_add_u64(words + par * RES_LIMB_W + 5 * k + lane, (unsigned long long)add);
        }
    }
}
template <int NV>
__device__ __forceinline__ void limb_collect(const unsigned long long* words, int par, const int (&ex)[NV],
                                             unsigned long long* s_prev, double (&out)[NV]) {
    __shared__ double stot[NV];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (wid < NV && lane < 5) {
        const int G = gridDim.x, w = par * RES_LIMB_W + 5 * wid + lane;
        const unsigned long long pv = s_prev[w];
        unsigned long long cur;
        unsigned spins = 0;
        while ((((cur = ld_relaxed_u64(words + w)) - pv) & 255ull) != (unsigned long long)G)
            if (++spins > RES_SPIN_LIMIT) __trap();
        s_prev[w] = cur;
        const double L = (double)(((long long)(cur - pv) - G) >> 8);   // exact: |.| < 2^49
        const double L0 = __shfl_sync(0x1fu, L, 0), L1 = __shfl_sync(0x1fu, L, 1);
        const double L2 = __shfl_sync(0x1fu, L, 2), L3 = __shfl_sync(0x1fu, L, 3);
        const double nbad = __shfl_sync(0x1fu, L, 4);
        if (lane == 0)
            stot[wid] = nbad != 0.0 ? __longlong_as_double(0x7ff8000000000000ll)
                                    : ldexp(((L3 * 0x1p20 + L2 * 0x1p-20) + L1 * 0x1p-60) + L0 * 0x1p-100, ex[wid]);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++) out[k] = stot[k];
}

// After this CTA's p stores: release its flag (all threads' stores ordered by
// the CTA barrier, then a gpu-scope release by thread 0).
__device__ __forceinline__ void halo_release(unsigned* flags, unsigned tag) {
    __syncthreads();
    if (threadIdx.x == 0) st_release_u32(flags + (size_t)blockIdx.x * RES_FLAG_STRIDE, tag);
}
// Before reading neighbours' p: acquire the flags of CTAs [blo, bhi].
__device__ __forceinline__ void halo_acquire(const unsigned* flags, int blo, int bhi, unsigned tag) {
    if (threadIdx.x < 32) {
        for (int b = blo + (int)threadIdx.x; b <= bhi; b += 32) {
            unsigned spins = 0;
            while (ld_acquire_u32(flags + (size_t)b * RES_FLAG_STRIDE) != tag)
                if (++spins > RES_SPIN_LIMIT) __trap();
        }
    }
    __syncthreads();
}

// CTA owning column col when ncol columns are split as [b ncol / G, (b+1) ncol / G).
__device__ __forceinline__ int res_owner(long long col, long long ncol, int G) {
    int b = (int)((col * G) / ncol);
    while (b > 0 && (long long)b * ncol / G > col) b--;
    while (b < G - 1 && (long long)(b + 1) * ncol / G <= col) b++;
    return b;
}

// Resident-path preconditioner application: z = r * rcp.approx(M) (~1 ulp;
// M > 0 is only the Jacobi preconditioner).
__device__ __forceinline__ float precond(float r, float M) {
    float inv;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(M));
    return r * inv;
}

// x += v (2 consecutive floats) at L2, no return value (the owner is the only
// writer of its x nodes).
__device__ __forceinline__ void red_add2(float* p, float2 v) {
    asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

// q = n / d for 0 <= n < 2^31 with a precomputed multiplier (no IDIV).
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

// The resident path stores every PE column with Pp = P rounded up to an even
// node count (zero padding), so a thread handles a pair of consecutive nodes
// of one column with 64-bit shared / global accesses, and in-plane
// neighbours (+-Pp, +-n2 Pp) stay 8-byte aligned.  (Groups of 4 would need
// 3 % more padding at P = 145 and 8 more registers per slot.)
__host__ __device__ inline int res_pad(int P) { return (P + 1) & ~1; }

// Global copy of p used for the in-plane halo: per pair (n1 + 2) x n2 x Pp
// floats with zero ghost planes at i = -1 and i = n1, so an i-neighbour read
// needs no existence test (a missing Neumann neighbour contributes 0 to the
// off-diagonal sum; its diagonal share is already excluded from M).
__host__ __device__ inline size_t res_ghost_pair_floats(const Geom& g) {
    return (size_t)(g.n1 + 2) * g.n2 * res_pad(g.P);
}
// Dynamic shared memory of one CTA: p, M, et with K x NT node pairs each (the
// slots past the CTA's ncl Pp nodes are zero-padding, so no slot loop needs a
// branch) and three 2-float zero guards.
__host__ __device__ inline size_t res_smem_bytes(int K) {
    return (size_t)(3 * 2 * K * RES_THREADS + 6) * sizeof(float);
}
// Slack (floats) after the last pair's ghost copy: the i+1 reads of padding
// slots of the last CTA stay inside the allocation (their values are unused).
__host__ __device__ inline size_t res_ghost_slack_floats(int K) { return (size_t)2 * K * RES_THREADS; }

// slot-mask fields (bit f + k for slot k < 12): pair valid, j-1 neighbour in
// this CTA, j+1 in this CTA, j-1 neighbour in the previous CTA, j+1 in the next
enum { RM_VAL = 0, RM_JML = RES_KMAX, RM_JPL = 2 * RES_KMAX, RM_JMR = 3 * RES_KMAX, RM_JPR = 4 * RES_KMAX };
struct SlotMask {                            // 5 fields x RES_KMAX slots = 90 bits
    unsigned long long lo, hi;
};
__device__ __forceinline__ bool mbit(const SlotMask& m, int b) {
    return b < 64 ? ((m.lo >> b) & 1ull) != 0 : ((m.hi >> (b - 64)) & 1ull) != 0;
}
__device__ __forceinline__ void mset(SlotMask& m, int b) {
    if (b < 64) m.lo |= 1ull << b;
    else m.hi |= 1ull << (b - 64);
}
__device__ __forceinline__ unsigned long long opaque64(unsigned long long v) {
    unsigned long long r;
    asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(v));
    return r;
}

// 2-D tiles (TILED kernels): CTA b = ti TJ + tj owns the TH x TW columns
// (i0 + li, j0 + lj), i0 = ti TH, j0 = tj TW (exact tiling: n1 = TI TH,
// n2 = TJ TW), numbered cl = li TW + lj in shared memory.  Against 1-D strips
// of consecutive columns (whose i-neighbours all live in the neighbouring
// CTAs), only the tile's perimeter talks to other CTAs: at the HCP 3T shape
// (tiles 42 x 3, 4 x 37 = 148) the L2 halo loads drop to 90 of 254 columns
// per CTA and the global copy of p is stored only for the 86 perimeter
// columns (tools/res_trace.cu ablations: halo loads cost 2.6 us and the copy
// stores 2.8 us of a 14.6 us iteration).  The global copy is kept per CTA in
// the CTA's own slot order (KNT node pairs per CTA), so a neighbour tile's
// value sits at a per-CTA constant offset from the reader's own slot:
//   j - 1 (lj = 0)      -> CTA b - 1,  slot q + (TW - 1) GPC
//   j + 1 (lj = TW - 1) -> CTA b + 1,  slot q - (TW - 1) GPC
//   i - 1 (li = 0)      -> CTA b - TJ, slot q + (TH - 1) TW GPC
//   i + 1 (li = TH - 1) -> CTA b + TJ, slot q - (TH - 1) TW GPC
// In-tile neighbours are shared-memory reads at q -+ GPC (j) and q -+ TW GPC
// (i).  The host picks tiles with TW GPC <= NT and (TH - 1) TW GPC >=
// (K - 1) NT, so only slot 0 holds first-row and only slot K - 1 last-row
// pairs: the i-direction needs no mask bits.
struct ResTile {
    int TI, TJ, TH, TW;
};
__host__ __device__ inline size_t res_tiled_ghost_floats(int G, int K) { return (size_t)G * 2 * K * RES_THREADS; }

// Before reading neighbours' p: acquire the flags of the (up to 4) listed CTAs.
__device__ __forceinline__ void halo_acquire_list(const unsigned* flags, const int (&nb)[4], unsigned tag) {
    if (threadIdx.x < 4) {
        const int b = nb[threadIdx.x];
        if (b >= 0) {
            unsigned spins = 0;
            while (ld_acquire_u32(flags + (size_t)b * RES_FLAG_STRIDE) != tag)
                if (++spins > RES_SPIN_LIMIT) __trap();
        }
    }
    __syncthreads();
}

// TRACE: phase stamps for tools/res_trace.cu (compiled out of the library's kernel).
template <int K, bool FIXED, bool TRACE = false, bool TILED = false>
__global__ void __launch_bounds__(RES_THREADS, 1)
    pcg_resident_kernel(Geom g, Ctl c, SolveParams sp, int pair, const float* __restrict__ grad,
                        const float* __restrict__ dt, const float* __restrict__ et, float* __restrict__ x,
                        float* __restrict__ xpad, float* __restrict__ pgh, double* __restrict__ gpart,
                        unsigned* __restrict__ flags, float wi, float wj, float* __restrict__ bcur,
                        float* __restrict__ bold, int batch, unsigned long long* trace = nullptr,
                        ResTile tl = ResTile{0, 0, 0, 0}) {
    constexpr int NT = RES_THREADS;
    static_assert(K <= RES_KMAX, "slot masks hold RES_KMAX slots per field");
    count_launch(c);
    if (!pcg_step_active(c.st[pair])) {      // uniform over the grid: no step (finished, or a search pending)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (!c.st[pair].gn_active) c.st[pair].ls_active = 0;
            if (pair == batch - 1)
                set_cond(c, COND_LS, any_pair(c, batch, [](volatile PairState* q2) { return q2->ls_active != 0; }));
        }
        return;
    }
    unsigned long long* trk = TRACE ? trace + ((size_t)blockIdx.x * 16 + 15) * 8 : nullptr;   // launch-level stamps
    if constexpr (TRACE) res_stamp(trk);
    extern __shared__ __align__(16) float smem_f[];
    const int P = g.P, Pp = res_pad(P), GPC = Pp >> 1, n2 = g.n2;
    // strips: columns [c0, c1); tiles: (ti, tj), TWG = pairs per tile row, RL = first last-row pair
    const int b = blockIdx.x;
    const int ti = TILED ? b / tl.TJ : 0, tj = TILED ? b - ti * tl.TJ : 0;
    const int TWG = TILED ? tl.TW * GPC : 0, RL = TILED ? (tl.TH - 1) * TWG : 0;
    const long long c0 = TILED ? 0 : (long long)b * g.ncol / gridDim.x;
    const long long c1 = TILED ? 0 : (long long)(b + 1) * g.ncol / gridDim.x;
    const int ncl = TILED ? tl.TH * tl.TW : (int)(c1 - c0);
    const int nq = ncl * GPC;                // node pairs owned by this CTA
    // shared layout (floats): [guard 2][p: KNT pairs][guard 2][M: KNT pairs][guard 2][et: KNT pairs]
    // Padding nodes (l >= P, and slots past the CTA's columns) have M = 1,
    // et = 0, r = 0, so their p and Hp stay exactly 0; et at l = n3 is 0, so
    // the PE coupling never crosses columns.
    constexpr int KNT2 = 2 * K * NT;
    float* sp_ = smem_f + 2;
    float* sM = sp_ + KNT2 + 2;
    float* se = sM + KNT2 + 2;
    float2* sp2 = reinterpret_cast<float2*>(sp_);
    float2* sM2 = reinterpret_cast<float2*>(sM);
    float2* se2 = reinterpret_cast<float2*>(se);
    const size_t n0 = (size_t)pair * g.ps + (size_t)c0 * P;
    // this CTA's first node in the ghost-padded global copy of p, and in xpad
    // (tiles: its own KNT-pair regions of both)
    float2* __restrict__ pgc2 =
        TILED ? reinterpret_cast<float2*>(pgh + (size_t)pair * res_tiled_ghost_floats(gridDim.x, K) +
                                          (size_t)b * KNT2)
              : reinterpret_cast<float2*>(pgh + (size_t)pair * res_ghost_pair_floats(g) + (size_t)(c0 + n2) * Pp);
    float2* __restrict__ xp2 = reinterpret_cast<float2*>(xpad + (TILED ? (size_t)b * KNT2 : (size_t)c0 * Pp));
    const int sI2 = n2 * GPC;                // i-neighbour distance in node pairs (strips)
    // tiles: offsets (in pairs) of the neighbour tiles' copies, relative to this CTA's
    const long long oJM = -(long long)KNT2 / 2 + (long long)(tl.TW - 1) * GPC;
    const long long oJP = (long long)KNT2 / 2 - (long long)(tl.TW - 1) * GPC;
    const long long oIM = -(long long)tl.TJ * (KNT2 / 2) + RL;
    const long long oIP = (long long)tl.TJ * (KNT2 / 2) - RL;
    const bool hasIM = TILED && ti > 0, hasIP = TILED && ti < tl.TI - 1;
    double* part0 = gpart;                          // [repl][G][2] r0.z0, r0.r0 (and the Armijo start)
    // limb words: set 0 p.Hp, set 1 (r0.z0, r0.r0) and (r.z, r.r) -- exact integer all-reduces
    unsigned long long* lw = reinterpret_cast<unsigned long long*>(gpart + 3 * RES_PART_DOUBLES);
    __shared__ unsigned long long s_prev[2 * RES_LIMB_W];
    const int tid = threadIdx.x;
    // flags[b * RES_FLAG_STRIDE]: p-halo flag of CTA b; flags[G * RES_FLAG_STRIDE]: launch counter
    const unsigned launch = *reinterpret_cast<volatile unsigned*>(flags + (size_t)gridDim.x * RES_FLAG_STRIDE);
    // CTAs owning this CTA's i-neighbour (+-n2) and j-neighbour (+-1) columns
    const int blo = TILED ? 0 : res_owner(c0 - n2 > 0 ? c0 - n2 : 0, g.ncol, gridDim.x);
    const int bhi = TILED ? 0 : res_owner(c1 - 1 + n2 < g.ncol ? c1 - 1 + n2 : g.ncol - 1, g.ncol, gridDim.x);
    const int nbl[4] = {TILED && tj > 0 ? b - 1 : -1, TILED && tj < tl.TJ - 1 ? b + 1 : -1, hasIM ? b - tl.TJ : -1,
                        hasIP ? b + tl.TJ : -1};

    if (tid < 6) smem_f[tid < 2 ? tid : tid < 4 ? 2 + KNT2 + (tid - 2) : 4 + 2 * KNT2 + (tid - 4)] = 0.f;
    limb_init(lw, s_prev);                   // before the start publish (halo_release's barrier)
    SlotMask msk{0ull, 0ull};
    float2 r[K], hv[K];
    float frz = 0.f, frr = 0.f;
    {
        FastDiv fdG, fdN2;
        fdG.init((unsigned)GPC);
        fdN2.init((unsigned)n2);
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int q = tid + k * NT;
            float2 rv = make_float2(0.f, 0.f), Mv = make_float2(1.f, 1.f), ev = make_float2(0.f, 0.f);
            if (q < nq) {
                const int cl = fdG.div(q);
                const int l0 = 2 * (q - cl * GPC);
                int i, j, lj = 0;
                if constexpr (TILED) {
                    const int li = cl / tl.TW;
                    lj = cl - li * tl.TW;
                    i = ti * tl.TH + li;
                    j = tj * tl.TW + lj;
                } else {
                    const long long col = c0 + cl;
                    i = fdN2.div((int)col);
                    j = (int)col - i * n2;
                }
                const float dl = (float)(g.ahd * diag_lxy(g, i, j));
                const size_t o = TILED ? (size_t)pair * g.ps + ((size_t)i * n2 + j) * P + l0 : n0 + (size_t)cl * P + l0;
                Mv.x = dt[o] + dl;
                ev.x = et[o];
                rv.x = -grad[o];
                if (l0 + 1 < P) {
                    Mv.y = dt[o + 1] + dl;
                    ev.y = et[o + 1];
                    rv.y = -grad[o + 1];
                }
                mset(msk, RM_VAL + k);
                if constexpr (TILED) {               // j-neighbours: in the tile, or the next tile's
                    if (j > 0) mset(msk, (lj > 0 ? RM_JML : RM_JMR) + k);
                    if (j < n2 - 1) mset(msk, (lj < tl.TW - 1 ? RM_JPL : RM_JPR) + k);
                } else {
                    if (j > 0) mset(msk, (cl > 0 ? RM_JML : RM_JMR) + k);
                    if (j < n2 - 1) mset(msk, (cl < ncl - 1 ? RM_JPL : RM_JPR) + k);
                }
                const float2 z = make_float2(precond(rv.x, Mv.x), precond(rv.y, Mv.y));
                frz = fmaf(rv.x, z.x, frz);
                frz = fmaf(rv.y, z.y, frz);
                frr = fmaf(rv.x, rv.x, frr);
                frr = fmaf(rv.y, rv.y, frr);
                sp2[q] = z;
                pgc2[q] = z;                   // x = 0 is written by the first update (or below)
            } else {
                sp2[q] = rv;
            }
            sM2[q] = Mv;
            se2[q] = ev;
            r[k] = rv;
            hv[k] = make_float2(0.f, 0.f);
        }
    }
    double v2[2] = {(double)frz, (double)frr}, t2[2];
    if constexpr (TRACE) res_stamp(trk + 1);
    halo_release(flags, res_tag(launch, 0));  // p0 published
    {   // r0.z0, r0.r0 on limbs, scaled by ||grad||^2 (= r0.r0) of the evaluation
        const int e0 = limb_exp(c.st[pair].gnorm2);
        const int ex0[2] = {e0, e0};
        limb_publish<2>(v2, ex0, lw, 1);
        limb_collect<2>(lw, 1, ex0, s_prev, t2);
    }
    if constexpr (TRACE) res_stamp(trk + 2);
    // Loop state kept out of registers (the r / Hp slots need 48 of the 80):
    // rr0 and the last r.r live in shared memory; the H-evaluation count, "x
    // already set" and "p barrier pending" all equal k_it > 0 / k_it.
    __shared__ double s_rr0, s_rr;
    double rz = t2[0];
    if (tid == 0) {
        s_rr0 = t2[1];
        s_rr = t2[1];
    }
    int k_it = 0;
    if (t2[1] > 0.0) {
        for (k_it = 0; k_it < sp.max_pcg;) {
            unsigned long long* tr = (TRACE && k_it < 16) ? trace + ((size_t)blockIdx.x * 16 + k_it) * 8 : nullptr;
            if constexpr (TRACE) res_stamp(tr);
            // ---- local part of Hp (own shared memory only; overlaps the p barrier):
            // M p + et_{l-1} p_{l-1} + et_l p_{l+1} - alpha hd / h2^2 (p_{j-1} + p_{j+1}).
            // Every slot loop is branch-free (padding slots compute zeros), so
            // all loads of a phase can be in flight together.
            {
                const int t0 = opaque(tid);
                const SlotMask m{opaque64(msk.lo), opaque64(msk.hi)};
                const float2* s2 = sp2 + t0;
                const float2* m2 = sM2 + t0;
                const float2* e2 = se2 + t0;
                const float* s1 = sp_ + 2 * t0;
                const float* e1 = se + 2 * t0;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int o = k * NT;
                    const float2 p = s2[o], M = m2[o], e = e2[o];
                    const float pm = s1[2 * o - 1], em = e1[2 * o - 1], pn = s1[2 * o + 2];
                    float2 h;
                    h.x = fmaf(e.x, p.y, fmaf(em, pm, M.x * p.x));
                    h.y = fmaf(e.y, pn, fmaf(e.x, p.x, M.y * p.y));
                    const float2 a = mbit(m, RM_JML + k) ? s2[o - GPC] : make_float2(0.f, 0.f);
                    const float2 b = mbit(m, RM_JPL + k) ? s2[o + GPC] : make_float2(0.f, 0.f);
                    h.x = fmaf(-wj, a.x + b.x, h.x);
                    h.y = fmaf(-wj, a.y + b.y, h.y);
                    if constexpr (TILED) {           // in-tile i-neighbours (first / last row: remote)
                        float2 ia, ib;
                        if (k == 0) ia = t0 >= TWG ? s2[o - TWG] : make_float2(0.f, 0.f);
                        else ia = s2[o - TWG];
                        if (k == K - 1) ib = t0 + o < RL ? s2[o + TWG] : make_float2(0.f, 0.f);
                        else ib = s2[o + TWG];
                        h.x = fmaf(-wi, ia.x + ib.x, h.x);
                        h.y = fmaf(-wi, ia.y + ib.y, h.y);
                    }
                    hv[k] = h;
                }
            }
            if constexpr (TILED) halo_acquire_list(flags, nbl, res_tag(launch, k_it));
            else halo_acquire(flags, blo, bhi, res_tag(launch, k_it));   // neighbours' p_k
            if constexpr (TRACE) res_stamp(tr ? tr + 1 : nullptr);
            // ---- remote part: i-neighbours (and j-neighbours across the CTA
            // boundary) from the global copy; p.Hp
            float fpq = 0.f;
            {
                const int t0 = opaque(tid);
                const SlotMask m{opaque64(msk.lo), opaque64(msk.hi)};
                const float2* gc = pgc2 + t0;
                const float2* s2 = sp2 + t0;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int o = k * NT;
                    float2 a = make_float2(0.f, 0.f), b = a, c = a, d = a;
                    if constexpr (TILED) {           // perimeter only: the neighbour tiles' copies
                        if (k == 0 && hasIM && t0 < TWG) a = __ldcg(gc + oIM);
                        if (k == K - 1 && hasIP && t0 + o >= RL && t0 + o < nq) b = __ldcg(gc + o + oIP);
                        if (mbit(m, RM_JMR + k)) c = __ldcg(gc + o + oJM);
                        if (mbit(m, RM_JPR + k)) d = __ldcg(gc + o + oJP);
                    } else {
#ifndef RES_ABLATE_REMOTE   // diagnostic builds only (tools/res_trace.cu): timing without the i-halo loads
                        a = __ldcg(gc + o - sI2);
                        b = __ldcg(gc + o + sI2);
#endif
                        if (mbit(m, RM_JMR + k)) c = __ldcg(gc + o - GPC);
                        if (mbit(m, RM_JPR + k)) d = __ldcg(gc + o + GPC);
                    }
                    float2 h = hv[k];
                    h.x = fmaf(-wi, a.x + b.x, fmaf(-wj, c.x + d.x, h.x));
                    h.y = fmaf(-wi, a.y + b.y, fmaf(-wj, c.y + d.y, h.y));
                    const bool v = mbit(m, RM_VAL + k);
                    h.x = v ? h.x : 0.f;
                    h.y = v ? h.y : 0.f;
                    hv[k] = h;
                    const float2 p = s2[o];
                    fpq = fmaf(p.x, h.x, fpq);
                    fpq = fmaf(p.y, h.y, fpq);
                }
            }
            if constexpr (TRACE) res_stamp(tr ? tr + 2 : nullptr);
            double v1[1] = {(double)fpq}, t1[1];
            const int ex1[1] = {limb_exp(rz)};        // p.Hp = rz / alpha
            limb_publish<1>(v1, ex1, lw, 0);
            if constexpr (TRACE) res_stamp(tr ? tr + 7 : nullptr);
            limb_collect<1>(lw, 0, ex1, s_prev, t1);
            if constexpr (TRACE) res_stamp(tr ? tr + 3 : nullptr);
            if (t1[0] <= 0.0) break;                  // breakdown (oracle pcg(): keep x)
            const float a = (float)(rz / t1[0]);
            // ---- r -= a Hp, z = r/M (kept in the dead Hp registers); r.z, r.r
            float frz2 = 0.f, frr2 = 0.f;
            {
                const int t0 = opaque(tid);
                const float2* m2 = sM2 + t0;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const float2 M = m2[k * NT];
                    float2 rn = r[k];
                    rn.x = fmaf(-a, hv[k].x, rn.x);
                    rn.y = fmaf(-a, hv[k].y, rn.y);
                    r[k] = rn;
                    const float2 z = make_float2(precond(rn.x, M.x), precond(rn.y, M.y));
                    hv[k] = z;
                    frz2 = fmaf(rn.x, z.x, frz2);
                    frz2 = fmaf(rn.y, z.y, frz2);
                    frr2 = fmaf(rn.x, rn.x, frr2);
                    frr2 = fmaf(rn.y, rn.y, frr2);
                }
            }
            double v3[2] = {(double)frz2, (double)frr2}, t3[2];
            const int ex3[2] = {limb_exp(rz), limb_exp(s_rr)};
            limb_publish<2>(v3, ex3, lw, 1);
            if constexpr (TRACE) res_stamp(tr ? tr + 4 : nullptr);
            // ---- x += a p while the r.z / r.r partials gather (fire-and-forget
            // L2 adds; x feeds no reduction)
            {
                const int t0 = opaque(tid);
                const SlotMask m{opaque64(msk.lo), opaque64(msk.hi)};
                const float2* s2 = sp2 + t0;
                float2* xt = xp2 + t0;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const float2 p = s2[k * NT];
                    const float2 v = make_float2(a * p.x, a * p.y);
                    if (mbit(m, RM_VAL + k)) {
#if defined(RES_ABLATE_XNONE)   // diagnostic builds only: timing without any x traffic (q invalid)
                        if (v.x == 12345.f) xt[k * NT] = v;
#elif defined(RES_ABLATE_X)
                        if (k_it > 0) xt[k * NT] = v;
#else
                        if (k_it > 0) red_add2(reinterpret_cast<float*>(xt + k * NT), v);
#endif
                        else xt[k * NT] = v;  // first update: x_1 = 0 + a p_0
                    }
                }
            }
            limb_collect<2>(lw, 1, ex3, s_prev, t3);
            if constexpr (TRACE) res_stamp(tr ? tr + 5 : nullptr);
            k_it += 1;
            if (tid == 0) s_rr = t3[1];              // (ex3 read it before limb_publish's barrier)
            const double beta = t3[0] / rz;
            rz = t3[0];
            if (k_it >= sp.max_pcg || (!FIXED && sqrt(t3[1] / s_rr0) < sp.pcg_rtol)) break;
            // ---- p = z + beta p on own columns and on the global halo copy
            const float be = (float)beta;
            {
                const int t0 = opaque(tid);
                const SlotMask m{opaque64(msk.lo), opaque64(msk.hi)};
                float2* s2 = sp2 + t0;
                float2* gt = pgc2 + t0;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int o = k * NT;
                    const float2 p = s2[o], z = hv[k];
                    const float2 pn = make_float2(fmaf(be, p.x, z.x), fmaf(be, p.y, z.y));
                    s2[o] = pn;
#ifndef RES_ABLATE_GHOST
                    if constexpr (TILED) {           // only the perimeter is read by other CTAs
                        const bool bnd = mbit(m, RM_JMR + k) || mbit(m, RM_JPR + k) ||
                                         (k == 0 && hasIM && t0 < TWG) ||
                                         (k == K - 1 && hasIP && t0 + o >= RL && t0 + o < nq);
                        if (bnd) gt[o] = pn;
                    } else {
                        if (mbit(m, RM_VAL + k)) gt[o] = pn;
                    }
#endif
                }
            }
            if constexpr (TRACE) res_stamp(tr ? tr + 6 : nullptr);
            halo_release(flags, res_tag(launch, k_it));            // p_{k+1} published
        }
    }
    // ---- q = x back to the node layout, fused with the start of the Armijo
    // search (A7; the work of trial_init_kernel): g.q, max|q|,
    // b_old = b, b = b + q (gamma = 1).  The CTA's nodes are contiguous in the
    // node layout, so this pass walks them in order (coalesced 128-bit
    // accesses) and gathers q from the padded xpad (fenced after the L2 adds).
    double agq = 0.0, aqm = 0.0;
    __threadfence();
    __syncthreads();
    if constexpr (TILED) {
        // tiles: TH runs of TW P contiguous nodes; flattened over the CTA so
        // every warp access is 32 consecutive nodes of one run (coalesced)
        const int RW = tl.TW * P, Nb = tl.TH * RW;
        FastDiv fdR, fdP;
        fdR.init((unsigned)RW);
        fdP.init((unsigned)P);
        const size_t base = (size_t)pair * g.ps + ((size_t)ti * tl.TH * n2 + (size_t)tj * tl.TW) * P;
        const float* xq = xpad + (size_t)b * KNT2;
        constexpr int U = 4;
        for (int e0 = tid; e0 < Nb; e0 += U * NT) {
            float qv[U], gv[U], bv[U];
            size_t o[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int e = min(e0 + u * NT, Nb - 1);
                const int row = fdR.div(e), t = e - row * RW;
                const int cj = fdP.div(t), l = t - cj * P;
                o[u] = base + (size_t)row * n2 * P + t;
                qv[u] = k_it == 0 ? 0.f : __ldcg(xq + (size_t)(row * tl.TW + cj) * Pp + l);
                gv[u] = grad[o[u]];
                bv[u] = bcur[o[u]];
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (e0 + u * NT < Nb) {
                    agq += (double)gv[u] * (double)qv[u];
                    aqm = fmax(aqm, (double)fabsf(qv[u]));
                    x[o[u]] = qv[u];
                    bold[o[u]] = bv[u];
                    bcur[o[u]] = bv[u] + qv[u];
                }
            }
        }
    } else {
        const int Nb = ncl * P;              // this CTA's nodes, from n0
        FastDiv fdP;
        fdP.init((unsigned)P);
        auto qval = [&](int t) -> float {    // q at CTA-local node t
            if (k_it == 0) return 0.f;
            const int cl = fdP.div(t);
            return __ldcg(xpad + (size_t)c0 * Pp + (size_t)cl * Pp + (t - cl * P));
        };
        // head: nodes before the first 16-byte boundary of the node arrays
        const int head = min((int)((4 - (n0 & 3)) & 3), Nb);
        for (int t = tid; t < head; t += NT) {
            const size_t o = n0 + t;
            const float qv = qval(t), bv = bcur[o];
            agq += (double)grad[o] * (double)qv;
            aqm = fmax(aqm, (double)fabsf(qv));
            x[o] = qv;
            bold[o] = bv;
            bcur[o] = bv + qv;
        }
        const int nv = (Nb - head) >> 2;     // aligned float4 groups
        for (int v = tid; v < nv; v += NT) {
            const int t = head + 4 * v;
            const size_t o = n0 + t;
            const float4 gv = *reinterpret_cast<const float4*>(grad + o);
            const float4 bv = *reinterpret_cast<const float4*>(bcur + o);
            const float4 qv = make_float4(qval(t), qval(t + 1), qval(t + 2), qval(t + 3));
            agq += (double)gv.x * qv.x + (double)gv.y * qv.y + (double)gv.z * qv.z + (double)gv.w * qv.w;
            aqm = fmax(aqm, (double)fmaxf(fmaxf(fabsf(qv.x), fabsf(qv.y)), fmaxf(fabsf(qv.z), fabsf(qv.w))));
            *reinterpret_cast<float4*>(x + o) = qv;
            *reinterpret_cast<float4*>(bold + o) = bv;
            *reinterpret_cast<float4*>(bcur + o) =
                make_float4(bv.x + qv.x, bv.y + qv.y, bv.z + qv.z, bv.w + qv.w);
        }
        for (int t = head + 4 * nv + tid; t < Nb; t += NT) {   // tail
            const size_t o = n0 + t;
            const float qv = qval(t), bv = bcur[o];
            agq += (double)grad[o] * (double)qv;
            aqm = fmax(aqm, (double)fabsf(qv));
            x[o] = qv;
            bold[o] = bv;
            bcur[o] = bv + qv;
        }
    }
    {
        double v4[2] = {agq, aqm}, t4[2];
        reduce_publish<2, 0x2u>(v4, part0, res_tag(launch, 31));
        reduce_collect<2, 0x2u>(part0, res_tag(launch, 31), t4);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            decide_trial(c.st[pair], t4);
            if (pair == batch - 1)
                set_cond(c, COND_LS, any_pair(c, batch, [](volatile PairState* q2) { return q2->ls_active != 0; }));
        }
    }
    if constexpr (TRACE) res_stamp(trk + 3);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // every CTA read `launch` before its first publish, which CTA 0 has
        // collected, so the counter can advance now
        *reinterpret_cast<volatile unsigned*>(flags + (size_t)gridDim.x * RES_FLAG_STRIDE) = launch + 1;
        PairState& s = c.st[pair];
        s.rz = rz;
        s.rr0 = s_rr0;
        s.pcg_k = k_it;
        s.pcg_iters += k_it;
        s.h_evals += k_it;                   // one H p per completed iteration (a breakdown stops before both)
        s.relres = s_rr0 > 0.0 ? sqrt(s_rr / s_rr0) : 0.0;
        s.pcg_active = 0;
    }
}

// Synchronisation floor of the resident PCG (profiling only, bench.py's
// roofline): the same launch (grid, block, dynamic shared memory, hence one
// CTA per SM) and per-iteration dependency chain of pcg_resident_kernel --
// neighbourhood p-halo acquire, tagged all-reduce of p.Hp, tagged all-reduce
// of (r.z, r.r), p-halo release -- with every slot loop (the arithmetic and
// the shared / L2 data movement) removed.  Its time per iteration is the
// latency floor a PCG iteration on this chip layout cannot go below.
template <int K, bool TILED = false>
__global__ void __launch_bounds__(RES_THREADS, 1)
    pcg_sync_floor_kernel(Geom g, int iters, double* __restrict__ gpart, unsigned* __restrict__ flags,
                          ResTile tl = ResTile{0, 0, 0, 0}) {
    const long long c0 = (long long)blockIdx.x * g.ncol / gridDim.x;
    const long long c1 = (long long)(blockIdx.x + 1) * g.ncol / gridDim.x;
    const int n2 = g.n2, b = blockIdx.x;
    const int ti = TILED ? b / tl.TJ : 0, tj = TILED ? b - ti * tl.TJ : 0;
    const unsigned launch = *reinterpret_cast<volatile unsigned*>(flags + (size_t)gridDim.x * RES_FLAG_STRIDE);
    const int blo = TILED ? 0 : res_owner(c0 - n2 > 0 ? c0 - n2 : 0, g.ncol, gridDim.x);
    const int bhi = TILED ? 0 : res_owner(c1 - 1 + n2 < g.ncol ? c1 - 1 + n2 : g.ncol - 1, g.ncol, gridDim.x);
    const int nbl[4] = {TILED && tj > 0 ? b - 1 : -1, TILED && tj < tl.TJ - 1 ? b + 1 : -1,
                        TILED && ti > 0 ? b - tl.TJ : -1, TILED && ti < tl.TI - 1 ? b + tl.TJ : -1};
    double* part0 = gpart;
    unsigned long long* lw = reinterpret_cast<unsigned long long*>(gpart + 3 * RES_PART_DOUBLES);
    __shared__ unsigned long long s_prev[2 * RES_LIMB_W];
    limb_init(lw, s_prev);
    double v2[2] = {1.0, 1.0}, t2[2];
    halo_release(flags, res_tag(launch, 0));
    {
        const int ex0[2] = {0, 0};
        limb_publish<2>(v2, ex0, lw, 1);
        limb_collect<2>(lw, 1, ex0, s_prev, t2);
    }
    for (int k = 0; k < iters; k++) {
        if constexpr (TILED) halo_acquire_list(flags, nbl, res_tag(launch, k));
        else halo_acquire(flags, blo, bhi, res_tag(launch, k));
        double v1[1] = {t2[0]}, t1[1];
        const int ex1[1] = {limb_exp(t2[0])};
        limb_publish<1>(v1, ex1, lw, 0);
        limb_collect<1>(lw, 0, ex1, s_prev, t1);
        double v3[2] = {t1[0], t2[1]};
        const int ex3[2] = {limb_exp(t1[0]), limb_exp(t2[1])};
        limb_publish<2>(v3, ex3, lw, 1);
        limb_collect<2>(lw, 1, ex3, s_prev, t2);
        if (k + 1 < iters) halo_release(flags, res_tag(launch, k + 1));
    }
    double v4[2] = {t2[0], t2[1]}, t4[2];
    reduce_publish<2, 0x2u>(v4, part0, res_tag(launch, 31));
    reduce_collect<2, 0x2u>(part0, res_tag(launch, 31), t4);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *reinterpret_cast<volatile unsigned*>(flags + (size_t)gridDim.x * RES_FLAG_STRIDE) = launch + 1;
}

}  // namespace hysco
