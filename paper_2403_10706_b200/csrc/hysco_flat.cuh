// hysco_flat.cuh — streaming Jacobi-PCG in two fused, vectorised launches per
// iteration (A5 + A6), for volumes whose PCG state does not fit on
// chip (HCP 7T, the 512x512x384 volume; fp64 builds).
//
// Layout: the node arrays are walked in FLAT node order t = (i n2 + j) P + l
// (not one warp per column): a thread owns V consecutive nodes (V = 4 fp32,
// 2 fp64: one 16-byte vector), so every own-array access is one aligned
// 128-bit load or store.  PE neighbours t-1 / t+1 come from the adjacent
// lanes' vectors (shuffles); the in-plane neighbours t +- P and t +- n2 P are
// 16-byte loads at a warp-uniform misalignment s (two aligned vectors and a
// uniform select; one when s = 0).  Each node group decomposes its flat index
// into (i, j, l) once (multiply-high division), for the Neumann flags (R3)
// and the Jacobi shift alpha hd diag(L_xy) (R13).
//
// Per PCG iteration k (52 B/node instead of 60 in three launches):
//   F1 pcg_dirmv_kernel:  p_k = z_k + beta_{k-1} p_{k-1}   (own node AND every
//                         stencil neighbour, formed from z and p_{k-1})
//                         x  += alpha_{k-1} p_{k-1}         (the update of the
//                         previous iteration, deferred here: p_{k-1} is read anyway)
//                         Hp = H p_k ;  p.Hp -> alpha_k      (decide_matvec)
//                         reads z, p_{k-1}, dt, et, x; writes p_k, Hp, x   (32 B/node)
//   F2 pcg_upd_kernel:    r -= alpha_k Hp ; z = r / M ; r.z, r.r -> beta_k,
//                         stop test (decide_update); reads r, Hp, M; writes r, z (20 B)
// (M = dt + alpha hd diag(L_xy) is formed once per GN step by the PCG start,
// so F2 is a pure stream.)
// p is double-buffered (neighbours of a CTA still read p_{k-1} while it
// writes p_k): p_k lives in buffer k & 1, the parity read from the pair's
// device state, so the same graph body serves the WHILE-loop form.  The last
// direction's update alpha p is folded into the Armijo start
// (trial_flat_kernel).  The arithmetic of every node is the same as in the
// three-kernel form (hysco_nodes.cuh); only where x += alpha p happens moves.
#pragma once

namespace hysco {

template <typename T> struct FlatVec;
template <> struct FlatVec<float> {
    static constexpr int V = 4;
    using type = float4;
    __device__ __forceinline__ static void ld(const float* p, float (&v)[4]) {
        const float4 a = *reinterpret_cast<const float4*>(p);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
    __device__ __forceinline__ static void st(float* p, const float (&v)[4]) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <> struct FlatVec<double> {
    static constexpr int V = 2;
    using type = double2;
    __device__ __forceinline__ static void ld(const double* p, double (&v)[2]) {
        const double2 a = *reinterpret_cast<const double2*>(p);
        v[0] = a.x; v[1] = a.y;
    }
    __device__ __forceinline__ static void st(double* p, const double (&v)[2]) {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    }
};

// Node buffers carry FLAT_GUARD elements of slack before and after (hysco_api.cu
// allocation): a node group that straddles a column or plane boundary may
// issue an in-plane neighbour vector load a few elements outside the pair
// whose values it masks.
constexpr int FLAT_GUARD = 32;

// n / d for 0 <= n < 2^31, d >= 1: ceil(2^p / d) with p = 31 + ceil(log2 d)
// and a 64-bit product (exact in that range; d = 1 included).
struct UDiv {
    unsigned long long m;
    int p;
    __device__ __forceinline__ void init(unsigned d) {
        int l = 0;
        while ((1ull << l) < d) l++;
        p = 31 + l;
        m = ((1ull << p) + d - 1) / d;
    }
    __device__ __forceinline__ int div(int n) const { return (int)(((unsigned long long)(unsigned)n * m) >> p); }
};

// Per-pair flat walk: group gi covers pair-relative nodes t0 .. t0 + V - 1,
// t0 = gi V - mis (mis = misalignment of the pair's first node).
struct FlatWalk {
    int mis, ngroups;
    int sj, si;            // (P mod V), (n2 P mod V): misalignment of the +P / +n2 P neighbours
    UDiv dP, dN2;
    __device__ __forceinline__ void init(const Geom& g, const void* pair0, int esz, int V) {
        mis = (int)(((uintptr_t)pair0 / esz) % V);
        ngroups = (int)((g.Nn + mis + V - 1) / V);
        sj = g.P % V;
        si = (int)(((long long)g.n2 * g.P) % V);
        dP.init((unsigned)g.P);
        dN2.init((unsigned)g.n2);
    }
};

// Column facts of the V nodes of a group (at most two columns: P >= V).
template <int V>
struct GroupCols {
    int l[V];             // position in the column (l < 0: node outside the pair)
    bool him[V], hip[V], hjm[V], hjp[V];
    float cmf[V];          // alpha hd diag(L_xy) (fp32 copy)
    double cmd[V];
};

template <int V>
__device__ __forceinline__ void group_cols(const Geom& g, const FlatWalk& w, long long t0, GroupCols<V>& gc,
                                           bool need_cm) {
    const long long tb = t0 < 0 ? 0 : t0;
    const int col0 = w.dP.div((int)tb);
    const int l0 = (int)(tb - (long long)col0 * g.P);
    const int i0 = w.dN2.div(col0), j0 = col0 - i0 * g.n2;
    // second column (col0 + 1)
    const int j1 = j0 + 1 == g.n2 ? 0 : j0 + 1, i1 = j0 + 1 == g.n2 ? i0 + 1 : i0;
    double cm0 = 0.0, cm1 = 0.0;
    if (need_cm) {
        cm0 = g.ahd * ((double)(has_im(g, i0) + has_ip(g, i0)) * g.ih1sq + (double)((j0 > 0) + (j0 < g.n2 - 1)) * g.ih2sq);
        cm1 = g.ahd * ((double)(has_im(g, i1) + has_ip(g, i1)) * g.ih1sq + (double)((j1 > 0) + (j1 < g.n2 - 1)) * g.ih2sq);
    }
#pragma unroll
    for (int m = 0; m < V; m++) {
        const long long t = t0 + m;
        const int lm = l0 + (int)(t - tb);
        const bool second = lm >= g.P;
        const bool in = t >= 0 && t < g.Nn;
        gc.l[m] = in ? (second ? lm - g.P : lm) : -1;
        const int i = second ? i1 : i0, j = second ? j1 : j0;
        gc.him[m] = in && has_im(g, i);
        gc.hip[m] = in && has_ip(g, i);
        gc.hjm[m] = in && j > 0;
        gc.hjp[m] = in && j < g.n2 - 1;
        gc.cmd[m] = second ? cm1 : cm0;
        gc.cmf[m] = (float)gc.cmd[m];
    }
}

template <typename T> __device__ __forceinline__ T cm_of(const GroupCols<FlatVec<T>::V>& gc, int m);
template <> __device__ __forceinline__ float cm_of<float>(const GroupCols<4>& gc, int m) { return gc.cmf[m]; }
template <> __device__ __forceinline__ double cm_of<double>(const GroupCols<2>& gc, int m) { return gc.cmd[m]; }

template <typename T>
__device__ __forceinline__ bool any_of(const bool (&f)[FlatVec<T>::V]) {
    bool a = false;
#pragma unroll
    for (int m = 0; m < FlatVec<T>::V; m++) a |= f[m];
    return a;
}

// PCG start (R14): x = 0, r = -grad, M = dt + alpha hd diag(L_xy) (stored once
// per GN step: the residual update then needs no column decomposition),
// z = r / M (the three-kernel form's rounding); r.z, r.r -> decide_pcg_init.
template <typename T>
__global__ void __launch_bounds__(256) pcg_init_flat_kernel(Geom g, Ctl c, const T* __restrict__ grad,
                                                            const T* __restrict__ dt, T* __restrict__ x,
                                                            T* __restrict__ r, T* __restrict__ z,
                                                            T* __restrict__ mdiag) {
    constexpr int V = FlatVec<T>::V;
    count_launch(c);
    const int pair = blockIdx.y;
    const bool active = pcg_step_active(c.st[pair]);
    const size_t po = (size_t)pair * g.ps;
    double arz = 0, arr = 0;
    if (active) {
        FlatWalk w;
        w.init(g, grad + po, sizeof(T), V);
        const T* gb = grad + po - w.mis;   // aligned group bases
        const T* db = dt + po - w.mis;
        T* xb = x + po - w.mis;
        T* rb = r + po - w.mis;
        T* zb = z + po - w.mis;
        T* mb = mdiag + po - w.mis;
        for (int gi = blockIdx.x * blockDim.x + threadIdx.x; gi < w.ngroups; gi += gridDim.x * blockDim.x) {
            const long long t0 = (long long)gi * V - w.mis;
            GroupCols<V> gc;
            group_cols<V>(g, w, t0, gc, true);
            T gv[V], dv[V], xo[V], ro[V], zo[V], mo[V];
            FlatVec<T>::ld(gb + (size_t)gi * V, gv);
            FlatVec<T>::ld(db + (size_t)gi * V, dv);
            const bool full = gc.l[0] >= 0 && gc.l[V - 1] >= 0;
#pragma unroll
            for (int m = 0; m < V; m++) {
                const bool ok = gc.l[m] >= 0;
                const T rv = ok ? -gv[m] : T(0);
                const T mi = ok ? dv[m] + cm_of<T>(gc, m) : T(1);
                const T zz = rv / mi;
                xo[m] = T(0);
                ro[m] = rv;
                zo[m] = zz;
                mo[m] = mi;
                arz += (double)rv * (double)zz;
                arr += (double)rv * (double)rv;
            }
            if (full) {
                FlatVec<T>::st(xb + (size_t)gi * V, xo);
                FlatVec<T>::st(rb + (size_t)gi * V, ro);
                FlatVec<T>::st(zb + (size_t)gi * V, zo);
                FlatVec<T>::st(mb + (size_t)gi * V, mo);
            } else {
#pragma unroll
                for (int m = 0; m < V; m++)
                    if (gc.l[m] >= 0) {
                        xb[(size_t)gi * V + m] = xo[m];
                        rb[(size_t)gi * V + m] = ro[m];
                        zb[(size_t)gi * V + m] = zo[m];
                        mb[(size_t)gi * V + m] = mo[m];
                    }
            }
        }
    }
    double v[2] = {arz, arr}, tot[2];
    if (!pair_reduce<2, 0u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {                       // slab: OP_PCG_INIT after the allreduce
        store_red(c, pair, gridDim.y, tot, 2, 0);
        return;
    }
    decide_pcg_init(c.st[pair], tot);
    if (last_pair(c)) set_cond(c, COND_PCG, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->pcg_active != 0; }));
}

// F1 as a plane march (2.5-D blocking) fed by bulk asynchronous copies.
// On B200 an L2 re-read costs about as much as an HBM read (a flat walk that
// fetches the in-plane neighbours itself pushed ~75 B per node through L2 for
// 32 B of HBM traffic and ran at 2.4 TB/s), so every value reaches a CTA
// once.  A CTA owns the columns [ja, jb) of a chunk of planes [ia, ib) and
// marches along dim 1.  For every plane q a stage of shared memory receives,
// by cp.async.bulk (the TMA engine; completion on an mbarrier, no registers,
// no thread issue):
//   z and p_{k-1} of the columns [ja - 1, jb]  (own + one halo column each side)
//   dt, et, x of the own columns                (own planes only)
// NST stages form a ring (three planes in use, the rest in flight); computing
// plane s reads all seven stencil values of p_k = z + beta p_{k-1} from the
// planes s-1, s, s+1, writes Hp, p_k and x += alpha_{k-1} p_{k-1} for its own
// nodes and reduces p.Hp.  Halo planes / columns are re-read from L2 by the
// neighbouring CTAs only ((C + 2) / C and (W + 2) / W of z and p_{k-1}).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MBW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MBW_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (16-byte aligned ends, bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Per-thread 16-byte asynchronous copies (LDGSTS) with completion on an
// mbarrier: every thread copies its share of a window and arrives once
// (.noinc: the barrier expects one arrival per thread).  The alternative to
// one bulk copy per window (HYSCO_MARCH_BULK); measured slower (7T march
// 2.5 vs 3.5 TB/s, C5 3.1 vs 4.0 TB/s), kept for the A/B.
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_arrive(unsigned long long* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// a window of `bytes` (multiple of 16) by all NT threads of the CTA
__device__ __forceinline__ void cp_window(void* dst, const void* src, unsigned bytes, int tid, int nt) {
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    for (unsigned i = (unsigned)tid * 16u; i < bytes; i += (unsigned)nt * 16u) cp16(d + i, s + i);
}
#ifndef HYSCO_MARCH_BULK
#define HYSCO_MARCH_BULK 1   // 0: per-thread 16-byte cp.async (measured slower: 7T 2.5 vs 3.5 TB/s)
#endif

// Shared-memory plan of one march stage (elements of T): [z | p_old] windows
// of LA, [dt | et | x] windows of LB, each a multiple of 16 bytes.
struct MarchPlan {
    int la, lb, nst, ms;
};
template <typename T>
__host__ __device__ inline MarchPlan march_plan(int wmax, int P, int nst) {
    const int q = 16 / (int)sizeof(T);
    MarchPlan m;
    m.la = (((wmax + 2) * P + q) + q - 1) / q * q;
    m.lb = ((wmax * P + 1 + q) + q - 1) / q * q;
    m.nst = nst;
    return m;
}
// Node slots per thread of pcg_march_kernel for tiles of wmax columns: the
// smallest instantiated MS with wmax P <= MS NT and (wmax + 2) P + Q <= (MS + 2) NT
// (0: none fits).
template <typename T>
inline int march_ms(int wmax, int P, int nt) {
    const int q = 16 / (int)sizeof(T);
    for (int ms : {2, 4, 8, 12})
        if (wmax * P <= ms * nt && (wmax + 2) * P + q <= (ms + 2) * nt) return ms;
    return 0;
}
template <typename T>
__host__ __device__ inline size_t march_stage_bytes(const MarchPlan& m) {
    return (size_t)(2 * m.la + 3 * m.lb) * sizeof(T);
}
template <typename T>
__host__ __device__ inline size_t march_smem_bytes(const MarchPlan& m) {
    return march_stage_bytes<T>(m) * m.nst + 16 * 8;   // + the stage barriers
}

#ifndef HYSCO_MARCH_CPS
#define HYSCO_MARCH_CPS 1   // march CTAs per SM (each with 1 / CPS of the shared memory and threads)
#endif
constexpr int MARCH_CPS = HYSCO_MARCH_CPS;
constexpr int MARCH_THREADS = 512 / MARCH_CPS;   // CPS = 1: one CTA per SM (shared memory), 16 warps

// FIRST (k = 0): p_0 = z, no p_{-1}, no x update.  MS: node slots per thread
// (the tile's own nodes of one plane, (jb - ja) P <= MS * MARCH_THREADS); every
// thread keeps the same nodes in every plane, so their offsets and Neumann
// flags are computed once, and the MS independent nodes of a slot loop give
// the two warps per scheduler instruction-level parallelism.
// fuse_up (slab path, defer mode, fixed counts): the previous residual
// update's decision (decide_update on the allreduced r.z, r.r in c.red) is
// not a separate decide_kernel launch: every CTA derives k, beta and the
// active flag from the pre-decision state and the totals, and the last CTA
// commits decide_update before it stores this launch's own partial totals.
template <typename T, bool FIRST, int MS>
__global__ void __launch_bounds__(MARCH_THREADS, MARCH_CPS) pcg_march_kernel(Geom g, Ctl c, int nJB, int C, MarchPlan mp,
                                                                     const T* __restrict__ dt,
                                                                     const T* __restrict__ et,
                                                                     const T* __restrict__ z, T* __restrict__ pbuf0,
                                                                     T* __restrict__ pbuf1, T* __restrict__ Hp,
                                                                     T* __restrict__ x, int fuse_up = 0,
                                                                     SolveParams sp = SolveParams{}) {
    extern __shared__ __align__(128) unsigned char march_raw[];
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(march_raw);
    T* stage0 = reinterpret_cast<T*>(march_raw + 16 * 8);
    count_launch(c);
    constexpr int NT = MARCH_THREADS;
    const int tid = threadIdx.x;
    const int pair = blockIdx.y;
    const PairState& st = c.st[pair];
    double acc = 0;
    const int bj = blockIdx.x % nJB, bc = blockIdx.x / nJB;
    const int n1 = g.n1, n2 = g.n2, P = g.P;
    const int ia = bc * C, ib = min(ia + C, n1);
    // the decision this launch starts from: committed state, or (fuse_up)
    // decide_update applied locally to the allreduced totals
    bool pact = st.pcg_active != 0;
    int kk = st.pcg_k;
    double bet = st.beta_c;
    const double* upd_tot = c.red + (size_t)pair * RED_W;
    if (fuse_up && pact) {
        kk = st.pcg_k + 1;
        bet = upd_tot[0] / st.rz;
        const double relres = sqrt(upd_tot[1] / st.rr0);
        pact = !(kk >= sp.max_pcg || (!sp.fixed && relres < sp.pcg_rtol));
    }
    // a launch of the other FIRST variant for this iteration parity does nothing
    if (pact && ia < n1 && ((kk == 0) == FIRST)) {
        const int k = kk;
        const T be = FIRST ? T(0) : (T)bet, ap = (T)st.alpha_c;
        const size_t po = (size_t)pair * g.ps;
        T* __restrict__ pnew = ((k & 1) ? pbuf1 : pbuf0) + po;
        const T* __restrict__ pold = ((k & 1) ? pbuf0 : pbuf1) + po;
        const T* __restrict__ zp = z + po;
        T* __restrict__ xp = x + po;
        T* __restrict__ hp = Hp + po;
        const int ja = (int)((long long)bj * n2 / nJB), jb = (int)((long long)(bj + 1) * n2 / nJB);
        const int jl = ja > 0 ? ja - 1 : 0, jh = jb < n2 ? jb : n2 - 1;   // window columns (inclusive)
        const int nown = (jb - ja) * P, nwin = (jh - jl + 1) * P;
        const int SE = 2 * mp.la + 3 * mp.lb;                             // stage pitch (elements)
        constexpr int Q = 16 / (int)sizeof(T);
        // planes loaded: [q0, qend); on a slab the halo planes -1 / n1 (exchanged
        // copies of the neighbouring ranks' boundary planes) where they exist
        const int q0 = ia > 0 ? ia - 1 : (has_im(g, 0) ? -1 : 0);
        const int qend = ib < n1 ? ib + 1 : (has_ip(g, n1 - 1) ? n1 + 1 : n1);
        // misalignment (elements below a 16-byte boundary) of plane q's windows:
        // (mis(0) + q (n2 P mod Q)) mod Q
        const long long plane = (long long)n2 * P;
        const int dq = (int)(plane % Q);
        const int mA0 = (int)(((uintptr_t)(zp + (size_t)jl * P) / sizeof(T)) % Q);
        const int mB0 = (int)(((uintptr_t)(zp + (size_t)ja * P - 1) / sizeof(T)) % Q);
        auto misA = [&](int q) { return ((mA0 + q * dq) % Q + Q) % Q; };
        auto misB = [&](int q) { return ((mB0 + q * dq) % Q + Q) % Q; };
        // the stage of plane q (called by every thread; bulk mode: thread 0 issues)
        auto issue = [&](int q) {
            const int s = (q - q0) % mp.nst;
            T* S = stage0 + (size_t)s * SE;
            const int dA = misA(q), dB = misB(q);
            const long long gA = (long long)q * plane + (long long)jl * P - dA;
            const long long gB = (long long)q * plane + (long long)ja * P - 1 - dB;
            const unsigned bA = (unsigned)(((nwin + dA) + Q - 1) / Q * 16);
            const unsigned bB = (unsigned)(((nown + 1 + dB) + Q - 1) / Q * 16);
            const bool own = q >= ia && q < ib;
#if HYSCO_MARCH_BULK
            if (tid != 0) return;
            const unsigned tot = bA * (FIRST ? 1u : 2u) + (own ? bB * (FIRST ? 2u : 3u) : 0u);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bars[s], tot);
            bulk_g2s(S, zp + gA, bA, &bars[s]);
            if (!FIRST) bulk_g2s(S + mp.la, pold + gA, bA, &bars[s]);
            if (own) {
                bulk_g2s(S + 2 * mp.la, dt + po + gB, bB, &bars[s]);
                bulk_g2s(S + 2 * mp.la + mp.lb, et + po + gB, bB, &bars[s]);
                if (!FIRST) bulk_g2s(S + 2 * mp.la + 2 * mp.lb, xp + gB, bB, &bars[s]);
            }
#else
            cp_window(S, zp + gA, bA, tid, NT);
            if (!FIRST) cp_window(S + mp.la, pold + gA, bA, tid, NT);
            if (own) {
                cp_window(S + 2 * mp.la, dt + po + gB, bB, tid, NT);
                cp_window(S + 2 * mp.la + mp.lb, et + po + gB, bB, tid, NT);
                if (!FIRST) cp_window(S + 2 * mp.la + 2 * mp.lb, xp + gB, bB, tid, NT);
            }
            cp_arrive(&bars[s]);
#endif
        };
        auto ready = [&](int q) {
            const int u = q - q0;
            mbar_wait(&bars[u % mp.nst], (unsigned)((u / mp.nst) & 1));
        };
        auto stage = [&](int q) { return stage0 + (size_t)((q - q0) % mp.nst) * SE; };
        // in place: window A's z slot becomes p_k = z + beta p_{k-1} (the p_{k-1}
        // slot is kept for the x update)
        constexpr int MW = MS + 2;   // window slots: (W + 2) P + Q <= (MS + 2) NT (host plan, march_ms)
        auto convert = [&](int q) {
            if (FIRST) return;
            T* S = stage(q);
            const int n = nwin + misA(q);
#pragma unroll
            for (int m = 0; m < MW; m++) {
                const int i = tid + m * NT;
                if (i < n) S[i] = fma(be, S[mp.la + i], S[i]);
            }
        };
        // this thread's nodes: e = tid + m NT of the tile (column cj = e / P, l = e mod P)
        int eo[MS];
        unsigned long long fl = 0;   // per slot 5 bits: valid, l > 0, l < n3, j-1, j+1 exist
#pragma unroll
        for (int m = 0; m < MS; m++) {
            const int e = tid + m * NT;
            const int cj = e / P, l = e - cj * P, j = ja + cj;
            eo[m] = e;
            if (e < nown) {
                const unsigned long long f =
                    1u | (l > 0 ? 2u : 0u) | (l < g.n3 ? 4u : 0u) | (j > 0 ? 8u : 0u) | (j < n2 - 1 ? 16u : 0u);
                fl |= f << (5 * m);   // MS <= 12: 60 bits
            }
        }
        if (tid == 0) {
            for (int s = 0; s < mp.nst; s++) mbar_init(&bars[s], HYSCO_MARCH_BULK ? 1 : NT);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        for (int q = q0; q < qend && q < q0 + mp.nst; q++) issue(q);
        for (int q = q0; q <= ia; q++) {   // prologue: planes q0 .. ia converted
            ready(q);
            convert(q);
        }
        const T ahd = gw<T>(g.ahd, g.f_ahd), ih1sq = gw<T>(g.ih1sq, g.f_ih1sq), ih2sq = gw<T>(g.ih2sq, g.f_ih2sq);
        const int base = (ja - jl) * P;
        for (int s = ia; s < ib; s++) {
            if (s + 1 < qend) {
                ready(s + 1);
                convert(s + 1);
            }
            __syncthreads();   // p of planes s-1, s, s+1 in place
            const bool him = has_im(g, s), hip = has_ip(g, s);
            const T* Sc = stage(s);
            const T* Pc = Sc + base + misA(s);
            const T* Pm = him ? stage(s - 1) + base + misA(s - 1) : Pc;
            const T* Pp = hip ? stage(s + 1) + base + misA(s + 1) : Pc;
            const T* DT = Sc + 2 * mp.la + 1 + misB(s);
            const T* ET = DT + mp.lb;
            const T* XS = ET + mp.lb;
            const T* PO = Pc + mp.la;                    // p_{k-1}
            const size_t go = (size_t)s * plane + (size_t)ja * P;
            T* hs = hp + go;
            T* ps = pnew + go;
            T* xs = xp + go;
#pragma unroll
            for (int m = 0; m < MS; m++) {
                const unsigned f = (unsigned)(fl >> (5 * m));
                if (f & 1u) {
                    const int e = eo[m];
                    const T pc = Pc[e];
                    // absent j-neighbours read the node itself (never outside the stage)
                    const T pl = Pc[e - 1], pr = Pc[e + 1];
                    const T pjm = Pc[(f & 8u) ? e - P : e], pjp = Pc[(f & 16u) ? e + P : e];
                    const T pim = Pm[e], pip = Pp[e];
                    const T em = ET[e - 1], ev = ET[e];
                    T h = DT[e] * pc;
                    if (f & 2u) h += em * pl;
                    if (f & 4u) h += ev * pr;
                    const T l1 = (him ? pc - pim : T(0)) + (hip ? pc - pip : T(0));
                    const T l2 = ((f & 8u) ? pc - pjm : T(0)) + ((f & 16u) ? pc - pjp : T(0));
                    h += ahd * (l1 * ih1sq + l2 * ih2sq);
                    hs[e] = h;
                    ps[e] = pc;
                    if (!FIRST) xs[e] = XS[e] + ap * PO[e];
                    acc += (double)pc * (double)h;
                }
            }
            __syncthreads();   // plane s-1's stage is free (last read in this step)
            if (s - 1 >= q0 && s - 1 + mp.nst < qend) issue(s - 1 + mp.nst);
        }
    }
    double v[1] = {acc}, tot[1];
    if (!pair_reduce<1, 0u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (fuse_up) {                       // every CTA has read the totals: commit their decision
        double ut[2] = {upd_tot[0], upd_tot[1]};
        decide_update(sp, c.st[pair], ut);
    }
    if (c.defer) {                       // slab: OP_MATVEC after the allreduce
        store_red(c, pair, gridDim.y, tot, 1, 0);
        return;
    }
    decide_matvec(c.st[pair], tot);
}

// F2: r -= alpha Hp, z = r / M; r.z, r.r -> beta, stop test.  Pure streaming
// (M from pcg_init_flat_kernel): 20 B per node.
// fuse_mv (slab path, defer mode): the march's decision (decide_matvec on the
// allreduced p.Hp) applied locally by every block, committed by the last.
template <typename T>
__global__ void __launch_bounds__(256) pcg_upd_kernel(Geom g, Ctl c, SolveParams sp, const T* __restrict__ mdiag,
                                                      const T* __restrict__ Hp, T* __restrict__ r,
                                                      T* __restrict__ z, int fuse_mv = 0) {
    constexpr int V = FlatVec<T>::V;
    count_launch(c);
    const int pair = blockIdx.y;
    bool active = c.st[pair].pcg_active != 0;
    double al = c.st[pair].alpha_c;
    const double mv_tot = fuse_mv ? c.red[(size_t)pair * RED_W] : 0.0;
    if (fuse_mv && active) {
        if (mv_tot <= 0.0) {             // breakdown (decide_matvec)
            active = false;
            al = 0.0;
        } else {
            al = c.st[pair].rz / mv_tot;
        }
    }
    const T a = (T)al;
    const size_t po = (size_t)pair * g.ps;
    double arz = 0, arr = 0;
    if (active) {
        const int mis = (int)(((uintptr_t)(r + po) / sizeof(T)) % V);
        const int ngroups = (int)((g.Nn + mis + V - 1) / V);
        const T* mb = mdiag + po - mis;
        const T* hb = Hp + po - mis;
        T* rb = r + po - mis;
        T* zb = z + po - mis;
        for (int gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ngroups; gi += gridDim.x * blockDim.x) {
            const long long t0 = (long long)gi * V - mis;
            T rv[V], hv[V], mv[V], ro[V], zo[V];
            FlatVec<T>::ld(rb + (size_t)gi * V, rv);
            FlatVec<T>::ld(hb + (size_t)gi * V, hv);
            FlatVec<T>::ld(mb + (size_t)gi * V, mv);
            const bool full = t0 >= 0 && t0 + V <= g.Nn;
#pragma unroll
            for (int m = 0; m < V; m++) {
                const T rn = rv[m] - a * hv[m];
                const T zz = rn / mv[m];
                ro[m] = rn;
                zo[m] = zz;
                if (full || (t0 + m >= 0 && t0 + m < g.Nn)) {
                    arz += (double)rn * (double)zz;
                    arr += (double)rn * (double)rn;
                }
            }
            if (full) {
                FlatVec<T>::st(rb + (size_t)gi * V, ro);
                FlatVec<T>::st(zb + (size_t)gi * V, zo);
            } else {
#pragma unroll
                for (int m = 0; m < V; m++)
                    if (t0 + m >= 0 && t0 + m < g.Nn) {
                        rb[(size_t)gi * V + m] = ro[m];
                        zb[(size_t)gi * V + m] = zo[m];
                    }
            }
        }
    }
    double v[2] = {arz, arr}, tot[2];
    if (!pair_reduce<2, 0u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (fuse_mv) {                       // every block has read the totals: commit their decision
        double mt[1] = {mv_tot};
        decide_matvec(c.st[pair], mt);
    }
    if (c.defer) {                       // slab: OP_UPDATE after the allreduce
        store_red(c, pair, gridDim.y, tot, 2, 0);
        return;
    }
    decide_update(sp, c.st[pair], tot);
    if (last_pair(c)) set_cond(c, COND_PCG, any_pair(c, gridDim.y, [](volatile PairState* q) { return q->pcg_active != 0; }));
}

// Armijo start (A7, R15) after a flat PCG: q = x + alpha p (the last
// direction's deferred update; alpha = 0 after a breakdown or when no
// iteration ran), x = q, b_old = b, b = b + q; g.q, max|q| -> decide_trial.
template <typename T>
__global__ void __launch_bounds__(256) trial_flat_kernel(Geom g, Ctl c, const T* __restrict__ grad,
                                                         T* __restrict__ x, const T* __restrict__ pbuf0,
                                                         const T* __restrict__ pbuf1, T* __restrict__ b,
                                                         T* __restrict__ bold) {
    constexpr int V = FlatVec<T>::V;
    count_launch(c);
    const int pair = blockIdx.y;
    const PairState& st = c.st[pair];
    const bool active = pcg_step_active(st);
    double agq = 0, aqm = 0;
    if (active) {
        const T ap = (T)st.alpha_c;
        const bool addp = st.alpha_c != 0.0;
        const T* pl = ((st.pcg_k - 1) & 1) ? pbuf1 : pbuf0;   // buffer of the last direction
        const size_t po = (size_t)pair * g.ps;
        FlatWalk w;
        w.init(g, x + po, sizeof(T), V);
        const T* gb = grad + po - w.mis;
        const T* plb = pl + po - w.mis;
        T* xb = x + po - w.mis;
        T* bb = b + po - w.mis;
        T* ob = bold + po - w.mis;
        for (int gi = blockIdx.x * blockDim.x + threadIdx.x; gi < w.ngroups; gi += gridDim.x * blockDim.x) {
            const long long t0 = (long long)gi * V - w.mis;
            bool okm[V];
            bool full = true;
#pragma unroll
            for (int m = 0; m < V; m++) {
                okm[m] = t0 + m >= 0 && t0 + m < g.Nn;
                full &= okm[m];
            }
            T gv[V], xv[V], bv[V], qv[V], bn[V];
            FlatVec<T>::ld(gb + (size_t)gi * V, gv);
            FlatVec<T>::ld(xb + (size_t)gi * V, xv);
            FlatVec<T>::ld(bb + (size_t)gi * V, bv);
            if (addp) {
                T pv[V];
                FlatVec<T>::ld(plb + (size_t)gi * V, pv);
#pragma unroll
                for (int m = 0; m < V; m++) qv[m] = xv[m] + ap * pv[m];
            } else {
#pragma unroll
                for (int m = 0; m < V; m++) qv[m] = xv[m];
            }
#pragma unroll
            for (int m = 0; m < V; m++) {
                bn[m] = bv[m] + qv[m];
                if (okm[m]) {
                    agq += (double)gv[m] * (double)qv[m];
                    aqm = fmax(aqm, (double)fabs(qv[m]));
                }
            }
            if (full) {
                FlatVec<T>::st(xb + (size_t)gi * V, qv);
                FlatVec<T>::st(ob + (size_t)gi * V, bv);
                FlatVec<T>::st(bb + (size_t)gi * V, bn);
            } else {
#pragma unroll
                for (int m = 0; m < V; m++)
                    if (okm[m]) {
                        xb[(size_t)gi * V + m] = qv[m];
                        ob[(size_t)gi * V + m] = bv[m];
                        bb[(size_t)gi * V + m] = bn[m];
                    }
            }
        }
    }
    double v[2] = {agq, aqm}, tot[2];
    if (!pair_reduce<2, 0x2u>(c, v, tot)) return;
    if (threadIdx.x != 0) return;
    if (c.defer) {                       // slab: OP_TRIAL after the allreduce
        store_red(c, pair, gridDim.y, tot, 1, 1);
        return;
    }
    decide_trial(c.st[pair], tot);
    if (last_pair(c)) set_cond(c, COND_LS, any_pair(c, gridDim.y, [](volatile PairState* q2) { return q2->ls_active != 0; }));
}

}  // namespace hysco
