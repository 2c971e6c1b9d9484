// hysco_api.cu — C ABI of libhysco.so (declared in include/hysco.h).
//
// Host side: context, memory plan (all scratch allocated at create), and the
// orchestration of the GN-PCG solve as ONE CUDA graph whose
// Gauss-Newton, PCG and Armijo loops are device-side conditional WHILE nodes
// (no host synchronisation inside a solve).  A host-loop fallback with the
// same kernels exists for drivers without conditional nodes (HYSCO_NO_GRAPH=1
// forces it).
#include "hysco.h"
#include "hysco_io.h"
#include "hysco_kernels.cuh"

#include <nccl.h>
#include <cufft.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

using namespace hysco;

// NVTX range around each public entry point (visible to nsys / ncu range
// filters; no cost without an attached tool).
struct NvtxRange {
    explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
    ~NvtxRange() { nvtxRangePop(); }
};

namespace {

// B_W, B_F: factors of the block preconditioner (R20); B_TMP also holds its z during a solve
enum { B_B = 0, B_BOLD, B_GRAD, B_DT, B_ET, B_X, B_R, B_P, B_HP, B_TMP, B_W, B_F, NBUF };

struct GraphKey {
    int kind;                 // 1 = solve, 2 = correct
    SolveParams sp;
    int blur;
    const void* ptr[8];
};

}  // namespace

struct hysco_ctx_s {
    hysco_config cfg{};
    Geom g{};
    int nsm = 0;
    size_t esz = 4;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    const void* Ip = nullptr;
    const void* Im = nullptr;
    void* buf[NBUF] = {};
    void* raw[NBUF] = {};     // allocations: buf[k] = raw[k] + FLAT_GUARD elements (hysco_flat.cuh)
    void* own_Ip = nullptr;   // host-entry image copies
    void* own_Im = nullptr;
    void* own_Tp = nullptr;   // host-entry corrected images
    // hysco_correct_host_stream: copy stream, 2 staging slots each way, events
    cudaStream_t copy_stream = nullptr;
    void* st_in[2][2] = {};       // [slot][I+, I-]
    void* st_out[2][3] = {};      // [slot][b, T+, T-]
    cudaEvent_t ev_h2d[2] = {}, ev_in_free[2] = {}, ev_out[2] = {}, ev_out_free[2] = {};
    bool stream_ready = false;
    // hysco_admm: cuFFT plans (R2C / C2R over (n1, n2), batch P), spectrum, rho / factors
    cufftHandle fft_fwd = 0, fft_inv = 0;
    void* admm_spec = nullptr;
    double* admm_rho = nullptr;     // [batch] device
    double* admm_fac = nullptr;     // [batch] device (u rescaling)
    double* admm_lam = nullptr;     // [n1][n2/2+1] periodic L_xy eigenvalues
    double* admm_stat = nullptr;    // [batch][4] iterations, r_norm, s_norm, converged (device)
    unsigned* admm_done = nullptr;  // device stop flags of the running ADMM solve: [0] all, [1 + p] pair p
    unsigned* h_admm_done = nullptr;                // [2] pinned copies of the flag
    cudaEvent_t admm_ev[2] = {nullptr, nullptr};    // recorded after each copy
    size_t admm_smem = 0;
    int admm_gx = 1;
    int admm_e = 0;                 // admm_b_kernel register-PCR width ceil(P / 32), 0 = shared-memory PCR
    bool admm_ready = false;
    struct AdmmSlab* admm_slab = nullptr;   // slab ADMM (transposed z-update), admm_slab_run
    void* own_Tm = nullptr;
    PairState* st = nullptr;
    PairState* h_st = nullptr;          // pinned mirror
    double* part = nullptr;
    unsigned* ctr = nullptr;
    unsigned* gctr = nullptr;
    unsigned long long* launches = nullptr;
    unsigned long long* h_launches = nullptr;
    // hysco_correct_host_stream: per-item pinned readback slots; while set,
    // run_path copies the final PairState / launch count there asynchronously
    // and returns without synchronising (the items then run back to back)
    PairState* defer_st = nullptr;
    unsigned long long* defer_launch = nullptr;
    PairState* h_items = nullptr;
    unsigned long long* h_items_l = nullptr;
    PairState* d_items = nullptr;              // device snapshots (one kernel per item, read once at the end)
    unsigned long long* d_items_l = nullptr;
    long long h_items_cap = 0;
    unsigned* dcond = nullptr;
    unsigned* h_cond = nullptr;
    Ctl ctl{};
    int gx_nodes = 1, gx_mv = 1, gx_cells = 1, gx_eval = 1, gx_apply = 1, gx_ot = 1, gx_flat = 1, gx_dmv = 1;
    // streaming PCG in the flat vectorised two-launch form (hysco_flat.cuh);
    // single-context paths with P >= the vector width (HYSCO_NO_FLAT=1: three-kernel form)
    bool flat = false;
    int mr_njb = 1, mr_c = 1;   // plane-march F1 tiling (pcg_march_kernel)
    MarchPlan mr_plan{};
    size_t smem_mr = 0;
    // launch view (PairView): the launchers address pairs [vp, vp + vb); the
    // resident path runs a batch pair by pair (one pair's arrays stay in L2
    // across its whole GN loop) with vb = 1 and the one-pair grids gx1
    int vb = 1;
    size_t vp = 0;
    bool vshare = false;
    bool last_per_pair = false;   // the last solve ran pair by pair on shared scratch
    int gx1[8] = {1, 1, 1, 1, 1, 1, 1, 1};
    int nch = 5;              // 32-node chunks per column segment of the node kernels
    size_t smem_eval = 0, smem_ot = 0, smem_apply = 0;
    bool state_valid = false;
    bool poisoned = false;
    bool no_graph = false;
    bool graph_broken = false;
    std::string err;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    GraphKey key{};
    bool have_key = false;
    // a second cached graph (hysco_correct_host_stream alternates two staging
    // slots, i.e. two pointer sets): swapped with the current one on a hit
    cudaGraph_t graph2 = nullptr;
    cudaGraphExec_t exec2 = nullptr;
    GraphKey key2{};
    bool have_key2 = false;
    long long last_launches = 0;
    void* flush = nullptr;    // profiling-only L2 flush scratch
    // on-chip-resident PCG (hysco_resident.cuh): fp32, one CTA per SM
    bool resident = false;
    int res_k = 0, res_grid = 0;
    bool res_tiled = false;      // 2-D tiles of columns per CTA (hysco_resident.cuh ResTile)
    ResTile res_tile{0, 0, 0, 0};
    size_t res_smem = 0;
    double* res_part = nullptr;
    unsigned* res_flags = nullptr;   // p-halo flags + launch counter (hysco_resident.cuh)
    float* res_pg = nullptr;     // ghost-padded global copy of p (halo source)
    float* res_x = nullptr;      // x of one pair in the padded resident layout
    float res_wi = 0.f, res_wj = 0.f;   // alpha hd / h1^2, alpha hd / h2^2 (in-plane Laplacian weights)
    // persistent L2-resident PCG (hysco_l2pcg.cuh): one CTA per SM, shares res_part / res_flags
    bool l2pcg = false;
    int l2_grid = 0;
    // slab decomposition (multi-rank)
    size_t plane_off = 0;        // elements from a pair's buffer start to local plane 0
    int rank = 0, nranks = 1;
    double* red = nullptr;       // [2][batch][RED_W] pair totals for the allreduce
    HistRec* hist = nullptr;     // [batch][HIST_MAX] per-GN-step history (hysco_history)
    struct CommBase* comm = nullptr;
    // slab path: recorded graph segments (run_slab_path) and the call shape they belong to
    std::vector<cudaGraphExec_t> seg_exec;
    std::vector<const void*> seg_key;
    SolveParams seg_sp{};
    bool seg_valid = false;
};

static hysco_status set_err(hysco_ctx c, hysco_status s, const std::string& m) {
    if (c) c->err = m;
    return s;
}

static hysco_status cuda_fail(hysco_ctx c, cudaError_t e, const char* what, int line) {
    char b[512];
    snprintf(b, sizeof b, "CUDA error %d (%s) at %s [hysco_api.cu:%d]", (int)e, cudaGetErrorString(e), what, line);
    cudaGetLastError();
    if (c) {
        c->poisoned = true;
        c->err = b;
    }
    return HYSCO_ERR_CUDA;
}

#define CK(call)                                                             \
    do {                                                                     \
        cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call, __LINE__);   \
    } while (0)

#define CK_C(c_, call)                                                        \
    do {                                                                      \
        cudaError_t e_ = (call);                                              \
        if (e_ != cudaSuccess) return cuda_fail((c_), e_, #call, __LINE__);   \
    } while (0)

#define CHECK_CTX()                                                                          \
    do {                                                                                     \
        if (!ctx) return HYSCO_ERR_ARG;                                                      \
        if (ctx->poisoned) return HYSCO_ERR_CUDA;                                            \
        cudaError_t e0_ = cudaSetDevice(ctx->cfg.device);                                    \
        if (e0_ != cudaSuccess) return cuda_fail(ctx, e0_, "cudaSetDevice", __LINE__);       \
    } while (0)

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
static bool getenv_is1(const char* n) {
    const char* e = getenv(n);
    return e && e[0] == '1';
}

static SolveParams to_params(const hysco_solve_opts& o, const hysco_ot_opts& t) {
    SolveParams s{};
    s.max_gn = o.max_gn;
    s.max_pcg = o.max_pcg;
    s.fixed = o.fixed_iters ? 1 : 0;
    s.ls_max = o.ls_max;
    s.pcg_rtol = o.pcg_rtol;
    s.c1 = o.armijo_c1;
    s.tol_grad_rel = o.tol_grad_rel;
    s.tol_dJ_rel = o.tol_dJ_rel;
    s.tol_db_rel = o.tol_db_rel;
    s.armijo = o.armijo ? 1 : 0;
    s.precond = o.precond;
    s.feas_cap = t.feas_cap;
    s.ot_eps = t.eps;
    return s;
}

static hysco_status check_opts(hysco_ctx ctx, const hysco_solve_opts& o, const hysco_ot_opts& t) {
    if (o.max_gn < 0 || o.max_pcg < 1 || o.ls_max < 1 || !(o.pcg_rtol >= 0) || !(o.armijo_c1 >= 0))
        return set_err(ctx, HYSCO_ERR_ARG, "bad hysco_solve_opts");
    if (!(t.eps >= 0) || !(t.feas_cap > 0)) return set_err(ctx, HYSCO_ERR_ARG, "bad hysco_ot_opts");
    if (o.precond != HYSCO_PRECOND_JACOBI && o.precond != HYSCO_PRECOND_PE_BLOCK)
        return set_err(ctx, HYSCO_ERR_ARG, "bad hysco_solve_opts.precond");
    return HYSCO_OK;
}

// ---------------------------------------------------------------------------
// Kernel launchers (typed)
// ---------------------------------------------------------------------------
// Node kernels take the number of 32-node chunks per column segment (NCH) as a
// compile-time parameter; pick_nch() chooses it from P = n3+1.
#define NCH_SWITCH(nch, ...)                      \
    switch (nch) {                                \
        case 2: {                                 \
            constexpr int NCH = 2;                \
            __VA_ARGS__;                          \
        } break;                                  \
        case 4: {                                 \
            constexpr int NCH = 4;                \
            __VA_ARGS__;                          \
        } break;                                  \
        case 5: {                                 \
            constexpr int NCH = 5;                \
            __VA_ARGS__;                          \
        } break;                                  \
        case 7: {                                 \
            constexpr int NCH = 7;                \
            __VA_ARGS__;                          \
        } break;                                  \
        default: {                                \
            constexpr int NCH = 8;                \
            __VA_ARGS__;                          \
        } break;                                  \
    }

static int pick_nch(int P) { return P <= 64 ? 2 : P <= 128 ? 4 : P <= 160 ? 5 : P <= 224 ? 7 : 8; }

template <typename T>
struct L {
    // per-pair view: b is the pair's own; the scratch arrays are pair 0's,
    // shared by the pairs run one after another (their L2 lines are reused)
    static T* b(hysco_ctx c, int k) {
        return static_cast<T*>(c->buf[k]) + c->plane_off + (k == B_B || !c->vshare ? c->vp : 0) * c->g.ps;
    }

    // bold / q given: a TRIAL evaluation forms the retry b itself (no ls_retry launch)
    static void eval(hysco_ctx c, const SolveParams& sp, int mode, const T* bsrc, const T* bold = nullptr,
                     const T* q = nullptr) {
        NCH_SWITCH(c->nch, eval_kernel<T, NCH><<<dim3(c->gx_eval, c->vb), 32 * EV_CT, c->smem_eval, c->stream>>>(
                               c->g, c->ctl, sp, mode, (const T*)c->Ip, (const T*)c->Im, bsrc, bold, q,
                               b(c, B_GRAD), b(c, B_DT), b(c, B_ET)));
    }
    static void pcg_init(hysco_ctx c) {
        NCH_SWITCH(c->nch, pcg_init_kernel<T, NCH><<<dim3(c->gx_nodes, c->vb), 256, 0, c->stream>>>(
                               c->g, c->ctl, b(c, B_GRAD), b(c, B_DT), b(c, B_X), b(c, B_R), b(c, B_P)));
    }
    static void pcg_iter(hysco_ctx c, const SolveParams& sp) {
        dim3 gr(c->gx_nodes, c->vb);
        NCH_SWITCH(c->nch,
                   matvec_kernel<T, NCH, true><<<dim3(c->gx_mv, c->vb), 256, 0, c->stream>>>(
                       c->g, c->ctl, b(c, B_DT), b(c, B_ET), b(c, B_P), b(c, B_HP));
                   pcg_update_kernel<T, NCH><<<gr, 256, 0, c->stream>>>(c->g, c->ctl, sp, b(c, B_DT), b(c, B_P),
                                                                       b(c, B_HP), b(c, B_X), b(c, B_R));
                   pcg_dir_kernel<T, NCH><<<gr, 256, 0, c->stream>>>(c->g, c->ctl, b(c, B_DT), b(c, B_R),
                                                                    b(c, B_P)));
    }
    // block preconditioner (R20): factor once per GN step, solve per iteration
    static dim3 gblk(hysco_ctx c) { return dim3((unsigned)((c->g.ncol + BLK_THREADS - 1) / BLK_THREADS), c->vb); }
    static void bfac(hysco_ctx c, int need_active) {
        bfac_kernel<T><<<gblk(c), BLK_THREADS, 0, c->stream>>>(c->g, c->ctl, b(c, B_DT), b(c, B_ET), b(c, B_W),
                                                               b(c, B_F), need_active);
    }
    static void psolve(hysco_ctx c, const T* r, T* z) {
        psolve_kernel<T><<<gblk(c), BLK_THREADS, 0, c->stream>>>(c->g, c->ctl, b(c, B_ET), b(c, B_W), b(c, B_F), r, z);
    }
    static void pcg_init_blk(hysco_ctx c, const SolveParams& sp) {
        bfac(c, 1);
        NCH_SWITCH(c->nch, pcg_blk_kernel<T, NCH, true><<<dim3(c->gx_nodes, c->vb), 256, 0, c->stream>>>(
                               c->g, c->ctl, sp, b(c, B_GRAD), b(c, B_P), b(c, B_HP), b(c, B_X), b(c, B_R),
                               b(c, B_W), b(c, B_ET), b(c, B_F), b(c, B_TMP)));
    }
    static void pcg_iter_blk(hysco_ctx c, const SolveParams& sp) {
        dim3 gr(c->gx_nodes, c->vb);
        NCH_SWITCH(c->nch,
                   matvec_kernel<T, NCH, true><<<dim3(c->gx_mv, c->vb), 256, 0, c->stream>>>(
                       c->g, c->ctl, b(c, B_DT), b(c, B_ET), b(c, B_P), b(c, B_HP));
                   pcg_blk_kernel<T, NCH, false><<<gr, 256, 0, c->stream>>>(
                       c->g, c->ctl, sp, b(c, B_GRAD), b(c, B_P), b(c, B_HP), b(c, B_X), b(c, B_R), b(c, B_W),
                       b(c, B_ET), b(c, B_F), b(c, B_TMP));
                   pcg_dir_blk_kernel<T, NCH><<<gr, 256, 0, c->stream>>>(c->g, c->ctl, b(c, B_TMP), b(c, B_P)));
    }
    // flat two-launch PCG (hysco_flat.cuh): z in B_TMP, p double-buffered in B_P / B_W
    // (B_F holds M = diag(H_J), formed by the PCG start)
    static void pcg_init_flat(hysco_ctx c) {
        pcg_init_flat_kernel<T><<<dim3(c->gx_flat, c->vb), 256, 0, c->stream>>>(
            c->g, c->ctl, b(c, B_GRAD), b(c, B_DT), b(c, B_X), b(c, B_R), b(c, B_TMP), b(c, B_F));
    }
    // first iteration (p_0 = z) and later ones are separate instantiations; the
    // unrolled form launches the one it needs, the WHILE body both (the other exits)
    // fuse: (slab, defer mode) apply the preceding allreduced decision in the
    // kernel instead of a decide_kernel launch (hysco_flat.cuh)
    template <bool FIRST, int MS>
    static void march_ms_t(hysco_ctx c, int fuse, const SolveParams& sp) {
        pcg_march_kernel<T, FIRST, MS><<<dim3(c->gx_dmv, c->vb), MARCH_THREADS, c->smem_mr, c->stream>>>(
            c->g, c->ctl, c->mr_njb, c->mr_c, c->mr_plan, b(c, B_DT), b(c, B_ET), b(c, B_TMP), b(c, B_P), b(c, B_W),
            b(c, B_HP), b(c, B_X), fuse, sp);
    }
    template <bool FIRST>
    static void march(hysco_ctx c, int fuse, const SolveParams& sp) {
        switch (c->mr_plan.ms) {
            case 2: march_ms_t<FIRST, 2>(c, fuse, sp); break;
            case 4: march_ms_t<FIRST, 4>(c, fuse, sp); break;
            case 8: march_ms_t<FIRST, 8>(c, fuse, sp); break;
            default: march_ms_t<FIRST, 12>(c, fuse, sp); break;
        }
    }
    static void pcg_dirmv(hysco_ctx c, bool first, int fuse = 0, const SolveParams& sp = SolveParams{}) {
        if (first) march<true>(c, 0, sp);
        else march<false>(c, fuse, sp);
    }
    static void pcg_upd(hysco_ctx c, const SolveParams& sp, int fuse = 0) {
        pcg_upd_kernel<T><<<dim3(c->gx_flat, c->vb), 256, 0, c->stream>>>(c->g, c->ctl, sp, b(c, B_F), b(c, B_HP),
                                                                         b(c, B_R), b(c, B_TMP), fuse);
    }
    static void pcg_iter_flat(hysco_ctx c, const SolveParams& sp, bool first) {
        pcg_dirmv(c, first);
        pcg_upd(c, sp);
    }
    static void trial_flat(hysco_ctx c, T* bdst, T* bold) {
        trial_flat_kernel<T><<<dim3(c->gx_flat, c->vb), 256, 0, c->stream>>>(c->g, c->ctl, b(c, B_GRAD), b(c, B_X),
                                                                            b(c, B_P), b(c, B_W), bdst, bold);
    }
    static void trial_init(hysco_ctx c) {
        NCH_SWITCH(c->nch, trial_init_kernel<T, NCH><<<dim3(c->gx_nodes, c->vb), 256, 0, c->stream>>>(
                               c->g, c->ctl, b(c, B_GRAD), b(c, B_X), b(c, B_B), b(c, B_BOLD)));
    }
    static void ls_body(hysco_ctx c, const SolveParams& sp) { eval(c, sp, EVAL_TRIAL, b(c, B_B), b(c, B_BOLD), b(c, B_X)); }
    static void matvec_plain(hysco_ctx c, const T* q, T* Hq) {
        NCH_SWITCH(c->nch, matvec_kernel<T, NCH, false><<<dim3(c->gx_mv, c->vb), 256, 0, c->stream>>>(
                               c->g, c->ctl, b(c, B_DT), b(c, B_ET), q, Hq));
    }
    static void diag(hysco_ctx c, T* out) {
        NCH_SWITCH(c->nch, hess_diag_kernel<T, NCH><<<dim3(c->gx_nodes, c->vb), 256, 0, c->stream>>>(
                               c->g, c->ctl, b(c, B_DT), out));
    }
    static void apply(hysco_ctx c, const T* bsrc, T* Tp, T* Tm, T* bout = nullptr) {
        apply_kernel<T><<<dim3(c->gx_apply, c->vb), 256, c->smem_apply, c->stream>>>(
            c->g, c->ctl, (const T*)c->Ip, (const T*)c->Im, bsrc, Tp, Tm, bout);
    }
    // OT init (+blur, guard) into buffer B_B
    static void ot(hysco_ctx c, const SolveParams& sp, int blur) {
        const T* Ip = (const T*)c->Ip;
        const T* Im = (const T*)c->Im;
        dim3 gn(c->gx_nodes, c->vb);
        ot_minmax_kernel<T><<<dim3(c->gx_cells, c->vb), 256, 0, c->stream>>>(c->g, c->ctl, sp, Ip, Im);
        T* dst = blur ? b(c, B_TMP) : b(c, B_B);
        ot_column_kernel<T><<<dim3(c->gx_ot, c->vb), 256, c->smem_ot, c->stream>>>(c->g, c->ctl, Ip, Im, dst);
        if (blur) {
            const double e = exp(-0.5), w0 = e / (1.0 + 2.0 * e), w1 = 1.0 / (1.0 + 2.0 * e);
            blur_axis_kernel<T, 1><<<gn, 256, 0, c->stream>>>(c->g, c->ctl, 0, w0, w1, b(c, B_TMP), b(c, B_R));
            blur_axis_kernel<T, 1><<<gn, 256, 0, c->stream>>>(c->g, c->ctl, 1, w0, w1, b(c, B_R), b(c, B_P));
            blur_pe_guard_kernel<T><<<gn, 256, 0, c->stream>>>(c->g, c->ctl, sp, w0, w1, b(c, B_P), b(c, B_B));
        } else {
            guard_max_kernel<T, 1><<<gn, 256, 0, c->stream>>>(c->g, c->ctl, sp, b(c, B_B));
        }
        guard_scale_kernel<T, 1><<<gn, 256, 0, c->stream>>>(c->g, c->ctl, b(c, B_B));
    }
};

// ---------------------------------------------------------------------------
// Runner: the same control structure either captured into a CUDA graph with
// conditional WHILE nodes, or executed with host-side loops.
// ---------------------------------------------------------------------------
struct Runner {
    hysco_ctx c;
    bool graph;
    cudaGraph_t cur = nullptr;
    std::vector<cudaGraphNode_t> tail;
    cudaError_t err = cudaSuccess;

    void seq(const std::function<void()>& fn) {
        if (err != cudaSuccess) return;
        if (!graph) {
            fn();
            err = cudaGetLastError();
            return;
        }
        err = cudaStreamBeginCaptureToGraph(c->stream, cur, tail.data(), nullptr, tail.size(),
                                            cudaStreamCaptureModeRelaxed);
        if (err != cudaSuccess) return;
        fn();
        cudaError_t le = cudaGetLastError();
        cudaStreamCaptureStatus cs;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        cudaError_t e2 = cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, nullptr, &deps, &nd);
        std::vector<cudaGraphNode_t> nt;
        if (e2 == cudaSuccess) nt.assign(deps, deps + nd);
        cudaGraph_t out = nullptr;
        cudaError_t e3 = cudaStreamEndCapture(c->stream, &out);
        err = le != cudaSuccess ? le : (e2 != cudaSuccess ? e2 : e3);
        tail = nt;
    }
    void handle(int slot) {
        if (err != cudaSuccess || !graph) return;
        cudaGraphConditionalHandle h;
        err = cudaGraphConditionalHandleCreate(&h, cur, 0, 0);
        if (err == cudaSuccess) {
            c->ctl.h[slot] = h;
            c->ctl.live |= 1u << slot;
        }
    }
    void loop(int slot, const std::function<void()>& body) {
        if (err != cudaSuccess) return;
        if (!graph) {
            for (int guard = 0; guard < 1000000; guard++) {
                err = cudaMemcpyAsync(c->h_cond + slot, c->dcond + slot, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                      c->stream);
                if (err == cudaSuccess) err = cudaStreamSynchronize(c->stream);
                if (err != cudaSuccess || c->h_cond[slot] == 0) return;
                body();
                if (err != cudaSuccess) return;
            }
            return;
        }
        cudaGraphNodeParams np{};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = c->ctl.h[slot];
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        err = cudaGraphAddNode(&node, cur, tail.data(), tail.size(), &np);
        if (err != cudaSuccess) return;
        cudaGraph_t saved = cur;
        cur = np.conditional.phGraph_out[0];
        tail.clear();
        body();
        cur = saved;
        tail.assign(1, node);
    }
};

// Resident PCG (fp32): K = node slots per thread, a compile-time parameter.
#define RES_K_SWITCH(k, ...)                                                   \
    switch (k) {                                                               \
        case RES_KMAX / 3: { constexpr int RK = RES_KMAX / 3; __VA_ARGS__; } break; \
        case 2 * RES_KMAX / 3: { constexpr int RK = 2 * RES_KMAX / 3; __VA_ARGS__; } break; \
        default: { constexpr int RK = RES_KMAX; __VA_ARGS__; } break;          \
    }

// bcur / bold: the trial b and b_old the fused Armijo start writes (B_B /
// B_BOLD in a solve; scratch when profiling).
static void launch_resident(hysco_ctx c, const SolveParams& sp, int pair, float* bcur, float* bold) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->res_grid, 1, 1);
    cfg.blockDim = dim3(RES_THREADS, 1, 1);
    cfg.dynamicSmemBytes = c->res_smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;   // co-residency of all CTAs (the spin waits rely on it)
    float* B[NBUF];
    for (int k = 0; k < NBUF; k++)   // the view's first pair (scratch shared in a per-pair view, L<T>::b)
        B[k] = static_cast<float*>(c->buf[k]) + (k == B_B || !c->vshare ? c->vp : 0) * c->g.ps;
    const int nb = c->vb;
#define RES_LAUNCH(FX, TL)                                                                                        \
    RES_K_SWITCH(c->res_k, cudaLaunchKernelEx(&cfg, pcg_resident_kernel<RK, FX, false, TL>, c->g, c->ctl, sp, pair, \
                                              (const float*)B[B_GRAD], (const float*)B[B_DT],                     \
                                              (const float*)B[B_ET], B[B_X], c->res_x, c->res_pg, c->res_part,    \
                                              c->res_flags, c->res_wi, c->res_wj, bcur, bold, nb,                 \
                                              (unsigned long long*)nullptr, c->res_tile))
    if (c->res_tiled) {
        if (sp.fixed) {
            RES_LAUNCH(true, true);
        } else {
            RES_LAUNCH(false, true);
        }
    } else {
        if (sp.fixed) {
            RES_LAUNCH(true, false);
        } else {
            RES_LAUNCH(false, false);
        }
    }
#undef RES_LAUNCH
}

// Persistent L2-resident PCG (hysco_l2pcg.cuh) for pair `pair` of the view.
template <typename T>
static void launch_l2pcg(hysco_ctx c, const SolveParams& sp, int pair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c->l2_grid, 1, 1);
    cfg.blockDim = dim3(L2P_THREADS, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;   // co-residency of all CTAs (the spin waits rely on it)
    T* B[NBUF];
    for (int k = 0; k < NBUF; k++) B[k] = L<T>::b(c, k);
    const int nb = c->vb;
    NCH_SWITCH(c->nch, {
        if (sp.fixed)
            cudaLaunchKernelEx(&cfg, pcg_l2_kernel<T, NCH, true>, c->g, c->ctl, sp, pair, (const T*)B[B_GRAD],
                               (const T*)B[B_DT], (const T*)B[B_ET], B[B_X], B[B_R], B[B_P], B[B_HP], B[B_B],
                               B[B_BOLD], c->res_part, c->res_flags, nb);
        else
            cudaLaunchKernelEx(&cfg, pcg_l2_kernel<T, NCH, false>, c->g, c->ctl, sp, pair, (const T*)B[B_GRAD],
                               (const T*)B[B_DT], (const T*)B[B_ET], B[B_X], B[B_R], B[B_P], B[B_HP], B[B_B],
                               B[B_BOLD], c->res_part, c->res_flags, nb);
    });
}

// Shared synchronisation buffers of the persistent PCG kernels (tagged
// all-reduce partials, p-halo flags + launch counter).
static bool alloc_persistent_sync(hysco_ctx ctx) {
    if (ctx->res_part) return true;
    const int G = ctx->nsm;
    if (cudaMalloc(&ctx->res_part, sizeof(double) * (3 * RES_PART_DOUBLES + RES_LIMB_DOUBLES)) != cudaSuccess ||
        cudaMalloc(&ctx->res_flags, sizeof(unsigned) * res_flags_words(G)) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaMemset(ctx->res_part, 0, sizeof(double) * (3 * RES_PART_DOUBLES + RES_LIMB_DOUBLES));
    cudaMemset(ctx->res_flags, 0, sizeof(unsigned) * res_flags_words(G));
    const unsigned first_launch = 1;      // tags of launch 0 would match the zeroed slots
    cudaMemcpy(ctx->res_flags + (size_t)G * RES_FLAG_STRIDE, &first_launch, sizeof(unsigned), cudaMemcpyHostToDevice);
    return true;
}

// The L2-resident persistent PCG, opt-in (HYSCO_L2PCG=1), when the
// shared-memory one does not apply and every pair has >= 1 column per SM.
// Measured at 7T (PCG working set 127 MB ~ the L2): 78 us per iteration,
// no faster than the three streaming kernels (the per-column arithmetic,
// not the launch boundaries, bounds both), so it is not the
// default.  Not on slab contexts (their exchanges are host-driven).
template <typename T>
static void setup_l2pcg(hysco_ctx ctx) {
    ctx->l2pcg = false;
    const char* e = getenv("HYSCO_L2PCG");
    if (!(e && e[0] == '1') || ctx->resident || ctx->g.slab) return;
    const Geom& g = ctx->g;
    const int G = ctx->nsm;
    if (g.ncol < G || G * 2 > RES_RSTRIDE) return;
    int occ = 0;
    NCH_SWITCH(ctx->nch, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pcg_l2_kernel<T, NCH, true>,
                                                                       L2P_THREADS, 0));
    int occ2 = 0;
    NCH_SWITCH(ctx->nch, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, pcg_l2_kernel<T, NCH, false>,
                                                                       L2P_THREADS, 0));
    if (occ < 1 || occ2 < 1 || !alloc_persistent_sync(ctx)) {
        cudaGetLastError();
        return;
    }
    ctx->l2_grid = G;
    ctx->l2pcg = true;
}

// Decide whether the PCG state of one pair fits on chip.
static void setup_resident(hysco_ctx ctx) {
    ctx->resident = false;
    const char* e = getenv("HYSCO_NO_RESIDENT");
    if ((e && e[0] == '1') || ctx->cfg.dtype != HYSCO_F32) return;
    const Geom& g = ctx->g;
    const int G = ctx->nsm;
    if (g.ncol < G) return;
    if (G >= 256) return;                // one arrival byte in the limb all-reduce words
    const long long ncl_max = (g.ncol + G - 1) / G;
    const long long nqmax = ncl_max * (res_pad(g.P) / 2);   // node pairs per CTA
    const long long need_k = (nqmax + RES_THREADS - 1) / RES_THREADS;
    if (need_k > RES_KMAX) return;
    const int k = need_k <= RES_KMAX / 3 ? RES_KMAX / 3 : need_k <= 2 * RES_KMAX / 3 ? 2 * RES_KMAX / 3 : RES_KMAX;
    // 2-D tiles (hysco_resident.cuh ResTile): an exact tiling n1 = TI TH, n2 = TJ TW
    // with TI TJ CTAs (>= 95 % of the SMs, <= G), TH TW columns in the same slot
    // count k, TW GPC <= NT and (TH - 1) TW GPC >= (k - 1) NT; fewest perimeter
    // columns (2 TH + 2 TW) wins.  HYSCO_RES_TILED=0: 1-D strips.
    ctx->res_tiled = false;
    if (!(getenv("HYSCO_RES_TILED") && getenv("HYSCO_RES_TILED")[0] == '0') && g.slab == 0) {
        const int GPC = res_pad(g.P) / 2;
        long long best = -1;
        for (int TH = 1; TH <= g.n1; TH++) {
            if (g.n1 % TH) continue;
            for (int TW = 1; TW <= g.n2; TW++) {
                if (g.n2 % TW) continue;
                const long long tiles = (long long)(g.n1 / TH) * (g.n2 / TW);
                const long long twg = (long long)TW * GPC, nq = (long long)TH * twg;
                if (tiles > G || tiles * 20 < (long long)G * 19 || nq > (long long)k * RES_THREADS) continue;
                if (twg > RES_THREADS || (TH - 1) * twg < (long long)(k - 1) * RES_THREADS) continue;
                const long long cost = 2LL * TH + 2LL * TW;
                if (best < 0 || cost < best) {
                    best = cost;
                    ctx->res_tile = ResTile{g.n1 / TH, g.n2 / TW, TH, TW};
                }
            }
        }
        ctx->res_tiled = best >= 0;
    }
    const size_t smem = res_smem_bytes(k);   // layout: hysco_resident.cuh
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->cfg.device);
    cudaFuncAttributes fa{};
    RES_K_SWITCH(k, cudaFuncGetAttributes(&fa, pcg_resident_kernel<RK, false>));
    if (smem + fa.sharedSizeBytes > (size_t)optin) return;
    cudaError_t err = cudaSuccess;
    RES_K_SWITCH(k, {
        const void* fns[6] = {(const void*)pcg_resident_kernel<RK, false>, (const void*)pcg_resident_kernel<RK, true>,
                              (const void*)pcg_resident_kernel<RK, false, false, true>,
                              (const void*)pcg_resident_kernel<RK, true, false, true>,
                              (const void*)pcg_sync_floor_kernel<RK>, (const void*)pcg_sync_floor_kernel<RK, true>};
        for (int f = 0; f < 6 && err == cudaSuccess; f++)
            err = cudaFuncSetAttribute(fns[f], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (err != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    int occ = 0;
    RES_K_SWITCH(k, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pcg_resident_kernel<RK, false>, RES_THREADS,
                                                                  smem));
    if (occ < 1) {
        cudaGetLastError();
        return;
    }
    const size_t ghost =
        std::max(res_ghost_pair_floats(g) * ctx->cfg.batch + res_ghost_slack_floats(k),
                 ctx->res_tiled ? res_tiled_ghost_floats(G, k) * ctx->cfg.batch : (size_t)0) * sizeof(float);
    const size_t xpadb = std::max((size_t)g.ncol * res_pad(g.P), ctx->res_tiled ? res_tiled_ghost_floats(G, k) : (size_t)0) *
                         sizeof(float);
    if (G * 2 > RES_RSTRIDE) return;   // replica layout of the partials (hysco_resident.cuh)
    if (!alloc_persistent_sync(ctx) || cudaMalloc(&ctx->res_pg, ghost) != cudaSuccess ||
        cudaMalloc(&ctx->res_x, xpadb) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaMemset(ctx->res_pg, 0, ghost);   // ghost planes stay zero forever
    ctx->res_k = k;
    ctx->res_wi = (float)(g.ahd * g.ih1sq);
    ctx->res_wj = (float)(g.ahd * g.ih2sq);
    ctx->res_grid = ctx->res_tiled ? ctx->res_tile.TI * ctx->res_tile.TJ : G;
    ctx->res_smem = smem;
    ctx->resident = true;
}

// ---------------------------------------------------------------------------
// Slab decomposition along dim 1.  Each rank's
// context owns planes [i0, i0 + n1) of every pair; node arrays carry one halo
// plane below and above.  Before every in-plane Laplacian application (eval
// on b, matvec on p, the periodic blur pass along dim 1) the boundary planes
// are exchanged; after every reduction the pair totals are allreduced and
// decide_kernel takes the (identical) decision on every rank.  Multi-rank
// solves are host-orchestrated (loop conditions read back per iteration);
// two transports: NCCL (one process per GPU) and a single-GPU loopback group
// (several contexts on one stream) that tests the same kernels and exchanges.
// ---------------------------------------------------------------------------
struct CommBase {
    virtual ~CommBase() {}
    virtual cudaError_t halo(std::vector<hysco_ctx>& R, int k, bool periodic) = 0;
    virtual cudaError_t allreduce(std::vector<hysco_ctx>& R, bool with_max) = 0;
};

// user node array (dense [batch][Nn]) <-> internal buffer (pair stride ps, halo planes)
static cudaError_t copy_nodes(hysco_ctx c, void* dst, const void* src, bool to_internal, cudaMemcpyKind kind) {
    const size_t w = (size_t)c->g.Nn * c->esz;
    if (c->g.ps == c->g.Nn && c->plane_off == 0)
        return cudaMemcpyAsync(dst, src, (size_t)c->cfg.batch * w, kind, c->stream);
    const size_t pitch = (size_t)c->g.ps * c->esz, off = c->plane_off * c->esz;
    if (to_internal)
        return cudaMemcpy2DAsync((char*)dst + off, pitch, src, w, w, c->cfg.batch, kind, c->stream);
    return cudaMemcpy2DAsync(dst, w, (const char*)src + off, pitch, w, c->cfg.batch, kind, c->stream);
}

__global__ void loopback_reduce_kernel(double* const* bufs, int nr, int n, int with_max) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double s = 0, m = -INFINITY;
        for (int r = 0; r < nr; r++) {          // fixed rank order: deterministic
            s += bufs[r][i];
            if (with_max) m = fmax(m, bufs[r][n + i]);
        }
        for (int r = 0; r < nr; r++) {
            bufs[r][i] = s;
            if (with_max) bufs[r][n + i] = m;
        }
    }
}

struct LoopbackComm : CommBase {
    std::vector<hysco_ctx> members;    // rank order; all on one device and one stream
    double** d_ptrs = nullptr;
    int refs = 0;                      // member contexts alive
    cudaStream_t stream = nullptr;     // shared by the members; owned here if created here
    bool own_stream = false;
    ~LoopbackComm() override {
        if (d_ptrs) cudaFree(d_ptrs);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
    cudaError_t halo(std::vector<hysco_ctx>& R, int k, bool periodic) override {
        const int n = (int)members.size();
        for (int r = 0; r < n; r++) {
            hysco_ctx c = members[r];
            const size_t plane = (size_t)c->g.n2 * c->g.P * c->esz;
            for (int p = 0; p < c->cfg.batch; p++) {
                char* base = (char*)c->buf[k] + (size_t)p * c->g.ps * c->esz;
                const int lo = r > 0 ? r - 1 : (periodic ? n - 1 : -1);
                const int hi = r < n - 1 ? r + 1 : (periodic ? 0 : -1);
                if (lo >= 0) {   // lower halo <- last plane of rank lo
                    hysco_ctx d = members[lo];
                    const char* src = (const char*)d->buf[k] + (size_t)p * d->g.ps * d->esz + d->plane_off * d->esz +
                                      (size_t)(d->g.n1 - 1) * plane;
                    cudaError_t e = cudaMemcpyAsync(base, src, plane, cudaMemcpyDeviceToDevice, c->stream);
                    if (e != cudaSuccess) return e;
                }
                if (hi >= 0) {   // upper halo <- first plane of rank hi
                    hysco_ctx d = members[hi];
                    const char* src = (const char*)d->buf[k] + (size_t)p * d->g.ps * d->esz + d->plane_off * d->esz;
                    cudaError_t e = cudaMemcpyAsync(base + c->plane_off * c->esz + (size_t)c->g.n1 * plane, src, plane,
                                                    cudaMemcpyDeviceToDevice, c->stream);
                    if (e != cudaSuccess) return e;
                }
            }
        }
        (void)R;
        return cudaSuccess;
    }
    cudaError_t allreduce(std::vector<hysco_ctx>& R, bool with_max) override {
        hysco_ctx c = members[0];
        loopback_reduce_kernel<<<1, 256, 0, c->stream>>>(d_ptrs, (int)members.size(), (int)(c->cfg.batch * RED_W),
                                                         with_max ? 1 : 0);
        (void)R;
        return cudaGetLastError();
    }
};

struct NcclComm : CommBase {
    ncclComm_t comm = nullptr;
    int rank = 0, n = 1;
    ncclResult_t last = ncclSuccess;
    ~NcclComm() override {
        if (comm) ncclCommDestroy(comm);
    }
    cudaError_t halo(std::vector<hysco_ctx>& R, int k, bool periodic) override {
        hysco_ctx c = R[0];
        const size_t cnt = (size_t)c->g.n2 * c->g.P;
        const ncclDataType_t ty = c->esz == 8 ? ncclDouble : ncclFloat;
        const int lo = rank > 0 ? rank - 1 : (periodic ? n - 1 : -1);
        const int hi = rank < n - 1 ? rank + 1 : (periodic ? 0 : -1);
        if (n == 1) {                      // periodic self-ring without NCCL
            if (!periodic) return cudaSuccess;
            for (int p = 0; p < c->cfg.batch; p++) {
                char* base = (char*)c->buf[k] + (size_t)p * c->g.ps * c->esz;
                char* own = base + c->plane_off * c->esz;
                const size_t pb = cnt * c->esz;
                cudaMemcpyAsync(base, own + (size_t)(c->g.n1 - 1) * pb, pb, cudaMemcpyDeviceToDevice, c->stream);
                cudaMemcpyAsync(own + (size_t)c->g.n1 * pb, own, pb, cudaMemcpyDeviceToDevice, c->stream);
            }
            return cudaGetLastError();
        }
        // phase A: first plane -> lower neighbour, upper halo <- upper neighbour;
        // phase B: last plane -> upper neighbour, lower halo <- lower neighbour
        // (this order keeps per-peer send/recv matching right for 2-rank rings)
        if ((last = ncclGroupStart()) != ncclSuccess) return cudaErrorUnknown;
        for (int ph = 0; ph < 2; ph++)
            for (int p = 0; p < c->cfg.batch; p++) {
                char* base = (char*)c->buf[k] + (size_t)p * c->g.ps * c->esz;
                char* own = base + c->plane_off * c->esz;
                const size_t pb = cnt * c->esz;
                if (ph == 0) {
                    if (lo >= 0) last = ncclSend(own, cnt, ty, lo, comm, c->stream);
                    if (hi >= 0) last = ncclRecv(own + (size_t)c->g.n1 * pb, cnt, ty, hi, comm, c->stream);
                } else {
                    if (hi >= 0) last = ncclSend(own + (size_t)(c->g.n1 - 1) * pb, cnt, ty, hi, comm, c->stream);
                    if (lo >= 0) last = ncclRecv(base, cnt, ty, lo, comm, c->stream);
                }
            }
        if ((last = ncclGroupEnd()) != ncclSuccess) return cudaErrorUnknown;
        return cudaSuccess;
    }
    cudaError_t allreduce(std::vector<hysco_ctx>& R, bool with_max) override {
        hysco_ctx c = R[0];
        if (n == 1) return cudaSuccess;
        const size_t cnt = (size_t)c->cfg.batch * RED_W;
        if ((last = ncclAllReduce(c->red, c->red, cnt, ncclDouble, ncclSum, comm, c->stream)) != ncclSuccess)
            return cudaErrorUnknown;
        if (with_max && (last = ncclAllReduce(c->red + cnt, c->red + cnt, cnt, ncclDouble, ncclMax, comm, c->stream)) !=
                            ncclSuccess)
            return cudaErrorUnknown;
        return cudaSuccess;
    }
};

// Multi-rank path: `R` = the contexts this process drives (one for NCCL, all
// ranks of a loopback group on one stream).  Straight-line parts -- OT, every
// GN step's PCG (fixed counts: unrolled) with its halo exchanges, allreduces
// and device-side decisions, the Armijo start -- are recorded once as CUDA
// graph segments (NCCL calls captured with the kernels) and replayed; only
// the loops whose trip count the device decides (the Armijo search; with the
// paper's stop rules also the GN and PCG loops) run on the host, one stream
// synchronisation per loop test.  A fixed 10 x 10 solve thus synchronises
// once per GN step instead of once per PCG iteration.  HYSCO_NO_GRAPH=1 runs
// every part eagerly.
struct SegExec {
    hysco_ctx c;                          // primary context: stream, segment cache
    bool graph = true;
    bool build = false;                   // recording (else replaying the cache)
    bool open = false, pending = false;
    int in_loop = 0;
    size_t idx = 0;
    cudaError_t err = cudaSuccess;
    void ok(cudaError_t e) {
        if (err == cudaSuccess && e != cudaSuccess) err = e;
    }
    template <typename F>
    void seq(F fn) {
        if (err != cudaSuccess) return;
        if (!graph || in_loop) {
            fn();
            ok(cudaGetLastError());
            return;
        }
        if (!build) {
            pending = true;
            return;
        }
        if (!open) {
            ok(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
            open = true;
        }
        fn();
        ok(cudaGetLastError());
    }
    void flush() {
        if (!graph || in_loop) return;
        if (build && open) {
            cudaGraph_t gr = nullptr;
            cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
            open = false;
            ok(e);
            cudaGraphExec_t ex = nullptr;
            if (err == cudaSuccess) ok(cudaGraphInstantiate(&ex, gr, 0));
            if (gr) cudaGraphDestroy(gr);
            if (err != cudaSuccess) return;
            c->seg_exec.push_back(ex);
            ok(cudaGraphLaunch(ex, c->stream));
            idx++;
        } else if (!build && pending) {
            if (idx >= c->seg_exec.size()) {
                ok(cudaErrorInvalidValue);
                return;
            }
            ok(cudaGraphLaunch(c->seg_exec[idx++], c->stream));
            pending = false;
        }
    }
};

template <typename T>
struct SlabRun {
    std::vector<hysco_ctx>& R;
    CommBase* comm;
    SolveParams sp;
    SegExec& x;
    cudaError_t err = cudaSuccess;

    void ok(cudaError_t e) {
        if (err == cudaSuccess && e != cudaSuccess) err = e;
    }
    template <typename F>
    void each(F fn) {
        for (hysco_ctx c : R) fn(c);
        ok(cudaGetLastError());
    }
    void reduce_decide(int op, int mode, bool with_max) {
        ok(comm->allreduce(R, with_max));
        each([&](hysco_ctx c) {
            decide_kernel<<<1, 256, 0, c->stream>>>(c->g, c->ctl, sp, op, mode, (int)c->cfg.batch);
        });
    }
    template <typename F>
    void seq(F fn) {
        x.seq([&] { fn(); });
        ok(x.err);
    }
    // a device-decided loop test: flush the recorded segment, read the flag
    bool cond(int slot) {
        x.flush();
        ok(x.err);
        hysco_ctx c = R[0];
        ok(cudaMemcpyAsync(c->h_cond + slot, c->dcond + slot, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
        for (hysco_ctx d : R) ok(cudaStreamSynchronize(d->stream));
        return err == cudaSuccess && c->h_cond[slot] != 0;
    }
    template <typename F>
    void loop(int slot, F body) {
        x.flush();
        ok(x.err);
        x.in_loop++;
        while (err == cudaSuccess && cond(slot)) body();
        x.in_loop--;
    }
    static dim3 gn(hysco_ctx c) { return dim3(c->gx_nodes, c->cfg.batch); }

    void ot(int blur) {
        each([&](hysco_ctx c) {
            ot_minmax_kernel<T><<<dim3(c->gx_cells, c->cfg.batch), 256, 0, c->stream>>>(c->g, c->ctl, sp,
                                                                                         (const T*)c->Ip,
                                                                                         (const T*)c->Im);
        });
        reduce_decide(OP_MINMAX, 0, true);
        each([&](hysco_ctx c) {
            ot_column_kernel<T><<<dim3(c->gx_ot, c->cfg.batch), 256, c->smem_ot, c->stream>>>(
                c->g, c->ctl, (const T*)c->Ip, (const T*)c->Im, L<T>::b(c, blur ? B_TMP : B_B));
        });
        if (blur) {
            const double e = exp(-0.5), w0 = e / (1.0 + 2.0 * e), w1 = 1.0 / (1.0 + 2.0 * e);
            ok(comm->halo(R, B_TMP, true));
            each([&](hysco_ctx c) {
                blur_axis_kernel<T, 1><<<gn(c), 256, 0, c->stream>>>(c->g, c->ctl, 0, w0, w1, L<T>::b(c, B_TMP),
                                                                    L<T>::b(c, B_R));
                blur_axis_kernel<T, 1><<<gn(c), 256, 0, c->stream>>>(c->g, c->ctl, 1, w0, w1, L<T>::b(c, B_R),
                                                                    L<T>::b(c, B_P));
                blur_axis_kernel<T, 1><<<gn(c), 256, 0, c->stream>>>(c->g, c->ctl, 2, w0, w1, L<T>::b(c, B_P),
                                                                    L<T>::b(c, B_B));
            });
        }
        each([&](hysco_ctx c) {
            guard_max_kernel<T, 1><<<gn(c), 256, 0, c->stream>>>(c->g, c->ctl, sp, L<T>::b(c, B_B));
        });
        reduce_decide(OP_GUARD, 0, true);
        each([&](hysco_ctx c) { guard_scale_kernel<T, 1><<<gn(c), 256, 0, c->stream>>>(c->g, c->ctl, L<T>::b(c, B_B)); });
    }
    void eval(int mode) {
        ok(comm->halo(R, B_B, false));
        each([&](hysco_ctx c) { L<T>::eval(c, sp, mode, L<T>::b(c, B_B)); });
        reduce_decide(OP_EVAL, mode, false);
    }
    // flat two-launch form on slabs (hysco_flat.cuh, defer mode): the march
    // reads z_k and p_{k-1} on the halo planes, so z is exchanged after the
    // PCG start and every residual update, p_k after every march
    bool flat() const { return R[0]->flat && sp.precond != HYSCO_PRECOND_PE_BLOCK; }
    void pcg_init(bool blk) {
        if (flat()) {
            each([&](hysco_ctx c) { L<T>::pcg_init_flat(c); });
            reduce_decide(OP_PCG_INIT, 0, false);
            ok(comm->halo(R, B_TMP, false));
            return;
        }
        if (blk) {
            each([&](hysco_ctx c) { L<T>::pcg_init_blk(c, sp); });
        } else {
            each([&](hysco_ctx c) {
                NCH_SWITCH(c->nch, pcg_init_kernel<T, NCH><<<gn(c), 256, 0, c->stream>>>(
                                       c->g, c->ctl, L<T>::b(c, B_GRAD), L<T>::b(c, B_DT), L<T>::b(c, B_X),
                                       L<T>::b(c, B_R), L<T>::b(c, B_P)));
            });
        }
        reduce_decide(OP_PCG_INIT, 0, false);
    }
    // one PCG iteration: p halo, matvec, allreduce + decision,
    // update (block: with the column Thomas solve, R20), allreduce + decision,
    // direction
    // fixed counts: the march / update apply the preceding allreduced decision
    // themselves (no decide_kernel launch), except after the last update, whose
    // decision the Armijo start needs committed
    bool fuse() const { return sp.fixed && !getenv_is1("HYSCO_SLAB_NO_FUSE"); }
    void pcg_iter(bool blk, int k) {
        if (flat()) {
            const bool fz = fuse();
            each([&](hysco_ctx c) { L<T>::pcg_dirmv(c, k == 0, fz && k > 0 ? 1 : 0, sp); });
            if (fz) ok(comm->allreduce(R, false));
            else reduce_decide(OP_MATVEC, 0, false);
            ok(comm->halo(R, (k & 1) ? B_W : B_P, false));   // p_k for the next march
            each([&](hysco_ctx c) { L<T>::pcg_upd(c, sp, fz ? 1 : 0); });
            if (fz && k + 1 < sp.max_pcg) ok(comm->allreduce(R, false));
            else reduce_decide(OP_UPDATE, 0, false);
            ok(comm->halo(R, B_TMP, false));                  // z_{k+1}
            return;
        }
        ok(comm->halo(R, B_P, false));
        each([&](hysco_ctx c) {
            NCH_SWITCH(c->nch, matvec_kernel<T, NCH, true><<<dim3(c->gx_mv, c->cfg.batch), 256, 0, c->stream>>>(
                                   c->g, c->ctl, L<T>::b(c, B_DT), L<T>::b(c, B_ET), L<T>::b(c, B_P),
                                   L<T>::b(c, B_HP)));
        });
        reduce_decide(OP_MATVEC, 0, false);
        if (blk) {
            each([&](hysco_ctx c) {
                NCH_SWITCH(c->nch, pcg_blk_kernel<T, NCH, false><<<gn(c), 256, 0, c->stream>>>(
                                       c->g, c->ctl, sp, L<T>::b(c, B_GRAD), L<T>::b(c, B_P), L<T>::b(c, B_HP),
                                       L<T>::b(c, B_X), L<T>::b(c, B_R), L<T>::b(c, B_W), L<T>::b(c, B_ET),
                                       L<T>::b(c, B_F), L<T>::b(c, B_TMP)));
            });
            reduce_decide(OP_UPDATE, 0, false);
            each([&](hysco_ctx c) {
                NCH_SWITCH(c->nch, pcg_dir_blk_kernel<T, NCH><<<gn(c), 256, 0, c->stream>>>(
                                       c->g, c->ctl, L<T>::b(c, B_TMP), L<T>::b(c, B_P)));
            });
        } else {
            each([&](hysco_ctx c) {
                NCH_SWITCH(c->nch, pcg_update_kernel<T, NCH><<<gn(c), 256, 0, c->stream>>>(
                                       c->g, c->ctl, sp, L<T>::b(c, B_DT), L<T>::b(c, B_P), L<T>::b(c, B_HP),
                                       L<T>::b(c, B_X), L<T>::b(c, B_R)));
            });
            reduce_decide(OP_UPDATE, 0, false);
            each([&](hysco_ctx c) {
                NCH_SWITCH(c->nch, pcg_dir_kernel<T, NCH><<<gn(c), 256, 0, c->stream>>>(
                                       c->g, c->ctl, L<T>::b(c, B_DT), L<T>::b(c, B_R), L<T>::b(c, B_P)));
            });
        }
    }
    void trial_start() {
        if (flat()) {
            each([&](hysco_ctx c) { L<T>::trial_flat(c, L<T>::b(c, B_B), L<T>::b(c, B_BOLD)); });
            reduce_decide(OP_TRIAL, 0, true);
            return;
        }
        each([&](hysco_ctx c) {
            NCH_SWITCH(c->nch, trial_init_kernel<T, NCH><<<gn(c), 256, 0, c->stream>>>(
                                   c->g, c->ctl, L<T>::b(c, B_GRAD), L<T>::b(c, B_X), L<T>::b(c, B_B),
                                   L<T>::b(c, B_BOLD)));
        });
        reduce_decide(OP_TRIAL, 0, true);
    }
    // Armijo search (R15): trial evaluation, then b = b_old + gamma q for the next try
    void line_search() {
        loop(COND_LS, [&] {
            seq([&] {
                eval(EVAL_TRIAL);
                each([&](hysco_ctx c) {
                    NCH_SWITCH(c->nch, ls_retry_kernel<T, NCH><<<gn(c), 256, 0, c->stream>>>(
                                           c->g, c->ctl, L<T>::b(c, B_X), L<T>::b(c, B_BOLD), L<T>::b(c, B_B)));
                });
            });
        });
    }
    void gn() {
        const bool blk = sp.precond == HYSCO_PRECOND_PE_BLOCK;   // column-local: no extra exchange (R20)
        seq([&] { eval(EVAL_GN_START); });
        if (sp.fixed) {   // fixed counts (R14-R16): GN steps and PCG iterations unrolled into the segments
            for (int k = 0; k < sp.max_gn && err == cudaSuccess; k++) {
                seq([&] {
                    pcg_init(blk);
                    for (int it = 0; it < sp.max_pcg; it++) pcg_iter(blk, it);
                    trial_start();
                });
                line_search();
            }
            return;
        }
        loop(COND_GN, [&] {   // paper stop rules: device-decided trip counts
            seq([&] { pcg_init(blk); });
            int it = 0;   // host iteration count = the device's pcg_k while the loop runs
            loop(COND_PCG, [&] { seq([&] { pcg_iter(blk, it++); }); });
            seq([&] { trial_start(); });
            line_search();
            seq([&] { each([&](hysco_ctx c) { gn_tail_kernel<<<1, 32, 0, c->stream>>>(c->ctl, (int)c->cfg.batch); }); });
        });
    }
};

// kind 1: solve from b (per-rank user arrays b_io[r]); kind 2: OT + solve + apply.
template <typename T>
static hysco_status run_slab_path(std::vector<hysco_ctx>& R, CommBase* comm, int kind, const SolveParams& sp,
                                  int blur, void* const* b_io, void* const* b_out, void* const* Tp, void* const* Tm) {
    hysco_ctx c0 = R[0];
    // segment cache of the primary context, valid for the same call shape
    std::vector<const void*> key;
    key.push_back((const void*)(uintptr_t)kind);
    key.push_back((const void*)(uintptr_t)blur);
    key.push_back((const void*)(uintptr_t)R.size());
    for (size_t r = 0; r < R.size(); r++) {
        key.push_back(R[r]);
        key.push_back(b_io ? b_io[r] : nullptr);
        key.push_back(b_out ? b_out[r] : nullptr);
        key.push_back(Tp ? Tp[r] : nullptr);
        key.push_back(Tm ? Tm[r] : nullptr);
        key.push_back(R[r]->Ip);
        key.push_back(R[r]->Im);
    }
    SegExec x{c0};
    x.graph = !c0->no_graph && !getenv_is1("HYSCO_NO_GRAPH");
    const bool hit = c0->seg_valid && c0->seg_key == key && memcmp(&c0->seg_sp, &sp, sizeof sp) == 0;
    if (x.graph && !hit) {
        for (cudaGraphExec_t e : c0->seg_exec) cudaGraphExecDestroy(e);
        c0->seg_exec.clear();
        c0->seg_valid = false;
    }
    x.build = x.graph && !hit;
    SlabRun<T> run{R, comm, sp, x};
    run.seq([&] {
        for (size_t r = 0; r < R.size(); r++) {
            hysco_ctx c = R[r];
            run.ok(cudaMemsetAsync(c->launches, 0, sizeof(unsigned long long), c->stream));
            if (kind == 1) run.ok(copy_nodes(c, c->buf[B_B], b_io[r], true, cudaMemcpyDeviceToDevice));
        }
        if (kind == 2) run.ot(blur);
    });
    run.gn();
    run.seq([&] {
        for (size_t r = 0; r < R.size(); r++) {
            hysco_ctx c = R[r];
            if (kind == 1) run.ok(copy_nodes(c, b_io[r], c->buf[B_B], false, cudaMemcpyDeviceToDevice));
            if (kind == 2) {
                if ((Tp && Tp[r]) || (Tm && Tm[r]))
                    L<T>::apply(c, L<T>::b(c, B_B), (T*)(Tp ? Tp[r] : nullptr), (T*)(Tm ? Tm[r] : nullptr));
                if (b_out && b_out[r]) run.ok(copy_nodes(c, b_out[r], c->buf[B_B], false, cudaMemcpyDeviceToDevice));
            }
        }
    });
    x.flush();
    run.ok(x.err);
    if (x.build && run.err == cudaSuccess) {
        c0->seg_key = key;
        c0->seg_sp = sp;
        c0->seg_valid = true;
    }
    for (size_t r = 0; r < R.size(); r++) {
        hysco_ctx c = R[r];
        run.ok(cudaGetLastError());
        run.ok(cudaMemcpyAsync(c->h_st, c->st, sizeof(PairState) * c->cfg.batch, cudaMemcpyDeviceToHost, c->stream));
        run.ok(cudaMemcpyAsync(c->h_launches, c->launches, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               c->stream));
    }
    for (hysco_ctx c : R) run.ok(cudaStreamSynchronize(c->stream));
    if (run.err != cudaSuccess) {
        cudaStreamCaptureStatus cs;
        if (cudaStreamIsCapturing(c0->stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
            cudaGraph_t tmp;
            cudaStreamEndCapture(c0->stream, &tmp);
            if (tmp) cudaGraphDestroy(tmp);
        }
        for (cudaGraphExec_t e : c0->seg_exec) cudaGraphExecDestroy(e);
        c0->seg_exec.clear();
        c0->seg_valid = false;
        const bool nccl = dynamic_cast<NcclComm*>(comm) && static_cast<NcclComm*>(comm)->last != ncclSuccess;
        for (hysco_ctx c : R) cuda_fail(c, run.err, nccl ? "slab solve (NCCL)" : "slab solve", __LINE__);
        return nccl ? HYSCO_ERR_NCCL : HYSCO_ERR_CUDA;
    }
    for (hysco_ctx c : R) c->last_launches = (long long)*c->h_launches;
    return HYSCO_OK;
}

// GN-PCG solve on buffer B_B, the structure of DESIGN.md "Solve graph".
template <typename T>
static void pcg_step(Runner& r, const SolveParams& sp, bool unrolled) {
    hysco_ctx c = r.c;
    const bool blk = sp.precond == HYSCO_PRECOND_PE_BLOCK;
    if (c->resident && !blk) {   // PCG + the Armijo start (trial_init) in one launch per pair
        r.seq([&] {
            for (int p = 0; p < c->vb; p++)
                launch_resident(c, sp, p, reinterpret_cast<float*>(L<T>::b(c, B_B)),
                                reinterpret_cast<float*>(L<T>::b(c, B_BOLD)));
        });
    } else if (c->l2pcg && !blk) {   // the same, state in L2 (hysco_l2pcg.cuh)
        r.seq([&] {
            for (int p = 0; p < c->vb; p++) launch_l2pcg<T>(c, sp, p);
        });
    } else if (c->flat && !blk) {   // two vectorised launches per iteration (hysco_flat.cuh)
        if (unrolled) {
            r.seq([&] {
                L<T>::pcg_init_flat(c);
                for (int k = 0; k < sp.max_pcg; k++) L<T>::pcg_iter_flat(c, sp, k == 0);
                L<T>::trial_flat(c, L<T>::b(c, B_B), L<T>::b(c, B_BOLD));
            });
        } else {
            r.handle(COND_PCG);
            // the first iteration (p_0 = z) outside the loop; its kernels exit
            // at once if the PCG start found nothing to do
            r.seq([&] {
                L<T>::pcg_init_flat(c);
                L<T>::pcg_iter_flat(c, sp, true);
            });
            r.loop(COND_PCG, [&] { r.seq([&] { L<T>::pcg_iter_flat(c, sp, false); }); });
            r.seq([&] { L<T>::trial_flat(c, L<T>::b(c, B_B), L<T>::b(c, B_BOLD)); });
        }
    } else if (unrolled) {   // fixed count: max_pcg iterations, kernels of finished pairs exit early
        r.seq([&] {
            if (blk) L<T>::pcg_init_blk(c, sp);
            else L<T>::pcg_init(c);
            for (int k = 0; k < sp.max_pcg; k++) {
                if (blk) L<T>::pcg_iter_blk(c, sp);
                else L<T>::pcg_iter(c, sp);
            }
            L<T>::trial_init(c);
        });
    } else {
        r.handle(COND_PCG);
        r.seq([&] {
            if (blk) L<T>::pcg_init_blk(c, sp);
            else L<T>::pcg_init(c);
        });
        r.loop(COND_PCG, [&] {
            r.seq([&] {
                if (blk) L<T>::pcg_iter_blk(c, sp);
                else L<T>::pcg_iter(c, sp);
            });
        });
        r.seq([&] { L<T>::trial_init(c); });
    }
}

// Fixed iteration counts (parity / timing, R14-R16) are unrolled in the graph:
// max_gn x (PCG step, first Armijo trial) with only the Armijo retries in a
// conditional WHILE node (usually skipped).  Each conditional node costs
// ~20-40 us of device-side scheduling on B200 (tools/timeline.py: 3T step
// gaps 617 -> 82 us), which the unrolled form avoids; kernels of finished
// pairs exit early.
// HYSCO_GRAPH_LOOPS=1 forces the WHILE-loop form.
template <typename T>
static void gn_sequence(Runner& r, const SolveParams& sp) {
    hysco_ctx c = r.c;
    const char* e = getenv("HYSCO_GRAPH_LOOPS");
    if (sp.fixed && r.graph && !(e && e[0] == '1') && c->resident && sp.precond != HYSCO_PRECOND_PE_BLOCK &&
        !getenv_is1("HYSCO_LS_WHILE")) {
        // resident PCG (one launch per GN step): max_gn unrolled slots of
        // (PCG step, trial / retry evaluation) with no conditional node inside;
        // a rejected trial's retry takes the next slot (whose PCG launch then
        // does nothing: pcg_step_active), and one WHILE node after the slots
        // finishes what the retries displaced (not entered when none did).
        // Each conditional node costs ~8 us of device-side scheduling (CUPTI
        // timeline: the gap before every resident launch after a WHILE node).
        r.handle(COND_GN);
        r.seq([&] { L<T>::eval(c, sp, EVAL_GN_START, L<T>::b(c, B_B)); });
        for (int k = 0; k < sp.max_gn; k++) {
            pcg_step<T>(r, sp, true);
            r.seq([&] { L<T>::ls_body(c, sp); });
        }
        r.loop(COND_GN, [&] {
            pcg_step<T>(r, sp, true);
            r.seq([&] { L<T>::ls_body(c, sp); });
        });
        return;
    }
    if (sp.fixed && r.graph && !(e && e[0] == '1')) {
        // a conditional node whose body runs costs ~95 us of device-side
        // scheduling (CUPTI timeline, 7T), so the first ls_unroll retries of a
        // search are plain launches (an evaluation with no search pending exits
        // at once, ~4 us) and only further ones go through the WHILE node
        const char* eu = getenv("HYSCO_LS_UNROLL");
        const int ls_unroll = eu ? std::max(0, atoi(eu)) : 2;
        r.seq([&] { L<T>::eval(c, sp, EVAL_GN_START, L<T>::b(c, B_B)); });
        for (int k = 0; k < sp.max_gn; k++) {
            pcg_step<T>(r, sp, true);
            r.handle(COND_LS);
            r.seq([&] {
                L<T>::ls_body(c, sp);                                          // first trial (gamma = 1)
                for (int u = 0; u < ls_unroll; u++) L<T>::ls_body(c, sp);     // first halvings / restore
            });
            r.loop(COND_LS, [&] { r.seq([&] { L<T>::ls_body(c, sp); }); });   // further halvings
        }
        return;
    }
    r.handle(COND_GN);
    r.seq([&] { L<T>::eval(c, sp, EVAL_GN_START, L<T>::b(c, B_B)); });
    r.loop(COND_GN, [&] {
        r.handle(COND_LS);
        pcg_step<T>(r, sp, false);
        r.loop(COND_LS, [&] { r.seq([&] { L<T>::ls_body(c, sp); }); });   // its last eval sets COND_GN
    });
}

// Narrow the launchers to pair p of a batch context (scoped): buffers, images
// and the per-pair control state (PairState, block partials, last-block
// counters) are offset to pair p, grids are the one-pair grids.
struct PairView {
    hysco_ctx c;
    Ctl ctl;
    const void *Ip, *Im;
    int gx[8];
    PairView(hysco_ctx ctx, int p) : c(ctx), ctl(ctx->ctl), Ip(ctx->Ip), Im(ctx->Im) {
        int* g[8] = {&c->gx_nodes, &c->gx_mv, &c->gx_cells, &c->gx_eval, &c->gx_apply, &c->gx_ot, &c->gx_flat, &c->gx_dmv};
        for (int k = 0; k < 8; k++) {
            gx[k] = *g[k];
            *g[k] = c->gx1[k];
        }
        c->vb = 1;
        c->vp = (size_t)p;
        c->vshare = true;
        c->ctl.st += p;
        c->ctl.part += (size_t)p * c->ctl.part_stride;
        c->ctl.ctr += p;
        c->ctl.hist += (size_t)p * HIST_MAX;
        c->Ip = static_cast<const char*>(Ip) + (size_t)p * c->g.Nc * c->esz;
        c->Im = static_cast<const char*>(Im) + (size_t)p * c->g.Nc * c->esz;
    }
    ~PairView() {
        int* g[8] = {&c->gx_nodes, &c->gx_mv, &c->gx_cells, &c->gx_eval, &c->gx_apply, &c->gx_ot, &c->gx_flat, &c->gx_dmv};
        for (int k = 0; k < 8; k++) *g[k] = gx[k];
        c->vb = (int)c->cfg.batch;
        c->vp = 0;
        c->vshare = false;
        c->ctl.st = ctl.st;
        c->ctl.part = ctl.part;
        c->ctl.ctr = ctl.ctr;
        c->ctl.hist = ctl.hist;
        c->Ip = Ip;
        c->Im = Im;
    }
};

// Build (kind 1: solve b in place; kind 2: correct = OT + solve + apply) and
// run either as a cached graph or host-looped.  With the resident PCG a batch
// runs pair by pair (the whole path of pair 0, then pair 1, ...): one pair's
// node arrays (~130 MB at 3T) then stay L2-resident between its kernels, so
// a pair costs the same in a batch as alone.
// hysco_correct_host_stream: copy the final per-pair states and the launch
// count of one item into its snapshot slot and reset the count for the next
// item -- one tiny kernel instead of a host synchronisation per item.
__global__ void state_snapshot_kernel(const PairState* __restrict__ st, int B, unsigned long long* launches,
                                      PairState* __restrict__ dst, unsigned long long* __restrict__ dl) {
    const int n = (int)(B * sizeof(PairState) / sizeof(int));
    const int* a = reinterpret_cast<const int*>(st);
    int* d = reinterpret_cast<int*>(dst);
    for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = a[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        *dl = *launches;
        *launches = 0;
    }
}

template <typename T>
static hysco_status run_path(hysco_ctx ctx, const GraphKey& key, void* b_io, void* b_out, void* Tp, void* Tm) {
    const bool per_pair = (ctx->resident || ctx->l2pcg) && ctx->cfg.batch > 1 && key.sp.precond != HYSCO_PRECOND_PE_BLOCK &&
                          !getenv_is1("HYSCO_BATCHED");
    ctx->last_per_pair = per_pair;
    auto body1 = [&](Runner& r) {
        const size_t nb = (size_t)ctx->vb * ctx->g.Nn * ctx->esz;
        const size_t on = ctx->vp * ctx->g.Nn * ctx->esz, oc = ctx->vp * ctx->g.Nc * ctx->esz;
        char* bio = b_io ? static_cast<char*>(b_io) + on : nullptr;
        char* bo = b_out ? static_cast<char*>(b_out) + on : nullptr;
        T* tp = Tp ? reinterpret_cast<T*>(static_cast<char*>(Tp) + oc) : nullptr;
        T* tm = Tm ? reinterpret_cast<T*>(static_cast<char*>(Tm) + oc) : nullptr;
        if (key.kind == 1) {
            r.seq([&] { cudaMemcpyAsync(L<T>::b(ctx, B_B), bio, nb, cudaMemcpyDeviceToDevice, ctx->stream); });
        } else {
            r.seq([&] { L<T>::ot(ctx, key.sp, key.blur); });
        }
        gn_sequence<T>(r, key.sp);
        r.seq([&] {
            if (key.kind == 1) {
                cudaMemcpyAsync(bio, L<T>::b(ctx, B_B), nb, cudaMemcpyDeviceToDevice, ctx->stream);
            } else {
                if (tp || tm) L<T>::apply(ctx, L<T>::b(ctx, B_B), tp, tm, (T*)bo);   // also copies b out
                else if (bo) cudaMemcpyAsync(bo, L<T>::b(ctx, B_B), nb, cudaMemcpyDeviceToDevice, ctx->stream);
            }
        });
    };
    auto body = [&](Runner& r) {
        if (!per_pair) {
            body1(r);
            return;
        }
        for (int p = 0; p < ctx->cfg.batch; p++) {
            PairView v(ctx, p);
            body1(r);
        }
    };
    // (deferred readback: the previous item's snapshot kernel reset the count)
    if (!ctx->defer_st) CK(cudaMemsetAsync(ctx->launches, 0, sizeof(unsigned long long), ctx->stream));
    bool use_graph = !ctx->no_graph && !ctx->graph_broken;
    if (use_graph) {
        bool hit = ctx->have_key && memcmp(&ctx->key, &key, sizeof key) == 0 && ctx->exec;
        if (!hit && ctx->have_key2 && memcmp(&ctx->key2, &key, sizeof key) == 0 && ctx->exec2) {
            std::swap(ctx->graph, ctx->graph2);
            std::swap(ctx->exec, ctx->exec2);
            std::swap(ctx->key, ctx->key2);
            std::swap(ctx->have_key, ctx->have_key2);
            hit = true;
        }
        if (!hit) {
            // the current graph becomes the spare; the old spare goes
            if (ctx->exec2) cudaGraphExecDestroy(ctx->exec2);
            if (ctx->graph2) cudaGraphDestroy(ctx->graph2);
            ctx->exec2 = ctx->have_key ? ctx->exec : nullptr;
            ctx->graph2 = ctx->have_key ? ctx->graph : nullptr;
            ctx->key2 = ctx->key;
            ctx->have_key2 = ctx->have_key && ctx->exec2;
            if (!ctx->have_key) {
                if (ctx->exec) cudaGraphExecDestroy(ctx->exec);
                if (ctx->graph) cudaGraphDestroy(ctx->graph);
            }
            ctx->exec = nullptr;
            ctx->graph = nullptr;
            ctx->have_key = false;
            Runner r{ctx, true};
            r.err = cudaGraphCreate(&ctx->graph, 0);
            r.cur = ctx->graph;
            ctx->ctl.use_graph = 1;
            ctx->ctl.live = 0;
            body(r);
            ctx->ctl.use_graph = 0;
            if (r.err == cudaSuccess) r.err = cudaGraphInstantiate(&ctx->exec, ctx->graph, 0);
            if (r.err != cudaSuccess) {
                // conditional nodes unavailable: fall back to host loops for this context
                cudaStreamCaptureStatus cs;
                if (cudaStreamIsCapturing(ctx->stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
                    cudaGraph_t tmp;
                    cudaStreamEndCapture(ctx->stream, &tmp);
                }
                cudaGetLastError();
                if (ctx->exec) cudaGraphExecDestroy(ctx->exec);
                if (ctx->graph) cudaGraphDestroy(ctx->graph);
                ctx->exec = nullptr;
                ctx->graph = nullptr;
                ctx->graph_broken = true;
                char m[256];
                snprintf(m, sizeof m, "graph build failed (%s); using host loops", cudaGetErrorString(r.err));
                ctx->err = m;
                use_graph = false;
            } else {
                ctx->key = key;
                ctx->have_key = true;
            }
        }
        if (use_graph) CK(cudaGraphLaunch(ctx->exec, ctx->stream));
    }
    if (!use_graph) {
        Runner r{ctx, false};
        ctx->ctl.use_graph = 0;
        body(r);
        if (r.err != cudaSuccess) return cuda_fail(ctx, r.err, "host-loop solve", __LINE__);
    }
    if (ctx->defer_st) {   // the caller reads all items' snapshots after one synchronisation
        state_snapshot_kernel<<<1, 128, 0, ctx->stream>>>(ctx->st, ctx->cfg.batch, ctx->launches, ctx->defer_st,
                                                          ctx->defer_launch);
        CK(cudaGetLastError());
        return HYSCO_OK;
    }
    CK(cudaMemcpyAsync(ctx->h_st, ctx->st, sizeof(PairState) * ctx->cfg.batch, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_launches, ctx->launches, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->last_launches = (long long)*ctx->h_launches;
    return HYSCO_OK;
}

static void fill_reports(hysco_ctx ctx, hysco_report* rep, bool* any_infeasible_start) {
    bool inf = false;
    for (int p = 0; p < ctx->cfg.batch; p++) {
        const PairState& s = ctx->h_st[p];
        if (s.stop_reason == STOP_INFEASIBLE) inf = true;
        if (!rep) continue;
        hysco_report& r = rep[p];
        r.gn_iters = s.gn_k;
        r.f_evals = s.f_evals;
        r.h_evals = s.h_evals;
        r.pcg_iters = s.pcg_iters;
        r.stop_reason = s.stop_reason;
        r.ls_halvings = s.ls_halvings;
        r.J = s.J;
        r.D = s.D;
        r.S = s.S;
        r.P = s.P;
        r.grad_norm = sqrt(s.gnorm2);
        r.last_relres = s.relres;
    }
    if (any_infeasible_start) *any_infeasible_start = inf;
}

template <typename K>
static int occ_blocks(K kernel, int threads, size_t smem) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess || n < 1) n = 1;
    return n;
}

template <typename T>
static hysco_status setup_typed(hysco_ctx ctx) {
    const Geom& g = ctx->g;
    const long long batch = ctx->cfg.batch;
    ctx->smem_eval = eval_smem_elems(g.n3) * sizeof(T);   // eval tile staging
    ctx->smem_apply = apply_smem_elems(g.n3) * sizeof(T);
    ctx->smem_ot = (size_t)8 * 2 * g.P * sizeof(double);
    if (ctx->smem_eval > 227 * 1024 || ctx->smem_ot > 227 * 1024 || ctx->smem_apply > 227 * 1024)
        return set_err(ctx, HYSCO_ERR_SHAPE, "n3 too large for the column-in-shared-memory kernels");
    NCH_SWITCH(pick_nch(g.P), CK(cudaFuncSetAttribute(eval_kernel<T, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)ctx->smem_eval)));
    CK(cudaFuncSetAttribute(apply_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->smem_apply));
    CK(cudaFuncSetAttribute(ot_column_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->smem_ot));
    auto per_pair = [&](long long work_blocks, int occ) {
        long long cap = ((long long)ctx->nsm * occ + batch - 1) / batch;
        long long gx = work_blocks < cap ? work_blocks : cap;
        return (int)(gx < 1 ? 1 : gx);
    };
    ctx->nch = pick_nch(g.P);
    int occ_n = 8, occ_m = 8;
    NCH_SWITCH(ctx->nch, {
        occ_n = occ_blocks(pcg_update_kernel<T, NCH>, 256, 0);
        const int o2 = occ_blocks(pcg_init_kernel<T, NCH>, 256, 0);
        if (o2 < occ_n) occ_n = o2;
        occ_m = occ_blocks(matvec_kernel<T, NCH, true>, 256, 0);
    });
    ctx->gx_nodes = per_pair((g.ncol + 7) / 8, occ_n);
    ctx->gx_mv = per_pair((g.ncol + 7) / 8, occ_m);
    ctx->gx_cells = per_pair((g.Nc + 255) / 256, occ_n);
    int occ_e = 1;
    NCH_SWITCH(ctx->nch, occ_e = occ_blocks(eval_kernel<T, NCH>, 32 * EV_CT, ctx->smem_eval));
    ctx->gx_eval = per_pair((g.ncol + EV_CT - 1) / EV_CT, occ_e);
    ctx->gx_apply = per_pair((g.ncol + 7) / 8, occ_blocks(apply_kernel<T>, 256, ctx->smem_apply));
    const long long flat_blocks = (g.Nn / FlatVec<T>::V + 2 + 255) / 256;
    int occ_f = occ_blocks(pcg_upd_kernel<T>, 256, 0);
    occ_f = std::min(occ_f, occ_blocks(pcg_init_flat_kernel<T>, 256, 0));
    occ_f = std::min(occ_f, occ_blocks(trial_flat_kernel<T>, 256, 0));
    ctx->gx_flat = per_pair(flat_blocks, occ_f);
    ctx->flat = g.P >= FlatVec<T>::V && !getenv_is1("HYSCO_NO_FLAT");
    {   // plane-march F1 (pcg_march_kernel): tiles of <= 16 columns, 5 bulk-copy stages in
        // <= 220 KB of shared memory (one CTA per SM), plane chunks for one wave of CTAs
        const size_t cap = 220 * 1024 / MARCH_CPS;
        int wmax = std::min(g.n2, 16);
        const int mslots = ctx->nsm * MARCH_CPS;   // co-resident march CTAs
        auto fits = [&](int w) {
            return march_ms<T>(w, g.P, MARCH_THREADS) > 0 && march_smem_bytes<T>(march_plan<T>(w, g.P, 5)) <= cap;
        };
        while (wmax > 0 && !fits(wmax)) wmax--;
        if (wmax == 0) {
            ctx->flat = false;
        } else {
            // column tiles: the widest (fewest halo columns, largest copies) unless its
            // nJB x floor(nsm / nJB) tiles leave > 10 % of the SMs idle; then, among
            // nJB up to twice that, the one filling the most SMs (C5: 128 -> 148 CTAs;
            // 7T keeps 14 x 10 = 140, narrower tiles measured slower)
            const int njb0 = (g.n2 + wmax - 1) / wmax;
            auto used = [&](int nj) {
                return nj <= mslots ? nj * std::min(std::max(1, mslots / nj), g.n1) : mslots;
            };
            int best = njb0, bestu = used(njb0);
            if (10 * bestu < 9 * std::min(mslots, g.n1 * njb0))
                for (int nj = njb0 + 1; nj <= std::min(2 * njb0, g.n2); nj++)
                    if (used(nj) > bestu) {
                        bestu = used(nj);
                        best = nj;
                    }
            ctx->mr_njb = best;
            wmax = (g.n2 + ctx->mr_njb - 1) / ctx->mr_njb;
            ctx->mr_plan = march_plan<T>(wmax, g.P, 5);
            ctx->mr_plan.ms = march_ms<T>(wmax, g.P, MARCH_THREADS);
            ctx->smem_mr = march_smem_bytes<T>(ctx->mr_plan);
            auto attr = [&](auto kern) {
                return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->smem_mr);
            };
            CK(attr(pcg_march_kernel<T, true, 2>));
            CK(attr(pcg_march_kernel<T, false, 2>));
            CK(attr(pcg_march_kernel<T, true, 4>));
            CK(attr(pcg_march_kernel<T, false, 4>));
            CK(attr(pcg_march_kernel<T, true, 8>));
            CK(attr(pcg_march_kernel<T, false, 8>));
            CK(attr(pcg_march_kernel<T, true, 12>));
            CK(attr(pcg_march_kernel<T, false, 12>));
            long long ncb = ctx->mr_njb <= mslots ? std::max(1, mslots / ctx->mr_njb) : 1;
            ncb = std::min<long long>(ncb, g.n1);
            ctx->mr_c = (int)((g.n1 + ncb - 1) / ncb);
            ncb = (g.n1 + ctx->mr_c - 1) / ctx->mr_c;
            ctx->gx_dmv = (int)(ctx->mr_njb * ncb);
        }
    }
    ctx->gx_ot = per_pair((g.ncol + 7) / 8, occ_blocks(ot_column_kernel<T>, 256, ctx->smem_ot));
    // one-pair grids (PairView)
    auto one = [&](long long work_blocks, int occ) {
        long long gx = std::min<long long>(work_blocks, (long long)ctx->nsm * occ);
        return (int)(gx < 1 ? 1 : gx);
    };
    ctx->gx1[0] = one((g.ncol + 7) / 8, occ_n);
    ctx->gx1[1] = one((g.ncol + 7) / 8, occ_m);
    ctx->gx1[2] = one((g.Nc + 255) / 256, occ_n);
    ctx->gx1[3] = one((g.ncol + EV_CT - 1) / EV_CT, occ_e);
    ctx->gx1[4] = one((g.ncol + 7) / 8, occ_blocks(apply_kernel<T>, 256, ctx->smem_apply));
    ctx->gx1[5] = one((g.ncol + 7) / 8, occ_blocks(ot_column_kernel<T>, 256, ctx->smem_ot));
    ctx->gx1[6] = one(flat_blocks, occ_f);
    ctx->gx1[7] = ctx->gx_dmv;   // independent of the batch (the tiling is per pair)
    ctx->vb = (int)batch;
    int mx = ctx->gx_nodes;
    for (int v : {ctx->gx_mv, ctx->gx_cells, ctx->gx_eval, ctx->gx_apply, ctx->gx_ot, ctx->gx_flat, ctx->gx_dmv}) mx = v > mx ? v : mx;
    for (int v : ctx->gx1) mx = v > mx ? v : mx;
    ctx->ctl.part_stride = mx * 8;
    return HYSCO_OK;
}

// admm_b_kernel is instantiated per E = ceil(P / 32) <= 8 (register PCR), 0 beyond
#define ADMM_E_SWITCH(e, ...)                                                 \
    switch (e) {                                                              \
        case 1: { constexpr int AE = 1; __VA_ARGS__; } break;                 \
        case 2: { constexpr int AE = 2; __VA_ARGS__; } break;                 \
        case 3: { constexpr int AE = 3; __VA_ARGS__; } break;                 \
        case 4: { constexpr int AE = 4; __VA_ARGS__; } break;                 \
        case 5: { constexpr int AE = 5; __VA_ARGS__; } break;                 \
        case 6: { constexpr int AE = 6; __VA_ARGS__; } break;                 \
        case 7: { constexpr int AE = 7; __VA_ARGS__; } break;                 \
        case 8: { constexpr int AE = 8; __VA_ARGS__; } break;                 \
        default: { constexpr int AE = 0; __VA_ARGS__; } break;                \
    }

template <typename T>
static hysco_status admm_setup(hysco_ctx ctx) {
    if (ctx->admm_ready) return HYSCO_OK;
    const Geom& g = ctx->g;
    int n[2] = {g.n1, g.n2}, ine[2] = {g.n1, g.n2}, one[2] = {g.n1, g.n2 / 2 + 1};
    const bool dbl = sizeof(T) == 8;
    if (cufftPlanMany(&ctx->fft_fwd, 2, n, ine, g.P, 1, one, g.P, 1, dbl ? CUFFT_D2Z : CUFFT_R2C, g.P) != CUFFT_SUCCESS ||
        cufftPlanMany(&ctx->fft_inv, 2, n, one, g.P, 1, ine, g.P, 1, dbl ? CUFFT_Z2D : CUFFT_C2R, g.P) != CUFFT_SUCCESS ||
        cufftSetStream(ctx->fft_fwd, ctx->stream) != CUFFT_SUCCESS ||
        cufftSetStream(ctx->fft_inv, ctx->stream) != CUFFT_SUCCESS)
        return set_err(ctx, HYSCO_ERR_CUDA, "cuFFT plan creation failed");
    const size_t spec = (size_t)g.n1 * (g.n2 / 2 + 1) * g.P;
    CK(cudaMalloc(&ctx->admm_spec, spec * 2 * sizeof(T) * ctx->cfg.batch));
    CK(cudaMalloc(&ctx->admm_rho, sizeof(double) * ctx->cfg.batch));
    CK(cudaMalloc(&ctx->admm_fac, sizeof(double) * ctx->cfg.batch));
    CK(cudaMalloc(&ctx->admm_lam, sizeof(double) * g.n1 * (g.n2 / 2 + 1)));
    CK(cudaMalloc(&ctx->admm_stat, sizeof(double) * 4 * ctx->cfg.batch));
    CK(cudaMalloc(&ctx->admm_done, sizeof(unsigned) * (1 + ctx->cfg.batch)));
    CK(cudaMallocHost(&ctx->h_admm_done, 2 * sizeof(unsigned)));
    for (int k = 0; k < 2; k++) CK(cudaEventCreateWithFlags(&ctx->admm_ev[k], cudaEventDisableTiming));
    admm_lambda_kernel<<<64, 256, 0, ctx->stream>>>(g, ctx->admm_lam);
    CK(cudaGetLastError());
    ctx->admm_smem = (size_t)ADMM_WARPS * admm_warp_elems(g.n3) * sizeof(T);
    if (ctx->admm_smem > 227 * 1024) return set_err(ctx, HYSCO_ERR_SHAPE, "n3 too large for the ADMM column kernel");
    ctx->admm_e = (g.P + 31) / 32 <= 8 ? (g.P + 31) / 32 : 0;
    int occ = 1;
    cudaError_t ea = cudaSuccess;
    ADMM_E_SWITCH(ctx->admm_e,
                  ea = cudaFuncSetAttribute(admm_b_kernel<T, AE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)ctx->admm_smem);
                  if (ea == cudaSuccess &&
                      (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, admm_b_kernel<T, AE>, 32 * ADMM_WARPS,
                                                                     ctx->admm_smem) != cudaSuccess || occ < 1))
                      occ = 1)
    CK(ea);
    const long long work = (g.ncol + ADMM_WARPS - 1) / ADMM_WARPS;
    const long long cap = ((long long)ctx->nsm * occ + ctx->cfg.batch - 1) / ctx->cfg.batch;
    ctx->admm_gx = (int)std::max(1LL, std::min(work, cap));
    ctx->admm_ready = true;
    return HYSCO_OK;
}

template <typename T>
static hysco_status admm_run(hysco_ctx ctx, void* d_b, const hysco_admm_opts& o, hysco_admm_report* reps) {
    if (hysco_status s0 = admm_setup<T>(ctx)) return s0;
    using C = typename std::conditional<sizeof(T) == 8, cufftDoubleComplex, cufftComplex>::type;
    const Geom& g = ctx->g;
    const int B = ctx->cfg.batch;
    const size_t nb = (size_t)B * g.Nn * sizeof(T);
    const long long spec = (long long)g.n1 * (g.n2 / 2 + 1) * g.P;
    cudaStream_t st = ctx->stream;
    T* b = L<T>::b(ctx, B_B);
    T* bprev = L<T>::b(ctx, B_BOLD);
    T* z = L<T>::b(ctx, B_R);
    T* u = L<T>::b(ctx, B_P);
    T* w = L<T>::b(ctx, B_HP);
    T* zn = L<T>::b(ctx, B_TMP);
    C* X = static_cast<C*>(ctx->admm_spec);
    const double rho0 = o.rho0 > 0 ? o.rho0 : g.alpha * (g.ih1sq + g.ih2sq);
    std::vector<double> rho(B, rho0), stat((size_t)4 * B, 0.0);
    CK(cudaMemsetAsync(ctx->launches, 0, sizeof(unsigned long long), st));
    CK(cudaMemcpyAsync(ctx->admm_rho, rho.data(), sizeof(double) * B, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(ctx->admm_done, 0, sizeof(unsigned) * (1 + B), st));
    CK(cudaMemsetAsync(ctx->admm_stat, 0, sizeof(double) * 4 * B, st));
    CK(cudaMemcpyAsync(b, d_b, nb, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(z, d_b, nb, cudaMemcpyDeviceToDevice, st));     // z0 = b0
    CK(cudaMemsetAsync(u, 0, nb, st));                                  // u0 = 0
    const dim3 gb(ctx->admm_gx, B), gn(ctx->gx_cells, B);
    const unsigned* done = ctx->admm_done;
    // The loop runs without a host round trip per iteration: residual balancing
    // and the stop test are admm_balance_kernel's; the host enqueues iteration
    // k after seeing the stop flag of iteration k - 2 (pinned copy + event), so
    // the GPU stays one iteration ahead.  Kernels of an iteration enqueued after
    // the stop are no-ops (only its two cuFFT calls still run, on scratch).
    for (int k = 0; k < o.max_iter; k++) {
        if (!o.fixed_iters && k >= 2) {
            CK(cudaEventSynchronize(ctx->admm_ev[k & 1]));
            if (ctx->h_admm_done[k & 1]) break;
        }
        CK(cudaMemcpyAsync(bprev, b, nb, cudaMemcpyDeviceToDevice, st));
        ADMM_E_SWITCH(ctx->admm_e,
                      admm_b_kernel<T, AE><<<gb, 32 * ADMM_WARPS, ctx->admm_smem, st>>>(
                          g, ctx->ctl, (const T*)ctx->Ip, (const T*)ctx->Im, b, z, u, ctx->admm_rho, o.inner,
                          o.armijo_c1, o.ls_max, o.col_tol, done))
        admm_rhs_kernel<T><<<gn, 256, 0, st>>>(g, ctx->ctl, b, u, w, done);
        for (int p = 0; p < B; p++) {
            cufftResult r = sizeof(T) == 8
                                ? cufftExecD2Z(ctx->fft_fwd, (cufftDoubleReal*)(w + (size_t)p * g.ps),
                                               (cufftDoubleComplex*)(X + (size_t)p * spec))
                                : cufftExecR2C(ctx->fft_fwd, (cufftReal*)(w + (size_t)p * g.ps),
                                               (cufftComplex*)(X + (size_t)p * spec));
            if (r != CUFFT_SUCCESS) return set_err(ctx, HYSCO_ERR_CUDA, "cuFFT forward transform failed");
        }
        admm_zscale_kernel<C><<<gn, 256, 0, st>>>(g, ctx->ctl, X, ctx->admm_rho, ctx->admm_lam, spec, done);
        for (int p = 0; p < B; p++) {
            cufftResult r = sizeof(T) == 8
                                ? cufftExecZ2D(ctx->fft_inv, (cufftDoubleComplex*)(X + (size_t)p * spec),
                                               (cufftDoubleReal*)(zn + (size_t)p * g.ps))
                                : cufftExecC2R(ctx->fft_inv, (cufftComplex*)(X + (size_t)p * spec),
                                               (cufftReal*)(zn + (size_t)p * g.ps));
            if (r != CUFFT_SUCCESS) return set_err(ctx, HYSCO_ERR_CUDA, "cuFFT inverse transform failed");
        }
        admm_u_kernel<T><<<gn, 256, 0, st>>>(g, ctx->ctl, b, bprev, zn, z, u, done);
        admm_balance_kernel<<<1, 256, 0, st>>>(ctx->ctl, B, ctx->admm_rho, ctx->admm_fac, ctx->admm_stat,
                                               ctx->admm_done, k, o.mu, o.tau, o.tol, o.fixed_iters);
        admm_scale_u_kernel<T><<<gn, 256, 0, st>>>(g, ctx->ctl, u, ctx->admm_fac);
        CK(cudaGetLastError());
        if (!o.fixed_iters) {
            CK(cudaMemcpyAsync(&ctx->h_admm_done[k & 1], ctx->admm_done, sizeof(unsigned), cudaMemcpyDeviceToHost,
                               st));
            CK(cudaEventRecord(ctx->admm_ev[k & 1], st));
        }
    }
    CK(cudaMemcpyAsync(stat.data(), ctx->admm_stat, sizeof(double) * 4 * B, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rho.data(), ctx->admm_rho, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(d_b, b, nb, cudaMemcpyDeviceToDevice, st));
    SolveParams sp{};
    L<T>::eval(ctx, sp, EVAL_PLAIN, b);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->h_st, ctx->st, sizeof(PairState) * B, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ctx->h_launches, ctx->launches, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->last_launches = (long long)*ctx->h_launches;   // ADMM kernels + the final evaluation (cuFFT not counted)
    for (int p = 0; p < B; p++) {
        if (!reps) break;
        const PairState& s = ctx->h_st[p];
        reps[p].iters = (int32_t)stat[4 * p + 0];
        reps[p].converged = stat[4 * p + 3] != 0.0;
        reps[p].rho = rho[p];
        reps[p].r_norm = stat[4 * p + 1];
        reps[p].s_norm = stat[4 * p + 2];
        reps[p].J = s.J;
        reps[p].D = s.D;
        reps[p].S = s.S;
        reps[p].P = s.P;
    }
    ctx->state_valid = false;
    return HYSCO_OK;
}

// ---------------------------------------------------------------------------
// ADMM on slabs (NEXT-2 at scale, "could be more scalable for datasets
// of considerably higher resolution"; R21-R26).  The b-update is column-local
// and runs on every rank's slab; the u-update is elementwise with its residual
// norms allreduced before the (identical) residual-balancing decision; the
// z-update -- a 2-D periodic solve over (n1, n2) per PE node l, which the slab
// split along dim 1 cuts -- runs after a transpose: every rank receives all
// n1 planes of its range of PE nodes [l0_r, l1_r) (l split evenly over the
// ranks), layout [n1][n2][Pl] (the batched-R2C layout of the single-context
// path with P -> Pl), transforms, scales, transforms back and returns the
// planes.  Each transpose is one strided 2-D copy per (pair, peer): a device
// copy between the members of a loopback group, NCCL send / receive (with a
// packed staging buffer) across processes.
// ---------------------------------------------------------------------------
struct AdmmSlab {
    int N = 1, me = 0;
    std::vector<int> i0, n1l;      // every rank's planes
    std::vector<int> l0, pl;       // every rank's PE-node range
    int n1g = 0;
    void* wT = nullptr;            // [B][n1g][n2][Pl]   (also the returned z)
    void* spec = nullptr;          // [B][n1g][n2/2+1][Pl] complex
    void* stage = nullptr;         // NCCL: [B][n1_local][n2][P] packing / receive buffer
    double* lam = nullptr;         // [n1g][n2/2+1]
    cufftHandle fwd = 0, inv = 0;
    bool plans = false;
};

static void admm_slab_free(hysco_ctx ctx);

template <typename T>
static hysco_status admm_slab_setup(hysco_ctx ctx, const std::vector<int>& i0, const std::vector<int>& n1l) {
    if (ctx->admm_slab) return HYSCO_OK;
    const Geom& g = ctx->g;
    AdmmSlab* a = new AdmmSlab();
    ctx->admm_slab = a;
    a->N = (int)i0.size();
    a->me = ctx->rank;
    a->i0 = i0;
    a->n1l = n1l;
    a->n1g = g.n1g;
    for (int r = 0; r < a->N; r++) {
        a->l0.push_back((int)((long long)r * g.P / a->N));
        a->pl.push_back((int)((long long)(r + 1) * g.P / a->N) - a->l0.back());
    }
    const int Pl = a->pl[a->me];
    if (Pl < 1) return set_err(ctx, HYSCO_ERR_SHAPE, "slab ADMM needs n3 + 1 >= number of ranks");
    const int B = (int)ctx->cfg.batch;
    const size_t nT = (size_t)a->n1g * g.n2 * Pl, nS = (size_t)a->n1g * (g.n2 / 2 + 1) * Pl;
    CK(cudaMalloc(&a->wT, nT * sizeof(T) * B));
    CK(cudaMalloc(&a->spec, nS * 2 * sizeof(T) * B));
    CK(cudaMalloc(&a->stage, (size_t)g.n1 * g.n2 * g.P * sizeof(T) * B));
    CK(cudaMalloc(&a->lam, sizeof(double) * a->n1g * (g.n2 / 2 + 1)));
    Geom gg = g;
    gg.n1 = a->n1g;                  // the periodic in-plane eigenvalues of the whole volume
    admm_lambda_kernel<<<64, 256, 0, ctx->stream>>>(gg, a->lam);
    CK(cudaGetLastError());
    int n[2] = {a->n1g, g.n2}, ine[2] = {a->n1g, g.n2}, one[2] = {a->n1g, g.n2 / 2 + 1};
    const bool dbl = sizeof(T) == 8;
    if (cufftPlanMany(&a->fwd, 2, n, ine, Pl, 1, one, Pl, 1, dbl ? CUFFT_D2Z : CUFFT_R2C, Pl) != CUFFT_SUCCESS ||
        cufftPlanMany(&a->inv, 2, n, one, Pl, 1, ine, Pl, 1, dbl ? CUFFT_Z2D : CUFFT_C2R, Pl) != CUFFT_SUCCESS ||
        cufftSetStream(a->fwd, ctx->stream) != CUFFT_SUCCESS || cufftSetStream(a->inv, ctx->stream) != CUFFT_SUCCESS)
        return set_err(ctx, HYSCO_ERR_CUDA, "cuFFT plan creation failed (slab ADMM)");
    a->plans = true;
    // the single-context ADMM state (rho, factors, stats, stop flags) is reused
    CK(cudaMalloc(&ctx->admm_rho, sizeof(double) * B));
    CK(cudaMalloc(&ctx->admm_fac, sizeof(double) * B));
    CK(cudaMalloc(&ctx->admm_stat, sizeof(double) * 4 * B));
    CK(cudaMalloc(&ctx->admm_done, sizeof(unsigned) * (1 + B)));
    CK(cudaMallocHost(&ctx->h_admm_done, 2 * sizeof(unsigned)));
    for (int k = 0; k < 2; k++) CK(cudaEventCreateWithFlags(&ctx->admm_ev[k], cudaEventDisableTiming));
    ctx->admm_smem = (size_t)ADMM_WARPS * admm_warp_elems(g.n3) * sizeof(T);
    if (ctx->admm_smem > 227 * 1024) return set_err(ctx, HYSCO_ERR_SHAPE, "n3 too large for the ADMM column kernel");
    ctx->admm_e = (g.P + 31) / 32 <= 8 ? (g.P + 31) / 32 : 0;
    int occ = 1;
    cudaError_t ea = cudaSuccess;
    ADMM_E_SWITCH(ctx->admm_e,
                  ea = cudaFuncSetAttribute(admm_b_kernel<T, AE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)ctx->admm_smem);
                  if (ea == cudaSuccess &&
                      (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, admm_b_kernel<T, AE>, 32 * ADMM_WARPS,
                                                                     ctx->admm_smem) != cudaSuccess || occ < 1))
                      occ = 1)
    CK(ea);
    const long long work = (g.ncol + ADMM_WARPS - 1) / ADMM_WARPS;
    const long long cap = ((long long)ctx->nsm * occ + B - 1) / B;
    ctx->admm_gx = (int)std::max(1LL, std::min(work, cap));
    return HYSCO_OK;
}

// Forward transpose: w (slabs, [n1_r][n2][P] per pair) -> wT of every rank
// ([n1g][n2][Pl_r'] per pair); backward: zT -> zn on the slabs.
template <typename T>
static cudaError_t admm_transpose(std::vector<hysco_ctx>& R, CommBase* comm, bool forward, int kw, int kz) {
    hysco_ctx c0 = R[0];
    const Geom& g = c0->g;
    const size_t es = sizeof(T);
    const int B = (int)c0->cfg.batch;
    NcclComm* nc1 = dynamic_cast<NcclComm*>(comm);
    if (dynamic_cast<LoopbackComm*>(comm) || (nc1 && nc1->n == 1)) {   // all ranks' buffers on this device
        const int N = (int)R.size();
        for (int r = 0; r < N; r++)
            for (int q = 0; q < N; q++) {
                hysco_ctx cr = R[r], cq = R[q];
                AdmmSlab *ar = cr->admm_slab, *aq = cq->admm_slab;
                const size_t nTq = (size_t)aq->n1g * g.n2 * aq->pl[q];
                for (int p = 0; p < B; p++) {
                    T* slab = L<T>::b(cr, forward ? kw : kz) + (size_t)p * cr->g.ps + ar->l0[q];
                    T* tq = static_cast<T*>(aq->wT) + (size_t)p * nTq + (size_t)ar->i0[r] * g.n2 * aq->pl[q];
                    cudaError_t e = forward
                        ? cudaMemcpy2DAsync(tq, aq->pl[q] * es, slab, (size_t)g.P * es, aq->pl[q] * es,
                                            (size_t)cr->g.n1 * g.n2, cudaMemcpyDeviceToDevice, c0->stream)
                        : cudaMemcpy2DAsync(slab, (size_t)g.P * es, tq, aq->pl[q] * es, aq->pl[q] * es,
                                            (size_t)cr->g.n1 * g.n2, cudaMemcpyDeviceToDevice, c0->stream);
                    if (e != cudaSuccess) return e;
                }
            }
        return cudaSuccess;
    }
    NcclComm* nc = dynamic_cast<NcclComm*>(comm);
    if (!nc) return cudaErrorInvalidValue;
    hysco_ctx c = R[0];
    AdmmSlab* a = c->admm_slab;
    const int N = a->N, me = a->me;
    const ncclDataType_t ty = es == 8 ? ncclDouble : ncclFloat;
    const size_t nT = (size_t)a->n1g * g.n2 * a->pl[me];
    const size_t nloc = (size_t)g.n1 * g.n2;      // columns of this slab
    T* st = static_cast<T*>(a->stage);
    for (int p = 0; p < B; p++) {
        T* slab = L<T>::b(c, forward ? kw : kz) + (size_t)p * g.ps;
        T* tme = static_cast<T*>(a->wT) + (size_t)p * nT;
        T* stp = st + (size_t)p * nloc * g.P;     // packed blocks [q][n1_local n2][Pl_q]
        if (forward) {
            for (int q = 0; q < N; q++) {         // pack this slab's l-range of rank q
                cudaError_t e = cudaMemcpy2DAsync(stp + nloc * a->l0[q], a->pl[q] * es, slab + a->l0[q], (size_t)g.P * es,
                                                  a->pl[q] * es, nloc, cudaMemcpyDeviceToDevice, c->stream);
                if (e != cudaSuccess) return e;
            }
            if ((nc->last = ncclGroupStart()) != ncclSuccess) return cudaErrorUnknown;
            for (int q = 0; q < N; q++) {
                nc->last = ncclSend(stp + nloc * a->l0[q], nloc * a->pl[q], ty, q, nc->comm, c->stream);
                nc->last = ncclRecv(tme + (size_t)a->i0[q] * g.n2 * a->pl[me], (size_t)a->n1l[q] * g.n2 * a->pl[me], ty, q,
                                    nc->comm, c->stream);
            }
            if ((nc->last = ncclGroupEnd()) != ncclSuccess) return cudaErrorUnknown;
        } else {
            if ((nc->last = ncclGroupStart()) != ncclSuccess) return cudaErrorUnknown;
            for (int q = 0; q < N; q++) {
                nc->last = ncclSend(tme + (size_t)a->i0[q] * g.n2 * a->pl[me], (size_t)a->n1l[q] * g.n2 * a->pl[me], ty, q,
                                    nc->comm, c->stream);
                nc->last = ncclRecv(stp + nloc * a->l0[q], nloc * a->pl[q], ty, q, nc->comm, c->stream);
            }
            if ((nc->last = ncclGroupEnd()) != ncclSuccess) return cudaErrorUnknown;
            for (int q = 0; q < N; q++) {         // unpack rank q's l-range
                cudaError_t e = cudaMemcpy2DAsync(slab + a->l0[q], (size_t)g.P * es, stp + nloc * a->l0[q], a->pl[q] * es,
                                                  a->pl[q] * es, nloc, cudaMemcpyDeviceToDevice, c->stream);
                if (e != cudaSuccess) return e;
            }
        }
    }
    return cudaSuccess;
}

// Spectrum scaling on the transposed layout [(k1 (n2/2+1) + k2) Pl + l].
template <typename C>
__global__ void __launch_bounds__(256) admm_zscale_t_kernel(Geom g, Ctl c, C* __restrict__ X,
                                                            const double* __restrict__ rho_p,
                                                            const double* __restrict__ lam, int n1g, int Pl,
                                                            long long spec, const unsigned* __restrict__ done) {
    count_launch(c);
    if (done[0] || done[1 + blockIdx.y]) return;
    const int pair = blockIdx.y, lane = threadIdx.x & 31;
    const double rho = rho_p[pair];
    const long long nk = (long long)n1g * (g.n2 / 2 + 1);
    const double sc = 1.0 / ((double)n1g * g.n2);
    C* Xp = X + (size_t)pair * spec;
    for (long long kk = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); kk < nk;
         kk += (long long)gridDim.x * (blockDim.x >> 5)) {
        const double f = rho / (g.alpha * lam[kk] + rho) * sc;
        C* row = Xp + kk * Pl;
        for (int l = lane; l < Pl; l += 32) {
            row[l].x *= f;
            row[l].y *= f;
        }
    }
}

template <typename T>
static hysco_status admm_slab_run(std::vector<hysco_ctx>& R, CommBase* comm, const hysco_admm_opts& o,
                                  void* const* d_b, hysco_admm_report* reps) {
    using C = typename std::conditional<sizeof(T) == 8, cufftDoubleComplex, cufftComplex>::type;
    hysco_ctx c0 = R[0];
    const int B = (int)c0->cfg.batch;
    // every rank's planes: loopback members directly, NCCL ranks by an allgather
    std::vector<int> i0, n1l;
    if (dynamic_cast<LoopbackComm*>(comm)) {
        for (hysco_ctx c : R) {
            i0.push_back(c->g.i0);
            n1l.push_back(c->g.n1);
        }
    } else {
        NcclComm* nc = dynamic_cast<NcclComm*>(comm);
        if (!nc) return set_err(c0, HYSCO_ERR_STATE, "slab ADMM needs a loopback group or an NCCL slab context");
        i0.assign(nc->n, 0);
        n1l.assign(nc->n, 0);
        if (nc->n == 1) {
            i0[0] = c0->g.i0;
            n1l[0] = c0->g.n1;
        } else if (!c0->admm_slab) {
            int* d = nullptr;
            CK_C(c0, cudaMalloc(&d, sizeof(int) * 2 * (nc->n + 1)));
            int mine[2] = {c0->g.i0, c0->g.n1};
            CK_C(c0, cudaMemcpy(d, mine, sizeof mine, cudaMemcpyHostToDevice));
            if ((nc->last = ncclAllGather(d, d + 2, 2, ncclInt32, nc->comm, c0->stream)) != ncclSuccess) {
                cudaFree(d);
                return set_err(c0, HYSCO_ERR_NCCL, "ncclAllGather of the slab bounds failed");
            }
            std::vector<int> h(2 * nc->n);
            CK_C(c0, cudaMemcpyAsync(h.data(), d + 2, sizeof(int) * 2 * nc->n, cudaMemcpyDeviceToHost, c0->stream));
            CK_C(c0, cudaStreamSynchronize(c0->stream));
            cudaFree(d);
            for (int r = 0; r < nc->n; r++) {
                i0[r] = h[2 * r];
                n1l[r] = h[2 * r + 1];
            }
        }
    }
    for (hysco_ctx c : R)
        if (hysco_status s = admm_slab_setup<T>(c, i0, n1l)) return s;
    const Geom& g = c0->g;
    const double rho0 = o.rho0 > 0 ? o.rho0 : g.alpha * (g.ih1sq + g.ih2sq);
    std::vector<double> rho(B, rho0), stat((size_t)4 * B, 0.0);
    cudaError_t err = cudaSuccess;
    auto ok = [&](cudaError_t e) {
        if (err == cudaSuccess && e != cudaSuccess) err = e;
    };
    for (size_t r = 0; r < R.size(); r++) {
        hysco_ctx c = R[r];
        const size_t nbl = (size_t)B * c->g.Nn * sizeof(T);
        ok(cudaMemsetAsync(c->launches, 0, sizeof(unsigned long long), c->stream));
        ok(cudaMemcpyAsync(c->admm_rho, rho.data(), sizeof(double) * B, cudaMemcpyHostToDevice, c->stream));
        ok(cudaMemsetAsync(c->admm_done, 0, sizeof(unsigned) * (1 + B), c->stream));
        ok(cudaMemsetAsync(c->admm_stat, 0, sizeof(double) * 4 * B, c->stream));
        ok(copy_nodes(c, c->buf[B_B], d_b[r], true, cudaMemcpyDeviceToDevice));
        ok(copy_nodes(c, c->buf[B_R], d_b[r], true, cudaMemcpyDeviceToDevice));   // z0 = b0
        for (int p = 0; p < B; p++)                                                 // u0 = 0
            ok(cudaMemsetAsync(L<T>::b(c, B_P) + (size_t)p * c->g.ps, 0, c->g.Nn * sizeof(T), c->stream));
        (void)nbl;
    }
    for (int k = 0; k < o.max_iter && err == cudaSuccess; k++) {
        if (!o.fixed_iters && k >= 2) {      // every rank holds the same stop flags (identical decisions)
            ok(cudaEventSynchronize(c0->admm_ev[k & 1]));
            if (c0->h_admm_done[k & 1]) break;
        }
        for (hysco_ctx c : R) {
            const dim3 gb(c->admm_gx, B), gn(c->gx_cells, B);
            for (int p = 0; p < B; p++)
                ok(cudaMemcpyAsync(L<T>::b(c, B_BOLD) + (size_t)p * c->g.ps, L<T>::b(c, B_B) + (size_t)p * c->g.ps,
                                   c->g.Nn * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
            ADMM_E_SWITCH(c->admm_e,
                          admm_b_kernel<T, AE><<<gb, 32 * ADMM_WARPS, c->admm_smem, c->stream>>>(
                              c->g, c->ctl, (const T*)c->Ip, (const T*)c->Im, L<T>::b(c, B_B), L<T>::b(c, B_R),
                              L<T>::b(c, B_P), c->admm_rho, o.inner, o.armijo_c1, o.ls_max, o.col_tol, c->admm_done))
            admm_rhs_kernel<T><<<gn, 256, 0, c->stream>>>(c->g, c->ctl, L<T>::b(c, B_B), L<T>::b(c, B_P),
                                                           L<T>::b(c, B_HP), c->admm_done);
        }
        ok(cudaGetLastError());
        ok(admm_transpose<T>(R, comm, true, B_HP, B_TMP));
        for (hysco_ctx c : R) {
            AdmmSlab* a = c->admm_slab;
            const int Pl = a->pl[a->me];
            const long long nT = (long long)a->n1g * g.n2 * Pl, nS = (long long)a->n1g * (g.n2 / 2 + 1) * Pl;
            for (int p = 0; p < B; p++) {
                T* wt = static_cast<T*>(a->wT) + (size_t)p * nT;
                C* X = static_cast<C*>(a->spec) + (size_t)p * nS;
                cufftResult r = sizeof(T) == 8 ? cufftExecD2Z(a->fwd, (cufftDoubleReal*)wt, (cufftDoubleComplex*)X)
                                               : cufftExecR2C(a->fwd, (cufftReal*)wt, (cufftComplex*)X);
                if (r != CUFFT_SUCCESS) return set_err(c, HYSCO_ERR_CUDA, "cuFFT forward transform failed (slab)");
            }
            admm_zscale_t_kernel<C><<<dim3(c->gx_cells, B), 256, 0, c->stream>>>(
                c->g, c->ctl, static_cast<C*>(a->spec), c->admm_rho, a->lam, a->n1g, Pl, nS, c->admm_done);
            for (int p = 0; p < B; p++) {
                T* wt = static_cast<T*>(a->wT) + (size_t)p * nT;
                C* X = static_cast<C*>(a->spec) + (size_t)p * nS;
                cufftResult r = sizeof(T) == 8 ? cufftExecZ2D(a->inv, (cufftDoubleComplex*)X, (cufftDoubleReal*)wt)
                                               : cufftExecC2R(a->inv, (cufftComplex*)X, (cufftReal*)wt);
                if (r != CUFFT_SUCCESS) return set_err(c, HYSCO_ERR_CUDA, "cuFFT inverse transform failed (slab)");
            }
        }
        ok(cudaGetLastError());
        ok(admm_transpose<T>(R, comm, false, B_HP, B_TMP));   // z_new on the slabs
        for (hysco_ctx c : R) {
            const dim3 gn(c->gx_cells, B);
            admm_u_kernel<T><<<gn, 256, 0, c->stream>>>(c->g, c->ctl, L<T>::b(c, B_B), L<T>::b(c, B_BOLD),
                                                         L<T>::b(c, B_TMP), L<T>::b(c, B_R), L<T>::b(c, B_P),
                                                         c->admm_done);
        }
        ok(cudaGetLastError());
        ok(comm->allreduce(R, false));        // residual norms of the whole volume
        for (hysco_ctx c : R) {
            const dim3 gn(c->gx_cells, B);
            admm_balance_kernel<<<1, 256, 0, c->stream>>>(c->ctl, B, c->admm_rho, c->admm_fac, c->admm_stat,
                                                           c->admm_done, k, o.mu, o.tau, o.tol, o.fixed_iters);
            admm_scale_u_kernel<T><<<gn, 256, 0, c->stream>>>(c->g, c->ctl, L<T>::b(c, B_P), c->admm_fac);
        }
        ok(cudaGetLastError());
        if (!o.fixed_iters) {
            ok(cudaMemcpyAsync(&c0->h_admm_done[k & 1], c0->admm_done, sizeof(unsigned), cudaMemcpyDeviceToHost,
                               c0->stream));
            ok(cudaEventRecord(c0->admm_ev[k & 1], c0->stream));
        }
    }
    // b out, then the objective of the result (slab evaluation: halo, allreduce, decision)
    for (size_t r = 0; r < R.size(); r++) ok(copy_nodes(R[r], d_b[r], R[r]->buf[B_B], false, cudaMemcpyDeviceToDevice));
    {
        SegExec x{c0};
        x.graph = false;
        SolveParams sp{};
        SlabRun<T> run{R, comm, sp, x};
        run.eval(EVAL_PLAIN);
        ok(run.err);
    }
    ok(cudaMemcpyAsync(stat.data(), c0->admm_stat, sizeof(double) * 4 * B, cudaMemcpyDeviceToHost, c0->stream));
    ok(cudaMemcpyAsync(rho.data(), c0->admm_rho, sizeof(double) * B, cudaMemcpyDeviceToHost, c0->stream));
    for (hysco_ctx c : R) {
        ok(cudaMemcpyAsync(c->h_st, c->st, sizeof(PairState) * B, cudaMemcpyDeviceToHost, c->stream));
        ok(cudaMemcpyAsync(c->h_launches, c->launches, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    }
    for (hysco_ctx c : R) ok(cudaStreamSynchronize(c->stream));
    if (err != cudaSuccess) {
        const bool nccl = dynamic_cast<NcclComm*>(comm) && static_cast<NcclComm*>(comm)->last != ncclSuccess;
        for (hysco_ctx c : R) cuda_fail(c, err, nccl ? "slab ADMM (NCCL)" : "slab ADMM", __LINE__);
        return nccl ? HYSCO_ERR_NCCL : HYSCO_ERR_CUDA;
    }
    for (hysco_ctx c : R) {
        c->last_launches = (long long)*c->h_launches;
        c->state_valid = false;
    }
    for (int p = 0; p < B && reps; p++) {
        const PairState& s = c0->h_st[p];
        reps[p].iters = (int32_t)stat[4 * p + 0];
        reps[p].converged = stat[4 * p + 3] != 0.0;
        reps[p].rho = rho[p];
        reps[p].r_norm = stat[4 * p + 1];
        reps[p].s_norm = stat[4 * p + 2];
        reps[p].J = s.J;
        reps[p].D = s.D;
        reps[p].S = s.S;
        reps[p].P = s.P;
    }
    return HYSCO_OK;
}

static void admm_slab_free(hysco_ctx ctx) {
    AdmmSlab* a = ctx->admm_slab;
    if (!a) return;
    if (a->plans) {
        cufftDestroy(a->fwd);
        cufftDestroy(a->inv);
    }
    for (void* q : {a->wT, a->spec, a->stage, (void*)a->lam})
        if (q) cudaFree(q);
    delete a;
    ctx->admm_slab = nullptr;
}

extern "C" {

void hysco_default_solve_opts(hysco_solve_opts* o) {
    if (!o) return;
    o->max_gn = 10;
    o->max_pcg = 10;
    o->pcg_rtol = 0.1;
    o->fixed_iters = 1;
    o->ls_max = 10;
    o->armijo_c1 = 1e-4;
    o->tol_grad_rel = 1e-2;
    o->tol_dJ_rel = 1e-4;
    o->tol_db_rel = 1e-3;
    o->armijo = 1;
    o->precond = HYSCO_PRECOND_JACOBI;
}

void hysco_default_ot_opts(hysco_ot_opts* o) {
    if (!o) return;
    o->eps = 1e-3;
    o->blur = 1;
    o->feas_cap = 0.95;
}

int32_t hysco_version(void) { return 1; }

}  // extern "C"

// Slab of a multi-rank decomposition along dim 1.
struct SlabSpec {
    int rank, nranks;
    long long n1g, i0;
};

static hysco_status create_impl(const hysco_config* cfg, const SlabSpec* slab, void* cuda_stream, hysco_ctx* out) {
    if (!cfg || !out) return HYSCO_ERR_ARG;
    *out = nullptr;
    if (cfg->n1 < 1 || cfg->n2 < 1 || cfg->n3 < 2 || cfg->batch < 1 || cfg->n3 > 8192 ||
        cfg->n1 * cfg->n2 * (cfg->n3 + 1) > (1ll << 40))
        return HYSCO_ERR_SHAPE;
    if (!(cfg->h1 > 0 && cfg->h2 > 0 && cfg->h3 > 0) || !(cfg->alpha >= 0) || !(cfg->beta >= 0))
        return HYSCO_ERR_ARG;
    if (cfg->dtype != HYSCO_F32 && cfg->dtype != HYSCO_F64) return HYSCO_ERR_ARG;
    hysco_ctx ctx = new hysco_ctx_s();
    ctx->cfg = *cfg;
    ctx->esz = cfg->dtype == HYSCO_F64 ? 8 : 4;
    const char* ng = getenv("HYSCO_NO_GRAPH");
    ctx->no_graph = ng && ng[0] == '1';
    Geom& g = ctx->g;
    g.n1 = (int)cfg->n1;
    g.n2 = (int)cfg->n2;
    g.n3 = (int)cfg->n3;
    g.P = g.n3 + 1;
    g.ncol = cfg->n1 * cfg->n2;
    g.Nc = g.ncol * g.n3;
    g.Nn = g.ncol * g.P;
    g.h1 = cfg->h1;
    g.h2 = cfg->h2;
    g.h3 = cfg->h3;
    g.hd = cfg->h1 * cfg->h2 * cfg->h3;
    g.alpha = cfg->alpha;
    g.beta = cfg->beta;
    g.ahd = cfg->alpha * g.hd;
    g.bh2 = 0.5 * cfg->beta * g.hd;
    g.ih1sq = 1.0 / (cfg->h1 * cfg->h1);
    g.ih2sq = 1.0 / (cfg->h2 * cfg->h2);
    g.ih3sq = 1.0 / (cfg->h3 * cfg->h3);
    g.ih3 = 1.0 / cfg->h3;
    geom_finish(g);
    g.ps = g.Nn;
    g.i0 = 0;
    g.n1g = g.n1;
    g.slab = 0;
    if (slab) {
        if (slab->nranks < 1 || slab->rank < 0 || slab->rank >= slab->nranks || slab->i0 < 0 ||
            slab->i0 + cfg->n1 > slab->n1g) {
            delete ctx;
            return HYSCO_ERR_SHAPE;
        }
        g.i0 = (int)slab->i0;
        g.n1g = (int)slab->n1g;
        g.slab = 1;
        g.ps = (long long)(g.n1 + 2) * g.n2 * g.P;      // one halo plane below and above
        ctx->plane_off = (size_t)g.n2 * g.P;
        ctx->rank = slab->rank;
        ctx->nranks = slab->nranks;
    }

    hysco_status st;
    auto bail = [&](hysco_status s) {
        hysco_destroy(ctx);
        return s;
    };
    {
        cudaError_t e = cudaSetDevice(cfg->device);
        if (e != cudaSuccess) return bail(cuda_fail(ctx, e, "cudaSetDevice", __LINE__));
        e = cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, cfg->device);
        if (e != cudaSuccess) return bail(cuda_fail(ctx, e, "cudaDeviceGetAttribute", __LINE__));
        if (cuda_stream) {
            ctx->stream = (cudaStream_t)cuda_stream;
        } else {
            e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
            if (e != cudaSuccess) return bail(cuda_fail(ctx, e, "cudaStreamCreate", __LINE__));
            ctx->own_stream = true;
        }
    }
    st = cfg->dtype == HYSCO_F64 ? setup_typed<double>(ctx) : setup_typed<float>(ctx);
    if (st != HYSCO_OK) return bail(st);
    const size_t nn = (size_t)cfg->batch * g.ps * ctx->esz, nc = (size_t)cfg->batch * g.Nc * ctx->esz;
    auto dalloc = [&](void** p, size_t n) -> bool {
        cudaError_t e = cudaMalloc(p, n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            ctx->err = "cudaMalloc failed";
            return false;
        }
        return true;
    };
    for (int k = 0; k < NBUF; k++) {   // FLAT_GUARD elements of slack on both sides (hysco_flat.cuh)
        if (!dalloc(&ctx->raw[k], nn + 2 * FLAT_GUARD * ctx->esz)) return bail(HYSCO_ERR_NOMEM);
        cudaMemset(ctx->raw[k], 0, FLAT_GUARD * ctx->esz);
        cudaMemset(static_cast<char*>(ctx->raw[k]) + FLAT_GUARD * ctx->esz + nn, 0, FLAT_GUARD * ctx->esz);
        ctx->buf[k] = static_cast<char*>(ctx->raw[k]) + FLAT_GUARD * ctx->esz;
    }
    if (!dalloc(&ctx->own_Ip, nc) || !dalloc(&ctx->own_Im, nc) || !dalloc(&ctx->own_Tp, nc) ||
        !dalloc(&ctx->own_Tm, nc))
        return bail(HYSCO_ERR_NOMEM);
    if (!dalloc((void**)&ctx->st, sizeof(PairState) * cfg->batch) ||
        !dalloc((void**)&ctx->part, sizeof(double) * ctx->ctl.part_stride * cfg->batch) ||
        !dalloc((void**)&ctx->ctr, sizeof(unsigned) * cfg->batch) || !dalloc((void**)&ctx->gctr, sizeof(unsigned)) ||
        !dalloc((void**)&ctx->launches, sizeof(unsigned long long)) ||
        !dalloc((void**)&ctx->dcond, sizeof(unsigned) * NCOND) ||
        !dalloc((void**)&ctx->red, sizeof(double) * 2 * RED_W * cfg->batch) ||
        !dalloc((void**)&ctx->hist, sizeof(HistRec) * HIST_MAX * cfg->batch))
        return bail(HYSCO_ERR_NOMEM);
    if (g.slab)   // halo planes must start at zero (Neumann ends never read them, blur ring does)
        for (int k = 0; k < NBUF; k++) cudaMemset(ctx->buf[k], 0, nn);
    if (cudaMallocHost((void**)&ctx->h_st, sizeof(PairState) * cfg->batch) != cudaSuccess ||
        cudaMallocHost((void**)&ctx->h_launches, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMallocHost((void**)&ctx->h_cond, sizeof(unsigned) * NCOND) != cudaSuccess) {
        cudaGetLastError();
        return bail(HYSCO_ERR_NOMEM);
    }
    cudaMemset(ctx->st, 0, sizeof(PairState) * cfg->batch);
    cudaMemset(ctx->ctr, 0, sizeof(unsigned) * cfg->batch);
    cudaMemset(ctx->gctr, 0, sizeof(unsigned));
    cudaMemset(ctx->launches, 0, sizeof(unsigned long long));
    cudaMemset(ctx->dcond, 0, sizeof(unsigned) * NCOND);
    {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return bail(cuda_fail(ctx, e, "create sync", __LINE__));
    }
    ctx->ctl.st = ctx->st;
    ctx->ctl.part = ctx->part;
    ctx->ctl.ctr = ctx->ctr;
    ctx->ctl.gctr = ctx->gctr;
    ctx->ctl.launches = ctx->launches;
    ctx->ctl.dcond = ctx->dcond;
    ctx->ctl.use_graph = 0;
    ctx->ctl.red = ctx->red;
    ctx->ctl.hist = ctx->hist;
    cudaMemset(ctx->hist, 0, sizeof(HistRec) * HIST_MAX * cfg->batch);
    ctx->ctl.defer = g.slab ? 1 : 0;     // slab runs are host-orchestrated: always decide after the allreduce
    if (!g.slab) setup_resident(ctx);
    if (!g.slab) {
        if (cfg->dtype == HYSCO_F64) setup_l2pcg<double>(ctx);
        else setup_l2pcg<float>(ctx);
    }
    *out = ctx;
    return HYSCO_OK;
}


// ---- push-forward simulation / least-squares correction (NEXT-3, R27-R29) ----
template <typename T, typename K>
static hysco_status lsq_grid(hysco_ctx ctx, K kern, int nT, int* gx, size_t* smem) {
    const Geom& g = ctx->g;
    *smem = (size_t)LSQ_WARPS * lsq_warp_bytes<T>(g.n3, nT);
    if (*smem > 227 * 1024) return set_err(ctx, HYSCO_ERR_SHAPE, "n3 too large for the least-squares column kernels");
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem));
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * LSQ_WARPS, *smem) != cudaSuccess || occ < 1)
        occ = 1;
    const long long work = (g.ncol + LSQ_WARPS - 1) / LSQ_WARPS;
    const long long cap = ((long long)ctx->nsm * occ + ctx->cfg.batch - 1) / ctx->cfg.batch;
    *gx = (int)std::max(1LL, std::min(work, cap));
    return HYSCO_OK;
}

template <typename T>
static hysco_status push_forward_run(hysco_ctx ctx, const void* b, const void* t, void* ip, void* im) {
    int gx;
    size_t smem;
    if (hysco_status s = lsq_grid<T>(ctx, push_forward_kernel<T>, 6, &gx, &smem)) return s;
    const int B = ctx->cfg.batch;
    CK(cudaMemsetAsync(ctx->red, 0, sizeof(double) * RED_W * B, ctx->stream));
    CK(cudaMemsetAsync(ctx->launches, 0, sizeof(unsigned long long), ctx->stream));
    push_forward_kernel<T><<<dim3(gx, B), 32 * LSQ_WARPS, smem, ctx->stream>>>(
        ctx->g, ctx->ctl, (const T*)b, (const T*)t, (T*)ip, (T*)im);
    CK(cudaGetLastError());
    std::vector<double> red((size_t)B * RED_W);
    CK(cudaMemcpyAsync(red.data(), ctx->red, sizeof(double) * B * RED_W, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_launches, ctx->launches, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->last_launches = (long long)*ctx->h_launches;
    for (int p = 0; p < B; p++)
        if (red[(size_t)p * RED_W + LSQ_ST_INFEAS] > 0) return HYSCO_INFEASIBLE;
    return HYSCO_OK;
}

template <typename T>
static hysco_status lsq_run(hysco_ctx ctx, const void* b, const hysco_lsq_opts& o, void* tout,
                            hysco_lsq_report* reps) {
    int gx;
    size_t smem;
    if (hysco_status s = lsq_grid<T>(ctx, lsq_kernel<T>, 9, &gx, &smem)) return s;
    const int B = ctx->cfg.batch;
    const double rtol = o.rtol > 0 ? o.rtol : (sizeof(T) == 8 ? 1e-12 : 1e-6);
    CK(cudaMemsetAsync(ctx->red, 0, sizeof(double) * RED_W * B, ctx->stream));
    CK(cudaMemsetAsync(ctx->launches, 0, sizeof(unsigned long long), ctx->stream));
    lsq_kernel<T><<<dim3(gx, B), 32 * LSQ_WARPS, smem, ctx->stream>>>(
        ctx->g, ctx->ctl, (const T*)b, (const T*)ctx->Ip, (const T*)ctx->Im, (T*)tout, o.lambda, o.max_iter, rtol);
    CK(cudaGetLastError());
    std::vector<double> red((size_t)B * RED_W);
    CK(cudaMemcpyAsync(red.data(), ctx->red, sizeof(double) * B * RED_W, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_launches, ctx->launches, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->last_launches = (long long)*ctx->h_launches;
    bool infeas = false;
    for (int p = 0; p < B; p++) {
        const double* t = &red[(size_t)p * RED_W];
        if (reps) {
            reps[p].max_iters = (int32_t)t[LSQ_ST_ITERS];
            reps[p].unconverged = (int64_t)t[LSQ_ST_UNCONV];
            reps[p].infeasible = (int64_t)t[LSQ_ST_INFEAS];
            reps[p].max_relres = t[LSQ_ST_RELRES];
        }
        infeas |= t[LSQ_ST_INFEAS] > 0;
    }
    return infeas ? HYSCO_INFEASIBLE : HYSCO_OK;
}

extern "C" {

hysco_status hysco_create(const hysco_config* cfg, void* cuda_stream, hysco_ctx* out) {
    return create_impl(cfg, nullptr, cuda_stream, out);
}

hysco_status hysco_bind_images(hysco_ctx ctx, const void* d_Iplus, const void* d_Iminus) {
    CHECK_CTX();
    if (!d_Iplus || !d_Iminus || !aligned16(d_Iplus) || !aligned16(d_Iminus))
        return set_err(ctx, HYSCO_ERR_ARG, "image pointers must be non-NULL and 16-byte aligned");
    // (graphs bake the image pointers; the cache key holds them)
    ctx->Ip = d_Iplus;
    ctx->Im = d_Iminus;
    ctx->state_valid = false;
    return HYSCO_OK;
}

static hysco_status need_images(hysco_ctx ctx) {
    if (!ctx->Ip || !ctx->Im) return set_err(ctx, HYSCO_ERR_STATE, "no images bound (hysco_bind_images)");
    return HYSCO_OK;
}

hysco_status hysco_ot_init(hysco_ctx ctx, const hysco_ot_opts* opts, void* d_b_out) {
    NvtxRange nvtx_("hysco_ot_init");
    CHECK_CTX();
    if (ctx->g.slab) return set_err(ctx, HYSCO_ERR_STATE, "slab contexts support solve / correct / correct_host");
    if (hysco_status s = need_images(ctx)) return s;
    if (!d_b_out || !aligned16(d_b_out)) return set_err(ctx, HYSCO_ERR_ARG, "d_b_out must be 16-byte aligned");
    hysco_ot_opts o;
    hysco_default_ot_opts(&o);
    if (opts) o = *opts;
    hysco_solve_opts so;
    hysco_default_solve_opts(&so);
    if (hysco_status s = check_opts(ctx, so, o)) return s;
    SolveParams sp = to_params(so, o);
    if (ctx->cfg.dtype == HYSCO_F64) L<double>::ot(ctx, sp, o.blur);
    else L<float>::ot(ctx, sp, o.blur);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(d_b_out, ctx->buf[B_B], (size_t)ctx->cfg.batch * ctx->g.Nn * ctx->esz,
                       cudaMemcpyDeviceToDevice, ctx->stream));
    return HYSCO_OK;
}

hysco_status hysco_objective_grad(hysco_ctx ctx, const void* d_b, double* JDSP, void* d_grad) {
    NvtxRange nvtx_("hysco_objective_grad");
    CHECK_CTX();
    if (ctx->g.slab) return set_err(ctx, HYSCO_ERR_STATE, "slab contexts support solve / correct / correct_host");
    if (hysco_status s = need_images(ctx)) return s;
    if (!d_b || !aligned16(d_b) || (d_grad && !aligned16(d_grad)))
        return set_err(ctx, HYSCO_ERR_ARG, "pointers must be 16-byte aligned");
    const size_t nb = (size_t)ctx->cfg.batch * ctx->g.Nn * ctx->esz;
    SolveParams sp{};
    CK(cudaMemcpyAsync(ctx->buf[B_B], d_b, nb, cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->cfg.dtype == HYSCO_F64) L<double>::eval(ctx, sp, EVAL_PLAIN, (const double*)ctx->buf[B_B]);
    else L<float>::eval(ctx, sp, EVAL_PLAIN, (const float*)ctx->buf[B_B]);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->h_st, ctx->st, sizeof(PairState) * ctx->cfg.batch, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    bool inf = false;
    for (int p = 0; p < ctx->cfg.batch; p++) {
        const PairState& s = ctx->h_st[p];
        inf = inf || s.infeasible;
        if (JDSP) {
            JDSP[4 * p + 0] = s.J;
            JDSP[4 * p + 1] = s.D;
            JDSP[4 * p + 2] = s.S;
            JDSP[4 * p + 3] = s.P;
        }
    }
    ctx->state_valid = !inf;
    if (inf) return HYSCO_INFEASIBLE;
    if (d_grad) {
        CK(cudaMemcpyAsync(d_grad, ctx->buf[B_GRAD], nb, cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return HYSCO_OK;
}

hysco_status hysco_hessvec(hysco_ctx ctx, const void* d_q, void* d_Hq) {
    NvtxRange nvtx_("hysco_hessvec");
    CHECK_CTX();
    if (ctx->g.slab) return set_err(ctx, HYSCO_ERR_STATE, "slab contexts support solve / correct / correct_host");
    if (!ctx->state_valid) return set_err(ctx, HYSCO_ERR_STATE, "hessvec needs a feasible objective_grad first");
    if (!d_q || !d_Hq || !aligned16(d_q) || !aligned16(d_Hq) || d_q == d_Hq)
        return set_err(ctx, HYSCO_ERR_ARG, "d_q/d_Hq must be distinct, 16-byte aligned");
    if (ctx->cfg.dtype == HYSCO_F64) L<double>::matvec_plain(ctx, (const double*)d_q, (double*)d_Hq);
    else L<float>::matvec_plain(ctx, (const float*)d_q, (float*)d_Hq);
    CK(cudaGetLastError());
    return HYSCO_OK;
}

hysco_status hysco_hess_diag(hysco_ctx ctx, void* d_diag) {
    NvtxRange nvtx_("hysco_hess_diag");
    CHECK_CTX();
    if (ctx->g.slab) return set_err(ctx, HYSCO_ERR_STATE, "slab contexts support solve / correct / correct_host");
    if (!ctx->state_valid) return set_err(ctx, HYSCO_ERR_STATE, "hess_diag needs a feasible objective_grad first");
    if (!d_diag || !aligned16(d_diag)) return set_err(ctx, HYSCO_ERR_ARG, "d_diag must be 16-byte aligned");
    if (ctx->cfg.dtype == HYSCO_F64) L<double>::diag(ctx, (double*)d_diag);
    else L<float>::diag(ctx, (float*)d_diag);
    CK(cudaGetLastError());
    return HYSCO_OK;
}

hysco_status hysco_precond_solve(hysco_ctx ctx, int kind, const void* d_r, void* d_z) {
    NvtxRange nvtx_("hysco_precond_solve");
    CHECK_CTX();
    if (ctx->g.slab) return set_err(ctx, HYSCO_ERR_STATE, "slab contexts support solve / correct / correct_host");
    if (!ctx->state_valid) return set_err(ctx, HYSCO_ERR_STATE, "precond_solve needs a feasible objective_grad first");
    if (!d_r || !d_z || !aligned16(d_r) || !aligned16(d_z) || d_r == d_z)
        return set_err(ctx, HYSCO_ERR_ARG, "d_r, d_z must be distinct 16-byte aligned device pointers");
    if (kind != HYSCO_PRECOND_JACOBI && kind != HYSCO_PRECOND_PE_BLOCK)
        return set_err(ctx, HYSCO_ERR_ARG, "bad preconditioner kind");
    const size_t nb = (size_t)ctx->cfg.batch * ctx->g.Nn * ctx->esz;
    if (kind == HYSCO_PRECOND_JACOBI) {   // z = r / diag(H_J): diag into B_TMP, then divide
        if (ctx->cfg.dtype == HYSCO_F64) {
            L<double>::diag(ctx, L<double>::b(ctx, B_TMP));
            jacobi_div_kernel<double><<<dim3(ctx->gx_nodes, ctx->cfg.batch), 256, 0, ctx->stream>>>(
                ctx->g, ctx->ctl, (const double*)d_r, L<double>::b(ctx, B_TMP), (double*)d_z);
        } else {
            L<float>::diag(ctx, L<float>::b(ctx, B_TMP));
            jacobi_div_kernel<float><<<dim3(ctx->gx_nodes, ctx->cfg.batch), 256, 0, ctx->stream>>>(
                ctx->g, ctx->ctl, (const float*)d_r, L<float>::b(ctx, B_TMP), (float*)d_z);
        }
    } else if (ctx->cfg.dtype == HYSCO_F64) {
        L<double>::bfac(ctx, 0);
        L<double>::psolve(ctx, (const double*)d_r, (double*)d_z);
    } else {
        L<float>::bfac(ctx, 0);
        L<float>::psolve(ctx, (const float*)d_r, (float*)d_z);
    }
    (void)nb;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    return HYSCO_OK;
}

void hysco_default_admm_opts(hysco_admm_opts* o) {
    if (!o) return;
    o->max_iter = 20;
    o->inner = 2;
    o->ls_max = 10;
    o->fixed_iters = 0;
    o->tol = 1e-3;
    o->rho0 = 0.0;
    o->mu = 10.0;
    o->tau = 2.0;
    o->armijo_c1 = 1e-4;
    o->col_tol = 1e-6;
}

hysco_status hysco_admm(hysco_ctx ctx, void* d_b_inout, const hysco_admm_opts* opts, hysco_admm_report* reports) {
    NvtxRange nvtx_("hysco_admm");
    CHECK_CTX();
    if (hysco_status s = need_images(ctx)) return s;
    if (!d_b_inout || !aligned16(d_b_inout)) return set_err(ctx, HYSCO_ERR_ARG, "d_b_inout must be 16-byte aligned");
    hysco_admm_opts o;
    hysco_default_admm_opts(&o);
    if (opts) o = *opts;
    if (o.max_iter < 0 || o.inner < 1 || o.ls_max < 1 || !(o.tol >= 0) || !(o.mu > 1) || !(o.tau > 1))
        return set_err(ctx, HYSCO_ERR_ARG, "bad hysco_admm_opts");
    if (ctx->g.slab) {   // one rank of a multi-process slab group (NCCL transposes)
        if (!dynamic_cast<NcclComm*>(ctx->comm))
            return set_err(ctx, HYSCO_ERR_STATE, "loopback slab contexts run ADMM with hysco_group_admm");
        std::vector<hysco_ctx> R{ctx};
        void* const bi[1] = {d_b_inout};
        return ctx->cfg.dtype == HYSCO_F64 ? admm_slab_run<double>(R, ctx->comm, o, bi, reports)
                                           : admm_slab_run<float>(R, ctx->comm, o, bi, reports);
    }
    return ctx->cfg.dtype == HYSCO_F64 ? admm_run<double>(ctx, d_b_inout, o, reports)
                                       : admm_run<float>(ctx, d_b_inout, o, reports);
}

hysco_status hysco_group_admm(hysco_ctx* ctxs, int32_t nranks, void* const* d_b_inout, const hysco_admm_opts* opts,
                              hysco_admm_report* reports) {
    NvtxRange nvtx_("hysco_group_admm");
    if (!ctxs || nranks < 1 || !d_b_inout) return HYSCO_ERR_ARG;
    LoopbackComm* lb = dynamic_cast<LoopbackComm*>(ctxs[0]->comm);
    if (!lb || (int)lb->members.size() != nranks) return set_err(ctxs[0], HYSCO_ERR_STATE, "not a loopback group");
    for (int r = 0; r < nranks; r++) {
        if (ctxs[r] != lb->members[r]) return set_err(ctxs[0], HYSCO_ERR_ARG, "contexts must be passed in rank order");
        if (ctxs[r]->poisoned) return HYSCO_ERR_CUDA;
        if (hysco_status s = need_images(ctxs[r])) return s;
        if (!d_b_inout[r]) return HYSCO_ERR_ARG;
    }
    hysco_admm_opts o;
    hysco_default_admm_opts(&o);
    if (opts) o = *opts;
    if (o.max_iter < 0 || o.inner < 1 || o.ls_max < 1 || !(o.tol >= 0) || !(o.mu > 1) || !(o.tau > 1))
        return set_err(ctxs[0], HYSCO_ERR_ARG, "bad hysco_admm_opts");
    std::vector<hysco_ctx> R(ctxs, ctxs + nranks);
    cudaSetDevice(ctxs[0]->cfg.device);
    return ctxs[0]->cfg.dtype == HYSCO_F64 ? admm_slab_run<double>(R, lb, o, d_b_inout, reports)
                                           : admm_slab_run<float>(R, lb, o, d_b_inout, reports);
}

void hysco_default_lsq_opts(hysco_lsq_opts* o) {
    if (!o) return;
    o->lambda = 0.05;
    o->max_iter = 200;
    o->rtol = 0.0;
}

hysco_status hysco_push_forward(hysco_ctx ctx, const void* d_b, const void* d_T, void* d_Iplus, void* d_Iminus) {
    NvtxRange nvtx_("hysco_push_forward");
    CHECK_CTX();
    // column-local: on a slab context it runs on the rank's planes, no exchange
    if (!d_b || !d_T || !d_Iplus || !d_Iminus || !aligned16(d_b) || !aligned16(d_T) || !aligned16(d_Iplus) ||
        !aligned16(d_Iminus))
        return set_err(ctx, HYSCO_ERR_ARG, "pointers must be non-NULL and 16-byte aligned");
    return ctx->cfg.dtype == HYSCO_F64 ? push_forward_run<double>(ctx, d_b, d_T, d_Iplus, d_Iminus)
                                       : push_forward_run<float>(ctx, d_b, d_T, d_Iplus, d_Iminus);
}

hysco_status hysco_lsq_correct(hysco_ctx ctx, const void* d_b, const hysco_lsq_opts* opts, void* d_T_out,
                               hysco_lsq_report* reports) {
    NvtxRange nvtx_("hysco_lsq_correct");
    CHECK_CTX();
    // column-local: on a slab context it runs on the rank's planes, no exchange
    if (hysco_status s = need_images(ctx)) return s;
    if (!d_b || !d_T_out || !aligned16(d_b) || !aligned16(d_T_out))
        return set_err(ctx, HYSCO_ERR_ARG, "pointers must be non-NULL and 16-byte aligned");
    hysco_lsq_opts o;
    hysco_default_lsq_opts(&o);
    if (opts) o = *opts;
    if (!(o.lambda >= 0) || o.max_iter < 0 || !(o.rtol >= 0))
        return set_err(ctx, HYSCO_ERR_ARG, "bad hysco_lsq_opts");
    return ctx->cfg.dtype == HYSCO_F64 ? lsq_run<double>(ctx, d_b, o, d_T_out, reports)
                                       : lsq_run<float>(ctx, d_b, o, d_T_out, reports);
}

hysco_status hysco_fieldmap_cells(hysco_ctx ctx, const void* d_b, void* d_out) {
    return hysco_fieldmap_cells_units(ctx, d_b, d_out, HYSCO_FIELDMAP_MM);
}

hysco_status hysco_fieldmap_cells_units(hysco_ctx ctx, const void* d_b, void* d_out, int32_t units) {
    CHECK_CTX();
    if (units != HYSCO_FIELDMAP_MM && units != HYSCO_FIELDMAP_VOXEL)
        return set_err(ctx, HYSCO_ERR_ARG, "units must be HYSCO_FIELDMAP_MM or HYSCO_FIELDMAP_VOXEL");
    const double scale = units == HYSCO_FIELDMAP_VOXEL ? 1.0 / ctx->g.h3 : 1.0;
    // column-local: on a slab context it runs on the rank's planes, no exchange
    if (!d_b || !d_out || !aligned16(d_b) || !aligned16(d_out))
        return set_err(ctx, HYSCO_ERR_ARG, "pointers must be non-NULL and 16-byte aligned");
    const long long total = (long long)ctx->cfg.batch * ctx->g.Nc;
    const int grid = (int)std::min<long long>((total + 255) / 256, (long long)ctx->nsm * 8);
    if (ctx->cfg.dtype == HYSCO_F64)
        fieldmap_cells_kernel<double><<<grid, 256, 0, ctx->stream>>>(ctx->g, ctx->ctl, (const double*)d_b,
                                                                    (double*)d_out, total, scale);
    else
        fieldmap_cells_kernel<float><<<grid, 256, 0, ctx->stream>>>(ctx->g, ctx->ctl, (const float*)d_b,
                                                                   (float*)d_out, total, (float)scale);
    CK(cudaGetLastError());
    return HYSCO_OK;
}

hysco_status hysco_apply(hysco_ctx ctx, const void* d_b, void* d_Iplus_corr, void* d_Iminus_corr) {
    NvtxRange nvtx_("hysco_apply");
    CHECK_CTX();
    if (ctx->g.slab) return set_err(ctx, HYSCO_ERR_STATE, "slab contexts support solve / correct / correct_host");
    if (hysco_status s = need_images(ctx)) return s;
    if (!d_b || !aligned16(d_b) || (d_Iplus_corr && !aligned16(d_Iplus_corr)) ||
        (d_Iminus_corr && !aligned16(d_Iminus_corr)))
        return set_err(ctx, HYSCO_ERR_ARG, "pointers must be 16-byte aligned");
    if (ctx->cfg.dtype == HYSCO_F64) L<double>::apply(ctx, (const double*)d_b, (double*)d_Iplus_corr, (double*)d_Iminus_corr);
    else L<float>::apply(ctx, (const float*)d_b, (float*)d_Iplus_corr, (float*)d_Iminus_corr);
    CK(cudaGetLastError());
    return HYSCO_OK;
}

static hysco_status solve_common(hysco_ctx ctx, int kind, const hysco_ot_opts* ot, const hysco_solve_opts* so,
                                 void* b_io, void* b_out, void* Tp, void* Tm, hysco_report* reports) {
    hysco_solve_opts o;
    hysco_default_solve_opts(&o);
    if (so) o = *so;
    hysco_ot_opts t;
    hysco_default_ot_opts(&t);
    if (ot) t = *ot;
    if (hysco_status s = check_opts(ctx, o, t)) return s;
    GraphKey key;
    memset(&key, 0, sizeof key);
    key.kind = kind;
    key.sp = to_params(o, t);
    key.blur = t.blur ? 1 : 0;
    key.ptr[0] = ctx->Ip;
    key.ptr[1] = ctx->Im;
    key.ptr[2] = b_io;
    key.ptr[3] = b_out;
    key.ptr[4] = Tp;
    key.ptr[5] = Tm;
    hysco_status s;
    if (ctx->g.slab) {
        if (!dynamic_cast<NcclComm*>(ctx->comm))
            return set_err(ctx, HYSCO_ERR_STATE, "loopback slab contexts are driven with hysco_group_*");
        std::vector<hysco_ctx> R{ctx};
        void* const bi[1] = {b_io};
        void* const bo[1] = {b_out};
        void* const tp[1] = {Tp};
        void* const tm[1] = {Tm};
        s = ctx->cfg.dtype == HYSCO_F64 ? run_slab_path<double>(R, ctx->comm, kind, key.sp, key.blur, bi, bo, tp, tm)
                                        : run_slab_path<float>(R, ctx->comm, kind, key.sp, key.blur, bi, bo, tp, tm);
    } else {
        s = ctx->cfg.dtype == HYSCO_F64 ? run_path<double>(ctx, key, b_io, b_out, Tp, Tm)
                                        : run_path<float>(ctx, key, b_io, b_out, Tp, Tm);
    }
    if (s != HYSCO_OK) return s;
    if (ctx->defer_st) return HYSCO_OK;   // reports after the caller's synchronisation
    bool inf = false;
    fill_reports(ctx, reports, &inf);
    // a pair-by-pair batch solve shares the Hessian scratch between pairs:
    // only the last pair's parts survive, so hessvec needs a new objective_grad
    ctx->state_valid = !inf && !ctx->last_per_pair;
    return inf ? HYSCO_INFEASIBLE : HYSCO_OK;
}

hysco_status hysco_solve(hysco_ctx ctx, void* d_b_inout, const hysco_solve_opts* opts, hysco_report* reports) {
    NvtxRange nvtx_("hysco_solve");
    CHECK_CTX();
    if (hysco_status s = need_images(ctx)) return s;
    if (!d_b_inout || !aligned16(d_b_inout)) return set_err(ctx, HYSCO_ERR_ARG, "d_b_inout must be 16-byte aligned");
    return solve_common(ctx, 1, nullptr, opts, d_b_inout, nullptr, nullptr, nullptr, reports);
}

hysco_status hysco_correct(hysco_ctx ctx, const hysco_ot_opts* ot, const hysco_solve_opts* so, void* d_b_out,
                           void* d_Iplus_corr, void* d_Iminus_corr, hysco_report* reports) {
    NvtxRange nvtx_("hysco_correct");
    CHECK_CTX();
    if (hysco_status s = need_images(ctx)) return s;
    for (void* p : {d_b_out, d_Iplus_corr, d_Iminus_corr})
        if (p && !aligned16(p)) return set_err(ctx, HYSCO_ERR_ARG, "output pointers must be 16-byte aligned");
    return solve_common(ctx, 2, ot, so, nullptr, d_b_out, d_Iplus_corr, d_Iminus_corr, reports);
}

hysco_status hysco_correct_host(hysco_ctx ctx, const void* h_Iplus, const void* h_Iminus, const hysco_ot_opts* ot,
                                const hysco_solve_opts* so, void* h_b_out, void* h_Iplus_corr, void* h_Iminus_corr,
                                hysco_report* reports) {
    NvtxRange nvtx_("hysco_correct_host");
    CHECK_CTX();
    if (!h_Iplus || !h_Iminus) return set_err(ctx, HYSCO_ERR_ARG, "host images must be non-NULL");
    const size_t nc = (size_t)ctx->cfg.batch * ctx->g.Nc * ctx->esz;
    const size_t nn = (size_t)ctx->cfg.batch * ctx->g.Nn * ctx->esz;
    CK(cudaMemcpyAsync(ctx->own_Ip, h_Iplus, nc, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->own_Im, h_Iminus, nc, cudaMemcpyHostToDevice, ctx->stream));
    if (hysco_status s = hysco_bind_images(ctx, ctx->own_Ip, ctx->own_Im)) return s;
    hysco_status s = solve_common(ctx, 2, ot, so, nullptr, nullptr, h_Iplus_corr ? ctx->own_Tp : nullptr,
                                  h_Iminus_corr ? ctx->own_Tm : nullptr, reports);
    if (s < 0) return s;
    if (h_b_out) CK(copy_nodes(ctx, h_b_out, ctx->buf[B_B], false, cudaMemcpyDeviceToHost));
    (void)nn;
    if (h_Iplus_corr) CK(cudaMemcpyAsync(h_Iplus_corr, ctx->own_Tp, nc, cudaMemcpyDeviceToHost, ctx->stream));
    if (h_Iminus_corr) CK(cudaMemcpyAsync(h_Iminus_corr, ctx->own_Tm, nc, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return s;
}

static hysco_status stream_setup(hysco_ctx ctx) {
    if (ctx->stream_ready) return HYSCO_OK;
    const size_t nc = (size_t)ctx->cfg.batch * ctx->g.Nc * ctx->esz;
    const size_t nn = (size_t)ctx->cfg.batch * ctx->g.Nn * ctx->esz;
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; k++) {
        CK(cudaMalloc(&ctx->st_in[k][0], nc));
        CK(cudaMalloc(&ctx->st_in[k][1], nc));
        CK(cudaMalloc(&ctx->st_out[k][0], nn));
        CK(cudaMalloc(&ctx->st_out[k][1], nc));
        CK(cudaMalloc(&ctx->st_out[k][2], nc));
        for (cudaEvent_t* e : {&ctx->ev_h2d[k], &ctx->ev_in_free[k], &ctx->ev_out[k], &ctx->ev_out_free[k]}) {
            CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            CK(cudaEventRecord(*e, ctx->copy_stream));   // slots start free
        }
    }
    ctx->stream_ready = true;
    return HYSCO_OK;
}

hysco_status hysco_correct_host_stream(hysco_ctx ctx, int32_t n_items, const void* const* h_Iplus,
                                       const void* const* h_Iminus, const hysco_ot_opts* ot,
                                       const hysco_solve_opts* so, void* const* h_b_out,
                                       void* const* h_Iplus_corr, void* const* h_Iminus_corr,
                                       hysco_report* reports) {
    NvtxRange nvtx_("hysco_correct_host_stream");
    CHECK_CTX();
    if (ctx->g.slab) return set_err(ctx, HYSCO_ERR_STATE, "slab contexts support solve / correct / correct_host");
    if (n_items < 0 || (n_items > 0 && (!h_Iplus || !h_Iminus)))
        return set_err(ctx, HYSCO_ERR_ARG, "host image arrays must be non-NULL");
    for (int k = 0; k < n_items; k++)
        if (!h_Iplus[k] || !h_Iminus[k]) return set_err(ctx, HYSCO_ERR_ARG, "host images must be non-NULL");
    if (hysco_status s0 = stream_setup(ctx)) return s0;
    const size_t nc = (size_t)ctx->cfg.batch * ctx->g.Nc * ctx->esz;
    const size_t nn = (size_t)ctx->cfg.batch * ctx->g.Nn * ctx->esz;
    auto out_ptr = [](void* const* a, int k) { return a ? a[k] : nullptr; };
    cudaStream_t cs = ctx->copy_stream, ks = ctx->stream;
    auto h2d = [&](int k) -> cudaError_t {       // item k -> input slot k % 2 (copy stream)
        const int sl = k & 1;
        cudaError_t e = cudaStreamWaitEvent(cs, ctx->ev_in_free[sl], 0);
        if (!e) e = cudaMemcpyAsync(ctx->st_in[sl][0], h_Iplus[k], nc, cudaMemcpyHostToDevice, cs);
        if (!e) e = cudaMemcpyAsync(ctx->st_in[sl][1], h_Iminus[k], nc, cudaMemcpyHostToDevice, cs);
        if (!e) e = cudaEventRecord(ctx->ev_h2d[sl], cs);
        return e;
    };
    const int B = ctx->cfg.batch;
    if ((long long)n_items * B > ctx->h_items_cap) {   // per-item readback slots (pinned, kept)
        if (ctx->h_items) cudaFreeHost(ctx->h_items);
        if (ctx->h_items_l) cudaFreeHost(ctx->h_items_l);
        ctx->h_items = nullptr;
        ctx->h_items_l = nullptr;
        ctx->h_items_cap = 0;
        const long long cap = std::max<long long>((long long)n_items * B, 8LL * B);
        if (ctx->d_items) cudaFree(ctx->d_items);
        if (ctx->d_items_l) cudaFree(ctx->d_items_l);
        ctx->d_items = nullptr;
        ctx->d_items_l = nullptr;
        CK(cudaMallocHost((void**)&ctx->h_items, sizeof(PairState) * cap));
        CK(cudaMallocHost((void**)&ctx->h_items_l, sizeof(unsigned long long) * cap));
        CK(cudaMalloc((void**)&ctx->d_items, sizeof(PairState) * cap));
        CK(cudaMalloc((void**)&ctx->d_items_l, sizeof(unsigned long long) * cap));
        ctx->h_items_cap = cap;
    }
    CK(cudaMemsetAsync(ctx->launches, 0, sizeof(unsigned long long), ctx->stream));   // item 0's count
    if (n_items > 0) CK(h2d(0));
    hysco_status first_err = HYSCO_OK;
    std::vector<char> ran(n_items, 0);
    struct DeferOff {   // the readback redirection ends with this call, however it returns
        hysco_ctx c;
        ~DeferOff() {
            c->defer_st = nullptr;
            c->defer_launch = nullptr;
        }
    } defer_off{ctx};
    // Item k runs on staging slot sl = k % 2: its images are read in place from
    // the input slot and its results written in place to the output slot (the
    // two slots' pointer sets are the context's two cached graphs), so no
    // device-to-device staging copies sit on the compute stream.
    for (int k = 0; k < n_items; k++) {
        const int sl = k & 1;
        if (k + 1 < n_items) CK(h2d(k + 1));     // next pair streams in during this correction
        CK(cudaStreamWaitEvent(ks, ctx->ev_h2d[sl], 0));
        CK(cudaStreamWaitEvent(ks, ctx->ev_out_free[sl], 0));   // item k - 2's results are out
        if (hysco_status s0 = hysco_bind_images(ctx, ctx->st_in[sl][0], ctx->st_in[sl][1])) return s0;
        void *hb = out_ptr(h_b_out, k), *hp = out_ptr(h_Iplus_corr, k), *hm = out_ptr(h_Iminus_corr, k);
        ctx->defer_st = ctx->d_items + (size_t)k * B;
        ctx->defer_launch = ctx->d_items_l + k;
        hysco_status s = solve_common(ctx, 2, ot, so, nullptr, hb ? ctx->st_out[sl][0] : nullptr,
                                      hp ? ctx->st_out[sl][1] : nullptr, hm ? ctx->st_out[sl][2] : nullptr, nullptr);
        CK(cudaEventRecord(ctx->ev_in_free[sl], ks));
        if (s < 0) {
            if (first_err == HYSCO_OK) first_err = s;
            continue;
        }
        if (s != HYSCO_OK && first_err == HYSCO_OK) first_err = s;
        ran[k] = 1;
        // results out to the host (copy stream)
        CK(cudaEventRecord(ctx->ev_out[sl], ks));
        CK(cudaStreamWaitEvent(cs, ctx->ev_out[sl], 0));
        if (hb) CK(cudaMemcpyAsync(hb, ctx->st_out[sl][0], nn, cudaMemcpyDeviceToHost, cs));
        if (hp) CK(cudaMemcpyAsync(hp, ctx->st_out[sl][1], nc, cudaMemcpyDeviceToHost, cs));
        if (hm) CK(cudaMemcpyAsync(hm, ctx->st_out[sl][2], nc, cudaMemcpyDeviceToHost, cs));
        CK(cudaEventRecord(ctx->ev_out_free[sl], cs));
    }
    if (n_items > 0) {
        CK(cudaMemcpyAsync(ctx->h_items, ctx->d_items, sizeof(PairState) * (size_t)n_items * B,
                           cudaMemcpyDeviceToHost, ks));
        CK(cudaMemcpyAsync(ctx->h_items_l, ctx->d_items_l, sizeof(unsigned long long) * n_items,
                           cudaMemcpyDeviceToHost, ks));
    }
    CK(cudaStreamSynchronize(cs));
    CK(cudaStreamSynchronize(ks));
    // reports and the state mirror from the per-item readbacks (in item order)
    ctx->state_valid = false;
    for (int k = 0; k < n_items; k++) {
        if (!ran[k]) continue;
        memcpy(ctx->h_st, ctx->h_items + (size_t)k * B, sizeof(PairState) * B);
        ctx->last_launches = (long long)ctx->h_items_l[k];
        bool inf = false;
        fill_reports(ctx, reports ? reports + (size_t)k * B : nullptr, &inf);
        if (inf && first_err == HYSCO_OK) first_err = HYSCO_INFEASIBLE;
        ctx->state_valid = k == n_items - 1 && !inf && !ctx->last_per_pair;   // as after hysco_correct
    }
    return first_err;
}

int64_t hysco_last_launch_count(hysco_ctx ctx) { return ctx ? ctx->last_launches : -1; }

int32_t hysco_pcg_path(hysco_ctx ctx, int32_t* tile_out) {
    if (!ctx) return -1;
    if (tile_out) {
        const bool t = ctx->resident && ctx->res_tiled;
        tile_out[0] = t ? ctx->res_tile.TI : 0;
        tile_out[1] = t ? ctx->res_tile.TJ : 0;
        tile_out[2] = t ? ctx->res_tile.TH : 0;
        tile_out[3] = t ? ctx->res_tile.TW : 0;
    }
    if (ctx->resident) return ctx->res_tiled ? 2 : 1;
    return ctx->l2pcg ? 3 : 0;
}

static_assert(sizeof(hysco_iter_record) == sizeof(HistRec), "hysco_iter_record mirrors HistRec");

hysco_status hysco_history(hysco_ctx ctx, int32_t pair, hysco_iter_record* out, int32_t max_records,
                           int32_t* n_records) {
    CHECK_CTX();
    if (pair < 0 || pair >= ctx->cfg.batch || !out || max_records < 0 || !n_records)
        return set_err(ctx, HYSCO_ERR_ARG, "hysco_history: bad pair / buffer");
    const PairState& s = ctx->h_st[pair];   // mirror of the last solve's final state
    int n = s.stop_reason == STOP_INFEASIBLE && s.f_evals <= 1 ? 1 : s.gn_k + 1;
    n = std::min(std::min(n, HIST_MAX), (int)max_records);
    *n_records = n;
    if (n == 0) return HYSCO_OK;
    CK(cudaMemcpyAsync(out, ctx->hist + (size_t)pair * HIST_MAX, sizeof(HistRec) * n, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return HYSCO_OK;
}

hysco_status hysco_nccl_unique_id(unsigned char id_out[128]) {
    if (!id_out) return HYSCO_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return HYSCO_ERR_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    memcpy(id_out, &id, 128);
    return HYSCO_OK;
}

hysco_status hysco_create_slab(const hysco_config* cfg, int32_t rank, int32_t nranks, int64_t n1_global, int64_t i0,
                               const unsigned char* nccl_id, void* cuda_stream, hysco_ctx* out) {
    if (!cfg || !out || (nranks > 1 && !nccl_id)) return HYSCO_ERR_ARG;
    SlabSpec sl{rank, nranks, n1_global, i0};
    hysco_status st = create_impl(cfg, &sl, cuda_stream, out);
    if (st != HYSCO_OK) return st;
    hysco_ctx ctx = *out;
    NcclComm* nc = new NcclComm();
    nc->rank = rank;
    nc->n = nranks;
    ctx->comm = nc;
    if (nranks > 1) {
        ncclUniqueId id;
        memcpy(&id, nccl_id, 128);
        if (ncclCommInitRank(&nc->comm, nranks, id, rank) != ncclSuccess) {
            ctx->err = "ncclCommInitRank failed";
            hysco_destroy(ctx);
            *out = nullptr;
            return HYSCO_ERR_NCCL;
        }
    }
    return HYSCO_OK;
}

hysco_status hysco_create_loopback(const hysco_config* cfg, int32_t nranks, void* cuda_stream, hysco_ctx* out) {
    if (!cfg || !out || nranks < 1 || nranks > cfg->n1) return HYSCO_ERR_ARG;
    LoopbackComm* lb = new LoopbackComm();
    cudaStream_t stream = (cudaStream_t)cuda_stream;
    bool own = false;
    if (!stream) {
        if (cudaSetDevice(cfg->device) != cudaSuccess || cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete lb;
            cudaGetLastError();
            return HYSCO_ERR_CUDA;
        }
        own = true;
    }
    for (int r = 0; r < nranks; r++) {
        const int64_t i0 = cfg->n1 * r / nranks, i1 = cfg->n1 * (r + 1) / nranks;
        hysco_config c = *cfg;
        c.n1 = i1 - i0;
        SlabSpec sl{r, nranks, cfg->n1, i0};
        hysco_status st = create_impl(&c, &sl, stream, &out[r]);
        if (st != HYSCO_OK) {
            if (r == 0) {
                delete lb;                       // no member holds it yet
            } else {
                for (int q = 0; q < r; q++) hysco_destroy(out[q]);   // the last one frees lb
            }
            return st;
        }
        out[r]->comm = lb;
        lb->members.push_back(out[r]);
        lb->refs++;
    }
    lb->stream = stream;                   // destroyed with the last member (~LoopbackComm)
    lb->own_stream = own;
    std::vector<double*> ptrs;
    for (auto* m : lb->members) ptrs.push_back(m->red);
    if (cudaMalloc(&lb->d_ptrs, sizeof(double*) * nranks) != cudaSuccess ||
        cudaMemcpy(lb->d_ptrs, ptrs.data(), sizeof(double*) * nranks, cudaMemcpyHostToDevice) != cudaSuccess) {
        for (int q = 0; q < nranks; q++) hysco_destroy(out[q]);
        return HYSCO_ERR_NOMEM;
    }
    return HYSCO_OK;
}

static hysco_status group_common(hysco_ctx* ctxs, int32_t n, int kind, const hysco_ot_opts* ot,
                                 const hysco_solve_opts* so, void* const* b_io, void* const* b_out,
                                 void* const* Tp, void* const* Tm, hysco_report* reports) {
    if (!ctxs || n < 1) return HYSCO_ERR_ARG;
    LoopbackComm* lb = dynamic_cast<LoopbackComm*>(ctxs[0]->comm);
    if (!lb || (int)lb->members.size() != n) return set_err(ctxs[0], HYSCO_ERR_STATE, "not a loopback group");
    for (int r = 0; r < n; r++) {
        hysco_ctx ctx = ctxs[r];
        if (ctx != lb->members[r]) return set_err(ctxs[0], HYSCO_ERR_ARG, "contexts must be passed in rank order");
        if (ctx->poisoned) return HYSCO_ERR_CUDA;
        if (hysco_status s = need_images(ctx)) return s;
    }
    hysco_solve_opts o;
    hysco_default_solve_opts(&o);
    if (so) o = *so;
    hysco_ot_opts t;
    hysco_default_ot_opts(&t);
    if (ot) t = *ot;
    if (hysco_status s = check_opts(ctxs[0], o, t)) return s;
    std::vector<hysco_ctx> R(ctxs, ctxs + n);
    cudaSetDevice(ctxs[0]->cfg.device);
    const SolveParams sp = to_params(o, t);
    hysco_status s = ctxs[0]->cfg.dtype == HYSCO_F64
                         ? run_slab_path<double>(R, lb, kind, sp, t.blur ? 1 : 0, b_io, b_out, Tp, Tm)
                         : run_slab_path<float>(R, lb, kind, sp, t.blur ? 1 : 0, b_io, b_out, Tp, Tm);
    if (s != HYSCO_OK) return s;
    bool inf = false;
    fill_reports(ctxs[0], reports, &inf);
    return inf ? HYSCO_INFEASIBLE : HYSCO_OK;
}

hysco_status hysco_group_correct(hysco_ctx* ctxs, int32_t nranks, const hysco_ot_opts* ot, const hysco_solve_opts* so,
                                 void* const* d_b_out, void* const* d_Iplus_corr, void* const* d_Iminus_corr,
                                 hysco_report* reports) {
    NvtxRange nvtx_("hysco_group_correct");
    return group_common(ctxs, nranks, 2, ot, so, nullptr, d_b_out, d_Iplus_corr, d_Iminus_corr, reports);
}

hysco_status hysco_group_solve(hysco_ctx* ctxs, int32_t nranks, void* const* d_b_inout, const hysco_solve_opts* so,
                               hysco_report* reports) {
    NvtxRange nvtx_("hysco_group_solve");
    if (!d_b_inout) return HYSCO_ERR_ARG;
    return group_common(ctxs, nranks, 1, nullptr, so, d_b_inout, nullptr, nullptr, nullptr, reports);
}

}  // extern "C"

template <typename T>
static hysco_status profile_typed(hysco_ctx ctx, int reps, int flush_l2, double* avg_ms) {
    // force the PCG kernels active (they early-exit on finished pairs)
    CK(cudaMemcpyAsync(ctx->h_st, ctx->st, sizeof(PairState) * ctx->cfg.batch, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int p = 0; p < ctx->cfg.batch; p++) {
        ctx->h_st[p].pcg_active = 1;
        ctx->h_st[p].gn_active = 1;     // resident PCG / trial_init run only for iterating pairs
        ctx->h_st[p].alpha_c = 0.0;     // x, r unchanged by update
        ctx->h_st[p].beta_c = 0.0;
        ctx->h_st[p].rz = 1.0;
        ctx->h_st[p].rr0 = 1.0;
    }
    SolveParams sp{};
    sp.max_pcg = 1 << 30;
    sp.fixed = 1;
    const size_t flush_bytes = (size_t)256 << 20;
    if (flush_l2 && !ctx->flush) CK(cudaMalloc(&ctx->flush, flush_bytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    dim3 gr(ctx->gx_nodes, ctx->cfg.batch);
    for (int k = 0; k < HYSCO_NPROF; k++) {
        double acc = 0;
        for (int r = 0; r < reps; r++) {
            CK(cudaMemcpyAsync(ctx->st, ctx->h_st, sizeof(PairState) * ctx->cfg.batch, cudaMemcpyHostToDevice,
                               ctx->stream));
            if (flush_l2) CK(cudaMemsetAsync(ctx->flush, r & 0xff, flush_bytes, ctx->stream));
            CK(cudaEventRecord(e0, ctx->stream));
            switch (k) {
                case HYSCO_PROF_MATVEC:
                    NCH_SWITCH(ctx->nch, matvec_kernel<T, NCH, true><<<dim3(ctx->gx_mv, ctx->cfg.batch), 256, 0,
                                                                       ctx->stream>>>(
                                             ctx->g, ctx->ctl, L<T>::b(ctx, B_DT), L<T>::b(ctx, B_ET),
                                             L<T>::b(ctx, B_P), L<T>::b(ctx, B_HP)));
                    break;
                case HYSCO_PROF_UPDATE:
                    NCH_SWITCH(ctx->nch, pcg_update_kernel<T, NCH><<<gr, 256, 0, ctx->stream>>>(
                                             ctx->g, ctx->ctl, sp, L<T>::b(ctx, B_DT), L<T>::b(ctx, B_P),
                                             L<T>::b(ctx, B_HP), L<T>::b(ctx, B_X), L<T>::b(ctx, B_R)));
                    break;
                case HYSCO_PROF_DIR:
                    NCH_SWITCH(ctx->nch, pcg_dir_kernel<T, NCH><<<gr, 256, 0, ctx->stream>>>(
                                             ctx->g, ctx->ctl, L<T>::b(ctx, B_DT), L<T>::b(ctx, B_R),
                                             L<T>::b(ctx, B_P)));
                    break;
                case HYSCO_PROF_RESIDENT: {
                    if (!ctx->resident) break;
                    SolveParams rp = sp;
                    rp.max_pcg = 10;          // one GN step's PCG solve
                    for (int p = 0; p < ctx->cfg.batch; p++)   // trial b to scratch: B_B stays
                        launch_resident(ctx, rp, p, reinterpret_cast<float*>(L<T>::b(ctx, B_TMP)),
                                        reinterpret_cast<float*>(L<T>::b(ctx, B_HP)));
                    break;
                }
                case HYSCO_PROF_RES_SYNC: {
                    if (!ctx->resident) break;
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(ctx->res_grid, 1, 1);
                    cfg.blockDim = dim3(RES_THREADS, 1, 1);
                    cfg.dynamicSmemBytes = ctx->res_smem;   // same occupancy as the real kernel
                    cfg.stream = ctx->stream;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeCooperative;
                    at[0].val.cooperative = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = 1;
                    if (ctx->res_tiled) {
                        RES_K_SWITCH(ctx->res_k, CK(cudaLaunchKernelEx(&cfg, pcg_sync_floor_kernel<RK, true>, ctx->g,
                                                                       10, ctx->res_part, ctx->res_flags,
                                                                       ctx->res_tile)));
                    } else {
                        RES_K_SWITCH(ctx->res_k, CK(cudaLaunchKernelEx(&cfg, pcg_sync_floor_kernel<RK>, ctx->g, 10,
                                                                       ctx->res_part, ctx->res_flags,
                                                                       ResTile{0, 0, 0, 0})));
                    }
                    break;
                }
                case HYSCO_PROF_L2PCG: {
                    if (!ctx->l2pcg) break;
                    SolveParams rp = sp;
                    rp.max_pcg = 10;          // one GN step's PCG solve
                    // the Armijo start writes b_old / b: point them at scratch for the profile
                    void* sb = ctx->buf[B_B];
                    void* so = ctx->buf[B_BOLD];
                    ctx->buf[B_B] = ctx->buf[B_TMP];
                    ctx->buf[B_BOLD] = ctx->buf[B_W];
                    for (int p = 0; p < ctx->cfg.batch; p++) launch_l2pcg<T>(ctx, rp, p);
                    ctx->buf[B_B] = sb;
                    ctx->buf[B_BOLD] = so;
                    break;
                }
                case HYSCO_PROF_TRIAL:
                    if (ctx->flat) {
                        L<T>::trial_flat(ctx, L<T>::b(ctx, B_TMP), L<T>::b(ctx, B_BOLD));
                        break;
                    }
                    NCH_SWITCH(ctx->nch, trial_init_kernel<T, NCH><<<gr, 256, 0, ctx->stream>>>(
                                             ctx->g, ctx->ctl, L<T>::b(ctx, B_GRAD), L<T>::b(ctx, B_X),
                                             L<T>::b(ctx, B_TMP), L<T>::b(ctx, B_BOLD)));
                    break;
                case HYSCO_PROF_DIRMV:
                    if (ctx->flat) L<T>::pcg_dirmv(ctx, false);
                    break;
                case HYSCO_PROF_UPD:
                    if (ctx->flat) L<T>::pcg_upd(ctx, sp);
                    break;
                default:
                    L<T>::eval(ctx, sp, EVAL_PLAIN, L<T>::b(ctx, B_B));
            }
            CK(cudaGetLastError());
            CK(cudaEventRecord(e1, ctx->stream));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            acc += ms;
        }
        avg_ms[k] = ((k == HYSCO_PROF_RESIDENT || k == HYSCO_PROF_RES_SYNC) && !ctx->resident) ||
                            (k == HYSCO_PROF_L2PCG && !ctx->l2pcg) ||
                            ((k == HYSCO_PROF_DIRMV || k == HYSCO_PROF_UPD) && !ctx->flat)
                        ? -1.0
                        : acc / reps;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // restore a consistent Hessian state at the current b
    L<T>::eval(ctx, sp, EVAL_PLAIN, L<T>::b(ctx, B_B));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    return HYSCO_OK;
}

extern "C" {

hysco_status hysco_profile_kernels(hysco_ctx ctx, int32_t reps, int32_t flush_l2, double* avg_ms) {
    NvtxRange nvtx_("hysco_profile_kernels");
    CHECK_CTX();
    if (hysco_status s = need_images(ctx)) return s;
    if (reps < 1 || !avg_ms) return set_err(ctx, HYSCO_ERR_ARG, "reps >= 1 and avg_ms[HYSCO_NPROF] required");
    return ctx->cfg.dtype == HYSCO_F64 ? profile_typed<double>(ctx, reps, flush_l2, avg_ms)
                                       : profile_typed<float>(ctx, reps, flush_l2, avg_ms);
}

const char* hysco_last_error(hysco_ctx ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

hysco_status hysco_destroy(hysco_ctx ctx) {
    if (!ctx) return HYSCO_ERR_ARG;
    cudaSetDevice(ctx->cfg.device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->exec) cudaGraphExecDestroy(ctx->exec);
    if (ctx->graph) cudaGraphDestroy(ctx->graph);
    if (ctx->exec2) cudaGraphExecDestroy(ctx->exec2);
    if (ctx->graph2) cudaGraphDestroy(ctx->graph2);
    for (cudaGraphExec_t e : ctx->seg_exec) cudaGraphExecDestroy(e);
    for (int k = 0; k < NBUF; k++)
        if (ctx->raw[k]) cudaFree(ctx->raw[k]);
    for (void* p : {ctx->own_Ip, ctx->own_Im, ctx->own_Tp, ctx->own_Tm, (void*)ctx->st, (void*)ctx->part,
                    (void*)ctx->ctr, (void*)ctx->gctr, (void*)ctx->launches, (void*)ctx->dcond})
        if (p) cudaFree(p);
    if (ctx->flush) cudaFree(ctx->flush);
    if (ctx->res_part) cudaFree(ctx->res_part);
    admm_slab_free(ctx);
    if (ctx->res_flags) cudaFree(ctx->res_flags);
    if (ctx->admm_ready) {
        cufftDestroy(ctx->fft_fwd);
        cufftDestroy(ctx->fft_inv);
    }
    for (int k = 0; k < 2; k++)
        if (ctx->admm_ev[k]) cudaEventDestroy(ctx->admm_ev[k]);
    if (ctx->h_admm_done) cudaFreeHost(ctx->h_admm_done);
    for (void* q : {ctx->admm_spec, (void*)ctx->admm_rho, (void*)ctx->admm_fac, (void*)ctx->admm_lam,
                    (void*)ctx->admm_stat, (void*)ctx->admm_done})
        if (q) cudaFree(q);
    if (ctx->stream_ready) {
        for (int k = 0; k < 2; k++) {
            for (void* q : {ctx->st_in[k][0], ctx->st_in[k][1], ctx->st_out[k][0], ctx->st_out[k][1], ctx->st_out[k][2]})
                if (q) cudaFree(q);
            for (cudaEvent_t e : {ctx->ev_h2d[k], ctx->ev_in_free[k], ctx->ev_out[k], ctx->ev_out_free[k]})
                if (e) cudaEventDestroy(e);
        }
        cudaStreamDestroy(ctx->copy_stream);
    }
    if (ctx->res_pg) cudaFree(ctx->res_pg);
    if (ctx->res_x) cudaFree(ctx->res_x);
    if (ctx->red) cudaFree(ctx->red);
    if (ctx->hist) cudaFree(ctx->hist);
    if (ctx->comm) {
        if (LoopbackComm* lb = dynamic_cast<LoopbackComm*>(ctx->comm)) {
            for (auto& m : lb->members)
                if (m == ctx) m = nullptr;
            if (--lb->refs == 0) delete lb;
        } else {
            delete ctx->comm;
        }
    }
    if (ctx->h_st) cudaFreeHost(ctx->h_st);
    if (ctx->h_launches) cudaFreeHost(ctx->h_launches);
    if (ctx->h_items) cudaFreeHost(ctx->h_items);
    if (ctx->h_items_l) cudaFreeHost(ctx->h_items_l);
    if (ctx->d_items) cudaFree(ctx->d_items);
    if (ctx->d_items_l) cudaFree(ctx->d_items_l);
    if (ctx->h_cond) cudaFreeHost(ctx->h_cond);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    cudaGetLastError();
    delete ctx;
    return HYSCO_OK;
}

}  // extern "C"
