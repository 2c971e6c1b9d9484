// res_trace.cu — phase timeline of the resident PCG kernel on a 3T-shaped
// problem (diagnostic; not part of the library).  Each CTA's thread 0 stamps
// %globaltimer at the phase boundaries of every iteration; we print, per
// phase, the mean over iterations of (last CTA end - first CTA start) and of
// the per-CTA durations, which separates compute from barrier skew.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2403_10706_b200/csrc -I include -o tools/res_trace tools/res_trace.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <string>
#include <cmath>
#include "hysco_kernels.cuh"

using namespace hysco;

int main(int argc, char** argv) {
    int n1 = 168, n2 = 111, n3 = 144;
    // usage: res_trace [tiled TI TJ TH TW] | [n1 n2 n3]
    ResTile tl{0, 0, 0, 0};
    const bool tiled = argc > 5 && std::string(argv[1]) == "tiled";
    if (tiled) tl = ResTile{atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atoi(argv[5])};
    else if (argc > 3) { n1 = atoi(argv[1]); n2 = atoi(argv[2]); n3 = atoi(argv[3]); }
    Geom g{};
    g.n1 = n1; g.n2 = n2; g.n3 = n3; g.P = n3 + 1; g.ncol = (long long)n1 * n2;
    g.Nc = g.ncol * n3; g.Nn = g.ncol * g.P; g.ps = g.Nn; g.i0 = 0; g.n1g = n1; g.slab = 0;
    g.h1 = g.h2 = g.h3 = 1.25; g.hd = 1.25 * 1.25 * 1.25; g.alpha = 300; g.beta = 1e-4;
    g.ahd = g.alpha * g.hd; g.bh2 = 0.5e-4 * g.hd;
    g.ih1sq = g.ih2sq = g.ih3sq = 1 / (1.25 * 1.25); g.ih3 = 1 / 1.25; geom_finish(g);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int G = nsm, NT = RES_THREADS, K = RES_KMAX;
    if (tiled && tl.TI * tl.TJ > G) { printf("too many tiles\n"); return 1; }
    const long long ncl = (g.ncol + G - 1) / G, knt = (long long)K * NT;
    if (ncl * (res_pad(g.P) / 2) > knt) { printf("does not fit K=RES_KMAX\n"); return 1; }
    size_t Nn = g.Nn;
    std::vector<float> hdt(Nn), het(Nn), hg(Nn);
    srand(1);
    for (size_t t = 0; t < Nn; t++) {
        hdt[t] = 1e5f + 1e4f * (rand() / (float)RAND_MAX);
        het[t] = ((t % g.P) == (size_t)n3) ? 0.f : -300.f - 4e4f * (rand() / (float)RAND_MAX);
        hg[t] = (rand() / (float)RAND_MAX) - 0.5f;
    }
    float *dt, *et, *grad, *x, *pgh, *xpad;
    cudaMalloc(&dt, Nn * 4); cudaMalloc(&et, Nn * 4); cudaMalloc(&grad, Nn * 4); cudaMalloc(&x, Nn * 4);
    cudaMalloc(&xpad, std::max((size_t)g.ncol * res_pad(g.P), res_tiled_ghost_floats(G, K)) * 4);
    float *bb, *bo; cudaMalloc(&bb, Nn * 4); cudaMalloc(&bo, Nn * 4); cudaMemset(bb, 0, Nn * 4);
    const float wi = (float)(g.ahd * g.ih1sq), wj = (float)(g.ahd * g.ih2sq);
    size_t ghost = std::max(res_ghost_pair_floats(g) + res_ghost_slack_floats(RES_KMAX), res_tiled_ghost_floats(G, K));
    cudaMalloc(&pgh, ghost * 4); cudaMemset(pgh, 0, ghost * 4);
    cudaMemcpy(dt, hdt.data(), Nn * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(et, het.data(), Nn * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(grad, hg.data(), Nn * 4, cudaMemcpyHostToDevice);
    PairState* st; cudaMalloc(&st, sizeof(PairState));
    PairState hs{}; hs.gn_active = 1; cudaMemcpy(st, &hs, sizeof hs, cudaMemcpyHostToDevice);
    unsigned long long* launches; cudaMalloc(&launches, 8);
    double* part; cudaMalloc(&part, sizeof(double) * (3 * RES_PART_DOUBLES + RES_LIMB_DOUBLES));
    unsigned* flags; cudaMalloc(&flags, 4 * res_flags_words(G)); cudaMemset(flags, 0, 4 * res_flags_words(G));
    cudaMemset(part, 0, sizeof(double) * (3 * RES_PART_DOUBLES + RES_LIMB_DOUBLES));
    { unsigned one = 1; cudaMemcpy(flags + (size_t)G * RES_FLAG_STRIDE, &one, 4, cudaMemcpyHostToDevice); }
    unsigned long long* trace; cudaMalloc(&trace, sizeof(unsigned long long) * G * 16 * 8);
    cudaMemset(trace, 0, sizeof(unsigned long long) * G * 16 * 8);
    unsigned* dcond; cudaMalloc(&dcond, 4 * NCOND);
    Ctl c{}; c.st = st; c.launches = launches; c.dcond = dcond; c.use_graph = 0;
    SolveParams sp{}; sp.max_pcg = 10; sp.fixed = 1;
    const size_t smem = res_smem_bytes(RES_KMAX);
    cudaFuncSetAttribute(pcg_resident_kernel<RES_KMAX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pcg_resident_kernel<RES_KMAX, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pcg_resident_kernel<RES_KMAX, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pcg_resident_kernel<RES_KMAX, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = tiled ? tl.TI * tl.TJ : G;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(NT); cfg.dynamicSmemBytes = smem; cfg.stream = 0;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms_notrace = 0, ms_trace = 0;
    for (int rep = 0; rep < 7; rep++) {
        cudaMemcpy(st, &hs, sizeof hs, cudaMemcpyHostToDevice);   // a fresh GN step (no search pending)
        cudaEventRecord(e0);
        if (tiled)
            cudaLaunchKernelEx(&cfg, pcg_resident_kernel<RES_KMAX, true, false, true>, g, c, sp, 0, (const float*)grad,
                               (const float*)dt, (const float*)et, x, xpad, pgh, part, flags, wi, wj, bb, bo, 1,
                               (unsigned long long*)nullptr, tl);
        else
            cudaLaunchKernelEx(&cfg, pcg_resident_kernel<RES_KMAX, true>, g, c, sp, 0, (const float*)grad, (const float*)dt,
                               (const float*)et, x, xpad, pgh, part, flags, wi, wj, bb, bo, 1, (unsigned long long*)nullptr, tl);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms_notrace, e0, e1);
    }
    cudaMemcpy(st, &hs, sizeof hs, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    if (tiled)
        cudaLaunchKernelEx(&cfg, pcg_resident_kernel<RES_KMAX, true, true, true>, g, c, sp, 0, (const float*)grad,
                           (const float*)dt, (const float*)et, x, xpad, pgh, part, flags, wi, wj, bb, bo, 1, trace, tl);
    else
        cudaLaunchKernelEx(&cfg, pcg_resident_kernel<RES_KMAX, true, true>, g, c, sp, 0, (const float*)grad, (const float*)dt,
                           (const float*)et, x, xpad, pgh, part, flags, wi, wj, bb, bo, 1, trace, tl);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms_trace, e0, e1);
    printf("err=%s  kernel %.1f us (untraced), %.1f us (traced), grid %d x %d, K %d\n",
           cudaGetErrorString(cudaGetLastError()), ms_notrace * 1e3, ms_trace * 1e3, G, NT, K);
    std::vector<unsigned long long> ht((size_t)G * 16 * 8);
    cudaMemcpy(ht.data(), trace, ht.size() * 8, cudaMemcpyDeviceToHost);
    // stamp slots in time order within an iteration; the last phase ends at the next iteration's slot 0
    const int order[8] = {0, 1, 2, 7, 3, 4, 5, 6};
    // phase k runs from stamp order[k] to stamp order[k + 1] (slot 0 = loop top,
    // 1 = after halo_acquire, 2 = after the remote loads, 7 = after publish #1,
    // 3 = after collect #1, 4 = after publish #2, 5 = after collect #2, 6 = after the p update)
    const char* names[8] = {"local Hp + halo acquire", "remote Hp + p.Hp", "publish #1 (p.Hp)", "collect #1",
                            "U-phase + publish #2", "x upd + collect #2", "p update (D-phase)",
                            "release + loop top"};
    // per phase: span = max_cta(end) - min_cta(start); per-CTA mean/max/min of (end - start)
    for (int k = 0; k < 8; k++) {
        double span = 0, mean_cta = 0, max_cta = 0, min_cta = 1e30;
        int nit = 0;
        for (int it = 1; it < 9; it++) {
            unsigned long long mn = ~0ull, mx = 0;
            double acc = 0, mxd = 0;
            for (int b = 0; b < G; b++) {
                unsigned long long a = ht[((size_t)b * 16 + it) * 8 + order[k]];
                unsigned long long z = k < 7 ? ht[((size_t)b * 16 + it) * 8 + order[k + 1]] : ht[((size_t)b * 16 + it + 1) * 8];
                mn = std::min(mn, a); mx = std::max(mx, z);
                double d = (double)(z - a); acc += d; mxd = std::max(mxd, d); min_cta = std::min(min_cta, d);
            }
            span += (double)(mx - mn); mean_cta += acc / G; max_cta += mxd; nit++;
        }
        printf("%-24s span %7.2f us | per-CTA mean %7.2f max %7.2f min %7.2f us\n", names[k],
               span / nit / 1e3, mean_cta / nit / 1e3, max_cta / nit / 1e3, min_cta / 1e3);
    }
    {   // launch-level stamps (slot 15): start, init loads done, init reduce done, loop done
        double a = 0, b2 = 0, c2 = 0, mx = 0;
        for (int b = 0; b < G; b++) {
            const unsigned long long* t = &ht[((size_t)b * 16 + 15) * 8];
            a += (double)(t[1] - t[0]); b2 += (double)(t[2] - t[1]); c2 += (double)(t[3] - t[2]);
            mx = std::max(mx, (double)(t[3] - t[0]));
        }
        printf("init loads %.2f us, init reduce %.2f us, loop %.2f us (per-CTA means), start->loop end max %.2f us\n",
               a / G / 1e3, b2 / G / 1e3, c2 / G / 1e3, mx / 1e3);
    }
    {   // collect #1 internals (clock64 cycles): first poll, spin phase, spin count
        double fp = 0, sp = 0, ns = 0, fpmax = 0, spmax = 0;
        int n = 0;
        for (int b = 0; b < G; b++)
            for (int it = 1; it < 8; it++) {
                const double a1 = (double)ht[((size_t)b * 16 + 12) * 8 + it], a2 = (double)ht[((size_t)b * 16 + 13) * 8 + it];
                fp += a1; sp += a2; ns += (double)ht[((size_t)b * 16 + 14) * 8 + it];
                fpmax = std::max(fpmax, a1); spmax = std::max(spmax, a2); n++;
            }
        printf("collect #1: first poll %.0f cyc (max %.0f), spin %.0f cyc (max %.0f), spins %.2f (means over CTAs x iterations)\n",
               fp / n, fpmax, sp / n, spmax, ns / n);
    }
    {   // skew: per CTA, mean over iterations of (publish #1 time - earliest CTA's publish #1) and
        // of its compute time (local + remote phases); slowest CTAs listed
        std::vector<std::pair<double, int>> late(G), comp(G);
        for (int b = 0; b < G; b++) { late[b] = {0.0, b}; comp[b] = {0.0, b}; }
        for (int it = 1; it < 9; it++) {
            unsigned long long mn = ~0ull;
            for (int b = 0; b < G; b++) mn = std::min(mn, ht[((size_t)b * 16 + it) * 8 + 2]);
            for (int b = 0; b < G; b++) {
                const unsigned long long* t = &ht[((size_t)b * 16 + it) * 8];
                late[b].first += (double)(t[2] - mn) / 8e3;
                comp[b].first += (double)((t[2] - t[1]) + (t[1] - t[0])) / 8e3;
            }
        }
        std::sort(late.begin(), late.end());
        std::sort(comp.begin(), comp.end());
        printf("remote-done lateness vs earliest CTA (us): min %.2f p50 %.2f p90 %.2f max %.2f; latest CTAs:",
               late[0].first, late[G / 2].first, late[G * 9 / 10].first, late[G - 1].first);
        for (int q = G - 1; q >= G - 8; q--) printf(" %d(%.2f)", late[q].second, late[q].first);
        printf("\nlocal+remote time per CTA (us): min %.2f p50 %.2f p90 %.2f max %.2f; slowest:", comp[0].first,
               comp[G / 2].first, comp[G * 9 / 10].first, comp[G - 1].first);
        for (int q = G - 1; q >= G - 8; q--) printf(" %d(%.2f)", comp[q].second, comp[q].first);
        printf("\n");
    }
    // iteration period
    double per = 0;
    for (int it = 1; it < 9; it++) per += (double)(ht[(size_t)it * 8 + 0] - ht[(size_t)(it - 1) * 8 + 0]);
    printf("iteration period (CTA 0): %.2f us\n", per / 8 / 1e3);
    PairState hs2; cudaMemcpy(&hs2, st, sizeof hs2, cudaMemcpyDeviceToHost);
    printf("pcg_k %d h_evals %d relres %.3e\n", hs2.pcg_k, hs2.h_evals, hs2.relres);
    if (tiled) {   // the tiled kernel's q against the strip kernel's (same problem)
        std::vector<float> xt(Nn), xs(Nn);
        cudaMemcpy(xt.data(), x, Nn * 4, cudaMemcpyDeviceToHost);
        cudaLaunchConfig_t c2 = cfg;
        c2.gridDim = dim3(G);
        cudaMemset(bb, 0, Nn * 4);
        cudaMemset(pgh, 0, ghost * 4);   // the strip layout's zero ghost planes (the tiled runs used the buffer)
        cudaMemcpy(st, &hs, sizeof hs, cudaMemcpyHostToDevice);
        cudaLaunchKernelEx(&c2, pcg_resident_kernel<RES_KMAX, true>, g, c, sp, 0, (const float*)grad, (const float*)dt,
                           (const float*)et, x, xpad, pgh, part, flags, wi, wj, bb, bo, 1, (unsigned long long*)nullptr, tl);
        cudaDeviceSynchronize();
        cudaMemcpy(xs.data(), x, Nn * 4, cudaMemcpyDeviceToHost);
        double num = 0, den = 0, mx = 0;
        for (size_t t = 0; t < Nn; t++) { const double d = (double)xt[t] - xs[t]; num += d * d; den += (double)xs[t] * xs[t]; mx = std::max(mx, fabs(d)); }
        printf("tiled vs strip q: rel L2 %.3e, max abs %.3e (err=%s)\n", sqrt(num / den), mx, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
