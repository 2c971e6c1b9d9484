// Microbenchmark: grid-wide deterministic fp64 all-reduce designs for the
// resident PCG (one 512-thread CTA per SM, cooperative launch), per
// all-reduce of NV = 2 values:
//  poll     : tagged partials published to 16 replicas, every CTA polls all
//             G partials (hysco_resident.cuh reduce_publish / reduce_collect)
//  flip     : partials stored plainly, then a flip barrier (one red.release
//             arrive per CTA on one word, acquire-poll of its phase bit),
//             then every CTA reads the G partials and folds them in order
//  flipsplit: the same with the word replicated per die half (two arrive
//             words; pollers read their own half's copy) -- not used
//  cg       : cooperative_groups grid.sync() then the fold
//  bar      : the flip barrier alone (no data)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/sync_bench tools/sync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
constexpr unsigned FULL = 0xffffffffu;
constexpr int REPL = 16, RSTR = 512, NV = 2;

__device__ __forceinline__ double ld_rel(const double* p) { double v; asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(double* p, double v) { asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_rlx32(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ double tagv(double v, unsigned t) { return __longlong_as_double((__double_as_longlong(v) & ~0xffll) | (long long)t); }
__device__ __forceinline__ unsigned vtag(double v) { return (unsigned)(__double_as_longlong(v) & 0xff); }

// block reduce of NV values; result valid in all threads via shared memory
__device__ __forceinline__ void block_red(double (&v)[NV], double (&out)[NV]) {
  __shared__ double s[NV][32];
  __shared__ double t[NV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k = 0; k < NV; k++) { double x = v[k]; for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o); if (lane == 0) s[k][wid] = x; }
  __syncthreads();
  if (wid < NV) { double x = lane < (int)(blockDim.x >> 5) ? s[wid][lane] : 0.0; for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o); if (lane == 0) t[wid] = x; }
  __syncthreads();
  for (int k = 0; k < NV; k++) out[k] = t[k];
}

// fold the G x NV partials at part (fixed order), by warps 0..NV-1, result in out
__device__ __forceinline__ void fold(const double* part, double (&out)[NV]) {
  __shared__ double t[NV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, G = gridDim.x;
  if (wid < NV) {
    double y = 0;
#pragma unroll
    for (int m = 0; m < 8; m++) { const int b = lane + 32 * m; if (b < G) y += ld_rel(part + b * NV + wid); }
    for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
    if (lane == 0) t[wid] = y;
  }
  __syncthreads();
  for (int k = 0; k < NV; k++) out[k] = t[k];
}

// ---------------- poll (current design)
__global__ void __launch_bounds__(512, 1) k_poll(double* part, int iters, double* out) {
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc = 0;
  __shared__ double tot[NV];
  for (int it = 0; it < iters; it++) {
    const unsigned tag = (unsigned)(it & 255);
    double v[NV] = {1.0 + threadIdx.x, 2.0}, b[NV];
    block_red(v, b);
    double* pb = part + (it % 3) * REPL * RSTR;
    if (wid < NV && lane < REPL) st_rel(pb + lane * RSTR + blockIdx.x * NV + wid, tagv(b[wid], tag));
    if (wid < NV) {
      const double* p = pb + (blockIdx.x % REPL) * RSTR;
      double x[8]; unsigned pend = 0;
      for (int m = 0; m < 8; m++) { const int bb = lane + 32 * m; x[m] = 0; if (bb < G) { x[m] = ld_rel(p + bb * NV + wid); if (vtag(x[m]) != tag) pend |= 1u << m; } }
      unsigned spins = 0;
      while (__any_sync(FULL, pend != 0)) { if (++spins > (1u << 24)) __trap(); for (int m = 0; m < 8; m++) if (pend & (1u << m)) { x[m] = ld_rel(p + (lane + 32 * m) * NV + wid); if (vtag(x[m]) == tag) pend &= ~(1u << m); } }
      double y = 0; for (int m = 0; m < 8; m++) y += x[m];
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
      if (lane == 0) tot[wid] = y;
    }
    __syncthreads();
    acc += tot[0] + tot[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

// ---------------- flip barrier + fold
__device__ __forceinline__ void flip_arrive(unsigned* bar) {
  red_rel(bar, blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u);
}
__device__ __forceinline__ void flip_wait(const unsigned* bar, unsigned phase) {
  unsigned spins = 0;
  while ((ld_acq(bar) & 0x80000000u) == phase) if (++spins > (1u << 26)) __trap();
}
template <bool SPLIT>
__global__ void __launch_bounds__(512, 1) k_flip(double* part, unsigned* bar, int iters, double* out) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0;
  unsigned phase = *reinterpret_cast<volatile unsigned*>(bar) & 0x80000000u;
  for (int it = 0; it < iters; it++) {
    double v[NV] = {1.0 + threadIdx.x, 2.0}, b[NV], t[NV];
    block_red(v, b);
    double* pb = part + (it & 1) * RSTR;     // double buffer: a CTA is < 1 all-reduce ahead
    if (wid < NV && lane == 0) st_rel(pb + blockIdx.x * NV + wid, b[wid]);
    __syncthreads();                          // both partial stores before the release
    if (threadIdx.x == 0) { flip_arrive(bar); flip_wait(bar, phase); }
    phase ^= 0x80000000u;
    __syncthreads();
    fold(pb, t);
    acc += t[0] + t[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

// ---------------- flip with the arrive by the partial-writing warps directly
// (warp k stores value k and arrives with red.release; no extra syncthreads)
__global__ void __launch_bounds__(512, 1) k_flip2(double* part, unsigned* bar, int iters, double* out) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0;
  unsigned phase = *reinterpret_cast<volatile unsigned*>(bar) & 0x80000000u;
  __shared__ double s[NV][32];
  __shared__ double tt[NV];
  for (int it = 0; it < iters; it++) {
    double v[NV] = {1.0 + threadIdx.x, 2.0};
    for (int k = 0; k < NV; k++) { double x = v[k]; for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o); if (lane == 0) s[k][wid] = x; }
    __syncthreads();
    double* pb = part + (it & 1) * RSTR;
    if (wid == 0) {
      // warp 0 folds both values (lanes 0..15 value 0, 16..31 value 1)
      const int k = lane >> 4, w = lane & 15;
      double x = w < (int)(blockDim.x >> 5) ? s[k][w] : 0.0;
      for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
      if (w == 0) st_rel(pb + blockIdx.x * NV + k, x);
      __syncwarp();
      if (lane == 0) { flip_arrive(bar); flip_wait(bar, phase); }
      __syncwarp();
      // fold: lane handles CTAs lane, lane+32, ...; both values
      double y0 = 0, y1 = 0;
      for (int m = 0; m < 8; m++) { const int b = lane + 32 * m; if (b < (int)gridDim.x) { y0 += ld_rel(pb + b * NV); y1 += ld_rel(pb + b * NV + 1); } }
      for (int o = 16; o > 0; o >>= 1) { y0 += __shfl_xor_sync(FULL, y0, o); y1 += __shfl_xor_sync(FULL, y1, o); }
      if (lane == 0) { tt[0] = y0; tt[1] = y1; }
    }
    phase ^= 0x80000000u;
    __syncthreads();
    acc += tt[0] + tt[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

// ---------------- cg grid sync + fold
__global__ void __launch_bounds__(512, 1) k_cg(double* part, int iters, double* out) {
  cg::grid_group gg = cg::this_grid();
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0;
  for (int it = 0; it < iters; it++) {
    double v[NV] = {1.0 + threadIdx.x, 2.0}, b[NV], t[NV];
    block_red(v, b);
    double* pb = part + (it & 1) * RSTR;
    if (wid < NV && lane == 0) st_rel(pb + blockIdx.x * NV + wid, b[wid]);
    gg.sync();
    fold(pb, t);
    acc += t[0] + t[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

// ---------------- barrier only
__global__ void __launch_bounds__(512, 1) k_bar(unsigned* bar, int iters, double* out) {
  unsigned phase = *reinterpret_cast<volatile unsigned*>(bar) & 0x80000000u;
  for (int it = 0; it < iters; it++) {
    __syncthreads();
    if (threadIdx.x == 0) { flip_arrive(bar); flip_wait(bar, phase); }
    phase ^= 0x80000000u;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = phase;
}

// ---------------- relaxed-poll barrier (ld.relaxed poll then one fence)
__global__ void __launch_bounds__(512, 1) k_bar_rlx(unsigned* bar, int iters, double* out) {
  unsigned phase = *reinterpret_cast<volatile unsigned*>(bar) & 0x80000000u;
  for (int it = 0; it < iters; it++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      flip_arrive(bar);
      unsigned spins = 0;
      while ((ld_rlx32(bar) & 0x80000000u) == phase) if (++spins > (1u << 26)) __trap();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    phase ^= 0x80000000u;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = phase;
}

// ---------------- neighbourhood flag wait (the p halo): release own flag,
// acquire flags of CTAs b-2..b+2
__global__ void __launch_bounds__(512, 1) k_halo(unsigned* flags, int iters, double* out) {
  const int G = gridDim.x;
  const int lo = max(0, (int)blockIdx.x - 2), hi = min(G - 1, (int)blockIdx.x + 2);
  for (int it = 1; it <= iters; it++) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"((unsigned)it) : "memory");
    if (threadIdx.x < 32) {
      for (int b = lo + (int)threadIdx.x; b <= hi; b += 32) { unsigned s = 0; while ((int)(ld_acq(flags + b * 32) - it) < 0) if (++s > (1u << 26)) __trap(); }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 1;
}


// ---------------- block reduction alone
__global__ void __launch_bounds__(512, 1) k_red(int iters, double* out) {
  double acc = 0;
  for (int it = 0; it < iters; it++) { double v[NV] = {1.0 + threadIdx.x + it, 2.0}, b[NV]; block_red(v, b); acc += b[0] + b[1]; }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}
// ---------------- barrier with relaxed arrive / relaxed poll (no fences: latency only)
__device__ __forceinline__ void red_rlx(unsigned* p, unsigned v) { asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__global__ void __launch_bounds__(512, 1) k_bar_nofence(unsigned* bar, int iters, double* out) {
  unsigned phase = *reinterpret_cast<volatile unsigned*>(bar) & 0x80000000u;
  for (int it = 0; it < iters; it++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      red_rlx(bar, blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u);
      unsigned spins = 0;
      while ((ld_rlx32(bar) & 0x80000000u) == phase) if (++spins > (1u << 26)) __trap();
    }
    phase ^= 0x80000000u;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = phase;
}
// ---------------- halo with relaxed flag store / relaxed poll
__global__ void __launch_bounds__(512, 1) k_halo_rlx(unsigned* flags, int iters, double* out) {
  const int G = gridDim.x;
  const int lo = max(0, (int)blockIdx.x - 2), hi = min(G - 1, (int)blockIdx.x + 2);
  for (int it = 1; it <= iters; it++) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"((unsigned)it) : "memory");
    if (threadIdx.x < 32) {
      for (int b = lo + (int)threadIdx.x; b <= hi; b += 32) { unsigned s = 0; while ((int)(ld_rlx32(flags + b * 32) - it) < 0) if (++s > (1u << 26)) __trap(); }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 1;
}
// ---------------- tagged poll without the block reduction: one warp publishes
// a per-CTA constant (NV values) and polls; isolates the poll round trip
template <int R>
__global__ void __launch_bounds__(512, 1) k_pollw(double* part, int iters, double* out) {
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc = 0;
  __shared__ double tot[NV];
  for (int it = 0; it < iters; it++) {
    const unsigned tag = (unsigned)(it & 255);
    double* pb = part + (it % 3) * REPL * RSTR;
    if (wid < NV && lane < R) st_rel(pb + lane * RSTR + blockIdx.x * NV + wid, tagv(1.0 + blockIdx.x, tag));
    if (wid < NV) {
      const double* p = pb + (blockIdx.x % R) * RSTR;
      double x[8]; unsigned pend = 0;
      for (int m = 0; m < 8; m++) { const int bb = lane + 32 * m; x[m] = 0; if (bb < G) { x[m] = ld_rel(p + bb * NV + wid); if (vtag(x[m]) != tag) pend |= 1u << m; } }
      unsigned spins = 0;
      while (__any_sync(FULL, pend != 0)) { if (++spins > (1u << 24)) __trap(); for (int m = 0; m < 8; m++) if (pend & (1u << m)) { x[m] = ld_rel(p + (lane + 32 * m) * NV + wid); if (vtag(x[m]) == tag) pend &= ~(1u << m); } }
      double y = 0; for (int m = 0; m < 8; m++) y += x[m];
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
      if (lane == 0) tot[wid] = y;
    }
    __syncthreads();
    acc += tot[0] + tot[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}
// ---------------- tagged poll, one word per CTA (both values packed as two
// fp32-tagged halves is not exact; instead NV values in ONE 16-byte store
// (v2.f64) and one 16-byte poll per CTA slot)
__device__ __forceinline__ void st_rel2(double* p, double a, double b) { asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory"); }
__device__ __forceinline__ void ld_rel2(const double* p, double& a, double& b) { asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p) : "memory"); }
__global__ void __launch_bounds__(512, 1) k_poll2(double* part, int iters, double* out) {
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc = 0;
  __shared__ double tot[NV];
  for (int it = 0; it < iters; it++) {
    const unsigned tag = (unsigned)(it & 255);
    double* pb = part + (it % 3) * REPL * RSTR;
    if (wid == 0 && lane < REPL) st_rel2(pb + lane * RSTR + blockIdx.x * 2, tagv(1.0 + blockIdx.x, tag), tagv(2.0, tag));
    if (wid == 0) {
      const double* p = pb + (blockIdx.x % REPL) * RSTR;
      double x[5], y2[5]; unsigned pend = 0;
      for (int m = 0; m < 5; m++) { const int bb = lane + 32 * m; x[m] = 0; y2[m] = 0; if (bb < G) { ld_rel2(p + bb * 2, x[m], y2[m]); if (vtag(x[m]) != tag || vtag(y2[m]) != tag) pend |= 1u << m; } }
      unsigned spins = 0;
      while (__any_sync(FULL, pend != 0)) { if (++spins > (1u << 24)) __trap(); for (int m = 0; m < 5; m++) if (pend & (1u << m)) { ld_rel2(p + (lane + 32 * m) * 2, x[m], y2[m]); if (vtag(x[m]) == tag && vtag(y2[m]) == tag) pend &= ~(1u << m); } }
      double s0 = 0, s1 = 0; for (int m = 0; m < 5; m++) { s0 += x[m]; s1 += y2[m]; }
      for (int o = 16; o > 0; o >>= 1) { s0 += __shfl_xor_sync(FULL, s0, o); s1 += __shfl_xor_sync(FULL, s1, o); }
      if (lane == 0) { tot[0] = s0; tot[1] = s1; }
    }
    __syncthreads();
    acc += tot[0] + tot[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

// ---------------- two-level tagged tree: members -> group leader (GS CTAs per
// group) -> every CTA polls the ngroups group sums (R replicas).  No fences,
// no atomics; every CTA folds the same values in the same order.
template <int GS, int R, bool BLOCKRED>
__global__ void __launch_bounds__(512, 1) k_tree(double* part, int iters, double* out) {
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ng = (G + GS - 1) / GS;
  double acc = 0;
  __shared__ double tot[NV];
  for (int it = 0; it < iters; it++) {
    const unsigned tag = (unsigned)(it & 255);
    double* p1 = part + (it % 3) * 2 * RSTR * 16;
    double* p2 = p1 + RSTR;
    double bv[NV] = {1.0 + blockIdx.x, 2.0};
    if (BLOCKRED) { double v[NV] = {1.0 + threadIdx.x, 2.0}; block_red(v, bv); }
    if (wid < NV) {
      if (lane == 0) st_rel(p1 + blockIdx.x * NV + wid, tagv(bv[wid], tag));
      if (blockIdx.x % GS == 0) {                 // group leader
        const int b = blockIdx.x + lane;
        double x = 0;
        if (lane < GS && b < G) { unsigned s = 0; do { x = ld_rel(p1 + b * NV + wid); if (++s > (1u << 24)) __trap(); } while (vtag(x) != tag); }
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
        if (lane < R) st_rel(p2 + lane * RSTR + (blockIdx.x / GS) * NV + wid, tagv(x, tag));
      }
      double y = 0;
      if (lane < ng) { const double* q = p2 + (blockIdx.x % R) * RSTR + lane * NV + wid; unsigned s = 0; do { y = ld_rel(q); if (++s > (1u << 24)) __trap(); } while (vtag(y) != tag); }
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
      if (lane == 0) tot[wid] = y;
    }
    __syncthreads();
    acc += tot[0] + tot[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

// ---------------- tree with every slot on its own 128-byte line (SL doubles apart)
template <int GS, int R, int SL, int NS>
__global__ void __launch_bounds__(512, 1) k_treep(double* part, int iters, double* out) {
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ng = (G + GS - 1) / GS;
  double acc = 0;
  __shared__ double tot[NV];
  for (int it = 0; it < iters; it++) {
    const unsigned tag = (unsigned)(it & 255);
    double* p1 = part + (it % 3) * (256 * NV * SL + R * 32 * NV * SL);
    double* p2 = p1 + 256 * NV * SL;
    if (wid < NV) {
      if (lane == 0) st_rel(p1 + (blockIdx.x * NV + wid) * SL, tagv(1.0 + blockIdx.x, tag));
      if (blockIdx.x % GS == 0) {
        const int b = blockIdx.x + lane;
        double x = 0;
        if (lane < GS && b < G) { unsigned s = 0; while (true) { x = ld_rel(p1 + (b * NV + wid) * SL); if (vtag(x) == tag) break; if (++s > (1u << 24)) __trap(); if (NS) __nanosleep(NS); } }
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
        if (lane < R) st_rel(p2 + ((lane * 32 + blockIdx.x / GS) * NV + wid) * SL, tagv(x, tag));
      }
      double y = 0;
      if (lane < ng) { const double* q = p2 + (((blockIdx.x % R) * 32 + lane) * NV + wid) * SL; unsigned s = 0; while (true) { y = ld_rel(q); if (vtag(y) == tag) break; if (++s > (1u << 24)) __trap(); if (NS) __nanosleep(NS); } }
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
      if (lane == 0) tot[wid] = y;
    }
    __syncthreads();
    acc += tot[0] + tot[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}
// ---------------- all-poll with padded slots: every CTA polls G lines
template <int SL, int R, int NS>
__global__ void __launch_bounds__(512, 1) k_pollp(double* part, int iters, double* out) {
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc = 0;
  __shared__ double tot[NV];
  for (int it = 0; it < iters; it++) {
    const unsigned tag = (unsigned)(it & 255);
    double* pb = part + (it % 3) * (R * 256 * NV * SL);
    if (wid < NV && lane < R) st_rel(pb + ((lane * 256 + blockIdx.x) * NV + wid) * SL, tagv(1.0 + blockIdx.x, tag));
    if (wid < NV) {
      const double* p = pb + ((blockIdx.x % R) * 256 * NV + wid) * SL;
      double x[8]; unsigned pend = 0;
      for (int m = 0; m < 8; m++) { const int bb = lane + 32 * m; x[m] = 0; if (bb < G) { x[m] = ld_rel(p + bb * NV * SL); if (vtag(x[m]) != tag) pend |= 1u << m; } }
      unsigned spins = 0;
      while (__any_sync(FULL, pend != 0)) { if (++spins > (1u << 24)) __trap(); if (NS) __nanosleep(NS); for (int m = 0; m < 8; m++) if (pend & (1u << m)) { x[m] = ld_rel(p + (lane + 32 * m) * NV * SL); if (vtag(x[m]) == tag) pend &= ~(1u << m); } }
      double y = 0; for (int m = 0; m < 8; m++) y += x[m];
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
      if (lane == 0) tot[wid] = y;
    }
    __syncthreads();
    acc += tot[0] + tot[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

// ---------------- exact fixed-point limb all-reduce: each value is scaled by
// a power of two S, split into NL 40-bit limbs, and each limb is added as
// (limb << 8) + 1 to a 64-bit word by red.relaxed (its own arrival count in
// the low byte); readers poll the words until every count reached G (words
// never reset: deltas against the previous final value, two parity buffers).
__device__ __forceinline__ void red_add_s64(unsigned long long* p, long long v) { asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ unsigned long long ld_rlx64(const unsigned long long* p) { unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
template <int WS>
__global__ void __launch_bounds__(512, 1) k_limb(unsigned long long* words, int iters, double* out) {
  // words: [2 parity][NV * 3 limbs] each WS u64 apart
  const int G = gridDim.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = NV * 3;
  double acc = 0;
  __shared__ double tot[NV];
  unsigned long long prev[2] = {0, 0};   // lane l < NW: last final value of its word, per parity
  if (wid == 0 && lane < NW) { prev[0] = ld_rlx64(words + lane * WS); prev[1] = ld_rlx64(words + (NW + lane) * WS); }
  for (int it = 0; it < iters; it++) {
    const int par = it & 1;
    if (wid == 0) {
      const double vals[NV] = {1.0 + blockIdx.x * 0.37, 2.0 - blockIdx.x * 1e-3};
      if (lane < NW) {
        const int k = lane / 3, li = lane % 3;
        const double q = vals[k] * 0x1p-8;              // S = 2^8 (example scale)
        const double a2 = floor(q * 0x1p20), r1 = q * 0x1p20 - a2;
        const double a1 = floor(r1 * 0x1p40), r0 = r1 * 0x1p40 - a1;
        const double a0 = rint(r0 * 0x1p40);
        const long long limb = li == 2 ? (long long)a2 : li == 1 ? (long long)a1 : (long long)a0;
        red_add_s64(words + (par * NW + lane) * WS, limb * 256 + 1);
        unsigned long long cur; unsigned s = 0;
        while (true) { cur = ld_rlx64(words + (par * NW + lane) * WS); if (((cur - prev[par]) & 255ull) == (unsigned long long)(G & 255)) break; if (++s > (1u << 24)) __trap(); }
        const long long d = (long long)(cur - prev[par]);
        prev[par] = cur;
        const double S = (double)((d - (G & 255)) >> 8);   // exact: |.| < 2^49
        // combine per value: lanes 3k..3k+2
        const double s2 = __shfl_sync(0x3fu, S, 3 * k + 2), s1 = __shfl_sync(0x3fu, S, 3 * k + 1), s0 = __shfl_sync(0x3fu, S, 3 * k);
        if (li == 0) tot[k] = ((s2 * 0x1p-20 + s1 * 0x1p-60) + s0 * 0x1p-100) * 0x1p8;
      }
    }
    __syncthreads();
    acc += tot[0] + tot[1];
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *part, *out; unsigned *bar, *flags;
  cudaMalloc(&part, 6 * 16 * sizeof(double) * REPL * RSTR); cudaMemset(part, 0xff, 6 * 16 * sizeof(double) * REPL * RSTR);
  cudaMalloc(&bar, 256); cudaMemset(bar, 0, 256);
  cudaMalloc(&flags, 4 * 32 * 256); cudaMemset(flags, 0, 4 * 32 * 256);
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  auto run = [&](const char* name, void* fn, void** args) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; rep++) {
      cudaMemset(flags, 0, 4 * 32 * 256);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel(fn, nsm, 512, args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float t; cudaEventElapsedTime(&t, e0, e1); if (t < best) best = t;
    }
    double r; cudaMemcpy(&r, out, 8, cudaMemcpyDeviceToHost);
    printf("%-10s %.3f us per op  (check %.6g) %s\n", name, best * 1e3 / iters, r, cudaGetErrorString(cudaGetLastError()));
  };
  void* ap[] = {&part, &iters, &out};
  void* af[] = {&part, &bar, &iters, &out};
  void* ab[] = {&bar, &iters, &out};
  void* ah[] = {&flags, &iters, &out};
  printf("G = %d CTAs x 512 threads\n", nsm);
  run("poll", (void*)k_poll, ap);
  run("flip", (void*)k_flip<false>, af);
  run("flip2", (void*)k_flip2, af);
  run("cg", (void*)k_cg, ap);
  run("bar", (void*)k_bar, ab);
  run("bar_rlx", (void*)k_bar_rlx, ab);
  run("halo", (void*)k_halo, ah);
  void* ai[] = {&iters, &out};
  run("red", (void*)k_red, ai);
  run("bar_nof", (void*)k_bar_nofence, ab);
  run("halo_rlx", (void*)k_halo_rlx, ah);
  run("pollw16", (void*)k_pollw<16>, ap);
  run("pollw1", (void*)k_pollw<1>, ap);
  run("pollw4", (void*)k_pollw<4>, ap);
  run("poll2v", (void*)k_poll2, ap);
  run("tree8r4", (void*)k_tree<8, 4, false>, ap);
  run("tree12r4", (void*)k_tree<12, 4, false>, ap);
  run("tree16r4", (void*)k_tree<16, 4, false>, ap);
  run("tree12r1", (void*)k_tree<12, 1, false>, ap);
  run("tree12r8", (void*)k_tree<12, 8, false>, ap);
  run("tree24r4", (void*)k_tree<24, 4, false>, ap);
  run("tree12r4B", (void*)k_tree<12, 4, true>, ap);
  run("poll_B", (void*)k_poll, ap);
  run("limb16", (void*)k_limb<16>, ap);
  run("limb1", (void*)k_limb<1>, ap);
  run("limb64", (void*)k_limb<64>, ap);
  run("treep12", (void*)k_treep<12, 4, 16, 0>, ap);
  run("treep16", (void*)k_treep<16, 4, 16, 0>, ap);
  run("treep12s", (void*)k_treep<12, 4, 16, 64>, ap);
  run("treep12_1", (void*)k_treep<12, 1, 16, 0>, ap);
  run("treep12_s4", (void*)k_treep<12, 4, 4, 0>, ap);
  run("pollp1", (void*)k_pollp<16, 1, 0>, ap);
  run("pollp4", (void*)k_pollp<16, 4, 0>, ap);
  run("pollp4s", (void*)k_pollp<16, 4, 100>, ap);
  run("pollw4s", (void*)k_pollp<1, 4, 100>, ap);
  return 0;
}
