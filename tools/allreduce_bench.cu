// Microbenchmark: grid-wide fp64 all-reduce latency with one 512-thread CTA
// per SM (cooperative launch), two deterministic designs:
//  (a) all-poll-all: every CTA publishes a tagged partial to 16 replicas and
//      polls all G partials (hysco_resident.cuh reduce_publish / collect);
//  (b) ticket: every CTA stores its partial and takes an arrival ticket
//      (atomicAdd); the last arriver folds the G partials in fixed order and
//      publishes the tagged total to 16 replicas; the others poll one replica.
#include <cstdio>
#include <cooperative_groups.h>
constexpr unsigned FULL = 0xffffffffu;
constexpr int REPL = 16, RSTR = 512;
__device__ __forceinline__ double ld_rel(const double* p) { double v; asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(double* p, double v) { asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }
__device__ __forceinline__ double tagv(double v, unsigned t) { return __longlong_as_double((__double_as_longlong(v) & ~0xffll) | (long long)t); }
__device__ __forceinline__ unsigned vtag(double v) { return (unsigned)(__double_as_longlong(v) & 0xff); }
__device__ double block_sum(double x) {
  __shared__ double s[32];
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = x;
  __syncthreads();
  double y = 0; if (threadIdx.x < 32) { y = threadIdx.x < (blockDim.x >> 5) ? s[threadIdx.x] : 0.0; for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o); }
  return y;   // valid in warp 0
}
__global__ void __launch_bounds__(512, 1) k_poll(double* part, int iters, double* out) {
  __shared__ double tot;
  const int G = gridDim.x; double acc = 0;
  for (int it = 0; it < iters; it++) {
    const unsigned tag = (unsigned)(it & 255);
    double x = block_sum(1.0 + threadIdx.x * 1e-3);
    double* pb = part + (it & 1) * REPL * RSTR;   // two buffers: a CTA is at most one all-reduce ahead
    if (threadIdx.x < 32 && threadIdx.x < REPL) st_rel(pb + threadIdx.x * RSTR + blockIdx.x, tagv(x, tag));
    if (threadIdx.x < 32) {
      const double* p = pb + (blockIdx.x % REPL) * RSTR; const int lane = threadIdx.x;
      double v[8]; unsigned pend = 0;
      for (int m = 0; m < 8; m++) { const int b = lane + 32 * m; v[m] = 0; if (b < G) { v[m] = ld_rel(p + b); if (vtag(v[m]) != tag) pend |= 1u << m; } }
      unsigned spins = 0;
      while (__any_sync(FULL, pend != 0) && ++spins < (1u << 22)) for (int m = 0; m < 8; m++) if (pend & (1u << m)) { v[m] = ld_rel(p + lane + 32 * m); if (vtag(v[m]) == tag) pend &= ~(1u << m); }
      double y = 0; for (int m = 0; m < 8; m++) y += v[m];
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
      if (lane == 0) tot = y;
    }
    __syncthreads();
    acc += tot;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}
__global__ void __launch_bounds__(512, 1) k_ticket(double* part, double* total, unsigned* ticket, int iters, double* out) {
  __shared__ double tot; __shared__ int last;
  const int G = gridDim.x; double acc = 0;
  for (int it = 0; it < iters; it++) {
    unsigned* tk = ticket + 32 * (it & 1);   // per-parity arrival counter, reset by its last arriver
    const unsigned tag = (unsigned)(it & 255);
    double x = block_sum(1.0 + threadIdx.x * 1e-3);
    if (threadIdx.x == 0) {
      st_rel(part + (it & 1) * RSTR + blockIdx.x, x);
      __threadfence();
      const unsigned t = atomicAdd(tk, 1u);
      last = t == (unsigned)(G - 1);
      if (last) *(volatile unsigned*)tk = 0;
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {   // fixed-order fold of all partials, then publish
      __threadfence();
      const int lane = threadIdx.x; double y = 0;
      for (int b = lane; b < G; b += 32) y += ld_rel(part + (it & 1) * RSTR + b);
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
      if (lane < REPL) st_rel(total + lane * RSTR, tagv(y, tag));
    }
    if (threadIdx.x == 0) {
      const double* p = total + (blockIdx.x % REPL) * RSTR; double y;
      unsigned spins = 0;
      do { y = ld_rel(p); if (++spins > (1u << 22)) __trap(); } while (vtag(y) != tag);
      tot = y;
    }
    __syncthreads();
    acc += tot;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}

__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) { unsigned o; asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }
__global__ void __launch_bounds__(512, 1) k_ticket2(double* part, double* total, unsigned* ticket, int iters, double* out) {
  __shared__ double tot; __shared__ int last;
  const int G = gridDim.x; double acc = 0;
  for (int it = 0; it < iters; it++) {
    unsigned* tk = ticket + 32 * (it & 1);
    const unsigned tag = (unsigned)(it & 255);
    double x = block_sum(1.0 + threadIdx.x * 1e-3);
    if (threadIdx.x == 0) {
      st_rel(part + (it & 1) * RSTR + blockIdx.x, x);
      const unsigned t = atom_add_acqrel(tk, 1u);      // release the partial, acquire the others' (last)
      last = t == (unsigned)(G - 1);
      if (last) *(volatile unsigned*)tk = 0;
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {
      const int lane = threadIdx.x; double y = 0;
      for (int b = lane; b < G; b += 32) y += ld_rel(part + (it & 1) * RSTR + b);
      for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
      if (lane < REPL) st_rel(total + lane * RSTR, tagv(y, tag));
    }
    if (threadIdx.x == 0) {
      const double* p = total + (blockIdx.x % REPL) * RSTR; double y;
      unsigned spins = 0;
      do { y = ld_rel(p); if (++spins > (1u << 22)) __trap(); } while (vtag(y) != tag);
      tot = y;
    }
    __syncthreads();
    acc += tot;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = acc;
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *part, *total, *out; unsigned* ticket;
  cudaMalloc(&part, 2 * sizeof(double) * REPL * RSTR); cudaMemset(part, 0xff, 2 * sizeof(double) * REPL * RSTR);
  cudaMalloc(&total, sizeof(double) * REPL * RSTR); cudaMemset(total, 0xff, sizeof(double) * REPL * RSTR);
  cudaMalloc(&ticket, 256); cudaMemset(ticket, 0, 256); cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; rep++) {
    int iters = 2000; float t1, t2;
    void* a1[] = {&part, &iters, &out}; void* a2[] = {&part, &total, &ticket, &iters, &out};
    cudaMemset(part, 0xfe, 2 * sizeof(double) * REPL * RSTR);
    cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_poll, nsm, 512, a1, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t1, e0, e1);
    double r1; cudaMemcpy(&r1, out, 8, cudaMemcpyDeviceToHost);
    cudaMemset(total, 0xfe, sizeof(double) * REPL * RSTR);
    cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_ticket, nsm, 512, a2, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t2, e0, e1);
    double r2; cudaMemcpy(&r2, out, 8, cudaMemcpyDeviceToHost);
    float t3; cudaMemset(total, 0xfd, sizeof(double) * REPL * RSTR);
    cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_ticket2, nsm, 512, a2, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t3, e0, e1);
    printf("ticket acq_rel atomic (no membar): %.3f us\n", t3 * 1e3 / iters);
    printf("G=%d: all-poll-all %.3f us, ticket %.3f us per all-reduce (sums %.6g %.6g) %s\n", nsm, t1 * 1e3 / iters, t2 * 1e3 / iters, r1, r2, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
