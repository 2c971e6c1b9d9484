// Microbenchmark: cost of one grid-wide barrier (148 CTAs x 768 threads, one per SM),
// comparing the generation barrier of hysco_resident.cuh with cooperative_groups grid.sync().
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) { unsigned o; asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o; }
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ void bar_gen(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) { const unsigned g0 = ld_acquire(gen);
    if (atom_add_acq_rel(count, 1u) == gridDim.x - 1) { *reinterpret_cast<volatile unsigned*>(count) = 0; red_release(gen, 1u); }
    else { while (ld_acquire(gen) == g0) {} } }
  __syncthreads();
}
// flip barrier with a fire-and-forget arrive: the phase bit is tracked locally
// (it cannot flip before this CTA arrives), so the arrive needs no return value
__device__ __forceinline__ void red_release_u32(unsigned* p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ void bar_flip(unsigned* bar, unsigned& phase) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_u32(bar, blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u);
    while ((ld_acquire(bar) & 0x80000000u) == phase) {}
  }
  phase ^= 0x80000000u;
  __syncthreads();
}
__global__ void k_flip(unsigned* b, int n, float* sink) {
  unsigned phase = *reinterpret_cast<volatile unsigned*>(b + 2) & 0x80000000u;
  float acc = 0; for (int i = 0; i < n; i++) { bar_flip(b + 2, phase); acc += i; } if (acc < 0) sink[0] = acc; }
__global__ void k_gen(unsigned* b, int n, float* sink) { float acc = 0; for (int i = 0; i < n; i++) { bar_gen(b, b + 1); acc += i; } if (acc < 0) sink[0] = acc; }
__global__ void k_cg(int n, float* sink) { cg::grid_group g = cg::this_grid(); float acc = 0; for (int i = 0; i < n; i++) { g.sync(); acc += i; } if (acc < 0) sink[0] = acc; }
__global__ void k_sync(int n, float* sink) { float acc = 0; for (int i = 0; i < n; i++) { __syncthreads(); acc += i; } if (acc < 0) sink[0] = acc; }
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned* b; cudaMalloc(&b, 16); cudaMemset(b, 0, 16); float* sink; cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int N = 2000;
  for (int threads : {256, 768}) {
    int n = N; void* a1[] = {&b, &n, &sink}; void* a2[] = {&n, &sink};
    for (int rep = 0; rep < 2; rep++) {
      float t1, t2, t3, t4;
      cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_flip, nsm, threads, a1, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t4, e0, e1);
      cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_gen, nsm, threads, a1, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t1, e0, e1);
      cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_cg, nsm, threads, a2, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t2, e0, e1);
      cudaEventRecord(e0); cudaLaunchCooperativeKernel((void*)k_sync, nsm, threads, a2, 0, 0); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t3, e0, e1);
      printf("threads %d: generation barrier %.3f us, cg grid.sync %.3f us, flip+red %.3f us, __syncthreads %.3f us (per barrier, %d SMs) err=%s\n", threads, t1 * 1e3 / N, t2 * 1e3 / N, t4 * 1e3 / N, t3 * 1e3 / N, nsm, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
