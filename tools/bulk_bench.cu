// Microbenchmark: cp.async.bulk (global -> shared, mbarrier completion) read
// throughput with one CTA per SM, vs plain 16-byte vector loads.  Each CTA
// streams `per_cta` bytes through a ring of NST stages of `chunk` bytes;
// `off` shifts every source address by off bytes (16-byte aligned, not 128).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(256, 1) k_bulk(const char* src, size_t per_cta, int chunk, int nst, int off, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned long long* bar = (unsigned long long*)sm;
  unsigned char* buf = sm + 128;
  const char* s0 = src + (size_t)blockIdx.x * per_cta + off;
  const int n = (int)(per_cta / chunk) - 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int i) {
    int s = i % nst;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(buf + (size_t)s * chunk)), "l"(s0 + (size_t)i * chunk), "r"(chunk), "r"(su(&bar[s])) : "memory");
  };
  if (threadIdx.x == 0) for (int i = 0; i < nst && i < n; i++) issue(i);
  float acc = 0;
  for (int i = 0; i < n; i++) {
    int s = i % nst; unsigned par = (i / nst) & 1;
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su(&bar[s])), "r"(par) : "memory");
    acc += ((float*)(buf + (size_t)s * chunk))[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && i + nst < n) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(i + nst); }
  }
  if (acc == 12345.f) sink[0] = acc;
}
__global__ void __launch_bounds__(256) k_ldg(const float4* src, size_t n4, float* sink) {
  float acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) { float4 v = src[i]; acc += v.x + v.y + v.z + v.w; }
  if (acc == 12345.f) sink[0] = acc;
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  size_t per_cta = 1 << 20; size_t tot = per_cta * nsm + 4096;
  char* src; cudaMalloc(&src, tot + (1 << 20)); cudaMemset(src, 1, tot + (1 << 20));
  float* sink; cudaMalloc(&sink, 4);
  char* flush; cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int chunk : {4096, 16384, 32768}) for (int nst : {2, 4, 6}) for (int off : {0, 16}) {
    size_t smem = 128 + (size_t)chunk * nst; if (smem > 220 * 1024) continue;
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
      cudaMemset(flush, r, 256 << 20);
      cudaEventRecord(e0); k_bulk<<<nsm, 256, smem>>>(src, per_cta, chunk, nst, off, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("bulk chunk %6d nst %d off %2d: %.0f GB/s  (%s)\n", chunk, nst, off, (double)(per_cta - chunk) * nsm / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  float best = 1e9;
  for (int r = 0; r < 5; r++) {
    cudaMemset(flush, r, 256 << 20);
    cudaEventRecord(e0); k_ldg<<<nsm * 8, 256>>>((const float4*)src, per_cta * nsm / 16, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("ldg.128 read: %.0f GB/s\n", (double)per_cta * nsm / (best * 1e-3) / 1e9);
  return 0;
}
