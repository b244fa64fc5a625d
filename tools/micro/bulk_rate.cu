// Microbenchmark: HBM streaming rate of cp.async.bulk (1-D bulk copies, mbarrier complete_tx)
// issued by ONE thread per CTA into a ring of STAGES x CHUNK bytes, vs grid size (CTAs per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const unsigned char* src, long long per_cta, int chunk, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned char* s = src + (long long)blockIdx.x * per_cta;
  const int n = (int)(per_cta / chunk);
  unsigned long long acc = 0;
  for (int i = 0; i < n + stages; ++i) {
    if (i >= stages) {  // consume chunk i - stages
      const int st = (i - stages) % stages;
      const uint32_t par = ((i - stages) / stages) & 1;
      uint32_t ok = 0;
      while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar[st])), "r"(par));
      acc += sm[st * chunk + (i & 63)];
    }
    if (i < n) {
      const int st = i % stages;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[st])), "r"(chunk));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + st * chunk)), "l"(s + (long long)i * chunk), "r"(chunk), "r"(su32(&bar[st])));
    }
  }
  sink[blockIdx.x] = acc;
}
int main() {
  const long long total = 1ll << 30;
  unsigned char* src;
  unsigned long long* sink;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  cudaMalloc(&sink, 8 * 4096);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct C { int chunk, stages, grid; };
  C cs[] = {{4096, 16, 148}, {8192, 10, 148}, {8192, 10, 296}, {8192, 6, 296}, {16384, 6, 148}, {16384, 6, 296},
            {16384, 12, 148}, {32768, 6, 148}, {8192, 20, 148}, {4096, 20, 296}, {8192, 10, 200}, {8192, 12, 444}};
  for (auto c : cs) {
    const long long per = (total / c.grid) / c.chunk * c.chunk;
    const int smem = c.chunk * c.stages;
    for (int r = 0; r < 2; ++r) k<<<c.grid, 32, smem>>>(src, per, c.chunk, c.stages, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k<<<c.grid, 32, smem>>>(src, per, c.chunk, c.stages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double gbs = 5.0 * per * c.grid / (ms * 1e-3) / 1e9;
    printf("chunk %6d stages %3d grid %4d (in flight/CTA %4d KB): %7.0f GB/s total, %5.1f GB/s per CTA (%s)\n", c.chunk,
           c.stages, c.grid, smem / 1024, gbs, gbs / c.grid, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
