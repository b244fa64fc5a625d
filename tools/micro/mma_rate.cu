// Microbenchmark: tcgen05.mma issue rate for small N (swap-AB GEMV shapes), A from smem vs
// TMEM, one accumulator vs alternating accumulators.  One CTA, one elected thread issues
// `iters` MMAs then commits; cycles measured with clock64 around issue+wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n) { return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24); }
template <int N, int MODE>  // MODE 0: SS one acc, 1: SS two accs alternating, 2: TS one acc, 3: TS 4 accs, 4: SS + commit per 8
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint64_t da = desc(su32(sm)), db = desc(su32(sm + 16384));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t d = tm + ((MODE == 1) ? (i & 1) * N : (MODE == 3 ? (i & 3) * N : 0));
      uint32_t acc = i >= 4;
      if (MODE == 4 && (i & 7) == 7)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)));
      if (MODE <= 1 || MODE == 4)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da + 2 * (i & 3)), "l"(db + 2 * (i & 3)), "r"(idesc(N)), "r"(acc));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(tm + 64 + 8 * (i & 7)), "l"(db + 2 * (i & 3)), "r"(idesc(N)), "r"(acc));
    }
    long long t1 = clock64();
    if (MODE == 4) t1 = 0;
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)));
    long long t2 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}

// two issuer threads (warp 0 and warp 1, lane 0) in ONE CTA, TS mode, separate accumulators
__global__ void k2iss(long long* out, int iters) {
  __shared__ __align__(1024) unsigned char sm[16384];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = slot;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < 2) {
    const uint64_t db = desc(su32(sm));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + w * 16), "r"(tm + 64 + 8 * (i & 7)), "l"(db + 2 * (i & 3)), "r"(idesc(16)), "r"((uint32_t)(i >= 4)));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[w])));
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar[w])));
    out[w] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}

// TS MMAs from warp 0 while warps 2..9 stream tcgen05.st into other TMEM columns (A-slot refills)
__global__ void kcont(long long* out, int iters, int st_on) {
  __shared__ __align__(1024) unsigned char sm[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int stop;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
  }
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = slot;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    if (lane == 0) {
      const uint64_t db = desc(su32(sm));
      long long t0 = clock64();
      for (int i = 0; i < iters; ++i)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm), "r"(tm + 64 + 8 * (i & 7)), "l"(db + 2 * (i & 3)), "r"(idesc(16)), "r"((uint32_t)(i >= 4)));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      uint32_t ok = 0;
      while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)));
      out[0] = clock64() - t0;
      stop = 1;
    }
  } else if (w >= 2 && st_on) {
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i * lane;
    const uint32_t base = tm + ((uint32_t)((w & 3) * 32) << 16) + 128 + ((w - 2) >> 2) * 32;
    long long n = 0;
    while (!stop) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(base + (uint32_t)(n & 3) * 64u),
        "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),"r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      ++n;
    }
    if (lane == 0) out[w] = n;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}
template <int N, int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  for (int iters : {64, 256, 1024}) {
    k<N, MODE><<<1, 128, 65536 + 1024>>>(d, iters);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-10s N=%3d iters=%5d issue %7lld cyc  done %7lld cyc  -> %.1f cyc/mma  (%s)\n", name, N, iters, h[0], h[1],
           (double)h[1] / iters, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(d);
}
template <int N, int MODE>
void run_grid(const char* name, int grid) {
  long long* d;
  cudaMalloc(&d, 16 * grid);
  cudaFuncSetAttribute(k<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  k<N, MODE><<<grid, 128, 65536 + 1024>>>(d, 1024);
  long long* h = new long long[2 * grid];
  cudaMemcpy(h, d, 16 * grid, cudaMemcpyDeviceToHost);
  double mx = 0, mn = 1e18;
  for (int i = 0; i < grid; ++i) { mx = h[2 * i + 1] > mx ? h[2 * i + 1] : mx; mn = h[2 * i + 1] < mn ? h[2 * i + 1] : mn; }
  printf("%-10s N=%3d grid=%4d per-CTA cyc/mma min %.1f max %.1f (%s)\n", name, N, grid, mn / 1024, mx / 1024, cudaGetErrorString(cudaGetLastError()));
  delete[] h;
  cudaFree(d);
}
int main() {
  {
    long long* d;
    cudaMalloc(&d, 16 * 8);
    for (int on = 0; on < 2; ++on) {
      cudaMemset(d, 0, 16 * 8);
      kcont<<<1, 320>>>(d, 4096, on);
      long long h[10];
      cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
      long long st = 0;
      for (int w = 2; w < 10; ++w) st += h[w];
      printf("TS MMA with%s concurrent tcgen05.st: %.1f cyc/MMA; %lld STTM.x32 (4 KB each) meanwhile -> %.1f B/cyc (%s)\n",
             on ? "" : "out", h[0] / 4096.0, st, st * 4096.0 / h[0], cudaGetErrorString(cudaGetLastError()));
    }
  }
  {
    long long* d;
    cudaMalloc(&d, 16);
    for (int rep = 0; rep < 2; ++rep) {
      k2iss<<<1, 64>>>(d, 1024);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("TS two issuers in one CTA: %.1f / %.1f cyc per MMA per issuer (%s)\n", h[0] / 1024.0, h[1] / 1024.0,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  run<16, 0>("SS 1acc");
  run<16, 4>("SS commit8");
  run_grid<16, 0>("SS 1acc", 148);
  run_grid<16, 0>("SS 1acc", 296);
  run_grid<16, 0>("SS 1acc", 444);
  run_grid<16, 2>("TS 1acc", 296);
  return 0;
}
