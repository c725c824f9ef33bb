// Probe: cycles per tcgen05.mma.kind::tf32 (K = 8) as a function of N, for
// one CTA (M = 128) and a CTA pair (M = 256), issued back to back by one
// elected thread of a warp-uniform loop with the descriptors in uniform
// registers -- the issue-rate ceiling of narrow tiles (conv1's N = 96 / 48
// window GEMMs, the FC layers).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, bool mn) {
  // K-major SW128 (SBO 1024) or MN-major SW128_BASE32B (LBO = 32 rows x 128 B, SBO 512)
  if (mn)
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(4096 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
           (1ull << 46) | (1ull << 61);
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n, int m, bool mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((mn ? 1u : 0u) << 15) | ((mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int N, bool PAIR, bool MN = false>
__global__ void __launch_bounds__(128, 1) probe(int reps, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    if (PAIR)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_holder)));
    else
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_holder)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_holder;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 1 && rank == 0) {
    const uint64_t a = desc(smem_u32(smem), MN), b = desc(smem_u32(smem) + 32768, MN);
    const uint32_t id = idesc(N, PAIR ? 256 : 128, MN);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      asm volatile(
          "{\n\t.reg .pred p, e;\n\t.reg .b32 x;\n\t"
          "setp.ne.b32 p, %4, 0;\n\t"
          "elect.sync x|e, 0xffffffff;\n\t"
          "@e tcgen05.mma.cta_group::%5.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(a + (uint64_t)((r & 3) * 2)), "l"(b + (uint64_t)((r & 3) * 2)), "r"(id), "r"(r), "n"(PAIR ? 2 : 1)
          : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b32 x;\n\telect.sync x|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::%1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)),
        "n"(PAIR ? 2 : 1)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar))
        : "memory");
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int N, bool PAIR, bool MN = false>
void run() {
  long long* d;
  cudaMalloc(&d, 2 * sizeof(long long));
  cudaMemset(d, 0, 2 * sizeof(long long));
  auto k = probe<N, PAIR, MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const int reps = 4096;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(PAIR ? 2 : 1);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 65536 + 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int it = 0; it < 2; ++it) cudaLaunchKernelEx(&cfg, k, reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
  const double per = (double)c / reps;
  const double macs = 128.0 * N * 8;   // per SM per MMA
  printf("%s%s N=%3d : %7.1f cycles/MMA  (%6.0f MAC/clk/SM; TF32 dense peak ~1415) %s\n", PAIR ? "pair  " : "single", MN ? " MN-major" : " K-major ", N,
         per, macs / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<16, false>();
  run<32, false>();
  run<48, false>();
  run<64, false>();
  run<96, false>();
  run<128, false>();
  run<192, false>();
  run<256, false>();
  run<32, true>();
  run<48, true>();
  run<64, true>();
  run<96, true>();
  run<128, true>();
  run<192, true>();
  run<256, true>();
  run<16, false, true>();
  run<32, false, true>();
  run<48, false, true>();
  run<64, false, true>();
  run<96, false, true>();
  run<128, false, true>();
  run<256, false, true>();
  run<96, true, true>();
  run<256, true, true>();
  return 0;
}
