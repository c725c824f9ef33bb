// Probe: can a tcgen05 shared-memory descriptor start at an arbitrary 128-byte
// (or 64-byte) row offset inside a TMA-swizzled tile, and what must the
// descriptor's base-offset field (bits 49-51) hold then?  The conv1 "window"
// implicit GEMM reads all 9 filter taps of a tile from ONE staged input window
// by shifting the A (fprop) / B (wgrad, MN-major) descriptor by the tap's row
// offset dy*57 + dx, which is only possible if such shifts are legal.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/desc_probe tools/desc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    auto e_ = (x);                                                            \
    if (e_ != 0) {                                                            \
      printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__);             \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

struct Case {
  int mode;   // 0: K-major SW128 A shift; 1: K-major SW64 A shift; 2: MN-major SW128_BASE32B B shift (along K)
  int r;      // row shift
  int bo;     // base_offset value
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW1:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra D1;\n\tbra W1;\n\tD1:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout,
                                         uint32_t bo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) | ((uint64_t)(bo & 7) << 49) |
         ((uint64_t)layout << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__host__ __device__ constexpr uint32_t idesc(int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// smem layout (1024-aligned):
//   A128 : 256 rows x 128 B  (K-major SW128, 32 tf32 of K per row)      0
//   B128 : 32 rows x 128 B   (K-major SW128, N = 32)                  32768
//   A64  : 256 rows x 64 B   (K-major SW64, 16 tf32 of K per row)     36864
//   B64  : 32 rows x 64 B    (K-major SW64)                           53248
//   BMN  : 256 rows x 128 B  (MN-major SW128_BASE32B: row = K, 32 N)  55296
//   bars                                                             88064
__global__ void probe(const __grid_constant__ CUtensorMap mA128, const __grid_constant__ CUtensorMap mB128,
                      const __grid_constant__ CUtensorMap mA64, const __grid_constant__ CUtensorMap mB64,
                      const __grid_constant__ CUtensorMap mBMN, const Case* cases, int ncases, float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  const uint32_t s = smem_u32(sm);
  const uint32_t A128 = s, B128 = s + 32768, A64 = s + 36864, B64 = s + 53248, BMN = s + 55296;
  const uint32_t bar_tma = s + 88064, bar_mma = s + 88072;
  __shared__ uint32_t tmem_holder;
  const int t = threadIdx.x;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_tma));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_mma));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        smem_u32(&tmem_holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_holder;
  if (t == 0) {
    const uint32_t bytes = 32768 + 4096 + 16384 + 2048 + 32768;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_tma), "r"(bytes));
    auto ld = [&](const CUtensorMap* m, uint32_t dst, int c0, int c1) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              dst),
          "l"((uint64_t)m), "r"(bar_tma), "r"(c0), "r"(c1)
          : "memory");
    };
    ld(&mA128, A128, 0, 0);
    ld(&mB128, B128, 0, 0);
    ld(&mA64, A64, 0, 0);
    ld(&mB64, B64, 0, 0);
    ld(&mBMN, BMN, 0, 0);
  }
  mbar_wait(bar_tma, 0);
  for (int ci = 0; ci < ncases; ++ci) {
    const Case c = cases[ci];
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (c.mode == 0) {   // A rows r..r+127 of A128, K = 32 (4 MMAs), B = B128
        for (int kk = 0; kk < 4; ++kk)
          mma(tmem, desc(A128 + c.r * 128 + kk * 32, 16, 1024, 2, c.bo), desc(B128 + kk * 32, 16, 1024, 2, 0),
              idesc(32, false, false), kk > 0);
      } else if (c.mode == 1) {   // SW64: K = 16 (2 MMAs)
        for (int kk = 0; kk < 2; ++kk)
          mma(tmem, desc(A64 + c.r * 64 + kk * 32, 16, 512, 4, c.bo), desc(B64 + kk * 32, 16, 512, 4, 0),
              idesc(32, false, false), kk > 0);
      } else {   // A = A128 rows 0..127 (K-major), B = BMN rows r..r+31 (K), MN-major, N = 32
        for (int kk = 0; kk < 4; ++kk)
          mma(tmem, desc(A128 + kk * 32, 16, 1024, 2, 0),
              desc(BMN + (c.r + 8 * kk) * 128, 32 * 128, 512, 1, c.bo), idesc(32, false, true), kk > 0);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_mma));
    }
    mbar_wait(bar_mma, ci & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[32];
    const uint32_t ta = tmem + ((uint32_t)((t / 32) * 32) << 16);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[16 * h + 0]), "=r"(r[16 * h + 1]), "=r"(r[16 * h + 2]), "=r"(r[16 * h + 3]),
            "=r"(r[16 * h + 4]), "=r"(r[16 * h + 5]), "=r"(r[16 * h + 6]), "=r"(r[16 * h + 7]),
            "=r"(r[16 * h + 8]), "=r"(r[16 * h + 9]), "=r"(r[16 * h + 10]), "=r"(r[16 * h + 11]),
            "=r"(r[16 * h + 12]), "=r"(r[16 * h + 13]), "=r"(r[16 * h + 14]), "=r"(r[16 * h + 15])
          : "r"(ta + 16 * h));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) out[((size_t)ci * 128 + t) * 32 + j] = __uint_as_float(r[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
  }
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}
static CUtensorMap tmap(float* g, int inner, int outer, int ld, int box_in, int box_out, CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t str[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_in, (cuuint32_t)box_out};
  cuuint32_t es[2] = {1, 1};
  CK(enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  return m;
}

int main() {
  // values exactly representable in tf32 (small integers / 8) so products are exact
  std::vector<float> A(256 * 32), B(32 * 32), A64(256 * 16), B64(32 * 16), BMN(256 * 32);
  srand(1);
  auto rv = [] { return (float)((rand() % 17) - 8) / 8.0f; };
  for (auto& v : A) v = rv();
  for (auto& v : B) v = rv();
  for (auto& v : A64) v = rv();
  for (auto& v : B64) v = rv();
  for (auto& v : BMN) v = rv();
  float *dA, *dB, *dA64, *dB64, *dBMN, *dout;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dA64, A64.size() * 4));
  CK(cudaMalloc(&dB64, B64.size() * 4));
  CK(cudaMalloc(&dBMN, BMN.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dA64, A64.data(), A64.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB64, B64.data(), B64.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dBMN, BMN.data(), BMN.size() * 4, cudaMemcpyHostToDevice));
  CUtensorMap mA = tmap(dA, 32, 256, 32, 32, 256, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap mB = tmap(dB, 32, 32, 32, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap mA6 = tmap(dA64, 16, 256, 16, 16, 256, CU_TENSOR_MAP_SWIZZLE_64B);
  CUtensorMap mB6 = tmap(dB64, 16, 32, 16, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  CUtensorMap mBM = tmap(dBMN, 32, 256, 32, 32, 256, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  std::vector<Case> cases;
  const int shifts[] = {0, 1, 2, 3, 4, 5, 7, 8, 9, 57, 58, 59, 114, 115, 116};
  for (int mode = 0; mode < 3; ++mode)
    for (int r : shifts) {
      const int lim = mode == 2 ? 256 - 32 : 256 - 128;
      if (r > lim) continue;
      const int rb = mode == 1 ? 64 : 128;
      const int ph = mode == 1 ? ((r * rb) >> 7) & 7 : mode == 2 ? ((r * rb) >> 7) & 3 : r & 7;
      cases.push_back({mode, r, 0});
      if (ph) cases.push_back({mode, r, ph});
      if (mode == 2 && (r & 7)) cases.push_back({mode, r, r & 7});
    }
  Case* dc;
  CK(cudaMalloc(&dc, cases.size() * sizeof(Case)));
  CK(cudaMemcpy(dc, cases.data(), cases.size() * sizeof(Case), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dout, cases.size() * 128 * 32 * 4));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  probe<<<1, 128, 100 * 1024>>>(mA, mB, mA6, mB6, mBM, dc, (int)cases.size(), dout);
  CK(cudaDeviceSynchronize());
  std::vector<float> out(cases.size() * 128 * 32);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  for (size_t ci = 0; ci < cases.size(); ++ci) {
    const Case c = cases[ci];
    double maxerr = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < 32; ++j) {
        double ref = 0;
        if (c.mode == 0)
          for (int k = 0; k < 32; ++k) ref += (double)A[(c.r + i) * 32 + k] * B[j * 32 + k];
        else if (c.mode == 1)
          for (int k = 0; k < 16; ++k) ref += (double)A64[(c.r + i) * 16 + k] * B64[j * 16 + k];
        else
          for (int k = 0; k < 32; ++k) ref += (double)A[i * 32 + k] * BMN[(c.r + k) * 32 + j];
        maxerr = fmax(maxerr, fabs(out[(ci * 128 + i) * 32 + j] - ref));
      }
    printf("mode %d (%s) shift %3d base_offset %d : max err %g %s\n", c.mode,
           c.mode == 0 ? "K-major SW128 A" : c.mode == 1 ? "K-major SW64 A " : "MN-major B32  B", c.r, c.bo,
           maxerr, maxerr == 0 ? "OK" : "WRONG");
  }
  return 0;
}
