// Window implicit GEMM for the space-to-depth first layer (CaffeNet conv1:
// 11x11 / stride 4 over 3 channels -> a 3x3 stride-1 conv over the
// 48-channel space-to-depth image, lower.cu) -- the layer the generic im2col
// path runs worst: its 128-pixel tiles re-read every input pixel once per
// filter tap (9 im2col boxes per channel block) and pad the 48 channels to 64.
//
// Padded-width indexing: with the s2d image flattened to rows
// q = (img * n2 + h) * n2 + w (pixel pitch cp = 48 floats), output pixel
// (img, h, w) of a stride-1 k2 x k2 conv without padding reads, for filter tap
// (kx, ky), exactly row q + kx * n2 + ky.  So a tile of 128 consecutive q
// needs ONE contiguous window of 128 + (k2-1)(n2+1) rows (244 for conv1), and
// each tap's A operand is that window shifted by a whole number of rows: the
// tcgen05 descriptor simply starts kx*n2+ky rows in (tools/desc_probe.cu: a
// descriptor may start at any 128 B / 64 B row of a TMA-swizzled tile).  Rows
// q with h >= m or w >= m are junk (6.9% for conv1) and never stored.
//
//  * fprop  (C[q, o] = sum_{tap, ch} X[q + off(tap), ch] W[o, tap, ch]):
//    CTA pairs (cta_group::2, M = 256 pixels, N = d_out); each CTA keeps its
//    half of ALL the weights resident in shared memory for the whole launch
//    and streams one 244-row window per tile: channels 0-31 as a 128-byte
//    swizzled box, 32-47 as a 64-byte swizzled box (K = 432, not 576).
//    A tile costs 244 rows x 192 B of L2->SM traffic instead of 9 x 128 rows
//    x 256 B plus the weights.
//  * wgrad  (dW[o, kx, ky, ch] = sum_pix dZ[pix, o] X[q(pix) + kx*n2 + ky, ch]):
//    M = (kx, ky*48 + ch) -- for a fixed kx the three ky taps' channels are
//    one contiguous 144-float run of the image -- in 32-channel MN-major
//    atoms, N = d_out, K = pixels, one output row per stage; the s2d rows stay
//    resident in a ring across the three output rows that read them (see the
//    wgrad section below).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace cwin {
using namespace gemm;

constexpr int CP = 48;        // space-to-depth channels (4 x 4 x 3)
constexpr int C0 = 32;        // channels in the 128-byte swizzled box
constexpr int C1 = CP - C0;   // channels in the 64-byte swizzled box
constexpr int K2 = 3;         // taps per dimension of the space-to-depth conv (11/4 -> 3)
constexpr int MAX_TAPS = K2 * K2;
constexpr int WIN_MAX = 256;  // TMA box rows

PFN_cuTensorMapEncodeTiled_v12000 encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

int tmap(CUtensorMap* m, const float* p, int rank, const cuuint64_t* dims, const cuuint64_t* strides_b,
         const cuuint32_t* box, CUtensorMapSwizzle sw) {
  auto fn = encode();
  if (!fn) {
    omni::set_error("cuTensorMapEncodeTiled unavailable");
    return OMNI_ECUDA;
  }
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(p), dims, strides_b, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    omni::set_error("conv window: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return OMNI_ECUDA;
  }
  return OMNI_OK;
}

// ------------------------------------------------------------- fprop ----
struct FParams {
  int b, n2, m, k2, n2sq;
  long long rows;     // b * n2 * n2
  int units;          // pair tiles of 256 padded pixels
  int win_rows;       // 128 + (k2 - 1) * (n2 + 1)
  int epilogue;
  const float* bias;
  float* Y;
  long long ldy;
  int debug;          // OMNI_WINDOW_DEBUG (timing probes only): 1 no stores, 2 no window
                      // reloads after the first STAGES tiles, 4 no MMAs
};

template <int BN>
struct FLayout {
  static constexpr int BNL = BN / 2;                 // weight rows (output channels) per CTA
  static constexpr int B0_TAP = BNL * 128;           // one tap: BNL rows x 32 K, SW128
  static constexpr int B1_TAP = BNL * 64;            // one tap: BNL rows x 16 K, SW64
  static constexpr int B1_OFF = MAX_TAPS * B0_TAP;
  static constexpr int B_ALLOC = (MAX_TAPS * (B0_TAP + B1_TAP) + 1023) / 1024 * 1024;
  static constexpr int A0 = WIN_MAX * 128;           // window, channels 0-31
  static constexpr int A1 = WIN_MAX * 64;            // window, channels 32-47
  static constexpr int STAGE = A0 + A1;
  static constexpr int STAGES = 2;
  static constexpr int STAGE_OFF = B_ALLOC;
  static constexpr int BAR_OFF = STAGE_OFF + STAGES * STAGE;
  static constexpr int BIAS_OFF = BAR_OFF + 256;    // BN floats
  // epilogue: EPI sets of 4 warps, set e drains accumulator columns
  // [e*CS, (e+1)*CS) of the 128 TMEM lanes (tiles are short: one set of four
  // warps cannot drain 96 columns as fast as the MMA warp fills them)
  static constexpr int EPI = 2;
  static constexpr int CS = BN / EPI;
  static constexpr int THREADS = 128 + 128 * EPI;
  static constexpr int STG_PITCH = 20;               // floats per staged row (16 + 4: conflict-free)
  static constexpr int STG_OFF = BIAS_OFF + 512;     // 4*EPI warps x 32 rows x STG_PITCH floats
  static constexpr int BYTES = STG_OFF + 4 * EPI * 32 * STG_PITCH * 4 + 1024;
  // a ring of NACC accumulators: tiles are short (54 MMAs), so the MMA warp
  // runs up to NACC - 1 tiles ahead of the epilogue and the cross-CTA
  // handoffs (commit -> epilogue -> release) overlap instead of pacing tiles
  static constexpr int NACC = 4;
  static constexpr int ACC_STRIDE = BN <= 32 ? 32 : (BN <= 64 ? 64 : 128);
  static constexpr int TMEM_COLS = NACC * ACC_STRIDE <= 128 ? 128 : (NACC * ACC_STRIDE <= 256 ? 256 : 512);
  static_assert(BYTES <= 232448, "fprop window layout exceeds shared memory");
  static_assert(B0_TAP % 1024 == 0 && B1_TAP % 512 == 0 && B1_OFF % 1024 == 0, "swizzle alignment");
};

template <int MODE>
__device__ __forceinline__ float fepi(float acc, const float* bias, int col) {
  if (MODE == OMNI_EPI_BIAS) return acc + bias[col];
  if (MODE == OMNI_EPI_BIAS_RELU) return fmaxf(acc + bias[col], 0.f);
  if (MODE == OMNI_EPI_RELU) return fmaxf(acc, 0.f);
  return acc;
}

// Apply the epilogue to one lane's 16 accumulator columns (bias: the 16
// matching values, in registers) and stage them as that lane's row of the
// warp's 32 x 16 staging tile (pitch 20 floats).
template <int MODE>
__device__ __forceinline__ void fstage16(float* srow, const uint32_t (&r)[16], const float* b16) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float4 v;
    v.x = fepi<MODE>(__uint_as_float(r[4 * j]), b16, 4 * j);
    v.y = fepi<MODE>(__uint_as_float(r[4 * j + 1]), b16, 4 * j + 1);
    v.z = fepi<MODE>(__uint_as_float(r[4 * j + 2]), b16, 4 * j + 2);
    v.w = fepi<MODE>(__uint_as_float(r[4 * j + 3]), b16, 4 * j + 3);
    *reinterpret_cast<float4*>(srow + 4 * j) = v;
  }
}

template <int BN>
__global__ void __launch_bounds__(FLayout<BN>::THREADS, 1)
    conv_window_fprop_kernel(const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmX1,
                             const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
                             const FParams p) {
  using L = FLayout<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + L::BAR_OFF;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 16u + 8u * s; };
  auto tfull_bar = [&](int a) { return bar0 + 32u + 8u * a; };    // a < NACC <= 4
  auto tempty_bar = [&](int a) { return bar0 + 64u + 8u * a; };
  const uint32_t bfull = bar0 + 96u;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::BAR_OFF + 104);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const int unit0 = (int)(blockIdx.x >> 1), units = (int)(gridDim.x >> 1);
  constexpr int taps = MAX_TAPS;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX0);
    tma_prefetch_desc(&tmX1);
    tma_prefetch_desc(&tmW0);
    tma_prefetch_desc(&tmW1);
    for (int s = 0; s < L::STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < L::NACC; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), 8 * L::EPI);  // 4 * EPI epilogue warps x 2 CTAs
    }
    mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "n"(L::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ---- producer: this CTA's half of every tap's weights, once --------
      const uint32_t bfb = mapa_rank0(bfull);
      if (rank == 0) mbar_expect_tx(bfull, (uint32_t)(2 * taps * (L::B0_TAP + L::B1_TAP)));
      for (int t = 0; t < taps; ++t) {
        tma_load_2d_pair(&tmW0, sbase + t * L::B0_TAP, bfb, t * CP, rank * L::BNL);
        tma_load_2d_pair(&tmW1, sbase + L::B1_OFF + t * L::B1_TAP, bfb, t * CP + C0, rank * L::BNL);
      }
      // ---- then one input window per tile --------------------------------
      const uint32_t win_bytes = (uint32_t)p.win_rows * (C0 + C1) * 4u;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int w = unit0; w < p.units; w += units, ++it) {
        mbar_wait(empty_bar(stage), phase ^ 1);
        if ((p.debug & 2) && it >= L::STAGES) {    // probe: reuse the staged window
          if (rank == 0) mbar_arrive(full_bar(stage));
          if (++stage == L::STAGES) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        if (rank == 0) mbar_expect_tx(full_bar(stage), 2u * win_bytes);
        const uint32_t fb = mapa_rank0(full_bar(stage));
        const int q0 = w * 256 + rank * 128;
        const uint32_t dst = sbase + L::STAGE_OFF + stage * L::STAGE;
        tma_load_2d_pair(&tmX0, dst, fb, 0, q0);
        tma_load_2d_pair(&tmX1, dst + L::A0, fb, C0, q0);
        if (++stage == L::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---- MMA issuer (whole warp, one elected thread issues): 9 taps x
      // (4 + 2) MMAs of K = 8 per tile; descriptors advance by adding the
      // byte offset >> 4 to the start-address field
      const uint32_t idesc = instr_desc_rt(BN, false, false, 256);
      const uint64_t b0d = make_desc(sbase, 16, 1024, 2);
      const uint64_t b1d = make_desc(sbase + L::B1_OFF, 16, 512, 4);
      mbar_wait_acq_cluster(bfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int w = unit0; w < p.units; w += units) {
        mbar_wait_acq_cluster(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        mbar_wait(full_bar(stage), phase);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * L::ACC_STRIDE);
        const uint32_t a0 = sbase + L::STAGE_OFF + stage * L::STAGE;
        const uint64_t a0d = make_desc(a0, 16, 1024, 2);
        const uint64_t a1d = make_desc(a0 + L::A0, 16, 512, 4);
#pragma unroll
        for (int t = 0; t < taps; ++t) {
          const uint32_t off = (uint32_t)((t / K2) * p.n2 + t % K2);   // t is a compile-time constant
          const uint64_t at0 = a0d + (uint64_t)(off * 8u), at1 = a1d + (uint64_t)(off * 4u);
          const uint64_t bt0 = b0d + (uint64_t)(t * (L::B0_TAP >> 4)), bt1 = b1d + (uint64_t)(t * (L::B1_TAP >> 4));
#pragma unroll
          for (int kk = 0; kk < C0 / 8; ++kk)
            tc_mma_tf32_pair_elect(d_tmem, at0 + 2u * kk, bt0 + 2u * kk, idesc, (t > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < C1 / 8; ++kk)
            tc_mma_tf32_pair_elect(d_tmem, at1 + 2u * kk, bt1 + 2u * kk, idesc, 1u);
        }
        tc_commit_pair_elect(empty_bar(stage));
        tc_commit_pair_elect(tfull_bar(acc));
        if (++stage == L::STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (++acc == L::NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> bias / ReLU -> NHWC rows (junk rows skipped) --
    const int ew = warp & 3;                 // TMEM lane quarter (rows ew*32 ..)
    const int es = (warp - 4) >> 2;          // column set
    // this set's bias values live in registers for the whole launch (a
    // shared-memory operand per element made the epilogue instruction-bound)
    float breg[L::CS];
#pragma unroll
    for (int j = 0; j < L::CS; ++j) breg[j] = p.bias ? __ldg(p.bias + es * L::CS + j) : 0.f;
    float* stg = reinterpret_cast<float*>(smem + L::STG_OFF) + (warp - 4) * 32 * L::STG_PITCH;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int w = unit0; w < p.units; w += units) {
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const long long q = (long long)w * 256 + rank * 128 + ew * 32 + lane;
      const int img = (int)(q / p.n2sq);
      const int r = (int)(q - (long long)img * p.n2sq);
      const int h = r / p.n2, x = r - (r / p.n2) * p.n2;
      const int valid = (img < p.b && h < p.m && x < p.m) ? 1 : 0;
      const int prow = valid ? (img * p.m + h) * p.m + x : 0;   // output pixel of this lane's row
      const uint32_t t_row = tmem_base + (uint32_t)(acc * L::ACC_STRIDE + es * L::CS) + ((uint32_t)(ew * 32) << 16);
      // this set's accumulator columns in one batch of TMEM loads, then the
      // accumulator goes straight back to the MMA warp
      uint32_t racc[L::CS / 16][16];
#pragma unroll
      for (int j = 0; j < L::CS / 16; ++j) tmem_ld16(t_row + (uint32_t)(16 * j), racc[j]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(mapa_rank0(tempty_bar(acc)));
      float* srow = stg + lane * L::STG_PITCH;
      const float* yb = p.Y + es * L::CS;
#pragma unroll
      for (int j = 0; j < L::CS / 16; ++j) {
        switch (p.epilogue) {
          case OMNI_EPI_BIAS: fstage16<OMNI_EPI_BIAS>(srow, racc[j], breg + 16 * j); break;
          case OMNI_EPI_BIAS_RELU: fstage16<OMNI_EPI_BIAS_RELU>(srow, racc[j], breg + 16 * j); break;
          case OMNI_EPI_RELU: fstage16<OMNI_EPI_RELU>(srow, racc[j], breg + 16 * j); break;
          default: fstage16<OMNI_EPI_STORE>(srow, racc[j], breg + 16 * j); break;
        }
        __syncwarp();
        // coalesced store: each instruction writes 8 whole 64-byte row segments
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int row = it * 8 + (lane >> 2), c4 = lane & 3;
          const int ok = __shfl_sync(0xffffffffu, valid, row);
          const int pr = __shfl_sync(0xffffffffu, prow, row);
          const float4 v = *reinterpret_cast<const float4*>(stg + row * L::STG_PITCH + 4 * c4);
          if (ok && !(p.debug & 1))
            *reinterpret_cast<float4*>(const_cast<float*>(yb) + (long long)pr * p.ldy + 16 * j + 4 * c4) = v;
        }
        __syncwarp();
      }
      if (++acc == L::NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(L::TMEM_COLS)
                 : "memory");
  }
}

// ------------------------------------------------------------- wgrad ----
// dW[o, kx, J] = sum_pix dZ[pix, o] X[q(pix) + kx*n2, J], J = ky*48 + ch in
// [0, 144): for a fixed kx the three ky taps' channels are ONE contiguous run
// of 144 floats of the flattened s2d image (pixel pitch 48), so with the image
// viewed as overlapping 160-float rows at a 192-byte pitch, M = (kx, J) is
// 3 x 4.5 MN-major 32-channel atoms -- no 48 -> 64 channel padding:
//   tiles 0-2 (M = 128): kx = t, J in [0, 128)   (atoms a0-a3 of s2d row h+t)
//   tile  3   (M = 128): J in [128, 160) of kx = 0, 1, 2 (16 real rows each)
//                        + a resident all-ones atom: rows 96-127 = the bias
//                        gradient (dZ column sums) at no extra MMA
// N = d_out, K = pixels: one output row (img, h) per stage, m = 55 pixels
// padded to 56 by the dZ box's zero fill.  The s2d rows' atoms a0-a3 sit in a
// 4-slot ring: output row h+1 reuses rows h+1 and h+2 of row h and loads only
// row h+3 (the A traffic of the 128-pixel im2col tiles drops 3x); the a4 atoms
// of the three rows and the dZ row are per-stage loads.  Each CTA reduces a
// contiguous range of output rows into TMEM (4 x d_out columns); a fixed-order
// reduction sums the per-CTA partials.
constexpr int W_TMEM_COLS = 512;
constexpr int W_RING = 4;            // s2d-row slots (rows h .. h+2 in use + 1 loading)
constexpr int W_STAGES = 2;          // per-output-row stages (a4 atoms + dZ)
constexpr int W_KB = 56;             // K rows per stage: one output row, 55 -> 56
constexpr uint32_t W_ATOM = W_KB * 128;   // 7168 B: one 32-float x 56-row MN-major atom
constexpr int W_COLS = 436;          // workspace row: 432 (kx, J) columns + bias + 3 pad
struct WParams {
  int n2, m;
  int units;        // output rows b * m
  int d_out;        // N (32, 64 or 96)
  uint32_t ring_off, stage_off, bar_off;
  float* ws;        // [gridDim.x][d_out][W_COLS] partial sums
};

__global__ void __launch_bounds__(256, 1)
    conv_window_wgrad_kernel(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmX,
                             const WParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + p.bar_off;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 32u + 8u * s; };
  const uint32_t acc_full = bar0 + 64u;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + p.bar_off + 80);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ring = sbase + p.ring_off;
  const uint32_t stg0 = sbase + p.stage_off;
  constexpr uint32_t STAGE_BYTES = 7 * W_ATOM;   // a4 x 3, ones, dZ x 3
  const int natoms_z = p.d_out / 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmG);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "n"(W_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  {  // each stage's all-ones atom (tile 3's rows 96-127; every element 1.0, so
     // its swizzle is irrelevant; TMA never writes it)
    for (int s = 0; s < W_STAGES; ++s) {
      float4* ones = reinterpret_cast<float4*>(smem + p.stage_off + s * STAGE_BYTES + 3 * W_ATOM);
      for (int i = threadIdx.x; i < (int)(W_ATOM / 16); i += blockDim.x) ones[i] = make_float4(1.f, 1.f, 1.f, 1.f);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // this CTA's contiguous range of output rows
  const int u0 = (int)(((long long)blockIdx.x * p.units) / gridDim.x);
  const int u1 = (int)(((long long)(blockIdx.x + 1) * p.units) / gridDim.x);

  if (warp == 0) {
    if (lane == 0) {
      int loads = 0;     // s2d rows loaded so far (ring slot = loads % W_RING)
      for (int u = u0; u < u1; ++u) {
        const int i = u - u0, stage = i % W_STAGES;
        const int img = u / p.m, h = u - (u / p.m) * p.m;
        const bool fresh = (i == 0) || (h == 0);
        mbar_wait(empty_bar(stage), ((i / W_STAGES) & 1) ^ 1);
        if (fresh && i > 0)   // a new image: its 3 rows overwrite slots the previous row still reads
          mbar_wait(empty_bar((i - 1) % W_STAGES), ((i - 1) / W_STAGES) & 1);
        const int nnew = fresh ? 3 : 1;
        mbar_expect_tx(full_bar(stage), (uint32_t)(nnew * 4 + 3 + natoms_z) * W_ATOM);
        const int rbase = img * p.n2;
        for (int j = 0; j < nnew; ++j) {
          const int r = fresh ? h + j : h + 2;
          const uint32_t slot = ring + (uint32_t)(loads % W_RING) * 4u * W_ATOM;
          ++loads;
          for (int a = 0; a < 4; ++a)
            tma_load_2d(&tmX, slot + a * W_ATOM, full_bar(stage), 32 * a, (rbase + r) * p.n2);
        }
        const uint32_t stg = stg0 + stage * STAGE_BYTES;
        for (int kx = 0; kx < 3; ++kx)
          tma_load_2d(&tmX, stg + kx * W_ATOM, full_bar(stage), 128, (rbase + h + kx) * p.n2);
        for (int j = 0; j < natoms_z; ++j)
          tma_load_3d(&tmG, stg + (4 + j) * W_ATOM, full_bar(stage), 32 * j, 0, u);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (whole warp, one elected thread issues) --------------
    const uint32_t idm = instr_desc_rt(p.d_out, true, true, 128);
    int loads = 0, sl0 = 0, sl1 = 0, sl2 = 0;   // ring slots of rows h, h+1, h+2
    for (int u = u0; u < u1; ++u) {
      const int i = u - u0, stage = i % W_STAGES;
      const int h = u - (u / p.m) * p.m;
      if (i == 0 || h == 0) {
        sl0 = loads % W_RING;
        sl1 = (loads + 1) % W_RING;
        sl2 = (loads + 2) % W_RING;
        loads += 3;
      } else {
        sl0 = sl1;
        sl1 = sl2;
        sl2 = loads % W_RING;
        loads += 1;
      }
      mbar_wait(full_bar(stage), (i / W_STAGES) & 1);
      tc_fence_after();
      const uint32_t stg = stg0 + stage * STAGE_BYTES;
      const uint32_t ra[3] = {ring + (uint32_t)sl0 * 4u * W_ATOM, ring + (uint32_t)sl1 * 4u * W_ATOM,
                              ring + (uint32_t)sl2 * 4u * W_ATOM};
#pragma unroll 1
      for (int kk = 0; kk < W_KB / 8; ++kk) {
        const uint32_t accf = (i > 0 || kk > 0) ? 1u : 0u;
        const uint32_t ko = (uint32_t)kk * 1024u;   // 8 K rows x 128 B
        const uint64_t bz = make_desc(stg + 4 * W_ATOM + ko, W_ATOM, 512, 1);
#pragma unroll
        for (int t = 0; t < 3; ++t)
          tc_mma_tf32_elect(tmem_base + (uint32_t)(t * p.d_out), make_desc(ra[t] + ko, W_ATOM, 512, 1), bz,
                            idm, accf);
        tc_mma_tf32_elect(tmem_base + (uint32_t)(3 * p.d_out), make_desc(stg + ko, W_ATOM, 512, 1), bz, idm,
                          accf);
      }
      tc_commit_elect(empty_bar(stage));
    }
    tc_commit_elect(acc_full);
  } else if (warp >= 4) {
    // ---- epilogue: the CTA's partial dW (d_out x W_COLS) -> workspace ----
    const int ew = warp - 4;
    const int L = ew * 32 + lane;            // TMEM lane = M row of every tile
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16);
    float* dst = p.ws + (long long)blockIdx.x * p.d_out * W_COLS;
#pragma unroll 1
    for (int t = 0; t < 4; ++t) {
      // tiles 0-2: (kx = t, J = L); tile 3: (kx = L / 32, J = 128 + L % 32), J < 144 real
      const int col = t < 3 ? t * 144 + L : (L >> 5) * 144 + 128 + (L & 31);
      const bool ok = t < 3 || ((L >> 5) < 3 && (L & 31) < 16);
#pragma unroll 1
      for (int o0 = 0; o0 < p.d_out; o0 += 16) {
        uint32_t rr[16];
        tmem_ld16(t_row + (uint32_t)(t * p.d_out + o0), rr);
        tmem_wait_ld();
        if (ok) {
#pragma unroll
          for (int j = 0; j < 16; ++j) dst[(long long)(o0 + j) * W_COLS + col] = __uint_as_float(rr[j]);
        } else if (t == 3 && L == 96) {   // an all-ones row: the bias gradient, + 3 pad columns
#pragma unroll
          for (int j = 0; j < 16; ++j)
            *reinterpret_cast<float4*>(dst + (long long)(o0 + j) * W_COLS + 432) =
                make_float4(__uint_as_float(rr[j]), 0.f, 0.f, 0.f);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(W_TMEM_COLS)
                 : "memory");
  }
}

// Y[o * ldy + c] = sum_s ws[s][o][c] in a fixed order (deterministic): 8 lanes
// per float4 output, lane j summing splits j, j+8, j+16, ... in ascending
// order (4 loads in flight), then a fixed xor-shuffle tree over the 8 sums.
// (One thread per output, 148 dependent loads each, took 30 us.)
__global__ void __launch_bounds__(256) window_reduce_kernel(const float* __restrict__ ws, int S, int d_out,
                                                            int ncols, float* __restrict__ Y, long long ldy) {
  const int n4 = ncols / 4;
  const int total = d_out * n4;
  const long long split = (long long)d_out * ncols;
  const int lane = threadIdx.x & 31, j = lane & 7;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int w = warp; w * 4 < total; w += nwarps) {   // warp-uniform: 4 outputs per warp
    const int i = w * 4 + (lane >> 3);
    const bool valid = i < total;
    const int ii = valid ? i : total - 1;
    const int o = ii / n4, c = (ii - o * n4) * 4;
    const float* src = ws + (long long)o * ncols + c;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int s = j;
    for (; s + 24 < S; s += 32) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(src + (s + 8 * u) * split));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
    for (; s < S; s += 8) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(src + s * split));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
#pragma unroll
    for (int m = 4; m >= 1; m >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, m);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, m);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, m);
      acc.w += __shfl_xor_sync(0xffffffffu, acc.w, m);
    }
    if (valid && j == 0) *reinterpret_cast<float4*>(Y + o * ldy + c) = acc;
  }
}

// ------------------------------------------------------------- host -----
struct Geo {
  int m, taps, win_f;
};

int geometry(int b, int n2, int cp, int k2, int d_out, Geo* g) {
  OMNI_REQUIRE(b >= 1 && n2 >= 1 && k2 >= 1 && d_out >= 1, "conv window: bad shape");
  OMNI_REQUIRE(cp == CP, "conv window: needs %d space-to-depth channels (got %d)", CP, cp);
  OMNI_REQUIRE(k2 == K2 && k2 <= n2, "conv window: k2 = %d unsupported (the kernels are built for %d)", k2, K2);
  g->m = n2 - k2 + 1;
  g->taps = k2 * k2;
  g->win_f = 128 + (k2 - 1) * (n2 + 1);
  OMNI_REQUIRE(g->win_f <= WIN_MAX,
               "conv window: image too wide for one window (n2 = %d)", n2);
  OMNI_REQUIRE((long long)b * n2 * n2 < (1LL << 31), "conv window: too many pixels");
  return OMNI_OK;
}

int wgrad_splits(int nblk) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = omni::sm_count_cached(dev);
  return nblk < sms ? nblk : sms;
}

template <int BN>
int launch_fprop(const FParams& p, const CUtensorMap& x0, const CUtensorMap& x1, const CUtensorMap& w0,
                 const CUtensorMap& w1, cudaStream_t st) {
  using L = FLayout<BN>;
  auto kern = conv_window_fprop_kernel<BN>;
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1ull << (dev & 63)))) {
    OMNI_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES));
    configured |= 1ull << (dev & 63);
  }
  const int pairs = omni::sm_count_cached(dev) / 2;
  const int grid = 2 * (p.units < pairs ? p.units : pairs);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(L::THREADS);
  cfg.dynamicSmemBytes = L::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OMNI_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, x0, x1, w0, w1, p));
  return omni::check_launch("conv_window_fprop");
}

}  // namespace cwin

extern "C" {

long long omni_conv_window_plan(int op, int b, int n2, int cp, int k2, int d_out) {
  cwin::Geo g;
  if (cwin::geometry(b, n2, cp, k2, d_out, &g)) return -1;
  if (op == OMNI_CONV_FPROP) return (d_out == 32 || d_out == 64 || d_out == 96 || d_out == 128) ? 0 : -1;
  if (op != OMNI_CONV_WGRAD_BIAS || d_out % 32 != 0 || d_out > 96 || g.m > cwin::W_KB) return -1;
  return (long long)cwin::wgrad_splits(b * g.m) * d_out * cwin::W_COLS * 4;
}

int omni_conv_window_f32(int op, const float* Xs, int b, int n2, int cp, int k2, int d_out, const float* G,
                         long long ldg, float* Y, long long ldy, int epilogue, const float* bias,
                         float* workspace, long long ws_bytes, void* stream) {
  cwin::Geo g;
  int rc = cwin::geometry(b, n2, cp, k2, d_out, &g);
  if (rc) return rc;
  OMNI_REQUIRE(((uintptr_t)Xs & 15) == 0 && ((uintptr_t)G & 15) == 0 && ((uintptr_t)Y & 15) == 0 &&
                   ldg % 4 == 0 && ldy % 4 == 0,
               "conv window: operands must be 16-byte aligned with leading dimensions %% 4 == 0");
  cudaStream_t st = omni::as_stream(stream);
  const long long rows = (long long)b * n2 * n2;
  const int taps = g.taps;
  if (op == OMNI_CONV_FPROP) {
    OMNI_REQUIRE(d_out == 32 || d_out == 64 || d_out == 96 || d_out == 128,
                 "conv window fprop: d_out must be 32, 64, 96 or 128 (got %d)", d_out);
    OMNI_REQUIRE(ldg >= (long long)taps * cwin::CP && ldy >= d_out, "conv window fprop: leading dimension too small");
    OMNI_REQUIRE(epilogue == OMNI_EPI_STORE || epilogue == OMNI_EPI_BIAS || epilogue == OMNI_EPI_BIAS_RELU ||
                     epilogue == OMNI_EPI_RELU,
                 "conv window fprop: unsupported epilogue %d", epilogue);
    OMNI_REQUIRE(!(epilogue == OMNI_EPI_BIAS || epilogue == OMNI_EPI_BIAS_RELU) || bias,
                 "conv window fprop: bias epilogue needs a bias vector");
    const int bnl = d_out / 2;
    CUtensorMap x0, x1, w0, w1;
    const cuuint64_t xd[2] = {(cuuint64_t)cwin::CP, (cuuint64_t)rows};
    const cuuint64_t xs[1] = {(cuuint64_t)cwin::CP * 4};
    const cuuint32_t bx0[2] = {32, (cuuint32_t)g.win_f}, bx1[2] = {16, (cuuint32_t)g.win_f};
    const cuuint64_t wd[2] = {(cuuint64_t)taps * cwin::CP, (cuuint64_t)d_out};
    const cuuint64_t ws_[1] = {(cuuint64_t)ldg * 4};
    const cuuint32_t bw0[2] = {32, (cuuint32_t)bnl}, bw1[2] = {16, (cuuint32_t)bnl};
    if ((rc = cwin::tmap(&x0, Xs, 2, xd, xs, bx0, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if ((rc = cwin::tmap(&x1, Xs, 2, xd, xs, bx1, CU_TENSOR_MAP_SWIZZLE_64B))) return rc;
    if ((rc = cwin::tmap(&w0, G, 2, wd, ws_, bw0, CU_TENSOR_MAP_SWIZZLE_128B))) return rc;
    if ((rc = cwin::tmap(&w1, G, 2, wd, ws_, bw1, CU_TENSOR_MAP_SWIZZLE_64B))) return rc;
    cwin::FParams p{};
    p.b = b;
    p.n2 = n2;
    p.m = g.m;
    p.k2 = k2;
    p.n2sq = n2 * n2;
    p.rows = rows;
    p.units = (int)omni::ceil_div(rows, 256);
    p.win_rows = g.win_f;
    p.epilogue = epilogue;
    p.bias = bias;
    p.Y = Y;
    p.ldy = ldy;
    p.debug = getenv("OMNI_WINDOW_DEBUG") ? atoi(getenv("OMNI_WINDOW_DEBUG")) : 0;
    switch (d_out) {
      case 32: return cwin::launch_fprop<32>(p, x0, x1, w0, w1, st);
      case 64: return cwin::launch_fprop<64>(p, x0, x1, w0, w1, st);
      case 96: return cwin::launch_fprop<96>(p, x0, x1, w0, w1, st);
      default: return cwin::launch_fprop<128>(p, x0, x1, w0, w1, st);
    }
  }
  OMNI_REQUIRE(op == OMNI_CONV_WGRAD_BIAS, "conv window: op must be FPROP or WGRAD_BIAS");
  OMNI_REQUIRE(d_out % 32 == 0 && d_out <= 96, "conv window wgrad: d_out must be 32, 64 or 96 (got %d)", d_out);
  OMNI_REQUIRE(g.m <= cwin::W_KB, "conv window wgrad: output rows wider than %d pixels", cwin::W_KB);
  const int ncols = taps * cwin::CP + 1;
  OMNI_REQUIRE(ldg >= d_out && ldy >= cwin::W_COLS,
               "conv window wgrad: leading dimension too small (ldg >= d_out, ldy >= %d)", cwin::W_COLS);
  (void)ncols;
  const int units = b * g.m;
  const int S = cwin::wgrad_splits(units);
  const long long need = (long long)S * d_out * cwin::W_COLS * 4;
  OMNI_REQUIRE(workspace && ws_bytes >= need && ((uintptr_t)workspace & 15) == 0,
               "conv window wgrad: workspace of %lld bytes required (got %lld)", need, ws_bytes);
  cwin::WParams p{};
  p.n2 = n2;
  p.m = g.m;
  p.units = units;
  p.d_out = d_out;
  p.ring_off = 0;
  p.stage_off = cwin::W_RING * 4 * cwin::W_ATOM;
  p.bar_off = p.stage_off + cwin::W_STAGES * 7 * cwin::W_ATOM;
  p.ws = workspace;
  CUtensorMap tg, tx;
  // dZ rows of one output row: (o, w < m, unit); w = m .. W_KB-1 zero-filled
  const cuuint64_t gd[3] = {(cuuint64_t)d_out, (cuuint64_t)g.m, (cuuint64_t)units};
  const cuuint64_t gs[2] = {(cuuint64_t)ldg * 4, (cuuint64_t)g.m * ldg * 4};
  const cuuint32_t gb[3] = {32, (cuuint32_t)cwin::W_KB, 1};
  // the s2d image as overlapping 160-float rows at the 48-float pixel pitch:
  // row q, column J = X[q * 48 + J] (J < 144: the three ky taps' channels).
  // The last two pixels are out of bounds (read as zeros); the last in-bounds
  // row reads 64 bytes past the image (caller-provided slack, junk M rows).
  const cuuint64_t xd[2] = {160, (cuuint64_t)(rows - 2)};
  const cuuint64_t xs[1] = {(cuuint64_t)cwin::CP * 4};
  const cuuint32_t xb[2] = {32, (cuuint32_t)cwin::W_KB};
  if ((rc = cwin::tmap(&tg, G, 3, gd, gs, gb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))) return rc;
  if ((rc = cwin::tmap(&tx, Xs, 2, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))) return rc;
  const int bytes = (int)(p.bar_off + 256 + 1024);
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1ull << (dev & 63)))) {
    OMNI_CUDA_TRY(cudaFuncSetAttribute(cwin::conv_window_wgrad_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    configured |= 1ull << (dev & 63);
  }
  cwin::conv_window_wgrad_kernel<<<S, 256, bytes, st>>>(tg, tx, p);
  rc = omni::check_launch("conv_window_wgrad");
  if (rc) return rc;
  const int total = d_out * (cwin::W_COLS / 4);
  cwin::window_reduce_kernel<<<omni::grid_for(8LL * total, 256), 256, 0, st>>>(workspace, S, d_out, cwin::W_COLS, Y,
                                                                         ldy);
  return omni::check_launch("conv_window_reduce");
}

}  // extern "C"
