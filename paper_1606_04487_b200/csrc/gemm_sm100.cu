// K2: the conv/FC contraction -- "one big GEMM per layer per batch"
// (tensors.py:193-210) -- as a persistent, warp-specialised
// tcgen05 kernel for sm_100a.
//
//   C[i,j] (op)= sum_r A(i,r) B(j,r)
//
// Pipeline per CTA (one CTA per SM, 128 x BN output tiles, BK = 32 fp32):
//   warp 0      TMA producer: 128B-swizzled A/B stages into a STAGES-deep
//               shared-memory ring (mbarrier full/empty pairs)
//   warp 1      MMA issuer: one thread issues tcgen05.mma.kind::tf32
//               (M=128, N=BN, K=8) into a double-buffered TMEM accumulator
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld 32 lanes x 16 columns -> registers ->
//               fused bias / ReLU / ReLU-mask / accumulate -> global
//   warps 8-11  (3xTF32 only) split every stage into hi (tf32-exact, in place)
//               and lo = x - hi copies so the MMA warp can issue
//               hi*hi + lo*hi + hi*lo: ~fp32 accuracy from tf32 tensor cores
//               with no extra HBM traffic.
// Operands may be K-major or MN-major (the weight-gradient products reduce
// over the long M = b*m^2 axis of both lowered operands, problems.py:263-267,
// so both operands are MN-major there); tcgen05 supports MN-major for tf32.
// Few-tile shapes (FC layers, weight gradients) use split-K into a caller
// workspace followed by a fixed-order reduction (deterministic, no atomics).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace gemm {

struct Params {
  int M, N, K;
  int m_tiles, n_tiles, k_tiles, splits, kt_per_split;
  int raster_m_inner;
  int epilogue;
  int vec_ok;         // C row stride % 4 == 0 and C 16-byte aligned
  int vec_aux;        // aux row stride % 4 == 0 and aux 16-byte aligned
  int use_tma_store;  // epilogue stages 32x32 sub-tiles in smem and TMA-stores them
  float* C;
  long long ldc;
  long long split_stride;  // elements between split-K partial outputs
  const float* bias;
  const float* aux;
  long long ld_aux;
  // implicit-GEMM convolution (IM2COL != 0): output size m, m*m, stride, pad,
  // kernel size, 32-channel blocks per filter tap
  int conv_m, conv_mm, conv_s, conv_pad, conv_k, conv_cblocks;
  int transpose_c;  // store C^T: C[j*ldc + i] (weight gradient with im2col as the A operand)
  int ones_chunk;   // IM2COL 3: 32-row A chunk loaded from the ones tile (bias gradient), or -1
  int px_dh, px_dw; // IM2COL 2/3: one k-tile of BKT pixels = px_dh output rows + px_dw columns
};

// CTA2: the tile is computed by a CTA pair (cluster of 2, tcgen05 cta_group::2,
// M = 256): each CTA stages its own 128 rows of A and half (BN/2) of B.
template <int BN, bool SPLIT3, int BKT = BK, bool CTA2 = false>
struct Layout {
  static constexpr int BNL = CTA2 ? BN / 2 : BN;  // B rows staged by this CTA
  static constexpr int A_BYTES = BM * BKT * 4;
  static constexpr int B_BYTES = BNL * BKT * 4;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGE_ALL = SPLIT3 ? 2 * STAGE : STAGE;
  static constexpr int STG_BYTES = 4 * 2 * 32 * 32 * 4;  // 4 epilogue warps x 2 x (32x32 fp32)
  static constexpr int BUDGET = 232448 - STG_BYTES - 256 - 1024;  // 227 KiB opt-in maximum
  static constexpr int STAGES = (BUDGET / STAGE_ALL) > 8 ? 8 : (BUDGET / STAGE_ALL);
  static constexpr int STG_OFF = STAGES * STAGE_ALL;
  static constexpr int BAR_OFF = STG_OFF + STG_BYTES;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;  // barriers + 1 KiB alignment slack
  static constexpr int TMEM_COLS = 2 * BN <= 32    ? 32
                                   : 2 * BN <= 64  ? 64
                                   : 2 * BN <= 128 ? 128
                                   : 2 * BN <= 256 ? 256
                                                   : 512;
  static constexpr int ACC_STRIDE = TMEM_COLS / 2;
  static constexpr int THREADS = SPLIT3 ? 384 : 256;
  static_assert(STAGES >= 2, "need at least two stages");
  static_assert(B_BYTES % 1024 == 0, "B tile must keep 1 KiB swizzle alignment");
};

// 3xTF32 operand split: hi = x rounded to the nearest tf32 (adding half an
// ulp of the 10-bit mantissa to the magnitude bits, then truncating), lo =
// x - hi (exact in fp32, |lo| <= 2^-11 |x|, either sign).  The tensor core
// truncates lo to tf32 again, so the dropped part is <= 2^-21 |x| and, lo's
// sign varying, unbiased -- a plain truncating split leaves lo >= 0 relative
// to x and its truncation error biased, which cancellation in long K sums
// turns into a ~4x larger normwise error.
__device__ __forceinline__ void split_tf32(uint32_t x, uint32_t& hi, uint32_t& lo) {
  hi = (x + 0x1000u) & 0xFFFFE000u;
  lo = __float_as_uint(__uint_as_float(x) - __uint_as_float(hi));
}

__device__ __forceinline__ void decode_work(const Params& p, int w, int& mt, int& nt, int& sp) {
  const int per = p.m_tiles * p.n_tiles;
  sp = w / per;
  const int r = w - sp * per;
  if (p.raster_m_inner) {
    nt = r / p.m_tiles;
    mt = r - nt * p.m_tiles;
  } else {
    mt = r / p.n_tiles;
    nt = r - mt * p.n_tiles;
  }
}

// With transpose_c the logical output is C^T: the bias indexes rows and the
// mask operand is read transposed, so both stay in the caller's layout.
template <int MODE>
__device__ __forceinline__ float epi_one(float acc, const Params& p, int row, int col,
                                         const float* Crow) {
  // The TMA-store epilogue evaluates whole 32 x 32 sub-tiles and lets the
  // tensor map clip the store at the M/N edges, so operand reads of
  // out-of-range elements must be masked here (the value is discarded).
  const bool in = row < p.M && col < p.N;
  const int bi = p.transpose_c ? row : col;
  if (MODE == OMNI_EPI_BIAS) return acc + (in ? __ldg(p.bias + bi) : 0.f);
  if (MODE == OMNI_EPI_BIAS_RELU) return fmaxf(acc + (in ? __ldg(p.bias + bi) : 0.f), 0.f);
  if (MODE == OMNI_EPI_ACCUM) return Crow[col] + acc;
  if (MODE == OMNI_EPI_MASK_AUX) {
    const long long ai = p.transpose_c ? (long long)col * p.ld_aux + row : (long long)row * p.ld_aux + col;
    return (in && __ldg(p.aux + ai) > 0.f) ? acc : 0.f;
  }
  if (MODE == OMNI_EPI_RELU) return fmaxf(acc, 0.f);
  return acc;
}

// Runtime-mode wrapper for the (rare) scalar paths.
__device__ __forceinline__ float epi_apply(int mode, float acc, const Params& p, int row, int col,
                                           const float* Crow) {
  switch (mode) {
    case OMNI_EPI_BIAS: return epi_one<OMNI_EPI_BIAS>(acc, p, row, col, Crow);
    case OMNI_EPI_BIAS_RELU: return epi_one<OMNI_EPI_BIAS_RELU>(acc, p, row, col, Crow);
    case OMNI_EPI_ACCUM: return epi_one<OMNI_EPI_ACCUM>(acc, p, row, col, Crow);
    case OMNI_EPI_MASK_AUX: return epi_one<OMNI_EPI_MASK_AUX>(acc, p, row, col, Crow);
    case OMNI_EPI_RELU: return epi_one<OMNI_EPI_RELU>(acc, p, row, col, Crow);
    default: return acc;
  }
}

// Apply the epilogue to N consecutive columns held in registers; the mode
// dispatch happens once per chunk, not per element.
template <int MODE, int N>
__device__ __forceinline__ void epi_chunk_t(float (&v)[N], const uint32_t* r, const Params& p,
                                            int row, int col0) {
  if (MODE == OMNI_EPI_MASK_AUX && p.vec_aux && !p.transpose_c && row < p.M && col0 + N <= p.N) {
    // each lane owns one row: read its N mask values as 16-byte vectors
    const float4* a = reinterpret_cast<const float4*>(p.aux + (long long)row * p.ld_aux + col0);
#pragma unroll
    for (int q = 0; q < N / 4; ++q) {
      const float4 m = __ldg(a + q);
      v[4 * q] = m.x > 0.f ? __uint_as_float(r[4 * q]) : 0.f;
      v[4 * q + 1] = m.y > 0.f ? __uint_as_float(r[4 * q + 1]) : 0.f;
      v[4 * q + 2] = m.z > 0.f ? __uint_as_float(r[4 * q + 2]) : 0.f;
      v[4 * q + 3] = m.w > 0.f ? __uint_as_float(r[4 * q + 3]) : 0.f;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = epi_one<MODE>(__uint_as_float(r[j]), p, row, col0 + j, nullptr);
}
template <int N>
__device__ __forceinline__ void epi_chunk(int mode, float (&v)[N], const uint32_t* r,
                                          const Params& p, int row, int col0) {
  switch (mode) {
    case OMNI_EPI_BIAS: epi_chunk_t<OMNI_EPI_BIAS, N>(v, r, p, row, col0); break;
    case OMNI_EPI_BIAS_RELU: epi_chunk_t<OMNI_EPI_BIAS_RELU, N>(v, r, p, row, col0); break;
    case OMNI_EPI_MASK_AUX: epi_chunk_t<OMNI_EPI_MASK_AUX, N>(v, r, p, row, col0); break;
    case OMNI_EPI_RELU: epi_chunk_t<OMNI_EPI_RELU, N>(v, r, p, row, col0); break;
    default: epi_chunk_t<OMNI_EPI_STORE, N>(v, r, p, row, col0); break;
  }
}

template <int BN, bool A_MN, bool B_MN, bool SPLIT3, int IM2COL, int BKT, bool CTA2>
__global__ void __launch_bounds__(Layout<BN, SPLIT3, BKT, CTA2>::THREADS, 1)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC,
                     const __grid_constant__ CUtensorMap tmO, const Params p) {
  // K-major operands hold exactly one 128-byte swizzle row (32 fp32) per stage;
  // deeper stages are for MN-major operands only.
  // BKT = K per pipeline stage.  MN-major operands stage BKT K-rows directly;
  // K-major operands stage KSUB = BKT / 32 sub-tiles of one 128-byte swizzle
  // row each (64-deep stages halve the stages, barriers and TMA issues per
  // byte -- the per-stage cost bounds the short-tile conv / FC GEMMs).
  static_assert(BKT == BK || BKT == 2 * BK, "BKT must be 32 or 64");
  static_assert(IM2COL != 4 || BKT == BK, "the transposed im2col form stages 32-deep");
  constexpr int KSUB = BKT / BK;
  // 3xTF32 on CTA pairs: each CTA's TMA signals its OWN full barrier (its
  // converter warps must see its stage land), each CTA splits its own half of
  // the stage, and the converters' per-warp arrivals gather on CTA 0's
  // conversion barrier, which the MMA issuer waits on.
  constexpr bool OWN_FULL = SPLIT3 || !CTA2;
  using L = Layout<BN, SPLIT3, BKT, CTA2>;
  constexpr int BM_T = CTA2 ? 2 * BM : BM;  // output rows per work tile
  constexpr int BNL = L::BNL;               // B rows this CTA stages
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + L::BAR_OFF;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (8 + s); };
  auto conv_bar = [&](int s) { return bar0 + 8u * (16 + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (24 + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (26 + a); };
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::BAR_OFF + 8 * 28);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA pair: rank 0 issues the MMAs for both; work units go to pairs
  const int rank = CTA2 ? (int)cluster_ctarank() : 0;
  const int unit0 = CTA2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int units = CTA2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.use_tma_store) tma_prefetch_desc(&tmC);
    if (IM2COL == 3 && p.ones_chunk >= 0) tma_prefetch_desc(&tmO);
    for (int s = 0; s < L::STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
      if (SPLIT3) mbar_init(conv_bar(s), CTA2 ? 2 : 1);  // one arrival per CTA's converters
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), CTA2 ? 8 : 128);  // pair: one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if (CTA2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_holder)),
                   "n"(L::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_holder)),
                   "n"(L::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CTA2) cluster_sync();  // peer barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int total = p.m_tiles * p.n_tiles * p.splits;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------- TMA producer --
      int stage = 0;
      uint32_t phase = 0;
      for (int w = unit0; w < total; w += units) {
        int mt, nt, sp;
        decode_work(p, w, mt, nt, sp);
        const int kt0 = sp * p.kt_per_split;
        const int kt1 = min(p.k_tiles, kt0 + p.kt_per_split);
        const int arow = mt * BM_T + rank * BM;  // first A row / B column this CTA stages
        const int bcol = nt * BN + rank * BNL;
        // im2col A (or B): window corner of this tile's first output pixel
        int a_img = 0, a_h0 = 0, a_w0 = 0, b_img = 0, b_h0 = 0, b_w0 = 0;
        if (IM2COL == 1) {
          const int m0 = arow;
          a_img = m0 / p.conv_mm;
          const int r = m0 - a_img * p.conv_mm;
          a_h0 = (r / p.conv_m) * p.conv_s - p.conv_pad;
          a_w0 = (r - (r / p.conv_m) * p.conv_m) * p.conv_s - p.conv_pad;
        }
        if (IM2COL == 4) {
          const int n0 = bcol;
          b_img = n0 / p.conv_mm;
          const int r = n0 - b_img * p.conv_mm;
          b_h0 = (r / p.conv_m) * p.conv_s - p.conv_pad;
          b_w0 = (r - (r / p.conv_m) * p.conv_m) * p.conv_s - p.conv_pad;
        }
        // This single thread paces the pipeline, so everything that does not
        // change along K is computed once per work unit and the K walk uses
        // division-free cursors.
        // IM2COL 2/3: (filter tap, channel block) of each 32-row im2col chunk
        constexpr int NCH = IM2COL == 3 ? BM / 32 : (IM2COL == 2 ? BNL / 32 : 1);
        int ch_c[NCH], ch_kx[NCH], ch_ky[NCH];  // ch_c < 0: the ones chunk
        // IM2COL 2/3: pixel cursor (image, output row, output column) of k-tile kt
        int px_img = 0, px_oh = 0, px_ow = 0;
        if (IM2COL == 2 || IM2COL == 3) {
          const int taps = p.conv_k * p.conv_k;
          const int first = (IM2COL == 3 ? arow : bcol) / 32;
#pragma unroll
          for (int j = 0; j < NCH; ++j) {
            const int blk = first + j;
            int tap = blk / p.conv_cblocks;
            const int cb = blk - tap * p.conv_cblocks;
            if (tap >= taps) tap = taps - 1;  // rows past M: any valid load, discarded
            ch_kx[j] = tap / p.conv_k;
            ch_ky[j] = tap - ch_kx[j] * p.conv_k;
            ch_c[j] = (IM2COL == 3 && blk == p.ones_chunk) ? -1 : cb * 32;
          }
          const int kc0 = kt0 * BKT;
          px_img = kc0 / p.conv_mm;
          const int r = kc0 - px_img * p.conv_mm;
          px_oh = r / p.conv_m;
          px_ow = r - px_oh * p.conv_m;
        }
        // IM2COL 1/4: (channel block, tap) cursor of k-tile kt, tap-major K
        int t_cb = 0, t_kx = 0, t_ky = 0;
        if (IM2COL == 1 || IM2COL == 4) {
          const int blk0 = kt0 * KSUB;   // first 32-wide K block of this work unit
          const int tap = blk0 / p.conv_cblocks;
          t_cb = blk0 - tap * p.conv_cblocks;
          t_kx = tap / p.conv_k;
          t_ky = tap - t_kx * p.conv_k;
        }
        for (int kt = kt0; kt < kt1; ++kt) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          if (OWN_FULL) mbar_expect_tx(full_bar(stage), (uint32_t)L::STAGE);
          else if (rank == 0) mbar_expect_tx(full_bar(stage), (uint32_t)(2 * L::STAGE));
          const uint32_t fb = OWN_FULL ? full_bar(stage) : mapa_rank0(full_bar(stage));
          auto load2d = [&](const CUtensorMap* map, uint32_t dst, int c0, int c1) {
            if (!OWN_FULL) tma_load_2d_pair(map, dst, fb, c0, c1);
            else tma_load_2d(map, dst, fb, c0, c1);
          };
          auto load_im2col = [&](const CUtensorMap* map, uint32_t dst, int c, int w_, int h_, int n_,
                                 uint16_t ow, uint16_t oh) {
            if (!OWN_FULL) tma_load_im2col_pair(map, dst, fb, c, w_, h_, n_, ow, oh);
            else tma_load_im2col(map, dst, fb, c, w_, h_, n_, ow, oh);
          };
          const uint32_t a_dst = sbase + stage * L::STAGE_ALL;
          const uint32_t b_dst = a_dst + L::A_BYTES;
          const int kc = kt * BKT;
          const int px_h0 = px_oh * p.conv_s - p.conv_pad, px_w0 = px_ow * p.conv_s - p.conv_pad;
          if (IM2COL == 1) {
            // K index = (tap, channel): tap-major, 32-channel blocks, KSUB per stage
#pragma unroll
            for (int sub = 0; sub < KSUB; ++sub) {
              // past the last block (odd block count): reload the last one, the MMA skips it
              const bool past = t_kx >= p.conv_k;
              load_im2col(&tmA, a_dst + sub * (BM * 128), (past ? p.conv_cblocks - 1 : t_cb) * 32, a_w0,
                          a_h0, a_img, (uint16_t)(past ? p.conv_k - 1 : t_ky),
                          (uint16_t)(past ? p.conv_k - 1 : t_kx));
              if (++t_cb == p.conv_cblocks) {
                t_cb = 0;
                if (++t_ky == p.conv_k) {
                  t_ky = 0;
                  ++t_kx;
                }
              }
            }
          } else if (IM2COL == 3) {
            // A(i = (tap, ch), r = pixel): BKT output pixels x 32 channels per 32-row chunk
#pragma unroll
            for (int j = 0; j < NCH; ++j) {
              if (ch_c[j] < 0)  // bias-gradient row: sum over pixels of dY
                load2d(&tmO, a_dst + j * (BKT * 128), 0, 0);
              else
                load_im2col(&tmA, a_dst + j * (BKT * 128), ch_c[j], px_w0, px_h0, px_img,
                            (uint16_t)ch_ky[j], (uint16_t)ch_kx[j]);
            }
          } else if (!A_MN) {
#pragma unroll
            for (int sub = 0; sub < KSUB; ++sub) load2d(&tmA, a_dst + sub * (BM * 128), kc + 32 * sub, arow);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 32; ++j)
              load2d(&tmA, a_dst + j * (BKT * 128), arow + 32 * j, kc);
          }
          if (IM2COL == 4) {
            // B(j = pixel, r = (tap, ch)): BN output pixels x 32 channels, K-major
            load_im2col(&tmB, b_dst, t_cb * 32, b_w0, b_h0, b_img, (uint16_t)t_ky, (uint16_t)t_kx);
          } else if (IM2COL == 2) {
            // B(j = (tap, ch), r = pixel): BKT output pixels x 32 channels per chunk
#pragma unroll
            for (int j = 0; j < NCH; ++j)
              load_im2col(&tmB, b_dst + j * (BKT * 128), ch_c[j], px_w0, px_h0, px_img,
                          (uint16_t)ch_ky[j], (uint16_t)ch_kx[j]);
          } else if (!B_MN) {
#pragma unroll
            for (int sub = 0; sub < KSUB; ++sub) load2d(&tmB, b_dst + sub * (BNL * 128), kc + 32 * sub, bcol);
          } else {
#pragma unroll
            for (int j = 0; j < BNL / 32; ++j)
              load2d(&tmB, b_dst + j * (BKT * 128), bcol + 32 * j, kc);
          }
          // advance the K cursors by one k-tile (IM2COL 1 advanced per sub-tile above)
          if (IM2COL == 4) {
            if (++t_cb == p.conv_cblocks) {
              t_cb = 0;
              if (++t_ky == p.conv_k) {
                t_ky = 0;
                ++t_kx;
              }
            }
          }
          if (IM2COL == 2 || IM2COL == 3) {
            px_ow += p.px_dw;  // BKT = px_dh * m + px_dw pixels
            px_oh += p.px_dh;
            if (px_ow >= p.conv_m) {
              px_ow -= p.conv_m;
              ++px_oh;
            }
            if (px_oh >= p.conv_m) {
              px_img += px_oh / p.conv_m;
              px_oh -= (px_oh / p.conv_m) * p.conv_m;
            }
          }
          if (++stage == L::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ------------------------------------------------------ MMA issuer --
      constexpr uint32_t idesc = instr_desc<BN, A_MN, B_MN, BM_T>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int w = unit0; w < total; w += units) {
        int mt, nt, sp;
        decode_work(p, w, mt, nt, sp);
        const int kt0 = sp * p.kt_per_split;
        const int kt1 = min(p.k_tiles, kt0 + p.kt_per_split);
        if (CTA2) mbar_wait_acq_cluster(tempty_bar(acc), acc_phase ^ 1);  // both CTAs drained it
        else mbar_wait(tempty_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * L::ACC_STRIDE);
        for (int kt = kt0; kt < kt1; ++kt) {
          if (SPLIT3 && CTA2) mbar_wait_acq_cluster(conv_bar(stage), phase);  // both CTAs converted
          else mbar_wait(SPLIT3 ? conv_bar(stage) : full_bar(stage), phase);
          tc_fence_after();
          const uint32_t a_addr = sbase + stage * L::STAGE_ALL;
          const uint32_t b_addr = a_addr + L::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BKT / 8; ++kk) {
            // an odd number of 32-wide K blocks: the last stage's second sub-tile is past K
            if (KSUB > 1 && kk > 0 && (kk & 3) == 0 && kt * BKT + kk * 8 >= p.K) break;
            const uint32_t a_off = A_MN ? kk * 1024u : (uint32_t)(kk >> 2) * (BM * 128u) + (kk & 3) * 32u;
            const uint32_t b_off = B_MN ? kk * 1024u : (uint32_t)(kk >> 2) * (BNL * 128u) + (kk & 3) * 32u;
            const uint64_t ad = smem_desc<A_MN, BKT>(a_addr + a_off);
            const uint64_t bd = smem_desc<B_MN, BKT>(b_addr + b_off);
            if (CTA2) tc_mma_tf32_pair(d_tmem, ad, bd, idesc, (kt > kt0 || kk > 0) ? 1u : 0u);
            else tc_mma_tf32(d_tmem, ad, bd, idesc, (kt > kt0 || kk > 0) ? 1u : 0u);
            if (SPLIT3) {
              const uint64_t ad_lo = smem_desc<A_MN, BKT>(a_addr + L::STAGE + a_off);
              const uint64_t bd_lo = smem_desc<B_MN, BKT>(b_addr + L::STAGE + b_off);
              if (CTA2) {
                tc_mma_tf32_pair(d_tmem, ad_lo, bd, idesc, 1u);
                tc_mma_tf32_pair(d_tmem, ad, bd_lo, idesc, 1u);
              } else {
                tc_mma_tf32(d_tmem, ad_lo, bd, idesc, 1u);
                tc_mma_tf32(d_tmem, ad, bd_lo, idesc, 1u);
              }
            }
          }
          // frees the stage (in both CTAs of a pair) once these MMAs have read it
          if (CTA2) tc_commit_pair(empty_bar(stage));
          else tc_commit(empty_bar(stage));
          if (++stage == L::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CTA2) tc_commit_pair(tfull_bar(acc));  // accumulator complete -> epilogues
        else tc_commit(tfull_bar(acc));
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // -------------------------------------------------------- epilogue --
    const int ew = warp - 4;  // TMEM lanes 32*ew .. 32*ew+31
    int acc = 0;
    uint32_t acc_phase = 0;
    const int mode = p.splits > 1 ? OMNI_EPI_STORE : p.epilogue;
    int st_chunk = 0;
    // hand a drained accumulator back to the MMA issuer (CTA 0 of a pair)
    auto release_acc = [&](int a) {
      tc_fence_before();
      if (CTA2) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(mapa_rank0(tempty_bar(a)));  // TMEM reads only: no store drain
      } else {
        mbar_arrive(tempty_bar(a));
      }
    };
    for (int w = unit0; w < total; w += units) {
      int mt, nt, sp;
      decode_work(p, w, mt, nt, sp);
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
      const int row0 = mt * BM_T + rank * BM + ew * 32;  // this warp's 32 output rows
      const int row = row0 + lane;
      const uint32_t t_row =
          tmem_base + (uint32_t)(acc * L::ACC_STRIDE) + ((uint32_t)(ew * 32) << 16);
      if (p.use_tma_store) {
        // 32 x 32 sub-tiles: registers -> 128B-swizzled smem -> TMA bulk store
        // (coalesced, clipped at the M/N edges by the tensor map).
        const uint32_t stg = sbase + L::STG_OFF + ew * 8192;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          const int col0 = nt * BN + c0;
          if (col0 >= p.N) break;  // warp-uniform
          uint32_t r[32];
          tmem_ld16(t_row + (uint32_t)c0, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
          tmem_ld16(t_row + (uint32_t)c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&r[16]));
          tmem_wait_ld();
          if (c0 + 32 >= BN || col0 + 32 >= p.N) {
            // last TMEM read of this accumulator: hand it back to the MMA warp early
            release_acc(acc);
          }
          const uint32_t buf = stg + (uint32_t)(st_chunk & 1) * 4096u;
          if (lane == 0) bulk_wait_read<1>();  // the store that last used `buf` has read it
          __syncwarp();
          float v[32];
          epi_chunk<32>(mode, v, r, p, row, col0);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(buf + (uint32_t)lane * 128u + ((uint32_t)(j ^ (lane & 7)) << 4), v[4 * j],
                         v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmC, buf, col0, row0, sp);
            bulk_commit();
          }
          ++st_chunk;
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        continue;
      }
      float* Crow = p.C + (long long)sp * p.split_stride + (long long)row * p.ldc;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        const int col0 = nt * BN + c0;
        if (col0 >= p.N) break;  // warp-uniform
        uint32_t r[16];
        tmem_ld16(t_row + (uint32_t)c0, r);
        tmem_wait_ld();
        if (p.transpose_c && row < p.M) {
          // C^T: for each column the warp's 32 lanes (consecutive rows) write 128 contiguous bytes
          float v[16];
          epi_chunk<16>(mode, v, r, p, row, col0);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (col0 + j < p.N) p.C[(long long)(col0 + j) * p.ldc + row] = v[j];
        } else if (row < p.M) {
          if (p.vec_ok && col0 + 16 <= p.N && mode != OMNI_EPI_ACCUM && mode != OMNI_EPI_MASK_AUX) {
            float v[16];
            epi_chunk<16>(mode, v, r, p, row, col0);
            float4* dst = reinterpret_cast<float4*>(Crow + col0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int col = col0 + j;
              if (col < p.N) Crow[col] = epi_apply(mode, __uint_as_float(r[j]), p, row, col, Crow);
            }
          }
        }
      }
      release_acc(acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (p.use_tma_store && lane == 0) bulk_wait_all();
  } else if (SPLIT3 && warp >= 8) {
    // ------------------------------------------- 3xTF32 hi/lo converters --
    const int t = threadIdx.x - 256;
    int stage = 0;
    uint32_t phase = 0;
    for (int w = unit0; w < total; w += units) {
      int mt, nt, sp;
      decode_work(p, w, mt, nt, sp);
      const int kt0 = sp * p.kt_per_split;
      const int kt1 = min(p.k_tiles, kt0 + p.kt_per_split);
      for (int kt = kt0; kt < kt1; ++kt) {
        mbar_wait(full_bar(stage), phase);
        uint4* hi = reinterpret_cast<uint4*>(smem + stage * L::STAGE_ALL);
        uint4* lo = reinterpret_cast<uint4*>(smem + stage * L::STAGE_ALL + L::STAGE);
        for (int i = t; i < L::STAGE / 16; i += 128) {
          const uint4 v = hi[i];
          uint4 h, l;
          split_tf32(v.x, h.x, l.x);
          split_tf32(v.y, h.y, l.y);
          split_tf32(v.z, h.z, l.z);
          split_tf32(v.w, h.w, l.w);
          hi[i] = h;
          lo[i] = l;
        }
        // converted stage -> async proxy (the MMA reads it, from CTA 0 for a
        // pair: hence the cluster-scope proxy fence), then one arrival per CTA
        // after all 128 converter threads are done (named barrier 1)
        if (CTA2) asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (t == 0) {
          if (CTA2) mbar_arrive_cluster(mapa_rank0(conv_bar(stage)));
          else mbar_arrive(conv_bar(stage));
        }
        if (++stage == L::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CTA2) cluster_sync();  // the peer's MMAs / commits into this CTA are complete
  if (warp == 2) {
    tc_fence_after();
    if (CTA2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(L::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(L::TMEM_COLS)
                   : "memory");
  }
}

// The ones tile behind OMNI_CONV_WGRAD_BIAS's bias-gradient row: a constant
// device array (TMA source), so no per-call fill launch.  kOnesBytes of the
// caller's workspace stay reserved for it (unchanged workspace contract).
constexpr int kOnesBytes = 64 * 32 * 4;  // BKT (<= 64) K-rows x 32 fp32
#define OMNI_ONES4 1.f, 1.f, 1.f, 1.f
#define OMNI_ONES16 OMNI_ONES4, OMNI_ONES4, OMNI_ONES4, OMNI_ONES4
#define OMNI_ONES64 OMNI_ONES16, OMNI_ONES16, OMNI_ONES16, OMNI_ONES16
#define OMNI_ONES256 OMNI_ONES64, OMNI_ONES64, OMNI_ONES64, OMNI_ONES64
__device__ __align__(128) float g_ones_tile[kOnesBytes / 4] = {
    OMNI_ONES256, OMNI_ONES256, OMNI_ONES256, OMNI_ONES256,
    OMNI_ONES256, OMNI_ONES256, OMNI_ONES256, OMNI_ONES256};
static_assert(kOnesBytes / 4 == 8 * 256, "ones tile initialiser size");

// Device address of g_ones_tile on the current device (cached per device).
const float* ones_tile() {
  static const float* addr[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!addr[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_ones_tile) != cudaSuccess) return nullptr;
    addr[dev] = static_cast<const float*>(p);
  }
  return addr[dev];
}

// Generic (scalar) split-K reduction.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws, int S,
                                                            int M, int N, Params p) {
  const long long total = (long long)M * N;
  const long long MN = total;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / N), col = (int)(idx - (idx / N) * N);
    float acc = 0.f;
    for (int s = 0; s < S; ++s) acc += ws[(long long)s * MN + idx];
    if (p.transpose_c) {
      p.C[(long long)col * p.ldc + row] = epi_apply(p.epilogue, acc, p, row, col, nullptr);
    } else {
      float* Crow = p.C + (long long)row * p.ldc;
      Crow[col] = epi_apply(p.epilogue, acc, p, row, col, Crow);
    }
  }
}

// Split-K reductions: C[i,j] = epi(sum_s ws[s][i][j]) in ascending s (the same
// order in every variant, so results do not depend on which one runs).
// Natural store, 4 columns per thread (N, ldc % 4 == 0, C 16-byte aligned).
template <int MODE>
__global__ void __launch_bounds__(256) splitk_reduce_v4_kernel(const float* __restrict__ ws, int S,
                                                               int M, int N, Params p) {
  const int n4 = N >> 2;
  const int total = M * n4;
  const long long MN = (long long)M * N;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int row = i / n4;
    const int col = (i - row * n4) << 2;
    const float* src = ws + (long long)row * N + col;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);  // 0 + sum, as the generic kernel
    int sp = 0;
    for (; sp + 4 <= S; sp += 4) {   // 4 split loads in flight, then the ordered adds
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(src + (sp + u) * MN));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
    for (; sp < S; ++sp) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(src + sp * MN));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    float* Crow = p.C + (long long)row * p.ldc;
    float4 out;
    out.x = epi_one<MODE>(acc.x, p, row, col, Crow);
    out.y = epi_one<MODE>(acc.y, p, row, col + 1, Crow);
    out.z = epi_one<MODE>(acc.z, p, row, col + 2, Crow);
    out.w = epi_one<MODE>(acc.w, p, row, col + 3, Crow);
    *reinterpret_cast<float4*>(Crow + col) = out;
  }
}

// Transposed store C[j*ldc + i] (weight gradients with im2col as A) through a
// 32 x 32 shared-memory tile: coalesced partial reads and C^T writes.
// One thread per element (1024-thread blocks): the split loop is the long,
// dependent part, so it gets all the parallelism.
template <int MODE>
__global__ void __launch_bounds__(1024) splitk_reduce_t_kernel(const float* __restrict__ ws, int S,
                                                               int M, int N, Params p) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const long long MN = (long long)M * N;
  {
    const int i = i0 + ty, j = j0 + tx;
    float acc = 0.f;
    if (i < M && j < N) {
      const float* src = ws + (long long)i * N + j;
      for (int sp = 0; sp < S; ++sp) acc += src[sp * MN];
    }
    tile[ty][tx] = acc;
  }
  __syncthreads();
  const int j = j0 + ty, i = i0 + tx;
  if (i < M && j < N) p.C[(long long)j * p.ldc + i] = epi_one<MODE>(tile[tx][ty], p, i, j, nullptr);
}

int launch_splitk_reduce(const float* ws, int S, int M, int N, const Params& q, cudaStream_t st) {
  const bool v4 = !q.transpose_c && N % 4 == 0 && q.ldc % 4 == 0 && ((uintptr_t)q.C & 15) == 0 &&
                  (long long)M * (N / 4) < (1LL << 31);
#define OMNI_REDUCE_MODES(KERNEL, GRID, BLOCK)                                                   \
  switch (q.epilogue) {                                                                        \
    case OMNI_EPI_BIAS: KERNEL<OMNI_EPI_BIAS><<<GRID, BLOCK, 0, st>>>(ws, S, M, N, q); break;   \
    case OMNI_EPI_BIAS_RELU:                                                                   \
      KERNEL<OMNI_EPI_BIAS_RELU><<<GRID, BLOCK, 0, st>>>(ws, S, M, N, q);                      \
      break;                                                                                   \
    case OMNI_EPI_ACCUM: KERNEL<OMNI_EPI_ACCUM><<<GRID, BLOCK, 0, st>>>(ws, S, M, N, q); break; \
    case OMNI_EPI_MASK_AUX:                                                                    \
      KERNEL<OMNI_EPI_MASK_AUX><<<GRID, BLOCK, 0, st>>>(ws, S, M, N, q);                       \
      break;                                                                                   \
    case OMNI_EPI_RELU: KERNEL<OMNI_EPI_RELU><<<GRID, BLOCK, 0, st>>>(ws, S, M, N, q); break;   \
    default: KERNEL<OMNI_EPI_STORE><<<GRID, BLOCK, 0, st>>>(ws, S, M, N, q); break;            \
  }
  if (q.transpose_c) {
    const dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
    OMNI_REDUCE_MODES(splitk_reduce_t_kernel, grid, 1024)
  } else if (v4) {
    const int grid = omni::grid_for((long long)M * (N / 4), 256);
    OMNI_REDUCE_MODES(splitk_reduce_v4_kernel, grid, 256)
  } else {
    splitk_reduce_kernel<<<omni::grid_for((long long)M * N, 256), 256, 0, st>>>(ws, S, M, N, q);
  }
#undef OMNI_REDUCE_MODES
  return omni::check_launch("splitk_reduce");
}


// CUDA-core fp32 reference GEMM (OMNI_PREC_FP32_SIMT): 16x16 tiles through
// shared memory.  Test reference only; never on the training path.
template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256) simt_gemm_kernel(const float* __restrict__ A, long long lda,
                                                        const float* __restrict__ B, long long ldb,
                                                        Params p) {
  __shared__ float As[16][17], Bs[16][17];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i = blockIdx.y * 16 + ty, j = blockIdx.x * 16 + tx;
  float acc = 0.f;
  for (int r0 = 0; r0 < p.K; r0 += 16) {
    {
      const int ii = blockIdx.y * 16 + ty, rr = r0 + tx;
      As[ty][tx] = (ii < p.M && rr < p.K) ? (A_MN ? A[(long long)rr * lda + ii]
                                                  : A[(long long)ii * lda + rr])
                                          : 0.f;
      const int jj = blockIdx.x * 16 + ty;
      Bs[ty][tx] = (jj < p.N && rr < p.K) ? (B_MN ? B[(long long)rr * ldb + jj]
                                                  : B[(long long)jj * ldb + rr])
                                          : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) acc = fmaf(As[ty][r], Bs[tx][r], acc);
    __syncthreads();
  }
  if (i < p.M && j < p.N) {
    float* Crow = p.C + (long long)i * p.ldc;
    Crow[j] = epi_apply(p.epilogue, acc, p, i, j, Crow);
  }
}

// ------------------------------------------------------------ host side --
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

int make_tmap_c(CUtensorMap* map, const float* ptr, long long N, long long M, long long ld,
                long long splits, long long split_stride) {
  auto fn = encode_fn();
  if (!fn) {
    omni::set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return OMNI_ECUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)splits};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)(split_stride > 0 ? split_stride : M * ld) * 4};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    omni::set_error("cuTensorMapEncodeTiled (C) failed (%d): N=%lld M=%lld ld=%lld", (int)r, N, M, ld);
    return OMNI_ECUDA;
  }
  return OMNI_OK;
}

int make_tmap(CUtensorMap* map, const float* ptr, long long inner, long long outer, long long ld,
              int box_inner, int box_outer, bool mn_major) {
  auto fn = encode_fn();
  if (!fn) {
    omni::set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return OMNI_ECUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    omni::set_error("cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld ld=%lld box=%dx%d",
                    (int)r, inner, outer, ld, box_inner, box_outer);
    return OMNI_ECUDA;
  }
  return OMNI_OK;
}

struct Plan {
  int bn, splits, kps, m_tiles, n_tiles, k_tiles, grid, raster_m_inner;
  int cta2;  // tiles of 256 rows computed by CTA pairs
};

constexpr int kBNs[] = {32, 64, 96, 128, 192, 256};

// Stage depth of the implicit weight gradient (im2col A, both operands
// MN-major): 64-deep in TF32 mode (OMNI_WGRAD_BKT=32 for the 32-deep variant).
int wgrad_bkt(int precision) {
  static const int env = getenv("OMNI_WGRAD_BKT") ? atoi(getenv("OMNI_WGRAD_BKT")) : 64;
  return (precision == OMNI_PREC_TF32 && env == 64) ? 64 : BK;
}

// Stage depth of every launch: 64-deep for TF32 plain GEMMs (FC) and implicit
// forward / data-gradient convs (OMNI_KMAJOR_BKT=32 for the 32-deep variant);
// the transposed im2col form and 3xTF32 (hi/lo copies double the stage) 32.
int stage_bkt(int precision, int im2col) {
  static const int env = getenv("OMNI_KMAJOR_BKT") ? atoi(getenv("OMNI_KMAJOR_BKT")) : 64;
  if (im2col == 3) return wgrad_bkt(precision);
  if ((im2col == 0 || im2col == 1) && precision == OMNI_PREC_TF32 && env == 64) return 64;
  return BK;
}

Plan make_plan(int M, int N, int K, int sms, int bkt = BK, bool cta2 = false, bool b_mn = false) {
  Plan pl{};
  pl.cta2 = cta2;
  const int bm = cta2 ? 2 * BM : BM;
  const int units = cta2 ? sms / 2 : sms;  // concurrent work units (SMs or SM pairs)
  if (N <= 256) {
    for (int b : kBNs)
      if (b >= N) {
        pl.bn = b;
        break;
      }
  }
  if (N > 192) {
    // Prefer wide tiles (fewer re-reads of A, better MMA/epilogue ratio) unless
    // they waste more than 8% of the MMA work on padding columns.
    pl.bn = 0;
    for (int b : {256, 192, 128}) {
      const long long padded = omni::ceil_div(N, b) * b;
      if (padded * 100 <= (long long)N * 108) {
        pl.bn = b;
        break;
      }
    }
    if (!pl.bn) {
      long long best = -1;
      for (int b : {256, 192, 128}) {
        const long long padded = omni::ceil_div(N, b) * b;
        if (best < 0 || padded < best) {
          best = padded;
          pl.bn = b;
        }
      }
    }
  }
  // a pair stages BN/2 columns of B per CTA: MN-major B needs whole 32-column chunks
  if (cta2 && b_mn && (pl.bn / 2) % 32 != 0) pl.bn = pl.bn < 64 ? 64 : pl.bn + 32;
  pl.m_tiles = (int)omni::ceil_div(M, bm);
  pl.n_tiles = (int)omni::ceil_div(N, pl.bn);
  pl.k_tiles = (int)omni::ceil_div(K, bkt);
  const long long tiles = (long long)pl.m_tiles * pl.n_tiles;
  int splits = 1;
  if (tiles < units && pl.k_tiles >= 8) {
    // Split-K cost model: the persistent grid finishes after ceil(tiles*s/sms)
    // rounds of (k_tiles/s) k-steps each; every extra split adds one M x N
    // fp32 partial written and re-read by the fixed-order reduction.
    const double t_kstep = 2.0 * bm * pl.bn * bkt / (650e12 / units);  // s per k-step per unit
    const int max_splits = pl.k_tiles / 4 < 64 ? pl.k_tiles / 4 : 64;  // >= 4 k-steps per split
    double best = 1e30;
    for (int s = 1; s <= max_splits; ++s) {
      const long long rounds = omni::ceil_div(tiles * s, units);
      const double t = rounds * omni::ceil_div(pl.k_tiles, s) * t_kstep +
                       (s > 1 ? s * (double)M * N * 8.0 / 6.0e12 : 0.0);
      if (t < best * 0.98) {   // prefer fewer splits unless clearly faster
        best = t;
        splits = s;
      }
    }
  }
  // tuning probes (tools/conv_probe.py sweeps): force a tile width / split count
  static const int force_bn = getenv("OMNI_FORCE_BN") ? atoi(getenv("OMNI_FORCE_BN")) : 0;
  static const int force_splits = getenv("OMNI_FORCE_SPLITS") ? atoi(getenv("OMNI_FORCE_SPLITS")) : 0;
  if (force_bn) {
    pl.bn = force_bn;
    pl.n_tiles = (int)omni::ceil_div(N, pl.bn);
  }
  if (force_splits) splits = force_splits < pl.k_tiles ? force_splits : pl.k_tiles;
  pl.kps = (int)omni::ceil_div(pl.k_tiles, splits);
  pl.splits = (int)omni::ceil_div(pl.k_tiles, pl.kps);
  const long long work = tiles * pl.splits;
  pl.grid = (int)(work < units ? work : units) * (cta2 ? 2 : 1);
  pl.raster_m_inner = pl.m_tiles < pl.n_tiles;
  return pl;
}

// CTA pairs (M = 256 tiles, half of B per CTA) for GEMMs with more than one
// 128-row tile: TF32 everywhere but the transposed conv form (im2col B,
// M = d_out <= 128); 3xTF32 on plain GEMMs only (OWN_FULL protocol: each
// CTA's converter warps split its own stage, CTA 0's MMA issuer waits for
// both; bit-identical to single CTAs, 4096^3 0.742 -> 0.644 ms) -- its conv
// forms measured slower on pairs (profiles/r02_3xtf32_pairs_ab.json).
// OMNI_NO_2CTA=1 disables pairs.
bool pair_ok(int precision, int M, int im2col) {
  static const bool off = getenv("OMNI_NO_2CTA") != nullptr;
  if (precision == OMNI_PREC_3XTF32) return !off && M > BM && im2col == 0;
  return !off && precision == OMNI_PREC_TF32 && M > BM && im2col != 4;
}

// The one planning entry point: launches and workspace queries agree on it.
Plan plan_for(int precision, int M, int N, int K, bool b_mn, int im2col) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int bkt = stage_bkt(precision, im2col);
  const bool b_mn_eff = b_mn || im2col == 2 || im2col == 3;
  // SMs left free for concurrent communication kernels (data parallel: the
  // persistent GEMM grids would otherwise hold every SM and delay NCCL)
  const int sms = omni::sm_count_cached(dev) - omni_get_sm_reserve();
  bool pair = pair_ok(precision, M, im2col);
  if (pair && b_mn_eff) {
    // MN-major B is split into 32-column halves: a tile width that does not
    // split (N = 96 -> BN 96) would have to grow and waste MMA work; stay single
    const Plan single = make_plan(M, N, K, sms, bkt, false, b_mn_eff);
    if ((single.bn / 2) % 32 != 0) return single;
  }
  return make_plan(M, N, K, sms, bkt, pair, b_mn_eff);
}

// Activation tensor behind an im2col operand (NHWC, pixel stride cs).
struct ConvGeom {
  const float* X;
  int b, n, c, cs, k, s, pad, m;
};

int make_tmap_im2col(CUtensorMap* map, const ConvGeom& g, int pixels, bool mn_major) {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(ptr);
  });
  if (!fn) {
    omni::set_error("cuTensorMapEncodeIm2col unavailable");
    return OMNI_ECUDA;
  }
  // dims (C, W, H, N) of the NHWC tensor; W is the fastest spatial index.
  cuuint64_t dims[4] = {(cuuint64_t)g.c, (cuuint64_t)g.n, (cuuint64_t)g.n, (cuuint64_t)g.b};
  cuuint64_t strides[3] = {(cuuint64_t)g.cs * 4, (cuuint64_t)g.n * g.cs * 4,
                           (cuuint64_t)g.n * g.n * g.cs * 4};
  // fprop bounding box (CUTLASS convention): lower = -pad, upper = pad - (k - 1)
  int lower[2] = {-g.pad, -g.pad};
  int upper[2] = {g.pad - (g.k - 1), g.pad - (g.k - 1)};
  cuuint32_t estr[4] = {1, (cuuint32_t)g.s, (cuuint32_t)g.s, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(g.X), dims, strides,
                  lower, upper, 32, (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    omni::set_error("cuTensorMapEncodeIm2col failed (%d): b=%d n=%d c=%d cs=%d k=%d s=%d pad=%d",
                    (int)r, g.b, g.n, g.c, g.cs, g.k, g.s, g.pad);
    return OMNI_ECUDA;
  }
  return OMNI_OK;
}

template <int BN, bool A_MN, bool B_MN, bool SPLIT3, int IM2COL, int BKT, bool CTA2>
int launch_tc(const Plan& pl, const float* A, long long lda, const float* B, long long ldb,
              const Params& p, cudaStream_t st, const ConvGeom* cg, const float* ones) {
  constexpr bool B_CHUNKED = B_MN || IM2COL == 2;  // B staged as 32-column MN-major chunks
  if constexpr (CTA2 && B_CHUNKED && (BN / 2) % 32 != 0) {
    omni::set_error("gemm: BN=%d cannot be split across a CTA pair with MN-major B", BN);
    return OMNI_EUNSUPPORTED;
  } else {
    using L = Layout<BN, SPLIT3, BKT, CTA2>;
    CUtensorMap ta, tb;
    int rc;
    if (IM2COL == 1) rc = make_tmap_im2col(&ta, *cg, BM, false);
    else if (IM2COL == 3) rc = make_tmap_im2col(&ta, *cg, BKT, true);
    else rc = A_MN ? make_tmap(&ta, A, p.M, p.K, lda, 32, BKT, true)
                   : make_tmap(&ta, A, p.K, p.M, lda, 32, BM, false);
    if (rc) return rc;
    if (IM2COL == 2) rc = make_tmap_im2col(&tb, *cg, BKT, true);
    else if (IM2COL == 4) rc = make_tmap_im2col(&tb, *cg, L::BNL, false);
    else rc = B_MN ? make_tmap(&tb, B, p.N, p.K, ldb, 32, BKT, true)
                   : make_tmap(&tb, B, p.K, p.N, ldb, 32, L::BNL, false);
    if (rc) return rc;
    CUtensorMap tc, to;
    memset(&tc, 0, sizeof(tc));
    memset(&to, 0, sizeof(to));
    if (p.use_tma_store) {
      rc = make_tmap_c(&tc, p.C, p.N, p.M, p.ldc, p.splits, p.split_stride);
      if (rc) return rc;
    }
    if (IM2COL == 3 && p.ones_chunk >= 0) {  // BKT x 32 ones, MN-major like an im2col chunk
      rc = make_tmap(&to, ones, 32, BKT, 32, 32, BKT, true);
      if (rc) return rc;
    }
    auto kern = gemm_tf32_kernel<BN, A_MN, B_MN, SPLIT3, IM2COL, BKT, CTA2>;
    // once per instantiation and device (so a launch inside CUDA-graph capture
    // makes no attribute calls)
    static unsigned long long configured = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured & (1ull << (dev & 63)))) {
      OMNI_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES));
      configured |= 1ull << (dev & 63);
    }
    if (CTA2) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)pl.grid);
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
      OMNI_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, to, p));
    } else {
      kern<<<pl.grid, L::THREADS, L::BYTES, st>>>(ta, tb, tc, to, p);
    }
    return omni::check_launch("gemm_tf32");
  }
}

template <bool A_MN, bool B_MN, bool SPLIT3, int IM2COL, int BKT, bool CTA2>
int dispatch_bn_t(const Plan& pl, const float* A, long long lda, const float* B, long long ldb,
                  const Params& p, cudaStream_t st, const ConvGeom* cg, const float* ones) {
#define OMNI_BN_CASE(X) \
  case X:               \
    return launch_tc<X, A_MN, B_MN, SPLIT3, IM2COL, BKT, CTA2>(pl, A, lda, B, ldb, p, st, cg, ones);
  switch (pl.bn) {
    OMNI_BN_CASE(32)
    OMNI_BN_CASE(64)
    OMNI_BN_CASE(96)
    OMNI_BN_CASE(128)
    OMNI_BN_CASE(192)
    OMNI_BN_CASE(256)
  }
#undef OMNI_BN_CASE
  omni::set_error("gemm: no kernel for BN=%d", pl.bn);
  return OMNI_EUNSUPPORTED;
}

template <bool A_MN, bool B_MN, bool SPLIT3, int IM2COL, int BKT = BK>
int dispatch_bn(const Plan& pl, const float* A, long long lda, const float* B, long long ldb,
                const Params& p, cudaStream_t st, const ConvGeom* cg = nullptr,
                const float* ones = nullptr) {
  if constexpr (!SPLIT3 && IM2COL != 4) {
    if (pl.cta2)
      return dispatch_bn_t<A_MN, B_MN, false, IM2COL, BKT, true>(pl, A, lda, B, ldb, p, st, cg, ones);
  }
  if constexpr (SPLIT3 && IM2COL == 0) {
    if (pl.cta2)
      return dispatch_bn_t<A_MN, B_MN, true, IM2COL, BKT, true>(pl, A, lda, B, ldb, p, st, cg, ones);
  }
  return dispatch_bn_t<A_MN, B_MN, SPLIT3, IM2COL, BKT, false>(pl, A, lda, B, ldb, p, st, cg, ones);
}

template <bool SPLIT3, int BKT = BK>
int dispatch_major(const Plan& pl, int a_mn, int b_mn, const float* A, long long lda,
                   const float* B, long long ldb, const Params& p, cudaStream_t st) {
  if (!a_mn && !b_mn) return dispatch_bn<false, false, SPLIT3, 0, BKT>(pl, A, lda, B, ldb, p, st);
  if (!a_mn && b_mn) return dispatch_bn<false, true, SPLIT3, 0, BKT>(pl, A, lda, B, ldb, p, st);
  if (a_mn && !b_mn) return dispatch_bn<true, false, SPLIT3, 0, BKT>(pl, A, lda, B, ldb, p, st);
  return dispatch_bn<true, true, SPLIT3, 0, BKT>(pl, A, lda, B, ldb, p, st);
}

// Shared tail of omni_gemm_f32 / omni_conv_implicit_f32: plan, workspace,
// output mode, launch (im2col variant when cg != nullptr), split-K reduce.
int run_gemm(int precision, int M, int N, int K, const float* A, long long lda, int a_mn,
             const float* B, long long ldb, int b_mn, float* C, long long ldc, int epilogue,
             const float* bias, const float* aux, long long ld_aux, float* workspace,
             long long ws_bytes, cudaStream_t st, const ConvGeom* cg, int im2col,
             const float* ones = nullptr) {
  Params p{};
  p.ones_chunk = (im2col == 3 && ones) ? (M - 1) / 32 : -1;  // last row = bias gradient
  p.M = M;
  p.N = N;
  p.K = K;
  p.epilogue = epilogue;
  p.bias = bias;
  p.aux = aux;
  p.ld_aux = ld_aux;
  p.vec_aux = aux && ld_aux % 4 == 0 && ((uintptr_t)aux & 15) == 0;
  // The implicit weight gradient (im2col A, both operands MN-major) runs 64-deep
  // K stages in TF32 mode: half the TMA ops per byte, 64-pixel im2col boxes.
  const int bkt = stage_bkt(precision, im2col);
  const Plan pl = plan_for(precision, M, N, K, b_mn != 0, im2col);
  p.m_tiles = pl.m_tiles;
  p.n_tiles = pl.n_tiles;
  p.k_tiles = pl.k_tiles;
  p.splits = pl.splits;
  p.kt_per_split = pl.kps;
  p.raster_m_inner = pl.raster_m_inner;
  if (cg) {
    p.conv_m = cg->m;
    p.conv_mm = cg->m * cg->m;
    p.conv_s = cg->s;
    p.conv_pad = cg->pad;
    p.conv_k = cg->k;
    p.conv_cblocks = (cg->c + 31) / 32;
    p.px_dh = bkt / cg->m;
    p.px_dw = bkt - p.px_dh * cg->m;
  }
  if (pl.splits > 1) {
    const long long need = (long long)pl.splits * M * N * 4;
    OMNI_REQUIRE(workspace && ws_bytes >= need,
                 "gemm: split-K workspace of %lld bytes required (got %lld)", need, ws_bytes);
    OMNI_REQUIRE(((uintptr_t)workspace & 15) == 0, "gemm: workspace must be 16-byte aligned");
    p.C = workspace;
    p.ldc = N;
    p.split_stride = (long long)M * N;
    p.vec_ok = (N % 4 == 0);
    p.use_tma_store = (N % 4 == 0);
  } else {
    p.C = C;
    p.ldc = ldc;
    p.split_stride = 0;
    p.vec_ok = (ldc % 4 == 0) && (((uintptr_t)C & 15) == 0);
    p.use_tma_store = p.vec_ok && epilogue != OMNI_EPI_ACCUM;
  }
  if (getenv("OMNI_NO_TMA_STORE")) p.use_tma_store = 0;
  if (im2col == 3 || im2col == 4) {
    p.transpose_c = pl.splits > 1 ? 0 : 1;  // partials are natural; the reduce transposes
    if (p.transpose_c) p.use_tma_store = 0;
  }
  int rc;
  const bool s3 = precision == OMNI_PREC_3XTF32;
  if (im2col == 1)
    rc = s3 ? dispatch_bn<false, false, true, 1>(pl, A, lda, B, ldb, p, st, cg)
       : bkt == 64 ? dispatch_bn<false, false, false, 1, 64>(pl, A, lda, B, ldb, p, st, cg)
                   : dispatch_bn<false, false, false, 1>(pl, A, lda, B, ldb, p, st, cg);
  else if (im2col == 3)
    rc = s3 ? dispatch_bn<true, true, true, 3>(pl, A, lda, B, ldb, p, st, cg, ones)
       : bkt == 64 ? dispatch_bn<true, true, false, 3, 64>(pl, A, lda, B, ldb, p, st, cg, ones)
                   : dispatch_bn<true, true, false, 3>(pl, A, lda, B, ldb, p, st, cg, ones);
  else if (im2col == 4)
    rc = s3 ? dispatch_bn<false, false, true, 4>(pl, A, lda, B, ldb, p, st, cg)
            : dispatch_bn<false, false, false, 4>(pl, A, lda, B, ldb, p, st, cg);
  else
    rc = s3 ? dispatch_major<true>(pl, a_mn, b_mn ? 1 : 0, A, lda, B, ldb, p, st)
       : bkt == 64 ? dispatch_major<false, 64>(pl, a_mn, b_mn ? 1 : 0, A, lda, B, ldb, p, st)
                   : dispatch_major<false>(pl, a_mn, b_mn ? 1 : 0, A, lda, B, ldb, p, st);
  if (rc) return rc;
  if (pl.splits > 1) {
    Params q = p;
    q.C = C;
    q.ldc = ldc;
    q.transpose_c = (im2col == 3 || im2col == 4);
    rc = launch_splitk_reduce(workspace, pl.splits, M, N, q, st);
  }
  return rc;
}

}  // namespace gemm

extern "C" {

long long omni_gemm_plan(int precision, int M, int N, int K, int a_mn_major, int b_mn_major,
                         int* splits, int* bn) {
  (void)a_mn_major;
  if (M < 1 || N < 1 || K < 1) return -1;
  if (precision == OMNI_PREC_FP32_SIMT) {
    if (splits) *splits = 1;
    if (bn) *bn = 16;
    return 0;
  }
  const gemm::Plan pl = gemm::plan_for(precision, M, N, K, b_mn_major != 0, 0);
  if (splits) *splits = pl.splits;
  if (bn) *bn = pl.bn;
  return pl.splits > 1 ? (long long)pl.splits * M * N * 4 : 0;
}

int omni_gemm_f32(int precision, int M, int N, int K, const float* A, long long lda,
                  int a_mn_major, const float* B, long long ldb, int b_mn_major, float* C,
                  long long ldc, int epilogue, const float* bias, const float* aux,
                  long long ld_aux, float* workspace, long long ws_bytes, void* stream) {
  OMNI_REQUIRE(M >= 1 && N >= 1 && K >= 1, "gemm: empty problem (M=%d N=%d K=%d)", M, N, K);
  OMNI_REQUIRE(precision >= 0 && precision <= 2, "gemm: unknown precision %d", precision);
  OMNI_REQUIRE(epilogue >= 0 && epilogue <= 5, "gemm: unknown epilogue %d", epilogue);
  OMNI_REQUIRE(lda >= (a_mn_major ? M : K) && ldb >= (b_mn_major ? N : K) && ldc >= N,
               "gemm: leading dimension too small (lda=%lld ldb=%lld ldc=%lld)", lda, ldb, ldc);
  OMNI_REQUIRE(!(epilogue == OMNI_EPI_BIAS || epilogue == OMNI_EPI_BIAS_RELU) || bias,
               "gemm: bias epilogue needs a bias vector");
  OMNI_REQUIRE(epilogue != OMNI_EPI_MASK_AUX || (aux && ld_aux >= N),
               "gemm: mask epilogue needs aux");
  cudaStream_t st = omni::as_stream(stream);
  if (precision == OMNI_PREC_FP32_SIMT) {
    gemm::Params p{};
    p.M = M;
    p.N = N;
    p.K = K;
    p.epilogue = epilogue;
    p.bias = bias;
    p.aux = aux;
    p.ld_aux = ld_aux;
    p.C = C;
    p.ldc = ldc;
    dim3 grid((unsigned)omni::ceil_div(N, 16), (unsigned)omni::ceil_div(M, 16));
    if (!a_mn_major && !b_mn_major)
      gemm::simt_gemm_kernel<false, false><<<grid, 256, 0, st>>>(A, lda, B, ldb, p);
    else if (!a_mn_major && b_mn_major)
      gemm::simt_gemm_kernel<false, true><<<grid, 256, 0, st>>>(A, lda, B, ldb, p);
    else if (a_mn_major && !b_mn_major)
      gemm::simt_gemm_kernel<true, false><<<grid, 256, 0, st>>>(A, lda, B, ldb, p);
    else
      gemm::simt_gemm_kernel<true, true><<<grid, 256, 0, st>>>(A, lda, B, ldb, p);
    return omni::check_launch("gemm_simt");
  }
  OMNI_REQUIRE(lda % 4 == 0 && ldb % 4 == 0,
               "gemm: lda/ldb must be multiples of 4 for TMA (lda=%lld ldb=%lld)", lda, ldb);
  OMNI_REQUIRE(((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0,
               "gemm: A and B must be 16-byte aligned for TMA");
  return gemm::run_gemm(precision, M, N, K, A, lda, a_mn_major, B, ldb, b_mn_major, C, ldc,
                        epilogue, bias, aux, ld_aux, workspace, ws_bytes, st, nullptr, 0);
}

// The transposed form trades 128 x d_out tiles for 128-row weight tiles against
// 256-pixel im2col boxes; its C^T epilogue store only pays off over a long
// reduction (conv2's data gradient: K = 6400 -> 615 TFLOP/s; CaffeNet conv1,
// K = 576, is faster untransposed).
static bool conv_fprop_transposed(int d_out, int pixels, int K) {
  static const bool off = getenv("OMNI_NO_TRANSPOSED_FPROP") != nullptr;
  static const bool force = getenv("OMNI_FORCE_TRANSPOSED_FPROP") != nullptr;   // tuning probe
  return !off && d_out <= 128 && pixels >= 128 * 148 && (K >= 2048 || force);
}

static int conv_shape(int op, int b, int n, int c, int k, int stride, int pad, int d_out, int* M,
                      int* N, int* K, int* m) {
  OMNI_REQUIRE(op == OMNI_CONV_FPROP || op == OMNI_CONV_WGRAD || op == OMNI_CONV_WGRAD_BIAS,
               "conv: unknown op %d", op);
  OMNI_REQUIRE(b >= 1 && n >= 1 && k >= 1 && stride >= 1 && pad >= 0 && d_out >= 1,
               "n, k, d_in, d_out, stride must be positive");
  OMNI_REQUIRE(c >= 1, "implicit conv needs d_in >= 1");
  // channels run in 32-wide im2col blocks: a partial last block reads the
  // missing channels as zeros (TMA out-of-bounds fill), so the GEMM's K index
  // per filter tap -- and the weight / weight-gradient rows -- are
  // round_up(d_in, 32) wide
  const int cpad = (c + 31) / 32 * 32;
  OMNI_REQUIRE(k <= n + 2 * pad && (n + 2 * pad - k) % stride == 0, "conv: bad geometry");
  OMNI_REQUIRE(pad <= 127 && k - 1 - pad <= 128, "conv: padding outside the im2col box range");
  *m = (n + 2 * pad - k) / stride + 1;
  const long long pix = (long long)b * (*m) * (*m);
  OMNI_REQUIRE(pix < (1LL << 31), "conv: too many output pixels");
  if (op == OMNI_CONV_FPROP) {
    *M = (int)pix;
    *N = d_out;
    *K = k * k * cpad;
  } else {
    *M = d_out;
    *N = k * k * cpad;
    *K = (int)pix;
  }
  return OMNI_OK;
}

long long omni_conv_implicit_plan(int precision, int op, int b, int n, int c, int k, int stride,
                                  int pad, int d_out) {
  int M, N, K, m;
  if (conv_shape(op, b, n, c, k, stride, pad, d_out, &M, &N, &K, &m)) return -1;
  // exactly the plans omni_conv_implicit_f32 launches
  if (op != OMNI_CONV_FPROP) {
    const int rows = op == OMNI_CONV_WGRAD_BIAS ? N + 1 : N;
    const gemm::Plan pl = gemm::plan_for(precision, rows, M, K, true, 3);
    return (op == OMNI_CONV_WGRAD_BIAS ? gemm::kOnesBytes : 0) +
           (pl.splits > 1 ? (long long)pl.splits * rows * M * 4 : 0);
  }
  const gemm::Plan pl = conv_fprop_transposed(d_out, M, K) ? gemm::plan_for(precision, N, M, K, false, 4)
                                                           : gemm::plan_for(precision, M, N, K, false, 1);
  return pl.splits > 1 ? (long long)pl.splits * M * N * 4 : 0;
}

int omni_conv_implicit_f32(int precision, int op, const float* X, int b, int n, int c, int cs,
                           int k, int stride, int pad, int d_out, const float* G, long long ldg,
                           float* Y, long long ldy, int epilogue, const float* bias,
                           const float* aux, long long ld_aux, float* workspace,
                           long long ws_bytes, void* stream) {
  int M, N, K, m;
  int rc = conv_shape(op, b, n, c, k, stride, pad, d_out, &M, &N, &K, &m);
  if (rc) return rc;
  OMNI_REQUIRE(precision == OMNI_PREC_TF32 || precision == OMNI_PREC_3XTF32,
               "conv: precision must be TF32 or 3xTF32");
  OMNI_REQUIRE(cs >= c && cs % 4 == 0 && ((uintptr_t)X & 15) == 0,
               "conv: X must be 16-byte aligned NHWC with cs %% 4 == 0");
  OMNI_REQUIRE(ldg % 4 == 0 && ((uintptr_t)G & 15) == 0, "conv: G must be 16-byte aligned, ldg %% 4 == 0");
  const bool with_bias = op == OMNI_CONV_WGRAD_BIAS;
  OMNI_REQUIRE(ldg >= (op == OMNI_CONV_FPROP ? K : d_out) && ldy >= N + (with_bias ? 1 : 0),
               "conv: leading dimension too small");
  OMNI_REQUIRE(epilogue >= 0 && epilogue <= 5, "conv: unknown epilogue %d", epilogue);
  OMNI_REQUIRE(!(epilogue == OMNI_EPI_BIAS || epilogue == OMNI_EPI_BIAS_RELU) || bias,
               "conv: bias epilogue needs a bias vector");
  OMNI_REQUIRE(epilogue != OMNI_EPI_MASK_AUX || (aux && ld_aux >= N), "conv: mask epilogue needs aux");
  gemm::ConvGeom cg{X, b, n, c, cs, k, stride, pad, m};
  cudaStream_t st = omni::as_stream(stream);
  if (op == OMNI_CONV_FPROP && conv_fprop_transposed(d_out, M, K))
    // few output channels: C^T = W im2col^T, im2col as the K-major B operand in
    // 256-pixel boxes (48 KB per 512 MMA cycles instead of 28 KB per 192 with
    // 128 x d_out tiles); epilogue stores C^T back into NHWC rows
    return gemm::run_gemm(precision, N, M, K, G, ldg, 0, nullptr, 0, 0, Y, ldy, epilogue, bias, aux,
                          ld_aux, workspace, ws_bytes, st, &cg, 4);
  if (op == OMNI_CONV_FPROP)   // A = im2col(X) (K-major), B = G weights (d_out x ldg, K-major)
    return gemm::run_gemm(precision, M, N, K, nullptr, 0, 0, G, ldg, 0, Y, ldy, epilogue, bias, aux,
                          ld_aux, workspace, ws_bytes, st, &cg, 1);
  // WGRAD: computed as C^T = im2col(X)^T dY with im2col as the MN-major A
  // operand (128 (tap, ch) rows = 128 im2col pixel-rows per stage, half of what
  // the B-side form needs) and dY (pixels x ldg) as the MN-major B operand;
  // the epilogue stores C^T, i.e. Y[o*ldy + (tap, ch)].
  OMNI_REQUIRE(epilogue == OMNI_EPI_STORE, "conv wgrad supports the plain store epilogue only");
  const float* ones = nullptr;
  if (with_bias) {
    // one more GEMM row (tap*c index k*k*c) fed by a ones chunk: the bias gradient
    OMNI_REQUIRE(workspace && ws_bytes >= gemm::kOnesBytes && ((uintptr_t)workspace & 15) == 0,
                 "conv wgrad+bias: workspace of at least %d bytes required", gemm::kOnesBytes);
    ones = gemm::ones_tile();
    OMNI_REQUIRE(ones, "conv wgrad+bias: ones tile address unavailable");
    workspace += gemm::kOnesBytes / 4;
    ws_bytes -= gemm::kOnesBytes;
  }
  return gemm::run_gemm(precision, N + (with_bias ? 1 : 0), M, K, nullptr, 0, 1, G, ldg, 1, Y, ldy,
                        epilogue, bias, aux, ld_aux, workspace, ws_bytes, st, &cg, 3, ones);
}

}  // extern "C"
