// Bandwidth-bound kernels of the CNN cascade: pooling (K3), softmax
// cross-entropy (K4), ReLU, bias gradient (K7), fused momentum SGD (K8) and
// the batch gather (K9).  Every reduction is a fixed-order gather or a
// two-pass tree so results are bit-reproducible run to run (no atomics).
#include <math.h>
#include <stdlib.h>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// n / d for 0 <= n < 2^32 by one wide multiply: m = ceil(2^(32+s) / d) with
// s = ceil(log2 d); the rounding error stays below 1/d, so the quotient is
// exact (index math of the issue-bound pooling backward).
struct FastDiv {
  unsigned long long m;
  int shift;
  int d;
};
inline FastDiv fast_div(int d) {
  int s = 0;
  while ((1ll << s) < d) ++s;
  FastDiv f;
  f.m = (unsigned long long)((((unsigned __int128)1 << (32 + s)) + d - 1) / d);
  f.shift = 32 + s;
  f.d = d;
  return f;
}
__device__ __forceinline__ int fdiv(int n, const FastDiv& f) {
  return (int)(((unsigned __int128)(unsigned)n * f.m) >> f.shift);
}

__host__ __device__ inline int pool_out(int n, int k, int s, int p, int ceil_mode) {
  const int span = n + 2 * p - k;
  int out = (ceil_mode ? (span + s - 1) / s : span / s) + 1;
  // Caffe's rule: the last window must start inside the (left-padded) input.
  if (p > 0 && (out - 1) * s >= n + p) --out;
  return out;
}

// One thread per (img, oy, ox, channel group of V).  Max: first maximum in
// (dy, dx) order, argmax = iy*w + ix (problems.py:213-216).  Avg: Caffe
// divisor.  V = 4 uses float4/int4 accesses (c, cs_in, cs_out multiples of 4).
// mark (max): windows whose maximum is not > 0 get the argmax sign bit set,
// so a backward without a ReLU mask routes nothing there (mode 2 below).
template <int MODE, int V, int KS = 0>
__global__ void __launch_bounds__(kThreads) pool_fwd_kernel(
    const float* __restrict__ X, int b, int h, int w, int c, int cs_in, int k_rt, int s, int p,
    int oh, int ow, float* __restrict__ Y, int cs_out, int32_t* __restrict__ argmax, int mark) {
  const int k = KS ? KS : k_rt;   // KS > 0: fully unrolled window, all loads in flight
  const int cv = c / V;
  const int total = b * oh * ow * cv;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int opix = idx / cv;
    const int ch = (idx - opix * cv) * V;
    const int img = opix / (oh * ow);
    const int r = opix - img * oh * ow;
    const int oy = r / ow, ox = r - (r / ow) * ow;
    int hs = oy * s - p, ws = ox * s - p;
    int he = min(hs + k, h + p), we = min(ws + k, w + p);
    const float inv = 1.f / (float)((he - hs) * (we - ws));
    hs = max(hs, 0);
    ws = max(ws, 0);
    he = min(he, h);
    we = min(we, w);
    const float* Xi = X + (long long)img * h * w * cs_in + ch;
    float best[V], acc[V];
    int arg[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      best[v] = -INFINITY;
      acc[v] = 0.f;
      arg[v] = hs * w + ws;
    }
    bool first = true;
    if constexpr (KS > 0 && V == 4) {
      // every window element loaded up front in one basic block (an element
      // outside the clipped window reads the window's first element and is
      // skipped by the fold), then folded in (dy, dx) order exactly as below:
      // one exposed load latency per output instead of one per element
      const int ny = he - hs, nx = we - ws;
      float4 t[KS][KS];
#pragma unroll
      for (int dy = 0; dy < KS; ++dy)
#pragma unroll
        for (int dx = 0; dx < KS; ++dx) {
          const int iy = hs + (dy < ny ? dy : 0), ix = ws + (dx < nx ? dx : 0);
          t[dy][dx] = __ldg(reinterpret_cast<const float4*>(Xi + (iy * w + ix) * cs_in));
        }
#pragma unroll
      for (int dy = 0; dy < KS; ++dy)
#pragma unroll
        for (int dx = 0; dx < KS; ++dx) {
          if (dy >= ny || dx >= nx) continue;
          const float val[4] = {t[dy][dx].x, t[dy][dx].y, t[dy][dx].z, t[dy][dx].w};
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            if (MODE == 0) {
              if (first || val[v] > best[v]) {
                best[v] = val[v];
                arg[v] = (hs + dy) * w + (ws + dx);
              }
            } else {
              acc[v] += val[v];
            }
          }
          first = false;
        }
    } else {
#pragma unroll
    for (int dy = 0; dy < (KS ? KS : 1); ++dy) {
      for (int iy = (KS ? hs + dy : hs); iy < (KS ? min(hs + dy + 1, he) : he); ++iy)
#pragma unroll
        for (int dx = 0; dx < (KS ? KS : 1); ++dx) {
          for (int ix = (KS ? ws + dx : ws); ix < (KS ? min(ws + dx + 1, we) : we); ++ix) {
            const float* src = Xi + (iy * w + ix) * cs_in;
            float val[V];
            if (V == 4) {
              const float4 t = __ldg(reinterpret_cast<const float4*>(src));
              val[0] = t.x; val[1 % V] = t.y; val[2 % V] = t.z; val[3 % V] = t.w;
            } else {
              val[0] = __ldg(src);
            }
#pragma unroll
            for (int v = 0; v < V; ++v) {
              if (MODE == 0) {
                if (first || val[v] > best[v]) {
                  best[v] = val[v];
                  arg[v] = iy * w + ix;
                }
              } else {
                acc[v] += val[v];
              }
            }
            first = false;
          }
        }
    }
    }
    float* dst = Y + (long long)opix * cs_out + ch;
    if (MODE == 0 && mark) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (!(best[v] > 0.f)) arg[v] |= (int)0x80000000;
    }
    if (MODE == 0) {
      if (V == 4) {
        *reinterpret_cast<float4*>(dst) = make_float4(best[0], best[1 % V], best[2 % V], best[3 % V]);
        *reinterpret_cast<int4*>(argmax + (long long)opix * c + ch) =
            make_int4(arg[0], arg[1 % V], arg[2 % V], arg[3 % V]);
      } else {
        dst[0] = best[0];
        argmax[(long long)opix * c + ch] = arg[0];
      }
    } else {
      if (V == 4)
        *reinterpret_cast<float4*>(dst) =
            make_float4(acc[0] * inv, acc[1 % V] * inv, acc[2 % V] * inv, acc[3 % V] * inv);
      else
        dst[0] = acc[0] * inv;
    }
  }
}

// Gather-form backward: each input pixel sums the output gradients of the
// windows that contain it, in ascending (oy, ox) order; fused ReLU mask.
template <int MODE, int V>
__global__ void __launch_bounds__(kThreads) pool_bwd_kernel(
    const float* __restrict__ dY, int b, int h, int w, int c, int cs_in, int k, int s, int p,
    int oh, int ow, int cs_out, const int32_t* __restrict__ argmax, const float* __restrict__ X,
    int relu_mask_x, float* __restrict__ dX) {
  const int cv = c / V;
  const int total = b * h * w * cv;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int pix = idx / cv;
    const int ch = (idx - pix * cv) * V;
    const int img = pix / (h * w);
    const int r = pix - img * h * w;
    const int iy = r / w, ix = r - (r / w) * w;
    const int oy0 = (iy + p < k) ? 0 : (iy + p - k) / s + 1;
    const int oy1 = min((iy + p) / s + 1, oh);
    const int ox0 = (ix + p < k) ? 0 : (ix + p - k) / s + 1;
    const int ox1 = min((ix + p) / s + 1, ow);
    const int obase = img * oh * ow;
    const int me = iy * w + ix;
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.f;
    for (int oy = oy0; oy < oy1; ++oy)
      for (int ox = ox0; ox < ox1; ++ox) {
        const int o = obase + oy * ow + ox;
        float g[V];
        if (V == 4) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(dY + (long long)o * cs_out + ch));
          g[0] = t.x; g[1 % V] = t.y; g[2 % V] = t.z; g[3 % V] = t.w;
        } else {
          g[0] = __ldg(dY + (long long)o * cs_out + ch);
        }
        if (MODE == 0) {
          int a[V];
          if (V == 4) {
            const int4 t = __ldg(reinterpret_cast<const int4*>(argmax + (long long)o * c + ch));
            a[0] = t.x; a[1 % V] = t.y; a[2 % V] = t.z; a[3 % V] = t.w;
          } else {
            a[0] = __ldg(argmax + (long long)o * c + ch);
          }
          if (relu_mask_x == 2) {  // X holds the pooled output: mask by the window max
            if (V == 4) {
              const float4 t = __ldg(reinterpret_cast<const float4*>(X + (long long)o * cs_out + ch));
              g[0] = t.x > 0.f ? g[0] : 0.f;
              g[1 % V] = t.y > 0.f ? g[1 % V] : 0.f;
              g[2 % V] = t.z > 0.f ? g[2 % V] : 0.f;
              g[3 % V] = t.w > 0.f ? g[3 % V] : 0.f;
            } else {
              g[0] = __ldg(X + (long long)o * cs_out + ch) > 0.f ? g[0] : 0.f;
            }
          }
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (a[v] == me) acc[v] += g[v];
        } else {
          const int hs = oy * s - p, ws = ox * s - p;
          const int he = min(hs + k, h + p), we = min(ws + k, w + p);
          const float inv = 1.f / (float)((he - hs) * (we - ws));
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v] += g[v] * inv;
        }
      }
    float* dst = dX + (long long)pix * cs_in + ch;
    if (relu_mask_x == 1) {
      const float* xm = X + (long long)pix * cs_in + ch;
      if (V == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(xm));
        acc[0] = t.x > 0.f ? acc[0] : 0.f;
        acc[1 % V] = t.y > 0.f ? acc[1 % V] : 0.f;
        acc[2 % V] = t.z > 0.f ? acc[2 % V] : 0.f;
        acc[3 % V] = t.w > 0.f ? acc[3 % V] : 0.f;
      } else {
        acc[0] = __ldg(xm) > 0.f ? acc[0] : 0.f;
      }
    }
    if (V == 4)
      *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1 % V], acc[2 % V], acc[3 % V]);
    else
      dst[0] = acc[0];
  }
}

// Stride-2 backward: one thread per 2x2 input block x 4 channels.  The four
// pixels of an aligned 2x2 block are covered by the same <= (k/2+1)^2 windows,
// so each window's dY and argmax are read once per block instead of once per
// pixel.  Per pixel the windows are still summed in ascending (oy, ox) order:
// bit-identical to pool_bwd_kernel.
// RM = relu_mask_x (compile time: the register budget follows the loads it needs).
template <int MODE, int RM>
__global__ void __launch_bounds__(kThreads) pool_bwd_s2_kernel(
    const float* __restrict__ dY, int b, int h, int w, int c, int cs_in, int k, int p, int oh,
    int ow, int cs_out, const int32_t* __restrict__ argmax, const float* __restrict__ X,
    float* __restrict__ dX, FastDiv dcv, FastDiv dbhw, FastDiv dbw) {
  constexpr int relu_mask_x = RM;
  const int cv = c / 4;
  const int bh = (h + 1) / 2, bw = (w + 1) / 2;
  const int total = b * bh * bw * cv;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int blk = fdiv(idx, dcv);
    const int ch = (idx - blk * cv) * 4;
    const int img = fdiv(blk, dbhw);
    const int r = blk - img * bh * bw;
    const int by = fdiv(r, dbw), bx = r - by * bw;
    const int y0 = 2 * by, x0 = 2 * bx;
    const int y1 = min(y0 + 1, h - 1), x1 = min(x0 + 1, w - 1);
    const int oy0 = (y0 + p < k) ? 0 : (y0 + p - k) / 2 + 1;
    const int oy1 = min((y1 + p) / 2 + 1, oh);
    const int ox0 = (x0 + p < k) ? 0 : (x0 + p - k) / 2 + 1;
    const int ox1 = min((x1 + p) / 2 + 1, ow);
    float acc[2][2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[a][e][v] = 0.f;
    const int obase = img * oh * ow;
    // at stride 2 with k <= 3 (or k = 4, even pad) at most 2 x 2 windows cover an
    // aligned 2x2 block: a fixed, unrolled candidate set whose loads are all
    // issued up front (a candidate outside [oy0, oy1) x [ox0, ox1) reads a
    // clamped in-range window and is skipped below)
    float4 gq[2][2], yq[2][2];
    int4 aq[2][2];
#pragma unroll
    for (int ty = 0; ty < 2; ++ty)
#pragma unroll
      for (int tx = 0; tx < 2; ++tx) {
        const int o = obase + min(oy0 + ty, oh - 1) * ow + min(ox0 + tx, ow - 1);
        gq[ty][tx] = __ldg(reinterpret_cast<const float4*>(dY + (long long)o * cs_out + ch));
        if (MODE == 0) {
          aq[ty][tx] = __ldg(reinterpret_cast<const int4*>(argmax + (long long)o * c + ch));
          if (relu_mask_x == 2)
            yq[ty][tx] = __ldg(reinterpret_cast<const float4*>(X + (long long)o * cs_out + ch));
        }
      }
#pragma unroll
    for (int ty = 0; ty < 2; ++ty)
#pragma unroll
      for (int tx = 0; tx < 2; ++tx) {
        const int oy = oy0 + ty, ox = ox0 + tx;
        if (oy >= oy1 || ox >= ox1) continue;
        const float4 g = gq[ty][tx];
        const float gv[4] = {g.x, g.y, g.z, g.w};
        if (MODE == 0) {
          const int4 t = aq[ty][tx];
          const int av[4] = {t.x, t.y, t.z, t.w};
          float gm[4] = {gv[0], gv[1], gv[2], gv[3]};
          if (relu_mask_x == 2) {  // X holds the pooled output: mask by the window max
            const float4 y = yq[ty][tx];
            gm[0] = y.x > 0.f ? gm[0] : 0.f;
            gm[1] = y.y > 0.f ? gm[1] : 0.f;
            gm[2] = y.z > 0.f ? gm[2] : 0.f;
            gm[3] = y.w > 0.f ? gm[3] : 0.f;
          }
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int me = (y0 + a) * w + (x0 + e);
#pragma unroll
              for (int v = 0; v < 4; ++v)
                if (av[v] == me) acc[a][e][v] += gm[v];
            }
        } else {
          const int hs = oy * 2 - p, ws = ox * 2 - p;
          const int he = min(hs + k, h + p), we = min(ws + k, w + p);
          const float inv = 1.f / (float)((he - hs) * (we - ws));
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int yy = y0 + a, xx = x0 + e;
              if (yy >= hs && yy < hs + k && xx >= ws && xx < ws + k)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[a][e][v] += gv[v] * inv;
            }
        }
      }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int yy = y0 + a, xx = x0 + e;
        if (yy >= h || xx >= w) continue;
        const long long pix = (long long)img * h * w + (long long)yy * w + xx;
        float4 out = make_float4(acc[a][e][0], acc[a][e][1], acc[a][e][2], acc[a][e][3]);
        if (relu_mask_x == 1) {
          const float4 m = __ldg(reinterpret_cast<const float4*>(X + pix * cs_in + ch));
          out.x = m.x > 0.f ? out.x : 0.f;
          out.y = m.y > 0.f ? out.y : 0.f;
          out.z = m.z > 0.f ? out.z : 0.f;
          out.w = m.w > 0.f ? out.w : 0.f;
        }
        *reinterpret_cast<float4*>(dX + pix * cs_in + ch) = out;
      }
  }
}

// Softmax cross-entropy, one warp per row.
// Launched as ONE cluster of kSoftmaxCtas CTAs (32 warps each): global warp
// g = rank*32 + warp owns rows g, g + 32*kSoftmaxCtas, ...; each CTA sums its
// warps in order, then CTA 0 sums the CTA partials in rank order through
// distributed shared memory -- a fixed tree, so the loss is bit-reproducible.
constexpr int kSoftmaxCtas = 8;
__global__ void __launch_bounds__(1024) softmax_xent_kernel(
    const float* __restrict__ Z, long long ld, const int32_t* __restrict__ y, int b, int C,
    float* __restrict__ loss, float* __restrict__ dZ, long long ldd, float scale) {
  __shared__ float warp_loss[32];
  __shared__ float cta_loss;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int gwarp = (int)rank * 32 + warp, nwarps = 32 * (int)gridDim.x;
  float my_loss = 0.f;
  if (C <= 1024) {
    // each lane keeps its <= 32 logits in registers: one batch of independent
    // loads per row instead of three dependent sweeps over memory
    for (int row = gwarp; row < b; row += nwarps) {
      const float* z = Z + (long long)row * ld;
      float v[32];
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int j = lane + 32 * i;
        v[i] = j < C ? __ldg(z + j) : -INFINITY;
        mx = fmaxf(mx, v[i]);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        v[i] = (lane + 32 * i) < C ? expf(v[i] - mx) : 0.f;
        sum += v[i];
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const int label = y[row];
      if (lane == 0) my_loss += (logf(sum) + mx) - z[label];
      if (dZ) {
        const float inv = 1.f / sum;
        float* d = dZ + (long long)row * ldd;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int j = lane + 32 * i;
          if (j < C) d[j] = (v[i] * inv - (j == label ? 1.f : 0.f)) * scale;
        }
      }
    }
  } else
  for (int row = gwarp; row < b; row += nwarps) {
    const float* z = Z + (long long)row * ld;
    float mx = -INFINITY;
    for (int j = lane; j < C; j += 32) mx = fmaxf(mx, z[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int j = lane; j < C; j += 32) sum += expf(z[j] - mx);
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const int label = y[row];
    if (lane == 0) my_loss += (logf(sum) + mx) - z[label];
    if (dZ) {
      const float inv = 1.f / sum;
      float* d = dZ + (long long)row * ldd;
      for (int j = lane; j < C; j += 32) {
        float pj = expf(z[j] - mx) * inv;
        if (j == label) pj -= 1.f;
        d[j] = pj * scale;
      }
    }
  }
  if (lane == 0) warp_loss[warp] = my_loss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int i = 0; i < 32; ++i) tot += warp_loss[i];
    cta_loss = tot;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(&cta_loss);
    float tot = 0.f;
    for (unsigned r = 0; r < gridDim.x; ++r) {
      uint32_t remote;
      float v;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
      tot += v;
    }
    loss[0] = tot / (float)b;
  }
  // keep every CTA's shared memory alive until CTA 0 has read it
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}

__global__ void __launch_bounds__(kThreads) relu_fwd_kernel(const float* __restrict__ X,
                                                             float* __restrict__ Y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    Y[i] = fmaxf(X[i], 0.f);
}

__global__ void __launch_bounds__(kThreads) relu_bwd_kernel(const float* __restrict__ dY,
                                                             const float* __restrict__ Y,
                                                             float* __restrict__ dX, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dX[i] = Y[i] > 0.f ? dY[i] : 0.f;
}

// Bias gradient pass 1: block (g, cb) sums rows [g*rpb, (g+1)*rpb) of columns
// [cb*32, cb*32+32); 8 row-lanes per column, combined in lane order.
__global__ void __launch_bounds__(256) bias_grad_pass1(const float* __restrict__ dY,
                                                       long long ld, int M, int N, int rpb,
                                                       float* __restrict__ ws) {
  __shared__ float part[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int col = blockIdx.y * 32 + tx;
  const long long r0 = (long long)blockIdx.x * rpb;
  const long long r1 = min((long long)M, r0 + rpb);
  float acc = 0.f;
  if (col < N)
    for (long long r = r0 + ty; r < r1; r += 8) acc += dY[r * ld + col];
  part[ty][tx] = acc;
  __syncthreads();
  if (ty == 0 && col < N) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += part[i][tx];
    ws[(long long)blockIdx.x * N + col] = s;
  }
}

// Pass 2: one warp per column; lane l sums partials l, l+32, ... then a fixed
// xor-shuffle tree -- deterministic, and G loads in flight instead of a chain.
__global__ void __launch_bounds__(256) bias_grad_pass2(const float* __restrict__ ws, int G, int N,
                                                       float* __restrict__ db) {
  const int lane = threadIdx.x & 31;
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (col >= N) return;
  float s = 0.f;
  for (int g = lane; g < G; g += 32) s += ws[(long long)g * N + col];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) db[col] = s;
}

inline void bias_grad_geometry(int M, int* G, int* rpb) {
  int r = (M + 295) / 296;  // about two row chunks per SM
  if (r < 64) r = 64;
  *rpb = r;
  *G = (M + r - 1) / r;
  if (*G < 1) *G = 1;
}

// V = mu*V - eta*(g + lam*w_read); W = W + V   (sgd.py:100-101), float4 body.
__global__ void __launch_bounds__(kThreads) sgd_kernel(float* __restrict__ W, float* __restrict__ V,
                                                       const float* __restrict__ g,
                                                       const float* w_read, float eta, float mu,
                                                       float lam, long long n) {
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    const float4 wr = reinterpret_cast<const float4*>(w_read)[i];
    float4 v = reinterpret_cast<float4*>(V)[i];
    float4 w = reinterpret_cast<float4*>(W)[i];
    v.x = mu * v.x - eta * (gv.x + lam * wr.x);
    v.y = mu * v.y - eta * (gv.y + lam * wr.y);
    v.z = mu * v.z - eta * (gv.z + lam * wr.z);
    v.w = mu * v.w - eta * (gv.w + lam * wr.w);
    w.x += v.x; w.y += v.y; w.z += v.z; w.w += v.w;
    reinterpret_cast<float4*>(V)[i] = v;
    reinterpret_cast<float4*>(W)[i] = w;
  }
  for (long long i = n4 * 4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const float v = mu * V[i] - eta * (g[i] + lam * w_read[i]);
    V[i] = v;
    W[i] = W[i] + v;
  }
}

__global__ void __launch_bounds__(kThreads) sgd_kernel_scalar(float* W, float* V,
                                                              const float* __restrict__ g,
                                                              const float* w_read, float eta,
                                                              float mu, float lam, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = mu * V[i] - eta * (g[i] + lam * w_read[i]);
    V[i] = v;
    W[i] = W[i] + v;
  }
}

// The g ordered updates of one compute-group round on a shard (groups.py):
// row m of `rows` is rank m's gradient shard; group i's gradient is the sum of
// its k members' rows in member order, applied with the group's snapshot as
// the regulariser's w_read (sgd.py:104-112), and W after update i becomes
// group i's next snapshot.  One pass over the shard instead of g*(k+2) eager
// launches; the per-element arithmetic is sgd_kernel's.
constexpr int kMaxGroupRanks = 64;
struct GroupUpdates {
  const float* rows;
  long long ld;
  float* W;
  float* V;
  float* snaps[kMaxGroupRanks];
  int members[kMaxGroupRanks];
  int g, k;
  float eta, mu, lam;
};

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

__global__ void __launch_bounds__(kThreads) group_updates_kernel(const __grid_constant__ GroupUpdates p,
                                                                 long long n, int vec) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const float eta = p.eta, mu = p.mu, lam = p.lam;
  if (vec) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += stride) {
      float4 w = reinterpret_cast<const float4*>(p.W)[i];
      float4 v = reinterpret_cast<const float4*>(p.V)[i];
      for (int gi = 0; gi < p.g; ++gi) {
        const int* mem = p.members + gi * p.k;
        float4 gv = reinterpret_cast<const float4*>(p.rows + mem[0] * p.ld)[i];
        for (int j = 1; j < p.k; ++j)
          gv = f4add(gv, reinterpret_cast<const float4*>(p.rows + mem[j] * p.ld)[i]);
        float4* sp = reinterpret_cast<float4*>(p.snaps[gi]) + i;
        const float4 wr = *sp;
        v.x = mu * v.x - eta * (gv.x + lam * wr.x);
        v.y = mu * v.y - eta * (gv.y + lam * wr.y);
        v.z = mu * v.z - eta * (gv.z + lam * wr.z);
        v.w = mu * v.w - eta * (gv.w + lam * wr.w);
        w.x += v.x; w.y += v.y; w.z += v.z; w.w += v.w;
        *sp = w;
      }
      reinterpret_cast<float4*>(p.V)[i] = v;
      reinterpret_cast<float4*>(p.W)[i] = w;
    }
    return;
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float w = p.W[i], v = p.V[i];
    for (int gi = 0; gi < p.g; ++gi) {
      const int* mem = p.members + gi * p.k;
      float gv = p.rows[mem[0] * p.ld + i];
      for (int j = 1; j < p.k; ++j) gv = gv + p.rows[mem[j] * p.ld + i];
      const float wr = p.snaps[gi][i];
      v = mu * v - eta * (gv + lam * wr);
      w = w + v;
      p.snaps[gi][i] = w;
    }
    p.V[i] = v;
    p.W[i] = w;
  }
}

// float64 K8 for the drop-in host API (sgd.py:92-101 keeps W, V in float64):
// the reference's NumPy expression evaluated in its exact order, one rounding
// per operation and no FMA contraction (the _rn intrinsics), so the result is
// bit-identical to  V' = mu*V - eta*(g + lam*w);  W' = W + V'.
__global__ void __launch_bounds__(kThreads) sgd_kernel_f64(double* W, double* V,
                                                           const double* __restrict__ g,
                                                           const double* w_read, double eta,
                                                           double mu, double lam, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double reg = __dadd_rn(g[i], __dmul_rn(lam, w_read[i]));
    const double v = __dsub_rn(__dmul_rn(mu, V[i]), __dmul_rn(eta, reg));
    V[i] = v;
    W[i] = __dadd_rn(W[i], v);
  }
}

// One block-stride loop per gathered row: no per-element division.
template <bool VEC4>
__global__ void __launch_bounds__(kThreads) gather_rows_kernel(const float* __restrict__ src,
                                                               long long row_elems,
                                                               const int64_t* __restrict__ idx,
                                                               int nidx, float* __restrict__ dst) {
  const long long per = VEC4 ? row_elems / 4 : row_elems;
  for (int i = blockIdx.y; i < nidx; i += gridDim.y) {
    const long long srow = idx[i];
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < per;
         j += (long long)gridDim.x * blockDim.x) {
      if (VEC4)
        reinterpret_cast<float4*>(dst)[i * per + j] =
            __ldg(reinterpret_cast<const float4*>(src) + srow * per + j);
      else
        dst[i * per + j] = __ldg(src + srow * per + j);
    }
  }
}

__global__ void gather_i32_kernel(const int32_t* __restrict__ src, const int64_t* __restrict__ idx,
                                  int nidx, int32_t* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nidx; i += gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void fill_kernel(float* X, float v, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    X[i] = v;
}

}  // namespace

extern "C" {

int omni_pool_out_size(int n, int k, int stride, int pad, int ceil_mode) {
  if (n < 1 || k < 1 || stride < 1 || pad < 0 || k > n + 2 * pad) return -1;
  return pool_out(n, k, stride, pad, ceil_mode);
}

int omni_pool_fwd_nhwc_f32(int mode, const float* X, int b, int h, int w, int c, int cs_in, int k,
                           int stride, int pad, int ceil_mode, float* Y, int cs_out,
                           int32_t* argmax, void* stream) {
  OMNI_REQUIRE(mode >= 0 && mode <= 2, "pool: mode must be 0 (max), 1 (avg) or 2 (max, marked argmax)");
  OMNI_REQUIRE(b >= 0 && h >= 1 && w >= 1 && c >= 1 && k >= 1 && stride >= 1 && pad >= 0 &&
                   pad < k && k <= h + 2 * pad && k <= w + 2 * pad && cs_in >= c && cs_out >= c,
               "pool: bad geometry");
  const int mark = mode == 2 ? 1 : 0;
  if (mode == 2) mode = 0;
  OMNI_REQUIRE(mode == 1 || argmax != nullptr, "pool: max mode needs an argmax buffer");
  const int oh = pool_out(h, k, stride, pad, ceil_mode), ow = pool_out(w, k, stride, pad, ceil_mode);
  const long long work = (long long)b * oh * ow * c;
  if (work == 0) return OMNI_OK;
  OMNI_REQUIRE((long long)b * h * w * cs_in < (1LL << 31) && work < (1LL << 31),
               "pool: tensor too large for 32-bit indexing");
  cudaStream_t st = omni::as_stream(stream);
  const bool v4 = c % 4 == 0 && cs_in % 4 == 0 && cs_out % 4 == 0 && aligned16(X) && aligned16(Y) &&
                  (mode == 1 || aligned16(argmax));
  const int grid = omni::grid_for(v4 ? work / 4 : work, kThreads);
#define OMNI_POOL_FWD(M, V, KS) \
  pool_fwd_kernel<M, V, KS><<<grid, kThreads, 0, st>>>(X, b, h, w, c, cs_in, k, stride, pad, oh, ow, Y, cs_out, argmax, mark)
  if (mode == 0) {
    if (v4 && k == 3) OMNI_POOL_FWD(0, 4, 3);
    else if (v4) OMNI_POOL_FWD(0, 4, 0);
    else OMNI_POOL_FWD(0, 1, 0);
  } else {
    if (v4 && k == 3) OMNI_POOL_FWD(1, 4, 3);
    else if (v4) OMNI_POOL_FWD(1, 4, 0);
    else OMNI_POOL_FWD(1, 1, 0);
  }
#undef OMNI_POOL_FWD
  return omni::check_launch("pool_fwd");
}

int omni_pool_bwd_nhwc_f32(int mode, const float* dY, int b, int h, int w, int c, int cs_in, int k,
                           int stride, int pad, int ceil_mode, int cs_out, const int32_t* argmax,
                           const float* X, int relu_mask_x, float* dX, void* stream) {
  OMNI_REQUIRE(mode == 0 || mode == 1, "pool: mode must be 0 (max) or 1 (avg)");
  OMNI_REQUIRE(b >= 0 && h >= 1 && w >= 1 && c >= 1 && k >= 1 && stride >= 1 && pad >= 0 &&
                   pad < k && cs_in >= c && cs_out >= c,
               "pool: bad geometry");
  OMNI_REQUIRE(mode == 1 || argmax != nullptr, "pool: max mode needs the forward argmax");
  OMNI_REQUIRE(relu_mask_x >= 0 && relu_mask_x <= 2 && (!relu_mask_x || X != nullptr),
               "pool: relu mask needs X");
  OMNI_REQUIRE(relu_mask_x != 2 || mode == 0, "pool: relu_mask_x = 2 (mask by the output) is max-pool only");
  const int oh = pool_out(h, k, stride, pad, ceil_mode), ow = pool_out(w, k, stride, pad, ceil_mode);
  const long long work = (long long)b * h * w * c;
  if (work == 0) return OMNI_OK;
  OMNI_REQUIRE((long long)b * h * w * cs_in < (1LL << 31), "pool: tensor too large for 32-bit indexing");
  cudaStream_t st = omni::as_stream(stream);
  const bool v4 = c % 4 == 0 && cs_in % 4 == 0 && cs_out % 4 == 0 && aligned16(dY) && aligned16(dX) &&
                  (mode == 1 || aligned16(argmax)) && (!relu_mask_x || aligned16(X));  // X: cs_in or cs_out rows, both % 4
  // the blocked kernel visits 2 x 2 candidate windows per aligned 2x2 input
  // block: enough for k <= 3, and for k = 4 only with even padding (odd
  // padding puts a third window over the block)
  if (v4 && stride == 2 && (k <= 3 || (k == 4 && pad % 2 == 0)) && !getenv("OMNI_POOL_BWD_PIXEL")) {
    const long long blocks = (long long)b * ((h + 1) / 2) * ((w + 1) / 2) * (c / 4);
    const int g2 = omni::grid_for(blocks, kThreads);
    const FastDiv dcv = fast_div(c / 4), dbhw = fast_div(((h + 1) / 2) * ((w + 1) / 2)),
                  dbw = fast_div((w + 1) / 2);
#define OMNI_POOL_BWD_S2(M, R)                                                                    \
  pool_bwd_s2_kernel<M, R><<<g2, kThreads, 0, st>>>(dY, b, h, w, c, cs_in, k, pad, oh, ow, cs_out, argmax, \
                                                    X, dX, dcv, dbhw, dbw)
    if (mode == 0) {
      if (relu_mask_x == 2) OMNI_POOL_BWD_S2(0, 2);
      else if (relu_mask_x == 1) OMNI_POOL_BWD_S2(0, 1);
      else OMNI_POOL_BWD_S2(0, 0);
    } else {
      if (relu_mask_x == 1) OMNI_POOL_BWD_S2(1, 1);
      else OMNI_POOL_BWD_S2(1, 0);
    }
#undef OMNI_POOL_BWD_S2
    return omni::check_launch("pool_bwd_s2");
  }
  const int grid = omni::grid_for(v4 ? work / 4 : work, kThreads);
#define OMNI_POOL_BWD(M, V)                                                                     \
  pool_bwd_kernel<M, V><<<grid, kThreads, 0, st>>>(dY, b, h, w, c, cs_in, k, stride, pad, oh, ow, \
                                                   cs_out, argmax, X, relu_mask_x, dX)
  if (mode == 0) {
    if (v4) OMNI_POOL_BWD(0, 4); else OMNI_POOL_BWD(0, 1);
  } else {
    if (v4) OMNI_POOL_BWD(1, 4); else OMNI_POOL_BWD(1, 1);
  }
#undef OMNI_POOL_BWD
  return omni::check_launch("pool_bwd");
}

int omni_softmax_xent_f32(const float* logits, long long ld, const int32_t* labels, int b, int C,
                          float* loss, float* dlogits, long long ldd, float scale, void* stream) {
  OMNI_REQUIRE(b >= 1 && C >= 1 && ld >= C && (dlogits == nullptr || ldd >= C),
               "softmax_xent: bad shape");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kSoftmaxCtas);
  cfg.blockDim = dim3(1024);
  cfg.stream = omni::as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kSoftmaxCtas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OMNI_CUDA_TRY(cudaLaunchKernelEx(&cfg, softmax_xent_kernel, logits, ld, labels, b, C, loss,
                                   dlogits, ldd, scale));
  return omni::check_launch("softmax_xent");
}

int omni_relu_fwd_f32(const float* X, float* Y, long long n, void* stream) {
  if (n <= 0) return OMNI_OK;
  relu_fwd_kernel<<<omni::grid_for(n, kThreads), kThreads, 0, omni::as_stream(stream)>>>(X, Y, n);
  return omni::check_launch("relu_fwd");
}

int omni_relu_bwd_f32(const float* dY, const float* Y, float* dX, long long n, void* stream) {
  if (n <= 0) return OMNI_OK;
  relu_bwd_kernel<<<omni::grid_for(n, kThreads), kThreads, 0, omni::as_stream(stream)>>>(dY, Y, dX,
                                                                                       n);
  return omni::check_launch("relu_bwd");
}

long long omni_bias_grad_ws_elems(int M, int N) {
  int G, rpb;
  bias_grad_geometry(M, &G, &rpb);
  return (long long)G * N;
}

int omni_bias_grad_f32(const float* dY, long long ld, int M, int N, float* db, float* ws,
                       void* stream) {
  OMNI_REQUIRE(M >= 1 && N >= 1 && ld >= N, "bias_grad: bad shape");
  int G, rpb;
  bias_grad_geometry(M, &G, &rpb);
  cudaStream_t st = omni::as_stream(stream);
  bias_grad_pass1<<<dim3(G, (N + 31) / 32), 256, 0, st>>>(dY, ld, M, N, rpb, ws);
  int rc = omni::check_launch("bias_grad_pass1");
  if (rc) return rc;
  bias_grad_pass2<<<(N * 32 + 255) / 256, 256, 0, st>>>(ws, G, N, db);
  return omni::check_launch("bias_grad_pass2");
}

int omni_sgd_momentum_f32(float* W, float* V, const float* g, const float* w_read, float eta,
                          float mu, float lam, long long n, void* stream) {
  OMNI_REQUIRE(n >= 0, "sgd: negative length");
  if (n == 0) return OMNI_OK;
  cudaStream_t st = omni::as_stream(stream);
  if (aligned16(W) && aligned16(V) && aligned16(g) && aligned16(w_read))
    sgd_kernel<<<omni::grid_for((n + 3) / 4, kThreads), kThreads, 0, st>>>(W, V, g, w_read, eta,
                                                                          mu, lam, n);
  else
    sgd_kernel_scalar<<<omni::grid_for(n, kThreads), kThreads, 0, st>>>(W, V, g, w_read, eta, mu,
                                                                       lam, n);
  return omni::check_launch("sgd_momentum");
}

int omni_group_updates_f32(const float* rows, int nrows, long long ld, const int* members, int g, int k,
                           float* W, float* V, float* const* snaps, long long n, float eta,
                           float mu, float lam, void* stream) {
  OMNI_REQUIRE(n >= 0 && g >= 1 && k >= 1 && g * k <= kMaxGroupRanks,
               "group_updates: need n >= 0, 1 <= g*k <= 64");
  OMNI_REQUIRE(rows && members && W && V && snaps, "group_updates: NULL argument");
  OMNI_REQUIRE(ld >= n, "group_updates: row pitch ld < n");
  if (n == 0) return OMNI_OK;
  GroupUpdates p{};
  p.rows = rows;
  p.ld = ld;
  p.W = W;
  p.V = V;
  p.g = g;
  p.k = k;
  p.eta = eta;
  p.mu = mu;
  p.lam = lam;
  bool vec = aligned16(rows) && aligned16(W) && aligned16(V) && ld % 4 == 0 && n % 4 == 0;
  for (int i = 0; i < g * k; ++i) {
    OMNI_REQUIRE(members[i] >= 0 && members[i] < nrows, "group_updates: member row out of range");
    p.members[i] = members[i];
  }
  for (int i = 0; i < g; ++i) {
    OMNI_REQUIRE(snaps[i] != nullptr, "group_updates: NULL snapshot");
    p.snaps[i] = snaps[i];
    vec = vec && aligned16(snaps[i]);
  }
  const long long work = vec ? n / 4 : n;
  group_updates_kernel<<<omni::grid_for(work, kThreads), kThreads, 0, omni::as_stream(stream)>>>(
      p, n, vec ? 1 : 0);
  return omni::check_launch("group_updates");
}

int omni_sgd_momentum_f64(double* W, double* V, const double* g, const double* w_read, double eta,
                          double mu, double lam, long long n, void* stream) {
  OMNI_REQUIRE(n >= 0, "sgd: negative length");
  if (n == 0) return OMNI_OK;
  sgd_kernel_f64<<<omni::grid_for(n, kThreads), kThreads, 0, omni::as_stream(stream)>>>(
      W, V, g, w_read, eta, mu, lam, n);
  return omni::check_launch("sgd_momentum_f64");
}

int omni_gather_rows_f32(const float* src, long long row_elems, const int64_t* idx, int nidx,
                         float* dst, void* stream) {
  OMNI_REQUIRE(row_elems >= 1 && nidx >= 0, "gather: bad shape");
  if (nidx == 0) return OMNI_OK;
  cudaStream_t st = omni::as_stream(stream);
  const bool v4 = (row_elems % 4 == 0) && aligned16(src) && aligned16(dst);
  const long long per = v4 ? row_elems / 4 : row_elems;
  const int gx = (int)omni::ceil_div(per, kThreads * 4) > 0 ? (int)omni::ceil_div(per, kThreads * 4) : 1;
  const dim3 grid(gx < 65535 ? gx : 65535, nidx < 65535 ? nidx : 65535);
  if (v4)
    gather_rows_kernel<true><<<grid, kThreads, 0, st>>>(src, row_elems, idx, nidx, dst);
  else
    gather_rows_kernel<false><<<grid, kThreads, 0, st>>>(src, row_elems, idx, nidx, dst);
  return omni::check_launch("gather_rows");
}

int omni_gather_i32(const int32_t* src, const int64_t* idx, int nidx, int32_t* dst, void* stream) {
  if (nidx <= 0) return OMNI_OK;
  gather_i32_kernel<<<omni::grid_for(nidx, kThreads), kThreads, 0, omni::as_stream(stream)>>>(
      src, idx, nidx, dst);
  return omni::check_launch("gather_i32");
}

int omni_fill_f32(float* X, float value, long long n, void* stream) {
  if (n <= 0) return OMNI_OK;
  fill_kernel<<<omni::grid_for(n, kThreads), kThreads, 0, omni::as_stream(stream)>>>(X, value, n);
  return omni::check_launch("fill");
}

}  // extern "C"
