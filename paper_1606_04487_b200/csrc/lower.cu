// K1 batched lowering (im2col over the whole mini-batch), lifting, the col2im
// adjoint, weight-layout staging and the batched transpose.
//
// All of these are pure data movement: they are HBM-bound and written so that
// consecutive threads produce consecutive output addresses (coalesced stores,
// 16-byte vectors when the row stride allows); the gathered reads hit L1/L2
// because every input element is re-read up to k*k/s^2 times in a short window.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;

// Reference column order (tensors.py:167-168): col = (ch*k + kx)*k + ky,
// row = img*m^2 + x*m + y, value = D[start+img, ch, x*s+kx-p, y*s+ky-p] or 0.
template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads) lower_nchw_kernel(
    const T* __restrict__ D, int c, int n, int k, int s, int p, int m, int start,
    long long rows, int K, long long ld, T* __restrict__ Dhat) {
  const long long cols_v = ld / VEC;
  const long long total = rows * cols_v;
  const int mm = m * m, kk = k * k;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long row = idx / cols_v;
    const int col0 = (int)(idx - row * cols_v) * VEC;
    const int img = (int)(row / mm);
    const int rem = (int)(row - (long long)img * mm);
    const int x = rem / m, y = rem - (rem / m) * m;
    const T* Dimg = D + (long long)(start + img) * c * n * n;
    T v[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const int col = col0 + j;
      T val = T(0);
      if (col < K) {
        const int ch = col / kk;
        const int t = col - ch * kk;
        const int kx = t / k, ky = t - (t / k) * k;
        const int ix = x * s + kx - p, iy = y * s + ky - p;
        if ((unsigned)ix < (unsigned)n && (unsigned)iy < (unsigned)n)
          val = __ldg(Dimg + ((long long)ch * n + ix) * n + iy);
      }
      v[j] = val;
    }
    T* out = Dhat + row * ld + col0;
    if constexpr (VEC == 4 && sizeof(T) == 4) {
      *reinterpret_cast<float4*>(out) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) out[j] = v[j];
    }
  }
}

// Tap-major lowering from NHWC (pixel stride cs): col = (kx*k + ky)*c + ch.
// One warp per lowered row (img, x, y).  For fixed kx the k taps ky = 0..k-1
// read consecutive input pixels iy0 + ky, so when cs == c the row is k
// contiguous runs of k*c floats copied from k input rows: coalesced loads,
// one contiguous 4*ld-byte store per warp.  VEC4 (c % 4 == 0): float4 lanes.
// With a padded pixel stride (cs > c) the runs break per tap (PER_TAP).
template <bool VEC4, bool PER_TAP>
__global__ void __launch_bounds__(kThreads) lower_nhwc_rows_kernel(
    const float* __restrict__ X, int n, int c, int cs, int k, int s, int p, int m,
    int rows, int K, int ld, int ones_col, float* __restrict__ Dhat) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int mm = m * m;
  const int kc = k * c;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += warps) {
    const int img = row / mm;
    const int rem = row - img * mm;
    const int x = rem / m, y = rem - (rem / m) * m;
    const int iy0 = y * s - p;
    float* out = Dhat + (long long)row * ld;
    const float* Ximg = X + (long long)img * n * n * cs;
    for (int kx = 0; kx < k; ++kx) {
      const int ix = x * s + kx - p;
      const bool row_ok = (unsigned)ix < (unsigned)n;
      const float* src = Ximg + ((long long)ix * n + iy0) * cs;  // pixel iy0 of input row ix
      float* dst = out + kx * kc;
      if constexpr (VEC4 && !PER_TAP) {
        const int c4 = c >> 2;
        for (int q = lane; q < (kc >> 2); q += 32) {
          const int ky = q / c4;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row_ok && (unsigned)(iy0 + ky) < (unsigned)n)
            v = __ldg(reinterpret_cast<const float4*>(src) + q);
          reinterpret_cast<float4*>(dst)[q] = v;
        }
      } else if constexpr (!PER_TAP) {
        for (int j = lane; j < kc; j += 32) {
          const int ky = j / c;
          float v = 0.f;
          if (row_ok && (unsigned)(iy0 + ky) < (unsigned)n) v = __ldg(src + j);
          dst[j] = v;
        }
      } else {
        for (int ky = 0; ky < k; ++ky) {
          const bool ok = row_ok && (unsigned)(iy0 + ky) < (unsigned)n;
          for (int ch = lane; ch < c; ch += 32)
            dst[ky * c + ch] = ok ? __ldg(src + (long long)ky * cs + ch) : 0.f;
        }
      }
    }
    for (int j = K + lane; j < ld; j += 32) out[j] = (ones_col && j == K) ? 1.f : 0.f;
  }
}

// Scalar-channel lowering (c % 4 != 0, e.g. the 3-channel first layer).  Each
// block builds two shared tables once: col -> offset of the source element
// relative to the window origin ((kx*n + ky)*cs + ch), and col -> (kx, ky).
// Rows whose window lies inside the image (all rows when pad == 0) take the
// fast path -- one table load, one global load, one store per element, lane
// j on column j for coalesced 128-byte stores; border rows check bounds.
__global__ void __launch_bounds__(kThreads) lower_nhwc_table_kernel(
    const float* __restrict__ X, int n, int c, int cs, int k, int s, int p, int m, int rows,
    int K, int ld, int ones_col, float* __restrict__ Dhat) {
  extern __shared__ int tab[];
  int* off = tab;       // [ld]
  int* kxy = tab + ld;  // [ld]: (kx << 16) | ky, or -1 (zero) / -2 (ones column)
  for (int j = threadIdx.x; j < ld; j += blockDim.x) {
    int o = 0, e = -1;
    if (j < K) {
      const int tap = j / c, ch = j - (j / c) * c;
      const int kx = tap / k, ky = tap - (tap / k) * k;
      o = (kx * n + ky) * cs + ch;
      e = (kx << 16) | ky;
    } else if (ones_col && j == K) {
      e = -2;
    }
    off[j] = o;
    kxy[j] = e;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int mm = m * m;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += warps) {
    const int img = row / mm;
    const int rem = row - img * mm;
    const int x = rem / m, y = rem - (rem / m) * m;
    const int ix0 = x * s - p, iy0 = y * s - p;
    float* out = Dhat + (long long)row * ld;
    if (ix0 >= 0 && iy0 >= 0 && ix0 + k <= n && iy0 + k <= n) {
      const float* org = X + (((long long)img * n + ix0) * n + iy0) * cs;
      for (int j0 = lane; j0 < ld; j0 += 128) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + 32 * u;
          float val = 0.f;
          if (j < ld) {
            const int e = kxy[j];
            val = e >= 0 ? __ldg(org + off[j]) : (e == -2 ? 1.f : 0.f);
          }
          v[u] = val;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + 32 * u < ld) out[j0 + 32 * u] = v[u];
      }
    } else {
      const float* Ximg = X + (long long)img * n * n * cs;
      for (int j = lane; j < ld; j += 32) {
        const int e = kxy[j];
        float val = e == -2 ? 1.f : 0.f;
        if (e >= 0) {
          const int ix = ix0 + (e >> 16), iy = iy0 + (e & 0xffff);
          if ((unsigned)ix < (unsigned)n && (unsigned)iy < (unsigned)n)
            val = __ldg(Ximg + ((long long)ix * n + iy) * cs + (off[j] - ((e >> 16) * n + (e & 0xffff)) * cs));
        }
        out[j] = val;
      }
    }
  }
}

// Adjoint of lower_nhwc: dX[img, ix, iy, ch] = sum over (kx, ky) with
// x = (ix+p-kx)/s, y = (iy+p-ky)/s integral and in [0, m) of
// dDhat[(img*m^2 + x*m + y)*ld + (kx*k + ky)*c + ch].  Fixed (kx, ky) order:
// deterministic, no atomics.
template <bool VEC4>
__global__ void __launch_bounds__(kThreads) col2im_nhwc_kernel(
    const float* __restrict__ dD, long long ld, int b, int n, int c, int cs, int k, int s, int p,
    int m, const float* __restrict__ mask_x, float* __restrict__ dX) {
  const int cv = VEC4 ? c / 4 : c;
  const long long total = (long long)b * n * n * cv;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long pix = idx / cv;
    const int chv = (int)(idx - pix * cv);
    const int ch = VEC4 ? chv * 4 : chv;
    const int img = (int)(pix / (n * n));
    const int r = (int)(pix - (long long)img * n * n);
    const int ix = r / n, iy = r - (r / n) * n;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int kx = 0; kx < k; ++kx) {
      const int tx = ix + p - kx;
      if (tx < 0) break;
      if (tx % s) continue;
      const int x = tx / s;
      if (x >= m) continue;
      for (int ky = 0; ky < k; ++ky) {
        const int ty = iy + p - ky;
        if (ty < 0) break;
        if (ty % s) continue;
        const int y = ty / s;
        if (y >= m) continue;
        const float* src =
            dD + ((long long)img * m * m + (long long)x * m + y) * ld + (kx * k + ky) * c + ch;
        if constexpr (VEC4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(src));
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        } else {
          acc.x += __ldg(src);
        }
      }
    }
    float* dst = dX + pix * cs + ch;
    if (mask_x) {  // fused ReLU backward: gradient flows only where the activation is > 0
      const float* mx = mask_x + pix * cs + ch;
      if constexpr (VEC4) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(mx));
        acc.x = a.x > 0.f ? acc.x : 0.f; acc.y = a.y > 0.f ? acc.y : 0.f;
        acc.z = a.z > 0.f ? acc.z : 0.f; acc.w = a.w > 0.f ? acc.w : 0.f;
      } else {
        acc.x = __ldg(mx) > 0.f ? acc.x : 0.f;
      }
    }
    if constexpr (VEC4) *reinterpret_cast<float4*>(dst) = acc;
    else *dst = acc.x;
  }
}

// OIHW (o, c, k, k) <-> tap-major rows Wt[o*ld + (kx*k+ky)*c + ch]; optional
// bias in column c*k*k (paired with the lowered matrix's ones column).
__global__ void __launch_bounds__(kThreads) weight_to_tap_kernel(
    const float* __restrict__ W, int o, int c, int k, float* __restrict__ Wt, long long ld,
    const float* __restrict__ bias) {
  const long long total = (long long)o * ld;
  const int K = c * k * k;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int oo = (int)(idx / ld);
    const int col = (int)(idx - (long long)oo * ld);
    float v = 0.f;
    if (col < K) {
      const int tap = col / c, ch = col - (col / c) * c;
      const int kx = tap / k, ky = tap - (tap / k) * k;
      v = W[(((long long)oo * c + ch) * k + kx) * k + ky];
    } else if (bias && col == K) {
      v = bias[oo];
    }
    Wt[idx] = v;
  }
}

__global__ void __launch_bounds__(kThreads) weight_from_tap_kernel(
    const float* __restrict__ Wt, int o, int c, int k, float* __restrict__ W, long long ld,
    float* __restrict__ bias) {
  const long long total = (long long)o * c * k * k;
  if (bias)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < o; i += gridDim.x * blockDim.x)
      bias[i] = Wt[(long long)i * ld + c * k * k];
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long r = idx;
    const int ky = (int)(r % k); r /= k;
    const int kx = (int)(r % k); r /= k;
    const int ch = (int)(r % c); r /= c;
    const int oo = (int)r;
    W[idx] = Wt[(long long)oo * ld + (kx * k + ky) * c + ch];
  }
}

// Data-gradient weights of a stride-1 conv: the spatially flipped, in/out
// transposed kernel in tap-major rows,
//   Wf[ch*ld + (kx*k + ky)*o + oo] = W[oo, ch, k-1-kx, k-1-ky]   (W is OIHW),
// so dX = conv(dY, Wf) with padding k-1-pad is one implicit forward GEMM.
__global__ void __launch_bounds__(kThreads) weight_flip_kernel(
    const float* __restrict__ W, int o, int c, int k, float* __restrict__ Wf, long long ld) {
  const long long total = (long long)c * ld;
  const int K = o * k * k;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(idx / ld);
    const int col = (int)(idx - (long long)ch * ld);
    float v = 0.f;
    if (col < K) {
      const int tap = col / o, oo = col - (col / o) * o;
      const int kx = tap / k, ky = tap - (tap / k) * k;
      v = W[(((long long)oo * c + ch) * k + (k - 1 - kx)) * k + (k - 1 - ky)];
    }
    Wf[idx] = v;
  }
}

// Space-to-depth with channel padding: X (b, n, n, cs) NHWC, c channels ->
// Y (b, n2, n2, cp) with Y[img, X, Y, (dx*s + dy)*c + ch] = X[img, s*X+dx, s*Y+dy, ch]
// (0 outside the image or for padded channels).  A stride-s k x k conv of X
// is then a stride-1 ceil(k/s)^2 conv of Y with s*s*c (-> cp) channels, which
// tiles the 32-channel TMA im2col boxes of the implicit GEMM.
// idx != nullptr: image img of Y is image idx[img] of X (fused batch gather).
__global__ void __launch_bounds__(kThreads) space_to_depth_kernel(
    const float* __restrict__ X, const int64_t* __restrict__ idx, int b, int n, int c, int cs,
    int s, float* __restrict__ Y, int n2, int cp) {
  // one block per output row (img, X2); shared decode table j -> (dx, dy, ch)
  extern __shared__ int s2d_tab[];
  const int sc = s * c;
  for (int j = threadIdx.x; j < cp; j += blockDim.x) {
    int e = -1;
    if (j < s * sc) {
      const int dx = j / sc, rem = j - (j / sc) * sc;
      const int dy = rem / c, ch = rem - (rem / c) * c;
      e = (dx << 24) | (dy << 16) | ch;
    }
    s2d_tab[j] = e;
  }
  __syncthreads();
  for (int row = blockIdx.x; row < b * n2; row += gridDim.x) {
    const int img = row / n2, X2 = row - (row / n2) * n2;
    const float* Xi = X + (idx ? idx[img] : (long long)img) * n * n * cs;
    float* out = Y + (long long)row * n2 * cp;
    const int total = n2 * cp;
    // 4 independent loads in flight per thread before the (coalesced) stores
    for (int q0 = threadIdx.x; q0 < total; q0 += 4 * blockDim.x) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * blockDim.x;
        float val = 0.f;
        if (q < total) {
          const int Y2 = q / cp, j = q - (q / cp) * cp;
          const int e = s2d_tab[j];
          if (e >= 0) {
            const int ix = s * X2 + (e >> 24), iy = s * Y2 + ((e >> 16) & 0xff);
            if (ix < n && iy < n) val = __ldg(Xi + ((long long)ix * n + iy) * cs + (e & 0xffff));
          }
        }
        v[u] = val;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < total) out[q] = v[u];
      }
    }
  }
}

// Fast path (cs == c, (s*c) % 4 == 0): every output float4 (4 consecutive j) is
// 4 contiguous input floats of one input row; table per group: (dx, dy of the
// group's first element, offset within the s-pixel run).
__global__ void __launch_bounds__(kThreads) space_to_depth_v4_kernel(
    const float* __restrict__ X, const int64_t* __restrict__ idx, int b, int n, int c, int s,
    float* __restrict__ Y, int n2, int cp) {
  extern __shared__ int s2d_tab[];
  const int sc = s * c, g4 = cp / 4;
  for (int t = threadIdx.x; t < g4; t += blockDim.x) {
    const int j = 4 * t;
    int e = -1;
    if (j < s * sc) {
      const int dx = j / sc, off = j - (j / sc) * sc;   // off = dy*c + ch, 4 contiguous floats
      e = (dx << 16) | off;
    }
    s2d_tab[t] = e;
  }
  __syncthreads();
  for (int row = blockIdx.x; row < b * n2; row += gridDim.x) {
    const int img = row / n2, X2 = row - (row / n2) * n2;
    const long long src_img = idx ? idx[img] : (long long)img;
    float4* out = reinterpret_cast<float4*>(Y + (long long)row * n2 * cp);
    const int total = n2 * g4;
    for (int q0 = threadIdx.x; q0 < total; q0 += 4 * blockDim.x) {
      float4 v[4];  // 4 independent 16-byte loads in flight per thread
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * blockDim.x;
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < total) {
          const int Y2 = q / g4, t = q - (q / g4) * g4;
          const int e = s2d_tab[t];
          const int ix = s * X2 + (e >> 16);
          if (e >= 0 && ix < n) {
            const int off = e & 0xffff;
            const float* src = X + ((src_img * n + ix) * n + (long long)s * Y2) * c + off;
            const int iy0 = s * Y2 + off / c;   // pixel of the first element; others may spill past n
            float a[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) a[w] = (iy0 + (off % c + w) / c < n) ? __ldg(src + w) : 0.f;
            r = make_float4(a[0], a[1], a[2], a[3]);
          }
        }
        v[u] = r;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + u * blockDim.x < total) out[q0 + u * blockDim.x] = v[u];
    }
  }
}

// Weights of the space-to-depth conv: Wt[o*ld + (kx2*k2 + ky2)*cp + (dx*s + dy)*c + ch]
// = W[o, ch, s*kx2+dx, s*ky2+dy] (0 past the original kernel / padded channels).
// inverse: read dWt, write the OIHW gradient (padded entries dropped).
__global__ void __launch_bounds__(kThreads) weight_s2d_kernel(
    float* __restrict__ W, int o, int c, int k, int s, int cp, float* __restrict__ Wt, long long ld,
    int inverse, float* __restrict__ bias) {
  const int k2 = (k + s - 1) / s;
  const int sc = s * c;
  if (inverse && bias) {   // bias-gradient row of OMNI_CONV_WGRAD_BIAS
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < o; i += gridDim.x * blockDim.x)
      bias[i] = Wt[(long long)i * ld + (long long)k2 * k2 * cp];
  }
  if (!inverse) {
    const long long total = (long long)o * ld;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
      const int oo = (int)(idx / ld);
      const int col = (int)(idx - (long long)oo * ld);
      float v = 0.f;
      if (col < k2 * k2 * cp) {
        const int tap = col / cp, j = col - (col / cp) * cp;
        if (j < s * sc) {
          const int kx2 = tap / k2, ky2 = tap - (tap / k2) * k2;
          const int dx = j / sc, rem = j - (j / sc) * sc;
          const int dy = rem / c, ch = rem - (rem / c) * c;
          const int kx = s * kx2 + dx, ky = s * ky2 + dy;
          if (kx < k && ky < k) v = W[(((long long)oo * c + ch) * k + kx) * k + ky];
        }
      }
      Wt[idx] = v;
    }
  } else {
    const long long total = (long long)o * c * k * k;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
      long long r = idx;
      const int ky = (int)(r % k); r /= k;
      const int kx = (int)(r % k); r /= k;
      const int ch = (int)(r % c); r /= c;
      const int oo = (int)r;
      const int tap = (kx / s) * k2 + (ky / s);
      const int j = ((kx % s) * s + (ky % s)) * c + ch;
      W[idx] = Wt[(long long)oo * ld + (long long)tap * cp + j];
    }
  }
}

// Batched tiled transpose through shared memory (32x33 tile: no bank conflicts).
template <typename T>
__global__ void __launch_bounds__(256) transpose_kernel(
    const T* __restrict__ src, long long lds, long long sb, int rows, int cols,
    T* __restrict__ dst, long long ldd, long long db, int batch) {
  __shared__ T tile[32][33];
  const int tiles_c = (cols + 31) / 32;
  const int tr = blockIdx.x / tiles_c, tc = blockIdx.x - (blockIdx.x / tiles_c) * tiles_c;
  for (int bi = blockIdx.y; bi < batch; bi += gridDim.y) {
    const T* S = src + (long long)bi * sb;
    T* Dd = dst + (long long)bi * db;
    const int r0 = tr * 32, c0 = tc * 32;
    for (int j = threadIdx.y; j < 32; j += 8) {
      const int r = r0 + j, cc = c0 + threadIdx.x;
      if (r < rows && cc < cols) tile[j][threadIdx.x] = S[(long long)r * lds + cc];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
      const int cc = c0 + j, r = r0 + threadIdx.x;
      if (r < rows && cc < cols) Dd[(long long)cc * ldd + r] = tile[threadIdx.x][j];
    }
    __syncthreads();
  }
}

template <typename T>
int launch_transpose(const T* src, long long lds, long long sb, int rows, int cols, T* dst,
                     long long ldd, long long db, int batch, cudaStream_t st) {
  if (rows == 0 || cols == 0 || batch == 0) return OMNI_OK;
  const long long tiles = omni::ceil_div(rows, 32) * omni::ceil_div(cols, 32);
  OMNI_REQUIRE(tiles < (1LL << 31), "transpose: too many tiles");
  dim3 grid((unsigned)tiles, (unsigned)(batch < 65535 ? batch : 65535));
  transpose_kernel<T><<<grid, dim3(32, 8), 0, st>>>(src, lds, sb, rows, cols, dst, ldd, db,
                                                    batch);
  return omni::check_launch("transpose");
}

int check_conv_geom(int b, int c, int n, int k, int stride, int pad, int* m) {
  OMNI_REQUIRE(b >= 0 && c >= 1 && n >= 1 && k >= 1 && stride >= 1 && pad >= 0,
               "n, k, d_in, d_out, stride must be positive");
  OMNI_REQUIRE(k <= n + 2 * pad, "kernel %d exceeds padded input %d", k, n + 2 * pad);
  OMNI_REQUIRE((n + 2 * pad - k) % stride == 0,
               "output size not integral: (n + 2*pad - k) = %d is not divisible by stride %d",
               n + 2 * pad - k, stride);
  *m = (n + 2 * pad - k) / stride + 1;
  return OMNI_OK;
}

template <typename T>
int lower_nchw(const T* D, int b, int c, int n, int k, int stride, int pad, int start, int b_p,
               T* Dhat, long long ld, void* stream) {
  int m = 0;
  int rc = check_conv_geom(b, c, n, k, stride, pad, &m);
  if (rc) return rc;
  OMNI_REQUIRE(b_p >= 1 && b_p <= b, "b_p=%d out of range [1, %d]", b_p, b);
  OMNI_REQUIRE(start >= 0 && start <= b - b_p, "start=%d leaves fewer than b_p=%d images", start,
               b_p);
  const int K = c * k * k;
  OMNI_REQUIRE(ld >= K, "ld=%lld < lowered width %d", ld, K);
  const long long rows = (long long)b_p * m * m;
  cudaStream_t st = omni::as_stream(stream);
  const bool vec = sizeof(T) == 4 && (ld % 4 == 0) && ((uintptr_t)Dhat % 16 == 0);
  if (vec) {
    lower_nchw_kernel<T, 4><<<omni::grid_for(rows * ld / 4, kThreads), kThreads, 0, st>>>(
        D, c, n, k, stride, pad, m, start, rows, K, ld, Dhat);
  } else {
    lower_nchw_kernel<T, 1><<<omni::grid_for(rows * ld, kThreads), kThreads, 0, st>>>(
        D, c, n, k, stride, pad, m, start, rows, K, ld, Dhat);
  }
  return omni::check_launch("lower_nchw");
}

}  // namespace

extern "C" {

int omni_lower_nchw_f32(const float* D, int b, int c, int n, int k, int stride, int pad,
                        int start, int b_p, float* Dhat, long long ld, void* stream) {
  return lower_nchw<float>(D, b, c, n, k, stride, pad, start, b_p, Dhat, ld, stream);
}

int omni_lower_nchw_f64(const double* D, int b, int c, int n, int k, int stride, int pad,
                        int start, int b_p, double* Dhat, long long ld, void* stream) {
  return lower_nchw<double>(D, b, c, n, k, stride, pad, start, b_p, Dhat, ld, stream);
}

int omni_lower_nhwc_f32(const float* X, int b, int n, int c, int cs, int k, int stride, int pad,
                        int ones_col, float* Dhat, long long ld, void* stream) {
  int m = 0;
  int rc = check_conv_geom(b, c, n, k, stride, pad, &m);
  if (rc) return rc;
  const int K = c * k * k;
  OMNI_REQUIRE(cs >= c, "pixel stride cs=%d < channels %d", cs, c);
  OMNI_REQUIRE(ld >= K + (ones_col ? 1 : 0) && ld % 4 == 0 && ld < (1LL << 31),
               "ld=%lld must be >= %d and a multiple of 4", ld, K + (ones_col ? 1 : 0));
  OMNI_REQUIRE((uintptr_t)Dhat % 16 == 0, "Dhat must be 16-byte aligned");
  if (b == 0) return OMNI_OK;
  const long long rows = (long long)b * m * m;
  OMNI_REQUIRE(rows < (1LL << 31), "too many lowered rows");
  cudaStream_t st = omni::as_stream(stream);
  const int grid = omni::grid_for(rows * 32, kThreads);
  if (cs == c && c % 4 == 0 && ((uintptr_t)X % 16 == 0)) {
    lower_nhwc_rows_kernel<true, false><<<grid, kThreads, 0, st>>>(
        X, n, c, cs, k, stride, pad, m, (int)rows, K, (int)ld, ones_col, Dhat);
  } else if (ld <= 8192) {
    const int smem = 2 * (int)ld * (int)sizeof(int);
    static int configured_max = 48 * 1024;
    if (smem > configured_max) {
      OMNI_CUDA_TRY(cudaFuncSetAttribute(lower_nhwc_table_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      configured_max = 64 * 1024;
    }
    lower_nhwc_table_kernel<<<grid, kThreads, smem, st>>>(
        X, n, c, cs, k, stride, pad, m, (int)rows, K, (int)ld, ones_col, Dhat);
  } else if (cs == c) {
    lower_nhwc_rows_kernel<false, false><<<grid, kThreads, 0, st>>>(
        X, n, c, cs, k, stride, pad, m, (int)rows, K, (int)ld, ones_col, Dhat);
  } else {
    lower_nhwc_rows_kernel<false, true><<<grid, kThreads, 0, st>>>(
        X, n, c, cs, k, stride, pad, m, (int)rows, K, (int)ld, ones_col, Dhat);
  }
  return omni::check_launch("lower_nhwc");
}

int omni_lift_nchw_f32(const float* Rhat, long long ld, int b, int m, int d_out, float* R,
                       void* stream) {
  OMNI_REQUIRE(b >= 0 && m >= 1 && d_out >= 1 && ld >= d_out, "lift: bad shape");
  // Per image, Rhat_img is (m^2 x d_out) with row stride ld; R_img is its transpose.
  return launch_transpose<float>(Rhat, ld, (long long)m * m * ld, m * m, d_out, R,
                                 (long long)m * m, (long long)d_out * m * m, b,
                                 omni::as_stream(stream));
}

int omni_lift_nchw_f64(const double* Rhat, long long ld, int b, int m, int d_out, double* R,
                       void* stream) {
  OMNI_REQUIRE(b >= 0 && m >= 1 && d_out >= 1 && ld >= d_out, "lift: bad shape");
  return launch_transpose<double>(Rhat, ld, (long long)m * m * ld, m * m, d_out, R,
                                  (long long)m * m, (long long)d_out * m * m, b,
                                  omni::as_stream(stream));
}

int omni_col2im_nhwc_f32(const float* dDhat, long long ld, int b, int n, int c, int cs, int k,
                         int stride, int pad, const float* relu_mask_x, float* dX, void* stream) {
  int m = 0;
  int rc = check_conv_geom(b, c, n, k, stride, pad, &m);
  if (rc) return rc;
  OMNI_REQUIRE(cs >= c && ld >= (long long)c * k * k, "col2im: bad strides");
  if (b == 0) return OMNI_OK;
  cudaStream_t st = omni::as_stream(stream);
  const bool v4 = (c % 4 == 0) && (cs % 4 == 0) && (ld % 4 == 0) &&
                  ((uintptr_t)dX % 16 == 0) && ((uintptr_t)dDhat % 16 == 0) &&
                  ((uintptr_t)relu_mask_x % 16 == 0);
  const long long work = (long long)b * n * n * (v4 ? c / 4 : c);
  if (v4)
    col2im_nhwc_kernel<true><<<omni::grid_for(work, kThreads), kThreads, 0, st>>>(
        dDhat, ld, b, n, c, cs, k, stride, pad, m, relu_mask_x, dX);
  else
    col2im_nhwc_kernel<false><<<omni::grid_for(work, kThreads), kThreads, 0, st>>>(
        dDhat, ld, b, n, c, cs, k, stride, pad, m, relu_mask_x, dX);
  return omni::check_launch("col2im_nhwc");
}

int omni_conv_weight_to_tap_f32(float* W, int o, int c, int k, float* Wt, long long ld,
                                int inverse, float* bias, void* stream) {
  OMNI_REQUIRE(o >= 1 && c >= 1 && k >= 1 && ld >= (long long)c * k * k + (bias ? 1 : 0),
               "weight staging: bad shape");
  cudaStream_t st = omni::as_stream(stream);
  if (!inverse) {
    weight_to_tap_kernel<<<omni::grid_for((long long)o * ld, kThreads), kThreads, 0, st>>>(
        W, o, c, k, Wt, ld, bias);
  } else {
    weight_from_tap_kernel<<<omni::grid_for((long long)o * c * k * k, kThreads), kThreads, 0,
                             st>>>(Wt, o, c, k, W, ld, bias);
  }
  return omni::check_launch("conv_weight_to_tap");
}

int omni_conv_weight_flip_f32(const float* W, int o, int c, int k, float* Wf, long long ld,
                              void* stream) {
  OMNI_REQUIRE(o >= 1 && c >= 1 && k >= 1 && ld >= (long long)o * k * k, "weight flip: bad shape");
  weight_flip_kernel<<<omni::grid_for((long long)c * ld, kThreads), kThreads, 0,
                       omni::as_stream(stream)>>>(W, o, c, k, Wf, ld);
  return omni::check_launch("conv_weight_flip");
}

static int space_to_depth(const float* X, const int64_t* idx, int b, int n, int c, int cs, int s,
                          float* Y, int n2, int cp, void* stream) {
  OMNI_REQUIRE(b >= 0 && n >= 1 && c >= 1 && cs >= c && s >= 1 && n2 * s >= n && cp >= s * s * c &&
                   cp % 4 == 0 && ((uintptr_t)Y % 16) == 0,
               "space_to_depth: bad shape");
  if (b == 0) return OMNI_OK;
  OMNI_REQUIRE(cp <= 12288, "space_to_depth: too many channels");
  const int rows = b * n2;
  int dev = 0;
  cudaGetDevice(&dev);
  const int grid = rows < omni::sm_count_cached(dev) * 16 ? rows : omni::sm_count_cached(dev) * 16;
  if (cs == c && (s * c) % 4 == 0)
    space_to_depth_v4_kernel<<<grid, kThreads, (cp / 4) * sizeof(int), omni::as_stream(stream)>>>(
        X, idx, b, n, c, s, Y, n2, cp);
  else
    space_to_depth_kernel<<<grid, kThreads, cp * sizeof(int), omni::as_stream(stream)>>>(
        X, idx, b, n, c, cs, s, Y, n2, cp);
  return omni::check_launch("space_to_depth");
}

int omni_space_to_depth_f32(const float* X, int b, int n, int c, int cs, int s, float* Y, int n2,
                            int cp, void* stream) {
  return space_to_depth(X, nullptr, b, n, c, cs, s, Y, n2, cp, stream);
}

int omni_space_to_depth_gather_f32(const float* X, const int64_t* idx, int b, int n, int c, int cs,
                                   int s, float* Y, int n2, int cp, void* stream) {
  OMNI_REQUIRE(idx != nullptr, "space_to_depth_gather: idx is NULL");
  return space_to_depth(X, idx, b, n, c, cs, s, Y, n2, cp, stream);
}

int omni_conv_weight_s2d_f32(float* W, int o, int c, int k, int s, int cp, float* Wt, long long ld,
                             int inverse, float* bias, void* stream) {
  const int k2 = (k + s - 1) / s;
  OMNI_REQUIRE(o >= 1 && c >= 1 && k >= 1 && s >= 1 && cp >= s * s * c &&
                   ld >= (long long)k2 * k2 * cp,
               "weight s2d: bad shape");
  OMNI_REQUIRE(!bias || (inverse && ld > (long long)k2 * k2 * cp),
               "weight s2d: the bias column needs inverse=1 and ld > ceil(k/s)^2 * cp");
  const long long work = inverse ? (long long)o * c * k * k : (long long)o * ld;
  weight_s2d_kernel<<<omni::grid_for(work, kThreads), kThreads, 0, omni::as_stream(stream)>>>(
      W, o, c, k, s, cp, Wt, ld, inverse, bias);
  return omni::check_launch("conv_weight_s2d");
}

int omni_transpose_f32(const float* src, long long lds, long long src_bstride, int rows, int cols,
                       float* dst, long long ldd, long long dst_bstride, int batch, void* stream) {
  OMNI_REQUIRE(rows >= 0 && cols >= 0 && batch >= 0 && lds >= cols && ldd >= rows,
               "transpose: bad shape");
  return launch_transpose<float>(src, lds, src_bstride, rows, cols, dst, ldd, dst_bstride, batch,
                                 omni::as_stream(stream));
}

}  // extern "C"
