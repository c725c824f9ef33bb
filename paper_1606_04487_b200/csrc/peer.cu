// Peer-memory data-parallel update over NVLink / NVSwitch: the gradient
// allreduce and the momentum update (K8, sgd.py:92-101) of one layer fused
// into ONE kernel that works directly on the other GPUs' memory.
//
// Each of the N ranks owns 1/N of every layer's parameter slice.  For its
// part it reads the N gradients straight out of the peers' HBM (CUDA IPC
// mappings), sums them in rank order 0..N-1 (fixed order: every rank ends
// with bit-identical weights, independent of arrival timing), applies
//     V = mu V - eta (G_sum + lam w_read);  W += V
// and stores the new W into every peer's W.  Traffic per rank and layer is
// (N-1)/N of the slice read and (N-1)/N written over NVLink -- what a ring
// allreduce moves -- with the separate update pass gone and no reduction
// staging buffer.  (The caller folds the 1/N of the mean into eta / lam.)
//
// Ordering between GPUs uses int64 flag slots in each rank's memory that the
// peers write with system-scope release stores and the owner polls with
// acquire loads:
//   flags[kind][src][slot],  kind 0 = "src's gradient of slot is final and
//   src no longer reads W of slot", kind 1 = "src has written its part of
//   slot's W into every peer".  Values are the step number, read from a
//   device counter (omni_p2p_step) so a captured CUDA graph replays a whole
//   data-parallel step unchanged; slots never need resetting.
// A wait gives up after 30 s and traps (a peer died) instead
// of hanging the GPU.

#include <cuda_runtime.h>
#include <stdlib.h>

#include "common.cuh"

namespace {

constexpr unsigned long long kTimeoutNs = 30ull * 1000000000ull;
constexpr int kMaxRanks = 8;

struct FlagPtrs {
  long long* f[kMaxRanks];   // each rank's flag block, [kind][src][slot]
};

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ long long ld_acquire_sys(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(long long* p, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void p2p_step_kernel(long long* step) { *step += 1; }

__global__ void p2p_signal_kernel(FlagPtrs fp, int n, int rank, int kind, int slot,
                                  int max_slots, const long long* __restrict__ step) {
  const int p = threadIdx.x;
  if (p >= n) return;
  const long long value = *step;
  asm volatile("fence.acq_rel.sys;" ::: "memory");   // prior kernels' (peer) stores first
  st_release_sys(fp.f[p] + ((long long)kind * n + rank) * max_slots + slot, value);
}

__global__ void p2p_wait_kernel(const long long* __restrict__ flags, int n, int rank, int kind,
                                int slot_lo, int slot_hi, int max_slots,
                                const long long* __restrict__ step) {
  const long long value = *step;
  const int per = slot_hi - slot_lo;
  const unsigned long long t0 = now_ns();
  for (int i = threadIdx.x; i < n * per; i += blockDim.x) {
    const int src = i / per, slot = slot_lo + i % per;
    const long long* f = flags + ((long long)kind * n + src) * max_slots + slot;
    while (ld_acquire_sys(f) < value) {
      if (now_ns() - t0 > kTimeoutNs) {
        printf("omni p2p wait: rank %d timed out on flag kind %d src %d slot %d (want %lld)\n",
               rank, kind, src, slot, value);
        __trap();
      }
      __nanosleep(200);
    }
  }
  __syncthreads();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

inline long long ceil_div_ll(long long a, long long b) { return (a + b - 1) / b; }

struct PeerPtrs {
  const float* g[kMaxRanks];
  float* w[kMaxRanks];
};

// U float4s of this rank's part (i, i + step, ...): every load is issued
// before any arithmetic, so U * N remote 16-byte loads are in flight per thread.
template <int N, int U>
__device__ __forceinline__ void update4(const PeerPtrs& pp, int n, int rank, long long i,
                                        long long step, long long end, float* V, float* Wl,
                                        const float* wr, float eta, float mu, float lam) {
  constexpr int NN = N ? N : kMaxRanks;
  float4 g[U][NN];
  float4 v[U], r[U], w[U];
  bool ok[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long long j = i + u * step;
    ok[u] = j < end;
    if (!ok[u]) continue;
#pragma unroll
    for (int p = 0; p < NN; ++p) {
      if (!N && p >= n) break;
      g[u][p] = *reinterpret_cast<const float4*>(pp.g[p] + j);
    }
    v[u] = *reinterpret_cast<const float4*>(V + j);
    r[u] = *reinterpret_cast<const float4*>(wr + j);
    w[u] = *reinterpret_cast<const float4*>(Wl + j);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (!ok[u]) continue;
    const long long j = i + u * step;
    float4 s = g[u][0];
#pragma unroll
    for (int p = 1; p < NN; ++p) {
      if (!N && p >= n) break;
      s.x += g[u][p].x; s.y += g[u][p].y; s.z += g[u][p].z; s.w += g[u][p].w;
    }
    float4 vv = v[u], ww = w[u];
    vv.x = mu * vv.x - eta * (s.x + lam * r[u].x);
    vv.y = mu * vv.y - eta * (s.y + lam * r[u].y);
    vv.z = mu * vv.z - eta * (s.z + lam * r[u].z);
    vv.w = mu * vv.w - eta * (s.w + lam * r[u].w);
    ww.x += vv.x; ww.y += vv.y; ww.z += vv.z; ww.w += vv.w;
    *reinterpret_cast<float4*>(V + j) = vv;
#pragma unroll
    for (int p = 0; p < NN; ++p) {
      if (!N && p >= n) break;
      if (pp.w[p] != nullptr) *reinterpret_cast<float4*>(pp.w[p] + j) = ww;
    }
  }
}

__device__ __forceinline__ void update1(const PeerPtrs& pp, int n, int rank, long long i, float* V,
                                        const float* wr, float eta, float mu, float lam) {
  float s = pp.g[0][i];
  for (int p = 1; p < n; ++p) s += pp.g[p][i];
  const float v = mu * V[i] - eta * (s + lam * wr[i]);
  const float w = pp.w[rank][i] + v;
  V[i] = v;
  for (int p = 0; p < n; ++p)
    if (pp.w[p] != nullptr) pp.w[p][i] = w;
}

template <int N, int U>
__global__ void __launch_bounds__(256) p2p_reduce_sgd_kernel(PeerPtrs pp, int n, int rank,
                                                             long long lo, long long hi, float* V,
                                                             float* Wl, const float* wr, float eta,
                                                             float mu, float lam) {
  // scalar head up to a 16-byte boundary (all buffers share element offsets)
  const long long a0 = min(hi, (lo + 3) & ~3ll);
  const long long a1 = a0 + ((hi - a0) & ~3ll);
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (tid < a0 - lo) update1(pp, n, rank, lo + tid, V, wr, eta, mu, lam);
  if (tid < hi - a1) update1(pp, n, rank, a1 + tid, V, wr, eta, mu, lam);
  for (long long i = a0 + 4 * tid; i < a1; i += 4 * stride * U)
    update4<N, U>(pp, n, rank, i, 4 * stride, a1, V, Wl, wr, eta, mu, lam);
}

template <int U>
void launch_reduce_sgd(int grid, cudaStream_t s, const PeerPtrs& pp, int n, int rank, long long lo,
                       long long hi, float* V, float* Wl, const float* wr, float eta, float mu,
                       float lam) {
  switch (n) {
    case 2: p2p_reduce_sgd_kernel<2, U><<<grid, 256, 0, s>>>(pp, n, rank, lo, hi, V, Wl, wr, eta, mu, lam); break;
    case 4: p2p_reduce_sgd_kernel<4, U><<<grid, 256, 0, s>>>(pp, n, rank, lo, hi, V, Wl, wr, eta, mu, lam); break;
    case 8: p2p_reduce_sgd_kernel<8, U><<<grid, 256, 0, s>>>(pp, n, rank, lo, hi, V, Wl, wr, eta, mu, lam); break;
    default: p2p_reduce_sgd_kernel<0, U><<<grid, 256, 0, s>>>(pp, n, rank, lo, hi, V, Wl, wr, eta, mu, lam);
  }
}

}  // namespace

extern "C" {

int omni_p2p_step(long long* step, void* stream) {
  OMNI_REQUIRE(step != nullptr, "omni_p2p_step: step is NULL");
  p2p_step_kernel<<<1, 1, 0, omni::as_stream(stream)>>>(step);
  return omni::check_launch("p2p_step_kernel");
}

int omni_p2p_signal(long long* const* flags, int nranks, int rank, int kind, int slot,
                    int max_slots, const long long* step, void* stream) {
  OMNI_REQUIRE(flags != nullptr && step != nullptr, "omni_p2p_signal: NULL argument");
  OMNI_REQUIRE(nranks >= 1 && nranks <= kMaxRanks && rank >= 0 && rank < nranks,
               "omni_p2p_signal: rank %d of %d (at most %d ranks)", rank, nranks, kMaxRanks);
  OMNI_REQUIRE((kind == OMNI_P2P_GRAD_READY || kind == OMNI_P2P_W_DONE) && slot >= 0 &&
                   slot < max_slots,
               "omni_p2p_signal: bad kind %d / slot %d of %d", kind, slot, max_slots);
  FlagPtrs fp{};
  for (int p = 0; p < nranks; ++p) {
    OMNI_REQUIRE(flags[p] != nullptr, "omni_p2p_signal: NULL flag block %d", p);
    fp.f[p] = flags[p];
  }
  p2p_signal_kernel<<<1, 32, 0, omni::as_stream(stream)>>>(fp, nranks, rank, kind, slot, max_slots,
                                                           step);
  return omni::check_launch("p2p_signal_kernel");
}

int omni_p2p_wait(const long long* flags, int nranks, int rank, int kind, int slot_lo, int slot_hi,
                  int max_slots, const long long* step, void* stream) {
  OMNI_REQUIRE(flags != nullptr && step != nullptr, "omni_p2p_wait: NULL argument");
  OMNI_REQUIRE(nranks >= 1 && nranks <= kMaxRanks && rank >= 0 && rank < nranks,
               "omni_p2p_wait: rank %d of %d (at most %d ranks)", rank, nranks, kMaxRanks);
  OMNI_REQUIRE((kind == OMNI_P2P_GRAD_READY || kind == OMNI_P2P_W_DONE) && slot_lo >= 0 &&
                   slot_lo <= slot_hi && slot_hi <= max_slots,
               "omni_p2p_wait: bad kind %d / slots [%d, %d) of %d", kind, slot_lo, slot_hi,
               max_slots);
  if (slot_lo == slot_hi) return OMNI_OK;
  p2p_wait_kernel<<<1, 256, 0, omni::as_stream(stream)>>>(flags, nranks, rank, kind, slot_lo,
                                                          slot_hi, max_slots, step);
  return omni::check_launch("p2p_wait_kernel");
}

int omni_p2p_reduce_sgd_f32(const float* const* grads, float* const* weights, int nranks, int rank,
                            long long lo, long long hi, float* V, const float* w_read, float eta,
                            float mu, float lam, void* stream) {
  OMNI_REQUIRE(grads != nullptr && weights != nullptr && V != nullptr && w_read != nullptr,
               "omni_p2p_reduce_sgd_f32: NULL argument");
  OMNI_REQUIRE(nranks >= 1 && nranks <= kMaxRanks && rank >= 0 && rank < nranks,
               "omni_p2p_reduce_sgd_f32: rank %d of %d (at most %d ranks)", rank, nranks,
               kMaxRanks);
  OMNI_REQUIRE(0 <= lo && lo <= hi, "omni_p2p_reduce_sgd_f32: bad range [%lld, %lld)", lo, hi);
  PeerPtrs pp{};
  for (int p = 0; p < nranks; ++p) {
    OMNI_REQUIRE(grads[p] != nullptr && (weights[p] != nullptr || p != rank),
                 "omni_p2p_reduce_sgd_f32: NULL pointer for rank %d", p);
    OMNI_REQUIRE(((uintptr_t)grads[p] & 15) == ((uintptr_t)grads[0] & 15) &&
                     (weights[p] == nullptr ||
                      ((uintptr_t)weights[p] & 15) == ((uintptr_t)grads[0] & 15)) &&
                     ((uintptr_t)V & 15) == ((uintptr_t)grads[0] & 15) &&
                     ((uintptr_t)w_read & 15) == ((uintptr_t)grads[0] & 15),
                 "omni_p2p_reduce_sgd_f32: buffers must share their 16-byte alignment");
    pp.g[p] = grads[p];
    pp.w[p] = weights[p];
  }
  OMNI_REQUIRE(((uintptr_t)grads[0] & 15) == 0,
               "omni_p2p_reduce_sgd_f32: buffers must be 16-byte aligned");
  if (hi == lo) return OMNI_OK;
  const long long n4 = (hi - lo + 3) / 4;
  static const int unroll = [] {
    const char* e = getenv("OMNI_P2P_UNROLL");   // probe knob: 1, 2 or 4 float4s per thread
    const int u = e ? atoi(e) : 2;
    return (u == 1 || u == 4) ? u : 2;
  }();
  const int grid = omni::grid_for(ceil_div_ll(n4, unroll), 256);
  cudaStream_t s = omni::as_stream(stream);
  float* Wl = weights[rank];
  if (unroll == 1) launch_reduce_sgd<1>(grid, s, pp, nranks, rank, lo, hi, V, Wl, w_read, eta, mu, lam);
  else if (unroll == 4) launch_reduce_sgd<4>(grid, s, pp, nranks, rank, lo, hi, V, Wl, w_read, eta, mu, lam);
  else launch_reduce_sgd<2>(grid, s, pp, nranks, rank, lo, hi, V, Wl, w_read, eta, mu, lam);
  return omni::check_launch("p2p_reduce_sgd_kernel");
}

int omni_copy_async(void* dst, const void* src, long long bytes, void* stream) {
  OMNI_REQUIRE(bytes >= 0 && (bytes == 0 || (dst != nullptr && src != nullptr)),
               "omni_copy_async: bad arguments");
  if (bytes == 0) return OMNI_OK;
  OMNI_CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault,
                                omni::as_stream(stream)));
  return OMNI_OK;
}

int omni_ipc_handle(const void* ptr, void* handle, long long* offset) {
  OMNI_REQUIRE(ptr != nullptr && handle != nullptr && offset != nullptr,
               "omni_ipc_handle: NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == OMNI_IPC_HANDLE_BYTES, "IPC handle size");
  // the handle names the whole allocation; report ptr's offset inside it
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<GetRange>(f);
  }();
  OMNI_REQUIRE(get_range != nullptr, "omni_ipc_handle: cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0) {
    omni::set_error("omni_ipc_handle: %p is not device memory", ptr);
    return OMNI_EINVAL;
  }
  cudaIpcMemHandle_t h;
  OMNI_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle, &h, sizeof(h));
  *offset = (long long)((uintptr_t)ptr - base);
  return OMNI_OK;
}

int omni_ipc_open(const void* handle, void** base) {
  OMNI_REQUIRE(handle != nullptr && base != nullptr, "omni_ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  OMNI_CUDA_TRY(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return OMNI_OK;
}

int omni_ipc_close(void* base) {
  if (base == nullptr) return OMNI_OK;
  OMNI_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return OMNI_OK;
}

}  // extern "C"
