// Status plumbing shared by every entry point of libomni.so.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>
#include <mutex>

#include "common.cuh"

namespace omni {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

static std::atomic<long long> g_launches{0};

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return OMNI_ECUDA;
  }
  // OMNI_DEBUG_SYNC=1: wait for every launch and name the kernel that faulted
  // (debugging aid; never set in production or inside graph capture)
  static const bool debug_sync = getenv("OMNI_DEBUG_SYNC") != nullptr;
  if (debug_sync) {
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      fprintf(stderr, "[omni] %s: kernel failed: %s\n", what, cudaGetErrorString(e));
      set_error("%s: kernel failed: %s", what, cudaGetErrorString(e));
      return OMNI_ECUDA;
    }
  }
  return OMNI_OK;
}

static int g_sm_count[64];
static std::once_flag g_sm_once[64];

int sm_count_cached(int dev) {
  if (dev < 0 || dev >= 64) return 148;
  std::call_once(g_sm_once[dev], [dev]() {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    g_sm_count[dev] = v;
  });
  return g_sm_count[dev];
}

int grid_for(long long work_items, int threads) {
  int dev = 0;
  cudaGetDevice(&dev);
  long long sms = sm_count_cached(dev);
  long long want = ceil_div(work_items, threads);
  long long cap = sms * 8;  // 8 resident 256-thread blocks per SM saturate HBM
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

}  // namespace omni

extern "C" {

const char* omni_last_error(void) { return omni::g_last_error.c_str(); }

int omni_version(void) { return 1; }

int omni_device_sm_count(int device) { return omni::sm_count_cached(device); }

long long omni_launch_count(void) { return omni::g_launches.load(std::memory_order_relaxed); }

static std::atomic<int> g_sm_reserve{-1};

int omni_set_sm_reserve(int sms) {
  OMNI_REQUIRE(sms >= 0 && sms <= 64, "sm reserve must be in [0, 64]");
  g_sm_reserve.store(sms);
  return OMNI_OK;
}

int omni_get_sm_reserve(void) {
  int r = g_sm_reserve.load();
  if (r < 0) {   // first use: OMNI_SM_RESERVE from the environment, default 0
    const char* e = getenv("OMNI_SM_RESERVE");
    r = e ? atoi(e) : 0;
    if (r < 0 || r > 64) r = 0;
    g_sm_reserve.store(r);
  }
  return r;
}

}  // extern "C"
