// Communicator entry points of the C-ABI (omni_comm_init_all,
// omni_comm_split, omni_allreduce_sum_f32, omni_comm_destroy), so a host that
// is not Python (the ctypes / C++ consumer in INTEGRATION.md) can run the
// multi-GPU path: a group's gradient allreduce (§8(e), the k GPUs of one
// compute group) and the server <-> group-leader snapshot / gradient
// transfers of the asynchronous runtime.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"): inside a PyTorch
// process that is the NCCL torch already loaded (same soname, one copy in the
// process), elsewhere the system library.
// Only <nccl.h> types are used at compile time; the library is never linked.

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string.h>

#include "common.cuh"

namespace {

struct Nccl {
  bool ok = false;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

Nccl g_nccl;
std::once_flag g_nccl_once;
std::string g_nccl_load_error;

template <class F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  if (!f) g_nccl_load_error = std::string("libnccl.so.2 lacks ") + name;
  return f != nullptr;
}

void load_nccl() {
  // Prefer a copy already mapped into the process (torch's), then the loader path.
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    const char* e = dlerror();
    g_nccl_load_error = std::string("dlopen(libnccl.so.2) failed: ") + (e ? e : "?");
    return;
  }
  Nccl n;
  bool ok = sym(h, "ncclGetErrorString", n.GetErrorString) && sym(h, "ncclGetVersion", n.GetVersion) &&
            sym(h, "ncclGetUniqueId", n.GetUniqueId) && sym(h, "ncclCommInitRank", n.CommInitRank) &&
            sym(h, "ncclCommInitAll", n.CommInitAll) && sym(h, "ncclCommSplit", n.CommSplit) &&
            sym(h, "ncclCommDestroy", n.CommDestroy) && sym(h, "ncclCommCount", n.CommCount) &&
            sym(h, "ncclCommUserRank", n.CommUserRank) && sym(h, "ncclAllReduce", n.AllReduce) &&
            sym(h, "ncclBroadcast", n.Broadcast) && sym(h, "ncclSend", n.Send) && sym(h, "ncclRecv", n.Recv) &&
            sym(h, "ncclAllGather", n.AllGather) &&
            sym(h, "ncclGroupStart", n.GroupStart) && sym(h, "ncclGroupEnd", n.GroupEnd);
  n.ok = ok;
  g_nccl = n;
}

int need_nccl() {
  std::call_once(g_nccl_once, load_nccl);
  if (!g_nccl.ok) {
    omni::set_error("NCCL unavailable: %s", g_nccl_load_error.c_str());
    return OMNI_EUNSUPPORTED;
  }
  return OMNI_OK;
}

}  // namespace

#define OMNI_NCCL_TRY(expr)                                                              \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess) {                                                             \
      omni::set_error("%s failed: %s", #expr, g_nccl.GetErrorString(_r));                \
      return _r == ncclInvalidArgument || _r == ncclInvalidUsage ? OMNI_EINVAL : OMNI_ECUDA; \
    }                                                                                    \
  } while (0)

#define OMNI_NEED_NCCL()          \
  do {                            \
    int _s = need_nccl();         \
    if (_s != OMNI_OK) return _s; \
  } while (0)

extern "C" {

int omni_comm_nccl_version(int* version) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(version != nullptr, "omni_comm_nccl_version: version is NULL");
  OMNI_NCCL_TRY(g_nccl.GetVersion(version));
  return OMNI_OK;
}

int omni_comm_unique_id(void* id) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(id != nullptr, "omni_comm_unique_id: id is NULL");
  static_assert(sizeof(ncclUniqueId) == OMNI_COMM_ID_BYTES, "NCCL unique id size");
  ncclUniqueId u;
  OMNI_NCCL_TRY(g_nccl.GetUniqueId(&u));
  memcpy(id, &u, sizeof(u));
  return OMNI_OK;
}

int omni_comm_init_rank(void** comm, int nranks, const void* id, int rank, int device) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr && id != nullptr, "omni_comm_init_rank: NULL argument");
  OMNI_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks,
               "omni_comm_init_rank: rank %d outside [0, %d)", rank, nranks);
  OMNI_CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  *comm = nullptr;
  OMNI_NCCL_TRY(g_nccl.CommInitRank(reinterpret_cast<ncclComm_t*>(comm), nranks, u, rank));
  return OMNI_OK;
}

int omni_comm_init_all(int ndev, const int* devs, void** comms) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(ndev >= 1 && comms != nullptr, "omni_comm_init_all: need ndev >= 1 and comms");
  static_assert(sizeof(ncclComm_t) == sizeof(void*), "ncclComm_t is a pointer");
  OMNI_NCCL_TRY(g_nccl.CommInitAll(reinterpret_cast<ncclComm_t*>(comms), ndev, devs));
  return OMNI_OK;
}

int omni_comm_split(void* comm, int color, int key, void** newcomm) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr && newcomm != nullptr, "omni_comm_split: NULL argument");
  OMNI_REQUIRE(color >= 0 || color == OMNI_COMM_SPLIT_NOCOLOR,
               "omni_comm_split: color must be >= 0 or OMNI_COMM_SPLIT_NOCOLOR");
  // Inside omni_comm_group_start/end NCCL completes the split at group end and
  // writes the handle then: hand it the caller's slot, not a local.
  *newcomm = nullptr;
  OMNI_NCCL_TRY(g_nccl.CommSplit(static_cast<ncclComm_t>(comm),
                                 color == OMNI_COMM_SPLIT_NOCOLOR ? NCCL_SPLIT_NOCOLOR : color, key,
                                 reinterpret_cast<ncclComm_t*>(newcomm), nullptr));
  return OMNI_OK;
}

int omni_comm_destroy(void* comm) {
  if (comm == nullptr) return OMNI_OK;
  OMNI_NEED_NCCL();
  OMNI_NCCL_TRY(g_nccl.CommDestroy(static_cast<ncclComm_t>(comm)));
  return OMNI_OK;
}

int omni_comm_size_rank(void* comm, int* size, int* rank) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr, "omni_comm_size_rank: comm is NULL");
  if (size) OMNI_NCCL_TRY(g_nccl.CommCount(static_cast<ncclComm_t>(comm), size));
  if (rank) OMNI_NCCL_TRY(g_nccl.CommUserRank(static_cast<ncclComm_t>(comm), rank));
  return OMNI_OK;
}

int omni_allreduce_sum_f32(void* comm, float* buf, size_t n, void* stream) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr, "omni_allreduce_sum_f32: comm is NULL");
  OMNI_REQUIRE(n == 0 || buf != nullptr, "omni_allreduce_sum_f32: buf is NULL");
  if (n == 0) return OMNI_OK;
  OMNI_NCCL_TRY(g_nccl.AllReduce(buf, buf, n, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm),
                                 omni::as_stream(stream)));
  return OMNI_OK;
}

int omni_broadcast_f32(void* comm, float* buf, size_t n, int root, void* stream) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr && (n == 0 || buf != nullptr), "omni_broadcast_f32: NULL argument");
  if (n == 0) return OMNI_OK;
  OMNI_NCCL_TRY(g_nccl.Broadcast(buf, buf, n, ncclFloat32, root, static_cast<ncclComm_t>(comm),
                                 omni::as_stream(stream)));
  return OMNI_OK;
}

int omni_send_f32(void* comm, const float* buf, size_t n, int peer, void* stream) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr && (n == 0 || buf != nullptr), "omni_send_f32: NULL argument");
  OMNI_NCCL_TRY(g_nccl.Send(buf, n, ncclFloat32, peer, static_cast<ncclComm_t>(comm),
                            omni::as_stream(stream)));
  return OMNI_OK;
}

int omni_recv_f32(void* comm, float* buf, size_t n, int peer, void* stream) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr && (n == 0 || buf != nullptr), "omni_recv_f32: NULL argument");
  OMNI_NCCL_TRY(g_nccl.Recv(buf, n, ncclFloat32, peer, static_cast<ncclComm_t>(comm),
                            omni::as_stream(stream)));
  return OMNI_OK;
}

int omni_allgather_f32(void* comm, const float* send, float* recv, size_t n, void* stream) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr && (n == 0 || (send != nullptr && recv != nullptr)),
               "omni_allgather_f32: NULL argument");
  if (n == 0) return OMNI_OK;
  OMNI_NCCL_TRY(g_nccl.AllGather(send, recv, n, ncclFloat32, static_cast<ncclComm_t>(comm),
                                 omni::as_stream(stream)));
  return OMNI_OK;
}

// Personalised all-to-all: parts[m] (n floats, any addresses) goes to rank m,
// rank m's part for this rank lands at recv + m*n.  One NCCL group of
// 2*(nranks-1) point-to-point calls; the self part is a device copy.
int omni_all_to_all_f32(void* comm, const float* const* parts, float* recv, size_t n,
                        void* stream) {
  OMNI_NEED_NCCL();
  OMNI_REQUIRE(comm != nullptr && parts != nullptr && (n == 0 || recv != nullptr),
               "omni_all_to_all_f32: NULL argument");
  if (n == 0) return OMNI_OK;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int size = 0, me = 0;
  OMNI_NCCL_TRY(g_nccl.CommCount(c, &size));
  OMNI_NCCL_TRY(g_nccl.CommUserRank(c, &me));
  for (int m = 0; m < size; ++m)
    OMNI_REQUIRE(parts[m] != nullptr, "omni_all_to_all_f32: NULL part");
  cudaStream_t st = omni::as_stream(stream);
  OMNI_CUDA_TRY(cudaMemcpyAsync(recv + (size_t)me * n, parts[me], n * sizeof(float),
                                cudaMemcpyDeviceToDevice, st));
  OMNI_NCCL_TRY(g_nccl.GroupStart());
  for (int m = 0; m < size; ++m) {
    if (m == me) continue;
    ncclResult_t r = g_nccl.Send(parts[m], n, ncclFloat32, m, c, st);
    if (r == ncclSuccess) r = g_nccl.Recv(recv + (size_t)m * n, n, ncclFloat32, m, c, st);
    if (r != ncclSuccess) {
      g_nccl.GroupEnd();
      omni::set_error("omni_all_to_all_f32: %s", g_nccl.GetErrorString(r));
      return OMNI_ECUDA;
    }
  }
  OMNI_NCCL_TRY(g_nccl.GroupEnd());
  return OMNI_OK;
}

int omni_comm_group_start(void) {
  OMNI_NEED_NCCL();
  OMNI_NCCL_TRY(g_nccl.GroupStart());
  return OMNI_OK;
}

int omni_comm_group_end(void) {
  OMNI_NEED_NCCL();
  OMNI_NCCL_TRY(g_nccl.GroupEnd());
  return OMNI_OK;
}

}  // extern "C"
