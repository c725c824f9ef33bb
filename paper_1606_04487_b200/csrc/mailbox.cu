// Host-side mailbox of the free-running compute-group runtime
// (async_groups.py): the update server and the group leaders -- separate
// processes, one per GPU -- hand gradients and snapshots to each other
// through a small POSIX shared-memory page of lock-free atomics, while the
// 250 MB payloads move GPU to GPU by copy-engine DMA over NVLink (IPC-mapped
// buffers, omni_copy_async).
//
//   ring:  a leader whose gradient has landed in its server lane takes a
//          ticket (fetch_add on `tail`) and writes its group id into the ring
//          slot; the server consumes tickets in order -- FIFO in order of
//          arrival, the serial server of simulator.py:3-7 / :170-205.
//   snap:  per group, the sequence number of the last snapshot the server
//          has written into that group's buffer (0 = none yet, -1 = stop).
//
// Waits spin with a pause and then yield, and give up after timeout_ms
// (returning OMNI_ETIMEOUT) so a dead peer never hangs a process.
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <string.h>

#include "common.cuh"

namespace {

constexpr int kMaxGroups = 64;
constexpr int kRing = 4096;   // > outstanding tickets (at most one per group)

struct Mailbox {
  std::atomic<long long> tail;                // tickets handed out
  std::atomic<long long> head;                // tickets consumed by the server
  std::atomic<int> ring[kRing];               // group id per ticket (-1 = not written yet)
  std::atomic<long long> snap[kMaxGroups];    // last snapshot sequence delivered (-1 = stop)
  std::atomic<long long> posted[kMaxGroups];  // gradients posted per group
  int ngroups;
  int magic;
};
constexpr int kMagic = 0x4f4d4e49;  // "OMNI"
static_assert(std::atomic<long long>::is_always_lock_free && std::atomic<int>::is_always_lock_free,
              "mailbox atomics must be lock-free to live in shared memory");

double now_ms() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

inline void backoff(int& spins) {
  if (++spins < 64) {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  } else {
    sched_yield();
  }
}

Mailbox* map_box(int fd) {
  void* p = mmap(nullptr, sizeof(Mailbox), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  return p == MAP_FAILED ? nullptr : static_cast<Mailbox*>(p);
}

}  // namespace

extern "C" {

long long omni_mailbox_bytes(void) { return (long long)sizeof(Mailbox); }

int omni_mailbox_create(const char* name, int ngroups, void** box) {
  OMNI_REQUIRE(name && box && ngroups >= 1 && ngroups <= kMaxGroups, "mailbox: 1 <= ngroups <= %d", kMaxGroups);
  shm_unlink(name);
  const int fd = shm_open(name, O_CREAT | O_RDWR | O_EXCL, 0600);
  OMNI_REQUIRE(fd >= 0, "mailbox: shm_open(%s) failed", name);
  if (ftruncate(fd, sizeof(Mailbox)) != 0) {
    close(fd);
    omni::set_error("mailbox: ftruncate failed");
    return OMNI_EINVAL;
  }
  Mailbox* m = map_box(fd);
  close(fd);
  OMNI_REQUIRE(m, "mailbox: mmap failed");
  m->tail.store(0);
  m->head.store(0);
  for (int i = 0; i < kRing; ++i) m->ring[i].store(-1);
  for (int i = 0; i < kMaxGroups; ++i) {
    m->snap[i].store(0);
    m->posted[i].store(0);
  }
  m->ngroups = ngroups;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  reinterpret_cast<std::atomic<int>*>(&m->magic)->store(kMagic, std::memory_order_release);
  *box = m;
  return OMNI_OK;
}

int omni_mailbox_open(const char* name, void** box, int timeout_ms) {
  OMNI_REQUIRE(name && box, "mailbox: bad arguments");
  const double t0 = now_ms();
  int spins = 0;
  for (;;) {
    const int fd = shm_open(name, O_RDWR, 0600);
    if (fd >= 0) {
      struct stat st;
      if (fstat(fd, &st) == 0 && st.st_size >= (off_t)sizeof(Mailbox)) {
        Mailbox* m = map_box(fd);
        close(fd);
        OMNI_REQUIRE(m, "mailbox: mmap failed");
        if (reinterpret_cast<std::atomic<int>*>(&m->magic)->load(std::memory_order_acquire) == kMagic) {
          *box = m;
          return OMNI_OK;
        }
        munmap(m, sizeof(Mailbox));
      } else {
        close(fd);
      }
    }
    if (now_ms() - t0 > timeout_ms) {
      omni::set_error("mailbox: %s not created within %d ms", name, timeout_ms);
      return OMNI_ETIMEOUT;
    }
    backoff(spins);
  }
}

int omni_mailbox_close(void* box, const char* unlink_name) {
  if (box) munmap(box, sizeof(Mailbox));
  if (unlink_name) shm_unlink(unlink_name);
  return OMNI_OK;
}

// Leader: its gradient is in the server lane -- take a ticket.
int omni_mailbox_post(void* box, int group, long long* ticket) {
  Mailbox* m = static_cast<Mailbox*>(box);
  OMNI_REQUIRE(m && group >= 0 && group < m->ngroups, "mailbox post: bad group %d", group);
  const long long t = m->tail.fetch_add(1, std::memory_order_acq_rel);
  m->posted[group].fetch_add(1, std::memory_order_relaxed);
  m->ring[t % kRing].store(group, std::memory_order_release);
  if (ticket) *ticket = t;
  return OMNI_OK;
}

// Server: the group of the next ticket, in ticket order.
int omni_mailbox_next(void* box, int* group, int timeout_ms) {
  Mailbox* m = static_cast<Mailbox*>(box);
  OMNI_REQUIRE(m && group, "mailbox next: bad arguments");
  const long long h = m->head.load(std::memory_order_relaxed);
  const double t0 = now_ms();
  int spins = 0;
  int g;
  while ((g = m->ring[h % kRing].load(std::memory_order_acquire)) < 0) {
    if (now_ms() - t0 > timeout_ms) {
      omni::set_error("mailbox next: no gradient within %d ms", timeout_ms);
      return OMNI_ETIMEOUT;
    }
    backoff(spins);
  }
  m->ring[h % kRing].store(-1, std::memory_order_relaxed);
  m->head.store(h + 1, std::memory_order_release);
  *group = g;
  return OMNI_OK;
}

// Server: snapshot `seq` of `group` is in place (seq < 0: stop).
int omni_mailbox_snap_post(void* box, int group, long long seq) {
  Mailbox* m = static_cast<Mailbox*>(box);
  OMNI_REQUIRE(m && group >= 0 && group < m->ngroups, "mailbox snap: bad group %d", group);
  m->snap[group].store(seq, std::memory_order_release);
  return OMNI_OK;
}

// Leader: wait until the group's snapshot sequence differs from `last`.
int omni_mailbox_snap_wait(void* box, int group, long long last, long long* seq, int timeout_ms) {
  Mailbox* m = static_cast<Mailbox*>(box);
  OMNI_REQUIRE(m && seq && group >= 0 && group < m->ngroups, "mailbox snap wait: bad group %d", group);
  const double t0 = now_ms();
  int spins = 0;
  long long v;
  while ((v = m->snap[group].load(std::memory_order_acquire)) == last) {
    if (now_ms() - t0 > timeout_ms) {
      omni::set_error("mailbox snap wait: group %d got no snapshot within %d ms", group, timeout_ms);
      return OMNI_ETIMEOUT;
    }
    backoff(spins);
  }
  *seq = v;
  return OMNI_OK;
}

}  // extern "C"
