// r2_oob_shm.cpp -- out-of-band control channel over POSIX shared memory.
//
// "When either endpoint detects an error, it immediately alerts its
// peer via a separate bootstrap network" -- on one 8xB200 box the ranks are
// processes of one host, so the OOB network is a host shared-memory segment,
// entirely off the NVLink data path.  It provides the r2_oob_t vtable:
// allgather / barrier (bootstrap, registration) and non-blocking post / poll
// of small control messages (notify, probe request/result, verdict, abort)
// through one single-producer ring per (src, dst) pair.
#include <errno.h>
#include <fcntl.h>
#include <sched.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <mutex>
#include <string>

#include "../../include/r2ccl.h"

namespace {

constexpr uint64_t kMagic = 0x5232434F4F423031ull;  // "R2COOB01"
constexpr int kSlots = 256;
constexpr int kMsg = 256;
constexpr size_t kAgBytes = 16384;

struct Ring {
  std::atomic<uint64_t> head;   // producer
  char pad0[56];
  std::atomic<uint64_t> tail;   // consumer
  char pad1[56];
  uint32_t len[kSlots];
  char data[kSlots][kMsg];
};

struct Header {
  std::atomic<uint64_t> magic;
  int world;
  int pad;
  std::atomic<int> attached;
  char pad0[44];
  std::atomic<uint64_t> bar_count;
  char pad1[56];
  std::atomic<uint64_t> bar_gen;
  char pad2[56];
};

struct Shm {
  std::string name;
  int rank, world;
  size_t size;
  char* base;
  Header* hdr;
  Ring* rings;     // [world][world]
  char* ag;        // [world][kAgBytes]
  int poll_start;
  std::mutex post_mu;
};

size_t seg_size(int world) {
  return sizeof(Header) + (size_t)world * world * sizeof(Ring) + (size_t)world * kAgBytes;
}

uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + ts.tv_nsec;
}

int shm_barrier(void* ctx) {
  Shm* s = (Shm*)ctx;
  uint64_t gen = s->hdr->bar_gen.load(std::memory_order_acquire);
  if (s->hdr->bar_count.fetch_add(1, std::memory_order_acq_rel) + 1 == (uint64_t)s->world) {
    s->hdr->bar_count.store(0, std::memory_order_relaxed);
    s->hdr->bar_gen.fetch_add(1, std::memory_order_acq_rel);
    return 0;
  }
  uint64_t t0 = now_ns();
  while (s->hdr->bar_gen.load(std::memory_order_acquire) == gen) {
    sched_yield();
    if (now_ns() - t0 > 300ull * 1000000000ull) return -1;
  }
  return 0;
}

int shm_allgather(void* ctx, const void* sendbuf, void* recvbuf, size_t bytes) {
  Shm* s = (Shm*)ctx;
  if (bytes > kAgBytes) return -2;
  memcpy(s->ag + (size_t)s->rank * kAgBytes, sendbuf, bytes);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  if (shm_barrier(ctx)) return -1;
  for (int r = 0; r < s->world; ++r) memcpy((char*)recvbuf + (size_t)r * bytes, s->ag + (size_t)r * kAgBytes, bytes);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  return shm_barrier(ctx);
}

int shm_post(void* ctx, int dst, const void* msg, size_t len) {
  Shm* s = (Shm*)ctx;
  if (dst < 0 || dst >= s->world || len > (size_t)kMsg) return -2;
  std::lock_guard<std::mutex> g(s->post_mu);
  Ring& rg = s->rings[(size_t)s->rank * s->world + dst];
  uint64_t h = rg.head.load(std::memory_order_relaxed);
  uint64_t t0 = now_ns();
  while (h - rg.tail.load(std::memory_order_acquire) >= (uint64_t)kSlots) {
    sched_yield();
    if (now_ns() - t0 > 10ull * 1000000000ull) return -1;
  }
  int slot = (int)(h % kSlots);
  memcpy(rg.data[slot], msg, len);
  rg.len[slot] = (uint32_t)len;
  rg.head.store(h + 1, std::memory_order_release);
  return 0;
}

int shm_poll(void* ctx, int* src, void* msg, size_t cap, size_t* len) {
  Shm* s = (Shm*)ctx;
  for (int i = 0; i < s->world; ++i) {
    int from = (s->poll_start + i) % s->world;
    Ring& rg = s->rings[(size_t)from * s->world + s->rank];
    uint64_t t = rg.tail.load(std::memory_order_relaxed);
    if (rg.head.load(std::memory_order_acquire) == t) continue;
    int slot = (int)(t % kSlots);
    size_t l = rg.len[slot];
    if (l > cap) l = cap;
    memcpy(msg, rg.data[slot], l);
    rg.tail.store(t + 1, std::memory_order_release);
    if (src) *src = from;
    if (len) *len = l;
    s->poll_start = (from + 1) % s->world;
    return 1;
  }
  return 0;
}

}  // namespace

extern "C" r2_result_t r2_oob_shm_open(const char* name, int rank, int world, r2_oob_t* out) {
  if (!name || !out || world < 1 || rank < 0 || rank >= world) return R2_ERR_INVALID_ARG;
  std::string nm = name[0] == '/' ? std::string(name) : std::string("/") + name;
  const size_t size = seg_size(world);
  int fd = -1;
  if (rank == 0) {
    shm_unlink(nm.c_str());
    fd = shm_open(nm.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) return R2_ERR_BOOTSTRAP;
    if (ftruncate(fd, (off_t)size) != 0) {
      close(fd);
      return R2_ERR_BOOTSTRAP;
    }
  } else {
    uint64_t t0 = now_ns();
    for (;;) {
      fd = shm_open(nm.c_str(), O_RDWR, 0600);
      if (fd >= 0) {
        struct stat st;
        if (fstat(fd, &st) == 0 && (size_t)st.st_size == size) break;
        close(fd);
        fd = -1;
      }
      if (now_ns() - t0 > 60ull * 1000000000ull) return R2_ERR_BOOTSTRAP;
      usleep(1000);
    }
  }
  void* p = mmap(nullptr, size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return R2_ERR_BOOTSTRAP;
  Shm* s = new Shm();
  s->name = nm;
  s->rank = rank;
  s->world = world;
  s->size = size;
  s->base = (char*)p;
  s->hdr = (Header*)p;
  s->rings = (Ring*)(s->base + sizeof(Header));
  s->ag = s->base + sizeof(Header) + (size_t)world * world * sizeof(Ring);
  s->poll_start = 0;
  if (rank == 0) {
    // fresh zero-filled segment: atomics start at 0
    s->hdr->world = world;
    s->hdr->magic.store(kMagic, std::memory_order_release);
  } else {
    uint64_t t0 = now_ns();
    while (s->hdr->magic.load(std::memory_order_acquire) != kMagic) {
      if (now_ns() - t0 > 60ull * 1000000000ull) {
        munmap(p, size);
        delete s;
        return R2_ERR_BOOTSTRAP;
      }
      usleep(100);
    }
  }
  s->hdr->attached.fetch_add(1, std::memory_order_acq_rel);
  uint64_t t0 = now_ns();
  while (s->hdr->attached.load(std::memory_order_acquire) < world) {
    if (now_ns() - t0 > 120ull * 1000000000ull) {
      munmap(p, size);
      delete s;
      return R2_ERR_BOOTSTRAP;
    }
    usleep(100);
  }
  if (rank == 0) shm_unlink(nm.c_str());   // everyone is attached: drop the name
  out->ctx = s;
  out->allgather = shm_allgather;
  out->post = shm_post;
  out->poll = shm_poll;
  out->barrier = shm_barrier;
  return R2_SUCCESS;
}

extern "C" r2_result_t r2_oob_shm_close(r2_oob_t* oob) {
  if (!oob || !oob->ctx) return R2_ERR_INVALID_ARG;
  Shm* s = (Shm*)oob->ctx;
  munmap(s->base, s->size);
  delete s;
  oob->ctx = nullptr;
  return R2_SUCCESS;
}
