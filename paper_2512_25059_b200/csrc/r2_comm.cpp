// r2_comm.cpp -- the C ABI of the R²CCL hot path: bootstrap + multi-
// registration, per-call planning (the
// planner reads the health records; plan-time Balance / HotRepair for dead
// channels), the allreduce launch, fault injection, probes and status.
#include "r2_comm.h"

#include <cuda.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <algorithm>
#include <chrono>
#include <thread>

namespace {

#define CK(x)                                  \
  do {                                         \
    cudaError_t e_ = (x);                      \
    if (e_ != cudaSuccess) return R2_ERR_CUDA; \
  } while (0)

int elem_bytes(r2_dtype_t dt) { return dt == R2_BFLOAT16 ? 2 : 4; }

constexpr int kMaxInflight = 16;   // outstanding collectives per communicator

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

ArenaLayout make_layout(int n, int K, int W, size_t chunk, size_t max_bytes, size_t ll_max_bytes, bool with_r2cc) {
  ArenaLayout L{};
  const size_t q = (size_t)n * K * 16;
  L.slot_bytes = std::max<size_t>(align_up(std::max<size_t>(max_bytes, 16), q) / n, 16 * K);
  // chunks per channel slice: a Broadcast's slice is the whole buffer / K (n times an
  // AllReduce slice)
  // a ring of any channel subset may carry the whole payload in one slice
  // (R²CCL-AllReduce rings run on channel subsets; chains cap chunks at 128 KiB)
  const size_t slice_cap = align_up(std::max<size_t>(max_bytes, 16), 16);
  const size_t bchunk = std::min<size_t>(chunk, (size_t)128 << 10);   // Broadcast chunk cap (r2_geometry_op)
  L.m_cap = (int)std::max<size_t>((slice_cap + bchunk - 1) / bchunk, (size_t)W);
  // LL: two 16-byte lines per 16-byte vector, one slot per ring step.  LL128
  // (reading R-12): each chunk owns whole 128-byte lines of 7 payload vectors,
  // so a slot needs <= K * (slice / 112 + chunks per slice + 1) lines; the
  // slot is sized for the larger of the two
  if (ll_max_bytes) {
    const size_t shard = std::max<size_t>(align_up(std::min(ll_max_bytes, max_bytes), q) / n, 16 * K);
    const size_t slice = shard / K;
    const size_t mmax = std::max<size_t>((size_t)W, (slice + chunk - 1) / chunk) + 1;
    // 128-byte multiple: every slot (and so every LL128 line) starts 128-byte aligned
    L.ll_slot_bytes = align_up(std::max<size_t>(2 * shard, (size_t)K * ((slice + 111) / 112 + mmax) * 128), 128);
  }
  const int steps = n > 1 ? 2 * n - 1 : 1;     // + the LL unpack step
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  L.scratch = take((size_t)2 * std::max(n - 1, 1) * L.slot_bytes);
  L.ll = take((size_t)2 * std::max(2 * n - 2, 1) * L.ll_slot_bytes);
  L.flags = take((size_t)steps * K * L.m_cap * 4);
  L.counters = take((size_t)steps * K * L.m_cap * 8);
  L.ep_dead = take((size_t)n * K * 4);
  L.link_dead = take((size_t)n * K * 4);
  L.alert = take(4);
  L.mailbox = take((size_t)n * K * 4);
  L.desc = take(8 * 8);
  L.misc = take(sizeof(MiscDev));
  L.stage = take(L.slot_bytes);
  L.dctrl = take(sizeof(DevCtrl));
  L.health = take((size_t)4 * n * K * 4);
  // ring 1 (R²CCL-AllReduce's partial ring over n-1 ranks, reading R-9) and the
  // stage-2 buffer where the degraded rank's contribution lands
  if (n >= 3 && with_r2cc) {
    const size_t q1 = (size_t)(n - 1) * K * 16;
    L.slot1_bytes = std::max<size_t>(align_up(std::max<size_t>(max_bytes, 16), q1) / (n - 1), 16 * K);
    L.scratch1 = take((size_t)2 * (n - 2) * L.slot1_bytes);
    L.flags1 = take((size_t)steps * K * L.m_cap * 4);
    L.counters1 = take((size_t)steps * K * L.m_cap * 8);
    L.misc1 = take(sizeof(MiscDev));
    L.stage1 = take(L.slot1_bytes);
    L.tailor_bytes = align_up(std::max<size_t>(max_bytes, 16), (size_t)K * 16);
    L.tailor = take(L.tailor_bytes);
  }
  L.total = align_up(off, 4096);
  return L;
}

// region 0: the arena as ring 0 sees it; region 1: ring 1's own scratch,
// flags, counters, misc and stage (per-rank state shared)
RankPtrs ptrs_of(char* base, const ArenaLayout& L, int region = 0) {
  RankPtrs p;
  p.scratch = base + (region ? L.scratch1 : L.scratch);
  p.ll = base + L.ll;
  p.flags = (unsigned int*)(base + (region ? L.flags1 : L.flags));
  p.counters = (unsigned long long*)(base + (region ? L.counters1 : L.counters));
  p.ep_dead = (unsigned int*)(base + L.ep_dead);
  p.link_dead = (unsigned int*)(base + L.link_dead);
  p.alert = (unsigned int*)(base + L.alert);
  p.mailbox = (unsigned int*)(base + L.mailbox);
  p.desc = (unsigned long long*)(base + L.desc);
  p.misc = (MiscDev*)(base + (region ? L.misc1 : L.misc));
  p.stage = base + (region ? L.stage1 : L.stage);
  p.dctrl = (DevCtrl*)(base + L.dctrl);
  p.health = (unsigned int*)(base + L.health);
  MiscDev* m0 = (MiscDev*)(base + L.misc);
  p.abort = &m0->abort_seq;
  p.bytes = m0->bytes;
  p.tailor = L.tailor ? base + L.tailor : nullptr;
  return p;
}

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

r2_result_t alloc_base(void* dptr, char** base, size_t* size) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
      return R2_ERR_CUDA;
    fn = (PFN_getAddressRange)f;
  }
  CUdeviceptr b = 0;
  size_t s = 0;
  if (fn(&b, &s, (CUdeviceptr)dptr) != CUDA_SUCCESS) return R2_ERR_INVALID_ARG;
  *base = (char*)b;
  *size = s;
  return R2_SUCCESS;
}

struct RegXchg {
  cudaIpcMemHandle_t h;
  unsigned long long base, dptr, bytes;
};

// Open (or reuse) the IPC mapping of `peer`'s allocation `base`.
r2_result_t open_peer(r2_comm* c, int peer, const RegXchg& x, void** out) {
  auto key = std::make_pair(peer, (unsigned long long)x.base);
  auto it = c->ipc_cache.find(key);
  if (it != c->ipc_cache.end()) {
    it->second.second++;
    *out = it->second.first;
    return R2_SUCCESS;
  }
  void* p = nullptr;
  if (cudaIpcOpenMemHandle(&p, x.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return R2_ERR_CUDA;
  c->ipc_cache[key] = std::make_pair(p, 1);
  *out = p;
  return R2_SUCCESS;
}

void close_peer(r2_comm* c, void* p) {
  for (auto it = c->ipc_cache.begin(); it != c->ipc_cache.end(); ++it)
    if (it->second.first == p) {
      if (--it->second.second == 0) {
        cudaIpcCloseMemHandle(p);
        c->ipc_cache.erase(it);
      }
      return;
    }
}

// Monitor threads of communicators never finalized (e.g. the caller exited on
// an error) are stopped at process exit, before the CUDA runtime unmaps the
// host-mapped control blocks they poll.
std::mutex g_live_mu;
std::vector<r2_comm*> g_live;
bool g_atexit_registered = false;

void stop_live_monitors() {
  std::lock_guard<std::mutex> g(g_live_mu);
  for (r2_comm* c : g_live) {
    c->stop.store(true);
    if (c->mon.joinable()) c->mon.join();
  }
  g_live.clear();
}

void track_live(r2_comm* c, bool add) {
  std::lock_guard<std::mutex> g(g_live_mu);
  if (add) {
    g_live.push_back(c);
    if (!g_atexit_registered) {
      std::atexit(stop_live_monitors);
      g_atexit_registered = true;
    }
  } else {
    g_live.erase(std::remove(g_live.begin(), g_live.end(), c), g_live.end());
  }
}

// Every resource r2_init may have acquired (null / empty members are
// skipped): the error path of r2_init and r2_finalize share it.
void release_resources(r2_comm* c) {
  for (auto& rg : c->regs)
    for (void* p : rg.opened) close_peer(c, p);
  c->regs.clear();
  for (void* p : c->peer_arena_opened)
    if (p) cudaIpcCloseMemHandle(p);
  c->peer_arena_opened.clear();
  for (char* a : c->arena)
    if (a) cudaFree(a);
  c->arena.clear();
  for (Ctrl* h : c->ctrl_host)
    if (h) cudaFreeHost(h);
  c->ctrl_host.clear();
  if (c->probe_res_host) cudaFreeHost((void*)c->probe_res_host);
  if (c->probe_t0_host) cudaFreeHost((void*)c->probe_t0_host);
  if (c->svc_host) cudaFreeHost(c->svc_host);
  if (c->flags_map_host) cudaFreeHost(c->flags_map_host);
  if (c->health_map_host) cudaFreeHost(c->health_map_host);
  if (c->health_pinned) cudaFreeHost(c->health_pinned);
  if (c->peers_dev) cudaFree(c->peers_dev);
  if (c->peers_dev1) cudaFree(c->peers_dev1);
  if (c->regtab_dev) cudaFree(c->regtab_dev);
  if (c->host_stage) cudaFree(c->host_stage);
  for (auto& ev : c->host_ev) cudaEventDestroy(ev);
  if (c->svc_ev) cudaEventDestroy(c->svc_ev);
  cudaStream_t streams[] = {c->h2d_stream, c->d2h_stream, c->mon_stream, c->health_stream, c->svc_stream};
  for (cudaStream_t s : streams)
    if (s) cudaStreamDestroy(s);
  for (int i = 0; i < r2_comm::kProbeStreams; ++i)
    if (c->probe_stream[i]) cudaStreamDestroy(c->probe_stream[i]);
}

// host-mapped pinned block: host pointer + device alias
template <class T>
bool alloc_mapped(size_t bytes, T** host, T** dev) {
  void* h = nullptr;
  if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped) != cudaSuccess) return false;
  memset(h, 0, bytes);
  *host = (T*)h;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return false;
  *dev = (T*)d;
  return true;
}

int take_async_error(r2_comm* c) {
  std::lock_guard<std::mutex> g(c->mu);
  int e = c->unreported_error;
  c->unreported_error = R2_SUCCESS;
  return e;
}

}  // namespace

int r2_debug = getenv("R2_DEBUG") ? atoi(getenv("R2_DEBUG")) : 0;

uint64_t r2_now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + ts.tv_nsec;
}

extern "C" void r2_config_default(r2_config_t* cfg) {
  if (!cfg) return;
  memset(cfg, 0, sizeof(*cfg));
  cfg->nchannels = 8;
  cfg->ctas_per_channel = 4;
  cfg->threads_per_cta = 512;
  cfg->chunk_bytes = 512 * 1024;
  cfg->max_bytes = (size_t)1 << 30;
  cfg->strategy = R2_BALANCE;
  cfg->probe_timeout_us = 50;
  cfg->watchdog_ms = 3000;
  cfg->use_channel_w = 0;
  cfg->rerank = 1;
  cfg->r2cc_stage1_eff_pct = 75;   // measured stage efficiencies (profiles/r02_summary.md, R²CCL stages)
  cfg->r2cc_stage2_eff_pct = 50;
  for (int i = 0; i < R2_MAX_CHANNELS; ++i) cfg->channel_w[i] = 1;
  cfg->sim_ranks = 1;
  cfg->protocol = R2_PROTO_AUTO;
  cfg->ll_max_bytes = (size_t)128 << 20;  // covers the LL128 / SIMPLE crossovers (reading R-12)
  // fitted to the forced-protocol sweeps at n = 2 and 4 (profiles/r02_protocols_n{2,4}.jsonl):
  // they reproduce the measured crossovers LL -> LL128 at 2 MB (n=2) / 3 MB (n=4)
  // and LL128 -> SIMPLE at ~21-25 MB (n=2) / ~60 MB (n=4)
  cfg->alpha_simple_ns = 6400;     // per ring step, SIMPLE (fence + completion word + publish)
  cfg->alpha_ll_ns = 2050;         // per ring step, LL (one line flight)
  cfg->beta_mbps = 700000;         // per-GPU NVLink store rate at large sizes
  cfg->reprobe_us = 2000;
  cfg->reprobe_max_us = 200000;
  cfg->allreduce_algo = R2_ALGO_AUTO;
  cfg->alpha_launch_ns = 6000;     // one cooperative launch + prologue (profiles/r01_host_overhead_n4.log)
  cfg->alpha_ll128_ns = 2850;      // per ring step, LL128 (one 128-byte line flight + the warp's flag check)
}

extern "C" r2_result_t r2_init(int rank, int world, int cuda_dev, const r2_oob_t* oob, const r2_config_t* cfg_in,
                               r2_comm_t* out) {
  if (!out) return R2_ERR_INVALID_ARG;
  *out = nullptr;
  r2_config_t cfg;
  if (cfg_in) cfg = *cfg_in;
  else r2_config_default(&cfg);
  if (world < 1 || rank < 0 || rank >= world) return R2_ERR_INVALID_ARG;
  if (cfg.nchannels < 1 || cfg.nchannels > R2_MAXK || cfg.ctas_per_channel < 1 || cfg.ctas_per_channel > R2_MAXW)
    return R2_ERR_INVALID_ARG;
  // warp 0 controls, warps 1.. move data: at least 2 warps per CTA
  if (cfg.threads_per_cta < 64 || cfg.threads_per_cta > 512 || cfg.threads_per_cta % 32) return R2_ERR_INVALID_ARG;
  if (cfg.chunk_bytes < 16 || cfg.chunk_bytes % 16 || cfg.max_bytes < 16) return R2_ERR_INVALID_ARG;
  if (cfg.strategy != R2_HOT_REPAIR && cfg.strategy != R2_BALANCE) return R2_ERR_INVALID_ARG;
  if (cfg.sim_ranks < 1 || cfg.sim_ranks > R2_MAXL || (world > 1 && cfg.sim_ranks != 1)) return R2_ERR_INVALID_ARG;
  if (world > 1 && (!oob || !oob->allgather || !oob->post || !oob->poll || !oob->barrier)) return R2_ERR_INVALID_ARG;
  if (world > R2_MAX_LOCAL * 4) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(cuda_dev) != cudaSuccess) return R2_ERR_CUDA;

  r2_comm* c = new r2_comm();
  c->rank = rank;
  c->world = world;
  c->dev = cuda_dev;
  c->cfg = cfg;
  c->sim = (world == 1 && cfg.sim_ranks > 1);
  c->n = c->sim ? cfg.sim_ranks : world;
  c->nlocal = c->sim ? c->n : 1;
  c->first_rank = c->sim ? 0 : rank;
  c->K = cfg.nchannels;
  c->W = cfg.ctas_per_channel;
  c->threads = cfg.threads_per_cta;
  c->ll_threads = getenv("R2_LL_THREADS") ? atoi(getenv("R2_LL_THREADS")) : 0;
  if (c->ll_threads != 0 && (c->ll_threads < 64 || c->ll_threads > 512 || c->ll_threads % 32)) c->ll_threads = 0;
  c->trace = getenv("R2_TRACE") ? atoi(getenv("R2_TRACE")) : 0;
  for (int k = 0; k < c->K; ++k) c->weights[k] = cfg.use_channel_w ? (unsigned)std::max(cfg.channel_w[k], 1) : 1u;
  if (oob) {
    c->oob = *oob;
    c->has_oob = world > 1;
  }
  if (cfg.protocol < R2_PROTO_AUTO || cfg.protocol > R2_PROTO_LL128) {
    delete c;
    return R2_ERR_INVALID_ARG;
  }
  if (cfg.allreduce_algo < R2_ALGO_AUTO || cfg.allreduce_algo > R2_ALGO_R2CC) {
    delete c;
    return R2_ERR_INVALID_ARG;
  }
  c->lay = make_layout(c->n, c->K, c->W, cfg.chunk_bytes, cfg.max_bytes, cfg.ll_max_bytes,
                       cfg.allreduce_algo != R2_ALGO_RING);
  auto fail = [&](r2_result_t e) {
    cudaDeviceSynchronize();
    release_resources(c);
    delete c;
    return e;
  };
  if (c->n > 1) {
    c->max_coop = r2_max_coop_ctas(std::max(std::max(c->threads, c->ll_threads), 512));
    if (c->nlocal * c->K * c->W > c->max_coop) return fail(R2_ERR_INVALID_ARG);
  }

  // ---- arenas (scratch, flags, counters, fabric state, mailboxes)
  c->arena.assign(c->nlocal, nullptr);
  c->ctrl_host.assign(c->nlocal, nullptr);
  c->ctrl_dev.assign(c->nlocal, nullptr);
  for (int l = 0; l < c->nlocal; ++l) {
    if (cudaMalloc(&c->arena[l], c->lay.total) != cudaSuccess) return fail(R2_ERR_CUDA);
    if (cudaMemset(c->arena[l], 0, c->lay.total) != cudaSuccess) return fail(R2_ERR_CUDA);
    void* h = nullptr;
    if (cudaHostAlloc(&h, sizeof(Ctrl), cudaHostAllocMapped) != cudaSuccess) return fail(R2_ERR_CUDA);
    memset(h, 0, sizeof(Ctrl));
    c->ctrl_host[l] = (Ctrl*)h;
    void* d = nullptr;
    if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return fail(R2_ERR_CUDA);
    c->ctrl_dev[l] = (Ctrl*)d;
  }
  {
    void* h = nullptr;
    if (cudaHostAlloc(&h, sizeof(int) * r2_comm::kProbeSlots, cudaHostAllocMapped) != cudaSuccess)
      return fail(R2_ERR_CUDA);
    c->probe_res_host = (volatile int*)h;
    for (int i = 0; i < r2_comm::kProbeSlots; ++i) c->probe_res_host[i] = -1;
    void* d = nullptr;
    if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return fail(R2_ERR_CUDA);
    c->probe_res_dev = (int*)d;
    if (cudaHostAlloc(&h, sizeof(unsigned long long) * r2_comm::kProbeSlots, cudaHostAllocMapped) != cudaSuccess)
      return fail(R2_ERR_CUDA);
    c->probe_t0_host = (volatile unsigned long long*)h;
    memset(h, 0, sizeof(unsigned long long) * r2_comm::kProbeSlots);
    if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return fail(R2_ERR_CUDA);
    c->probe_t0_dev = (unsigned long long*)d;
    if (!alloc_mapped(sizeof(SvcBlock), &c->svc_host, &c->svc_dev)) return fail(R2_ERR_CUDA);
    const size_t flag_words = (size_t)(c->n > 1 ? 2 * c->n - 1 : 1) * c->K * c->lay.m_cap;
    if (!alloc_mapped(flag_words * 4, &c->flags_map_host, &c->flags_map_dev)) return fail(R2_ERR_CUDA);
    if (!alloc_mapped((size_t)4 * c->n * c->K * 4, &c->health_map_host, &c->health_map_dev)) return fail(R2_ERR_CUDA);
    if (cudaStreamCreateWithFlags(&c->svc_stream, cudaStreamNonBlocking) != cudaSuccess) return fail(R2_ERR_CUDA);
    if (cudaEventCreateWithFlags(&c->svc_ev, cudaEventDisableTiming) != cudaSuccess) return fail(R2_ERR_CUDA);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(R2_ERR_CUDA);

  // ---- map every peer's arena (multi-registration at init)
  c->peers_host.assign((size_t)c->nlocal * c->n, RankPtrs{});
  c->peers_host1.assign((size_t)c->nlocal * c->n, RankPtrs{});
  if (c->sim) {
    for (int l = 0; l < c->nlocal; ++l)
      for (int p = 0; p < c->n; ++p) {
        c->peers_host[l * c->n + p] = ptrs_of(c->arena[p], c->lay);
        c->peers_host1[l * c->n + p] = ptrs_of(c->arena[p], c->lay, 1);
      }
  } else if (world == 1) {
    c->peers_host[0] = ptrs_of(c->arena[0], c->lay);
    c->peers_host1[0] = ptrs_of(c->arena[0], c->lay, 1);
  } else {
    RegXchg mine{};
    if (cudaIpcGetMemHandle(&mine.h, c->arena[0]) != cudaSuccess) return fail(R2_ERR_CUDA);
    mine.base = (unsigned long long)c->arena[0];
    std::vector<RegXchg> all(world);
    if (c->oob.allgather(c->oob.ctx, &mine, all.data(), sizeof(RegXchg))) return fail(R2_ERR_BOOTSTRAP);
    c->peer_arena_opened.assign(world, nullptr);
    for (int p = 0; p < world; ++p) {
      char* b = c->arena[0];
      if (p != rank) {
        void* op = nullptr;
        if (cudaIpcOpenMemHandle(&op, all[p].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
          return fail(R2_ERR_CUDA);
        c->peer_arena_opened[p] = op;
        b = (char*)op;
      }
      c->peers_host[p] = ptrs_of(b, c->lay);
      c->peers_host1[p] = ptrs_of(b, c->lay, 1);
    }
  }
  for (int region = 0; region < 2; ++region) {
    std::vector<RankPtrs>& h = region ? c->peers_host1 : c->peers_host;
    RankPtrs*& d = region ? c->peers_dev1 : c->peers_dev;
    if (cudaMalloc(&d, sizeof(RankPtrs) * h.size()) != cudaSuccess) return fail(R2_ERR_CUDA);
    if (cudaMemcpy(d, h.data(), sizeof(RankPtrs) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(R2_ERR_CUDA);
  }
  c->regtab_host.assign((size_t)R2_MAX_REGS * c->n, 0ull);
  if (cudaMalloc(&c->regtab_dev, sizeof(unsigned long long) * c->regtab_host.size()) != cudaSuccess)
    return fail(R2_ERR_CUDA);
  if (cudaMemset(c->regtab_dev, 0, sizeof(unsigned long long) * c->regtab_host.size()) != cudaSuccess)
    return fail(R2_ERR_CUDA);

  c->health.assign((size_t)4 * c->n * c->K, 0u);
  if (cudaStreamCreateWithFlags(&c->health_stream, cudaStreamNonBlocking) != cudaSuccess) return fail(R2_ERR_CUDA);
  c->handled_err.assign((size_t)c->nlocal * c->K, 0);
  c->timeout_seq.assign(c->nlocal, 0);
  c->epoch.assign(c->nlocal, 0);
  c->plan_seq.assign(c->nlocal, 0);
  c->cur_plan.assign(c->nlocal, {});
  if (cudaStreamCreateWithFlags(&c->mon_stream, cudaStreamNonBlocking) != cudaSuccess) return fail(R2_ERR_CUDA);
  for (int i = 0; i < r2_comm::kProbeStreams; ++i)
    if (cudaStreamCreateWithFlags(&c->probe_stream[i], cudaStreamNonBlocking) != cudaSuccess)
      return fail(R2_ERR_CUDA);
  {
    void* h = nullptr;
    if (cudaHostAlloc(&h, c->health.size() * sizeof(uint32_t), cudaHostAllocDefault) != cudaSuccess)
      return fail(R2_ERR_CUDA);
    c->health_pinned = (uint32_t*)h;
  }
  if (c->n > 1) {
    // pre-load the kernels (see r2_warmup): a healthy self-probe
    const RankPtrs& me = c->peers_host[c->first_rank];
    ProbeParams pp{};
    pp.target_mailbox = me.mailbox + c->first_rank * c->K;
    pp.ep_dead = me.ep_dead;
    pp.link_dead = me.link_dead;
    pp.prober = pp.target = c->first_rank;
    pp.channel = 0;
    pp.n = c->n;
    pp.K = c->K;
    pp.token = 0x5eed;
    pp.timeout_ns = 1000000ull;
    pp.result = c->probe_res_dev + (r2_comm::kProbeSlots - 1);
    if (r2_warmup(pp, c->mon_stream) != 0) return fail(R2_ERR_CUDA);
    c->probe_res_host[r2_comm::kProbeSlots - 1] = -1;
    // host CLOCK_MONOTONIC <-> device %globaltimer offset (failover timelines):
    // best of a few probe launches, midpoint of the host window
    pp.t_start = c->probe_t0_dev + (r2_comm::kProbeSlots - 1);
    long long best_w = -1;
    for (int i = 0; i < 5; ++i) {
      c->probe_t0_host[r2_comm::kProbeSlots - 1] = 0;
      const uint64_t h0 = r2_now_ns();
      if (r2_launch_probe(pp, c->mon_stream) != 0) return fail(R2_ERR_CUDA);
      while (c->probe_t0_host[r2_comm::kProbeSlots - 1] == 0) {
      }
      const uint64_t h1 = r2_now_ns();
      const long long w = (long long)(h1 - h0);
      if (best_w < 0 || w < best_w) {
        best_w = w;
        c->clk_offset = (long long)c->probe_t0_host[r2_comm::kProbeSlots - 1] - (long long)((h0 + h1) / 2);
      }
    }
    cudaStreamSynchronize(c->mon_stream);
    c->probe_res_host[r2_comm::kProbeSlots - 1] = -1;
  }
  if (c->has_oob && c->oob.barrier(c->oob.ctx)) return fail(R2_ERR_BOOTSTRAP);
  if (c->n > 1) {
    c->mon = std::thread(r2_monitor_main, c);
    track_live(c, true);
  }
  *out = c;
  return R2_SUCCESS;
}

extern "C" r2_result_t r2_register_multi(r2_comm_t c, void* dptr, size_t bytes, uint64_t* reg_out) {
  if (!c || !dptr || !reg_out) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(c->dev) != cudaSuccess) return R2_ERR_CUDA;
  if (c->sim || c->world == 1) {
    Reg rg{(uint64_t)c->regs.size(), true, (char*)dptr, bytes, {}, {}};
    c->regs.push_back(rg);
    *reg_out = rg.id;
    return R2_SUCCESS;
  }
  if (c->regs.size() >= R2_MAX_REGS) return R2_ERR_INVALID_ARG;
  char* base = nullptr;
  size_t size = 0;
  r2_result_t e = alloc_base(dptr, &base, &size);
  if (e != R2_SUCCESS) return e;
  if ((char*)dptr + bytes > base + size) return R2_ERR_INVALID_ARG;
  RegXchg mine{};
  CK(cudaIpcGetMemHandle(&mine.h, base));
  mine.base = (unsigned long long)base;
  mine.dptr = (unsigned long long)dptr;
  mine.bytes = bytes;
  std::vector<RegXchg> all(c->world);
  if (c->oob.allgather(c->oob.ctx, &mine, all.data(), sizeof(RegXchg))) return R2_ERR_BOOTSTRAP;
  Reg rg;
  rg.id = c->regs.size();
  rg.active = true;
  rg.dptr = (char*)dptr;
  rg.bytes = bytes;
  rg.peer_ptr.assign(c->world, 0);
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) {
      rg.peer_ptr[p] = (unsigned long long)dptr;
      continue;
    }
    void* op = nullptr;
    e = open_peer(c, p, all[p], &op);
    if (e != R2_SUCCESS) return e;
    rg.opened.push_back(op);
    rg.peer_ptr[p] = (unsigned long long)op + (all[p].dptr - all[p].base);
  }
  for (int p = 0; p < c->world; ++p) c->regtab_host[rg.id * c->n + p] = rg.peer_ptr[p];
  CK(cudaMemcpy(c->regtab_dev + rg.id * c->n, &c->regtab_host[rg.id * c->n], sizeof(unsigned long long) * c->n,
                cudaMemcpyHostToDevice));
  c->regs.push_back(rg);
  *reg_out = rg.id;
  return R2_SUCCESS;
}

extern "C" r2_result_t r2_deregister(r2_comm_t c, uint64_t reg) {
  if (!c || reg >= c->regs.size() || !c->regs[reg].active) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(c->dev) != cudaSuccess) return R2_ERR_CUDA;
  if (c->has_oob && c->oob.barrier(c->oob.ctx)) return R2_ERR_BOOTSTRAP;
  Reg& rg = c->regs[reg];
  for (void* p : rg.opened) close_peer(c, p);
  rg.opened.clear();
  rg.active = false;
  return R2_SUCCESS;
}

extern "C" r2_result_t r2_inject_fault(r2_comm_t c, const r2_fault_t* f) {
  if (!c || !f) return R2_ERR_INVALID_ARG;
  if (f->kind < R2_FAULT_LOCAL || f->kind > R2_FAULT_HEAL) return R2_ERR_INVALID_ARG;
  if (f->src_rank < 0 || f->src_rank >= c->n || f->channel < 0 || f->channel >= c->K) return R2_ERR_INVALID_ARG;
  if (f->origin_channel < -1 || f->origin_channel >= c->K) return R2_ERR_INVALID_ARG;
  if (f->kind <= R2_FAULT_LINK && (f->step < 0 || f->chunk < 0)) return R2_ERR_INVALID_ARG;
  if (f->at_seq <= c->seq) return R2_ERR_INVALID_ARG;   // must precede the targeted collective
  c->faults.push_back(*f);
  return R2_SUCCESS;
}

// One ring of a launch: which ranks in which order, on which channels, over
// which part of the user buffers (r2_internal.h LaunchParams).
struct RingSpec {
  r2_op_t op = R2_OP_ALLREDUCE;
  const void* send = nullptr;                // region start in the user buffers
  void* recv = nullptr;
  size_t count = 0;                          // elements of the region (op convention)
  int root = 0;                              // chain collectives: root's ring position
  std::vector<int> order;                    // global rank at each ring position
  std::vector<int> chans;                    // global channels, ring-local order
  int region = 0;                            // arena region set (0 / 1)
  size_t peer_recv_off = 0;                  // bytes: region start inside a peer's registered recv
  bool allow_ll = true;                      // the alpha-beta protocol choice may pick LL
  size_t row_elems = 0;                      // sim mode: elements of a full rank row (0: the region's own)
};

RingSpec standard_ring(const r2_comm* c, r2_op_t op, const void* send, void* recv, size_t count, int root) {
  RingSpec rs;
  rs.op = op;
  rs.send = send;
  rs.recv = recv;
  rs.count = count;
  rs.root = root;
  for (int r = 0; r < c->n; ++r) rs.order.push_back(r);
  for (int k = 0; k < c->K; ++k) rs.chans.push_back(k);
  return rs;
}

// Geometry, protocol and every LaunchParams field of one ring (no faults).
r2_result_t prep_ring(r2_comm* c, const RingSpec& rs, r2_dtype_t dt, uint32_t seq, LaunchParams& p, RingInfo& ri) {
  const r2_op_t op = rs.op;
  const int E = elem_bytes(dt);
  const int n = (int)rs.order.size(), K = (int)rs.chans.size();
  const size_t count = rs.count;
  r2_geometry_t g;
  r2_result_t e = r2_geometry_op(op, count, dt, n, K, c->W, c->cfg.chunk_bytes, &g);
  if (e != R2_SUCCESS) return e;
  const size_t slot = rs.region ? c->lay.slot1_bytes : c->lay.slot_bytes;
  const bool chain = op == R2_OP_BROADCAST || op == R2_OP_R2CC_STAGE2;
  if ((!chain && g.shard * E > slot) || g.m > c->lay.m_cap) return R2_ERR_INVALID_ARG;
  if (op == R2_OP_R2CC_STAGE2 && g.Np * E > c->lay.tailor_bytes) return R2_ERR_INVALID_ARG;
  // protocol: alpha-beta model over the ring's steps; LL
  // moves twice the bytes, LL128 8/7 of them, but neither pays a fence per
  // step (r2ccl.h "Protocols").  ll: 0 SIMPLE, 1 LL, 2 LL128
  int ll = 0;
  const bool lines_ok = rs.allow_ll && rs.region == 0 && c->lay.ll_slot_bytes;
  const bool ll_fits = lines_ok && 2 * g.shard * (size_t)E <= c->lay.ll_slot_bytes;
  const size_t lc = (g.chunk / g.V + 6) / 7;                       // LL128 lines per chunk
  const bool l128_fits = lines_ok && (size_t)K * g.m * lc * 128 <= c->lay.ll_slot_bytes;
  if (chain || !rs.allow_ll) {
    ll = 0;                                            // chains: always SIMPLE (r2ccl.h)
  } else if (c->cfg.protocol == R2_PROTO_LL) {
    if (!ll_fits) return R2_ERR_INVALID_ARG;
    ll = 1;
  } else if (c->cfg.protocol == R2_PROTO_LL128) {
    if (!l128_fits) return R2_ERR_INVALID_ARG;
    ll = 2;
  } else if (c->cfg.protocol == R2_PROTO_AUTO && (ll_fits || l128_fits)) {
    const double wire = (double)(op == R2_OP_ALLREDUCE ? 2 : 1) * (n - 1) * (double)g.shard * E;
    const double bpns = std::max(c->cfg.beta_mbps, 1) / 1000.0;
    const int unpack = op != R2_OP_REDUCE_SCATTER;
    double best = g.steps * (double)c->cfg.alpha_simple_ns + wire / bpns;
    if (ll_fits) {
      const double t = (g.steps + unpack) * (double)c->cfg.alpha_ll_ns + 2 * wire / bpns;
      if (t < best) best = t, ll = 1;
    }
    if (l128_fits) {
      const double t = (g.steps + unpack) * (double)c->cfg.alpha_ll128_ns + 8.0 / 7.0 * wire / bpns;
      if (t < best) best = t, ll = 2;
    }
  }
  const int steps = g.steps + (ll && op != R2_OP_REDUCE_SCATTER ? 1 : 0);   // + the LL unpack step
  const int local_step = ll && op != R2_OP_REDUCE_SCATTER ? steps - 1 : g.local_step;

  memset(&p, 0, sizeof(p));
  p.seq = seq;
  p.n = n;
  p.K = K;
  p.W = c->W;
  p.m = g.m;
  p.steps = steps;
  p.first_rank = c->first_rank;
  p.ng = c->n;
  p.Kg = c->K;
  p.ring_id = rs.region;
  for (int i = 0; i < n; ++i) p.ring[i] = rs.order[i];
  for (int i = 0; i < K; ++i) p.chan[i] = rs.chans[i];
  // participants: this process's ranks that are on the ring
  for (int l = 0; l < c->nlocal; ++l)
    if (std::find(rs.order.begin(), rs.order.end(), c->first_rank + l) != rs.order.end()) p.part_l[p.nlocal++] = l;
  p.dtype = dt == R2_INT32 ? R2D_INT32 : (dt == R2_FLOAT32 ? R2D_FLOAT32 : R2D_BF16);
  p.elem_bytes = E;
  p.V = g.V;
  p.op = op;
  p.t0 = g.t0;
  p.local_step = local_step;
  p.fin_step = local_step >= 0 ? local_step - 1 : steps - 1;   // last step with incoming words
  p.peer_recv = !ll && op != R2_OP_REDUCE_SCATTER;
  p.peer_recv_off = rs.peer_recv_off;
  p.ll = ll;
  p.ll_slot_bytes = c->lay.ll_slot_bytes;
  if (c->cfg.channel_gbps > 0)          // lane rate = channel rate / W
    p.lane_ps_per_byte = (unsigned int)((1000ull * c->W + c->cfg.channel_gbps / 2) / c->cfg.channel_gbps);
  p.cvec_full = (unsigned int)(g.chunk / g.V);
  p.cvec_last = g.m ? (unsigned int)((g.slice - (uint64_t)(g.m - 1) * g.chunk) / g.V) : 0u;
  p.lc128 = (p.cvec_full + 6) / 7;
  p.sstride = g.stride;
  p.slen = op == R2_OP_ALLREDUCE ? g.shard : count;
  const size_t shard_bytes = count * (size_t)E;
  const void* send = rs.send;
  void* recv = rs.recv;
  p.inplace = op == R2_OP_ALLREDUCE && send == recv;
  if (op == R2_OP_ALL_GATHER && !c->sim)
    p.ag_inplace = (const char*)send == (const char*)recv + (size_t)c->rank * shard_bytes;
  if (c->sim && (op == R2_OP_REDUCE_SCATTER || op == R2_OP_ALL_GATHER) && (send == recv))
    return R2_ERR_INVALID_ARG;   // sim: out-of-place only
  if (chain) {
    p.root = rs.root;
    p.ag_inplace = send == recv;                       // root: no local copy
  }
  p.strategy = c->cfg.strategy;
  p.sim = c->sim;
  p.N = g.N;
  p.Np = g.Np;
  p.shard = g.shard;
  p.slice = g.slice;
  p.chunk = g.chunk;
  p.slot_bytes = slot;
  p.watchdog_ns = (unsigned long long)c->cfg.watchdog_ms * 1000000ull;
  p.trace = c->trace;
  for (int k = 0; k < K; ++k) p.weights[k] = c->weights[rs.chans[k]];
  p.peers = rs.region ? c->peers_dev1 : c->peers_dev;
  p.regtab = c->regtab_dev;
  p.svc = c->svc_dev;
  p.grid_exited = &((MiscDev*)(c->arena[0] + c->lay.misc))->grid_exited;   // local rank 0, ring-0 misc

  // rank buffers: sim mode rows of the FULL user buffers (16-B aligned); the
  // region starts at send / recv of rank 0's row
  const size_t full = align_up((size_t)rs.row_elems * E, 16);
  const size_t part = align_up(count * E, 16);
  const size_t sstride = rs.row_elems ? full : (op == R2_OP_ALL_GATHER ? part : align_up((size_t)g.N * E, 16));
  const size_t rstride = rs.row_elems ? full : (op == R2_OP_REDUCE_SCATTER ? part : align_up((size_t)g.N * E, 16));
  for (int l = 0; l < c->nlocal; ++l) {
    p.send[l] = (const char*)send + (size_t)l * sstride;
    p.recv[l] = (char*)recv + (size_t)l * rstride;
    p.ctrl[l] = c->ctrl_dev[l];
  }
  if (!c->sim && p.peer_recv) {
    const size_t rbytes = (size_t)g.N * E;
    int found = -1;
    for (size_t i = 0; i < c->regs.size(); ++i) {
      const Reg& rg = c->regs[i];
      if (rg.active && (char*)recv >= rg.dptr && (char*)recv + rbytes <= rg.dptr + rg.bytes) {
        found = (int)i;
        break;
      }
    }
    if (found < 0) return R2_ERR_NOT_REGISTERED;
    p.recv_reg[0] = found;
    p.recv_off[0] = (unsigned long long)((char*)recv - c->regs[found].dptr);
  }

  memset(&ri, 0, sizeof(ri));
  ri.op = op;
  ri.root = rs.root;
  ri.local_step = local_step;
  ri.ll = ll;
  ri.m = g.m;
  ri.steps = steps;
  ri.V = g.V;
  ri.slice = g.slice;
  ri.chunk = g.chunk;
  ri.n = n;
  ri.K = K;
  ri.region = rs.region;
  for (int i = 0; i < n; ++i) ri.order[i] = rs.order[i];
  for (int i = 0; i < K; ++i) {
    ri.chans[i] = rs.chans[i];
    ri.chan_mask |= 1u << rs.chans[i];
  }
  return R2_SUCCESS;
}

// One launch (one seq): its rings run concurrently in one cooperative grid
// (+ the service CTA).  Faults armed for the seq go to the ring carrying
// their channel (ring-local step / chunk / origin).
r2_result_t launch_rings(r2_comm* c, std::vector<RingSpec>& rings, r2_dtype_t dt, void* stream) {
  const uint64_t t_in = r2_debug >= 2 ? r2_now_ns() : 0;
  const uint32_t seq = (uint32_t)(c->seq + 1);
  LaunchSet S;
  memset(&S, 0, sizeof(S));
  LaunchInfo li{};
  li.seq = seq;
  S.nrings = 0;
  unsigned int exit_target = 0;
  for (size_t i = 0; i < rings.size(); ++i) {
    LaunchParams& p = S.ring[S.nrings];
    RingInfo& ri = li.ring[S.nrings];
    r2_result_t e = prep_ring(c, rings[i], dt, seq, p, ri);
    if (e != R2_SUCCESS) return e;
    if (p.nlocal == 0) continue;                       // none of this process's ranks is on the ring
    S.nctas[S.nrings] = p.nlocal * p.K * p.W;
    exit_target += (unsigned)p.nlocal;
    S.nrings++;
  }
  li.nrings = S.nrings;
  if (S.nrings == 0) return R2_SUCCESS;
  int total = 0;
  for (int i = 0; i < S.nrings; ++i) total += S.nctas[i];
  if (total > c->max_coop) return R2_ERR_INVALID_ARG;
  for (int i = 0; i < S.nrings; ++i) S.ring[i].exit_target = exit_target;

  // faults armed for this seq; REPAIRs take effect before it (stand-in for
  // re-probe); HEALs only repair the emulated fabric (found by re-probing)
  std::vector<std::pair<int, int>> repairs, heals;
  for (const r2_fault_t& f : c->faults) {
    if (f.at_seq != seq) continue;
    if (f.kind == R2_FAULT_REPAIR || f.kind == R2_FAULT_HEAL) {
      (f.kind == R2_FAULT_REPAIR ? repairs : heals).push_back({f.src_rank, f.channel});
      continue;
    }
    const int origin = f.origin_channel < 0 ? f.channel : f.origin_channel;
    for (int i = 0; i < S.nrings; ++i) {
      LaunchParams& p = S.ring[i];
      const RingInfo& ri = li.ring[i];
      const int ci = ri.local_of(f.channel), oi = ri.local_of(origin);
      if (ci < 0 || oi < 0 || ri.pos_of(f.src_rank) < 0) continue;       // not this ring's connection
      if (f.step >= p.steps || f.chunk >= p.m || f.step == p.local_step) continue;   // no such send: never fires
      const int pos = ri.pos_of(f.src_rank);
      const bool std_link = ri.order[(pos + 1) % ri.n] == (f.src_rank + 1) % c->n;
      if (f.kind == R2_FAULT_LINK && !std_link) continue;      // reading R-10: no such link
      if ((p.op == R2_OP_BROADCAST || p.op == R2_OP_R2CC_STAGE2) &&
          f.step != ((pos - p.root) % p.n + p.n) % p.n)
        continue;
      if (p.nfaults >= R2_MAXF || li.nfaults >= R2_MAXF) return R2_ERR_INVALID_ARG;
      FaultDev& d = p.faults[p.nfaults++];
      d.rank = f.src_rank;
      d.channel = f.channel;                          // global (matched against the CTA's global channel)
      d.origin = oi;                                  // ring-local (geometry)
      d.kind = f.kind;
      d.t = f.step;
      d.j = f.chunk;
      d.b = f.byte_offset;
      d.detect_delay_us = f.detect_delay_us;
      d.poison = f.poison;
      FaultDev& h = li.faults[li.nfaults++];          // the monitor's copy: global ids
      h = d;
      h.origin = origin;
    }
  }
  {
    std::lock_guard<std::mutex> gl(c->mu);
    // REPAIR re-admits (rank, channel) from this seq on (seq-indexed: no
    // ordering against collectives already in flight is needed)
    for (auto& rc : repairs) r2_declare_repaired(c, rc.first, rc.second, seq);
    // connections the monitor's re-probes found healthy again (f4)
    const bool readmit = !c->readmit_pending.empty();
    for (auto& rc : c->readmit_pending) r2_declare_conn_repaired(c, rc.first, rc.second, seq);
    c->readmit_pending.clear();
    if ((!repairs.empty() || readmit) && r2_push_health(c) != 0) return R2_ERR_CUDA;
    // speculation (line protocols, reading R-6) on every ring, static degraded
    // plans included: a mid-call plan change makes the lanes abandon their
    // spinning items before they take on a residual (r2_kernels.cu
    // control_run), which breaks the cycle a static Balance plan could
    // otherwise close (parts of one channel in another channel's lane)
    static const int no_spec = getenv("R2_NO_SPECULATION") ? atoi(getenv("R2_NO_SPECULATION")) : 0;
    for (int i = 0; i < S.nrings; ++i) S.ring[i].spec_ok = !no_spec;
    // a ring connection with no healthy channel left: the chain is exhausted
    for (int i = 0; i < S.nrings; ++i) {
      const RingInfo& ri = li.ring[i];
      for (int j = 0; j < S.ring[i].nlocal; ++j) {
        const int r = c->first_rank + S.ring[i].part_l[j], to = ri.next_of(r);
        bool any = false;
        for (int k = 0; k < ri.K; ++k) any |= r2_conn_ok_to(c, r, to, ri.chans[k], seq);
        if (!any) return R2_ERR_NO_BACKUP;
      }
    }
  }
  // the emulated fabric heals in stream order
  for (auto& h : heals) repairs.push_back(h);
  for (auto& rc : repairs)
    for (int l = 0; l < c->nlocal; ++l) {
      const RankPtrs& me = c->peers_host[l * c->n + c->first_rank + l];
      CK(cudaMemsetAsync(me.ep_dead + rc.first * c->K + rc.second, 0, 4, (cudaStream_t)stream));
      CK(cudaMemsetAsync(me.link_dead + rc.first * c->K + rc.second, 0, 4, (cudaStream_t)stream));
    }
  {
    std::lock_guard<std::mutex> gl(c->mu);
    c->launches[seq] = li;
    while (c->launches.size() > 64) c->launches.erase(c->launches.begin());
  }
  // bounded run-ahead: a full device launch queue would block the monitor's
  // standalone service kernel behind a spinning collective, so at most
  // kMaxInflight collectives are outstanding
  const uint64_t t_win0 = r2_debug >= 2 ? r2_now_ns() : 0;
  {
    const uint64_t t0 = r2_now_ns();
    for (;;) {
      uint32_t done = 0xFFFFFFFFu;
      for (int l = 0; l < c->nlocal; ++l) done = std::min(done, (uint32_t)c->ctrl_host[l]->done_seq);
      if ((int32_t)(seq - done) <= kMaxInflight) break;
      // every kernel ends within its watchdog (the service lane publishes
      // done_seq on any exit): twice that is a broken device
      const uint64_t waited = r2_now_ns() - t0;
      if (waited > (uint64_t)c->cfg.watchdog_ms * 2000000ull) return R2_ERR_TIMEOUT;
      if (waited > 1000000ull) std::this_thread::sleep_for(std::chrono::microseconds(20));
      else std::this_thread::yield();
    }
  }
  c->seq = seq;
  c->last_protocol = S.ring[0].ll == 2 ? R2_PROTO_LL128 : S.ring[0].ll ? R2_PROTO_LL : R2_PROTO_SIMPLE;
  const uint64_t t_pre = r2_debug >= 2 ? r2_now_ns() : 0;
  static uint64_t sum_win = 0;
  if (r2_debug >= 2) sum_win += t_pre - t_win0;
  // worker CTAs of every ring + the service CTA (r2_kernels.cu service_main)
  // LL128 launches run 512 threads per CTA (15 data warps: twice the lines in
  // flight; measured 32 MiB 146 -> 128 us, 64 MiB 253 -> 220 us at N=4,
  // profiles/r02_summary.md); R2_LL_THREADS overrides both line protocols
  const int threads = S.ring[0].ll && c->ll_threads ? c->ll_threads : S.ring[0].ll == 2 ? 512 : c->threads;
  int rc = r2_launch_allreduce(S, threads, stream);
  if (r2_debug >= 2) {                       // host enqueue cost breakdown (diagnostics)
    static uint64_t n_calls = 0, sum_pre = 0, sum_launch = 0;
    const uint64_t t_post = r2_now_ns();
    sum_pre += t_pre - t_in;
    sum_launch += t_post - t_pre;
    if (++n_calls % 500 == 0)
      fprintf(stderr, "[r2 enqueue] rank %d: host prep %.2f us (of which in-flight window wait %.2f), "
              "cooperative launch %.2f us per call\n", c->rank, sum_pre / 1e3 / 500, sum_win / 1e3 / 500,
              sum_launch / 1e3 / 500), sum_pre = sum_launch = sum_win = 0;
  }
  c->last_stream = stream;
  if (rc != 0) return R2_ERR_CUDA;
  return R2_SUCCESS;
}

// One standard ring collective (AllReduce, or the standalone ReduceScatter /
// AllGather halves of SURVEY §8(f) f1, or Broadcast).  `count`: AllReduce
// elements; RS recvcount; AG sendcount.
static r2_result_t enqueue_coll(r2_comm* c, r2_op_t op, const void* send, void* recv, size_t count, r2_dtype_t dt,
                                void* stream, int root = 0) {
  const int E = elem_bytes(dt);
  if (c->n == 1) {
    if (send != recv) CK(cudaMemcpyAsync(recv, send, count * E, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    c->last_stream = stream;
    return R2_SUCCESS;
  }
  std::vector<RingSpec> rings{standard_ring(c, op, send, recv, count, root)};
  return launch_rings(c, rings, dt, stream);
}

// ---------------------------------------------------------------- re-ranking
// SURVEY §8(f) f4 (Algorithm 1, App. D; §6; readings C-19,
// R-13): the ring order of the next AllReduce from the health records of its
// seq ("the planner inspects the health status records").
std::vector<int> rerank_plan(r2_comm* c, uint32_t q) {
  const int n = c->n, K = c->K;
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  if (n < 3) return order;
  std::vector<uint32_t> rails(n, 0), dead(n, 0);
  {
    std::lock_guard<std::mutex> g(c->mu);
    for (int r = 0; r < n; ++r)
      for (int k = 0; k < K; ++k) {
        if (!r2_ep_dead_at(c, r, k, q)) rails[r] |= 1u << k;
        if (r2_link_dead_at(c, r, k, q)) dead[r] |= 1u << k;
      }
  }
  std::vector<int> out(n);
  if (r2_rerank(n, order.data(), rails.data(), dead.data(), out.data()) <= 0) return order;
  return out;
}

// ---------------------------------------------------------------- R²CCL-AllReduce
// SURVEY §8(f) f2 (App. A; reading R-9) and the strategy
// choice of f3 (reading R-11).
struct R2ccPlan {
  bool applies = false;
  int f = -1;                                // the degraded rank
  double X = 0, Y = 0;                       // lost bandwidth fraction, partial-AllReduce share
  size_t NA = 0, NP = 0;                     // elements: global ring prefix / partial ring suffix
  std::vector<int> A, P;                     // f's healthy / dead channels (global ids)
};

// App. A (g = 1 GPU per "server"): threshold n/(3n-2); above it
// Y* = X + X(1-X) / (X + (n-2) n) (Step 1 with g = 1), else 0 (Step 3).
double r2cc_partition(int n, double X) {
  const double th = (double)n / (3.0 * n - 2.0);
  if (X <= th) return 0.0;
  return X + X * (1.0 - X) / (X + (double)(n - 2) * n);
}

R2ccPlan r2cc_plan(r2_comm* c, size_t count, r2_dtype_t dt, uint32_t q) {
  R2ccPlan pl;
  const int n = c->n, K = c->K;
  if (n < 3 || c->cfg.allreduce_algo == R2_ALGO_RING || !c->lay.tailor) return pl;
  std::lock_guard<std::mutex> g(c->mu);
  for (int r = 0; r < n; ++r)
    for (int k = 0; k < K; ++k) {
      if (r2_link_dead_at(c, r, k, q)) return pl;          // a dead link: not the single-degraded-rank case
      if (r2_ep_dead_at(c, r, k, q)) {
        if (pl.f >= 0 && pl.f != r) return pl;             // two degraded ranks: Balance (f4 territory)
        pl.f = r;
      }
    }
  if (pl.f < 0) return pl;
  double wd = 0, wt = 0;
  for (int k = 0; k < K; ++k) {
    wt += c->weights[k];
    if (r2_ep_dead_at(c, pl.f, k, q)) {
      wd += c->weights[k];
      pl.P.push_back(k);
    } else {
      pl.A.push_back(k);
    }
  }
  if (pl.A.empty()) return pl;                             // NO_BACKUP: left to the ring path
  pl.X = wd / wt;
  pl.Y = r2cc_partition(n, pl.X);
  const size_t V = 16 / (size_t)elem_bytes(dt);
  // reading R-9: N_A = N - floor(Y N / V) V rounded up to whole vectors (the
  // partial region starts 16-byte aligned), at most N; N_P = N - N_A
  const size_t np0 = (size_t)floor(pl.Y * (double)count / (double)V) * V;
  pl.NA = std::min(count, (count - std::min(np0, count) + V - 1) / V * V);
  pl.NP = count - pl.NA;
  pl.applies = pl.Y > 0 && pl.NP > 0 && pl.NA > 0;
  return pl;
}

// alpha-beta cost of the two algorithms on the degraded communicator (reading
// R-11): the ring is throttled to (1-X) of the per-GPU rate at the degraded
// rank; R²CCL-AllReduce pays max(T1, T2) + T3 (the paper's model
// with B = beta) plus its extra ring steps and the second launch.
bool r2cc_faster(const r2_comm* c, const R2ccPlan& pl, size_t count, r2_dtype_t dt) {
  const int n = c->n;
  const double S = (double)count * elem_bytes(dt);
  const double B = std::max(c->cfg.beta_mbps, 1) / 1000.0;            // bytes per ns
  const double a = c->cfg.alpha_simple_ns;
  const double X = pl.X, Y = (double)pl.NP / (double)count;
  const double t_ring = (2 * n - 2) * a + 2.0 * (n - 1) / n * S / ((1 - X) * B);
  const double T1 = 2.0 * (n - 1) / n * (1 - Y) * S / ((1 - X) * B);
  const double T2 = 2.0 * (n - 2) / (n - 1) * Y * S / (X * B);
  const double T3 = Y * S / (X * B);
  // stage efficiencies: the fraction of its bandwidth model each stage reaches
  // on this implementation (reading R-11; measured, tools/r2cc_stages.py)
  const double e1 = std::max(c->cfg.r2cc_stage1_eff_pct, 1) / 100.0, e2 = std::max(c->cfg.r2cc_stage2_eff_pct, 1) / 100.0;
  const double t_r2cc = (2 * n - 2) * a + std::max(T1, T2) / e1 + n * a + T3 / e2 + c->cfg.alpha_launch_ns;
  return t_r2cc < t_ring;
}

// Stage 1 (one launch): global ring over [0, N_A) on f's healthy channels
// concurrently with the partial ring over [N_A, N) among the n-1 healthy ranks
// on f's dead channels.  Stage 2 (a second launch): the tailored broadcast of
// [N_A, N) from f around the ring.
r2_result_t r2cc_enqueue(r2_comm* c, const R2ccPlan& pl, const void* send, void* recv, size_t count, r2_dtype_t dt,
                         void* stream) {
  const size_t E = (size_t)elem_bytes(dt);
  const size_t shiftb = pl.NA * E;
  std::vector<RingSpec> st1;
  RingSpec g = standard_ring(c, R2_OP_ALLREDUCE, send, recv, pl.NA, 0);
  g.chans = pl.A;
  g.allow_ll = false;
  g.row_elems = count;
  st1.push_back(g);
  RingSpec pr = standard_ring(c, R2_OP_ALLREDUCE, (const char*)send + shiftb, (char*)recv + shiftb, pl.NP, 0);
  pr.order.erase(std::find(pr.order.begin(), pr.order.end(), pl.f));
  pr.chans = pl.P;
  pr.region = 1;
  pr.peer_recv_off = shiftb;
  pr.allow_ll = false;
  pr.row_elems = count;
  st1.push_back(pr);
  // diagnostics only (tools/r2cc_stages.py): R2_R2CC_ONLY_STAGE=1/2 launches
  // one stage alone to time it -- the result is then incomplete
  static const int only = getenv("R2_R2CC_ONLY_STAGE") ? atoi(getenv("R2_R2CC_ONLY_STAGE")) : 0;
  r2_result_t e = R2_SUCCESS;
  if (only != 2) e = launch_rings(c, st1, dt, stream);
  if (e != R2_SUCCESS) return e;
  std::vector<RingSpec> st2{standard_ring(c, R2_OP_R2CC_STAGE2, (const char*)send + shiftb, (char*)recv + shiftb,
                                          pl.NP, pl.f)};
  st2[0].row_elems = count;
  st2[0].allow_ll = false;
  if (only != 1) e = launch_rings(c, st2, dt, stream);
  if (e != R2_SUCCESS) return e;
  std::lock_guard<std::mutex> gl(c->mu);
  c->last_r2cc.seq = c->seq;
  c->last_r2cc.f = pl.f;
  c->last_r2cc.X = pl.X;
  c->last_r2cc.Y = pl.Y;
  c->last_r2cc.NA = pl.NA;
  c->last_r2cc.NP = pl.NP;
  c->n_r2cc++;
  return R2_SUCCESS;
}

extern "C" r2_result_t r2_allreduce(r2_comm_t c, const void* send, void* recv, size_t count, r2_dtype_t dt,
                                    void* stream) {
  if (!c) return R2_ERR_INVALID_ARG;
  int ae = take_async_error(c);
  if (ae != R2_SUCCESS) return (r2_result_t)ae;
  if (dt != R2_INT32 && dt != R2_FLOAT32 && dt != R2_BFLOAT16) return R2_ERR_INVALID_ARG;
  if (count == 0) return R2_SUCCESS;
  if (!send || !recv || ((uintptr_t)send & 15) || ((uintptr_t)recv & 15)) return R2_ERR_INVALID_ARG;
  if (count * (size_t)elem_bytes(dt) > c->cfg.max_bytes) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(c->dev) != cudaSuccess) return R2_ERR_CUDA;
  if (c->n > 1 && c->cfg.allreduce_algo != R2_ALGO_RING) {
    // the planner reads the health records of the next seq
    const R2ccPlan pl = r2cc_plan(c, count, dt, (uint32_t)c->seq + 1);
    if (pl.applies && (c->cfg.allreduce_algo == R2_ALGO_R2CC || r2cc_faster(c, pl, count, dt)))
      return r2cc_enqueue(c, pl, send, recv, count, dt, stream);
  }
  if (c->n == 1) return enqueue_coll(c, R2_OP_ALLREDUCE, send, recv, count, dt, stream);
  std::vector<RingSpec> rings{standard_ring(c, R2_OP_ALLREDUCE, send, recv, count, 0)};
  if (c->cfg.rerank) rings[0].order = rerank_plan(c, (uint32_t)c->seq + 1);
  const bool reranked = !std::is_sorted(rings[0].order.begin(), rings[0].order.end());
  r2_result_t e = launch_rings(c, rings, dt, stream);
  if (e == R2_SUCCESS) {
    std::lock_guard<std::mutex> gl(c->mu);
    c->last_ring = rings[0].order;
    c->n_rerank += reranked;
  }
  return e;
}

// ReduceScatter / AllGather (f1).  The shard stride count * elem need not be
// a multiple of 16 bytes: the kernel then uses element-wise user accesses.
static r2_result_t rs_ag(r2_comm_t c, r2_op_t op, const void* send, void* recv, size_t count, r2_dtype_t dt,
                         void* stream) {
  if (!c) return R2_ERR_INVALID_ARG;
  int ae = take_async_error(c);
  if (ae != R2_SUCCESS) return (r2_result_t)ae;
  if (dt != R2_INT32 && dt != R2_FLOAT32 && dt != R2_BFLOAT16) return R2_ERR_INVALID_ARG;
  if (count == 0) return R2_SUCCESS;
  if (!send || !recv) return R2_ERR_INVALID_ARG;
  const size_t E = (size_t)elem_bytes(dt);
  // the n-shard buffer is 16-byte aligned; the one-shard buffer only needs
  // element alignment when it is the own shard of the other (in place)
  const void* big = op == R2_OP_REDUCE_SCATTER ? send : (const void*)recv;
  if ((uintptr_t)big & 15) return R2_ERR_INVALID_ARG;
  const void* small = op == R2_OP_REDUCE_SCATTER ? (const void*)recv : send;
  const bool own_shard = !c->sim && (const char*)small == (const char*)big + (size_t)c->rank * count * E;
  if (!own_shard && ((uintptr_t)small & 15)) return R2_ERR_INVALID_ARG;
  if ((uintptr_t)small % E) return R2_ERR_INVALID_ARG;
  if ((size_t)c->n * count * E > c->cfg.max_bytes) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(c->dev) != cudaSuccess) return R2_ERR_CUDA;
  return enqueue_coll(c, op, send, recv, count, dt, stream);
}

extern "C" r2_result_t r2_broadcast(r2_comm_t c, const void* send, void* recv, size_t count, r2_dtype_t dt, int root,
                                    void* stream) {
  if (!c) return R2_ERR_INVALID_ARG;
  int ae = take_async_error(c);
  if (ae != R2_SUCCESS) return (r2_result_t)ae;
  if (dt != R2_INT32 && dt != R2_FLOAT32 && dt != R2_BFLOAT16) return R2_ERR_INVALID_ARG;
  if (root < 0 || root >= c->n) return R2_ERR_INVALID_ARG;
  if (count == 0) return R2_SUCCESS;
  const bool reads_send = c->sim || c->rank == root;
  if (!recv || ((uintptr_t)recv & 15) || (reads_send && (!send || ((uintptr_t)send & 15)))) return R2_ERR_INVALID_ARG;
  if (count * (size_t)elem_bytes(dt) > c->cfg.max_bytes) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(c->dev) != cudaSuccess) return R2_ERR_CUDA;
  return enqueue_coll(c, R2_OP_BROADCAST, reads_send ? send : recv, recv, count, dt, stream, root);
}

extern "C" r2_result_t r2_reduce_scatter(r2_comm_t c, const void* send, void* recv, size_t recvcount, r2_dtype_t dt,
                                         void* stream) {
  return rs_ag(c, R2_OP_REDUCE_SCATTER, send, recv, recvcount, dt, stream);
}

extern "C" r2_result_t r2_all_gather(r2_comm_t c, const void* send, void* recv, size_t sendcount, r2_dtype_t dt,
                                     void* stream) {
  return rs_ag(c, R2_OP_ALL_GATHER, send, recv, sendcount, dt, stream);
}

extern "C" r2_result_t r2_allreduce_host(r2_comm_t c, const void* send, void* recv, size_t count, r2_dtype_t dt,
                                         void* stream) {
  if (!c || !send || !recv) return R2_ERR_INVALID_ARG;
  int ae = take_async_error(c);
  if (ae != R2_SUCCESS) return (r2_result_t)ae;
  if (dt != R2_INT32 && dt != R2_FLOAT32 && dt != R2_BFLOAT16) return R2_ERR_INVALID_ARG;
  if (count == 0) return R2_SUCCESS;
  const size_t bytes = count * (size_t)elem_bytes(dt);
  if (bytes > c->cfg.max_bytes) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(c->dev) != cudaSuccess) return R2_ERR_CUDA;
  const size_t stride = align_up(bytes, 16);
  const size_t need = (align_up(c->cfg.max_bytes, 16) + 4096) * c->nlocal;   // + per-segment row padding
  if (!c->host_stage) {
    CK(cudaMalloc(&c->host_stage, need));
    c->host_stage_bytes = need;
    r2_result_t e = r2_register_multi(c, c->host_stage, need, &c->host_stage_reg);
    if (e != R2_SUCCESS) return e;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (bytes >= ((size_t)8 << 20)) {
    // Pipelined: segment i's H2D (copy stream), allreduce (caller's stream) and
    // D2H (second copy stream) overlap with the neighbouring segments'; PCIe
    // is full duplex, so the call costs about one direction's transfer.  Every
    // rank derives the same segmentation from count (each segment is one
    // collective).  Simulated ranks: segment i of every rank row is packed into
    // its own stage region [nlocal][roundup(seg_i, 16 B)] (2-D copies), the row
    // layout a sim-mode collective of seg_i elements expects.
    const size_t V = 16 / (size_t)elem_bytes(dt);
    const size_t E = (size_t)elem_bytes(dt);
    const int nseg = (int)std::min<size_t>(8, std::max<size_t>(1, bytes / ((size_t)4 << 20)));
    const size_t seg = (count + nseg - 1) / nseg / V * V + V;      // elements, 16-byte multiple
    if (!c->h2d_stream) {
      CK(cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
      c->host_ev.resize(3 * 8 + 1);
      for (auto& ev : c->host_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    cudaEvent_t ev_begin = c->host_ev[3 * 8];
    CK(cudaEventRecord(ev_begin, s));                             // after the caller's earlier work
    CK(cudaStreamWaitEvent(c->h2d_stream, ev_begin, 0));          // (the previous call's D2H included)
    const char* hs = (const char*)send;
    char* hr = (char*)recv;
    int last = -1;
    size_t region = 0;                                             // stage offset of segment i's rows
    for (int i = 0; i < nseg; ++i) {
      const size_t lo = (size_t)i * seg;
      if (lo >= count) break;
      const size_t n_i = std::min(seg, count - lo), off = lo * E, b_i = n_i * E;
      const size_t pitch = align_up(b_i, 16);                      // sim rows of this segment
      char* st = c->host_stage + region;
      cudaEvent_t e_in = c->host_ev[3 * i], e_ar = c->host_ev[3 * i + 1], e_out = c->host_ev[3 * i + 2];
      CK(cudaMemcpy2DAsync(st, pitch, hs + off, stride, b_i, c->nlocal, cudaMemcpyHostToDevice, c->h2d_stream));
      CK(cudaEventRecord(e_in, c->h2d_stream));
      CK(cudaStreamWaitEvent(s, e_in, 0));
      r2_result_t e = enqueue_coll(c, R2_OP_ALLREDUCE, st, st, n_i, dt, stream);
      if (e != R2_SUCCESS) return e;
      CK(cudaEventRecord(e_ar, s));
      CK(cudaStreamWaitEvent(c->d2h_stream, e_ar, 0));
      CK(cudaMemcpy2DAsync(hr + off, stride, st, pitch, b_i, c->nlocal, cudaMemcpyDeviceToHost, c->d2h_stream));
      CK(cudaEventRecord(e_out, c->d2h_stream));
      region += pitch * c->nlocal;
      last = i;
    }
    if (last >= 0) CK(cudaStreamWaitEvent(s, c->host_ev[3 * last + 2], 0));   // the caller's stream sees it all
    return R2_SUCCESS;
  }
  // one contiguous copy each way when the host rows are packed like the stage
  if (stride == bytes || c->nlocal == 1) {
    CK(cudaMemcpyAsync(c->host_stage, send, bytes * c->nlocal, cudaMemcpyHostToDevice, s));
  } else {
    for (int l = 0; l < c->nlocal; ++l)
      CK(cudaMemcpyAsync(c->host_stage + l * stride, (const char*)send + l * stride, bytes, cudaMemcpyHostToDevice, s));
  }
  r2_result_t e = enqueue_coll(c, R2_OP_ALLREDUCE, c->host_stage, c->host_stage, count, dt, stream);
  if (e != R2_SUCCESS) return e;
  if (stride == bytes || c->nlocal == 1) {
    CK(cudaMemcpyAsync(recv, c->host_stage, bytes * c->nlocal, cudaMemcpyDeviceToHost, s));
  } else {
    for (int l = 0; l < c->nlocal; ++l)
      CK(cudaMemcpyAsync((char*)recv + l * stride, c->host_stage + l * stride, bytes, cudaMemcpyDeviceToHost, s));
  }
  return R2_SUCCESS;
}

// Deterministic: once the stream is synchronised every kernel up to c->seq
// has exited, and a rank whose kernel left without a complete result (watchdog,
// abort, exhausted chain) wrote Ctrl.fail_seq / fail_code before exiting.  A
// kernel that exits normally has every incoming completion word, so its
// result is complete: SUCCESS is never returned for a wrong buffer.
extern "C" r2_result_t r2_sync(r2_comm_t c) {
  if (!c) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(c->dev) != cudaSuccess) return R2_ERR_CUDA;
  if (cudaStreamSynchronize((cudaStream_t)c->last_stream) != cudaSuccess) return R2_ERR_CUDA;
  int err = R2_SUCCESS;
  if (c->n > 1)
    for (int l = 0; l < c->nlocal; ++l) {
      const uint32_t fs = c->ctrl_host[l]->fail_seq;
      if (fs && fs > c->reported_seq && fs <= c->seq) err = (int)c->ctrl_host[l]->fail_code;
    }
  std::lock_guard<std::mutex> g(c->mu);
  if (err == R2_SUCCESS) err = c->unreported_error;
  c->unreported_error = R2_SUCCESS;
  c->reported_seq = c->seq;
  if (err != R2_SUCCESS && c->last_error == R2_SUCCESS) {
    c->last_error = err;
    c->last_error_seq = c->seq;
  }
  return (r2_result_t)err;
}

extern "C" r2_result_t r2_trace(r2_comm_t c, int rank_local, uint64_t out[64]) {
  if (!c || !out || !c->trace || c->n < 2 || rank_local < 0 || rank_local >= c->nlocal) return R2_ERR_INVALID_ARG;
  if (cudaSetDevice(c->dev) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return R2_ERR_CUDA;
  const RankPtrs& me = c->peers_host[rank_local * c->n + c->first_rank + rank_local];
  unsigned long long* dev = me.misc->trace;
  if (cudaMemcpy(out, dev, sizeof(unsigned long long) * R2_TRACE_SLOTS, cudaMemcpyDeviceToHost) != cudaSuccess)
    return R2_ERR_CUDA;
  unsigned long long arm[R2_TRACE_SLOTS];
  for (int i = 0; i < R2_TRACE_SLOTS; ++i) arm[i] = (i == 0 || i == 2 || (i >= 32 && i < 60)) ? ~0ull : 0ull;
  if (cudaMemcpy(dev, arm, sizeof(arm), cudaMemcpyHostToDevice) != cudaSuccess) return R2_ERR_CUDA;
  return R2_SUCCESS;
}

extern "C" r2_result_t r2_probe(r2_comm_t c, int rank_local, int peer, int channel, r2_verdict_t* out) {
  if (!c || !out || c->n < 2) return R2_ERR_INVALID_ARG;
  if (rank_local < 0 || rank_local >= c->nlocal || peer < 0 || peer >= c->n || channel < 0 || channel >= c->K)
    return R2_ERR_INVALID_ARG;
  const int a = c->first_rank + rank_local;
  if (peer == a) return R2_ERR_INVALID_ARG;
  uint32_t id;
  {
    std::lock_guard<std::mutex> g(c->pmu);
    id = ((uint32_t)a << 24) | (++c->round_counter & 0xFFFFFF);
    c->probe_requests.push_back({rank_local, {peer, channel}});
    c->probe_request_ids.push_back(id);
  }
  uint64_t t0 = r2_now_ns();
  for (;;) {
    {
      std::lock_guard<std::mutex> g(c->pmu);
      auto it = c->finished_rounds.find(id);
      if (it != c->finished_rounds.end()) {
        *out = it->second;
        c->finished_rounds.erase(it);
        return R2_SUCCESS;
      }
    }
    if (r2_now_ns() - t0 > 10ull * 1000000000ull) return R2_ERR_TIMEOUT;
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

extern "C" r2_result_t r2_status(r2_comm_t c, r2_status_t* out) {
  if (!c || !out) return R2_ERR_INVALID_ARG;
  memset(out, 0, sizeof(*out));
  {
    std::lock_guard<std::mutex> g(c->mu);
    out->seq = c->seq;
    out->last_error = c->last_error;
    out->last_error_seq = c->last_error_seq;
    out->n_events = (int)c->events.size();
    out->world = c->n;
    out->nlocal = c->nlocal;
    out->nchannels = c->K;
    out->last_protocol = c->last_protocol;
    out->n_readmits = c->n_readmits;
    out->n_reprobes = c->n_reprobes;
    out->n_service_kernels = c->n_svc_kicks;
    out->n_r2cc = c->n_r2cc;
    out->r2cc_rank = c->last_r2cc.f;
    out->r2cc_X = c->last_r2cc.X;
    out->r2cc_Y = c->last_r2cc.Y;
    out->r2cc_NA = c->last_r2cc.NA;
    out->r2cc_NP = c->last_r2cc.NP;
    out->r2cc_seq = c->last_r2cc.seq;
    out->n_rerank = c->n_rerank;
    for (int i = 0; i < c->n && i < R2_MAX_RANKS; ++i)
      out->ring_order[i] = i < (int)c->last_ring.size() ? c->last_ring[i] : i;
    const uint32_t q = (uint32_t)c->seq + 1;   // the view of the next collective
    for (int r = 0; r < c->n && r < R2_MAX_LOCAL * 4; ++r)
      for (int k = 0; k < c->K; ++k) {
        if (r2_ep_dead_at(c, r, k, q)) out->dead_endpoints[r] |= 1u << k;
        if (r2_link_dead_at(c, r, k, q)) out->dead_links[r] |= 1u << k;
      }
  }
  if (c->n > 1) {
    if (cudaSetDevice(c->dev) != cudaSuccess) return R2_ERR_CUDA;
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    std::vector<MiscDev> m(c->nlocal);
    for (int l = 0; l < c->nlocal; ++l) {
      const RankPtrs& me = c->peers_host[l * c->n + c->first_rank + l];
      CK(cudaMemcpyAsync(&m[l], me.misc, sizeof(MiscDev), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    cudaStreamDestroy(s);
    for (int l = 0; l < c->nlocal; ++l)
      for (int k = 0; k < c->K; ++k) out->bytes[l][k] = m[l].bytes[k];
  }
  return R2_SUCCESS;
}

extern "C" r2_result_t r2_get_event(r2_comm_t c, int idx, r2_event_t* out) {
  if (!c || !out) return R2_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> g(c->mu);
  if (idx < 0 || idx >= (int)c->events.size()) return R2_ERR_INVALID_ARG;
  *out = c->events[idx];
  return R2_SUCCESS;
}

extern "C" r2_result_t r2_finalize(r2_comm_t c) {
  if (!c) return R2_ERR_INVALID_ARG;
  cudaSetDevice(c->dev);
  cudaDeviceSynchronize();
  if (c->has_oob) c->oob.barrier(c->oob.ctx);
  track_live(c, false);
  c->stop.store(true);
  if (c->mon.joinable()) c->mon.join();
  cudaDeviceSynchronize();                  // a standalone service kernel, if any
  for (auto& rg : c->regs)
    for (void* p : rg.opened) close_peer(c, p);
  c->regs.clear();
  for (void* p : c->peer_arena_opened)
    if (p) cudaIpcCloseMemHandle(p);
  c->peer_arena_opened.clear();
  if (c->has_oob) c->oob.barrier(c->oob.ctx);
  release_resources(c);
  delete c;
  return R2_SUCCESS;
}
