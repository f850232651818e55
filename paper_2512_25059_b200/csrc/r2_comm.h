// r2_comm.h -- the communicator object behind r2_comm_t (host side).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/r2ccl.h"
#include "r2_internal.h"

// OOB control messages (P:11 bilateral notify; P:16-19 probes/verdict).
enum MsgType : uint32_t {
  MSG_NOTIFY = 1,        // detector -> all: connection (a -> b, c) failed in seq
  MSG_PROBE_REQ = 2,     // round owner -> prober: run probe prober -> target
  MSG_PROBE_RES = 3,     // prober -> round owner: outcome
  MSG_VERDICT = 4,       // round owner -> all: triangulated verdict
  MSG_ABORT = 5,         // any -> all: collective seq is unrecoverable
  MSG_NOTIFY_ACK = 6,    // every rank -> detector: NOTIFY received ("notifies both sides")
};

struct Msg {
  uint32_t type;
  uint32_t seq;
  int32_t src, dst;      // sender / destination rank (sim mode routes on dst)
  int32_t round_owner;
  uint32_t round_id;
  int32_t a, b, aux, channel;
  int32_t slot;          // probe slot 0..3 (A->B, B->A, aux->A, aux->B)
  int32_t prober, target;
  int32_t outcome;
  int32_t verdict;
  int32_t outcomes[4];
  int32_t error;
  uint64_t t_fire;
};

struct Reg {
  uint64_t id;
  bool active;
  char* dptr;
  size_t bytes;
  std::vector<unsigned long long> peer_ptr;  // per rank, in this process's VA
  std::vector<void*> opened;                 // IPC bases opened for this reg (to close)
};

struct RingInfo {                            // one ring of a launch (r2_internal.h LaunchParams)
  int op, root;                              // r2_op_t; chain root (ring position)
  int local_step;                            // LOCAL step (own completion words) or -1
  bool ll;                                   // LL protocol
  int m, steps, V;
  unsigned long long slice, chunk;
  int n, K, region;                          // positions, channels, region set (0 / 1)
  int order[R2_MAXR];                        // global rank at ring position
  int chans[R2_MAXK];                        // global channel of ring-local channel
  uint32_t chan_mask;                        // global channels of this ring
  int pos_of(int r) const {
    for (int i = 0; i < n; ++i)
      if (order[i] == r) return i;
    return -1;
  }
  int next_of(int r) const { const int p = pos_of(r); return p < 0 ? -1 : order[(p + 1) % n]; }
  int local_of(int cg) const {
    for (int i = 0; i < K; ++i)
      if (chans[i] == cg) return i;
    return -1;
  }
};

struct LaunchInfo {                          // what the monitor needs about a seq
  uint32_t seq;
  int nrings;
  RingInfo ring[R2_MAXRINGS];
  int nfaults;
  FaultDev faults[R2_MAXF];                  // global rank / channel / origin channel
  // the ring carrying global channel cg (nullptr: none)
  const RingInfo* ring_of(int cg) const {
    for (int i = 0; i < nrings; ++i)
      if (ring[i].chan_mask >> cg & 1u) return &ring[i];
    return nullptr;
  }
};

struct Round {                               // one triangulation round
  uint32_t id, seq;
  int a, b, aux, channel, local;             // local: index of A in this process
  bool reprobe;                              // recovery check of a dead connection: local only
  int outcomes[4];
  int need;
  uint64_t t_start;
};

struct Replan {                              // a dead outgoing connection to re-place
  uint32_t seq;
  int l, channel;
  r2_verdict_t verdict;
  int stage;                                 // 0 quiesce, 1 freeze-wait, 2 done
  uint32_t freeze_epoch;
  bool froze;                                // adopted work was frozen: rollback reads completion words
  uint64_t t_detect, t_verdict;
  uint64_t t_fire_dev;
};

struct PendingProbe {
  int prober, target, channel, slot, local_prober;
  int round_owner;
  uint32_t round_id, seq;
  volatile int* res_host;
  int res_index;
};

struct NotifyState {                         // one NOTIFY broadcast by this process
  uint32_t seq;
  int a, channel;                            // detecting sender, its channel
  int expected, acks, resends;
  uint64_t acked_by;                         // bit per acknowledging rank (duplicates after a resend)
  uint64_t t_sent, t_last_send, t_acked;     // host CLOCK_MONOTONIC
  bool peer_acked;                           // the other endpoint (a+1) confirmed: no half-open side
  bool dirty;                                // event records to update
  Msg msg;
};

struct EventTiming {                         // finalize failover_ms later
  int event_index;
  int l;
  uint32_t seq, epoch;
  uint64_t t_fire_dev;
};

struct r2_comm {
  int rank = 0, world = 1, dev = 0;
  int n = 1, nlocal = 1, first_rank = 0;
  bool sim = false;
  r2_config_t cfg{};
  int K = 8, W = 4, threads = 512;
  int ll_threads = 0;   // threads per CTA of line-protocol launches (0: threads; R2_LL_THREADS)
  int trace = 0;                             // R2_TRACE=1: record the device timeline (r2_trace)
  int last_protocol = 0;                     // r2_protocol_t of the last enqueued collective
  struct { uint64_t seq; int f; double X, Y; size_t NA, NP; } last_r2cc{0, -1, 0, 0, 0, 0};   // (mu)
  int n_r2cc = 0;                                                                        // (mu)
  int n_rerank = 0;                                                                      // (mu)
  std::vector<int> last_ring;   // ring order of the last ring AllReduce (f4 re-ranking)  (mu)
  // re-probing of dead connections ("periodically reprobes to detect
  // component recovery ... adapting probe frequency")
  struct Reprobe { int r, ch; uint64_t next_ns, interval_ns; uint32_t round_id; };
  std::vector<Reprobe> reprobes;             // monitor only
  std::vector<std::pair<int, int>> readmit_pending;   // (rank, channel) -> next enqueue (mu)
  int n_readmits = 0, n_reprobes = 0;        // (mu)
  uint64_t reprobe_scan_ns = 0;
  uint32_t reprobe_counter = 0;
  unsigned int weights[R2_MAXK]{};
  ArenaLayout lay{};
  r2_oob_t oob{};
  bool has_oob = false;

  // per local rank
  std::vector<char*> arena;                  // own arenas (device)
  std::vector<Ctrl*> ctrl_host, ctrl_dev;
  std::vector<RankPtrs> peers_host;          // [nlocal][n]  ring-0 region set
  RankPtrs* peers_dev = nullptr;
  std::vector<RankPtrs> peers_host1;         // [nlocal][n]  ring-1 region set (R²CCL-AllReduce partial ring)
  RankPtrs* peers_dev1 = nullptr;
  const RankPtrs& rp(int region, int l, int q) const {
    return (region ? peers_host1 : peers_host)[(size_t)l * n + q];
  }
  std::vector<void*> peer_arena_opened;      // real mode: IPC-opened peer arenas
  unsigned long long* regtab_dev = nullptr;  // [R2_MAX_REGS][n]
  std::vector<unsigned long long> regtab_host;
  std::vector<Reg> regs;
  std::map<std::pair<int, unsigned long long>, std::pair<void*, int>> ipc_cache;  // (peer, base)->(ptr, refs)

  // probe result slots (host-mapped)
  volatile int* probe_res_host = nullptr;
  int* probe_res_dev = nullptr;
  volatile unsigned long long* probe_t0_host = nullptr;   // probe start, device clock
  long long clk_offset = 0;                  // device %globaltimer - host CLOCK_MONOTONIC (ns)
  unsigned long long* probe_t0_dev = nullptr;
  int probe_res_next = 0;
  static const int kProbeSlots = 256;

  // collective state
  uint64_t seq = 0;
  std::vector<r2_fault_t> faults;
  void* last_stream = nullptr;
  int max_coop = 0;

  // host-buffer path
  char* host_stage = nullptr;
  uint64_t host_stage_reg = 0;
  size_t host_stage_bytes = 0;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;   // pipelined host path
  std::vector<cudaEvent_t> host_ev;

  // shared with the monitor (mu)
  std::mutex mu;
  std::vector<uint32_t> health;              // host knowledge [4][n*K] seq-indexed (r2_internal.h)
  struct RepairRec { int r, c; uint32_t seq; };
  std::vector<RepairRec> repairs_applied;    // REPAIRs already enqueued (closing later deaths)
  cudaStream_t health_stream = nullptr;
  std::vector<r2_event_t> events;
  int last_error = R2_SUCCESS;
  uint64_t last_error_seq = 0;
  int unreported_error = R2_SUCCESS;
  uint64_t reported_seq = 0;                 // errors of collectives <= this were returned by r2_sync
  std::map<uint32_t, LaunchInfo> launches;

  // monitor
  std::thread mon;
  std::atomic<bool> stop{false};
  cudaStream_t mon_stream = nullptr;
  static const int kProbeStreams = 4;        // the probes of a round run concurrently
  cudaStream_t probe_stream[kProbeStreams] = {};
  int probe_stream_next = 0;
  uint32_t* health_pinned = nullptr;         // pinned staging of the health records
  // service ring (r2_internal.h SvcBlock): posted by the monitor thread only
  SvcBlock* svc_host = nullptr;
  SvcBlock* svc_dev = nullptr;
  uint32_t svc_posted = 0;                   // requests posted (= last tag)
  uint64_t svc_tpost[R2_SVC_RING] = {};      // host time each slot's request was posted
  cudaStream_t svc_stream = nullptr;         // standalone service kernel
  cudaEvent_t svc_ev = nullptr;
  bool svc_launched = false;
  int n_svc_kicks = 0;
  unsigned int* flags_map_host = nullptr;    // rollback: receiver's completion words (host-mapped)
  unsigned int* flags_map_dev = nullptr;
  uint32_t* health_map_host = nullptr;       // health records staged for a service COPY
  uint32_t* health_map_dev = nullptr;
  std::mutex qmu;                            // local message queue (sim + self)
  std::deque<Msg> localq;
  std::vector<uint32_t> handled_err;         // [nlocal*K] last handled err seq
  std::vector<uint32_t> timeout_seq;         // [nlocal] last reported watchdog seq
  std::vector<Round> rounds;
  std::vector<Replan> replans;
  std::vector<PendingProbe> probes;
  std::vector<EventTiming> timings;
  std::vector<NotifyState> notifies;         // outstanding / recent NOTIFYs (monitor)
  std::map<std::pair<uint32_t, int>, int> planned;  // (seq, l*K+c) already re-placed
  std::vector<uint32_t> epoch;               // [nlocal] last epoch written
  std::vector<uint32_t> plan_seq;            // [nlocal] seq the ctrl block serves
  std::vector<std::vector<PlanEntry>> cur_plan;      // [nlocal] entries published
  uint32_t round_counter = 0;
  // r2_probe (main thread) <-> monitor
  std::mutex pmu;
  std::map<uint32_t, r2_verdict_t> finished_rounds;
  std::deque<std::pair<int, std::pair<int, int>>> probe_requests;  // (local, (peer, channel)) -> round ids
  std::deque<uint32_t> probe_request_ids;
  unsigned int probe_token = 1;
};

// tracing (R2_DEBUG=1): control-plane events with host timestamps
#include <stdio.h>
extern int r2_debug;
uint64_t r2_now_ns();
#define R2LOG(...)                                                          \
  do {                                                                      \
    if (r2_debug) {                                                         \
      fprintf(stderr, "[r2 %.6f] ", (double)r2_now_ns() / 1e9);             \
      fprintf(stderr, __VA_ARGS__);                                         \
      fputc('\n', stderr);                                                  \
    }                                                                       \
  } while (0)

// one load of a CTA record's seq|state word
inline void rec_ss(const CtaRec& r, uint32_t* seq, uint32_t* state) {
  unsigned long long v = r.ss;
  *seq = (uint32_t)(v >> 32);
  *state = (uint32_t)(v & 0xFFFFFFFFu);
}

// r2_monitor.cpp
void r2_monitor_main(r2_comm* comm);
// service ring (monitor thread): post a request (tag returned), ask whether it
// is done, launch the standalone service kernel when no resident service lane
// will take it, wait for a request (kicking as needed; false on timeout)
uint32_t r2_svc_post(r2_comm* comm, SvcReq& r);
bool r2_svc_done(const r2_comm* comm, uint32_t tag);
void r2_svc_kick(r2_comm* comm);
bool r2_svc_wait(r2_comm* comm, uint32_t tag, uint64_t timeout_ns);
int r2_push_health_svc(r2_comm* comm);                                 // monitor: via the service ring
void r2_send_msg(r2_comm* comm, int dst, Msg m);
uint64_t r2_now_ns();

// r2_hostlogic.cpp (internal helpers; health calls need comm->mu held)
int r2_first_healthy_in_chain(int origin, uint32_t mask, int K);
bool r2_conn_ok_at(const r2_comm* comm, int r, int c, uint32_t q);     // connection r->r+1 on c, seq q
bool r2_conn_ok_to(const r2_comm* comm, int r, int to, int c, uint32_t q);   // connection r->to (reading R-10)
uint32_t r2_conn_mask_at(const r2_comm* comm, int r, uint32_t q);
bool r2_ep_dead_at(const r2_comm* comm, int r, int c, uint32_t q);
bool r2_link_dead_at(const r2_comm* comm, int r, int c, uint32_t q);
void r2_declare_dead(r2_comm* comm, int kind, int r, int c, uint32_t from_seq);   // kind 0 ep, 1 link
void r2_declare_repaired(r2_comm* comm, int r, int c, uint32_t at_seq);
void r2_declare_conn_repaired(r2_comm* comm, int r, int c, uint32_t at_seq);   // ep r, ep r+1, link r
int r2_push_health(r2_comm* comm);                                     // mirror to every local arena
cudaError_t r2_spin_sync(cudaStream_t s);
