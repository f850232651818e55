// r2_internal.h -- structures shared by the host control code (r2_comm.cpp,
// r2_monitor.cpp) and the sm_100a kernels (r2_kernels.cu).
//
// Memory layout per rank (one cudaMalloc "arena", IPC-exported to every peer,
// P:27 "register each GPU buffer with all NICs" -> here: mapped into every
// peer process once, at init):
//
//   scratch   [2 parities][n-1 RS slots][slot_bytes]   peer-written partials
//   flags     u32 [2n-2 steps][K][m_cap]               completion words (=seq)
//   counters  u64 [2n-2][K][m_cap]                     Balance part counters
//   ep_dead   u32 [n][K]   link_dead u32 [n][K]        emulated fabric state
//   alert     u32                                      seq of last fault firing
//   mailbox   u32 [n][K]                               probe-flag targets
//   desc      u64 [2][4]                               recv publication
//   misc      delivered/exited/copy counters, bytes[K]
//   stage     [slot_bytes]                             in-place own shard y
#pragma once
#include <stddef.h>
#include <stdint.h>

#define R2_MAXL 16
#define R2_MAXK 16
#define R2_MAXW 16
#define R2_MAXF 8
#define R2_MAX_REGS 64
#define R2_MAX_CTAS_PER_RANK (R2_MAXK * R2_MAXW)
#define R2_MAXR 64          // ranks of a communicator (R2_MAX_LOCAL * 4)
#define R2_MAXRINGS 2       // rings of one launch (R²CCL-AllReduce stage 1: global + partial)

enum { R2D_INT32 = 0, R2D_FLOAT32 = 1, R2D_BF16 = 2 };

// CTA states written to the host-mapped control block
enum { CTA_IDLE = 0, CTA_RUNNING = 1, CTA_DRAINING = 2, CTA_STOPPED = 3, CTA_EXITED = 4 };
// stop causes
enum { STOP_NONE = 0, STOP_FAULT_FIRED = 1, STOP_FAULT_TABLE = 2, STOP_DEATH = 3, STOP_HOST = 4,
       STOP_ABORT = 5, STOP_TIMEOUT = 6, STOP_NOBACKUP = 7 };
// plan entry modes
enum { PLAN_NONE = 0, PLAN_HOT = 1, PLAN_BAL = 2 };

// r2_trace slots: [0] first CTA start (min), [1] last CTA init done (max),
// [2] first publish (min), [4+t] last own chunk of step t retired (max),
// [32+t] first own chunk of step t published (min), [60] last control END,
// [61] last drain done, [62] last CTA exit (max)
#define R2_TRACE_SLOTS 64
struct MiscDev {
  unsigned int delivered;     // items whose flag this rank set in this collective
  unsigned int exited;        // CTAs that left the kernel
  unsigned int copy_next;     // in-place staging copy work counter
  unsigned int abort_seq;     // == seq: a CTA of this rank timed out, all stop
  unsigned long long bytes[R2_MAXK];  // cumulative bytes pushed per carrier channel
  unsigned long long first_retx_ns;   // min over adopters (debug)
  unsigned long long trace[R2_TRACE_SLOTS];  // %globaltimer timeline when LaunchParams.trace (r2_trace)
  // service lane (local rank 0's arena only): request claim state shared by the
  // resident service CTA and the standalone service kernel, and the count of
  // local ranks whose worker CTAs have all left the kernel
  unsigned int svc_lock, svc_tail, grid_exited, pad_svc;
};

struct PlanEntry {           // dynamic re-placement of one origin channel
  unsigned int origin, mode, assignee, mask;   // residual: chunks of origin without a completion word
};

// Device-resident mirror of the plan fields of Ctrl, one per rank arena.
// The CTAs poll THIS (an L2 hit) instead of host memory: thousands of PCIe
// reads per microsecond from every CTA of every GPU saturate the host path
// (measured: ~90 us per poll under load).  The monitor pushes updates with a
// one-thread kernel on its own stream (r2_launch_ctrl_push): body first, then
// (after a fence) the word that publishes it.
struct DevCtrl {
  unsigned int plan_seq, epoch, freeze, abort, stop_mask, nentries, pad0, pad1;
  PlanEntry entries[R2_MAXK];
};

// One rank's arena as seen from some process.  A launch runs up to two rings
// (r2_internal.h LaunchSet); each ring has its own table whose per-ring
// regions (scratch, ll, flags, counters, misc, stage) are disjoint, while the
// per-rank state (fabric, alert, mailbox, desc, dctrl, health, abort word,
// byte counters, tailored-broadcast buffer) is the same memory in both.
struct RankPtrs {
  char* scratch;
  char* ll;                  // LL line slots [2 parities][2n-2 steps][ll_slot_bytes]
  unsigned int* flags;
  unsigned long long* counters;
  unsigned int* ep_dead;
  unsigned int* link_dead;
  unsigned int* alert;
  unsigned int* mailbox;
  unsigned long long* desc;
  MiscDev* misc;
  char* stage;
  DevCtrl* dctrl;            // plan/stop/abort mirror polled by the CTAs
  unsigned int* health;      // [4][n*K] host health records: ep dead/repair seq, link dead/repair seq
  unsigned int* abort;       // per-rank abort word (= seq: a CTA of this rank timed out; ring-0 misc)
  unsigned long long* bytes; // [K] bytes pushed per global channel (ring-0 misc)
  char* tailor;              // R²CCL-AllReduce stage 2: the degraded rank's contribution lands here
};

// Health records are seq-indexed so that collectives enqueued ahead of a
// verdict plan consistently: an endpoint/link declared dead while collective
// q runs is dead from q+1 on; a REPAIR armed for seq s' re-admits it from s'.
#define R2_H_EP_DEAD 0
#define R2_H_EP_REP 1
#define R2_H_LINK_DEAD 2
#define R2_H_LINK_REP 3
#ifdef __cplusplus
inline __host__ __device__ bool r2_dead_at(unsigned int dseq, unsigned int rseq, unsigned int q) {
  // a REPAIR armed at the seq a death takes effect wins (it was issued later)
  return dseq != 0 && dseq <= q && !(rseq >= dseq && rseq <= q);
}
#endif

struct ArenaLayout {
  size_t scratch, ll, flags, counters, ep_dead, link_dead, alert, mailbox, desc, misc, stage, dctrl, health, total;
  // ring 1 (R²CCL-AllReduce's partial ring over n-1 ranks) and stage 2's buffer
  size_t scratch1, flags1, counters1, misc1, stage1, tailor;
  size_t slot1_bytes;         // one ring-1 scratch slot (>= max_bytes / (n-1))
  size_t tailor_bytes;        // stage-2 buffer (>= max_bytes)
  size_t slot_bytes;          // one RS scratch slot (>= max shard bytes)
  size_t ll_slot_bytes;       // one LL slot (2 x the largest LL shard)
  int m_cap;
};

// ------------------------------------------------------------------ control


struct CtaRec {                       // written by one CTA, read by the monitor
  volatile unsigned long long ss;    // seq << 32 | state   (one store: never torn)
  volatile unsigned long long ack;   // seq << 32 | acknowledged plan epoch
  volatile unsigned int cause, adopt_tag, wait_idx, wait_val;  // adopt_tag = seq<<8 | epoch; watchdog diagnostics
  volatile unsigned long long t_stop, t_first_adopt;
  volatile unsigned long long t_apply, t_pub_adopt, t_prev_poll;
  volatile unsigned int npoll, apply_src;   // diagnostics: plan applied / first adopted chunk published
  volatile unsigned long long stop_key;  // own chunks with key >= stop_key are not complete (set with the state)
};
#define R2_SS(seq, state) (((unsigned long long)(seq) << 32) | (unsigned long long)(state))

struct ErrRec {              // one per channel: the stop that needs handling
  volatile unsigned int seq, cause, origin, q;
  volatile unsigned long long t_fire;
};

struct Ctrl {                // host-mapped, one per local rank
  volatile unsigned int plan_seq, epoch, freeze, abort;
  volatile unsigned int stop_mask, nentries, done_seq, pad1;   // done_seq: last collective finished
  // last collective this rank's kernel left WITHOUT a complete result (watchdog,
  // abort, exhausted chain) and its r2_result_t: written by the exiting CTAs
  // before the kernel ends, so r2_sync reads it deterministically after the
  // stream synchronisation (never SUCCESS for an aborted collective)
  volatile unsigned int fail_code, fail_seq;
  PlanEntry entries[R2_MAXK];
  ErrRec err[R2_MAXK];
  CtaRec cta[R2_MAX_CTAS_PER_RANK];
};

// ------------------------------------------------------------------ service
// The monitor's device-side work (probe-flag stores and read-backs, installs of
// the plan mirror DevCtrl, copies of health records / completion words) is a
// ring of requests in host-mapped memory.  It is served by the SERVICE CTA of
// the resident collective kernel (one extra CTA in the cooperative grid; its
// warp 0 polls the ring), so failover needs no second kernel to run next to
// the persistent one (profilers and sanitizers serialise kernels; other work
// may hold the spare SMs).  With no collective resident, the monitor launches
// the standalone service kernel, which serves the same ring.  Requests are
// claimed under a device-memory lock (svc_lock/svc_tail in MiscDev), in order.
enum { SVC_PROBE = 1, SVC_MIRROR = 2, SVC_COPY = 3, SVC_STORE = 4 };   // STORE: u32 nwords -> *dst
#define R2_SVC_RING 64
#define R2_SVC_MAXPROBES 8
struct SvcReq {
  unsigned int kind, mode, tag, nwords;   // MIRROR mode: 0 new collective (plan_seq last), 1 update (epoch last);
                                          // STORE: nwords is the value
  unsigned long long src, dst;            // COPY: nwords u32 src -> dst; MIRROR: dst = DevCtrl
  unsigned long long mailbox, ep_dead, link_dead, result, t_start;   // PROBE (device addresses)
  int prober, target, channel, n, K;
  unsigned int token;
  unsigned long long timeout_ns;
  DevCtrl v;                              // MIRROR: the snapshot to install
};
struct SvcBlock {                         // host-mapped, one per process
  volatile unsigned int head, pad;        // requests posted (host)
  volatile unsigned long long alive;      // seq << 32 | 1 while a resident service lane polls, | 0 after
  volatile unsigned int ack[R2_SVC_RING]; // = tag once request tag is done
  SvcReq req[R2_SVC_RING];
};

// ------------------------------------------------------------------ launch
struct FaultDev {
  unsigned int rank, channel, origin, kind;
  unsigned int t, j, detect_delay_us, poison;
  unsigned long long b;
};

// One ring of a launch.  Positions 0..n-1 of the ring hold global ranks
// ring[pos] (the standard ring: ring[pos] = pos); the ring runs on K of the
// communicator's Kg channels, ring-local channel ci being global channel
// chan[ci].  Geometry (shards, slices, flags, plan entries in the kernel) is in
// ring positions / ring-local channels; fabric state, health records, fault
// table, control block and byte counters are in global ranks / channels.
struct LaunchParams {
  unsigned int seq;
  int n, K, W, m, steps, nlocal, first_rank;   // nlocal: participating local ranks of this ring
  int ng, Kg;                            // communicator ranks / channels
  int ring_id;                           // 0 / 1: which region set (RankPtrs table)
  unsigned char ring[R2_MAXR];           // global rank at ring position
  unsigned char chan[R2_MAXK];           // global channel of ring-local channel
  unsigned char part_l[R2_MAXL];         // process-local index of participant i (sim mode: its global rank)
  unsigned long long peer_recv_off;      // bytes added to a downstream rank's registered recv (ring region)
  unsigned int* grid_exited;             // local rank 0's ring-0 misc: (ring, rank) pairs done
  unsigned int exit_target;              // (ring, local rank) pairs of the whole launch
  int dtype, elem_bytes, V, inplace, strategy, sim;
  int op;                                // r2_op_t
  int t0;                                // AllReduce step of op-step 0 (AllGather: n-1)
  int local_step;                        // op-step of LOCAL items (ReduceScatter: n-1) or -1
  int fin_step;                          // last op-step with incoming completion words
  int peer_recv;                         // some step writes the downstream rank's recv
  int ag_inplace;                        // AllGather with send == own shard of recv; Broadcast root send == recv
  int root;                              // Broadcast root
  unsigned long long N, Np, shard, slice, chunk;   // elements (N: the whole user buffer)
  unsigned long long sstride, slen;      // shard stride in the user buffers / valid elements per shard
  size_t slot_bytes;
  int ll;                                // 0 SIMPLE, 1 LL, 2 LL128 (r2ccl.h "Protocols")
  unsigned int cvec_full, cvec_last, lc128;   // vectors per chunk / in a slice's last chunk; LL128 lines
                                             // per chunk (host-computed: no 64-bit divisions per chunk)
  int spec_ok;                           // line protocols: speculative publishing allowed (reading R-6;
                                         // R2_NO_SPECULATION=1 turns it off for diagnostics)
  unsigned int lane_ps_per_byte;         // channel bandwidth model: pacing per lane (0 = off)
  size_t ll_slot_bytes;
  unsigned long long watchdog_ns;
  int trace;                             // record the r2_trace timeline
  int nfaults;
  FaultDev faults[R2_MAXF];
  unsigned int weights[R2_MAXK];
  const char* send[R2_MAXL];
  char* recv[R2_MAXL];
  int recv_reg[R2_MAXL];                 // registration id of recv (real mode)
  unsigned long long recv_off[R2_MAXL];  // offset of recv inside the registration
  const RankPtrs* peers;                 // [nlocal][n] device array
  const unsigned long long* regtab;      // [R2_MAX_REGS][n] peer registered bases
  Ctrl* ctrl[R2_MAXL];                   // device aliases of host-mapped blocks
  SvcBlock* svc;                         // device alias of the host-mapped service ring
};

struct LaunchSet {                       // the kernel's parameter: rings + service CTA
  int nrings;
  int nctas[R2_MAXRINGS];                // worker CTAs of each ring (grid = sum + 1 service CTA)
  LaunchParams ring[R2_MAXRINGS];
};

struct ProbeParams {
  unsigned int* target_mailbox;          // &mailbox[prober][channel] in target arena
  const unsigned int* ep_dead;           // prober's replicated fabric state
  const unsigned int* link_dead;
  int prober, target, channel, n, K;
  unsigned int token;
  unsigned long long timeout_ns;
  volatile int* result;                  // host-mapped: r2_probe_outcome_t
  volatile unsigned long long* t_start;  // host-mapped: %globaltimer at probe start (failover timeline)
};

// host-side launchers implemented in r2_kernels.cu
#ifdef __cplusplus
extern "C++" {
#endif
int r2_launch_allreduce(const LaunchSet& s, int threads, void* stream);
int r2_launch_probe(const ProbeParams& p, void* stream);
int r2_kernel_smem_bytes();
int r2_max_coop_ctas(int threads);
int r2_warmup(const ProbeParams& p, void* stream);
// standalone service kernel: serves the ring until it is empty
int r2_launch_service(SvcBlock* svc, MiscDev* misc0, void* stream);
#ifdef __cplusplus
}
#endif
