// r2_kernels.cu -- sm_100a kernels of the R²CCL hot path (arXiv 2512.25059).
//
// r2_allreduce_kernel: one persistent (cooperative) launch per collective.
// CTA (l, c, w) serves local rank l, channel c (a CTA group = the bandwidth
// unit standing in for a NIC, SURVEY reading C-1) and chunk lane w (chunks
// j = w, w+W, ...).  It walks its work list in global (step, origin, chunk)
// order -- own items and adopted items merged -- which keeps adoption
// deadlock-free (SURVEY §7 hard part 3):
//
//   RS  step t <= n-2 : x_r[shard] (+ scratch partial) -> peer scratch  (Fig. 3)
//   t = n-1 (fused)   : partial + x_r[own shard] -> own recv + peer recv
//   AG  step t >= n   : own recv[shard] -> peer recv
//
// Every item moves 16-byte vectors straight into the peer's memory over
// NVLink (CUDA-IPC mapping), then one thread issues fence.acq_rel.sys and
// stores the completion word (= seq) into the RECEIVER's flag array (the
// RDMA work-completion analogue; reading C-4).
//
// Fault path: an armed fault fires at (rank, channel, step,
// origin, chunk): the first b bytes reach the peer, no flag is written, the
// emulated fabric state is marked dead on every rank, an error record is
// posted to the host-mapped control block and the channel stops.  The host
// monitor (r2_monitor.cpp) notifies peers out of band, triangulates with
// r2_probe_kernel, rolls back from the flags and publishes a re-placement
// plan; surviving CTAs adopt the residual chunks (HotRepair: the first
// healthy channel of the failover chain; Balance: a weight-proportional part
// of every residual chunk on every healthy channel) and deliver them to the
// canonical addresses with the canonical flags.
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/r2ccl.h"
#include "r2_internal.h"

namespace {

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ unsigned int ld_acquire_sys(const volatile unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_acquire_gpu(const volatile unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Completion words are polled with RELAXED loads (an acquire per poll cost
// ~1.5 us, tools/pingpong.cu, profiles/r01_pingpong.log); once a word is
// seen, one ld.acquire.sys of it makes the receiver side formally ordered
// (try_publish).
__device__ __forceinline__ unsigned int ld_relaxed_sys(const volatile unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys64(const volatile unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(volatile unsigned int* p, unsigned int v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// r2_trace timeline (LaunchParams.trace): slot layout in r2_internal.h.
// trace = 1: min / max over all CTAs of the rank (contended atomics: they
// stretch a latency-bound run by ~1-2 us per event); trace = 2: CTA 0 of the
// rank only, plain stores (one lane's undisturbed timeline)
#define TRACE_MIN(k, i)                                                                  \
  do {                                                                                   \
    if ((k).p->trace == 1) atomicMin(&(k).me->misc->trace[(i)], gtimer());                \
    else if ((k).p->trace == 2 && (k).cta_in_rank == 0 && (k).me->misc->trace[(i)] == ~0ull) \
      (k).me->misc->trace[(i)] = gtimer();                                                \
  } while (0)
#define TRACE_MAX(k, i)                                                                  \
  do {                                                                                   \
    if ((k).p->trace == 1) atomicMax(&(k).me->misc->trace[(i)], gtimer());                \
    else if ((k).p->trace == 2 && (k).cta_in_rank == 0) (k).me->misc->trace[(i)] = gtimer(); \
  } while (0)
__device__ __forceinline__ uint4 ld_cg(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ------------------------------------------------------------------ one hop
// int32: two's-complement wrap (C-9); fp32: IEEE RN add (no FMA, no FTZ);
// bf16: fp32 add then cvt.rn (RNE) back to bf16 at every hop (C-8).
__device__ __forceinline__ unsigned int add_bf16x2(unsigned int a, unsigned int b) {
  float a_lo = __uint_as_float(a << 16), a_hi = __uint_as_float(a & 0xFFFF0000u);
  float b_lo = __uint_as_float(b << 16), b_hi = __uint_as_float(b & 0xFFFF0000u);
  float s_lo = __fadd_rn(a_lo, b_lo), s_hi = __fadd_rn(a_hi, b_hi);
  unsigned int d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(s_hi), "f"(s_lo));
  return d;
}
template <int DT>
__device__ __forceinline__ unsigned int add32(unsigned int a, unsigned int b) {
  if (DT == R2D_INT32) return a + b;
  if (DT == R2D_FLOAT32) return __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(b)));
  return add_bf16x2(a, b);
}
template <int DT>
__device__ __forceinline__ uint4 vadd(uint4 a, uint4 b) {
  return make_uint4(add32<DT>(a.x, b.x), add32<DT>(a.y, b.y), add32<DT>(a.z, b.z), add32<DT>(a.w, b.w));
}

// masked (tail) user-buffer access: lanes >= valid read as 0 / are not written
__device__ __forceinline__ uint4 ld_user(const char* p, int valid, int E, bool aligned = true) {
  if (aligned && valid >= 16 / E) return ld_cg(p);
  unsigned int w[4] = {0, 0, 0, 0};
  if (valid > 0) {
    if (E == 4) {
      for (int i = 0; i < valid; ++i) w[i] = ((const volatile unsigned int*)p)[i];
    } else {
      for (int i = 0; i < valid; ++i) {
        unsigned int h = ((const volatile unsigned short*)p)[i];
        w[i >> 1] |= h << (16 * (i & 1));
      }
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ void st_user(char* p, uint4 v, int valid, int E, bool aligned = true) {
  if (aligned && valid >= 16 / E) { st_v4(p, v); return; }
  unsigned int w[4] = {v.x, v.y, v.z, v.w};
  if (E == 4) {
    for (int i = 0; i < valid; ++i) ((volatile unsigned int*)p)[i] = w[i];
  } else {
    for (int i = 0; i < valid; ++i) ((volatile unsigned short*)p)[i] = (unsigned short)(w[i >> 1] >> (16 * (i & 1)));
  }
}

enum { MODE_RS = 0, MODE_FUSED = 1, MODE_AG = 2 };
enum { ST_OK = 0, ST_STOP = 1, ST_REPLAN = 2, ST_ABORT = 3, ST_TIMEOUT = 4, ST_NOTREADY = 5 };

// ---------------------------------------------------------- mbarrier (PTX)
__device__ __forceinline__ unsigned int smem_u32(const void* p) {
  return static_cast<unsigned int>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_test(unsigned long long* b, unsigned int parity) {
  unsigned int ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned int parity) {
  unsigned int ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}

// Warp-specialized pipeline: warp 0 (control) publishes chunk descriptors into
// a ring of NSLOT shared-memory slots, the other warps move the data; each
// slot has a `full` (control -> data) and an `empty` (data -> control)
// mbarrier.  The control warp retires finished chunks in order with ONE
// fence.acq_rel.sys for all chunks finished since its last retire.
// 8 slots: the control lane publishes a whole small collective's items
// before its first retire (same-box A/B vs 4 slots: N=4 LL calls 32.4 ->
// 31.1 us; N=2 and >= 4 MiB within run-to-run noise; profiles/r02_nslot.txt)
#ifndef R2_NSLOT
#define R2_NSLOT 8
#endif
#define NSLOT R2_NSLOT
enum { SLOT_GO = 0, SLOT_END = 1 };
enum { META_ITEM = 0, META_FIRE = 1, META_END = 2 };

struct Slot {                 // read by the data warps
  int status;
  int poison;
  unsigned int nvec, total;   // vectors to move / vectors of the part (poison tail)
  const char* src;
  const char* s_in;
  char* d_rem;
  char* d_loc;
  int rem_user, loc_user, rs;
  int src_ll;                 // LL protocol: src is an LL slot (else user memory)
  int aligned;                // every user-buffer pointer 16-byte aligned (ReduceScatter /
                              // AllGather shards at a ragged stride may not be)
  unsigned long long e0;
  unsigned long long lim;     // one past the last valid element of the item's shard
  unsigned int lo_c, cvec;    // LL128: the part's first vector in its chunk / vectors of the chunk
};

struct Meta {                 // read by the control warp at retirement
  int kind;
  int t, o, j;
  unsigned int parts, epoch, nbytes;
  int own, fault, local;
};

struct Shared {
  int decision;
  int cause;
  unsigned int abort_code;    // r2_result_t of a monitor abort (DevCtrl.abort)
  int pipe_status;
  unsigned int seen_epoch;
  int dynamic;
  int freeze;
  int nent;
  int alerted;
  int flag;
  unsigned int piece;
  unsigned int pub, fin;      // control: slots published / retired (monotone across pipeline runs)
  unsigned long long stop_key;  // first own chunk that will not complete (recorded at a stop)
  char* recv_next;
  unsigned long long first_adopt;
  unsigned long long wait_t0;
  unsigned long long t_poll, t_prev_poll;   // diagnostics
  unsigned long long t_ctl;                 // last control / fabric check of try_publish
  unsigned long long ph[6];                 // R2_TRACE=3: SM cycles per try_publish phase
  unsigned long long pace_next;             // channel bandwidth model: earliest next send
  unsigned int npoll;
  unsigned long long full[NSLOT];
  unsigned long long empty[NSLOT];
  Slot slot[NSLOT];
  Meta meta[NSLOT];
  PlanEntry ent[R2_MAXK];
  unsigned long long sbase[2 * R2_MAXR];   // per op-step: first element of the shard this rank sends
  unsigned long long slim[2 * R2_MAXR];    //   and one past its last valid element
  int abandon;                // control lane -> data warps: give up spinning line items
  int reissue;                // own items may have been abandoned: re-yield those without a completion
  int slot_ab[NSLOT];         // data warps -> control lane: the slot's item was abandoned
  RankPtrs rp[2];             // this rank's / the ring successor's arena pointers (Cta::me / nx):
                              // the control lane reads them on every chunk, so they live here
                              // and not in the device-memory peers table (an L2 round trip each)
};

struct Cta {
  const LaunchParams* p;
  // l: process-local rank index (send/recv/ctrl/peers rows); r, r1: global
  // ranks of this CTA and of its ring successor; pos: ring position (shard
  // arithmetic); c: ring-local channel (geometry, flags, plan entries);
  // cg: global channel (fabric, health, faults, control block, counters)
  int l, r, r1, pos, c, cg, w, tid, nthr, cta_in_rank;
  unsigned int seq;
  int par;
  bool fault_channel;
  bool own_alive;
  unsigned int conn_mask;   // static plan: outgoing channels healthy for this seq (health records)
  bool all_healthy;         // conn_mask covers every channel (O(1) own-item walk)
  int t_act;                // Broadcast: this rank's chain position (sends only at that step); else -1
  const RankPtrs* me;        // this rank's / the ring successor's arena (copies in Shared::rp)
  const RankPtrs* nx;
  Ctrl* ctrl;
  unsigned int total_items;
  unsigned long long own_next_key;
};

__device__ __forceinline__ unsigned long long keyof(int t, int o, int j) {
  return ((unsigned long long)t << 40) | ((unsigned long long)o << 32) | (unsigned int)j;
}
__device__ __forceinline__ size_t fidx(const LaunchParams& p, int t, int o, int j) {
  return ((size_t)t * p.K + o) * (size_t)p.m + j;
}
__device__ __forceinline__ char* scratch_slot(const RankPtrs& rp, const LaunchParams& p, int par, int slot) {
  return rp.scratch + ((size_t)par * (p.n - 1) + slot) * p.slot_bytes;
}

// The launch parameters, the Cta's arena pointers and Shared live in shared
// memory but reach the control-lane functions through generic pointers; the
// assumption lets the compiler emit shared-space loads (LDS) for them.
#define R2_ASSUME_SHARED(k, sh)                     \
  do {                                              \
    __builtin_assume(__isShared((k).p));            \
    __builtin_assume(__isShared((k).me));           \
    __builtin_assume(__isShared((k).nx));           \
    __builtin_assume(__isShared(&(sh)));            \
  } while (0)

// back-off of the data warps' line polls (ns); R2_SPIN_NS=0 at build time disables it
#ifndef R2_SPIN_NS
#define R2_SPIN_NS 0
#endif
#if R2_SPIN_NS > 0
#define R2_SPIN_PAUSE() __nanosleep(R2_SPIN_NS)
#else
#define R2_SPIN_PAUSE() ((void)0)
#endif

// ------------------------------------------------------------ LL protocol
// One 16-byte vector {w0, w1, w2, w3} travels as two 16-byte lines
// {w0, seq, w1, seq}, {w2, seq, w3, seq} (r2ccl.h "Protocols"): a line is valid
// when both its flags equal the collective's seq (stale lines of earlier
// collectives carry older seqs), so the payload needs no fence.
__device__ __forceinline__ char* ll_slot(const RankPtrs& rp, const LaunchParams& p, int par, int slot) {
  return rp.ll + ((size_t)par * (2 * p.n - 2) + slot) * p.ll_slot_bytes;
}
__device__ __forceinline__ void ll_store(char* q, uint4 v, unsigned int seq) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(q), "r"(v.x), "r"(seq), "r"(v.y), "r"(seq)
               : "memory");
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(q + 16), "r"(v.z), "r"(seq), "r"(v.w),
               "r"(seq)
               : "memory");
}
__device__ __forceinline__ uint4 ll_line(const char* q) {
  uint4 a;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
               : "l"(q)
               : "memory");
  return a;
}
// The control lane publishes an LL item only after the sender's completion
// word for its input (written after the sender issued every line), so the
// lines are in flight and the spin is short; the abort word bounds it anyway.
// `bail` (Shared::abandon): the control lane asks the data warps to give up
// spinning items (a new plan needs the lane, reading R-6); *gave is set then.
__device__ __forceinline__ uint4 ll_load(const char* q, unsigned int seq, const volatile unsigned int* abort_word,
                                         const volatile int* bail, bool* gave) {
  uint4 a = ll_line(q), b = ll_line(q + 16);
  unsigned int spins = 0;
  while (a.y != seq || a.w != seq || b.y != seq || b.w != seq) {
    if ((++spins & 0x3Fu) == 0 && *bail) {
      *gave = true;
      break;
    }
    if ((spins & 0x3FFu) == 0 && *abort_word == seq) break;
    // back off: a warp re-polling at full rate keeps the SM's load queue full,
    // and the control lane's own loads / stores then wait behind the polls
    R2_SPIN_PAUSE();
    if (a.y != seq || a.w != seq) a = ll_line(q);
    if (b.y != seq || b.w != seq) b = ll_line(q + 16);
  }
  return make_uint4(a.x, a.z, b.x, b.z);
}

// Balance part of channel c in an item of V vectors (reading C-15):
// floor(V*w/Σw) per healthy channel in id order, remainder to the top weight
// (ties -> lowest id).  Same rule as r2_balance_shares on the host.
__device__ void bal_part(unsigned int V, unsigned int mask, const unsigned int* w, int K, int c,
                         unsigned int& lo, unsigned int& hi, unsigned int& parts) {
  unsigned long long tot = 0;
  int top = -1;
  for (int k = 0; k < K; ++k)
    if (mask >> k & 1u) {
      tot += w[k];
      if (top < 0 || w[k] > w[top]) top = k;
    }
  lo = hi = 0;
  parts = 0;
  if (tot == 0) return;
  unsigned long long sum = 0;
  for (int k = 0; k < K; ++k)
    if (mask >> k & 1u) sum += (unsigned long long)V * w[k] / tot;
  unsigned int rem = V - (unsigned int)sum;
  unsigned int off = 0;
  for (int k = 0; k < K; ++k) {
    if (!(mask >> k & 1u)) continue;
    unsigned int sh = (unsigned int)((unsigned long long)V * w[k] / tot) + (k == top ? rem : 0u);
    if (sh) parts++;
    if (k == c) {
      lo = off;
      hi = off + sh;
    }
    off += sh;
  }
}

// --------------------------------------------------------------- data mover
// Vectors [0, nvec) of one item part; e0 = global element of vector 0.
//   src    : x (RS/fused) or own recv (AG), user memory (masked by N)
//   s_in   : scratch partial (RS t>0, fused) or null
//   d_rem  : peer scratch (RS, full vectors) or peer recv (fused/AG, masked)
//   d_loc  : fused only: own stage (in-place, full) or own recv (masked)
//   (d_rem null: the ReduceScatter's LOCAL final add)
//   lim    : one past the last valid element of the shard; aligned: user
//            pointers 16-byte aligned (else element-wise user accesses)
template <int DT>
__device__ void move(const LaunchParams& p, unsigned int tid, unsigned int nthr, const char* src, const char* s_in,
                     char* d_rem, bool rem_user, char* d_loc, bool loc_user, unsigned long long e0,
                     unsigned int nvec, unsigned long long lim, bool aligned) {
  const int E = p.elem_bytes, V = p.V;
  const unsigned int stride = nthr;
  if (aligned && d_rem && e0 + (unsigned long long)nvec * V <= lim) {
    // fast path: every vector is inside the user buffer.  UNR vectors per
    // thread per iteration: all loads issued before any use (memory-level
    // parallelism is what bounds this HBM/NVLink-bound loop)
#ifndef R2_UNR
#define R2_UNR 8   // measured: 8 -> 0.956, 4 -> 0.923 of the HBM roof (N=1, profiles/r01_summary.md)
#endif
    constexpr int UNR = R2_UNR;
    unsigned int v = tid;
    for (; v + (UNR - 1) * stride < nvec; v += UNR * stride) {
      uint4 a[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) a[u] = ld_cg(src + (size_t)(v + u * stride) * 16);
      if (s_in) {
        uint4 b[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) b[u] = ld_cg(s_in + (size_t)(v + u * stride) * 16);
#pragma unroll
        for (int u = 0; u < UNR; ++u) a[u] = vadd<DT>(b[u], a[u]);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) st_v4(d_rem + (size_t)(v + u * stride) * 16, a[u]);
      if (d_loc) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) st_v4(d_loc + (size_t)(v + u * stride) * 16, a[u]);
      }
    }
    for (; v < nvec; v += stride) {
      uint4 a = ld_cg(src + (size_t)v * 16);
      if (s_in) a = vadd<DT>(ld_cg(s_in + (size_t)v * 16), a);
      st_v4(d_rem + (size_t)v * 16, a);
      if (d_loc) st_v4(d_loc + (size_t)v * 16, a);
    }
    return;
  }
  // tail path: vectors straddling / beyond the shard's end, unaligned user
  // buffers, or a LOCAL item (no remote destination)
  for (unsigned int v = tid; v < nvec; v += stride) {
    long long ev = (long long)(e0 + (unsigned long long)v * V);
    long long left = (long long)lim - ev;
    int valid = left <= 0 ? 0 : (left >= V ? V : (int)left);
    uint4 a = ld_user(src + (size_t)v * 16, valid, E, aligned);
    if (s_in) a = vadd<DT>(ld_cg(s_in + (size_t)v * 16), a);
    if (d_rem) {
      if (rem_user) st_user(d_rem + (size_t)v * 16, a, valid, E, aligned);
      else st_v4(d_rem + (size_t)v * 16, a);
    }
    if (d_loc) {
      if (loc_user) st_user(d_loc + (size_t)v * 16, a, valid, E, aligned);
      else st_v4(d_loc + (size_t)v * 16, a);
    }
  }
}

// LL item: src user memory (or an LL slot when src_ll), s_in an LL slot, d_rem
// an LL slot at the peer, d_loc user memory / stage.  Padding vectors travel
// as zeros so that the receiver can validate every line.
template <int DT>
__device__ bool move_ll(const LaunchParams& p, unsigned int tid, unsigned int nthr, const char* src, bool src_ll,
                        const char* s_in, char* d_rem, char* d_loc, bool loc_user, unsigned long long e0,
                        unsigned int nvec, unsigned long long lim, bool aligned, unsigned int seq,
                        const volatile unsigned int* abort_word, const volatile int* bail) {
  const int E = p.elem_bytes, V = p.V;
  bool gave = false;
  for (unsigned int v = tid; v < nvec && !gave; v += nthr) {
    const long long ev = (long long)(e0 + (unsigned long long)v * V);
    const long long left = (long long)lim - ev;
    const int valid = left <= 0 ? 0 : (left >= V ? V : (int)left);
    uint4 a = src_ll ? ll_load(src + (size_t)v * 32, seq, abort_word, bail, &gave)
                     : ld_user(src + (size_t)v * 16, valid, E, aligned);
    if (s_in) a = vadd<DT>(ll_load(s_in + (size_t)v * 32, seq, abort_word, bail, &gave), a);
    if (gave) break;                       // an abandoned item writes nothing more
    if (d_rem) ll_store(d_rem + (size_t)v * 32, a, seq);
    if (d_loc) {
      if (loc_user) st_user(d_loc + (size_t)v * 16, a, valid, E, aligned);
      else st_v4(d_loc + (size_t)v * 16, a);
    }
  }
  return gave;
}

// ------------------------------------------------------------ LL128 protocol
// (reading R-12; r2ccl.h "Protocols").  A chunk's vectors travel in 128-byte
// lines of 7 payload vectors + one flag vector {seq, seq, seq, seq}: line L of
// a chunk holds its vectors 7L .. 7L+6 (the last line zero-padded).  Eight
// consecutive lanes of a warp own one line, so ONE warp-wide 16-byte store
// instruction writes four whole lines and one 16-byte load instruction reads
// them back: the receiver accepts a line when its flag vector equals the
// collective's seq, which relies on a 128-byte line written by one warp store
// being observed whole across NVLink (the property NCCL's LL128 relies on;
// checked by tools/ll128_tear.cu).  Every line a part touches is written
// WHOLE by that part (vectors outside the part are recomputed from the same
// inputs, so two parts sharing a boundary line write identical bytes).
#define LL128_PAY 7
// line groups per warp per iteration: 2 for items of up to R2_LL128_SMALL
// lines, 4 above (U = 2 measured 8 % faster at 16 MiB, 4 % at 32 MiB and 3 %
// slower at 64-128 MiB than U = 4 at N=4; U = 3 and U = 8 slower:
// profiles/r02_ll128_unroll.txt)
#ifndef R2_LL128_SMALL
#define R2_LL128_SMALL 1024
#endif
#ifndef R2_LL128_ULARGE
#define R2_LL128_ULARGE 4
#endif
#ifndef R2_LL128_TINY
#define R2_LL128_TINY 256        // chunks of up to this many lines: one line group per iteration
#endif
template <int U>
__device__ __forceinline__ bool ll128_validate(uint4 (&x)[U], const bool (&act)[U], const char* q,
                                               const unsigned int (&L)[U], unsigned int lane, unsigned int seq,
                                               const volatile unsigned int* abort_word, const volatile int* bail) {
  const unsigned int pos = lane & 7u;
  for (unsigned int spins = 0;; ++spins) {
    bool ok = true;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool f = !act[u] || (x[u].x == seq && x[u].y == seq && x[u].z == seq && x[u].w == seq);
      ok &= __shfl_sync(0xFFFFFFFFu, f, lane | 7u);      // the line's flag lane decides
    }
    if (__all_sync(0xFFFFFFFFu, ok)) return true;
    if ((spins & 0x3Fu) == 0x3Fu) {
      const int gv = __shfl_sync(0xFFFFFFFFu, lane == 0 ? (int)(*bail != 0) : 0, 0);
      if (gv) return false;                              // abandoned (Shared::abandon)
    }
    if ((spins & 0x3FFu) == 0x3FFu) {
      const int ab = __shfl_sync(0xFFFFFFFFu, lane == 0 ? (int)(*abort_word == seq) : 0, 0);
      if (ab) return true;
    }
    // reload every line of the warp: the 8 lanes of a line must read it with
    // ONE converged load instruction (a line read in pieces can pair a new
    // flag with an old payload)
    R2_SPIN_PAUSE();
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (act[u]) x[u] = ll_line(q + (size_t)L[u] * 128 + pos * 16);
  }
}

// Part [lo, lo + nvec) of a chunk of cvec vectors.  src: user memory at the
// part's first vector, or (src_ll) the chunk's lines in an LL128 slot; s_in:
// the chunk's lines (or null); d_rem: the chunk's lines at the peer (or null);
// d_loc: user memory / stage at the part's first vector (or null).  dtid / dn:
// thread index / count over the data warps (multiples of 32).  Line loads and
// line stores are issued by the converged warp (__syncwarp before each), so
// the 8 lanes of a line always access it in one instruction.
template <int DT, int U>
__device__ bool move_ll128(const LaunchParams& p, unsigned int dtid, unsigned int dn, const char* src, bool src_ll,
                           const char* s_in, char* d_rem, char* d_loc, bool loc_user, unsigned long long e0,
                           unsigned int lo, unsigned int nvec, unsigned int cvec, unsigned long long lim,
                           bool aligned, unsigned int seq, const volatile unsigned int* abort_word,
                           const volatile int* bail) {
  const int E = p.elem_bytes, V = p.V;
  const unsigned int lane = dtid & 31u, wid = dtid >> 5, nw = dn >> 5;
  const unsigned int pos = lane & 7u;
  const unsigned int L0 = lo / LL128_PAY, L1 = (lo + nvec + LL128_PAY - 1) / LL128_PAY;
  const uint4 flag = make_uint4(seq, seq, seq, seq);
  for (unsigned int base = L0 + wid * 4u * U; base < L1; base += nw * 4u * U) {
    uint4 a[U], b[U];
    bool act[U];
    unsigned int L[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      L[u] = base + (unsigned int)u * 4u + (lane >> 3);
      act[u] = L[u] < L1;                 // the same for the 8 lanes of a line
      a[u] = make_uint4(0u, 0u, 0u, 0u);
      b[u] = make_uint4(0u, 0u, 0u, 0u);
    }
    // 1. line loads (converged), validated
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (src_ll && act[u]) a[u] = ll_line(src + (size_t)L[u] * 128 + pos * 16);
      if (s_in && act[u]) b[u] = ll_line(s_in + (size_t)L[u] * 128 + pos * 16);
    }
    // 2. user loads (independent of the lines: issued before the validation
    //    waits on them; may diverge -- masked tails, unaligned buffers)
    if (!src_ll) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned int vc = L[u] * LL128_PAY + pos;
        if (act[u] && pos < LL128_PAY && vc < cvec) {
          const long long ev = (long long)e0 + ((long long)vc - (long long)lo) * V;
          const long long left = (long long)lim - ev;
          const int valid = left <= 0 ? 0 : (left >= V ? V : (int)left);
          a[u] = ld_user(src + ((long long)vc - (long long)lo) * 16, valid, E, aligned);
        }
      }
    }
    if (src_ll && !ll128_validate<U>(a, act, src, L, lane, seq, abort_word, bail)) return true;
    if (s_in && !ll128_validate<U>(b, act, s_in, L, lane, seq, abort_word, bail)) return true;
    // 3. sums, then the line stores (converged) and the part's local copies
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned int vc = L[u] * LL128_PAY + pos;
      const bool pay = pos < LL128_PAY && vc < cvec;
      uint4 v = pay ? a[u] : make_uint4(0u, 0u, 0u, 0u);
      if (pay && s_in) v = vadd<DT>(b[u], v);
      a[u] = pos == LL128_PAY ? flag : v;
    }
    if (d_rem) {
      __syncwarp();
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (act[u]) st_v4(d_rem + (size_t)L[u] * 128 + pos * 16, a[u]);
    }
    if (d_loc) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned int vc = L[u] * LL128_PAY + pos;
        if (act[u] && pos < LL128_PAY && vc < cvec && vc >= lo && vc < lo + nvec) {
          const long long ev = (long long)e0 + ((long long)vc - (long long)lo) * V;
          if (loc_user) {
            const long long left = (long long)lim - ev;
            const int valid = left <= 0 ? 0 : (left >= V ? V : (int)left);
            st_user(d_loc + (size_t)(vc - lo) * 16, a[u], valid, E, aligned);
          } else {
            st_v4(d_loc + (size_t)(vc - lo) * 16, a[u]);
          }
        }
      }
    }
  }
  return false;
}

// ------------------------------------------------------------ control polls
// Thread 0 only.  Looks at the device-local abort word, the alert word
// (set on every rank by a firing fault) and, once alerted, the host-mapped
// control block (abort, stop mask, plan epoch).
__device__ int poll_control(const Cta& k, Shared& sh) {
  R2_ASSUME_SHARED(k, sh);
  sh.t_prev_poll = sh.t_poll;
  sh.t_poll = gtimer();
  sh.npoll++;
  if (ld_relaxed_sys(k.me->abort) == k.seq) return ST_ABORT;
  if (!sh.alerted) {
    if (ld_relaxed_sys(k.me->alert) == k.seq) sh.alerted = 1;
  }
  if (sh.alerted) {
    DevCtrl* C = k.me->dctrl;
    if (ld_relaxed_sys(&C->plan_seq) == k.seq) {
      const unsigned int ab = ld_relaxed_sys(&C->abort);
      if (ab) {
        sh.cause = STOP_ABORT;
        sh.abort_code = ab;
        return ST_ABORT;
      }
      if (ld_relaxed_sys(&C->stop_mask) >> k.cg & 1u) {
        sh.cause = STOP_HOST;
        return ST_STOP;
      }
      if (ld_acquire_gpu(&C->epoch) != sh.seen_epoch) return ST_REPLAN;
    }
  }
  return ST_OK;
}

__device__ __forceinline__ bool conn_phys_dead(const Cta& k) {
  if (k.fault_channel) return false;   // deterministic stop rule applies instead
  const LaunchParams& p = *k.p;
  // a LINK is the standard ring's r -> r+1 (reading R-10): other pairs only die with an endpoint
  const bool std_link = k.r1 == (k.r + 1) % p.ng;
  return ld_relaxed_sys(k.me->ep_dead + k.r * p.Kg + k.cg) | ld_relaxed_sys(k.me->ep_dead + k.r1 * p.Kg + k.cg) |
         (std_link ? ld_relaxed_sys(k.me->link_dead + k.r * p.Kg + k.cg) : 0u);
}

// watchdog: returns true when expired
__device__ __forceinline__ bool watchdog(const Cta& k, Shared& sh) {
  unsigned long long now = gtimer();
  if (sh.wait_t0 == 0) { sh.wait_t0 = now; return false; }
  return now - sh.wait_t0 > k.p->watchdog_ns;
}

// control lane: peer's recv pointer for this seq, without blocking (real
// mode: the descriptor the downstream rank publishes at kernel start)
__device__ bool try_recv_next(const Cta& k, Shared& sh) {
  const LaunchParams& p = *k.p;
  if (sh.recv_next) return true;
  if (p.sim) {
    sh.recv_next = p.recv[k.r1 - p.first_rank];
    return true;
  }
  const volatile unsigned long long* d = k.nx->desc + k.par * 4;
  if ((unsigned int)ld_relaxed_sys64(d) != k.seq) return false;
  fence_sys();
  unsigned long long reg = ld_relaxed_sys64(d + 1), off = ld_relaxed_sys64(d + 2);
  sh.recv_next = (char*)(p.regtab[reg * p.ng + k.r1] + off + p.peer_recv_off);
  return true;
}

// thread 0: fire an armed fault ("Failures may occur mid-chunk").
__device__ void fire_fault(const Cta& k, const FaultDev& f, int t, int o, int j) {
  const LaunchParams& p = *k.p;
  unsigned long long t_fire = gtimer();
  fence_sys();
  for (int q = 0; q < p.ng; ++q) {
    const RankPtrs& rp = p.peers[k.l * p.ng + q];
    if (f.kind == 2) st_relaxed_sys(rp.link_dead + k.r * p.Kg + k.cg, 1u);        // LINK
    else if (f.kind == 0) st_relaxed_sys(rp.ep_dead + k.r * p.Kg + k.cg, 1u);     // LOCAL
    else st_relaxed_sys(rp.ep_dead + k.r1 * p.Kg + k.cg, 1u);                     // REMOTE
  }
  fence_sys();
  for (int q = 0; q < p.ng; ++q) st_relaxed_sys(p.peers[k.l * p.ng + q].alert, k.seq);
  fence_sys();
  // the sender's transport error surfaces after detect_delay_us (reading C-17)
  unsigned long long delay = (unsigned long long)f.detect_delay_us * 1000ull;
  while (gtimer() - t_fire < delay) {
  }
  ErrRec& e = k.ctrl->err[k.cg];
  e.cause = STOP_FAULT_FIRED;
  e.origin = (unsigned int)p.chan[o];
  e.q = (unsigned int)(t * p.m + j);
  e.t_fire = t_fire;
  __threadfence_system();
  e.seq = k.seq;
  __threadfence_system();
}

// control lane: item delivered -> completion word (+ Balance counter).  The
// caller has issued the release fence (one for every chunk retired together).
// dl_acc / by_acc: the rank's delivered-items and this channel's byte
// counters, accumulated over a retire batch by the caller (one atomic each
// per batch instead of two per chunk)
__device__ void complete_item(const Cta& k, Shared& sh, int t, int o, int j, unsigned int parts,
                              unsigned int epoch, bool own, unsigned int nbytes, bool local, unsigned int& dl_acc,
                              unsigned long long& by_acc) {
  const LaunchParams& p = *k.p;
  bool last = true;
  const size_t fi = fidx(p, t, o, j);
  if (parts > 1) {
    unsigned long long* ctr = k.me->counters + fi;
    const unsigned long long tag = (unsigned long long)(((k.seq & 0xFFFFFFu) << 8) | (epoch & 0xFFu)) << 32;
    unsigned long long old = *(volatile unsigned long long*)ctr, prev, nw;
    unsigned int cnt;
    for (;;) {
      cnt = ((old & 0xFFFFFFFF00000000ull) == tag) ? (unsigned int)(old & 0xFFFFFFFFu) + 1u : 1u;
      nw = tag | cnt;
      prev = atomicCAS(ctr, old, nw);
      if (prev == old) break;
      old = prev;
    }
    last = cnt == parts;
    if (last && !p.ll) fence_sys();
  }
  if (last) {
    // the completion word lives with its consumer: the receiver, or this rank
    // itself for a LOCAL item (ReduceScatter's final add, reading R-5)
    st_relaxed_sys((local ? k.me->flags : k.nx->flags) + fi, k.seq);
    dl_acc++;
  }
  if (!local) by_acc += nbytes;
  if (!own && sh.first_adopt == 0) {
    // failover latency endpoint: first retransmitted chunk's flag
    sh.first_adopt = gtimer();
    CtaRec& rec = k.ctrl->cta[k.cta_in_rank];
    rec.t_first_adopt = sh.first_adopt;
    __threadfence_system();
    rec.adopt_tag = (k.seq << 8) | (epoch & 0xFFu);
  }
}

// ------------------------------------------------------------ work list
// The merged work list of one CTA in (step, origin, chunk) order: its own
// chunks (j = w, w+W, ...) and the chunks it adopts for dead origins (static
// plan: plan-time placement from the health records; dynamic plan: the
// monitor's plan entries; a re-placed chunk is skipped once its completion
// word is set).  Resumable iterator of the control lane.
struct Iter {
  int t, o, j;
};
struct ItemRef {
  int t, o, j;
  unsigned int lo, hi, parts, epoch;
  bool own;
};

__device__ bool iter_next(const Cta& k, const Shared& sh, Iter& it, ItemRef& out) {
  R2_ASSUME_SHARED(k, sh);
  const LaunchParams& p = *k.p;
  if (k.all_healthy && !sh.dynamic && !sh.freeze) {
    // healthy static plan: the lane's own chunks only, (t, c, j = w, w+W, ...)
    // in order -- O(1) per item (the general walk below visits all K origins
    // of every step, a few microseconds per item for one thread)
    const int m = p.m, W = p.W;
    while (it.t < p.steps) {
      if (k.t_act >= 0 && it.t != k.t_act) {         // Broadcast: only this rank's chain step
        if (it.t > k.t_act) return false;
        it.t = k.t_act;                              // (the last rank of the chain: t_act = steps)
        it.o = 0;
        it.j = k.w;
        continue;
      }
      if (it.o < k.c) {
        it.o = k.c;
        it.j = k.w;
      }
      if (it.o == k.c && it.j < m) {
        const int j = it.j;
        it.j += W;
        if (keyof(it.t, k.c, j) < k.own_next_key) continue;
        out.t = it.t;
        out.o = k.c;
        out.j = j;
        out.lo = 0;
        out.hi = j == m - 1 ? p.cvec_last : p.cvec_full;
        out.parts = 1;
        out.epoch = 0;
        out.own = true;
        return true;
      }
      it.o = 0;
      it.j = k.w;
      it.t++;
    }
    return false;
  }
  while (it.t < p.steps) {
    if (k.t_act >= 0 && it.t != k.t_act) {           // Broadcast: only this rank's chain step
      if (it.t > k.t_act) return false;
      it.t = k.t_act;
      it.o = 0;
      it.j = k.w;
      continue;
    }
    const int t = it.t, o = it.o;
    const bool own = (o == k.c) && k.own_alive;
    unsigned int mode = PLAN_NONE, mask = 0, assignee = 0, epoch = 0;
    bool dyn = false;
    bool usable = true;
    if (!own) {
      if (sh.freeze) {
        usable = false;
      } else if (sh.dynamic) {
        for (int e = 0; e < sh.nent; ++e)
          if ((int)sh.ent[e].origin == o) {
            mode = sh.ent[e].mode;
            mask = sh.ent[e].mask;
            assignee = sh.ent[e].assignee;
            dyn = true;
          }
        epoch = sh.seen_epoch;
      } else if (!(k.conn_mask >> o & 1u)) {
        mask = k.conn_mask;
        if (p.strategy == 0) {
          mode = PLAN_HOT;
          assignee = 0xFFFFFFFFu;
          for (int d = 1; d < p.K; ++d)
            if (mask >> ((o + d) % p.K) & 1u) {
              assignee = (unsigned int)((o + d) % p.K);
              break;
            }
        } else {
          mode = PLAN_BAL;
        }
      }
      if (mode == PLAN_NONE) usable = false;
      else if (mode == PLAN_HOT && assignee != (unsigned int)k.c) usable = false;
      else if (mode == PLAN_BAL && !(mask >> k.c & 1u)) usable = false;
    }
    if (usable) {
      for (; it.j < p.m; it.j += p.W) {
        const int j = it.j;
        const unsigned long long key = keyof(t, o, j);
        if (own && key < k.own_next_key) continue;
        // after an abandonment own items from the abandoned key on come back:
        // those already completed are skipped (never completed twice)
        if (own && sh.reissue &&
            (int)(ld_relaxed_sys((t == p.local_step ? k.me->flags : k.nx->flags) + fidx(p, t, o, j)) - k.seq) >= 0)
          continue;
        // re-placed chunks: exactly those without a completion (reading C-7);
        // the origin's own lanes have quiesced and no part of an older plan
        // is in flight (freeze), so the receiver's flags are stable evidence
        if (dyn && (int)(ld_relaxed_sys((t == p.local_step ? k.me->flags : k.nx->flags) + fidx(p, t, o, j)) - k.seq) >= 0)
          continue;
        const unsigned int Vj = j == p.m - 1 ? p.cvec_last : p.cvec_full;
        unsigned int lo = 0, hi = Vj, parts = 1;
        if (!own && mode == PLAN_BAL) {
          bal_part(Vj, mask, p.weights, p.K, k.c, lo, hi, parts);
          if (hi == lo) continue;
        }
        out.t = t;
        out.o = o;
        out.j = j;
        out.lo = lo;
        out.hi = hi;
        out.parts = parts;
        out.epoch = epoch;
        out.own = own;
        it.j += p.W;
        return true;
      }
    }
    it.o++;
    it.j = k.w;
    if (it.o == p.K) {
      it.o = 0;
      it.t++;
    }
  }
  return false;
}

// ------------------------------------------------------------ control lane
// Decide one chunk (fault table, control block, emulated death, input
// arrived?) and, when ready, publish its descriptor into the next slot.
// Returns ST_OK (published; *fired if it carries an armed fault),
// ST_NOTREADY, or a terminal status (cause in sh.cause).
__device__ int try_publish(Cta& k, Shared& sh, const ItemRef& it, bool first_try, bool* fired) {
  R2_ASSUME_SHARED(k, sh);
  const LaunchParams& p = *k.p;
  const int n = p.n;
  int fire = 0;
  unsigned int fire_nvec = 0;
  int poison = 0;
  const bool prof = p.trace == 3 && k.cta_in_rank == 0 && k.l == 0;
  long long q0 = prof ? clock64() : 0;
#define R2_PH(i)                \
  if (prof) {                   \
    const long long q = clock64(); \
    sh.ph[i] += q - q0;         \
    q0 = q;                     \
  }
  const unsigned long long key = keyof(it.t, it.o, it.j);
  for (int i = 0; i < p.nfaults; ++i) {
    const FaultDev& f = p.faults[i];
    if ((int)f.rank != k.r || (int)f.channel != k.cg || f.kind > 2) continue;
    const unsigned long long kf = keyof(f.t, f.origin, f.j);
    // own-origin faults: deterministic "dead from k* on" for every lane of the
    // channel (reading R-1); adopted-chunk faults fire when (and if) carried
    if (key > kf && (int)f.origin == k.c) {
      sh.cause = STOP_FAULT_TABLE;
      return ST_STOP;
    }
    if (key == kf) {
      fire = 1 + i;
      const unsigned long long bv = f.b / 16;
      fire_nvec = (unsigned int)(bv < (it.hi - it.lo) ? bv : (it.hi - it.lo));
      poison = f.poison;
    }
  }
  R2_PH(0);
  // control words and the emulated fabric state: at most once per ~10 us
  // (40k SM cycles; each check is a handful of global loads, ~2.5 us per
  // publish when done every time -- it was the latency floor of small LL
  // collectives).  Faults of this lane's own channel stop it
  // deterministically (above); a death caused elsewhere, a stop or a new
  // plan is noticed within the interval (failover takes ~300 us).
  if (first_try) {
    const unsigned long long now = (unsigned long long)clock64();   // SM cycles: cheap to read
    if (now - sh.t_ctl >= 40000ull) {
      sh.t_ctl = now;
      const int st = poll_control(k, sh);
      if (st != ST_OK) return st;
      if (conn_phys_dead(k)) {
        sh.cause = STOP_DEATH;
        return ST_STOP;
      }
    }
  }
  // LL speculation: while this rank's plan is the healthy static one (no
  // alert, no adoption), an LL item is published before its input's
  // completion word -- the data warps wait on the self-validating lines
  // themselves, so a ring step costs one line flight instead of line + word.
  // Deadlock-free: every lane then holds only its own items, in key order,
  // and an own item's inputs never depend on a later item of the same lane.
  // Once alerted, items wait for the completion word again (an adopted
  // residual must never queue behind a spinning item that needs it).
  R2_PH(1);
  const bool spec = p.ll && p.spec_ok && !sh.alerted && !sh.dynamic;
  if (it.t > 0 && !spec) {
    const unsigned int* w = k.me->flags + fidx(p, it.t - 1, it.o, it.j);
    if ((int)(ld_relaxed_sys(w) - k.seq) < 0) return ST_NOTREADY;
    // the word is there: ONE sys-scope acquire of it (not one per poll) orders
    // the data warps' payload loads after the sender's release -- thread 0's
    // acquire, then the slot's mbarrier release/acquire (CTA scope), form the
    // causality chain of the PTX memory model
    if (!p.ll) (void)ld_acquire_sys(w);
  }
  R2_PH(2);
  const int t = it.t;
  const int ta = t + p.t0;                            // the AllReduce step this op-step is
  const bool local = t == p.local_step;
  if (p.peer_recv && (ta >= n - 1 || p.op == R2_OP_BROADCAST || (p.op == R2_OP_R2CC_STAGE2 && t > 0)) && !local &&
      !try_recv_next(k, sh))
    return ST_NOTREADY;
  if (p.lane_ps_per_byte && !local) {
    // channel bandwidth model (r2ccl.h channel_gbps): a token bucket per lane
    const unsigned long long now = gtimer();
    if (now < sh.pace_next) return ST_NOTREADY;
    const unsigned long long wire = (unsigned long long)(it.hi - it.lo) * (p.ll == 2 ? 18ull : p.ll ? 32ull : 16ull);
    sh.pace_next = (now > sh.pace_next ? now : sh.pace_next) + wire * p.lane_ps_per_byte / 1000ull;
  }

  R2_PH(3);
  const int E = p.elem_bytes, V = p.V;
  const bool chain = p.op == R2_OP_BROADCAST || p.op == R2_OP_R2CC_STAGE2;
  // shard of this step (computed once per CTA: sh.sbase / sh.slim, worker_main)
  const unsigned long long off =
      (unsigned long long)it.o * p.slice + (unsigned long long)it.j * p.chunk + (unsigned long long)it.lo * V;
  const unsigned long long sbase = sh.sbase[t];
  const unsigned long long e0 = sbase + off;
  const unsigned int u = sh.pub % NSLOT;
  // built in registers and stored to the slot at the end: a field-by-field
  // store into shared memory, which also holds the launch parameters, made the
  // compiler re-issue every later parameter load behind each store
  Slot d{};
  Meta m{};
  sh.slot_ab[u] = 0;
  d.status = SLOT_GO;
  d.nvec = fire ? fire_nvec : (it.hi - it.lo);
  d.total = it.hi - it.lo;
  d.poison = fire && poison;
  d.e0 = e0;
  d.lim = sh.slim[t];
  d.rs = ta <= n - 2;
  d.src_ll = 0;
  if (p.op == R2_OP_R2CC_STAGE2) {
    // R²CCL-AllReduce's tailored broadcast (reading R-9): the degraded
    // rank (position 0) sends its input into the next rank's tailor buffer;
    // position 1 adds it to its partial result (IEEE addition commutes:
    // hop_add(p, x_f) bit for bit), keeps the sum and sends it on; the chain
    // forwards it back around to the degraded rank
    d.rs = 0;
    d.s_in = nullptr;
    d.d_loc = nullptr;
    d.loc_user = 1;
    if (t == 0) {
      d.src = p.send[k.l] + off * E;
      d.d_rem = k.nx->tailor + off * E;
      d.rs = 1;                                       // library memory: whole vectors
    } else {
      d.src = (const char*)p.recv[k.l] + off * E;
      d.d_rem = sh.recv_next + off * E;
      if (t == 1) {
        d.s_in = k.me->tailor + off * E;
        d.d_loc = p.recv[k.l] + off * E;
      }
    }
    d.rem_user = !d.rs;
  } else if (p.op == R2_OP_BROADCAST) {
    // chain: the root's input (t = 0), else what arrived here; into the next rank's recv
    d.rs = 0;
    d.src = (t == 0 ? p.send[k.l] : (const char*)p.recv[k.l]) + off * E;
    d.s_in = nullptr;
    d.d_rem = sh.recv_next + off * E;
    d.rem_user = 1;
    d.d_loc = (t == 0 && !p.ag_inplace) ? p.recv[k.l] + off * E : nullptr;
    d.loc_user = 1;
  } else if (p.ll) {
    // LL: scratch traffic as lines; slot index = the AllReduce step that sends
    // into it (RS hops 0..n-2, AG sends n-1..2n-3), offsets doubled.  LL128:
    // each chunk owns ceil(chunk vectors / 7) whole lines of the slot; the
    // slot pointers address the chunk's first line, the user pointers the
    // part's first vector (move_ll128)
    const unsigned long long lo =
        p.ll == 2 ? ((unsigned long long)it.o * p.m + it.j) * p.lc128 * 128ull : off * E * 2;
    d.cvec = it.j == p.m - 1 ? p.cvec_last : p.cvec_full;
    d.lo_c = it.lo;
    d.rs = 1;                                         // d_rem is library scratch
    if (ta <= n - 2) {                                // reduce-scatter hop
      d.src = p.send[k.l] + e0 * E;
      d.s_in = t > 0 ? ll_slot(*k.me, p, k.par, ta - 1) + lo : nullptr;
      d.d_rem = ll_slot(*k.nx, p, k.par, ta) + lo;
      d.d_loc = nullptr;
      d.loc_user = 0;
    } else if (ta == n - 1 && p.op == R2_OP_ALLREDUCE) {   // final add + first all-gather send
      d.src = p.send[k.l] + e0 * E;
      d.s_in = ll_slot(*k.me, p, k.par, n - 2) + lo;
      d.d_rem = ll_slot(*k.nx, p, k.par, n - 1) + lo;
      d.d_loc = p.inplace ? (k.me->stage + off * E) : (p.recv[k.l] + e0 * E);
      d.loc_user = !p.inplace;
    } else if (ta == n - 1 && p.op == R2_OP_REDUCE_SCATTER) {   // final add into the own output
      d.src = p.send[k.l] + e0 * E;
      d.s_in = ll_slot(*k.me, p, k.par, n - 2) + lo;
      d.d_rem = nullptr;
      d.d_loc = p.recv[k.l] + off * E;
      d.loc_user = 1;
    } else if (ta == n - 1) {                         // all-gather: the owner sends its own shard
      d.src = p.send[k.l] + off * E;
      d.s_in = nullptr;
      d.d_rem = ll_slot(*k.nx, p, k.par, n - 1) + lo;
      d.d_loc = p.ag_inplace ? nullptr : (p.recv[k.l] + e0 * E);
      d.loc_user = 1;
    } else if (!local) {                              // all-gather forward: unpack + send on
      d.src = ll_slot(*k.me, p, k.par, ta - 1) + lo;
      d.src_ll = 1;
      d.s_in = nullptr;
      d.d_rem = ll_slot(*k.nx, p, k.par, ta) + lo;
      d.d_loc = p.recv[k.l] + e0 * E;
      d.loc_user = 1;
    } else {                                          // the last all-gather step, unpacked locally
      d.src = ll_slot(*k.me, p, k.par, ta - 1) + lo;
      d.src_ll = 1;
      d.s_in = nullptr;
      d.d_rem = nullptr;
      d.d_loc = p.recv[k.l] + e0 * E;
      d.loc_user = 1;
    }
    d.rem_user = 0;
  } else if (ta <= n - 2) {                           // reduce-scatter hop
    d.src = p.send[k.l] + e0 * E;
    d.s_in = t > 0 ? scratch_slot(*k.me, p, k.par, t - 1) + off * E : nullptr;
    d.d_rem = scratch_slot(*k.nx, p, k.par, t) + off * E;
    d.rem_user = 0;
    d.d_loc = nullptr;
    d.loc_user = 0;
  } else if (ta == n - 1 && p.op == R2_OP_ALLREDUCE) {   // final add + first all-gather send
    d.src = p.send[k.l] + e0 * E;
    d.s_in = scratch_slot(*k.me, p, k.par, n - 2) + off * E;
    d.d_rem = sh.recv_next + e0 * E;
    d.rem_user = 1;
    d.d_loc = p.inplace ? (k.me->stage + off * E) : (p.recv[k.l] + e0 * E);
    d.loc_user = !p.inplace;
  } else if (ta == n - 1 && p.op == R2_OP_REDUCE_SCATTER) {   // final add into the own output (LOCAL)
    d.src = p.send[k.l] + e0 * E;
    d.s_in = scratch_slot(*k.me, p, k.par, n - 2) + off * E;
    d.d_rem = nullptr;
    d.rem_user = 0;
    d.d_loc = p.recv[k.l] + off * E;
    d.loc_user = 1;
  } else if (ta == n - 1) {                           // all-gather: the owner sends its own shard
    d.src = p.send[k.l] + off * E;
    d.s_in = nullptr;
    d.d_rem = sh.recv_next + e0 * E;
    d.rem_user = 1;
    d.d_loc = p.ag_inplace ? nullptr : (p.recv[k.l] + e0 * E);
    d.loc_user = 1;
  } else {                                            // all-gather forward
    d.src = p.recv[k.l] + e0 * E;
    d.s_in = nullptr;
    d.d_rem = sh.recv_next + e0 * E;
    d.rem_user = 1;
    d.d_loc = nullptr;
    d.loc_user = 0;
  }
  d.aligned = ((((d.src_ll ? 0ull : (unsigned long long)d.src)) | (d.rem_user ? (unsigned long long)d.d_rem : 0ull) |
                (d.loc_user ? (unsigned long long)d.d_loc : 0ull)) & 15ull) == 0;
  m.kind = fire ? META_FIRE : META_ITEM;
  m.local = local;
  m.t = t;
  m.o = it.o;
  m.j = it.j;
  m.parts = it.parts;
  m.epoch = it.epoch;
  m.nbytes = (it.hi - it.lo) * 16u;
  m.own = it.own;
  m.fault = fire - 1;
  R2_PH(4);
  sh.slot[u] = d;
  sh.meta[u] = m;
  mbar_arrive(&sh.full[u]);
  if (p.trace == 2 && k.cta_in_rank == 0 && sh.pub < 8) k.me->misc->trace[24 + sh.pub] = gtimer();  // publish i
  sh.pub++;
  if (it.own) {
    k.own_next_key = key + 1;
    if (t < 28) TRACE_MIN(k, 32 + t);
    TRACE_MIN(k, 2);
  }
  *fired = fire != 0;
  R2_PH(5);
#undef R2_PH
  return ST_OK;
}

// Thread 0: the monitor's plan entries (global channel ids, both rings of a
// launch) -> this ring's entries in ring-local channel ids (origins of other
// rings dropped; masks and assignees translated).
__device__ void load_entries(const Cta& k, Shared& sh, int nent) {
  const LaunchParams& p = *k.p;
  const volatile unsigned int* src = (const volatile unsigned int*)k.me->dctrl->entries;
  int out = 0;
  for (int e = 0; e < nent && e < R2_MAXK; ++e) {
    const unsigned int og = ld_relaxed_sys(src + 4 * e + 0), mode = ld_relaxed_sys(src + 4 * e + 1);
    const unsigned int ag = ld_relaxed_sys(src + 4 * e + 2), gmask = ld_relaxed_sys(src + 4 * e + 3);
    int o = -1, a = 0;
    unsigned int mask = 0;
    for (int ci = 0; ci < p.K; ++ci) {
      if ((unsigned int)p.chan[ci] == og) o = ci;
      if ((unsigned int)p.chan[ci] == ag) a = ci;
      if (gmask >> p.chan[ci] & 1u) mask |= 1u << ci;
    }
    if (o < 0) continue;
    sh.ent[out].origin = (unsigned int)o;
    sh.ent[out].mode = mode;
    sh.ent[out].assignee = (unsigned int)a;
    sh.ent[out].mask = mask;
    ++out;
  }
  sh.nent = out;
}

// Control lane: apply a new plan epoch in place (no pipeline drain: chunks
// already published have their inputs and complete on their own).  A freeze
// is acknowledged once no adopted chunk of the old plan is in flight.
__device__ void apply_plan(const Cta& k, Shared& sh) {
  DevCtrl* C = k.me->dctrl;
  const unsigned int e = ld_acquire_gpu(&C->epoch);
  sh.seen_epoch = e;
  sh.freeze = (int)ld_relaxed_sys(&C->freeze);
  const int nent = (int)ld_relaxed_sys(&C->nentries);
  sh.nent = 0;
  sh.first_adopt = 0;
  if (!sh.freeze) {
    load_entries(k, sh, nent);
    sh.dynamic = 1;
    k.ctrl->cta[k.cta_in_rank].t_apply = gtimer();
    k.ctrl->cta[k.cta_in_rank].t_prev_poll = sh.t_prev_poll;
    k.ctrl->cta[k.cta_in_rank].npoll = sh.npoll;
    k.ctrl->cta[k.cta_in_rank].apply_src = 1;
  }
}

// Control lane (thread 0): run the work list through the slot ring until it
// is exhausted or a stop / abort / timeout is decided; every published chunk
// is retired before returning, then an END slot releases the data warps.
// Returns the status (also in sh.pipe_status).
__device__ int control_run(Cta& k, Shared& sh) {
  R2_ASSUME_SHARED(k, sh);
  const LaunchParams& p = *k.p;
  Iter it{0, 0, k.w};
  ItemRef cur;
  // R2_TRACE=3 (diagnostics): SM cycles the control lane of CTA 0 spends in
  // try_publish / iter_next / retiring, into trace slots 50..56
  const bool prof = p.trace == 3 && k.cta_in_rank == 0 && k.l == 0;
  long long c_pub = 0, c_it = 0, c_ret = 0, n_pub = 0, n_it = 0, n_ret = 0;
  const long long c_start = clock64();
  long long c0 = clock64();
  bool have = iter_next(k, sh, it, cur);
  if (prof) c_it += clock64() - c0, n_it++;
  bool first_try = true;
  int pending = ST_OK;
  unsigned int idle = 0;
  unsigned long long t_idle = 0;
  unsigned long long fired_key = ~0ull;   // own chunk that carried a fired fault
  unsigned int last_adopt_pub = 0;        // 1 + slot index of the newest published adopted chunk
  unsigned int ack_epoch = 0;             // freeze epoch still to acknowledge
  // a new plan while line items are in flight: published speculative items may
  // be spinning on inputs that now depend on this lane's residual, so they
  // are abandoned first (Shared::abandon), then the plan is applied and the
  // abandoned items re-issued (reading R-6)
  bool defer_plan = false;
  unsigned long long ab_min = ~0ull;      // smallest abandoned own key
  auto replan_now = [&]() {
    apply_plan(k, sh);
    if (sh.freeze) ack_epoch = sh.seen_epoch;
    it = Iter{0, 0, k.w};                 // rescan: own chunks skip by key, re-placed ones by flag
    have = iter_next(k, sh, it, cur);
    first_try = true;
  };
  auto on_replan = [&]() {
    if (p.ll && sh.pub != sh.fin) {
      sh.abandon = 1;
      defer_plan = true;
    } else {
      replan_now();
    }
  };
  for (;;) {
    bool progress = false;
    // 1. publish as many chunks as possible (slot free, input arrived) BEFORE
    //    retiring: the retire's fence blocks this lane until the retired
    //    chunks' stores have landed, and the data warps must not idle meanwhile
    //    (publishing after the fence cost one chunk transfer per chunk)
    bool replanned = false;
    while (pending == ST_OK && have && !defer_plan && sh.pub - sh.fin < NSLOT) {
      bool fired = false;
      if (prof) c0 = clock64();
      int st = try_publish(k, sh, cur, first_try, &fired);
      if (prof) c_pub += clock64() - c0, n_pub++;
      first_try = false;
      if (st == ST_REPLAN) {
        on_replan();
        replanned = !defer_plan;
        break;
      }
      if (st == ST_OK) {
        progress = true;
        first_try = true;
        if (!cur.own) {
          if (!last_adopt_pub) k.ctrl->cta[k.cta_in_rank].t_pub_adopt = gtimer();
          last_adopt_pub = sh.pub;
        }
        if (fired) {
          if (cur.own) fired_key = keyof(cur.t, cur.o, cur.j);
          pending = ST_STOP;
          sh.cause = STOP_FAULT_FIRED;
          have = false;
        } else {
          if (prof) c0 = clock64();
          have = iter_next(k, sh, it, cur);
          if (prof) c_it += clock64() - c0, n_it++;
        }
      } else {
        if (st != ST_NOTREADY) {
          pending = st;
          have = false;
        }
        break;
      }
    }
    if (replanned) continue;
    // 2. retire finished chunks in order: ONE release fence for all of them
    unsigned int nd = 0;
    while (sh.fin + nd != sh.pub) {
      const unsigned int u = sh.fin + nd;
      if (!mbar_test(&sh.empty[u % NSLOT], (u / NSLOT) & 1u)) break;
      ++nd;
    }
    if (nd) {
      if (prof) c0 = clock64(), n_ret += nd;
      bool any = false;
      for (unsigned int i = 0; i < nd; ++i) any |= sh.meta[(sh.fin + i) % NSLOT].kind != META_END;
      if (any && !p.ll) fence_sys();   // LL lines validate themselves: no fence
      unsigned int dl_acc = 0;
      unsigned long long by_acc = 0;
      for (unsigned int i = 0; i < nd; ++i) {
        const Meta& m = sh.meta[(sh.fin + i) % NSLOT];
        if (m.kind == META_ITEM && sh.slot_ab[(sh.fin + i) % NSLOT]) {
          // abandoned: no completion; re-issued after the new plan
          if (m.own) {
            const unsigned long long key = keyof(m.t, m.o, m.j);
            ab_min = key < ab_min ? key : ab_min;
            sh.reissue = 1;
          }
        } else if (m.kind == META_ITEM) {
          complete_item(k, sh, m.t, m.o, m.j, m.parts, m.epoch, m.own, m.nbytes, m.local != 0, dl_acc, by_acc);
          if (m.own && m.t < 28) TRACE_MAX(k, 4 + m.t);
        } else if (m.kind == META_FIRE) {
          atomicAdd(&k.me->bytes[k.cg], (unsigned long long)sh.slot[(sh.fin + i) % NSLOT].nvec * 16ull);
          fire_fault(k, p.faults[m.fault], m.t, m.o, m.j);
        }
      }
      if (dl_acc) atomicAdd(&k.me->misc->delivered, dl_acc);
      if (by_acc) atomicAdd(&k.me->bytes[k.cg], by_acc);
      if (p.trace == 2 && k.cta_in_rank == 0)
        for (unsigned int i = 0; i < nd; ++i)
          if (sh.fin + i < 8) k.me->misc->trace[16 + sh.fin + i] = gtimer();   // retire i
      sh.fin += nd;
      progress = true;
      if (prof) c_ret += clock64() - c0;
    }
    // 1a. the deferred plan, once every line item in flight came back
    if (defer_plan && sh.fin == sh.pub) {
      sh.abandon = 0;
      if (ab_min < k.own_next_key) k.own_next_key = ab_min;
      ab_min = ~0ull;
      defer_plan = false;
      replan_now();
      continue;
    }
    // 1b. acknowledge a freeze once no adopted chunk is in flight
    if (ack_epoch && sh.fin >= last_adopt_pub) {
      __threadfence_system();            // completion words before the acknowledgement
      k.ctrl->cta[k.cta_in_rank].ack = R2_SS(k.seq, ack_epoch);
      ack_epoch = 0;
    }
    // 2b. an abort / timeout also releases data warps spinning on LL lines
    if ((pending == ST_ABORT || pending == ST_TIMEOUT) && sh.fin != sh.pub && ld_relaxed_sys(k.me->abort) != k.seq)
      st_relaxed_sys(k.me->abort, k.seq);
    // 3. done: everything published is retired -> END releases the data warps
    if ((!have || pending != ST_OK) && sh.fin == sh.pub && !ack_epoch) {
      const unsigned int u = sh.pub % NSLOT;
      sh.slot[u].status = SLOT_END;
      sh.meta[u].kind = META_END;
      sh.pipe_status = pending;
      sh.stop_key = fired_key != ~0ull ? fired_key : k.own_next_key;
      TRACE_MAX(k, 60);
      if (prof) {
        unsigned long long* tr = k.me->misc->trace;
        tr[50] = (unsigned long long)c_pub, tr[51] = (unsigned long long)n_pub;
        tr[52] = (unsigned long long)c_it, tr[53] = (unsigned long long)n_it;
        tr[54] = (unsigned long long)c_ret, tr[55] = (unsigned long long)n_ret;
        tr[56] = (unsigned long long)(clock64() - c_start);
        for (int i = 0; i < 6; ++i) tr[40 + i] = sh.ph[i];
      }
      mbar_arrive(&sh.full[u]);
      sh.pub++;
      return pending;
    }
    // 4. idle: periodic control polls (new plan, stop, abort), emulated death,
    //    watchdog while waiting for an input
    if (progress) {
      idle = 0;
      t_idle = 0;
    } else if ((++idle & 31u) == 0 && pending == ST_OK && !defer_plan) {
      int st = poll_control(k, sh);
      if (st == ST_REPLAN) {
        on_replan();
        continue;
      }
      if (st == ST_OK && have && conn_phys_dead(k)) {
        st = ST_STOP;
        sh.cause = STOP_DEATH;
      }
      if (st != ST_OK) {
        pending = st;
        have = false;
        continue;
      }
      if (have) {
        const unsigned long long now = gtimer();
        if (t_idle == 0) {
          t_idle = now;
        } else if (now - t_idle > p.watchdog_ns) {
          pending = ST_TIMEOUT;
          sh.cause = STOP_TIMEOUT;
          CtaRec& rec = k.ctrl->cta[k.cta_in_rank];     // diagnostics: the input we gave up on
          if (cur.t > 0) {
            const size_t fi = fidx(p, cur.t - 1, cur.o, cur.j);
            rec.wait_idx = (unsigned int)fi;
            rec.wait_val = k.me->flags[fi];
          } else {
            rec.wait_idx = 0x40000000u;
            rec.wait_val = 0;
          }
          have = false;
        }
      }
    }
  }
}

// Data warps: move the published chunks (16-byte vectors straight into the
// peer's memory over NVLink), then signal the slot empty.
template <int DT>
__device__ void data_run(const Cta& k, Shared& sh, unsigned int& dcount) {
  const LaunchParams& p = *k.p;
  const unsigned int dtid = k.tid - 32, dn = k.nthr - 32, lane = k.tid & 31u;
  for (;;) {
    const unsigned int u = dcount % NSLOT, ph = (dcount / NSLOT) & 1u;
    mbar_wait(&sh.full[u], ph);
    ++dcount;
    if (p.trace == 2 && k.cta_in_rank == 0 && k.tid == 32 && dcount <= 8)
      k.me->misc->trace[40 + dcount - 1] = gtimer();   // data warps take item dcount-1
    const Slot d = sh.slot[u];
    if (d.status == SLOT_END) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[u]);
      return;
    }
    bool gave = false;
    if (p.ll == 2)
      gave = d.cvec <= R2_LL128_TINY * LL128_PAY
                 ? move_ll128<DT, 1>(p, dtid, dn, d.src, d.src_ll != 0, d.s_in, d.d_rem, d.d_loc, d.loc_user != 0,
                                     d.e0, d.lo_c, d.nvec, d.cvec, d.lim, d.aligned != 0, k.seq, k.me->abort,
                                     &sh.abandon)
             : d.cvec <= R2_LL128_SMALL * LL128_PAY
                 ? move_ll128<DT, 2>(p, dtid, dn, d.src, d.src_ll != 0, d.s_in, d.d_rem, d.d_loc, d.loc_user != 0,
                                     d.e0, d.lo_c, d.nvec, d.cvec, d.lim, d.aligned != 0, k.seq, k.me->abort,
                                     &sh.abandon)
                 : move_ll128<DT, R2_LL128_ULARGE>(p, dtid, dn, d.src, d.src_ll != 0, d.s_in, d.d_rem, d.d_loc,
                                                   d.loc_user != 0,
                                     d.e0, d.lo_c, d.nvec, d.cvec, d.lim, d.aligned != 0, k.seq, k.me->abort,
                                     &sh.abandon);
    else if (p.ll)
      gave = move_ll<DT>(p, dtid, dn, d.src, d.src_ll != 0, d.s_in, d.d_rem, d.d_loc, d.loc_user != 0, d.e0, d.nvec,
                         d.lim, d.aligned != 0, k.seq, k.me->abort, &sh.abandon);
    else
      move<DT>(p, dtid, dn, d.src, d.s_in, d.d_rem, d.rem_user, d.d_loc, d.loc_user, d.e0, d.nvec, d.lim,
               d.aligned != 0);
    if (d.poison && d.d_rem && p.ll == 2) {
      // LL128: whole lines after the delivered prefix arrive invalid (flag ~0)
      const unsigned int Lf = (d.lo_c + d.nvec + LL128_PAY - 1) / LL128_PAY;
      const unsigned int Le = (d.lo_c + d.total + LL128_PAY - 1) / LL128_PAY;
      for (unsigned int x0 = Lf * 8; x0 < Le * 8; x0 += dn) {
        __syncwarp();
        if (x0 + dtid < Le * 8) st_v4(d.d_rem + (size_t)(x0 + dtid) * 16, make_uint4(~0u, ~0u, ~0u, ~0u));
      }
    } else if (d.poison && d.d_rem && p.ll) {
      // LL: the rest of the faulted part arrives as invalid lines (reading C-6)
      for (unsigned int v = d.nvec + dtid; v < d.total; v += dn) {
        st_v4(d.d_rem + (size_t)v * 32, make_uint4(~0u, ~0u, ~0u, ~0u));
        st_v4(d.d_rem + (size_t)v * 32 + 16, make_uint4(~0u, ~0u, ~0u, ~0u));
      }
    } else if (d.poison && d.d_rem) {
      // poison the rest of the faulted part at the peer (reading C-6)
      for (unsigned int v = d.nvec + dtid; v < d.total; v += dn) {
        const long long ev = (long long)(d.e0 + (unsigned long long)v * p.V);
        const long long left = (long long)d.lim - ev;
        const int valid = left <= 0 ? 0 : (left >= p.V ? p.V : (int)left);
        if (d.rs) st_v4(d.d_rem + (size_t)v * 16, make_uint4(~0u, ~0u, ~0u, ~0u));
        else st_user(d.d_rem + (size_t)v * 16, make_uint4(~0u, ~0u, ~0u, ~0u), valid, p.elem_bytes, d.aligned != 0);
      }
    }
    if (__any_sync(0xFFFFFFFFu, gave) && lane == 0) sh.slot_ab[u] = 1;   // before this warp's arrival
    __syncwarp();
    if (p.trace == 2 && k.cta_in_rank == 0 && k.tid == 32 && dcount <= 8)
      k.me->misc->trace[48 + dcount - 1] = gtimer();   // warp 1 done with item dcount-1
    if (lane == 0) mbar_arrive(&sh.empty[u]);
  }
}

// thread 0 writes this CTA's record
// (one 64-bit store of seq|state).  Only when the monitor may act on it (a
// fault is in flight, or a stop) is it ordered after this CTA's completion
// words with a system fence; the healthy path pays no PCIe round trip.
__device__ void post_state(const Cta& k, const Shared& sh, unsigned int state, unsigned int cause) {
  CtaRec& rec = k.ctrl->cta[k.cta_in_rank];
  if (cause) rec.cause = cause;
  // own chunks with key >= stop_key are not complete (every published chunk
  // was retired before the state changes; a fired chunk never completes)
  rec.stop_key = state == CTA_STOPPED ? sh.stop_key : k.own_next_key;
  if (sh.alerted || state == CTA_STOPPED) {
    rec.t_stop = gtimer();
    __threadfence_system();
  }
  rec.ss = R2_SS(k.seq, state);
}

// all threads: pull the dynamic plan from the control block
__device__ void load_plan(Cta& k, Shared& sh) {
  if (k.tid == 0) {
    DevCtrl* C = k.me->dctrl;
    unsigned int e = ld_acquire_gpu(&C->epoch);
    sh.seen_epoch = e;
    sh.freeze = (int)ld_relaxed_sys(&C->freeze);
    sh.flag = (int)ld_relaxed_sys(&C->nentries);
    sh.nent = 0;
    sh.first_adopt = 0;
  }
  __syncthreads();
  if (!sh.freeze) {
    if (k.tid == 0) {
      load_entries(k, sh, sh.flag);
      sh.dynamic = 1;
      k.ctrl->cta[k.cta_in_rank].t_apply = gtimer();
      k.ctrl->cta[k.cta_in_rank].t_prev_poll = sh.t_prev_poll;
      k.ctrl->cta[k.cta_in_rank].npoll = sh.npoll;
      k.ctrl->cta[k.cta_in_rank].apply_src = 2;
    }
  }
  __syncthreads();
  if (k.tid == 0) {
    __threadfence_system();   // completion words before the acknowledgement
    k.ctrl->cta[k.cta_in_rank].ack = R2_SS(k.seq, sh.seen_epoch);
  }
  __syncthreads();
}

// all threads: wait for the whole rank to finish (delivered + final flags)
__device__ int drain(Cta& k, Shared& sh) {
  const LaunchParams& p = *k.p;
  if (k.tid == 0) {
    post_state(k, sh, CTA_DRAINING, 0);
    sh.wait_t0 = 0;
  }
  bool first = true;
  for (;;) {
    if (k.tid == 0) {
      // first pass: the rank's delivered count first -- when it is complete
      // (the common case) the control words need no look (two dependent
      // global loads); every later pass polls them (a freeze must be
      // acknowledged while this CTA waits for incoming words)
      const unsigned int dl0 = ld_relaxed_sys((volatile unsigned int*)&k.me->misc->delivered);
      int st = first && dl0 >= k.total_items ? ST_OK : poll_control(k, sh);
      first = false;
      int cand = 0;
      if (st == ST_OK) {
        const unsigned int dl = dl0 >= k.total_items ? dl0 : ld_relaxed_sys((volatile unsigned int*)&k.me->misc->delivered);
        cand = dl >= k.total_items;
        if (!cand) {
          if (watchdog(k, sh)) {
            st = ST_TIMEOUT;
            sh.cause = STOP_TIMEOUT;
            k.ctrl->cta[k.cta_in_rank].wait_idx = 0x80000000u | (dl & 0xFFFFFFu);   // drain: delivered
            k.ctrl->cta[k.cta_in_rank].wait_val = k.total_items;
          } else {
            __nanosleep(200);
          }
        }
      }
      sh.decision = st;
      sh.flag = cand;
    }
    __syncthreads();
    const int st = sh.decision;
    const int cand = sh.flag;
    __syncthreads();
    if (st != ST_OK) return st;
    if (!cand) continue;
    // all final incoming completion words present?
    int ok = 1;
    const int nf = p.K * p.m;
    // the root of a Broadcast receives nothing; under LL the last incoming step
    // is consumed by this rank's own unpack items (already delivered)
    const int fs = p.op == R2_OP_BROADCAST      ? k.t_act - 1
                   : p.op == R2_OP_R2CC_STAGE2 ? (k.t_act == 0 ? p.n - 1 : k.t_act - 1)
                   : (p.ll && p.local_step >= 0 ? -1 : p.fin_step);
    const unsigned int* fin = k.me->flags + fidx(p, fs < 0 ? 0 : fs, 0, 0);
    for (int i = k.tid; fs >= 0 && i < nf; i += k.nthr)
      if ((int)(ld_relaxed_sys(fin + i) - k.seq) < 0) ok = 0;
    if (__syncthreads_and(ok)) {
      if (k.tid == 0) TRACE_MAX(k, 61);
      return ST_OK;
    }
    if (k.tid == 0) sh.flag = watchdog(k, sh) ? -1 : 0;
    __syncthreads();
    const int expired = sh.flag == -1;
    __syncthreads();
    if (expired) {
      if (k.tid == 0) {
        sh.cause = STOP_TIMEOUT;
        k.ctrl->cta[k.cta_in_rank].wait_idx = 0xC0000000u;    // drain: final completion words
        k.ctrl->cta[k.cta_in_rank].wait_val = 0;
      }
      return ST_TIMEOUT;
    }
  }
}

// in-place: copy the staged own shard into recv (pieces grabbed atomically)
__device__ void copy_stage(Cta& k, Shared& sh) {
  const LaunchParams& p = *k.p;
  const unsigned long long shard_vec = p.shard / p.V;   // AllReduce only (sstride == shard)
  const unsigned int PIECE = 4096;
  const unsigned long long npieces = (shard_vec + PIECE - 1) / PIECE;
  __threadfence();
  for (;;) {
    if (k.tid == 0) sh.piece = atomicAdd(&k.me->misc->copy_next, 1u);
    __syncthreads();
    const unsigned long long pc = sh.piece;
    __syncthreads();
    if (pc >= npieces) break;
    const unsigned long long v0 = pc * PIECE;
    const unsigned int nv = (unsigned int)min((unsigned long long)PIECE, shard_vec - v0);
    const unsigned long long e0 = (unsigned long long)k.pos * p.shard + v0 * p.V;
    if (e0 >= p.N) continue;
    for (unsigned int v = k.tid; v < nv; v += k.nthr) {
      long long ev = (long long)(e0 + (unsigned long long)v * p.V);
      long long left = (long long)p.N - ev;
      int valid = left <= 0 ? 0 : (left >= p.V ? p.V : (int)left);
      if (!valid) continue;
      uint4 a = ld_cg(k.me->stage + (v0 + v) * 16);
      st_user(p.recv[k.l] + (size_t)ev * p.elem_bytes, a, valid, p.elem_bytes);
    }
  }
}

// thread 0, once per CTA on the way out.  The last CTA of the rank resets
// the per-collective counters (nobody reads them any more in this launch) and
// counts its (ring, rank) pair out; the last pair publishes done_seq and the
// service lane leaves (service_main).
__device__ void last_out(const Cta& k) {
  const unsigned int per_rank = (unsigned int)(k.p->K * k.p->W);
  TRACE_MAX(k, 62);
  if (atomicAdd(&k.me->misc->exited, 1u) == per_rank - 1) {
    k.me->misc->delivered = 0;
    k.me->misc->copy_next = 0;
    __threadfence();
    atomicExch(&k.me->misc->exited, 0u);
    __threadfence();
    // one (ring, rank) pair done (service_main); the last pair of the launch
    // publishes done_seq (posted host writes: the host only paces its
    // in-flight window and drops stale re-plans with it)
    if (atomicAdd(k.p->grid_exited, 1u) == k.p->exit_target - 1) {
      for (int l = 0; l < R2_MAXL && k.p->ctrl[l]; ++l) k.p->ctrl[l]->done_seq = k.seq;   // every local rank
    }
  }
}

// thread 0: this rank's kernel leaves without a complete result (watchdog,
// abort, exhausted chain): record it for r2_sync before the kernel ends
__device__ void post_failure(const Cta& k, unsigned int code) {
  k.ctrl->fail_code = code;
  __threadfence_system();
  k.ctrl->fail_seq = k.seq;
  __threadfence_system();
}

template <int DT>
__device__ void cta_main(Cta& k, Shared& sh) {
  int st;
  unsigned int exit_state = CTA_EXITED;
  if (k.conn_mask == 0) {
    // every outgoing channel of this rank is dead: the chain is exhausted
    // before the collective starts -- abort, the monitor reports it
    if (k.tid == 0) {
      st_relaxed_sys(k.me->abort, k.seq);
      k.ctrl->cta[k.cta_in_rank].cause = STOP_NOBACKUP;
      post_failure(k, R2_ERR_NO_BACKUP);
      k.ctrl->cta[k.cta_in_rank].ss = R2_SS(k.seq, CTA_EXITED);
      last_out(k);
    }
    return;
  }
  unsigned int dcount = 0;   // data warps: slots consumed (monotone across pipeline runs)
  for (;;) {
    // warp-specialized work list: thread 0 controls, warps 1.. move data
    if (k.tid < 32) {
      if (k.tid == 0) control_run(k, sh);
      __syncwarp();
    } else {
      data_run<DT>(k, sh, dcount);
    }
    __syncthreads();
    st = sh.pipe_status;
    __syncthreads();
    if (st == ST_REPLAN) {
      load_plan(k, sh);
      continue;
    }
    if (st != ST_OK) break;
    st = drain(k, sh);
    if (st == ST_REPLAN) {
      load_plan(k, sh);
      continue;
    }
    break;
  }
  if (st == ST_OK) {
    if (k.p->inplace) copy_stage(k, sh);
  } else if (k.tid == 0) {
    exit_state = (st == ST_STOP) ? CTA_STOPPED : CTA_EXITED;
    if (st == ST_TIMEOUT) {
      // local abort: the rest of this rank stops waiting too
      st_relaxed_sys(k.me->abort, k.seq);
    }
    if (st == ST_TIMEOUT || st == ST_ABORT)
      post_failure(k, st == ST_ABORT && sh.abort_code ? sh.abort_code : (unsigned int)R2_ERR_TIMEOUT);
    if (st == ST_STOP && sh.cause == STOP_DEATH) {
      // bilateral awareness starts at the detecting sender; the
      // surviving CTAs of every rank must start reading the control block
      const LaunchParams& p = *k.p;
      for (int q = 0; q < p.ng; ++q) st_relaxed_sys(p.peers[k.l * p.ng + q].alert, k.seq);
      ErrRec& e = k.ctrl->err[k.cg];
      if (e.seq != k.seq) {
        e.cause = STOP_DEATH;
        e.origin = (unsigned int)k.cg;
        e.q = 0;
        e.t_fire = gtimer();
        __threadfence_system();
        e.seq = k.seq;
      }
    }
  }
  if (k.tid == 0) {
    post_state(k, sh, exit_state, st == ST_OK ? 0u : (unsigned int)sh.cause);
    last_out(k);
  }
}

// ------------------------------------------------------------ service lane
// Warp 0 of the service CTA (the last CTA of the cooperative grid) or of the
// standalone service kernel serves the monitor's request ring (r2_internal.h
// SvcBlock): probe-flag stores + read-backs (reading C-11), installs of
// the plan mirror (DevCtrl) and word copies (health records, completion words
// for rollback).  Requests are claimed in order under svc_lock; probes run
// concurrently (up to R2_SVC_MAXPROBES, lanes 0..7 watch one each).
struct SvcProbe {
  int active, dropped;
  unsigned int tag, token, slot;
  unsigned long long t0, timeout_ns, mailbox, result;
};
struct SvcShared {
  SvcReq rq;
  SvcProbe pr[R2_SVC_MAXPROBES];
  int go, nactive;
};

__device__ __forceinline__ void svc_ack(SvcBlock* S, unsigned int slot, unsigned int tag) {
  __threadfence_system();
  S->ack[slot] = tag;
}

// lane 0: start one probe (completion is watched by svc_probes)
__device__ void svc_probe_start(SvcBlock* S, SvcShared& ss, unsigned int slot) {
  const SvcReq& r = ss.rq;
  const unsigned int* ep = (const unsigned int*)r.ep_dead;
  const unsigned int* lk = (const unsigned int*)r.link_dead;
  const int K = r.K, c = r.channel;
  if (r.t_start) *(volatile unsigned long long*)r.t_start = gtimer();
  if (ld_relaxed_sys(ep + r.prober * K + c)) {         // the prober's own endpoint: immediate local error
    *(volatile int*)r.result = R2_PROBE_LOCAL_ERROR;
    svc_ack(S, slot, r.tag);
    return;
  }
  const bool link = ((r.target == (r.prober + 1) % r.n) && ld_relaxed_sys(lk + r.prober * K + c)) ||
                    ((r.prober == (r.target + 1) % r.n) && ld_relaxed_sys(lk + r.target * K + c));
  const bool dropped = link || ld_relaxed_sys(ep + r.target * K + c);
  if (!dropped) {
    st_relaxed_sys((volatile unsigned int*)r.mailbox, r.token);
    fence_sys();
  }
  for (int i = 0; i < R2_SVC_MAXPROBES; ++i)
    if (!ss.pr[i].active) {
      SvcProbe& q = ss.pr[i];
      q.dropped = dropped;
      q.tag = r.tag;
      q.token = r.token;
      q.slot = slot;
      q.t0 = gtimer();
      q.timeout_ns = r.timeout_ns;
      q.mailbox = r.mailbox;
      q.result = r.result;
      q.active = 1;
      ss.nactive++;
      return;
    }
}

// lanes 0..7: finish probes whose read-back arrived or whose timeout expired
__device__ void svc_probes(SvcBlock* S, SvcShared& ss, unsigned int lane) {
  if (lane < R2_SVC_MAXPROBES && ss.pr[lane].active) {
    SvcProbe& q = ss.pr[lane];
    int res = -1;
    if (!q.dropped && ld_acquire_sys((const volatile unsigned int*)q.mailbox) == q.token) res = R2_PROBE_SUCCESS;
    else if (gtimer() - q.t0 >= q.timeout_ns) res = R2_PROBE_TIMEOUT;
    if (res >= 0) {
      *(volatile int*)q.result = res;
      svc_ack(S, q.slot, q.tag);
      q.active = 0;
      atomicSub(&ss.nactive, 1);
    }
  }
  __syncwarp();
}

// whole warp: claim and execute the posted requests (returns with the lock
// released).  A probe request waits for a free probe slot.
__device__ void svc_take(SvcBlock* S, MiscDev* m0, SvcShared& ss, unsigned int lane) {
  if (lane == 0) ss.go = atomicCAS(&m0->svc_lock, 0u, 1u) == 0u;
  __syncwarp();
  if (!ss.go) return;
  for (;;) {
    if (lane == 0) {
      __threadfence();
      const unsigned int tail = *(volatile unsigned int*)&m0->svc_tail;
      const unsigned int head = S->head;
      ss.go = (tail != head) && ss.nactive < R2_SVC_MAXPROBES;
    }
    __syncwarp();
    if (!ss.go) break;
    const unsigned int tail = *(volatile unsigned int*)&m0->svc_tail;
    const unsigned int slot = tail % R2_SVC_RING;
    // the request (host-mapped): every lane loads 8-byte words, one PCIe round trip
    {
      const volatile unsigned long long* src = (const volatile unsigned long long*)&S->req[slot];
      unsigned long long* dst = (unsigned long long*)&ss.rq;
      for (unsigned int i = lane; i < sizeof(SvcReq) / 8; i += 32) dst[i] = src[i];
    }
    __syncwarp();
    const SvcReq& r = ss.rq;
    if (r.kind == SVC_MIRROR) {
      // body, fence, then the word that publishes it (plan_seq for a new
      // collective, epoch for an update): same order as the CTAs read it
      volatile unsigned int* d = (volatile unsigned int*)r.dst;
      const unsigned int* v = (const unsigned int*)&r.v;
      for (unsigned int i = 2 + lane; i < sizeof(DevCtrl) / 4; i += 32) d[i] = v[i];
      __threadfence();
      __syncwarp();
      if (lane == 0) {
        d[1] = r.v.epoch;
        if (r.mode == 0) {
          __threadfence();
          d[0] = r.v.plan_seq;
        }
        __threadfence();
        svc_ack(S, slot, r.tag);
      }
    } else if (r.kind == SVC_COPY) {
      const volatile unsigned int* a = (const volatile unsigned int*)r.src;
      volatile unsigned int* b = (volatile unsigned int*)r.dst;
      for (unsigned int i = lane; i < r.nwords; i += 32) b[i] = ld_relaxed_sys(a + i);
      __threadfence_system();
      __syncwarp();
      if (lane == 0) svc_ack(S, slot, r.tag);
    } else if (r.kind == SVC_STORE) {
      if (lane == 0) {
        st_relaxed_sys((volatile unsigned int*)r.dst, r.nwords);
        svc_ack(S, slot, r.tag);
      }
    } else if (r.kind == SVC_PROBE) {
      if (lane == 0) svc_probe_start(S, ss, slot);
    } else if (lane == 0) {
      svc_ack(S, slot, r.tag);                        // unknown kind: consumed
    }
    __syncwarp();
    if (lane == 0) {
      *(volatile unsigned int*)&m0->svc_tail = tail + 1;
      __threadfence();
    }
    __syncwarp();
  }
  if (lane == 0) {
    __threadfence();
    atomicExch(&m0->svc_lock, 0u);
  }
  __syncwarp();
}

// Resident flavour (the service CTA of a collective): serve until every local
// rank's worker CTAs have left (the last of them published done_seq).
__device__ void service_main(const LaunchParams& p) {
  __shared__ SvcShared ss;
  const unsigned int lane = threadIdx.x & 31u;
  SvcBlock* S = p.svc;
  MiscDev* m0 = p.peers[p.first_rank].misc;             // local rank 0's ring-0 misc (svc lock / tail)
  if (lane == 0) {
    ss.nactive = 0;
    for (int i = 0; i < R2_SVC_MAXPROBES; ++i) ss.pr[i].active = 0;
    S->alive = R2_SS(p.seq, 1);
  }
  __syncwarp();
  unsigned long long t_head = gtimer();
  unsigned int head_seen = 0, tail_seen = 0;
  // the host's head word costs a PCIe round trip (~1 us): it is loaded every
  // ~2 us and its value used only at the NEXT load, so the lane never stalls
  // on it (the exit check below stays prompt when the last worker leaves)
  unsigned int head_inflight = S->head;
  for (;;) {
    int take = 0;
    if (lane == 0) {
      const unsigned long long now = gtimer();
      if (now - t_head >= 2000ull) {
        t_head = now;
        head_seen = head_inflight;
        head_inflight = S->head;
        tail_seen = *(volatile unsigned int*)&m0->svc_tail;
      }
      take = head_seen != tail_seen;
    }
    take = __shfl_sync(0xFFFFFFFFu, take, 0);
    if (take) {
      svc_take(S, m0, ss, lane);
      if (lane == 0) {                                // look again right away
        head_seen = head_inflight = S->head;
        tail_seen = *(volatile unsigned int*)&m0->svc_tail;
        t_head = gtimer();
      }
    }
    if (ss.nactive) svc_probes(S, ss, lane);
    int out = 0;
    if (lane == 0)
      out = ss.nactive == 0 && ld_relaxed_sys((const volatile unsigned int*)p.grid_exited) == p.exit_target;
    out = __shfl_sync(0xFFFFFFFFu, out, 0);
    if (out) break;
    __nanosleep(64);
  }
  if (lane == 0) {
    *p.grid_exited = 0;                               // nobody else touches it in this launch
    S->alive = R2_SS(p.seq, 0);                       // posted: the monitor only uses it as a hint
  }
}

// Standalone flavour: no collective resident; serve until the ring is empty
// and no probe is outstanding.
__global__ void r2_service_kernel(SvcBlock* S, MiscDev* m0) {
  __shared__ SvcShared ss;
  const unsigned int lane = threadIdx.x & 31u;
  if (threadIdx.x >= 32) return;
  if (lane == 0) {
    ss.nactive = 0;
    for (int i = 0; i < R2_SVC_MAXPROBES; ++i) ss.pr[i].active = 0;
  }
  __syncwarp();
  for (;;) {
    svc_take(S, m0, ss, lane);
    if (ss.nactive) svc_probes(S, ss, lane);
    int out = 0;
    if (lane == 0) {
      __threadfence();
      out = ss.nactive == 0 && S->head == *(volatile unsigned int*)&m0->svc_tail;
    }
    out = __shfl_sync(0xFFFFFFFFu, out, 0);
    if (out) break;
  }
}

// Worker CTA (participant i, ring-local channel ci, lane w) of ring RI; the
// ring index is a template argument so that every parameter access is a
// constant-bank load at a fixed offset (a run-time ring index made them
// indexed and cost registers: spills in the data path).
template <int RI>
__device__ __forceinline__ void worker_main(const LaunchParams& p, unsigned int b) {
  const int per_rank = p.K * p.W;
  __shared__ Shared sh;
  // the launch parameters in shared memory: every later access goes through
  // Cta::p, a generic pointer, which into the parameter space is a slow
  // generic load -- the control lane reads dozens of fields per chunk
  __shared__ __align__(16) LaunchParams sp;
  {
    static_assert(sizeof(LaunchParams) % 4 == 0, "LaunchParams copy");
    const unsigned int* src = reinterpret_cast<const unsigned int*>(&p);
    unsigned int* dst = reinterpret_cast<unsigned int*>(&sp);
    for (unsigned int i = threadIdx.x; i < sizeof(LaunchParams) / 4; i += blockDim.x) dst[i] = src[i];
  }
  Cta k;
  k.p = &sp;
  k.l = p.part_l[b / per_rank];
  k.c = (int)(b % per_rank) / p.W;
  k.w = (int)(b % per_rank) % p.W;
  k.cg = p.chan[k.c];
  k.cta_in_rank = k.cg * p.W + k.w;                      // control-block record: global channel
  k.r = p.first_rank + k.l;
  k.pos = 0;
  for (int q = 0; q < p.n; ++q)
    if (p.ring[q] == k.r) k.pos = q;
  k.r1 = p.ring[(k.pos + 1) % p.n];
  k.tid = threadIdx.x;
  k.nthr = blockDim.x;
  k.seq = p.seq;
  k.par = (int)(p.seq & 1u);
  if (k.tid < 2) sh.rp[k.tid] = p.peers[k.l * p.ng + (k.tid == 0 ? k.r : k.r1)];
  // per op-step shard tables (the control lane's per-chunk arithmetic without
  // integer divisions; SURVEY §8 header: RS sends shard (pos-1-t) mod n, AG
  // shard (pos-(t-n+1)) mod n, chains one shard)
  for (int t = k.tid; t < p.steps; t += k.nthr) {
    const int n = p.n, ta = t + p.t0;
    const bool chain = p.op == R2_OP_BROADCAST || p.op == R2_OP_R2CC_STAGE2;
    const int s_ = chain ? 0 : (ta <= n - 2) ? ((k.pos - 1 - ta) % n + n) % n : ((k.pos - (ta - n + 1)) % n + n) % n;
    const unsigned long long sb = (unsigned long long)s_ * p.sstride;
    sh.sbase[t] = sb;
    sh.slim[t] = sb + p.slen < p.N ? sb + p.slen : p.N;
  }
  __syncthreads();
  k.me = &sh.rp[0];
  k.nx = &sh.rp[1];
  k.ctrl = p.ctrl[k.l];
  // chain collectives: this rank's position in the chain from the root
  k.t_act = (p.op == R2_OP_BROADCAST || p.op == R2_OP_R2CC_STAGE2) ? ((k.pos - p.root) % p.n + p.n) % p.n : -1;
  k.total_items = p.op == R2_OP_BROADCAST     ? (k.t_act <= p.n - 2 ? (unsigned int)(p.K * p.m) : 0u)
                  : p.op == R2_OP_R2CC_STAGE2 ? (unsigned int)(p.K * p.m)
                                              : (unsigned int)(p.steps * p.K * p.m);
  if (k.tid == 0) TRACE_MIN(k, 0);
  // plan-time placement: read the host's health records for this seq;
  // every CTA of the rank computes the same mask (records for this seq are
  // never rewritten while it runs, see r2_internal.h)
  {
    // all records loaded up front (independent loads in flight together; the
    // short-circuit form issued them one dependent round trip at a time)
    const unsigned int nk = (unsigned int)(p.ng * p.Kg);
    const unsigned int* h = k.me->health;
    const bool std_link = k.r1 == (k.r + 1) % p.ng;       // reading R-10
    unsigned int mask = 0;
#pragma unroll 4
    for (int c = 0; c < p.K; ++c) {
      const unsigned int a = k.r * p.Kg + p.chan[c], b2 = k.r1 * p.Kg + p.chan[c];
      const unsigned int ead = h[R2_H_EP_DEAD * nk + a], ear = h[R2_H_EP_REP * nk + a];
      const unsigned int ebd = h[R2_H_EP_DEAD * nk + b2], ebr = h[R2_H_EP_REP * nk + b2];
      const unsigned int lad = h[R2_H_LINK_DEAD * nk + a], lar = h[R2_H_LINK_REP * nk + a];
      const bool dead = r2_dead_at(ead, ear, k.seq) | r2_dead_at(ebd, ebr, k.seq) |
                        (std_link && r2_dead_at(lad, lar, k.seq));
      if (!dead) mask |= 1u << c;
    }
    k.conn_mask = mask;
  }
  k.own_alive = (k.conn_mask >> k.c) & 1u;
  k.all_healthy = k.conn_mask == (p.K >= 32 ? 0xFFFFFFFFu : ((1u << p.K) - 1u));
  k.own_next_key = 0;
  k.fault_channel = false;
  for (int i = 0; i < p.nfaults; ++i)
    if ((int)p.faults[i].rank == k.r && (int)p.faults[i].channel == k.cg && p.faults[i].kind <= 2 &&
        (int)p.faults[i].origin == k.c)
      k.fault_channel = true;
  if (k.tid == 0) {
    sh.decision = 0;
    sh.cause = 0;
    sh.abort_code = 0;
    sh.pipe_status = 0;
    sh.pub = 0;
    sh.fin = 0;
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&sh.full[s], 1);                          // the control lane's publish
      mbar_init(&sh.empty[s], (k.nthr >> 5) - 1);         // one arrival per data warp
    }
    sh.seen_epoch = 0;
    sh.abandon = 0;
    sh.reissue = 0;
    for (int s2 = 0; s2 < NSLOT; ++s2) sh.slot_ab[s2] = 0;
    sh.dynamic = 0;
    sh.freeze = 0;
    sh.nent = 0;
    sh.alerted = 0;
    sh.recv_next = nullptr;
    sh.first_adopt = 0;
    sh.wait_t0 = 0;
    sh.t_poll = sh.t_prev_poll = 0;
    sh.t_ctl = (unsigned long long)clock64();   // the plan was read just now: first check after the interval
    for (int i = 0; i < 6; ++i) sh.ph[i] = 0;
    sh.pace_next = 0;
    sh.npoll = 0;
    CtaRec& rec = k.ctrl->cta[k.cta_in_rank];
    rec.cause = 0;
    rec.ss = R2_SS(k.seq, CTA_RUNNING);
    if (!p.sim && p.peer_recv && p.ring_id == 0 && k.c == 0 && k.w == 0) {
      // publish our recv (registration id, offset) for the upstream rank(s)
      volatile unsigned long long* d = k.me->desc + k.par * 4;
      d[1] = (unsigned long long)p.recv_reg[k.l];
      d[2] = p.recv_off[k.l];
      fence_sys();
      d[0] = k.seq;
    }
  }
  __syncthreads();
  if (k.tid == 0) TRACE_MAX(k, 1);
  if (p.dtype == R2D_INT32) cta_main<R2D_INT32>(k, sh);
  else if (p.dtype == R2D_FLOAT32) cta_main<R2D_FLOAT32>(k, sh);
  else cta_main<R2D_BF16>(k, sh);
}

// Grid: ring 0's worker CTAs, ring 1's (R²CCL-AllReduce stage 1 only), then
// the service CTA.
__global__ void __launch_bounds__(512, 1) r2_allreduce_kernel(const __grid_constant__ LaunchSet S) {
  unsigned int b = blockIdx.x;
  if (b < (unsigned)S.nctas[0]) {
    worker_main<0>(S.ring[0], b);
    return;
  }
  b -= (unsigned)S.nctas[0];
  if (S.nrings > 1 && b < (unsigned)S.nctas[1]) {
    worker_main<1>(S.ring[1], b);
    return;
  }
  if (threadIdx.x < 32) service_main(S.ring[0]);        // the service CTA (last in the grid)
}

// The single-ring flavour (every launch but R²CCL-AllReduce's stage 1): half
// the parameter block to push per launch (measured on the small-call floor)
__global__ void __launch_bounds__(512, 1) r2_ring_kernel(const __grid_constant__ LaunchParams P, int nctas) {
  if (blockIdx.x < (unsigned)nctas) {
    worker_main<0>(P, blockIdx.x);
    return;
  }
  if (threadIdx.x < 32) service_main(P);
}

// ------------------------------------------------------------ probe kernel
// Zero-byte probe: a flag-only store into the target's per-(prober,
// channel) mailbox over the peer mapping, then a read-back of the same word
// (the completion).  Emulated outcome (reading C-11): LOCAL_ERROR if the
// prober's endpoint is dead; the store is dropped (-> TIMEOUT after the
// timeout) if the target's endpoint or a link between them is dead.
__global__ void r2_probe_kernel(const __grid_constant__ ProbeParams p) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (p.t_start) *p.t_start = gtimer();
  int res;
  const int K = p.K, c = p.channel;
  if (ld_relaxed_sys(p.ep_dead + p.prober * K + c)) {
    res = 1;
  } else {
    bool link = ((p.target == (p.prober + 1) % p.n) && ld_relaxed_sys(p.link_dead + p.prober * K + c)) ||
                ((p.prober == (p.target + 1) % p.n) && ld_relaxed_sys(p.link_dead + p.target * K + c));
    bool dropped = link || ld_relaxed_sys(p.ep_dead + p.target * K + c);
    if (!dropped) {
      st_relaxed_sys(p.target_mailbox, p.token);
      fence_sys();
    }
    res = 2;
    unsigned long long t0 = gtimer();
    while (gtimer() - t0 < p.timeout_ns) {
      if (!dropped && ld_acquire_sys(p.target_mailbox) == p.token) {
        res = 0;
        break;
      }
    }
  }
  *p.result = res;
  __threadfence_system();
}

}  // namespace

int r2_launch_allreduce(const LaunchSet& s, int threads, void* stream) {
  int nctas = 1;                                         // + the service CTA
  for (int i = 0; i < s.nrings; ++i) nctas += s.nctas[i];
  cudaError_t e;
  // (a plain launch instead of the cooperative one measured the same per-call
  // time: the co-residency guarantee costs nothing here)
  if (s.nrings == 1) {
    int nw = s.nctas[0];
    void* args[] = {(void*)&s.ring[0], (void*)&nw};
    e = cudaLaunchCooperativeKernel((const void*)r2_ring_kernel, dim3(nctas), dim3(threads), args, 0,
                                    (cudaStream_t)stream);
  } else {
    void* args[] = {(void*)&s};
    e = cudaLaunchCooperativeKernel((const void*)r2_allreduce_kernel, dim3(nctas), dim3(threads), args, 0,
                                    (cudaStream_t)stream);
  }
  return (int)e;
}

int r2_launch_probe(const ProbeParams& p, void* stream) {
  r2_probe_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

int r2_kernel_smem_bytes() { return (int)sizeof(Shared); }

// Load both kernels at init.  With CUDA 12 lazy module loading, the first
// launch of a not-yet-loaded kernel can wait for the running persistent
// allreduce kernel -- which itself waits for the probe verdict (deadlock
// until the watchdog).  A warm-up launch of the probe kernel (self-probe of a
// healthy mailbox) and an attribute query of the allreduce kernel load them.
int r2_launch_service(SvcBlock* svc, MiscDev* misc0, void* stream) {
  r2_service_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(svc, misc0);
  return (int)cudaGetLastError();
}

int r2_warmup(const ProbeParams& p, void* stream) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, r2_allreduce_kernel);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncGetAttributes(&a, r2_ring_kernel);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncGetAttributes(&a, r2_probe_kernel);
  if (e != cudaSuccess) return (int)e;
  e = cudaFuncGetAttributes(&a, r2_service_kernel);
  if (e != cudaSuccess) return (int)e;
  r2_probe_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return (int)e;
  return (int)cudaStreamSynchronize((cudaStream_t)stream);
}

// Worker CTAs available to one cooperative launch: the service CTA takes one
// more SM; one stays free for the standalone service kernel (no failover step
// depends on it while a collective is resident).
int r2_max_coop_ctas(int threads) {
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int per1 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, r2_allreduce_kernel, threads, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, r2_ring_kernel, threads, 0);
  return (nsm - 2) * std::min(per, per1);
}
