/*
 * r2ccl.h -- C ABI of the B200-native R²CCL hot path (arXiv 2512.25059).
 *
 * A fault-tolerant, chunked, multi-channel ring allreduce over NVLink 5 /
 * NVSwitch peer mappings, one process per GPU (or k simulated ranks on one
 * GPU).  Citations: P:n = reference PAPER.md line n, S:n = SPEC.md line n.
 *
 * The paper's statement of the problem: a drop-in collective
 * library; communicators come from a one-time bootstrap; a failure
 * during a collective must not crash the process but be intercepted and
 * survived transparently.
 *
 * Conventions (all entry points):
 *   - Return codes, never abort: every call returns an r2_result_t.
 *   - Plain pointers and sizes only.  Device pointers are CUDA device
 *     addresses of the caller's GPU; "stream" is a cudaStream_t passed as
 *     void* (NULL = legacy default stream).
 *   - Ownership: the caller owns send/recv buffers and streams; the library
 *     owns its scratch, flags, mailboxes, IPC mappings, host-mapped control
 *     blocks and its monitor thread (released by r2_finalize).
 *   - Threading: one host thread per communicator issues calls (like NCCL);
 *     only r2_status / r2_get_event may be called concurrently.
 *   - "collective": every rank of the communicator must make the same call
 *     in the same order.
 */
#ifndef R2CCL_H
#define R2CCL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define R2_MAX_CHANNELS 16   /* K upper bound                                   */
#define R2_MAX_LOCAL 16      /* simulated ranks per process upper bound         */
#define R2_MAX_RANKS 64      /* ranks of a communicator upper bound             */

typedef enum {
  R2_SUCCESS = 0,
  R2_ERR_INVALID_ARG = 1,    /* bad pointer / size / config / alignment          */
  R2_ERR_CUDA = 2,           /* a CUDA runtime call failed                       */
  R2_ERR_BOOTSTRAP = 3,      /* out-of-band bootstrap failed                     */
  R2_ERR_NOT_REGISTERED = 4, /* recv not inside an r2_register_multi range       */
  R2_ERR_NO_BACKUP = 5,      /* failover chain exhausted                 */
  R2_ERR_TIMEOUT = 6,        /* watchdog expired (reading C-13)                  */
  R2_ERR_INTERNAL = 7
} r2_result_t;

typedef enum { R2_INT32 = 0, R2_FLOAT32 = 1, R2_BFLOAT16 = 2 } r2_dtype_t;

/* Collectives on the ring (SURVEY §8(f) f1 for the standalone halves). */
typedef enum { R2_OP_ALLREDUCE = 0, R2_OP_REDUCE_SCATTER = 1, R2_OP_ALL_GATHER = 2, R2_OP_BROADCAST = 3,
               R2_OP_R2CC_STAGE2 = 4  /* internal: R²CCL-AllReduce stage 2 (tailored broadcast, reading R-9) */
} r2_op_t;

/* Single-failure strategies (P:57 HotRepair; P:73 R²CCL-Balance). */
typedef enum { R2_HOT_REPAIR = 0, R2_BALANCE = 1 } r2_strategy_t;

/* Emulated fault kinds (App. C; SURVEY reading C-14). */
typedef enum {
  R2_FAULT_LOCAL = 0,   /* sender endpoint (src_rank, channel) dies           */
  R2_FAULT_REMOTE = 1,  /* receiver endpoint (src_rank+1, channel) dies       */
  R2_FAULT_LINK = 2,    /* ring link src_rank -> src_rank+1 on channel dies   */
  R2_FAULT_REPAIR = 3,  /* re-admit (src_rank, channel): stand-in for the
                           periodic re-probe of P:19 / S:345                  */
  R2_FAULT_HEAL = 4     /* the emulated endpoint (src_rank, channel) and link
                           src_rank -> src_rank+1 recover before at_seq; the
                           library learns it only by re-probing (f4)    */
} r2_fault_kind_t;

/* Probe outcomes and verdicts (reading C-10). */
typedef enum { R2_PROBE_SUCCESS = 0, R2_PROBE_LOCAL_ERROR = 1, R2_PROBE_TIMEOUT = 2,
               R2_PROBE_NOT_RUN = 3 } r2_probe_outcome_t;
typedef enum {
  R2_V_NONE = 0, R2_V_LOCAL_ENDPOINT = 1, R2_V_REMOTE_ENDPOINT = 2, R2_V_LINK = 3,
  R2_V_ENDPOINT_UNREACHABLE_A = 4, R2_V_ENDPOINT_UNREACHABLE_B = 5,
  R2_V_DUAL_ENDPOINT = 6, R2_V_TWO_LOCAL = 7, R2_V_INCONCLUSIVE = 8
} r2_verdict_kind_t;

typedef struct r2_comm* r2_comm_t;

/*
 * Out-of-band transport ("a separate bootstrap network").  A
 * vtable so that the library is independent of the launcher.  All functions
 * return 0 on success.  allgather/barrier are collective and blocking;
 * post is non-blocking (msg <= 256 bytes); poll is non-blocking and returns 1
 * when a message was received (src, len filled), 0 when none.
 * r2_oob_shm_open below provides a POSIX shared-memory implementation for
 * ranks of one node.
 */
typedef struct {
  void* ctx;
  int (*allgather)(void* ctx, const void* sendbuf, void* recvbuf, size_t bytes);
  int (*post)(void* ctx, int dst, const void* msg, size_t len);
  int (*poll)(void* ctx, int* src, void* msg, size_t cap, size_t* len);
  int (*barrier)(void* ctx);
} r2_oob_t;

/*
 * Configuration.  r2_config_default fills the defaults listed here.
 *   nchannels         K channels (default 8, mirrors 8 NICs/server)
 *   ctas_per_channel  W CTAs per channel (default 4)
 *   threads_per_cta   512
 *   chunk_bytes       per (connection, step) chunk, multiple of 16 (512 KiB;
 *                     reading C-3)
 *   max_bytes         largest allreduce payload per rank (scratch sizing;
 *                     default 1 GiB)
 *   strategy          R2_BALANCE
 *   probe_timeout_us  50 (reading C-13)
 *   watchdog_ms       3000: a kernel waiting longer aborts with R2_ERR_TIMEOUT
 *   channel_w         K integer weights (NULL = equal) for Balance
 *   sim_ranks         world == 1 only: k >= 1 simulated ranks on one GPU
 *                     (send/recv then hold k rank buffers back to back)
 *   protocol          R2_PROTO_AUTO (default): per call, the alpha-beta model
 *                     below picks SIMPLE, LL or LL128;
 *                     R2_PROTO_SIMPLE / R2_PROTO_LL / R2_PROTO_LL128 force one
 *                     (a forced LL/LL128 call whose payload exceeds the line
 *                     scratch returns R2_ERR_INVALID_ARG)
 *   ll_max_bytes      largest per-rank payload the LL / LL128 protocols may
 *                     carry (sizes their shared line scratch: 4 x payload per
 *                     rank; default 128 MiB, 0 disables both)
 *   reprobe_us        first re-probe of a dead connection after this many
 *                     microseconds, then exponential back-off ("adapting
 *                     probe frequency"); default 2000, 0 disables re-probing
 *   reprobe_max_us    back-off cap (default 200000)
 *   channel_gbps      bandwidth model of a channel (0 = off, the default): every
 *                     lane paces its sends to channel_gbps / W, so a channel is
 *                     a bandwidth unit like the paper's NIC (reading C-1: without
 *                     it channels share the GPU's NVLink ports and a dead channel
 *                     only removes CTAs)
 *   rerank            1 (default): before every ring AllReduce the planner
 *                     applies Algorithm 1 (App. D, §6; r2_rerank) to the
 *                     health records of that seq -- rails S_u = channels alive
 *                     on rank u; a neighbour pair with no live link left has
 *                     capacity 0 (reading R-13) -- and runs the collective on the
 *                     re-ranked ring R' (AllReduce only: its result does not
 *                     depend on which rank owns which shard); 0 keeps rank order
 *   r2cc_stage1_eff_pct, r2cc_stage2_eff_pct
 *                     the AUTO algorithm choice divides R²CCL-AllReduce's stage
 *                     bandwidth terms by these measured efficiencies
 *                     (defaults 75 / 50: stage 1 0.79 ms vs 0.59 modelled, the
 *                     tailored broadcast 0.89 vs 0.44; reading R-11); 100 / 100
 *                     is the paper's model as written
 *   alpha_simple_ns, alpha_ll_ns, alpha_ll128_ns, beta_mbps
 *                     cost model: T = (#ring steps) * alpha + (wire bytes per
 *                     rank) / beta, LL moving twice the bytes and LL128 8/7 of
 *                     them (defaults from profiles/r01_pingpong.log,
 *                     r01_sizes_n4.jsonl and the round-2 protocol sweeps)
 *
 * Protocols.  SIMPLE: 16-byte vectors straight into the peer's memory, one
 * fence.acq_rel.sys per retired batch, then the completion word (P:33's
 * work completion).  LL ("low latency", latency-bound sizes): every 16-byte
 * vector travels as two 16-byte lines {w0, seq, w1, seq}, {w2, seq, w3, seq}
 * into library scratch, self-validating at the receiver, so the completion
 * word needs no fence; the receiver unpacks the last all-gather step locally
 * (reading R-6).  LL128 (mid sizes, reading R-12): a chunk travels as
 * 128-byte lines of 7 payload vectors + 1 flag vector {seq x 4}, each line
 * written by one warp store instruction and accepted by the receiver when its
 * flag vector equals seq: 8/7 of the bytes and no fence per step.  All three
 * keep the per-chunk completion words, rollback and re-placement unchanged.
 */
typedef struct {
  int nchannels;
  int ctas_per_channel;
  int threads_per_cta;
  size_t chunk_bytes;
  size_t max_bytes;
  int strategy;
  int probe_timeout_us;
  int watchdog_ms;
  int channel_w[R2_MAX_CHANNELS];
  int use_channel_w;
  int sim_ranks;
  int protocol;
  size_t ll_max_bytes;
  int alpha_simple_ns, alpha_ll_ns;
  int beta_mbps;
  int reprobe_us, reprobe_max_us;
  int channel_gbps;
  int allreduce_algo;   /* r2_algo_t (default AUTO)                                  */
  int alpha_launch_ns;  /* cost model: one more collective launch (R²CCL stage 2)    */
  int alpha_ll128_ns;   /* cost model: per ring step under LL128                     */
  int rerank;           /* 1 (default): ring AllReduce on Algorithm 1's re-ranked ring */
  int r2cc_stage1_eff_pct, r2cc_stage2_eff_pct;  /* cost model: measured efficiency of
                           R²CCL-AllReduce's stages vs their bandwidth terms (75, 50) */
} r2_config_t;

/*
 * AllReduce algorithm under a degraded rank (P:106-136,
 * App. A).  RING: always the ring (Balance / HotRepair re-placement
 * of the dead channels).  R2CC: R²CCL-AllReduce whenever it applies -- exactly
 * one rank f has dead channel endpoints (no dead link), n >= 3, and App. A's
 * planner gives Y > 0 (lost fraction X > n/(3n-2)): stage 1 runs the global
 * ring on f's healthy channels over the first (1-Y) of the buffer concurrently
 * with a partial ring over the n-1 healthy ranks on f's dead channels over the
 * rest; stage 2 (a second launch, its own seq) is the tailored broadcast f ->
 * f+1 (adds f's contribution) -> ... -> f-1 -> f (reading R-9).  AUTO: the
 * alpha-beta cost model picks the faster of the two per call (reading R-11).
 * A call that runs R²CCL-AllReduce enqueues two collectives (two seqs).
 */
typedef enum { R2_ALGO_AUTO = 0, R2_ALGO_RING = 1, R2_ALGO_R2CC = 2 } r2_algo_t;

typedef enum { R2_PROTO_AUTO = 0, R2_PROTO_SIMPLE = 1, R2_PROTO_LL = 2, R2_PROTO_LL128 = 3 } r2_protocol_t;

/*
 * An injected channel fault.  Fires in collective number
 * at_seq (1 = first r2_allreduce of the communicator) when channel `channel`
 * of sender `src_rank` starts the item (step, chunk) of origin channel
 * `origin_channel` (-1 = its own items): the first byte_offset bytes of that
 * item's part reach the peer (rounded down to 16 bytes), no completion flag
 * is written (reading C-6), the transport is dead from then on
 * (every later item of that channel, in (step, origin, chunk) order, is
 * undelivered).  The sender's error becomes visible after detect_delay_us.
 * poison: fill the rest of the faulted item at the peer with 0xFF.
 * REPAIR: before collective at_seq, the endpoint/link is healthy again.
 */
typedef struct {
  uint64_t at_seq;
  int src_rank;
  int channel;
  int origin_channel;
  int kind;          /* r2_fault_kind_t */
  int step;
  int chunk;
  uint64_t byte_offset;
  int detect_delay_us;
  int poison;
} r2_fault_t;

typedef struct {
  int kind;          /* r2_verdict_kind_t */
  int a, b, aux;     /* endpoint ranks A (detector), B (its peer), aux (-1 none) */
  int channel;
  int outcome[4];    /* A->B, B->A, aux->A, aux->B (r2_probe_outcome_t)      */
} r2_verdict_t;

/* One failover record: a re-planned origin channel of one sender rank. */
typedef struct {
  uint64_t seq;
  int rank;               /* sender rank of the connection                    */
  int origin_channel;     /* whose items were rolled back / re-placed          */
  int stopped_channel;    /* the stopped channel that triggered it             */
  r2_verdict_t verdict;
  int resume;             /* first stream position without completion  */
  int floor;              /* last contiguously confirmed position             */
  int retransmit;         /* items re-placed (exactly those w/o completion)   */
  int strategy;
  int assignee;           /* HOT_REPAIR: adopting channel; -1 otherwise       */
  int chain_pos;          /* its position in the failover chain        */
  int shares[R2_MAX_CHANNELS]; /* BALANCE: 16-B vectors of a full chunk/channel */
  int error;              /* R2_SUCCESS or R2_ERR_NO_BACKUP                   */
  /* timing: device %globaltimer ns on the sender's GPU, host CLOCK_MONOTONIC ns */
  uint64_t t_fire_dev_ns, t_first_retx_dev_ns;
  uint64_t t_detect_host_ns, t_verdict_host_ns, t_plan_host_ns;
  double failover_ms;     /* t_first_retx_dev - t_fire_dev (-1 if unknown)     */
  /* bilateral notification ("notifies both sides to avoid
     half-open states"): the detector's NOTIFY and the acknowledgements of
     every rank (the other endpoint included); filled in on the detecting
     rank's record once the acknowledgements arrive                          */
  int notify_acks;        /* acknowledgements received (expected: world)      */
  int notify_peer_acked;  /* the connection's other endpoint acknowledged     */
  double notify_ack_ms;   /* NOTIFY sent -> last acknowledgement (-1 pending) */
} r2_event_t;

typedef struct {
  uint64_t seq;               /* collectives enqueued so far                       */
  int last_error;             /* most recent asynchronous error (r2_result_t)     */
  uint64_t last_error_seq;
  int n_events;
  int world, nlocal, nchannels;
  uint32_t dead_endpoints[R2_MAX_LOCAL * 4]; /* bit c of word r: endpoint (r,c) */
  uint32_t dead_links[R2_MAX_LOCAL * 4];     /* bit c of word r: link r->r+1    */
  uint64_t bytes[R2_MAX_LOCAL][R2_MAX_CHANNELS]; /* bytes pushed per local rank/channel */
  int last_protocol;          /* r2_protocol_t the last enqueued collective used  */
  int n_readmits;             /* connections re-admitted after a successful re-probe */
  int n_reprobes;             /* re-probe rounds run                              */
  int n_service_kernels;      /* standalone service-kernel launches (monitor work
                                 with no collective resident to serve it)         */
  /* R²CCL-AllReduce (f2): calls that ran it, and the planner's choice for the
     last one (degraded rank f, lost fraction X, partial share Y = App. A's
     optimal partition, element split N_A + N_P, the seq of its stage 2)        */
  int n_r2cc;
  int r2cc_rank;
  double r2cc_X, r2cc_Y;
  uint64_t r2cc_NA, r2cc_NP, r2cc_seq;
  /* Re-ranking (f4, Algorithm 1): AllReduce calls that ran on a re-ranked
     ring, and the ring order of the last ring AllReduce (ranks by position) */
  int n_rerank;
  int ring_order[R2_MAX_RANKS];
} r2_status_t;

/* Fill *cfg with the defaults documented above. */
void r2_config_default(r2_config_t* cfg);

/*
 * r2_init -- collective.  One-time bootstrap + multi-registration
 * (P:25-27): allocates this rank's scratch (2(n-1)/n * max_bytes),
 * per-chunk flag words, part counters, emulated link state and probe
 * mailboxes, exports them over CUDA IPC and maps EVERY peer's (not only the
 * ring neighbours'), so that no mapping is created on the recovery path.
 * Starts the monitor thread.  rank in [0, world); cuda_dev = device ordinal.
 * world == 1 with cfg->sim_ranks = k runs k simulated ranks (oob may be NULL).
 * Errors: INVALID_ARG, CUDA, BOOTSTRAP.  *out is NULL on error.
 */
r2_result_t r2_init(int rank, int world, int cuda_dev, const r2_oob_t* oob,
                    const r2_config_t* cfg, r2_comm_t* out);

/*
 * r2_register_multi -- collective.  Registers the allocation that contains
 * [dptr, dptr+bytes) with every peer (IPC export + open on all ranks,
 * P:27 "registering each GPU buffer with multiple NICs at initialization").
 * recv buffers of r2_allreduce must lie in a registered range; send buffers
 * need not.  *reg_out receives an id (same on all ranks).
 * Errors: INVALID_ARG (NULL / not a device pointer), CUDA, BOOTSTRAP.
 */
r2_result_t r2_register_multi(r2_comm_t comm, void* dptr, size_t bytes, uint64_t* reg_out);

/* r2_deregister -- collective.  Unmaps a registration on every rank (the
 * inverse of r2_register_multi's multi-NIC registration, P:27 / P:741; SPEC
 * register_multi S:225-233).  reg: the id r2_register_multi returned.  Errors:
 * R2_ERR_NOT_REGISTERED for an unknown id, R2_ERR_BOOTSTRAP if the OOB fails. */
r2_result_t r2_deregister(r2_comm_t comm, uint64_t reg);

/*
 * r2_allreduce -- collective, asynchronous on `stream`.  Sum-allreduce of
 * `count` elements (P:94 ring ReduceScatter + AllGather).  send == recv
 * (in-place) is allowed.  Both pointers 16-byte aligned.  count == 0 is a
 * no-op; count * elem size <= cfg.max_bytes.  In sim mode (k ranks) send and
 * recv each hold k rank buffers of count elements, rank l's starting at byte
 * l * roundup(count * elem size, 16), and need no registration.  Result (reading C-8): for element i of shard s,
 * y[i] = fold(x_{s+1}[i], ..., x_{s+n-1}[i], x_s[i]) with per-hop rounding
 * (int32 wraps, fp32 RN, bf16 = RNE(fp32 add)); bit-identical with and without
 * faults.  A channel fault mid-collective is recovered inside the call's
 * stream work; the stream is released only when the result is complete.  An
 * unrecoverable failure (NO_BACKUP, TIMEOUT) still releases the stream (result
 * undefined) and is reported by the next r2_* call and r2_status.last_error.
 * Errors: INVALID_ARG, NOT_REGISTERED, CUDA, and pending async errors.
 */
r2_result_t r2_allreduce(r2_comm_t comm, const void* send, void* recv, size_t count,
                         r2_dtype_t dt, void* stream);

/*
 * r2_reduce_scatter -- collective, asynchronous ("a
 * ReduceScatter retains only a 1/n shard"; P:353/572 Balance on RS).  send
 * holds n * recvcount elements (shard s at element s * recvcount); rank r's
 * recv receives recvcount elements: shard r reduced with the AllReduce's
 * ring fold, fold(x_{r+1}, ..., x_{r-1}, x_r) per element, per-hop rounding as
 * r2_allreduce.  In-place: recv == send + r * recvcount.  recv needs no
 * registration (peers write only into library scratch).  Same fault handling
 * (rollback, failover chain / Balance; the owner's final add is a LOCAL item
 * that uses no connection, reading R-5).  Sim mode: send rows of n * recvcount
 * elements and recv rows of recvcount elements, each row 16-byte aligned.
 * Errors: as r2_allreduce.
 */
r2_result_t r2_reduce_scatter(r2_comm_t comm, const void* send, void* recv, size_t recvcount,
                              r2_dtype_t dt, void* stream);

/*
 * r2_all_gather -- collective, asynchronous (f1; "an AllGather must
 * receive the same amount").  send holds sendcount elements; every rank's
 * recv receives n * sendcount elements, rank s's input at element
 * s * sendcount (bits preserved).  In-place: send == recv + r * sendcount.
 * recv must lie in a registered range (peers write into it).  Sim mode: send
 * rows of sendcount and recv rows of n * sendcount elements, 16-byte aligned.
 * Errors: as r2_allreduce.
 */
r2_result_t r2_all_gather(r2_comm_t comm, const void* send, void* recv, size_t sendcount,
                          r2_dtype_t dt, void* stream);

/*
 * r2_broadcast -- collective, asynchronous (f1; "in a Broadcast, the
 * root sends D_total while all others receive it").  The root's send (count
 * elements) arrives in every rank's recv, bits preserved, over a pipelined
 * chain root -> root+1 -> ... along the ring (reading R-8); send is read on the
 * root only (may be NULL elsewhere); in-place on the root: send == recv.  recv
 * must lie in a registered range.  Same fault handling (rollback, failover
 * chain / Balance).  Always the SIMPLE protocol.  Sim mode: send / recv rows of
 * count elements, 16-byte aligned.  Errors: as r2_allreduce; root out of range.
 */
r2_result_t r2_broadcast(r2_comm_t comm, const void* send, void* recv, size_t count, r2_dtype_t dt, int root,
                         void* stream);

/*
 * r2_allreduce_host -- as r2_allreduce, but send/recv are HOST buffers (pinned
 * memory recommended).  Copies into a library-owned registered device buffer,
 * allreduces, copies back; the caller synchronizes `stream` before reading
 * recv.  From 8 MiB on the payload is cut into up to 8
 * segments, each its own collective, whose H2D copy, allreduce and D2H copy
 * overlap the neighbouring segments' (two library copy streams, ordered with
 * `stream` by events).  The result is that of r2_allreduce applied to each
 * segment (the fold order follows the segment's shards): segment size
 * ceil(count / nseg) rounded down to a 16-byte multiple plus one vector,
 * nseg = min(8, bytes / 4 MiB).
 */
r2_result_t r2_allreduce_host(r2_comm_t comm, const void* send, void* recv, size_t count,
                              r2_dtype_t dt, void* stream);

/*
 * r2_inject_fault -- collective (same descriptor on all ranks, before the
 * targeted seq; like SPEC's scenario fault list S:362).  Arms an emulated
 * channel fault (NVLink faults cannot be injected on a live box).
 * Errors: INVALID_ARG.
 */
r2_result_t r2_inject_fault(r2_comm_t comm, const r2_fault_t* f);

/*
 * r2_probe -- one three-point triangulation round for connection
 * (rank -> peer, channel) started by this rank: zero-byte probe-flag kernels
 * A->B, B->A, aux->A, aux->B (aux = lowest rank not in {A,B}, reading C-12),
 * outcome per reading C-11, verdict per reading C-10.  Peer and aux answer
 * through their monitor threads (no call needed on their side).  Blocks
 * until the verdict.  In sim mode `rank_local` selects the simulated prober.
 */
r2_result_t r2_probe(r2_comm_t comm, int rank_local, int peer, int channel, r2_verdict_t* out);

/* r2_status -- thread-safe snapshot (waits for nothing): the observable
 * state of the method -- health records ("inspects the health status
 * records"), failover records (P:31-36 rollback, P:27 chain, P:73 Balance),
 * per-channel bytes, protocol / R²CCL / ring-order choices -- the
 * counterpart of SPEC's Report.  *out is caller-owned; fields
 * are a consistent snapshot under the communicator's lock. */
r2_result_t r2_status(r2_comm_t comm, r2_status_t* out);

/* r2_get_event -- idx-th failover record (0 <= idx < n_events). */
r2_result_t r2_get_event(r2_comm_t comm, int idx, r2_event_t* out);

/*
 * r2_sync -- synchronize the last stream used by r2_allreduce and return the
 * async error of the collectives completed since the previous r2_sync.
 */
r2_result_t r2_sync(r2_comm_t comm);

/*
 * r2_trace -- diagnostics.  Returns the device-clock (%globaltimer, ns)
 * timeline of the collectives launched since the previous r2_trace call on
 * local rank `rank_local` (64 slots: first CTA start, per-step first publish
 * and last retire, control end, drain end, exit; 0 / ~0 = not reached) and
 * re-arms it.  Recording is enabled by the environment variable R2_TRACE=1 at
 * r2_init; otherwise INVALID_ARG.  Synchronizes the device.
 */
r2_result_t r2_trace(r2_comm_t comm, int rank_local, uint64_t out[64]);

/* r2_finalize -- collective.  Stops the monitor, unmaps peers, frees all
 * (the end of the communicator the bootstrap of P:657 created).  Must not be
 * called with a collective of this communicator in flight on any stream
 * (synchronise first); after it, comm is invalid.  Errors: R2_ERR_CUDA if a
 * device resource cannot be released (the rest is still freed). */
r2_result_t r2_finalize(r2_comm_t comm);

const char* r2_strerror(r2_result_t r);

/* ------------------------------------------------------------------------
 * Host logic, exposed for parity tests (no GPU needed).
 * ---------------------------------------------------------------------- */

/* Decision table C-10.  outcome[2..3] ignored if !has_aux. */
int r2_triangulate(const int outcome[4], int has_aux);

/* Balance shares (reading C-15): floor(R*w_c/Σw) over
 * channels whose bit is set in healthy_mask, remainder to the largest weight
 * (ties: lowest id).  shares_out[K].  Returns R2_ERR_NO_BACKUP if mask empty. */
r2_result_t r2_balance_shares(uint64_t R, const int* w, uint32_t healthy_mask, int K,
                              uint64_t* shares_out);

/* Failover chain of channel c (reading C-2): c+1, ..., c+K-1 mod K. */
void r2_failover_chain(int c, int K, int* out);

/* Rollback on a completion ledger. */
void r2_rollback(const uint8_t* completed, int npos, int* resume, int* floor);

/* Topology-aware logical re-ranking: Algorithm 1 (App. D, §6
 * P:726 "pairs of neighbors whose rail overlap falls below a bandwidth
 * threshold are separated by inserting 'bridge' nodes").  ring_in[0..n): the
 * ring order (a permutation of ranks 0..n-1); rails[u]: bitmask of the
 * channels whose endpoint on rank u is alive (the rail set S_u, reading
 * C-1); dead_links[u] (may be NULL): channels whose standard link u -> u+1
 * mod n is dead (reading R-13: an edge whose links are dead on every common
 * channel has capacity 0, else |S_u ∩ S_v|).  Writes
 * R' to ring_out[0..n) (caller-owned).  Returns the number of relocations,
 * or -1 on invalid arguments (n outside 1..R2_MAX_RANKS, NULL pointers). */
int r2_rerank(int n, const int* ring_in, const uint32_t* rails, const uint32_t* dead_links, int* ring_out);

/* Geometry of one collective (SURVEY §8 header, reading C-3).
 * Chunk = chunk_bytes, capped at ceil(slice bytes / W) rounded up to 16
 * bytes: every one of a channel's W lanes gets a chunk per ring step.
 * AllReduce: N = count, shards of Np/n at stride shard.
 * Broadcast (f1): N = count, one shard of roundup(count, K*V) = Np, steps
 * n-1 (rank r sends only at its chain position (r - root) mod n), chunks
 * capped at 128 KiB.
 * ReduceScatter / AllGather (f1): N = n * count (the n-shard user buffer),
 * shard = roundup(count, K*V) (the channel split), stride = count (shard
 * distance in the user buffers); steps n (RS: t = n-1 is the owner's LOCAL
 * final add, local_step = n-1) / n-1 (AG: op-step t is AllReduce step
 * t + t0, t0 = n-1). */
typedef struct {
  uint64_t N, Np, shard, slice, chunk; /* elements */
  int n, K, W, V, m, steps;
  uint64_t stride;                     /* elements between shards in the user buffers */
  int t0, local_step;                  /* AllReduce step of op-step 0; LOCAL step or -1 */
} r2_geometry_t;
r2_result_t r2_geometry(uint64_t count, r2_dtype_t dt, int n, int K, int W,
                        size_t chunk_bytes, r2_geometry_t* out);
r2_result_t r2_geometry_op(r2_op_t op, uint64_t count, r2_dtype_t dt, int n, int K, int W,
                           size_t chunk_bytes, r2_geometry_t* out);

/* POSIX shared-memory OOB for ranks of one node.  `name` must be identical
 * on all ranks and unique per communicator (e.g. from the launcher's store).
 * Rank 0 creates the segment; others attach (waits up to 60 s). */
r2_result_t r2_oob_shm_open(const char* name, int rank, int world, r2_oob_t* out);
r2_result_t r2_oob_shm_close(r2_oob_t* oob);

#ifdef __cplusplus
}
#endif
#endif /* R2CCL_H */
