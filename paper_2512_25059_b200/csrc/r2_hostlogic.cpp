// r2_hostlogic.cpp -- pure host logic of the R²CCL control plane.
//   r2_triangulate      decision table C-10
//   r2_balance_shares   R²CCL-Balance integer shares (C-15)
//   r2_failover_chain   ordered backups (C-2)
//   r2_rollback         sender resume / receiver floor
//   r2_geometry         shards / slices / chunks (SURVEY §8 header, C-3)
//   r2_rerank           bridge-based logical re-ranking (Algorithm 1; C-19, R-13)
#include <string.h>

#include <algorithm>

#include "r2_comm.h"

extern "C" int r2_triangulate(const int o[4], int has_aux) {
  const int S = R2_PROBE_SUCCESS, L = R2_PROBE_LOCAL_ERROR, T = R2_PROBE_TIMEOUT;
  const int ab = o[0], ba = o[1];
  if (ab == L && ba == L) return R2_V_TWO_LOCAL;
  if (ab == L) return R2_V_LOCAL_ENDPOINT;
  if (ba == L) return R2_V_REMOTE_ENDPOINT;
  if (ab == S && ba == S) return R2_V_NONE;
  if ((ab == T && ba == S) || (ab == S && ba == T)) return R2_V_LINK;
  // both endpoints timed out
  if (!has_aux) return R2_V_INCONCLUSIVE;
  const int xa = o[2], xb = o[3];
  if (xa == L || xb == L) return R2_V_INCONCLUSIVE;
  if (xa == S && xb == S) return R2_V_LINK;
  if (xa == T && xb == S) return R2_V_ENDPOINT_UNREACHABLE_A;
  if (xa == S && xb == T) return R2_V_ENDPOINT_UNREACHABLE_B;
  return R2_V_DUAL_ENDPOINT;
}

extern "C" r2_result_t r2_balance_shares(uint64_t R, const int* w, uint32_t mask, int K, uint64_t* out) {
  if (!w || !out || K <= 0 || K > R2_MAX_CHANNELS) return R2_ERR_INVALID_ARG;
  uint64_t tot = 0;
  int top = -1;
  for (int k = 0; k < K; ++k) {
    out[k] = 0;
    if ((mask >> k & 1u) && w[k] > 0) {
      tot += (uint64_t)w[k];
      if (top < 0 || w[k] > w[top]) top = k;
    }
  }
  if (tot == 0) return R2_ERR_NO_BACKUP;
  uint64_t sum = 0;
  for (int k = 0; k < K; ++k)
    if ((mask >> k & 1u) && w[k] > 0) {
      out[k] = (uint64_t)((unsigned __int128)R * (uint64_t)w[k] / tot);
      sum += out[k];
    }
  out[top] += R - sum;
  return R2_SUCCESS;
}

extern "C" void r2_failover_chain(int c, int K, int* out) {
  for (int d = 1; d < K; ++d) out[d - 1] = (c + d) % K;
}

extern "C" void r2_rollback(const uint8_t* completed, int npos, int* resume, int* floor) {
  int r = npos;
  for (int q = 0; q < npos; ++q)
    if (!completed[q]) {
      r = q;
      break;
    }
  if (resume) *resume = r;
  if (floor) *floor = r - 1;
}

static int elem_bytes_of(r2_dtype_t dt) { return dt == R2_BFLOAT16 ? 2 : 4; }

extern "C" r2_result_t r2_geometry(uint64_t count, r2_dtype_t dt, int n, int K, int W, size_t chunk_bytes,
                                   r2_geometry_t* g) {
  return r2_geometry_op(R2_OP_ALLREDUCE, count, dt, n, K, W, chunk_bytes, g);
}

extern "C" r2_result_t r2_geometry_op(r2_op_t op, uint64_t count, r2_dtype_t dt, int n, int K, int W,
                                      size_t chunk_bytes, r2_geometry_t* g) {
  if (!g || n < 1 || K < 1 || W < 1 || chunk_bytes < 16 || chunk_bytes % 16) return R2_ERR_INVALID_ARG;
  if (dt != R2_INT32 && dt != R2_FLOAT32 && dt != R2_BFLOAT16) return R2_ERR_INVALID_ARG;
  if (op != R2_OP_ALLREDUCE && op != R2_OP_REDUCE_SCATTER && op != R2_OP_ALL_GATHER && op != R2_OP_BROADCAST &&
      op != R2_OP_R2CC_STAGE2)
    return R2_ERR_INVALID_ARG;
  const bool chain = op == R2_OP_BROADCAST || op == R2_OP_R2CC_STAGE2;   // one shard: the whole buffer
  const int E = elem_bytes_of(dt), V = 16 / E;
  const uint64_t Nmin = count ? count : 1;
  uint64_t Np_cap;
  if (op == R2_OP_ALLREDUCE) {
    const uint64_t q = (uint64_t)n * K * V;
    Np_cap = (Nmin + q - 1) / q * q;
  } else if (chain) {
    const uint64_t q = (uint64_t)K * V;              // one shard: the whole buffer
    Np_cap = (Nmin + q - 1) / q * q;
  } else {
    const uint64_t q = (uint64_t)K * V;              // each shard padded for the channel split
    Np_cap = (uint64_t)n * ((Nmin + q - 1) / q * q);
  }
  const uint64_t slice = Np_cap / ((uint64_t)(chain ? 1 : n) * K);
  const uint64_t slice_bytes = slice * E;
  // reading C-3: capped at ceil(slice / W) -- one chunk per lane per step.
  // (Four chunks per lane per step, to pipeline across ring steps, was
  // measured slower at 4-64 MiB: the control lane's per-chunk cost (~1.7 us
  // per publish) outweighs the overlap -- profiles/r02_lane_chunks.txt)
  uint64_t per_worker = ((slice_bytes + W - 1) / W + 15) / 16 * 16;
  // a Broadcast chain pipelines per chunk (fill = (n-2) chunk hops): 128 KiB cap (reading R-8)
  const uint64_t cap = chain && chunk_bytes > (128u << 10) ? (128u << 10) : chunk_bytes;
  uint64_t chunkb = cap < per_worker ? cap : per_worker;
  if (chunkb < 16) chunkb = 16;
  memset(g, 0, sizeof(*g));
  g->N = (op == R2_OP_ALLREDUCE || chain) ? count : (uint64_t)n * count;
  g->Np = count ? Np_cap : 0;
  g->shard = chain ? g->Np : g->Np / n;
  g->stride = (op == R2_OP_ALLREDUCE || chain) ? g->shard : count;
  g->t0 = op == R2_OP_ALL_GATHER ? n - 1 : 0;
  g->local_step = op == R2_OP_REDUCE_SCATTER ? n - 1 : -1;
  g->slice = count ? slice : 0;
  g->chunk = chunkb / E;
  g->n = n;
  g->K = K;
  g->W = W;
  g->V = V;
  g->m = count ? (int)((g->slice + g->chunk - 1) / g->chunk) : 0;
  // AG, BCAST: n-1; R²CCL stage 2: n (the chain returns to the degraded rank, reading R-9)
  g->steps = op == R2_OP_ALLREDUCE ? 2 * n - 2
             : op == R2_OP_REDUCE_SCATTER ? n
             : op == R2_OP_R2CC_STAGE2 ? n
                                       : n - 1;
  return R2_SUCCESS;
}

int r2_first_healthy_in_chain(int origin, uint32_t mask, int K) {
  for (int d = 1; d < K; ++d) {
    int c = (origin + d) % K;
    if (mask >> c & 1u) return c;
  }
  return -1;
}

// ---- seq-indexed health records (the planner's "health status records")
static inline const uint32_t* hrow(const r2_comm* c, int which) {
  return c->health.data() + (size_t)which * c->n * c->K;
}

bool r2_ep_dead_at(const r2_comm* c, int r, int k, uint32_t q) {
  const int i = r * c->K + k;
  return r2_dead_at(hrow(c, R2_H_EP_DEAD)[i], hrow(c, R2_H_EP_REP)[i], q);
}

bool r2_link_dead_at(const r2_comm* c, int r, int k, uint32_t q) {
  const int i = r * c->K + k;
  return r2_dead_at(hrow(c, R2_H_LINK_DEAD)[i], hrow(c, R2_H_LINK_REP)[i], q);
}

bool r2_conn_ok_at(const r2_comm* c, int r, int k, uint32_t q) {
  const int r1 = (r + 1) % c->n;
  return !r2_ep_dead_at(c, r, k, q) && !r2_ep_dead_at(c, r1, k, q) && !r2_link_dead_at(c, r, k, q);
}

// Reading R-10: a LINK record is the standard ring's link r -> r+1; any other
// pair of ranks (a re-ranked or partial ring) is dead only with an endpoint.
bool r2_conn_ok_to(const r2_comm* c, int r, int to, int k, uint32_t q) {
  if (to == (r + 1) % c->n) return r2_conn_ok_at(c, r, k, q);
  return !r2_ep_dead_at(c, r, k, q) && !r2_ep_dead_at(c, to, k, q);
}

uint32_t r2_conn_mask_at(const r2_comm* c, int r, uint32_t q) {
  uint32_t m = 0;
  for (int k = 0; k < c->K; ++k)
    if (r2_conn_ok_at(c, r, k, q)) m |= 1u << k;
  return m;
}

// A death opens a new interval from `from_seq` (a collective that has not
// started on any rank whose plan depends on this record, see on_verdict).
void r2_declare_dead(r2_comm* c, int kind, int r, int k, uint32_t from_seq) {
  const int i = r * c->K + k;
  const size_t nk = (size_t)c->n * c->K;
  uint32_t& d = c->health[(kind == 0 ? R2_H_EP_DEAD : R2_H_LINK_DEAD) * nk + i];
  uint32_t& rs = c->health[(kind == 0 ? R2_H_EP_REP : R2_H_LINK_REP) * nk + i];
  if (r2_dead_at(d, rs, from_seq)) return;          // already dead then
  d = from_seq;
  // a REPAIR already enqueued for a later collective closes this interval
  uint32_t best = 0;
  for (const auto& rp : c->repairs_applied)
    if (rp.r == r && rp.c == k && rp.seq >= from_seq && (!best || rp.seq < best)) best = rp.seq;
  rs = best;
}

// A record may only change in ways that leave the view of every collective
// before `at_seq` untouched (kernels in flight read it): a REPAIR only closes
// an open death interval (dead since d <= at_seq, not yet repaired); an
// already repaired or never-dead record keeps its values.
void r2_declare_repaired(r2_comm* c, int r, int k, uint32_t at_seq) {
  const int i = r * c->K + k;
  const size_t nk = (size_t)c->n * c->K;
  c->repairs_applied.push_back({r, k, at_seq});
  if (c->repairs_applied.size() > 4096) c->repairs_applied.erase(c->repairs_applied.begin());
  for (int pair = 0; pair < 2; ++pair) {
    uint32_t& d = c->health[(pair ? R2_H_LINK_DEAD : R2_H_EP_DEAD) * nk + i];
    uint32_t& rs = c->health[(pair ? R2_H_LINK_REP : R2_H_EP_REP) * nk + i];
    if (d != 0 && rs < d && at_seq >= d) rs = at_seq;
  }
}

// A successful re-probe of connection r -> r+1 on channel k proves both
// endpoints and the link alive: close those three records (only open
// intervals, as r2_declare_repaired).
void r2_declare_conn_repaired(r2_comm* c, int r, int k, uint32_t at_seq) {
  const size_t nk = (size_t)c->n * c->K;
  const int r1 = (r + 1) % c->n;
  const struct { int kind; int rank; } recs[3] = {{0, r}, {0, r1}, {1, r}};
  for (const auto& x : recs) {
    const int i = x.rank * c->K + k;
    uint32_t& d = c->health[(x.kind ? R2_H_LINK_DEAD : R2_H_EP_DEAD) * nk + i];
    uint32_t& rs = c->health[(x.kind ? R2_H_LINK_REP : R2_H_EP_REP) * nk + i];
    if (d != 0 && rs < d && at_seq >= d) rs = at_seq;
  }
}

int r2_push_health(r2_comm* c) {
  const size_t bytes = c->health.size() * sizeof(uint32_t);
  memcpy(c->health_pinned, c->health.data(), bytes);     // pinned: true async DMA, no staging
  for (int l = 0; l < c->nlocal; ++l) {
    const RankPtrs& me = c->peers_host[l * c->n + c->first_rank + l];
    if (cudaMemcpyAsync(me.health, c->health_pinned, bytes, cudaMemcpyHostToDevice, c->health_stream) !=
        cudaSuccess)
      return -1;
  }
  return r2_spin_sync(c->health_stream) == cudaSuccess ? 0 : -1;
}

// Busy-wait for a stream (the monitor is on the failover critical path; a
// blocking synchronize can take 100+ us to wake up under load).
cudaError_t r2_spin_sync(cudaStream_t s) {
  cudaError_t e;
  while ((e = cudaStreamQuery(s)) == cudaErrorNotReady) {
  }
  return e;
}

extern "C" const char* r2_strerror(r2_result_t r) {
  switch (r) {
    case R2_SUCCESS: return "success";
    case R2_ERR_INVALID_ARG: return "invalid argument";
    case R2_ERR_CUDA: return "CUDA error";
    case R2_ERR_BOOTSTRAP: return "out-of-band bootstrap error";
    case R2_ERR_NOT_REGISTERED: return "recv buffer not registered";
    case R2_ERR_NO_BACKUP: return "failover chain exhausted (no healthy channel)";
    case R2_ERR_TIMEOUT: return "watchdog timeout";
    case R2_ERR_INTERNAL: return "internal error";
  }
  return "unknown error";
}

// Algorithm 1 (§6): bridge-based repair of a ring order.
// Rails of rank u = channels whose endpoint on u is alive; the capacity of
// the ring edge u -> v is |S_u ∩ S_v|, or 0 when the link u -> v is dead on
// every common channel (reading R-13; only standard links u -> u+1 mod n have
// link state, reading R-10).  Scan order, tie-breaks and skipped pairs: reading
// C-19 / R-13.
namespace {
struct RerankCtx {
  int n;
  const uint32_t* rails;
  const uint32_t* dead_links;
  int cap(int u, int v) const {
    const uint32_t m = rails[u] & rails[v];
    if (dead_links && v == (u + 1) % n && (m & ~dead_links[u]) == 0) return 0;   // no direct path left
    return __builtin_popcount(m);
  }
};
int ring_index(const int* R, int n, int u) {
  for (int i = 0; i < n; ++i)
    if (R[i] == u) return i;
  return -1;
}
}  // namespace

extern "C" int r2_rerank(int n, const int* ring_in, const uint32_t* rails, const uint32_t* dead_links,
                         int* ring_out) {
  if (n <= 0 || n > R2_MAX_RANKS || !ring_in || !rails || !ring_out) return -1;
  RerankCtx cx{n, rails, dead_links};
  int R[R2_MAX_RANKS];
  for (int i = 0; i < n; ++i) R[i] = ring_out[i] = ring_in[i];
  if (n < 3) return 0;
  int B = 1 << 30;                                   // line 2: B_global = min |S_u|
  for (int i = 0; i < n; ++i) B = std::min(B, __builtin_popcount(rails[ring_in[i]]));
  // lines 3-9: candidate edges of the input ring, gap descending, position ascending
  int cu[R2_MAX_RANKS], cv[R2_MAX_RANKS], gap[R2_MAX_RANKS], nc = 0;
  for (int i = 0; i < n; ++i) {
    const int u = ring_in[i], v = ring_in[(i + 1) % n], c = cx.cap(u, v);
    if (c >= B) continue;
    int at = nc++;
    while (at > 0 && gap[at - 1] < B - c) {          // stable insertion: ties keep position order
      cu[at] = cu[at - 1], cv[at] = cv[at - 1], gap[at] = gap[at - 1];
      --at;
    }
    cu[at] = u, cv[at] = v, gap[at] = B - c;
  }
  int moved = 0;
  for (int k = 0; k < nc; ++k) {
    const int u = cu[k], v = cv[k];
    int iu = ring_index(R, n, u);
    if (R[(iu + 1) % n] != v && R[(iu + n - 1) % n] != v) continue;   // already separated
    int best = -1;
    for (int i = 0; i < n && best < 0; ++i) {        // line 13: R' index order from position 0
      const int w = R[i];
      if (w == u || w == v) continue;
      const int x = R[(i + n - 1) % n], y = R[(i + 1) % n];
      if (std::min(cx.cap(u, w), cx.cap(w, v)) >= B && cx.cap(x, y) >= B) best = w;   // lines 15-19
    }
    if (best < 0) continue;
    // Relocate(best, between u and v)
    int ib = ring_index(R, n, best);
    for (int i = ib; i < n - 1; ++i) R[i] = R[i + 1];
    iu = ring_index(R, n - 1, u);
    const int at = R[(iu + 1) % (n - 1)] == v ? iu + 1 : iu;
    for (int i = n - 1; i > at; --i) R[i] = R[i - 1];
    R[at] = best;
    ++moved;
  }
  for (int i = 0; i < n; ++i) ring_out[i] = R[i];
  return moved;
}
