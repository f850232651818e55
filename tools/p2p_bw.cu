// p2p_bw.cu -- NVLink peer-store ceiling for the data mover's access pattern.
// One process, G GPUs (2 or 4), peer access enabled; GPU g streams a local
// buffer into GPU (g+1)%G's buffer with SM stores (the ring's traffic shape),
// all GPUs at once.  Reports per-GPU egress GB/s for several CTA / thread /
// vector-width / unroll choices, plus the copy engine for reference.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_bw tools/p2p_bw.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <int VB, int UNR, bool ADD>
__global__ void push(const char* __restrict__ src, const char* __restrict__ src2, char* __restrict__ dst,
                     size_t bytes) {
  const size_t nvec = bytes / VB;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (VB == 16) {
    for (; v + (UNR - 1) * stride < nvec; v += UNR * stride) {
      uint4 a[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) a[u] = __ldcg((const uint4*)src + v + u * stride);
      if (ADD) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          uint4 b = __ldcg((const uint4*)src2 + v + u * stride);
          a[u].x += b.x; a[u].y += b.y; a[u].z += b.z; a[u].w += b.w;
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) ((uint4*)dst)[v + u * stride] = a[u];
    }
  } else {
    for (; v + (UNR - 1) * stride < nvec; v += UNR * stride) {
      unsigned int a[UNR][8];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const char* p = src + (v + u * stride) * 32;
        asm volatile("ld.global.cg.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(a[u][0]), "=r"(a[u][1]), "=r"(a[u][2]), "=r"(a[u][3]), "=r"(a[u][4]), "=r"(a[u][5]),
                       "=r"(a[u][6]), "=r"(a[u][7])
                     : "l"(p));
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        char* p = dst + (v + u * stride) * 32;
        asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a[u][0]), "r"(a[u][1]),
                     "r"(a[u][2]), "r"(a[u][3]), "r"(a[u][4]), "r"(a[u][5]), "r"(a[u][6]), "r"(a[u][7])
                     : "memory");
      }
    }
  }
}

typedef void (*Kern)(const char*, const char*, char*, size_t);

// TMA bulk path: one thread per CTA streams B-byte pieces global -> smem
// (cp.async.bulk + mbarrier) -> peer global (cp.async.bulk bulk_group).
template <int B, int S>
__global__ void push_tma(const char* __restrict__ src, const char* __restrict__ src2, char* __restrict__ dst,
                         size_t bytes) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) unsigned long long bar[S];
  if (threadIdx.x != 0) return;
  const size_t npieces = bytes / B;
  for (int s = 0; s < S; ++s) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  unsigned int phase[S];
  for (int s = 0; s < S; ++s) phase[s] = 0;
  auto load = [&](size_t piece, int s) {
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * B);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(B) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                 "l"(src + piece * B), "r"(B), "r"(a)
                 : "memory");
  };
  size_t first = blockIdx.x, step = gridDim.x;
  size_t p = first;
  int issued = 0;
  for (int s = 0; s < S && first + (size_t)s * step < npieces; ++s) load(first + (size_t)s * step, s), ++issued;
  int i = 0;
  for (p = first; p < npieces; p += step, ++i) {
    const int s = i % S;
    unsigned a = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                   : "=r"(ok)
                   : "r"(a), "r"(phase[s])
                   : "memory");
    phase[s] ^= 1u;
    unsigned sm = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * B);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + p * B), "r"(sm), "r"(B)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill the stage of the previous piece once its store has read smem
    if (i >= 1) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const size_t nxt = p + (size_t)(S - 1) * step;
      if (nxt < npieces) load(nxt, (i - 1) % S);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int VB, int UNR>
__global__ void pull(const char* __restrict__ src, const char* __restrict__ src2, char* __restrict__ dst,
                     size_t bytes) {
  // src here is the PEER's buffer, dst local
  const size_t nvec = bytes / 16;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; v + (UNR - 1) * stride < nvec; v += UNR * stride) {
    uint4 a[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) a[u] = __ldcg((const uint4*)src + v + u * stride);
#pragma unroll
    for (int u = 0; u < UNR; ++u) ((uint4*)dst)[v + u * stride] = a[u];
  }
}

int main(int argc, char** argv) {
  int G = argc > 1 ? atoi(argv[1]) : 2;
  size_t bytes = (argc > 2 ? atoll(argv[2]) : 256ll) << 20;
  char *src[8], *src2[8], *dst[8];
  cudaStream_t st[8];
  cudaEvent_t e0[8], e1[8];
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMalloc(&src2[g], bytes));
    CK(cudaMalloc(&dst[g], bytes));
    CK(cudaMemset(src[g], 1, bytes));
    CK(cudaMemset(src2[g], 2, bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  struct Cfg {
    const char* name;
    Kern k;
  } cfgs[] = {
      {"v16 unr4", push<16, 4, false>}, {"v16 unr8", push<16, 8, false>}, {"v32 unr4", push<32, 4, false>},
      {"v16 unr8 +add(2 local reads)", push<16, 8, true>}, {"pull v16 unr8", pull<16, 8>},
      {"tma 16K x4", push_tma<16384, 4>}, {"tma 32K x4", push_tma<32768, 4>}, {"tma 32K x6", push_tma<32768, 6>},
      {"tma 64K x3", push_tma<65536, 3>},
  };
  int ctas_list[] = {32, 64, 96, 128, 146};
  int thr_list[] = {32, 256, 512, 1024};
  const int iters = 10;
  // copy engine reference
  {
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaMemcpyPeerAsync(dst[(g + 1) % G], (g + 1) % G, src[g], g, bytes, st[g]));
    }
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaStreamSynchronize(st[g]));
      CK(cudaEventRecord(e0[g], st[g]));
      for (int i = 0; i < iters; ++i) CK(cudaMemcpyPeerAsync(dst[(g + 1) % G], (g + 1) % G, src[g], g, bytes, st[g]));
      CK(cudaEventRecord(e1[g], st[g]));
    }
    float worst = 0;
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventSynchronize(e1[g]));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
      if (ms > worst) worst = ms;
    }
    printf("G=%d %zu MiB copy-engine peer copy: %.1f GB/s per GPU\n", G, bytes >> 20, bytes * iters / (worst * 1e6));
  }
  CK(cudaSetDevice(0));
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFuncSetAttribute(push_tma<16384, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
    CK(cudaFuncSetAttribute(push_tma<32768, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
    CK(cudaFuncSetAttribute(push_tma<32768, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768));
    CK(cudaFuncSetAttribute(push_tma<65536, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536));
  }
  // hybrid: SM stores on a fraction of the bytes, the copy engine on the rest
  if (getenv("HYBRID")) {
    cudaStream_t st2[8];
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaStreamCreateWithFlags(&st2[g], cudaStreamNonBlocking));
    }
    for (int pct : {0, 20, 30, 40, 50, 60, 100}) {
      const size_t ce = (bytes * pct / 100) & ~(size_t)65535, sm = bytes - ce;
      float worst = 0;
      for (int rep = 0; rep < 2; ++rep) {
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaStreamSynchronize(st[g]));
          CK(cudaStreamSynchronize(st2[g]));
        }
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventRecord(e0[g], st[g]));
          CK(cudaStreamWaitEvent(st2[g], e0[g], 0));
          for (int i = 0; i < iters; ++i) {
            if (sm) push<16, 8, false><<<128, 512, 0, st[g]>>>(src[g], src2[g], dst[(g + 1) % G], sm);
            if (ce) CK(cudaMemcpyPeerAsync(dst[(g + 1) % G] + sm, (g + 1) % G, src[g] + sm, g, ce, st2[g]));
          }
          cudaEvent_t j;
          CK(cudaEventCreate(&j));
          CK(cudaEventRecord(j, st2[g]));
          CK(cudaStreamWaitEvent(st[g], j, 0));
          CK(cudaEventRecord(e1[g], st[g]));
        }
        worst = 0;
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventSynchronize(e1[g]));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
          if (ms > worst) worst = ms;
        }
      }
      printf("G=%d hybrid CE %d%%: %.1f GB/s per GPU\n", G, pct, bytes * iters / (worst * 1e6));
    }
    // two destinations: half the CTAs to g+1, half to g-1
    for (int ctas : {64, 128}) {
      float worst = 0;
      for (int rep = 0; rep < 2; ++rep) {
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventRecord(e0[g], st[g]));
          for (int i = 0; i < iters; ++i) {
            push<16, 8, false><<<ctas, 512, 0, st[g]>>>(src[g], src2[g], dst[(g + 1) % G], bytes / 2);
            push<16, 8, false><<<ctas, 512, 0, st2[g]>>>(src[g] + bytes / 2, src2[g], dst[(g + G - 1) % G] + bytes / 2,
                                                          bytes / 2);
          }
          cudaEvent_t j;
          CK(cudaEventCreate(&j));
          CK(cudaEventRecord(j, st2[g]));
          CK(cudaStreamWaitEvent(st[g], j, 0));
          CK(cudaEventRecord(e1[g], st[g]));
        }
        worst = 0;
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventSynchronize(e1[g]));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
          if (ms > worst) worst = ms;
        }
      }
      printf("G=%d two-peer SM push 2x%d CTAs: %.1f GB/s per GPU\n", G, ctas, bytes * iters / (worst * 1e6));
    }
    return 0;
  }
  for (auto& c : cfgs)
    for (int thr : thr_list)
      for (int ctas : ctas_list) {
        const bool tma = c.name[0] == 't', pl = c.name[0] == 'p';
        if (tma && thr != 32) continue;
        if (!tma && thr == 32) continue;
        size_t smem = 0;
        if (tma) {
          int B = atoi(c.name + 4) * 1024, S = atoi(strchr(c.name, 'x') + 1);
          smem = (size_t)B * S;
        }
        cudaFuncAttributes fa;
        CK(cudaFuncGetAttributes(&fa, c.k));
        if (fa.maxThreadsPerBlock < thr) continue;
        const char* s_of[8];
        char* d_of[8];
        for (int g = 0; g < G; ++g) {
          s_of[g] = pl ? src[(g + G - 1) % G] : src[g];
          d_of[g] = pl ? dst[g] : dst[(g + 1) % G];
        }
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          c.k<<<ctas, thr, smem, st[g]>>>(s_of[g], src2[g], d_of[g], bytes);
          CK(cudaGetLastError());
        }
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaStreamSynchronize(st[g]));
        }
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventRecord(e0[g], st[g]));
          for (int i = 0; i < iters; ++i) c.k<<<ctas, thr, smem, st[g]>>>(s_of[g], src2[g], d_of[g], bytes);
          CK(cudaEventRecord(e1[g], st[g]));
        }
        float worst = 0;
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventSynchronize(e1[g]));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
          if (ms > worst) worst = ms;
        }
        printf("G=%d %s thr=%d ctas=%d: %.1f GB/s per GPU\n", G, c.name, thr, ctas, bytes * iters / (worst * 1e6));
      }
  return 0;
}
