// pingpong.cu -- per-hop latency floor of the ring's completion protocols
// between two B200s over NVLink (one process, peer access, one CTA per GPU).
// Each hop: GPU a writes B payload bytes into GPU b, makes them visible, and
// signals; GPU b waits for the signal (and the data) and answers.  Reports
// one-way latency = round trip / 2 for:
//   flag     : a flag store only (no payload)
//   fence    : payload st.v4, fence.acq_rel.sys, flag store   (the ring's protocol)
//   release  : payload st.v4, __syncthreads, st.release.sys flag
//   ll       : payload as LL lines {d0, seq, d1, seq} (st.volatile.v4); the
//              receiver polls every line (no fence, no separate flag)
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pingpong tools/pingpong.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ unsigned ld_acq(const volatile unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const volatile unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx(volatile unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel(volatile unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// mode 0 flag, 1 fence, 2 release, 3 ll
__global__ void hop(int mode, int first, int iters, unsigned bytes, char* peer_data, const char* my_data,
                    volatile unsigned* peer_flag, volatile unsigned* my_flag, unsigned long long* out_ns) {
  const unsigned nvec = bytes / 16;
  __shared__ int ok;
  unsigned long long t0 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    const unsigned seq = (unsigned)i;
    const bool send_now = first || true;
    // wait for the peer's hop i (the second GPU) / i-1 (the first)
    const unsigned want = first ? seq - 1 : seq;
    if (want > 0) {
      if (mode == 3) {
        // every thread polls its LL lines
        for (unsigned v = threadIdx.x; v < nvec * 2; v += blockDim.x) {
          const volatile uint4* l = (const volatile uint4*)(my_data + (size_t)v * 16);
          for (;;) {
            uint4 x;
            asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                         : "l"(l));
            if (x.y == want && x.w == want) break;
          }
        }
        if (nvec == 0 && threadIdx.x == 0)
          while (ld_rlx(my_flag) != want) {
          }
        __syncthreads();
      } else {
        if (threadIdx.x == 0) {
          while (ld_rlx(my_flag) != want) {
          }
          asm volatile("fence.acq_rel.sys;" ::: "memory");
        }
        __syncthreads();
      }
    }
    (void)send_now;
    // send hop
    if (mode == 0) {
      if (threadIdx.x == 0) st_rlx(peer_flag, seq);
    } else if (mode == 3) {
      for (unsigned v = threadIdx.x; v < nvec * 2; v += blockDim.x) {
        asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(peer_data + (size_t)v * 16), "r"(v),
                     "r"(seq), "r"(v + 1), "r"(seq)
                     : "memory");
      }
      if (nvec == 0 && threadIdx.x == 0) st_rlx(peer_flag, seq);
    } else {
      for (unsigned v = threadIdx.x; v < nvec; v += blockDim.x) {
        uint4 a = make_uint4(v, seq, v, seq);
        asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(peer_data + (size_t)v * 16), "r"(a.x),
                     "r"(a.y), "r"(a.z), "r"(a.w)
                     : "memory");
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (mode == 1) {
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          st_rlx(peer_flag, seq);
        } else {
          st_rel(peer_flag, seq);
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *out_ns = t1 - t0;
  }
  (void)ok;
}

int main() {
  char *data[2];
  unsigned* flag[2];
  unsigned long long* ns[2];
  cudaStream_t st[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&data[g], 8 << 20));
    CK(cudaMalloc(&flag[g], 4096));
    CK(cudaMallocManaged(&ns[g], 8));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
  }
  const char* names[] = {"flag", "fence", "release", "ll"};
  unsigned sizes[] = {0, 128, 4096, 65536};
  const int iters = 2000;
  for (int mode = 0; mode < 4; ++mode)
    for (unsigned b : sizes) {
      if (mode == 0 && b) continue;
      for (int thr : {32, 512}) {
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaMemset(data[g], 0, 8 << 20));
          CK(cudaMemset(flag[g], 0, 4096));
          CK(cudaDeviceSynchronize());
        }
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          hop<<<1, thr, 0, st[g]>>>(mode, g == 0, iters, b, data[1 - g], data[g], flag[1 - g], flag[g], ns[g]);
          CK(cudaGetLastError());
        }
        for (int g = 0; g < 2; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaStreamSynchronize(st[g]));
        }
        printf("%-8s %6u B  %3d thr: one-way %.2f us\n", names[mode], b, thr, (double)*ns[0] / iters / 2 / 1e3);
        fflush(stdout);
      }
    }
  return 0;
}
