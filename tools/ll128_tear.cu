// ll128_tear.cu -- checks the property the LL128 protocol (reading R-12,
// r2_kernels.cu move_ll128) relies on: a 128-byte line written by ONE warp
// store instruction (8 lanes x 16 B) through an NVLink peer mapping is
// observed whole by a reader that loads it with one warp load instruction.
//
// GPU 0 rewrites L lines in GPU 1's memory over and over; every write of round
// s puts payload words h(s, line, word) and the flag vector {s, s, s, s}.
// GPU 1 reads the lines concurrently; a read whose flag vector is {s, s, s, s}
// must carry h(s, line, word) in all 28 payload words, otherwise it is a TEAR.
// Also counted: flag vectors that are themselves mixed (not one s).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ll128_tear tools/ll128_tear.cu
//   tools/bin/ll128_tear [seconds=5] [lines=4096]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

__device__ __forceinline__ unsigned int h(unsigned int s, unsigned int line, unsigned int w) {
  unsigned int x = s * 0x9E3779B1u ^ line * 0x85EBCA77u ^ w * 0xC2B2AE3Du;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  return x | 1u;   // never 0 (fresh memory is 0)
}

__global__ void writer(char* lines, int L, volatile int* stop, unsigned int* rounds) {
  const unsigned int lane = threadIdx.x & 31u, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned int nwarps = (gridDim.x * blockDim.x) >> 5, pos = lane & 7u;
  unsigned int s = 1;
  for (; !*stop; ++s) {
    for (unsigned int base = warp * 4; base < (unsigned int)L; base += nwarps * 4) {
      const unsigned int line = base + (lane >> 3);
      uint4 v;
      if (pos == 7) v = make_uint4(s, s, s, s);
      else v = make_uint4(h(s, line, pos * 4), h(s, line, pos * 4 + 1), h(s, line, pos * 4 + 2), h(s, line, pos * 4 + 3));
      if (line < (unsigned int)L)
        asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(lines + (size_t)line * 128 + pos * 16),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *rounds = s;
}

__global__ void reader(const char* lines, int L, volatile int* stop, unsigned long long* stats) {
  const unsigned int lane = threadIdx.x & 31u, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned int nwarps = (gridDim.x * blockDim.x) >> 5, pos = lane & 7u;
  unsigned long long reads = 0, valid = 0, tears = 0, mixed = 0;
  while (!*stop) {
    for (unsigned int base = warp * 4; base < (unsigned int)L; base += nwarps * 4) {
      const unsigned int line = base + (lane >> 3);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (line < (unsigned int)L)
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(lines + (size_t)line * 128 + pos * 16)
                     : "memory");
      const unsigned int s = __shfl_sync(0xFFFFFFFFu, v.x, lane | 7u);
      const bool fl_ok = __shfl_sync(0xFFFFFFFFu, (int)(v.x == v.y && v.y == v.z && v.z == v.w), lane | 7u);
      bool bad = false;
      if (fl_ok && s != 0 && pos < 7)
        bad = v.x != h(s, line, pos * 4) || v.y != h(s, line, pos * 4 + 1) || v.z != h(s, line, pos * 4 + 2) ||
              v.w != h(s, line, pos * 4 + 3);
      const unsigned int badm = __ballot_sync(0xFFFFFFFFu, bad);
      if (pos == 0 && line < (unsigned int)L) {
        ++reads;
        if (!fl_ok) ++mixed;
        else if (s != 0) {
          ++valid;
          if ((badm >> (lane & ~7u)) & 0xFFu) ++tears;
        }
      }
    }
  }
  atomicAdd(&stats[0], reads);
  atomicAdd(&stats[1], valid);
  atomicAdd(&stats[2], tears);
  atomicAdd(&stats[3], mixed);
}

int main(int argc, char** argv) {
  const double secs = argc > 1 ? atof(argv[1]) : 5.0;
  const int L = argc > 2 ? atoi(argv[2]) : 4096;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  char* lines;
  int* stop;
  unsigned long long* stats;
  unsigned int* rounds;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&lines, (size_t)L * 128));
  CK(cudaMemset(lines, 0, (size_t)L * 128));
  CK(cudaMalloc(&stats, 4 * sizeof(unsigned long long)));
  CK(cudaMemset(stats, 0, 4 * sizeof(unsigned long long)));
  CK(cudaHostAlloc(&stop, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostAlloc(&rounds, sizeof(unsigned int), cudaHostAllocMapped | cudaHostAllocPortable));
  *stop = 0;
  CK(cudaDeviceSynchronize());
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaSetDevice(1));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  reader<<<64, 256, 0, s1>>>(lines, L, stop, stats);
  CK(cudaSetDevice(0));
  writer<<<64, 256, 0, s0>>>(lines, L, stop, rounds);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  do {
    clock_gettime(CLOCK_MONOTONIC, &t1);
  } while ((t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec) < secs);
  *stop = 1;
  CK(cudaStreamSynchronize(s0));
  CK(cudaSetDevice(1));
  CK(cudaStreamSynchronize(s1));
  unsigned long long st[4];
  CK(cudaMemcpy(st, stats, sizeof(st), cudaMemcpyDeviceToHost));
  printf("lines %d, %.1f s, writer rounds %u: line reads %llu, flag-valid %llu, TEARS %llu, mixed flag vectors %llu\n",
         L, secs, *rounds, st[0], st[1], st[2], st[3]);
  return st[2] ? 2 : 0;
}
