// fence_bg.cu -- does fence.acq_rel.sys by one warp wait for OTHER warps'
// outstanding NVLink stores?  Warp 0 stores 128 B to the peer, fences, and
// times the fence; warps 1..B stream `bg` bytes to the peer concurrently.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence_bg tools/fence_bg.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s\n", cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void k(char* peer, size_t bg, int reps, unsigned long long* out) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    unsigned long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      if (lane < 8) ((uint4*)peer)[lane] = make_uint4(r, r, r, r);
      __syncwarp();
      unsigned long long t0, t1;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
      if (lane == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
      __syncwarp();
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
      tot += t1 - t0;
    }
    if (lane == 0) out[blockIdx.x] = tot / reps;
  } else {
    const size_t nvec = bg / 16;
    const int nthr = blockDim.x - 32, tid = threadIdx.x - 32;
    for (size_t v = tid; v < nvec; v += nthr) ((uint4*)(peer + 4096))[v] = make_uint4(v, v, v, v);
  }
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  char* peer;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&peer, 64 << 20));
  CK(cudaSetDevice(0));
  unsigned long long* out;
  CK(cudaMallocManaged(&out, 8 * 256));
  for (size_t bg : {(size_t)0, (size_t)64 << 10, (size_t)1 << 20, (size_t)8 << 20}) {
    for (int threads : {64, 512}) {
      k<<<1, threads>>>(peer, bg, 20, out);
      CK(cudaDeviceSynchronize());
      k<<<1, threads>>>(peer, bg, 20, out);
      CK(cudaDeviceSynchronize());
      printf("bg %8zu B  threads %3d : fence %6.2f us (avg of 20)\n", bg, threads, out[0] / 1965.0);
    }
  }
  return 0;
}
