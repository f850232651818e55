// Test-only helper (tests/test_gpu_service.py): a kernel that fills every SM
// left free by a resident collective (2 x 1024 threads per SM = the SM's
// thread limit) and spins on %globaltimer, so no other kernel can start
// while it runs.  Built by the test with nvcc; not part of the product.
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 2) r2t_spin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

extern "C" int r2t_spin(unsigned long long ns, int blocks, void* stream) {
  r2t_spin_kernel<<<blocks, 1024, 0, (cudaStream_t)stream>>>(ns);
  return (int)cudaGetLastError();
}
