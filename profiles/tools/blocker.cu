// Diagnostics helper: occupy `grid` SMs (one CTA each, `smem` bytes of
// dynamic shared memory) for `ns` nanoseconds of %globaltimer, optionally
// streaming `bytes` per CTA from `src` meanwhile (HBM load of a concurrent
// kernel).  Built by profiles/tools/build.sh into profiles/tools/libblocker.so.
#include <cuda_runtime.h>
#include <cstdint>

__global__ void spin_kernel(long long ns, const uint4* src, long long per_cta, int* sink, int* counter) {
  extern __shared__ int sm[];
  if (counter != nullptr && threadIdx.x == 0) atomicAdd(counter, 1);
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned acc = 0;
  if (src != nullptr) {
    const uint4* p = src + blockIdx.x * per_cta;
    for (long long i = threadIdx.x; i < per_cta; i += blockDim.x) {
      uint4 v = __ldcs(p + i);
      acc ^= v.x;
    }
  }
  for (;;) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= static_cast<unsigned long long>(ns)) break;
  }
  if (threadIdx.x == 0) sm[0] = acc;
  __syncthreads();
  if (sm[0] == 0x7654321 && sink) sink[0] = 1;
}

// spins until *counter >= target (every blocker CTA is resident)
__global__ void wait_kernel(const int* counter, int target) {
  while (atomicAdd(const_cast<int*>(counter), 0) < target) __nanosleep(100);
}

extern "C" int waiter_launch(const void* counter, int target, void* stream) {
  wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const int*>(counter), target);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int blocker_launch(int grid, int smem, long long ns, const void* src, long long bytes_per_cta,
                              void* counter, void* stream) {
  cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  spin_kernel<<<grid, 384, smem, static_cast<cudaStream_t>(stream)>>>(
      ns, static_cast<const uint4*>(src), bytes_per_cta / 16, nullptr, static_cast<int*>(counter));
  return static_cast<int>(cudaGetLastError());
}
