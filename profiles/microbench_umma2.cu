// Microbenchmark: tcgen05.mma issue rate of a CTA pair (cta_group::2,
// M = 256 across the two SMs of a cluster) against the single-CTA M = 128
// instruction, and the single-CTA rate for N = 32 / 64 / 128 / 256 issued
// warp-wide with elect.sync.  One
// cluster of 2 CTAs per SM pair, the leader's elected lane issues `iters`
// K = 16 MMAs back to back, then commits; cycles per MMA and per-SM MAC rate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o profiles/mb_umma2 profiles/microbench_umma2.cu && profiles/mb_umma2
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2402_14808_b200/csrc/rb_common.cuh"

using namespace rb;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, bool PAIR>
__global__ void __launch_bounds__(128, 1) k_umma2(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 196 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 196 * 1024 + 64);
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 196 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (threadIdx.x < 32) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(slot, 512);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x < 32 && rank == 0) {
    const uint32_t a_base = smem_u32(smem), b_base = smem_u32(smem + 64 * 1024);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      ad[kk] = make_smem_desc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
      bd[kk] = make_smem_desc_sw128(b_base + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
    }
    const uint32_t id = make_idesc_bf16_f32(PAIR ? 256 : 128, N, 0, 0);
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
      const uint32_t d = tmem + ((it >> 3) & 1) * 256;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (PAIR) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "elect.sync r|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(ad[kk]), "l"(bd[kk]), "r"(id), "r"(kk > 0 ? 1u : 0u)
              : "memory");
        } else {
          umma_f16_ss_elect(d, ad[kk], bd[kk], id, kk > 0 ? 1u : 0u);
        }
      }
    }
    if (PAIR) {
      asm volatile(
          "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\t"
          "elect.sync r|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
              smem_u32(bar)),
          "h"(static_cast<unsigned short>(1))
          : "memory");
    } else {
      umma_commit_elect(bar);
    }
    if (threadIdx.x == 0) {
      mbar_wait(bar, 0);
      out[blockIdx.x] = static_cast<unsigned long long>(clock64() - t0);
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();
  tc_fence_after();
  if (threadIdx.x < 32) {
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      tmem_dealloc(tmem, 512);
  }
}

template <int N, bool PAIR>
void run(int sms, unsigned long long* d_out) {
  const int smem = 197 * 1024;
  auto kern = k_umma2<N, PAIR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 8192;
  const int grid = (sms / 2) * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  cudaError_t err = cudaSuccess;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    err = cudaLaunchKernelEx(&cfg, kern, iters, d_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    printf("launch failed: %s\n", cudaGetErrorString(err));
    return;
  }
  unsigned long long h[256];
  cudaMemcpy(h, d_out, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  double cyc = 0;
  int n = 0;
  for (int i = 0; i < grid; i += PAIR ? 2 : 1, ++n) cyc += static_cast<double>(h[i]);
  cyc /= n;
  const double per = cyc / iters;
  const double macs_per_sm = 128.0 * N * 16;   // each SM's share of one instruction
  const double tf = 2.0 * macs_per_sm * iters * grid / (ms * 1e-3) / 1e12;
  printf("%s M=%d N=%3d: %6.1f cycles/MMA  %6.0f MAC/clk/SM  %7.0f TFLOP/s (%d CTAs, %.3f ms)\n",
         PAIR ? "cta_group::2" : "cta_group::1", PAIR ? 256 : 128, N, per, macs_per_sm / per, tf, grid, ms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 256 * sizeof(unsigned long long));
  run<32, false>(sms, d_out);
  run<64, false>(sms, d_out);
  run<128, false>(sms, d_out);
  run<256, false>(sms, d_out);
  run<64, true>(sms, d_out);
  run<128, true>(sms, d_out);
  run<256, true>(sms, d_out);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
