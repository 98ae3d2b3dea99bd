// Microbenchmark: tcgen05.mma issue throughput per SM for the shapes and
// operand sources of the GQA system kernels (no TMA traffic, no softmax):
// one CTA per SM, one thread issues `iters` MMAs of K = 16 back to back into
// two alternating TMEM accumulators, then waits on a commit.  Reports cycles
// per MMA and the per-SM MAC rate against the 128 x N / 256-cycle floor of
// /opt/skills/guides/B300_MICROARCH.md (tcgen05 floor).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o profiles/mb_umma profiles/microbench_umma.cu && profiles/mb_umma
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2402_14808_b200/csrc/rb_common.cuh"

using namespace rb;

// mode: 0 SS (A, B K-major), 1 SS B MN-major, 2 TS (A in TMEM) B K-major,
// 3 TS B MN-major
// tcgen05.mma issued by the whole warp with one elected lane (operands warp-
// uniform), so the descriptors can live in uniform registers
__device__ __forceinline__ void umma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int N>
__global__ void __launch_bounds__(128, 1) k_umma(int mode, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 196 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 196 * 1024 + 64);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 196 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (threadIdx.x < 32) tmem_alloc(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (mode >= 6 && threadIdx.x < 32) {
    // whole warp, elected issue, precomputed descriptors
    const uint32_t a_base = smem_u32(smem), b_base = smem_u32(smem + 64 * 1024);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      ad[kk] = make_smem_desc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
      bd[kk] = make_smem_desc_sw128(b_base + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
    }
    const uint32_t id = make_idesc_bf16_f32(128, N, 0, 0);
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
      const uint32_t d = tmem + ((it >> 3) & 1) * 256;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (mode == 6)
          umma_ss_elect(d, ad[kk], bd[kk], id, kk > 0 ? 1u : 0u);
        else
          umma_ts_elect(d, tmem + 384 + kk * 8, bd[kk], id, kk > 0 ? 1u : 0u);
      }
    }
    if (threadIdx.x == 0) {
      umma_commit(bar);
      mbar_wait(bar, 0);
      out[blockIdx.x] = static_cast<unsigned long long>(clock64() - t0);
    }
    __syncwarp();
  } else if (mode < 6 && threadIdx.x == 0) {
    const uint32_t a_base = smem_u32(smem);               // 128 rows x 128 K (32 KB)
    const uint32_t b_base = smem_u32(smem + 64 * 1024);   // N rows x 128 K
    const bool bmn = mode == 1 || mode == 3, ts = mode >= 2;
    const uint32_t idesc = make_idesc_bf16_f32(128, N, 0, bmn ? 1 : 0);
    const long long t0 = clock64();
    if (mode >= 4) {
      // precomputed descriptors, 8 MMAs unrolled per iteration (SS, B K-major)
      uint64_t ad[8], bd[8];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        ad[kk] = make_smem_desc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
        bd[kk] = make_smem_desc_sw128(b_base + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
      }
      const uint32_t id = make_idesc_bf16_f32(128, N, 0, 0);
      for (int it = 0; it < iters; it += 8) {
        const uint32_t d = tmem + ((it >> 3) & 1) * 256;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (mode == 4)
            umma_f16_ss(d, ad[kk], bd[kk], id, kk > 0 ? 1u : 0u);
          else
            umma_f16_ts(d, tmem + 384 + kk * 8, bd[kk], id, kk > 0 ? 1u : 0u);
        }
      }
    } else {
    for (int it = 0; it < iters; ++it) {
      const int kk = it & 7;
      const uint32_t d = tmem + ((it >> 3) & 1) * 256;
      const uint64_t b = bmn ? make_smem_desc_sw128(b_base + kk * 2048, 16384, 1024)
                             : make_smem_desc_sw128(b_base + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
      if (ts) {
        umma_f16_ts(d, tmem + 384 + kk * 8, b, idesc, kk > 0 ? 1u : 0u);
      } else {
        const uint64_t a = make_smem_desc_sw128(a_base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
        umma_f16_ss(d, a, b, idesc, kk > 0 ? 1u : 0u);
      }
    }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N>
void run(int sms, int mode, unsigned long long* d_out) {
  const int smem = 197 * 1024;
  cudaFuncSetAttribute(k_umma<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 8192;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_umma<N><<<sms, 128, smem>>>(mode, iters, d_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  unsigned long long h[256];
  cudaMemcpy(h, d_out, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < sms; ++i) cyc += static_cast<double>(h[i]);
  cyc /= sms;
  const double per = cyc / iters;
  const double macs = 128.0 * N * 16;
  const double tf = 2.0 * macs * iters * sms / (ms * 1e-3) / 1e12;
  const char* names[] = {"SS  B K-major", "SS  B MN-major", "TS  B K-major", "TS  B MN-major",
                         "SS  precomp x8", "TS  precomp x8", "SS  warp elect", "TS  warp elect"};
  printf("M=128 N=%3d %s: %6.1f cycles/MMA (floor %3d)  %6.0f MAC/clk/SM  %7.0f TFLOP/s (%d SMs, %.3f ms)\n",
         N, names[mode], per, 128 * N / 256, macs / per, tf, sms, ms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 256 * sizeof(unsigned long long));
  for (int mode = 0; mode < 4; ++mode) {
    run<64>(sms, mode, d_out);
    run<128>(sms, mode, d_out);
    if (mode < 2) run<256>(sms, mode, d_out);  // (TS: A sits in columns 384+)
  }
  run<64>(sms, 4, d_out);
  run<128>(sms, 4, d_out);
  run<256>(sms, 4, d_out);
  run<64>(sms, 5, d_out);
  run<128>(sms, 5, d_out);
  run<64>(sms, 6, d_out);
  run<128>(sms, 6, d_out);
  run<256>(sms, 6, d_out);
  run<64>(sms, 7, d_out);
  run<128>(sms, 7, d_out);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
