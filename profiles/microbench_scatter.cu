// Microbenchmark: per-SM throughput of loading SCATTERED fixed-size blocks
// (the paged-KV pattern) through the TMA bulk-copy engine vs the LSU
// (cp.async 16 B per lane), by block size and by the size of the region the
// blocks are drawn from (address-translation reach).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o profiles/mb_scatter profiles/microbench_scatter.cu && profiles/mb_scatter
//
// One CTA per SM.  engine 0: one issuing lane, ring of 8 x 16 KB slots of
// cp.async.bulk.  engine 1: 4 warps, each keeps 8 groups of one block
// (lanes x 16 B cp.async) in flight (cp.async.wait_group).
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2402_14808_b200/csrc/rb_common.cuh"

using namespace rb;

constexpr int kSlots = 8;
constexpr int kSlotBytes = 16384;

__device__ __forceinline__ long long pick(long long op, long long nblocks) {
  const unsigned long long h =
      (static_cast<unsigned long long>(blockIdx.x) * 0x9E3779B97F4A7C15ull +
       static_cast<unsigned long long>(op) * 0xBF58476D1CE4E5B9ull) >> 17;
  return static_cast<long long>(h % nblocks);
}

__global__ void __launch_bounds__(128, 1)
    k_tma(const uint8_t* base, long long region, int bytes, long long n_ops) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSlots * kSlotBytes);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int per_slot = kSlotBytes / bytes;
  const long long nblocks = region / bytes;
  const long long slots = n_ops / per_slot;
  long long op = 0;
  for (long long it = 0; it < slots + kSlots; ++it) {
    const int s = static_cast<int>(it % kSlots);
    if (it >= kSlots) mbar_wait(&full[s], static_cast<uint32_t>(((it / kSlots) - 1) & 1));
    if (it >= slots) continue;
    mbar_arrive_expect_tx(&full[s], per_slot * bytes);
    for (int k = 0; k < per_slot; ++k, ++op)
      bulk_copy_g2s(smem + s * kSlotBytes + k * bytes, base + pick(op, nblocks) * bytes, bytes,
                    &full[s]);
  }
}

__global__ void __launch_bounds__(128, 1)
    k_lsu(const uint8_t* base, long long region, int bytes, long long n_ops) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warp w owns 32 KB of smem: 8 groups of up to 4 KB
  uint8_t* mine = smem + warp * 32768;
  const int gbytes = bytes < 4096 ? bytes : 4096;  // per group
  const long long nblocks = region / bytes;
  const long long my_ops = n_ops / 4;
  const int parts = bytes / gbytes;
  long long g = 0;
  for (long long op = 0; op < my_ops; ++op) {
    const uint8_t* src = base + pick(op * 4 + warp, nblocks) * bytes;
    for (int pp = 0; pp < parts; ++pp, ++g) {
      uint8_t* dst = mine + (g % 8) * 4096;
      for (int o = lane * 16; o < gbytes; o += 512) cp_async_16(dst + o, src + pp * gbytes + o, 16);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 7;" ::: "memory");
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// engine 2: the context kernel's pattern -- `ctas` CTAs per SM x 4 warps, each
// warp keeps `depth` chunks (K 4 KB + V 4 KB from two random blocks) in flight
template <int DEPTH>
__global__ void __launch_bounds__(128)
    k_lsu_kv(const uint8_t* base, long long region, long long n_chunks) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* mine = smem + warp * DEPTH * 8192;
  const long long nblocks = region / 4096;
  const long long my = n_chunks / 4;
  for (long long c = 0; c < my; ++c) {
    const long long op = (c * 4 + warp) * 2;
    const uint8_t* ks = base + pick(op, nblocks) * 4096;
    const uint8_t* vs = base + pick(op + 1, nblocks) * 4096;
    uint8_t* dst = mine + (c % DEPTH) * 8192;
    for (int o = lane * 16; o < 4096; o += 512) {
      cp_async_16(dst + o, ks + o, 16);
      cp_async_16(dst + 4096 + o, vs + o, 16);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1) : "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long max_region = 1ll << 30;
  uint8_t* buf = nullptr;
  if (cudaMalloc(&buf, max_region) != cudaSuccess) return 1;
  cudaMemset(buf, 1, max_region);
  const int smem = kSlots * kSlotBytes + 1024;
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_lsu, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("engine,region_MB,block_bytes,GB/s_total,GB/s_per_SM\n");
  for (int eng = 0; eng < 2; ++eng)
    for (long long mb : {16ll, 64ll, 256ll, 1024ll})
      for (int bytes : {4096, 16384}) {
        const long long per_cta_bytes = 8ll << 20;
        const long long n_ops = per_cta_bytes / bytes;
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (eng == 0)
            k_tma<<<sms, 128, smem>>>(buf, mb << 20, bytes, n_ops);
          else
            k_lsu<<<sms, 128, smem>>>(buf, mb << 20, bytes, n_ops);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
        }
        const double gbs = static_cast<double>(per_cta_bytes) * sms / (ms * 1e-3) / 1e9;
        printf("%s,%lld,%d,%.0f,%.1f\n", eng == 0 ? "tma_bulk" : "lsu_cp_async", mb, bytes, gbs,
               gbs / sms);
      }
  // the context kernel's configuration
  for (int ctas : {1, 2, 3}) {
    for (int depth : {2, 3, 6}) {
      const long long per_cta_bytes = 4ll << 20;
      const long long n_chunks = per_cta_bytes / 8192;
      const int sm_bytes = 4 * depth * 8192;
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (depth == 2) {
          cudaFuncSetAttribute(k_lsu_kv<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes);
          k_lsu_kv<2><<<sms * ctas, 128, sm_bytes>>>(buf, 1ll << 30, n_chunks);
        } else if (depth == 3) {
          cudaFuncSetAttribute(k_lsu_kv<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes);
          k_lsu_kv<3><<<sms * ctas, 128, sm_bytes>>>(buf, 1ll << 30, n_chunks);
        } else {
          cudaFuncSetAttribute(k_lsu_kv<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes);
          k_lsu_kv<6><<<sms * ctas, 128, sm_bytes>>>(buf, 1ll << 30, n_chunks);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double gbs = static_cast<double>(per_cta_bytes) * sms * ctas / (ms * 1e-3) / 1e9;
      printf("lsu_kv ctas/SM %d depth %d (in flight %d KB/SM): %.0f GB/s, %.1f per SM\n", ctas, depth,
             ctas * 4 * depth * 8, gbs, gbs / sms);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
