// Microbenchmark: per-SM load throughput of TMA tensor boxes vs bulk copies by
// box size (the context tiles of the relay step are many small paged boxes).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include \
//        -o /tmp/mb_tma profiles/microbench_tma.cu -lcuda && /tmp/mb_tma
//
// One CTA per SM, one issuing lane, a ring of 8 x 16 KB slots kept full; every
// CTA streams its own contiguous 64 MB slice of a 9.5 GB buffer (no L2 reuse).
// mode 0: 3-D tensor box {64, rows, 1} with SWIZZLE_128B (rows * 128 B per box)
// mode 1: 1-D cp.async.bulk of `bytes` per copy
// mode 2: 1-D cp.async.bulk from pseudo-random `bytes`-aligned offsets of a
//         shared 256 MB region (the paged-KV pattern: scattered blocks)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../paper_2402_14808_b200/csrc/rb_common.cuh"

using namespace rb;

constexpr int kSlots = 8;
constexpr int kSlotBytes = 16384;

__global__ void __launch_bounds__(32, 1)
    mb_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* base, int mode,
              int bytes_per_op, int ops_per_slot, long long slot_iters, long long cta_bytes,
              unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSlots * kSlotBytes);
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int i = 0; i < kSlots; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const long long cta_off = static_cast<long long>(blockIdx.x) * cta_bytes;
  const int rows_per_op = bytes_per_op / 128;
  const unsigned long long t0 = clock64();
  if (lane == 0) {
    long long op = 0;
    for (long long it = 0; it < slot_iters; ++it) {
      const int s = static_cast<int>(it % kSlots);
      if (it >= kSlots) mbar_wait(&full[s], static_cast<uint32_t>(((it / kSlots) - 1) & 1));
      mbar_arrive_expect_tx(&full[s], ops_per_slot * bytes_per_op);
      for (int k = 0; k < ops_per_slot; ++k, ++op) {
        uint8_t* dst = smem + s * kSlotBytes + k * bytes_per_op;
        if (mode == 0) {
          // rows of 128 B (= 64 bf16) of a [total_rows][64] view
          const long long row = (cta_off / 128) + op * rows_per_op;
          tma_load_3d(dst, &tm, &full[s], 0, static_cast<int>(row % 65536),
                      static_cast<int>(row / 65536), l2_policy_evict_first());
        } else if (mode == 1) {
          bulk_copy_g2s(dst, base + cta_off + op * bytes_per_op, bytes_per_op, &full[s]);
        } else {
          const unsigned long long hsh =
              (static_cast<unsigned long long>(blockIdx.x) * 0x9E3779B97F4A7C15ull +
               static_cast<unsigned long long>(op) * 0xBF58476D1CE4E5B9ull) >> 20;
          const long long nslots = (256ll << 20) / bytes_per_op;
          bulk_copy_g2s(dst, base + (static_cast<long long>(hsh % nslots)) * bytes_per_op,
                        bytes_per_op, &full[s]);
        }
      }
    }
    for (long long it = slot_iters; it < slot_iters + kSlots; ++it) {
      const int s = static_cast<int>(it % kSlots);
      if (it >= kSlots) mbar_wait(&full[s], static_cast<uint32_t>(((it / kSlots) - 1) & 1));
    }
  }
  __syncwarp();
  if (lane == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long cta_bytes = 64ll << 20;
  const size_t total = cta_bytes * sms;
  uint8_t* buf = nullptr;
  if (cudaMalloc(&buf, total) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(buf, 1, total);
  unsigned long long* cyc = nullptr;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int smem = kSlots * kSlotBytes + 1024;
  cudaFuncSetAttribute(mb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("mode,bytes_per_op,ops_per_slot,GB/s_total,GB/s_per_SM,ns_per_op\n");
  for (int mode = 0; mode < 3; ++mode) {
    for (int bpo : {1024, 2048, 4096, 8192, 16384}) {
      CUtensorMap tm;
      const long long rows_total = total / 128;
      const int rows = bpo / 128;
      cuuint64_t dims[3] = {64, 65536, (cuuint64_t)(rows_total / 65536)};
      cuuint64_t strides[2] = {128, 128ull * 65536};
      cuuint32_t box[3] = {64, (cuuint32_t)(rows > 256 ? 256 : rows), 1};
      cuuint32_t es[3] = {1, 1, 1};
      if (mode == 0 && rows > 256) continue;
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int ops_per_slot = kSlotBytes / bpo;
      const long long slot_iters = (cta_bytes / 4) / kSlotBytes;  // 16 MB per CTA
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        mb_kernel<<<sms, 32, smem>>>(tm, buf, mode, bpo, ops_per_slot, slot_iters, cta_bytes, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = static_cast<double>(slot_iters) * kSlotBytes * sms;
      const double gbs = bytes / (ms * 1e-3) / 1e9;
      const double ops = static_cast<double>(slot_iters) * ops_per_slot;
      printf("%s,%d,%d,%.0f,%.1f,%.1f\n", mode == 0 ? "tma_tensor" : mode == 1 ? "bulk" : "bulk_random", bpo, ops_per_slot,
             gbs, gbs / sms, ms * 1e6 / ops);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
