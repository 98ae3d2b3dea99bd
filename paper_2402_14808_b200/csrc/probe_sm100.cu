// Layout probes of the relay step's tcgen05 operands (tests only).
//
// Paged-context operands:
// one CTA builds a 128-key K and V tile in the PagedKvCache block layout
// ([128 d][bs tokens] per block, paged_swizzle applied), Q and P in the
// K-major SW128 layout, and runs exactly the descriptors relay_step_kernel
// uses for context tiles:
//   S^T[128 keys x 32] = K (A, MN-major, Swizzle(2*bs)) . Q^T (B, K-major SW128)
//   O^T[128 d x 32]    = V^T (A, K-major, Swizzle(2*bs)) . P^T (B, K-major SW128)
#include "rb_common.cuh"
#include "rb_plan.h"

namespace rb {

constexpr int kKvTileBytes = RB_KEY_TILE * RB_HEAD_DIM * 2;  // 32 KB

__global__ void ctx_probe_kernel(const __nv_bfloat16* k, const __nv_bfloat16* q,
                                 const __nv_bfloat16* v, const __nv_bfloat16* p, int bs,
                                 float* s_out, float* o_out) {
  constexpr int NQ = 32;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sk = smem;
  uint8_t* sv = smem + 32768;
  uint8_t* sq = smem + 65536;
  uint8_t* sp = sq + NQ * 256;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sp + NQ * 256);
  uint32_t* tm = reinterpret_cast<uint32_t*>(bar + 2);
  const uint32_t rb = 2 * bs;
  for (int idx = threadIdx.x; idx < 128 * 128; idx += blockDim.x) {
    const int t = idx / 128, d = idx % 128;  // key t, dim d
    const uint32_t off = (t / bs) * bs * 256 + paged_swizzle(d * rb + (t % bs) * 2, rb);
    *reinterpret_cast<__nv_bfloat16*>(sk + off) = k[idx];
    *reinterpret_cast<__nv_bfloat16*>(sv + off) = v[idx];
  }
  for (int idx = threadIdx.x; idx < NQ * 128; idx += blockDim.x) {
    const int row = idx / 128, col = idx % 128;
    const uint32_t off = (col >> 6) * (NQ * 128) + sw128_offset(row, col & 63);
    *reinterpret_cast<__nv_bfloat16*>(sq + off) = q[idx];
    *reinterpret_cast<__nv_bfloat16*>(sp + off) = p[idx];
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(tm, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tm;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc_qk = make_idesc_bf16_f32(128, NQ, 1, 0);
    constexpr uint32_t idesc_pv = make_idesc_bf16_f32(128, NQ, 0, 0);
    const uint32_t k_base = smem_u32(sk), v_base = smem_u32(sv);
    const uint32_t q_base = smem_u32(sq), p_base = smem_u32(sp);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t b =
          make_smem_desc_sw128(q_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
      umma_f16_ss(tbase, ctx_k_desc(k_base, kk, bs), b, idesc_qk, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar[0]);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t b =
          make_smem_desc_sw128(p_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
      umma_f16_ss(tbase + 64, ctx_v_desc(v_base, kk, bs), b, idesc_pv, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar[1]);
  }
  __syncwarp();
  mbar_wait(&bar[0], 0);
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t laddr = tbase + (static_cast<uint32_t>(warp * 32) << 16);
  for (int c0 = 0; c0 < NQ; c0 += 8) {
    float s[8], o[8];
    tmem_ld_32x32b<8>(laddr + c0, s);
    tmem_ld_32x32b<8>(laddr + 64 + c0, o);
    tmem_wait_ld();
    for (int c = 0; c < 8; ++c) {
      s_out[(warp * 32 + lane) * NQ + c0 + c] = s[c];
      o_out[(warp * 32 + lane) * NQ + c0 + c] = o[c];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tbase, 128);
  }
}

cudaError_t launch_ctx_probe(const __nv_bfloat16* k, const __nv_bfloat16* q,
                             const __nv_bfloat16* v, const __nv_bfloat16* p, int bs, float* s_out,
                             float* o_out, cudaStream_t stream) {
  if (bs != 16 && bs != 32 && bs != 64) return cudaErrorInvalidValue;
  const int smem = 65536 + 2 * 32 * 256 + 64;
  cudaError_t e =
      cudaFuncSetAttribute(ctx_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  ctx_probe_kernel<<<1, 128, smem, stream>>>(k, q, v, p, bs, s_out, o_out);
  return cudaGetLastError();
}

// ------------------------------------------- system-tile layout probe
// One-CTA check of the exact operand layouts / descriptors the system kernel
// uses (K, V in the TMA SW128 box layout; Q, P in the K-major SW128 layout).
template <int NQ>
__global__ void umma_probe_kernel(const __nv_bfloat16* k, const __nv_bfloat16* q,
                                  const __nv_bfloat16* v, const __nv_bfloat16* p, float* s_out,
                                  float* o_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sk = smem;
  uint8_t* sv = smem + kKvTileBytes;
  uint8_t* sq = smem + 2 * kKvTileBytes;
  uint8_t* sp = sq + NQ * 256;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sp + NQ * 256);
  uint32_t* tm = reinterpret_cast<uint32_t*>(bar + 2);
  for (int idx = threadIdx.x; idx < 128 * 128; idx += blockDim.x) {
    const int row = idx / 128, col = idx % 128;
    const uint32_t off = (col >> 6) * (kKvTileBytes / 2) + sw128_offset(row, col & 63);
    *reinterpret_cast<__nv_bfloat16*>(sk + off) = k[idx];
    *reinterpret_cast<__nv_bfloat16*>(sv + off) = v[idx];
  }
  for (int idx = threadIdx.x; idx < NQ * 128; idx += blockDim.x) {
    const int row = idx / 128, col = idx % 128;
    const uint32_t off = (col >> 6) * (NQ * 128) + sw128_offset(row, col & 63);
    *reinterpret_cast<__nv_bfloat16*>(sq + off) = q[idx];
    *reinterpret_cast<__nv_bfloat16*>(sp + off) = p[idx];
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(tm, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tm;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc_qk = make_idesc_bf16_f32(128, NQ, 0, 0);
    constexpr uint32_t idesc_pv = make_idesc_bf16_f32(128, NQ, 1, 0);
    const uint32_t k_base = smem_u32(sk), v_base = smem_u32(sv);
    const uint32_t q_base = smem_u32(sq), p_base = smem_u32(sp);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a =
          make_smem_desc_sw128(k_base + (kk >> 2) * (kKvTileBytes / 2) + (kk & 3) * 32, 16, 1024);
      const uint64_t b = make_smem_desc_sw128(q_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
      umma_f16_ss(tbase, a, b, idesc_qk, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar[0]);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a = make_smem_desc_sw128(v_base + kk * 2048, kKvTileBytes / 2, 1024);
      const uint64_t b = make_smem_desc_sw128(p_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
      umma_f16_ss(tbase + 64, a, b, idesc_pv, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar[1]);
  }
  __syncwarp();
  mbar_wait(&bar[0], 0);
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t laddr = tbase + (static_cast<uint32_t>(warp * 32) << 16);
  for (int c0 = 0; c0 < NQ; c0 += 8) {
    float s[8], o[8];
    tmem_ld_32x32b<8>(laddr + c0, s);
    tmem_ld_32x32b<8>(laddr + 64 + c0, o);
    tmem_wait_ld();
    for (int c = 0; c < 8; ++c) {
      s_out[(warp * 32 + lane) * NQ + c0 + c] = s[c];
      o_out[(warp * 32 + lane) * NQ + c0 + c] = o[c];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tbase, 128);
  }
}

template <int N>
static cudaError_t launch_probe_n(const __nv_bfloat16* k, const __nv_bfloat16* q,
                                  const __nv_bfloat16* v, const __nv_bfloat16* p, float* s_out,
                                  float* o_out, cudaStream_t stream) {
  const int smem = 2 * kKvTileBytes + 2 * 64 * 256 + 64;
  cudaError_t e =
      cudaFuncSetAttribute(umma_probe_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  umma_probe_kernel<N><<<1, 128, smem, stream>>>(k, q, v, p, s_out, o_out);
  return cudaGetLastError();
}

cudaError_t launch_umma_probe(const __nv_bfloat16* k, const __nv_bfloat16* q,
                              const __nv_bfloat16* v, const __nv_bfloat16* p, int nq,
                              float* s_out, float* o_out, cudaStream_t stream) {
  switch (nq) {
    case 16: return launch_probe_n<16>(k, q, v, p, s_out, o_out, stream);
    case 32: return launch_probe_n<32>(k, q, v, p, s_out, o_out, stream);
    case 64: return launch_probe_n<64>(k, q, v, p, s_out, o_out, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rb
