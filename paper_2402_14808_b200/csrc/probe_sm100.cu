// Layout probe for the paged-context operands of the relay step (tests only):
// one CTA builds a 128-key K and V tile in the PagedKvCache block layout
// ([128 d][bs tokens] per block, paged_swizzle applied), Q and P in the
// K-major SW128 layout, and runs exactly the descriptors relay_step_kernel
// uses for context tiles:
//   S^T[128 keys x 32] = K (A, MN-major, Swizzle(2*bs)) . Q^T (B, K-major SW128)
//   O^T[128 d x 32]    = V^T (A, K-major, Swizzle(2*bs)) . P^T (B, K-major SW128)
#include "rb_common.cuh"

namespace rb {

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

}  // namespace rb
