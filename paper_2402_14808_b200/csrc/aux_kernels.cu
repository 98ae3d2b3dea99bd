// Small kernels around the relay step: the standalone relay fusion and the
// paged KV append.
#include "rb_common.cuh"
#include "rb_plan.h"

namespace rb {

// ----------------------------------------------------------- relay fusion
// Standalone LSE merge of two segment results (attention.py:137-157), fp32.
// out = w_s * o_sys + w_c * o_ctx with max-subtracted weights (no overflow at
// |lse gap| > 88); lse_out = logaddexp(lse_sys, lse_ctx).
__global__ void relay_fusion_kernel(const float* __restrict__ o_sys, const float* __restrict__ lse_sys,
                                    const float* __restrict__ o_ctx, const float* __restrict__ lse_ctx,
                                    float* __restrict__ out, float* __restrict__ lse_out,
                                    long long n_vec, int d) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n_vec * d) return;
  const long long vi = idx / d;
  const float ls = lse_sys[vi], lc = lse_ctx[vi];
  const float mx = fmaxf(ls, lc);
  const float ws = __expf(ls - mx), wc = __expf(lc - mx);
  const float inv = 1.f / (ws + wc);
  out[idx] = (ws * o_sys[idx] + wc * o_ctx[idx]) * inv;
  if (lse_out != nullptr && idx % d == 0) lse_out[vi] = mx + __logf(ws + wc);
}

cudaError_t launch_relay_fusion(const float* o_sys, const float* lse_sys, const float* o_ctx,
                                const float* lse_ctx, float* out, float* lse_out, long long n_vec,
                                int d, cudaStream_t stream) {
  const long long n = n_vec * d;
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  relay_fusion_kernel<<<static_cast<unsigned>((n + threads - 1) / threads), threads, 0, stream>>>(
      o_sys, lse_sys, o_ctx, lse_ctx, out, lse_out, n_vec, d);
  return cudaGetLastError();
}

// ----------------------------------------------------------- paged append
// Write n_tok new (k, v) rows [n_tok][hkv][128] into the pool at
// slot_mapping[t] = block_id * bs + offset (kvcache.py:207-235).  A pool block
// of one kv head is [128 d][bs tokens] with paged_swizzle applied (the UMMA
// operand layout the relay step copies verbatim), so token `offset` of dim d
// lands at byte paged_swizzle(d * 2bs + offset * 2).  One thread per
// (token, head, dim) of K and V; reads are coalesced over d.
__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ k_new,
                                 const __nv_bfloat16* __restrict__ v_new,
                                 const int* __restrict__ slots, unsigned char* k_pool,
                                 unsigned char* v_pool, int n_tok, int hkv, int bs,
                                 long long block_bytes, long long head_bytes) {
  const long long n = static_cast<long long>(n_tok) * hkv * RB_HEAD_DIM;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= 2 * n) return;
  const bool is_v = idx >= n;
  const long long e = is_v ? idx - n : idx;
  const int d = static_cast<int>(e % RB_HEAD_DIM);
  const int h = static_cast<int>((e / RB_HEAD_DIM) % hkv);
  const int t = static_cast<int>(e / (RB_HEAD_DIM * hkv));
  const int slot = __ldg(slots + t);
  const int blk = slot / bs, off = slot % bs;
  const uint32_t rb = 2 * bs;
  const long long dst = blk * block_bytes + h * head_bytes + paged_swizzle(d * rb + off * 2, rb);
  const __nv_bfloat16 val = is_v ? v_new[e] : k_new[e];
  *reinterpret_cast<__nv_bfloat16*>((is_v ? v_pool : k_pool) + dst) = val;
}

cudaError_t launch_kv_append(const __nv_bfloat16* k_new, const __nv_bfloat16* v_new,
                             const int* slots, void* k_pool, void* v_pool, int n_tok, int hkv,
                             int bs, long long block_bytes, long long head_bytes,
                             cudaStream_t stream) {
  if (n_tok == 0) return cudaSuccess;
  const long long total = 2LL * n_tok * hkv * RB_HEAD_DIM;
  const int threads = 256;
  kv_append_kernel<<<static_cast<unsigned>((total + threads - 1) / threads), threads, 0, stream>>>(
      k_new, v_new, slots, static_cast<unsigned char*>(k_pool), static_cast<unsigned char*>(v_pool),
      n_tok, hkv, bs, block_bytes, head_bytes);
  return cudaGetLastError();
}

}  // namespace rb
