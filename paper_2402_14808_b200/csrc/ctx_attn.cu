// Request-context attention over paged KV, with the relay fusion fused into
// the epilogue; plus the standalone relay-fusion kernel and the paged KV
// append used by the decode step.
//
// One kernel, three roles (selected by the arguments, not by a backend):
//  * context attention  -- `_context_attention` / causal `attention_with_lse`
//    (/root/reference/pkg/src/relayserve/attention.py:96-134,160-174):
//    query row t of request r attends context keys 0 .. c_r - m_r + t.
//  * relay              -- the same plus, in the epilogue, the LSE merge with
//    the system partial (o_sys, lse_sys) of the same (row, head)
//    (`relay_fusion`, attention.py:137-157), writing the fused output and
//    the fused LSE: the two partial outputs never make an extra HBM trip.
//  * naive baseline     -- a shared prefix segment (the system K/V, shared in
//    storage) read again by every request before its context: the
//    per-request `baseline_attention` (attention.py:266-296), i.e. the
//    "vLLM-PS" baseline the paper compares against.
//
// Memory-bound design (HBM roofline): grid = (request,
// kv head, row tile); 4 warps stride over 16-token chunks; a half-warp reads
// one 256-byte K (or V) row with 16 B per lane (128-bit coalesced loads,
// L1::no_allocate), dot products reduce with 4 xor-shuffles, online softmax
// in the log2 domain per half-warp, then an smem merge of the 8 partial
// states, the fusion, and one coalesced store per row.
#include "rb_common.cuh"
#include "rb_args.cuh"

namespace rb {



constexpr int kCtxThreads = 128;
constexpr int kChunk = 16;

__device__ __forceinline__ const __nv_bfloat16* ctx_row(const KvView& kv, const __nv_bfloat16* base,
                                                        int r, int t, int h) {
  long long off;
  if (kv.block_table != nullptr) {
    const int blk = __ldg(kv.block_table + static_cast<long long>(r) * kv.bt_stride + t / kv.block_size);
    off = static_cast<long long>(blk) * kv.stride_block +
          static_cast<long long>(t % kv.block_size) * kv.stride_tok;
  } else {
    off = (kv.req_offset[r] + t) * kv.stride_tok;
  }
  return base + off + h * kv.stride_head;
}

template <int R>
struct RowState {
  float m[R], l[R], acc[R][8];
};

// Process one 16-key chunk for a half-warp: keys key0 + 2p + hw, p = 0..7.
// `lim[i]` is the exclusive key bound of row i inside this segment.
template <int R>
__device__ __forceinline__ void chunk_update(RowState<R>& st, const float (&qf)[R][8],
                                             const uint4 (&kr)[8], const uint4 (&vr)[8],
                                             int key0, int hw, const int (&lim)[R], float scale_log2) {
  float x[R][8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    float kf[8];
    kf[0] = bf16_lo(kr[p].x); kf[1] = bf16_hi(kr[p].x);
    kf[2] = bf16_lo(kr[p].y); kf[3] = bf16_hi(kr[p].y);
    kf[4] = bf16_lo(kr[p].z); kf[5] = bf16_hi(kr[p].z);
    kf[6] = bf16_lo(kr[p].w); kf[7] = bf16_hi(kr[p].w);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) s = fmaf(qf[i][e], kf[e], s);
      x[i][p] = s;
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      float s = x[i][p];
      s += __shfl_xor_sync(0xffffffffu, s, 8);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      const int key = key0 + 2 * p + hw;
      x[i][p] = key < lim[i] ? s * scale_log2 : -INFINITY;
    }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    float cm = x[i][0];
#pragma unroll
    for (int p = 1; p < 8; ++p) cm = fmaxf(cm, x[i][p]);
    if (cm == -INFINITY) continue;  // no valid key of this row in this chunk half
    const float mn = fmaxf(st.m[i], cm);
    const float al = (st.m[i] == -INFINITY) ? 0.f : fast_exp2(st.m[i] - mn);
    st.m[i] = mn;
    float ps = 0.f;
    float a[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] = st.acc[i][e] * al;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const float pr = fast_exp2(x[i][p] - mn);
      ps += pr;
      a[0] = fmaf(pr, bf16_lo(vr[p].x), a[0]); a[1] = fmaf(pr, bf16_hi(vr[p].x), a[1]);
      a[2] = fmaf(pr, bf16_lo(vr[p].y), a[2]); a[3] = fmaf(pr, bf16_hi(vr[p].y), a[3]);
      a[4] = fmaf(pr, bf16_lo(vr[p].z), a[4]); a[5] = fmaf(pr, bf16_hi(vr[p].z), a[5]);
      a[6] = fmaf(pr, bf16_lo(vr[p].w), a[6]); a[7] = fmaf(pr, bf16_hi(vr[p].w), a[7]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) st.acc[i][e] = a[e];
    st.l[i] = st.l[i] * al + ps;
  }
}

template <int R>
__global__ void __launch_bounds__(kCtxThreads)
    ctx_attn_kernel(const CtxArgs a) {
  const int r = blockIdx.x;
  const int h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hw = lane >> 4, l16 = lane & 15;
  const int row0 = a.q_start[r];
  const int m_r = a.q_start[r + 1] - row0;
  const int nrows_total = m_r * a.g;          // (token, group) rows of this (r, h)
  const int rbase = blockIdx.z * R;           // first local row of this CTA
  if (rbase >= nrows_total) return;
  const int c_r = a.ctx_lens[r];

  // queries (fp32, 8 dims per lane) and per-row key limits
  float qf[R][8];
  int lim_ctx[R], lim_pre[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int li = rbase + i;
    if (li < nrows_total) {
      const int t = li / a.g, jj = li % a.g;
      const __nv_bfloat16* qp = a.q + static_cast<long long>(row0 + t) * a.q_row_stride +
                                static_cast<long long>(h * a.g + jj) * a.q_head_stride + l16 * 8;
      const uint4 u = *reinterpret_cast<const uint4*>(qp);
      qf[i][0] = bf16_lo(u.x); qf[i][1] = bf16_hi(u.x);
      qf[i][2] = bf16_lo(u.y); qf[i][3] = bf16_hi(u.y);
      qf[i][4] = bf16_lo(u.z); qf[i][5] = bf16_hi(u.z);
      qf[i][6] = bf16_lo(u.w); qf[i][7] = bf16_hi(u.w);
      lim_ctx[i] = a.causal ? c_r - m_r + t + 1 : c_r;
      lim_pre[i] = a.s_prefix;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) qf[i][e] = 0.f;
      lim_ctx[i] = 0;
      lim_pre[i] = 0;
    }
  }
  int max_lim = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) max_lim = max(max_lim, lim_ctx[i]);

  RowState<R> st;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    st.m[i] = -INFINITY;
    st.l[i] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) st.acc[i][e] = 0.f;
  }

  // ---- shared prefix segment (naive baseline only)
  if (a.s_prefix > 0) {
    const long long hoff = static_cast<long long>(h) * a.p_stride_head + l16 * 8;
    for (int c0 = warp * kChunk; c0 < a.s_prefix; c0 += 4 * kChunk) {
      uint4 kr[8], vr[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int t = min(c0 + 2 * p + hw, a.s_prefix - 1);
        kr[p] = ld_nc_v4(a.pk + static_cast<long long>(t) * a.p_stride_tok + hoff);
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int t = min(c0 + 2 * p + hw, a.s_prefix - 1);
        vr[p] = ld_nc_v4(a.pv + static_cast<long long>(t) * a.p_stride_tok + hoff);
      }
      chunk_update<R>(st, qf, kr, vr, c0, hw, lim_pre, a.scale_log2);
    }
  }
  // ---- request context segment (paged or ragged)
  for (int c0 = warp * kChunk; c0 < max_lim; c0 += 4 * kChunk) {
    uint4 kr[8], vr[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int t = min(c0 + 2 * p + hw, max_lim - 1);
      kr[p] = ld_nc_v4(ctx_row(a.ctx, a.ctx.k, r, t, h) + l16 * 8);
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int t = min(c0 + 2 * p + hw, max_lim - 1);
      vr[p] = ld_nc_v4(ctx_row(a.ctx, a.ctx.v, r, t, h) + l16 * 8);
    }
    chunk_update<R>(st, qf, kr, vr, c0, hw, lim_ctx, a.scale_log2);
  }

  // ---- merge the 8 (warp, half) partial states per row through smem
  __shared__ float s_acc[8][R][128];
  __shared__ float s_m[8][R], s_l[8][R];
  const int wh = warp * 2 + hw;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    *reinterpret_cast<float4*>(&s_acc[wh][i][l16 * 8]) =
        make_float4(st.acc[i][0], st.acc[i][1], st.acc[i][2], st.acc[i][3]);
    *reinterpret_cast<float4*>(&s_acc[wh][i][l16 * 8 + 4]) =
        make_float4(st.acc[i][4], st.acc[i][5], st.acc[i][6], st.acc[i][7]);
    if (l16 == 0) {
      s_m[wh][i] = st.m[i];
      s_l[wh][i] = st.l[i];
    }
  }
  __syncthreads();
  const int dcol = threadIdx.x;  // 128 threads = 128 head dims
#pragma unroll 1
  for (int i = 0; i < R; ++i) {
    const int li = rbase + i;
    if (li >= nrows_total) break;
    float M = -INFINITY;
#pragma unroll
    for (int k = 0; k < 8; ++k) M = fmaxf(M, s_m[k][i]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float w = (s_m[k][i] == -INFINITY) ? 0.f : fast_exp2(s_m[k][i] - M);
        L = fmaf(s_l[k][i], w, L);
        O = fmaf(s_acc[k][i][dcol], w, O);
      }
    }
    float o = (L > 0.f) ? O / L : 0.f;
    float lse2 = (L > 0.f) ? M + __log2f(L) : -INFINITY;
    const int t = li / a.g, jj = li % a.g;
    const long long oidx = static_cast<long long>(row0 + t) * a.hq + h * a.g + jj;
    if (a.o_sys != nullptr) {
      const float ls2 = a.lse_sys[oidx] * kLog2e;
      const float os = a.o_sys[oidx * 128 + dcol];
      const float mx = fmaxf(ls2, lse2);
      const float wc = (lse2 == -INFINITY) ? 0.f : fast_exp2(lse2 - mx);
      const float ws = (ls2 == -INFINITY) ? 0.f : fast_exp2(ls2 - mx);
      const float inv = 1.f / (wc + ws);
      o = (wc * o + ws * os) * inv;
      lse2 = mx + __log2f(wc + ws);
    }
    if (a.out_fp32)
      reinterpret_cast<float*>(a.out)[oidx * 128 + dcol] = o;
    else
      reinterpret_cast<__nv_bfloat16*>(a.out)[oidx * 128 + dcol] = __float2bfloat16_rn(o);
    if (a.lse_out != nullptr && dcol == 0) a.lse_out[oidx] = lse2 * kLn2;
  }
}

cudaError_t launch_context_attention(const CtxArgs& a, int max_rows, cudaStream_t stream) {
  // max_rows = max over requests of m_r * g
  int R = 1;
  if (max_rows >= 8) R = 8;
  else if (max_rows >= 4) R = 4;
  else if (max_rows >= 2) R = 2;
  dim3 grid(a.b, a.hkv, (max_rows + R - 1) / R);
  switch (R) {
    case 1: ctx_attn_kernel<1><<<grid, kCtxThreads, 0, stream>>>(a); break;
    case 2: ctx_attn_kernel<2><<<grid, kCtxThreads, 0, stream>>>(a); break;
    case 4: ctx_attn_kernel<4><<<grid, kCtxThreads, 0, stream>>>(a); break;
    default: ctx_attn_kernel<8><<<grid, kCtxThreads, 0, stream>>>(a); break;
  }
  return cudaGetLastError();
}

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
// slot_mapping[t] = block_id * block_size + offset (kvcache.py:207-235).
__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ k_new,
                                 const __nv_bfloat16* __restrict__ v_new,
                                 const int* __restrict__ slots, __nv_bfloat16* k_pool,
                                 __nv_bfloat16* v_pool, int n_tok, int hkv, int block_size,
                                 long long stride_block, long long stride_tok,
                                 long long stride_head) {
  const int t = blockIdx.x;
  const int slot = slots[t];
  const int blk = slot / block_size, off = slot % block_size;
  for (int idx = threadIdx.x; idx < hkv * 16; idx += blockDim.x) {
    const int h = idx / 16, c = idx % 16;
    const long long src = (static_cast<long long>(t) * hkv + h) * 128 + c * 8;
    const long long dst = blk * stride_block + off * stride_tok + h * stride_head + c * 8;
    *reinterpret_cast<uint4*>(k_pool + dst) = *reinterpret_cast<const uint4*>(k_new + src);
    *reinterpret_cast<uint4*>(v_pool + dst) = *reinterpret_cast<const uint4*>(v_new + src);
  }
}

cudaError_t launch_kv_append(const __nv_bfloat16* k_new, const __nv_bfloat16* v_new,
                             const int* slots, __nv_bfloat16* k_pool, __nv_bfloat16* v_pool,
                             int n_tok, int hkv, int block_size, long long stride_block,
                             long long stride_tok, long long stride_head, cudaStream_t stream) {
  if (n_tok == 0) return cudaSuccess;
  kv_append_kernel<<<n_tok, 128, 0, stream>>>(k_new, v_new, slots, k_pool, v_pool, n_tok, hkv,
                                              block_size, stride_block, stride_tok, stride_head);
  return cudaGetLastError();
}

}  // namespace rb
