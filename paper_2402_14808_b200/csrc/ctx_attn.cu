// Request-context attention over paged KV (the context segment of the relay
// decode step), the relay fusion, and the paged KV append.
//
// One kernel (ctx_cta_kernel), three roles selected by the arguments:
//  * context attention  -- `_context_attention` / causal `attention_with_lse`
//    (/root/reference/pkg/src/relayserve/attention.py:96-134,160-174):
//    query row t of request r attends context keys 0 .. c_r - m_r + t;
//    optionally fused with a given system partial (o_sys, lse_sys):
//    `relay_fusion` (attention.py:137-157) in the epilogue.
//  * relay              -- inside rb_relay_attention, concurrently with the
//    system kernel on other SMs: each (row, head) state is merged with the
//    system kernel's stream-K parts of its unit (`relay_fusion`,
//    attention.py:137-157) as soon as the unit is published; rows whose
//    unit is not yet complete are fused at the end of the CTA.
//  * naive baseline     -- a shared prefix segment (the system K/V, shared in
//    storage) read again by every request before its context: the
//    per-request `baseline_attention` (attention.py:266-296), i.e. the
//    "vLLM-PS" baseline the paper compares against.
//
// Memory-bound design (HBM roofline).  Work item =
// (request, kv head, row tile of up to R query rows); items are claimed
// dynamically by persistent CTAs (2 per SM).  Per CTA: a scheduler warp
// publishes items (geometry, block-table entries, query rows) in a smem
// queue; 4 worker warps split each item's 16-token chunks (K 4 KB + V 4 KB
// per chunk, streamed with cp.async through per-warp 3-slot rings -- the LSU
// path sustains HBM rate on scattered 4 KB paged blocks where the bulk-copy
// engine manages ~19 GB/s per SM, profiles/microbench_scatter.cu) and run
// QK^T / PV on the tensor cores with mma.sync (16 query rows x 16 keys per
// chunk); a merger warp combines the 4 partial states and writes the result.
#include <type_traits>

#include "rb_common.cuh"
#include "rb_args.cuh"

namespace rb {

constexpr int kChunk = 16;                       // tokens per chunk
constexpr int kRowBytes = RB_HEAD_DIM * 2;       // 256 B per key row
constexpr int kSlotBytes = 2 * kChunk * kRowBytes;  // K + V of one chunk: 8 KB

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


// Work item = (request r, kv head h, row tile z).  Geometry of one item.
template <int R>
struct CtxItem {
  int r, h, z, row0, m_r, nrows, c_r, max_lim, n_chunks;
  long long roff;  // ragged mode: first token of request r
};

// Issue the cp.async copies of one 16-token chunk (rows 0 .. n-1 of K at kb
// and V at vb, row stride tok_stride elements) into an 8 KB slot [K|V][16
// rows][256 B] whose 16-byte columns are XOR-swizzled by (row & 7), so the
// ldmatrix reads of the MMA path are bank-conflict free.  Lane (row0 = lane
// / 16, c16 = lane % 16) copies 16 B of rows row0 + 2i; rows >= n are
// zero-filled (never stale: their probabilities are 0 but 0 * NaN is not).
__device__ __forceinline__ uint32_t slot_off(int row, int c16) {
  return static_cast<uint32_t>(row * kRowBytes + ((c16 ^ (row & 7)) << 4));
}
__device__ __forceinline__ void chunk_cp_async(uint8_t* slot, const __nv_bfloat16* kb,
                                               const __nv_bfloat16* vb, long long tok_stride, int n,
                                               int lane) {
  const int row0 = lane >> 4, c16 = lane & 15;
  // row = row0 + 2i, (row & 7) = row0 | (2i & 6): swizzled column c16 ^ row0 ^ (2i & 6)
  const int cx = c16 ^ row0;
  uint8_t* d = slot + row0 * kRowBytes;
  const char* ks = reinterpret_cast<const char*>(kb + row0 * tok_stride + c16 * 8);
  const char* vs = reinterpret_cast<const char*>(vb + row0 * tok_stride + c16 * 8);
  const long long st2 = 4 * tok_stride;  // bytes between rows row and row + 2
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool ok = row0 + 2 * i < n;
    const uint32_t off = i * 2 * kRowBytes + ((cx ^ ((2 * i) & 6)) << 4);
    cp_async_16(d + off, ok ? ks + i * st2 : ks, ok ? 16u : 0u);
    cp_async_16(d + kChunk * kRowBytes + off, ok ? vs + i * st2 : vs, ok ? 16u : 0u);
  }
}

// Cold path of the chunk copy (blocks not a multiple of 16 tokens, or other
// row layouts): per-row addresses through the block table.  Out of line so
// the hot loop stays small (instruction-cache resident).
__device__ __noinline__ void chunk_cp_async_rows(uint8_t* dst, KvView kv, int r, int t0, int h, int n,
                                                 int lane) {
  const int row0 = lane >> 4, c16 = lane & 15;
  for (int i = 0; i < 8; ++i) {
    const int row = row0 + 2 * i;
    const bool ok = row < n;
    const __nv_bfloat16* ks = ok ? ctx_row(kv, kv.k, r, t0 + row, h) : kv.k;
    const __nv_bfloat16* vs = ok ? ctx_row(kv, kv.v, r, t0 + row, h) : kv.v;
    const uint32_t so = slot_off(row, c16);
    cp_async_16(dst + so, ks + c16 * 8, ok ? 16u : 0u);
    cp_async_16(dst + kChunk * kRowBytes + so, vs + c16 * 8, ok ? 16u : 0u);
  }
}

// Tensor-core (mma.sync m16n8k16) update of one 16-key chunk for up to 16
// query rows: S = Q K^T (2 n-tiles x 8 k-steps), online softmax in the log2
// domain on the accumulator fragments, O += P V (16 n-tiles).  Lane (g =
// lane / 4, t = lane % 4) holds rows g and g + 8.  lim0 / lim1: exclusive key
// bounds (segment-relative) of those rows; key0: this chunk's first key.
// mask = false: every key of the chunk is valid for every valid row (rows
// past the item's rows compute harmless values that are never written).
// Lazy rescale: the running max moves only when a score exceeds it by more
// than kCtxTau (log2 units), so O is rescaled rarely; p <= 2^kCtxTau.
constexpr float kCtxTau = 8.f;
struct MmaRowState {
  float o[16][4];
  float m[2], l[2];
};

__device__ __forceinline__ void chunk_mma(MmaRowState& st, const uint32_t (&qa)[8][4], uint32_t slot,
                                          int lane, int key0, int lim0, int lim1, float scale_log2,
                                          bool mask) {
  const int mi = lane >> 3, rr = lane & 7, t = lane & 3;
  float s[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) s[nt][e] = 0.f;
  {
    const int key = (mi >> 1) * 8 + rr;
    const uint32_t kaddr = slot + key * kRowBytes;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t b[4];
      ldsm_x4(b, kaddr + (((ks * 2 + (mi & 1)) ^ (key & 7)) << 4));
      mma_bf16_16816(s[0], qa[ks], b[0], b[1]);
      mma_bf16_16816(s[1], qa[ks], b[2], b[3]);
    }
  }
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int key = key0 + nt * 8 + 2 * t + e;
      s[nt][e] = (!mask || key < lim0) ? s[nt][e] * scale_log2 : -INFINITY;
      s[nt][2 + e] = (!mask || key < lim1) ? s[nt][2 + e] * scale_log2 : -INFINITY;
      mx0 = fmaxf(mx0, s[nt][e]);
      mx1 = fmaxf(mx1, s[nt][2 + e]);
    }
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
  // lazy max: keep the reference unless the chunk exceeds it by > kCtxTau
  const float mn0 = (mx0 > st.m[0] + kCtxTau) ? mx0 : st.m[0];
  const float mn1 = (mx1 > st.m[1] + kCtxTau) ? mx1 : st.m[1];
  const float b0 = (mn0 == -INFINITY) ? 0.f : mn0, b1 = (mn1 == -INFINITY) ? 0.f : mn1;
  float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      s[nt][e] = fast_exp2(s[nt][e] - b0);
      s[nt][2 + e] = fast_exp2(s[nt][2 + e] - b1);
      sum0 += s[nt][e];
      sum1 += s[nt][2 + e];
    }
  sum0 += __shfl_xor_sync(0xffffffffu, sum0, 1);
  sum1 += __shfl_xor_sync(0xffffffffu, sum1, 1);
  sum0 += __shfl_xor_sync(0xffffffffu, sum0, 2);
  sum1 += __shfl_xor_sync(0xffffffffu, sum1, 2);
  if (mn0 != st.m[0] || mn1 != st.m[1]) {
    const float al0 = (st.m[0] == -INFINITY) ? 0.f : fast_exp2(st.m[0] - mn0);
    const float al1 = (st.m[1] == -INFINITY) ? 0.f : fast_exp2(st.m[1] - mn1);
    st.l[0] *= al0;
    st.l[1] *= al1;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      st.o[nt][0] *= al0;
      st.o[nt][1] *= al0;
      st.o[nt][2] *= al1;
      st.o[nt][3] *= al1;
    }
    st.m[0] = mn0;
    st.m[1] = mn1;
  }
  st.l[0] += sum0;
  st.l[1] += sum1;
  const uint32_t pa[4] = {pack_bf16x2(s[0][0], s[0][1]), pack_bf16x2(s[0][2], s[0][3]),
                          pack_bf16x2(s[1][0], s[1][1]), pack_bf16x2(s[1][2], s[1][3])};
  {
    const int key = (mi & 1) * 8 + rr;
    const uint32_t vaddr = slot + kChunk * kRowBytes + key * kRowBytes;
#pragma unroll
    for (int dp = 0; dp < 8; ++dp) {
      uint32_t b[4];
      ldsm_x4_trans(b, vaddr + (((dp * 2 + (mi >> 1)) ^ (key & 7)) << 4));
      mma_bf16_16816(st.o[2 * dp], pa, b[0], b[1]);
      mma_bf16_16816(st.o[2 * dp + 1], pa, b[2], b[3]);
    }
  }
}

template <int R>
struct RowState {
  float m[R], l[R], acc[R][8];
};

// CUDA-core update of one 16-key chunk for a half-warp (R <= 2 query rows,
// where 16-row MMA tiles would be mostly padding): keys key0 + 2p + hw,
// p = 0..7, K/V rows already in registers; dot products reduce with 4
// xor-shuffles, online softmax in the log2 domain.  `lim[i]` is the exclusive key bound of row i inside
// this segment; keys at or past it contribute nothing (their V rows may hold
// stale data and are zeroed, never multiplied).
template <int R>
__device__ __forceinline__ void chunk_update(RowState<R>& st, const float (&qf)[R][8],
                                             const uint4 (&kr)[8], uint4 (&vr)[8],
                                             int key0, int hw, const int (&lim)[R], float scale_log2,
                                             int max_lim) {
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
      // packed pairs: 4 FFMA2 + 1 FADD instead of 8 FFMA
      float2 s2 = make_float2(qf[i][0] * kf[0], qf[i][1] * kf[1]);
#pragma unroll
      for (int e = 2; e < 8; e += 2)
        s2 = ffma2(make_float2(qf[i][e], qf[i][e + 1]), make_float2(kf[e], kf[e + 1]), s2);
      x[i][p] = s2.x + s2.y;
    }
    if (key0 + 2 * p + hw >= max_lim) vr[p] = make_uint4(0, 0, 0, 0);
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
      const float2 pp = make_float2(pr, pr);
      float2 a01 = ffma2(pp, make_float2(bf16_lo(vr[p].x), bf16_hi(vr[p].x)), make_float2(a[0], a[1]));
      float2 a23 = ffma2(pp, make_float2(bf16_lo(vr[p].y), bf16_hi(vr[p].y)), make_float2(a[2], a[3]));
      float2 a45 = ffma2(pp, make_float2(bf16_lo(vr[p].z), bf16_hi(vr[p].z)), make_float2(a[4], a[5]));
      float2 a67 = ffma2(pp, make_float2(bf16_lo(vr[p].w), bf16_hi(vr[p].w)), make_float2(a[6], a[7]));
      a[0] = a01.x; a[1] = a01.y; a[2] = a23.x; a[3] = a23.y;
      a[4] = a45.x; a[5] = a45.y; a[6] = a67.x; a[7] = a67.y;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) st.acc[i][e] = a[e];
    st.l[i] = st.l[i] * al + ps;
  }
}


// Per-worker compute policies of ctx_cta_kernel: same interface, chosen by
// the rows per item.  R <= 2 (decode): CUDA cores, a half-warp per key pair
// (no padded MMA rows).  R >= 4: mma.sync tiles of 16 query rows.
template <int R>
struct SimtCompute {
  float qf[R][8];
  int lim_ctx[R], lim_pre[R];
  RowState<R> st;

  __device__ __forceinline__ void load(const uint8_t* qrows, const uint8_t* /*qzero*/,
                                       const CtxItem<R>& it, int item, const CtxArgs& a, int lane) {
    const int l16 = lane & 15, rbase = it.z * R;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int li = rbase + i;
      const bool ok = item >= 0 && it.n_chunks > 0 && li < it.nrows;
      if (ok) {
        const uint4 u = *reinterpret_cast<const uint4*>(qrows + i * kRowBytes + l16 * 16);
        qf[i][0] = bf16_lo(u.x); qf[i][1] = bf16_hi(u.x);
        qf[i][2] = bf16_lo(u.y); qf[i][3] = bf16_hi(u.y);
        qf[i][4] = bf16_lo(u.z); qf[i][5] = bf16_hi(u.z);
        qf[i][6] = bf16_lo(u.w); qf[i][7] = bf16_hi(u.w);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) qf[i][e] = 0.f;
      }
      lim_ctx[i] = ok ? (a.causal ? it.c_r - it.m_r + li / a.g + 1 : it.c_r) : 0;
      lim_pre[i] = ok ? a.s_prefix : 0;
    }
  }
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      st.m[i] = -INFINITY;
      st.l[i] = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) st.acc[i][e] = 0.f;
    }
  }
  __device__ __forceinline__ void chunk(const uint8_t* slot, int key0, bool pre, int max_lim,
                                        bool /*mask*/, const CtxArgs& a, int lane) {
    const int hw = lane >> 4, l16 = lane & 15;
    uint4 kr[8], vr[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const uint32_t off = slot_off(2 * p + hw, l16);
      kr[p] = *reinterpret_cast<const uint4*>(slot + off);
      vr[p] = *reinterpret_cast<const uint4*>(slot + kChunk * kRowBytes + off);
    }
    chunk_update<R>(st, qf, kr, vr, key0, hw, pre ? lim_pre : lim_ctx, a.scale_log2,
                    pre ? a.s_prefix : max_lim);
  }
  // fold the two half-warp states, then half-warp 0 writes rows < R
  __device__ __forceinline__ void handoff(float* macc, float* mml, int lane) {
    const int hw = lane >> 4, l16 = lane & 15;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const float mo = __shfl_xor_sync(0xffffffffu, st.m[i], 16);
      const float lo = __shfl_xor_sync(0xffffffffu, st.l[i], 16);
      const float M = fmaxf(st.m[i], mo);
      const float ws = (st.m[i] == -INFINITY) ? 0.f : fast_exp2(st.m[i] - M);
      const float wo = (mo == -INFINITY) ? 0.f : fast_exp2(mo - M);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float ao = __shfl_xor_sync(0xffffffffu, st.acc[i][e], 16);
        st.acc[i][e] = st.acc[i][e] * ws + ao * wo;
      }
      const float L = st.l[i] * ws + lo * wo;
      if (hw == 0) {
        *reinterpret_cast<float4*>(macc + i * 128 + l16 * 8) =
            make_float4(st.acc[i][0], st.acc[i][1], st.acc[i][2], st.acc[i][3]);
        *reinterpret_cast<float4*>(macc + i * 128 + l16 * 8 + 4) =
            make_float4(st.acc[i][4], st.acc[i][5], st.acc[i][6], st.acc[i][7]);
        if (l16 == 0) {
          mml[i * 2] = M;
          mml[i * 2 + 1] = L;
        }
      }
    }
  }
};

template <int R>
struct MmaCompute {
  uint32_t qa[8][4];
  int lim_ctx[2], lim_pre[2];
  MmaRowState st;

  __device__ __forceinline__ void load(const uint8_t* qrows, const uint8_t* qzero,
                                       const CtxItem<R>& it, int item, const CtxArgs& a, int lane) {
    // Q rows as MMA A fragments (rows past R read the zero row)
    const int qrow = (lane & 7) + ((lane >> 3) & 1) * 8;
    const uint32_t qaddr = qrow < R ? smem_u32(qrows + qrow * kRowBytes) : smem_u32(qzero);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) ldsm_x4(qa[ks], qaddr + ((ks * 2 + (lane >> 4)) << 4));
    const int g8 = lane >> 2, rbase = it.z * R;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int rr = g8 + 8 * hr, li = rbase + rr;
      const bool ok = item >= 0 && it.n_chunks > 0 && rr < R && li < it.nrows;
      lim_ctx[hr] = ok ? (a.causal ? it.c_r - it.m_r + li / a.g + 1 : it.c_r) : 0;
      lim_pre[hr] = ok ? a.s_prefix : 0;
    }
  }
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) st.o[nt][e] = 0.f;
    st.m[0] = st.m[1] = -INFINITY;
    st.l[0] = st.l[1] = 0.f;
  }
  __device__ __forceinline__ void chunk(const uint8_t* slot, int key0, bool pre, int /*max_lim*/,
                                        bool mask, const CtxArgs& a, int lane) {
    chunk_mma(st, qa, smem_u32(slot), lane, key0, pre ? lim_pre[0] : lim_ctx[0],
              pre ? lim_pre[1] : lim_ctx[1], a.scale_log2, mask);
  }
  __device__ __forceinline__ void handoff(float* macc, float* mml, int lane) {
    const int g8 = lane >> 2, tq = lane & 3;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int rr = g8 + 8 * hr;
      if (rr < R) {
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
          *reinterpret_cast<float2*>(macc + rr * 128 + nt * 8 + 2 * tq) =
              make_float2(st.o[nt][2 * hr], st.o[nt][2 * hr + 1]);
        if (tq == 0) {
          mml[rr * 2] = st.m[hr];
          mml[rr * 2 + 1] = st.l[hr];
        }
      }
    }
  }
};

template <int R>
using CtxCompute = typename std::conditional<(R <= 2), SimtCompute<R>, MmaCompute<R>>::type;

// Relay fusion of one (row, head) pair (`relay_fusion`, attention.py:137-157):
// the context state (O unnormalised, m log2, l) merged with every stream-K
// part of the pair's system unit in slot order (deterministic), normalised
// and written.  One warp, lane = 4 head dims.  The unit must be published.
// Split in two so the merger can issue the first parts' loads before it
// waits for the workers (RelayParts carries them in registers).
struct RelayParts {
  long long base;
  int np, col;
  float mk[4], lk[4];
  float4 ak[4];
};

__device__ __forceinline__ void relay_parts_load(const rb_sys_plan& SP, const float* part_acc,
                                                 const float* part_ml, long long base, int np,
                                                 int col, int k0, int lane, float* mk, float* lk,
                                                 float4* ak) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int k = min(k0 + kk, np - 1);
    const float* pml = part_ml + (base + k) * 2 * SP.nq;
    mk[kk] = __ldcg(pml + col);
    lk[kk] = __ldcg(pml + SP.nq + col);
    ak[kk] = __ldcg(reinterpret_cast<const float4*>(part_acc + ((base + k) * SP.nq + col) * RB_HEAD_DIM + lane * 4));
  }
}

__device__ __forceinline__ RelayParts relay_parts_begin(const rb_sys_plan& SP, int hq, long long pair,
                                                        const float* part_acc, const float* part_ml,
                                                        int lane) {
  RelayParts P;
  const int row = static_cast<int>(pair / hq), hh = static_cast<int>(pair % hq);
  const long long f = static_cast<long long>(row) * SP.g + hh % SP.g;
  const int qt = static_cast<int>(f / SP.nq);
  P.col = static_cast<int>(f % SP.nq);
  const int u = (hh / SP.g) * SP.n_qt + qt;
  P.np = rb_unit_parts(&SP, u);
  P.base = static_cast<long long>(u) * SP.max_parts;
  relay_parts_load(SP, part_acc, part_ml, P.base, P.np, P.col, 0, lane, P.mk, P.lk, P.ak);
  return P;
}

__device__ __forceinline__ void relay_fuse_finish(const rb_sys_plan& SP, RelayParts& P, long long pair,
                                                  const float* part_acc, const float* part_ml,
                                                  float4 O, float mt, float lt, void* out, int out_fp32,
                                                  float* lse_out, int lane) {
  const int d0 = lane * 4;
  for (int k0 = 0; k0 < P.np; k0 += 4) {
    if (k0 > 0) relay_parts_load(SP, part_acc, part_ml, P.base, P.np, P.col, k0, lane, P.mk, P.lk, P.ak);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      if (k0 + kk >= P.np) break;
      const float mn = fmaxf(mt, P.mk[kk]);
      const float so = (mt == -INFINITY) ? 0.f : fast_exp2(mt - mn);
      const float sk = fast_exp2(P.mk[kk] - mn);
      lt = lt * so + P.lk[kk] * sk;
      O.x = O.x * so + P.ak[kk].x * sk;
      O.y = O.y * so + P.ak[kk].y * sk;
      O.z = O.z * so + P.ak[kk].z * sk;
      O.w = O.w * so + P.ak[kk].w * sk;
      mt = mn;
    }
  }
  const float inv = 1.f / lt;
  if (out_fp32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + pair * 128 + d0) =
        make_float4(O.x * inv, O.y * inv, O.z * inv, O.w * inv);
  } else {
    uint2 pk;
    pk.x = pack_bf16x2(O.x * inv, O.y * inv);
    pk.y = pack_bf16x2(O.z * inv, O.w * inv);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + pair * 128 + d0) = pk;
  }
  if (lse_out != nullptr && lane == 0) lse_out[pair] = (mt + __log2f(lt)) * kLn2;
}

__device__ __forceinline__ void relay_fuse_pair(const rb_sys_plan& SP, int hq, long long pair,
                                                const float* part_acc, const float* part_ml,
                                                float4 O, float mt, float lt, void* out, int out_fp32,
                                                float* lse_out, int lane) {
  RelayParts P = relay_parts_begin(SP, hq, pair, part_acc, part_ml, lane);
  relay_fuse_finish(SP, P, pair, part_acc, part_ml, O, mt, lt, out, out_fp32, lse_out, lane);
}

// Is the system unit of `pair` published (all its parts written)?  Lane 0
// probes with acquire semantics; the answer is broadcast to the warp.
__device__ __forceinline__ bool relay_unit_ready(const rb_sys_plan& SP, int hq, long long pair,
                                                 const int* ready, int lane, bool block) {
  const int row = static_cast<int>(pair / hq), hh = static_cast<int>(pair % hq);
  const long long f = static_cast<long long>(row) * SP.g + hh % SP.g;
  const int u = (hh / SP.g) * SP.n_qt + static_cast<int>(f / SP.nq);
  const int np = rb_unit_parts(&SP, u);
  int ok = 1;
  if (lane == 0) {
    ok = ld_acquire_gpu(ready + u) >= np;
    while (!ok && block) {
      __nanosleep(128);
      ok = ld_acquire_gpu(ready + u) >= np;
    }
  }
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// Is the system unit of `pair` in the merger's bitmask of published units?
__device__ __forceinline__ bool relay_unit_published(const rb_sys_plan& SP, int hq, long long pair,
                                                     unsigned long long pub) {
  const int row = static_cast<int>(pair / hq), hh = static_cast<int>(pair % hq);
  const long long f = static_cast<long long>(row) * SP.g + hh % SP.g;
  const int u = (hh / SP.g) * SP.n_qt + static_cast<int>(f / SP.nq);
  return (pub >> u) & 1;
}

constexpr int kWorkers = 4;
constexpr int kDepth = 3;                      // chunks in flight per worker
static_assert(kDepth == 3, "wait_group ladder in ctx_cta_kernel assumes 3");
constexpr int kIQ = 3;                         // item queue depth (claim-ahead bound)
constexpr int kNB = 3;                         // merge buffers
constexpr int kCtxThreadsPC = 32 * (2 + kWorkers);  // scheduler + workers + merger
constexpr int kMergerWarp = 1 + kWorkers;
constexpr int kPartStride = 132;               // floats per relay context partial: O[128], m, l
constexpr int kMaxDefer = 62;                  // relay rows per CTA awaiting their system unit

// Relay fusion of a parked pair (the end phase): 8 lanes per pair, lane
// sub = lane & 7 owning head dims [16 sub, 16 sub + 16), so one warp fuses
// four pairs with all their loads in flight at once.  Waits for the pair's
// system unit; same merge order and arithmetic as relay_fuse_pair.
__device__ __forceinline__ void relay_fuse_parked8(const rb_sys_plan& SP, int hq, long long pair,
                                                   bool valid, const int* ready, const float* ctx_part,
                                                   const float* part_acc, const float* part_ml,
                                                   void* out, int out_fp32, float* lse_out, int lane) {
  const int sub = lane & 7;
  int u = 0, col = 0, np = 0;
  if (valid) {
    const int row = static_cast<int>(pair / hq), hh = static_cast<int>(pair % hq);
    const long long f = static_cast<long long>(row) * SP.g + hh % SP.g;
    col = static_cast<int>(f % SP.nq);
    u = (hh / SP.g) * SP.n_qt + static_cast<int>(f / SP.nq);
    np = rb_unit_parts(&SP, u);
    if (sub == 0)
      while (ld_acquire_gpu(ready + u) < np) __nanosleep(64);
  }
  __syncwarp();
  if (!valid) return;
  const int d0 = sub * 16;
  const float* cp = ctx_part + pair * kPartStride;
  float4 O[4];
#pragma unroll
  for (int v = 0; v < 4; ++v) O[v] = __ldcg(reinterpret_cast<const float4*>(cp + d0 + 4 * v));
  const float2 ml = __ldcg(reinterpret_cast<const float2*>(cp + 128));
  float mt = ml.x, lt = ml.y;
  const long long base = static_cast<long long>(u) * SP.max_parts;
  for (int k = 0; k < np; ++k) {  // the first part's loads fly with the context part's
    const float* pml = part_ml + (base + k) * 2 * SP.nq;
    const float mk = __ldcg(pml + col), lk = __ldcg(pml + SP.nq + col);
    const float* pa = part_acc + ((base + k) * SP.nq + col) * RB_HEAD_DIM + d0;
    float4 ak[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) ak[v] = __ldcg(reinterpret_cast<const float4*>(pa + 4 * v));
    const float mn = fmaxf(mt, mk);
    const float so = (mt == -INFINITY) ? 0.f : fast_exp2(mt - mn);
    const float sk = fast_exp2(mk - mn);
    lt = lt * so + lk * sk;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      O[v].x = O[v].x * so + ak[v].x * sk;
      O[v].y = O[v].y * so + ak[v].y * sk;
      O[v].z = O[v].z * so + ak[v].z * sk;
      O[v].w = O[v].w * so + ak[v].w * sk;
    }
    mt = mn;
  }
  const float inv = 1.f / lt;
  if (out_fp32) {
    float* o = reinterpret_cast<float*>(out) + pair * 128 + d0;
#pragma unroll
    for (int v = 0; v < 4; ++v)
      reinterpret_cast<float4*>(o)[v] = make_float4(O[v].x * inv, O[v].y * inv, O[v].z * inv, O[v].w * inv);
  } else {
    uint4 pk[2];
    uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      w[2 * v] = pack_bf16x2(O[v].x * inv, O[v].y * inv);
      w[2 * v + 1] = pack_bf16x2(O[v].z * inv, O[v].w * inv);
    }
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + pair * 128 + d0);
    o[0] = pk[0];
    o[1] = pk[1];
  }
  if (lse_out != nullptr && sub == 0) lse_out[pair] = (mt + __log2f(lt)) * kLn2;
}


template <int R>
struct ItemSlot {
  CtxItem<R> it;
  int item;                                    // -1: no more work
  int bt[32];                                  // block ids of context blocks 0..31
};

template <int R>
struct CtaSmem {
  // [kIQ][R][128] bf16 query rows, then one zero row (MMA rows past R)
  static constexpr int kOffQ = kWorkers * kDepth * kSlotBytes;
  static constexpr int kOffQZero = kOffQ + kIQ * R * kRowBytes;
  static constexpr int kOffAcc = kOffQZero + kRowBytes;                  // [kNB][kWorkers][R][128] f32
  static constexpr int kOffML = kOffAcc + kNB * kWorkers * R * 128 * 4;  // [kNB][kWorkers][R][2]
  static constexpr int kOffMIt = (kOffML + kNB * kWorkers * R * 8 + 15) & ~15;  // [kNB] CtxItem
  static constexpr int kOffItems =
      (kOffMIt + kNB * static_cast<int>(sizeof(CtxItem<R>)) + 15) & ~15;  // [kIQ] ItemSlot
  static constexpr int kOffBar = (kOffItems + kIQ * static_cast<int>(sizeof(ItemSlot<R>)) + 7) & ~7;
  static constexpr int kOffDefer = kOffBar + (3 * kIQ + 2 * kNB) * 8;  // [1 + kMaxDefer] int
  static constexpr int kBytes = kOffDefer + (1 + kMaxDefer) * 4;
};

template <int R>
__global__ void __launch_bounds__(kCtxThreadsPC, 2)
    ctx_cta_kernel(const CtxArgs a, int n_items, int n_z) {
  using SM = CtaSmem<R>;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_pre = (a.s_prefix + kChunk - 1) / kChunk;
  float* s_acc = reinterpret_cast<float*>(smem + SM::kOffAcc);
  float* s_ml = reinterpret_cast<float*>(smem + SM::kOffML);
  ItemSlot<R>* iq = reinterpret_cast<ItemSlot<R>*>(smem + SM::kOffItems);
  uint64_t* i_meta = reinterpret_cast<uint64_t*>(smem + SM::kOffBar);
  uint64_t* i_full = i_meta + kIQ;
  uint64_t* i_empty = i_full + kIQ;
  uint64_t* m_full = i_empty + kIQ;
  uint64_t* m_empty = m_full + kNB;

  if (threadIdx.x == 0) {
    reinterpret_cast<int*>(smem + SM::kOffDefer)[0] = 0;
    for (int i = 0; i < kIQ; ++i) {
      mbar_init(&i_meta[i], 1);
      mbar_init(&i_full[i], 1);
      mbar_init(&i_empty[i], kWorkers + 1);  // workers + merger
    }
    for (int i = 0; i < kNB; ++i) {
      mbar_init(&m_full[i], kWorkers);
      mbar_init(&m_empty[i], 1);
    }
    fence_mbar_init();
  }
  // the zero query row stands in for MMA rows past R (16-row tiles)
  if (threadIdx.x < kRowBytes / 16)
    reinterpret_cast<uint4*>(smem + SM::kOffQZero)[threadIdx.x] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  pdl_launch_dependents();
  unsigned long long* dts = (RB_DIAG && a.debug_ts) ? a.debug_ts + blockIdx.x * 8 : nullptr;
  if (dts && threadIdx.x == 0) {
    dts[0] = global_timer_ns();
    dts[1] = smid();
  }

  if (warp == 0) {
    // ----------------------------------------------------------- scheduler
    // Software pipeline: publish item j, load item j+1's metadata, claim
    // item j+3 (the atomic resolves while the scheduler waits for a free
    // queue slot).  With `sched` every item is claimed from the global
    // counter (the first three in one atomic), so CTAs that start late --
    // after the concurrent system kernel frees their SM -- still share the
    // remaining work; without it the order is static (b + k * grid).
    int* sched = a.sched;
    const int bt_lanes = a.ctx.block_table != nullptr ? min(32, a.ctx.bt_stride) : 0;
    struct Raw {
      int item, qs0, qs1, clen, bte;
      long long roff;
    };
    auto load_raw = [&](int item) {
      Raw w;
      w.item = item;
      w.qs0 = w.qs1 = w.clen = w.bte = 0;
      w.roff = 0;
      if (item < n_items) {
        const int r = item / (n_z * a.hkv);
        w.qs0 = __ldg(a.q_start + r);
        w.qs1 = __ldg(a.q_start + r + 1);
        w.clen = __ldg(a.ctx_lens + r);
        if (a.ctx.req_offset != nullptr) w.roff = __ldg(a.ctx.req_offset + r);
        // rows of the table are bt_stride long: the first min(32, bt_stride) are in bounds
        if (lane < bt_lanes)
          w.bte = __ldg(a.ctx.block_table + static_cast<long long>(r) * a.ctx.bt_stride + lane);
      }
      return w;
    };
    const int G = static_cast<int>(gridDim.x);
    int id0 = blockIdx.x, id1 = blockIdx.x + G, id2 = blockIdx.x + 2 * G;
    if (sched != nullptr) {
      int base = 0;
      if (lane == 0) base = atomicAdd(sched, 3);
      base = __shfl_sync(0xffffffffu, base, 0);
      id0 = base;
      id1 = base + 1;
      id2 = base + 2;
    }
    Raw cur = load_raw(id0);
    for (int j = 0;; ++j) {
      const int item = cur.item;
      const int qs = j % kIQ;
      ItemSlot<R>& slot = iq[qs];
      // claim item j+3 and load item j+1 while this one is published
      int p = id2 + G;
      if (sched != nullptr && lane == 0) p = atomicAdd(sched, 1);
      const Raw nxt = load_raw(id1);
      mbar_wait(&i_empty[qs], ((j / kIQ) & 1) ^ 1);
      if (item >= n_items) {
        if (lane == 0) {
          slot.item = -1;
          mbar_arrive(&i_meta[qs]);
          mbar_arrive(&i_full[qs]);
        }
        break;
      }
      CtxItem<R> it;
      it.z = item % n_z;
      it.h = (item / n_z) % a.hkv;
      it.r = item / (n_z * a.hkv);
      it.row0 = cur.qs0;
      it.m_r = cur.qs1 - cur.qs0;
      it.nrows = it.m_r * a.g;
      it.c_r = cur.clen;
      it.roff = cur.roff;
      const int rbase = it.z * R;
      if (rbase >= it.nrows) {
        it.max_lim = 0;
        it.n_chunks = 0;
      } else {
        const int t_last = (min(rbase + R, it.nrows) - 1) / a.g;
        it.max_lim = a.causal ? it.c_r - it.m_r + t_last + 1 : it.c_r;
        it.n_chunks = n_pre + (it.max_lim + kChunk - 1) / kChunk;
      }
      const int nvalid = it.n_chunks > 0 ? max(0, min(R, it.nrows - rbase)) : 0;
      slot.bt[lane] = cur.bte;
      if (lane == 0) {
        slot.it = it;
        slot.item = item;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&i_meta[qs]);
        mbar_arrive_expect_tx(&i_full[qs], nvalid * kRowBytes);
      }
      __syncwarp();
      // query rows of the item: one 256-byte bulk copy per row
      if (lane < nvalid) {
        const int li = rbase + lane;
        const int t = li / a.g, jj = li % a.g;
        const __nv_bfloat16* qp = a.q + static_cast<long long>(it.row0 + t) * a.q_row_stride +
                                  static_cast<long long>(it.h * a.g + jj) * a.q_head_stride;
        bulk_copy_g2s(smem + SM::kOffQ + (qs * R + lane) * kRowBytes, qp, kRowBytes, &i_full[qs]);
      }
      cur = nxt;
      id1 = id2;
      id2 = (sched != nullptr) ? __shfl_sync(0xffffffffu, p, 0) : p;
    }
    if (sched != nullptr && lane == 0) {
      // every scheduler's last claim precedes its arrival here, so the last
      // CTA to arrive can rearm the counters for the next launch
      if (atomicAdd(sched + 1, 1) == static_cast<int>(gridDim.x) - 1) {
        atomicExch(sched, 0);
        atomicExch(sched + 1, 0);
      }
    }
    return;
  }

  if (warp == kMergerWarp) {
    // --------------------------------------------------------------- merger
    // Walks the item queue like the workers (metadata only), waits for the
    // workers' states of each item (m_full), combines them (lane = 4 head
    // dims) and writes: the relay context partial (unnormalised O, m, l) to
    // the workspace, or the final output (+ optional fusion with a given
    // system partial o_sys / lse_sys).
    bool waited = false;
    int jp = 0;  // queue cursor
    // diagnostics (debug timestamps only): waits and work of the merger
    unsigned long long d_mfull = 0, d_work = 0, d_imeta = 0, d_t = 0;
    // relay with <= 64 system units: the publication counters are polled in
    // the background (lane l: units l, l + 32; loads issued one item ahead,
    // consumed at the next) into a bitmask of published units, so deciding
    // fuse-or-park costs no round trip on the merger's critical path
    const bool poll = a.ctx_part != nullptr && a.sys_plan.n_units <= 64;
    unsigned long long pub = 0;
    int pv0 = 0, pv1 = 0, np0 = 0x7fffffff, np1 = 0x7fffffff;
    if (poll) {
      if (lane < a.sys_plan.n_units) np0 = rb_unit_parts(&a.sys_plan, lane);
      if (lane + 32 < a.sys_plan.n_units) np1 = rb_unit_parts(&a.sys_plan, lane + 32);
      if (np0 != 0x7fffffff) pv0 = ld_acquire_gpu(a.sys_ready + lane);
      if (np1 != 0x7fffffff) pv1 = ld_acquire_gpu(a.sys_ready + lane + 32);
    }
    for (int mi = 0;; ++mi) {
      // next non-empty item off the queue
      int item = -1;
      CtxItem<R> it;
      for (;;) {
        const int qs = jp % kIQ;
        if (dts) d_t = global_timer_ns();
        mbar_wait(&i_meta[qs], static_cast<uint32_t>((jp / kIQ) & 1));
        if (dts) d_imeta += global_timer_ns() - d_t;
        item = iq[qs].item;
        it = iq[qs].it;
        __syncwarp();
        if (lane == 0) mbar_arrive(&i_empty[qs]);
        ++jp;
        if (item < 0 || it.n_chunks > 0) break;
      }
      if (item < 0) break;
      // relay: if row 0's system unit is already published, issue its
      // parts' loads now so they land while the workers finish the item
      bool pre = false;
      RelayParts pp;
      if (poll) {
        // fold in the previous poll, then issue the next one
        const unsigned b0 = __ballot_sync(0xffffffffu, pv0 >= np0);
        const unsigned b1 = __ballot_sync(0xffffffffu, pv1 >= np1);
        pub |= static_cast<unsigned long long>(b0) | (static_cast<unsigned long long>(b1) << 32);
        __syncwarp();  // the acquiring lanes' loads precede every lane's part reads
        if (np0 != 0x7fffffff && !((pub >> lane) & 1)) pv0 = ld_acquire_gpu(a.sys_ready + lane);
        if (np1 != 0x7fffffff && !((pub >> (lane + 32)) & 1))
          pv1 = ld_acquire_gpu(a.sys_ready + lane + 32);
      }
      if (a.ctx_part != nullptr && it.z * R < it.nrows) {
        const long long o0 = static_cast<long long>(it.row0 + (it.z * R) / a.g) * a.hq +
                             it.h * a.g + (it.z * R) % a.g;
        pre = poll ? relay_unit_published(a.sys_plan, a.hq, o0, pub)
                   : relay_unit_ready(a.sys_plan, a.hq, o0, a.sys_ready, lane, false);
        if (pre) pp = relay_parts_begin(a.sys_plan, a.hq, o0, a.sys_part_acc, a.sys_part_ml, lane);
      }
      if (!waited && a.ctx_part == nullptr) {
        // before the first output write / o_sys read: the previous grid (a
        // system kernel producing o_sys, or a reader of out) must be done
        pdl_wait_primary();
        waited = true;
      }
      const int mb = mi % kNB;
      const uint32_t mph = static_cast<uint32_t>((mi / kNB) & 1);
      if (dts) d_t = global_timer_ns();
      mbar_wait(&m_full[mb], mph);
      if (dts) {
        const unsigned long long t1 = global_timer_ns();
        d_mfull += t1 - d_t;
        d_t = t1;
      }
      const float* bacc = s_acc + mb * kWorkers * R * 128;
      const float* bml = s_ml + mb * kWorkers * R * 2;
      const int rbase = it.z * R;
      const int d0 = lane * 4;
#pragma unroll 1
      for (int i = 0; i < R; ++i) {
        const int li = rbase + i;
        if (li >= it.nrows) break;
        const int t = li / a.g, jj = li % a.g;
        const long long oidx = static_cast<long long>(it.row0 + t) * a.hq + it.h * a.g + jj;
        float M = -INFINITY;
#pragma unroll
        for (int k = 0; k < kWorkers; ++k) M = fmaxf(M, bml[(k * R + i) * 2]);
        float Ls = 0.f, O[4] = {0.f, 0.f, 0.f, 0.f};
        if (M != -INFINITY) {
#pragma unroll
          for (int k = 0; k < kWorkers; ++k) {
            const float mk = bml[(k * R + i) * 2];
            const float wt = (mk == -INFINITY) ? 0.f : fast_exp2(mk - M);
            Ls = fmaf(bml[(k * R + i) * 2 + 1], wt, Ls);
            const float4 av = *reinterpret_cast<const float4*>(bacc + (k * R + i) * 128 + d0);
            O[0] = fmaf(av.x, wt, O[0]);
            O[1] = fmaf(av.y, wt, O[1]);
            O[2] = fmaf(av.z, wt, O[2]);
            O[3] = fmaf(av.w, wt, O[3]);
          }
        }
        if (a.ctx_part != nullptr) {
          // relay: fuse now if the pair's system unit is published, else
          // park the unnormalised partial and fuse it at the end of the CTA
          int* defer = reinterpret_cast<int*>(smem + SM::kOffDefer);
          const bool full = defer[0] >= kMaxDefer;
          if (i == 0 && pre) {
            relay_fuse_finish(a.sys_plan, pp, oidx, a.sys_part_acc, a.sys_part_ml,
                              make_float4(O[0], O[1], O[2], O[3]), M, Ls, a.out, a.out_fp32,
                              a.lse_out, lane);
          } else if (poll ? (relay_unit_published(a.sys_plan, a.hq, oidx, pub) ||
                             (full && relay_unit_ready(a.sys_plan, a.hq, oidx, a.sys_ready, lane, true)))
                          : relay_unit_ready(a.sys_plan, a.hq, oidx, a.sys_ready, lane, full)) {
            relay_fuse_pair(a.sys_plan, a.hq, oidx, a.sys_part_acc, a.sys_part_ml,
                            make_float4(O[0], O[1], O[2], O[3]), M, Ls, a.out, a.out_fp32,
                            a.lse_out, lane);
          } else {
            float* dst = a.ctx_part + oidx * kPartStride;
            __stcg(reinterpret_cast<float4*>(dst + d0), make_float4(O[0], O[1], O[2], O[3]));
            if (lane == 0) __stcg(reinterpret_cast<float2*>(dst + 128), make_float2(M, Ls));
            __syncwarp();
            if (lane == 0) defer[1 + defer[0]++] = static_cast<int>(oidx);
            __syncwarp();
          }
          continue;
        }
        float o[4];
        float lse2;
        {
          const float inv = (Ls > 0.f) ? 1.f / Ls : 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) o[e] = O[e] * inv;
          lse2 = (Ls > 0.f) ? M + __log2f(Ls) : -INFINITY;
        }
        if (a.o_sys != nullptr) {
          const float ls2 = __ldcg(a.lse_sys + oidx) * kLog2e;
          const float4 sv = __ldcg(reinterpret_cast<const float4*>(a.o_sys + oidx * 128 + d0));
          const float mx = fmaxf(ls2, lse2);
          const float wc = (lse2 == -INFINITY) ? 0.f : fast_exp2(lse2 - mx);
          const float ws = (ls2 == -INFINITY) ? 0.f : fast_exp2(ls2 - mx);
          const float inv = 1.f / (wc + ws);
          o[0] = (wc * o[0] + ws * sv.x) * inv;
          o[1] = (wc * o[1] + ws * sv.y) * inv;
          o[2] = (wc * o[2] + ws * sv.z) * inv;
          o[3] = (wc * o[3] + ws * sv.w) * inv;
          lse2 = mx + __log2f(wc + ws);
        }
        if (a.out_fp32) {
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + oidx * 128 + d0) =
              make_float4(o[0], o[1], o[2], o[3]);
        } else {
          uint2 pk;
          pk.x = pack_bf16x2(o[0], o[1]);
          pk.y = pack_bf16x2(o[2], o[3]);
          *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.out) + oidx * 128 + d0) = pk;
        }
        if (a.lse_out != nullptr && lane == 0) a.lse_out[oidx] = lse2 * kLn2;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&m_empty[mb]);
      if (dts) d_work += global_timer_ns() - d_t;
    }
    if (dts && lane == 0) {
      dts[6] = global_timer_ns();
      unsigned long long* acc = dts + 3072 * 8;
      acc[0] = d_mfull;
      acc[1] = static_cast<unsigned long long>(jp);
      acc[2] = d_work;
      acc[5] = d_imeta;
    }
  } else {
  // ---------------------------------------------------------------- workers
  const int w = warp - 1;                       // 0 .. kWorkers-1
  const uint32_t ring = smem_u32(smem + w * kDepth * kSlotBytes);
  uint8_t* ring_p = smem + w * kDepth * kSlotBytes;

  // issue cursor: queue item ji, next chunk ki (= w mod kWorkers)
  int ji = 0, ki = w, iss_item = 0, iss_bte = 0;
  int iss_r = 0, iss_h = 0, iss_lim = 0, iss_nch = 0;
  long long iss_roff = 0;
  bool have_iss = false;
  int issued = 0, consumed = 0, iss_sl = 0;

  // Issue chunks while the ring has room.  The cursor blocks on the item
  // queue only for items <= jc (already published); for later items it
  // polls, so a worker never waits on an item its CTA cannot publish yet.
  auto try_issue = [&](int jc) {
    while (issued < consumed + kDepth) {
      if (!have_iss) {
        const int qs = ji % kIQ;
        const uint32_t par = static_cast<uint32_t>((ji / kIQ) & 1);
        if (ji <= jc)
          mbar_wait(&i_meta[qs], par);
        else if (!mbar_test(&i_meta[qs], par))
          return;
        iss_item = iq[qs].item;
        iss_r = iq[qs].it.r;
        iss_h = iq[qs].it.h;
        iss_lim = iq[qs].it.max_lim;
        iss_nch = iq[qs].it.n_chunks;
        iss_roff = iq[qs].it.roff;
        iss_bte = iq[qs].bt[lane];
        have_iss = true;
        ki = w;
      }
      if (iss_item < 0) return;
      if (ki >= iss_nch) {
        ++ji;
        have_iss = false;
        continue;
      }
      const int k = ki;
      uint8_t* dst = ring_p + iss_sl * kSlotBytes;
      const __nv_bfloat16 *kb = a.ctx.k, *vb = a.ctx.v;
      long long tok_stride = a.ctx.stride_tok;
      int n;
      bool rows_ok = true;  // rows t0 .. t0 + 15 share one block / run
      if (k < n_pre) {
        const int t0 = k * kChunk;
        const long long off = static_cast<long long>(iss_h) * a.p_stride_head + t0 * a.p_stride_tok;
        kb = a.pk + off;
        vb = a.pv + off;
        tok_stride = a.p_stride_tok;
        n = min(kChunk, a.s_prefix - t0);
      } else {
        const int t0 = (k - n_pre) * kChunk;
        n = min(kChunk, iss_lim - t0);
        long long off;
        if (a.ctx.block_table == nullptr) {
          off = (iss_roff + t0) * a.ctx.stride_tok;
        } else if (a.ctx.block_size % kChunk == 0) {
          const int bi = t0 / a.ctx.block_size;
          const int v0 = __shfl_sync(0xffffffffu, iss_bte, bi & 31);
          const int blk = bi < 32 ? v0
                                  : __ldg(a.ctx.block_table +
                                          static_cast<long long>(iss_r) * a.ctx.bt_stride + bi);
          off = static_cast<long long>(blk) * a.ctx.stride_block +
                static_cast<long long>(t0 % a.ctx.block_size) * a.ctx.stride_tok;
        } else {
          off = 0;
          rows_ok = false;
        }
        off += iss_h * a.ctx.stride_head;
        kb += off;
        vb += off;
        if (!rows_ok) chunk_cp_async_rows(dst, a.ctx, iss_r, t0, iss_h, n, lane);
      }
      if (rows_ok) chunk_cp_async(dst, kb, vb, tok_stride, n, lane);
      asm volatile("cp.async.commit_group;" ::: "memory");
      ++issued;
      iss_sl = (iss_sl + 1 == kDepth) ? 0 : iss_sl + 1;
      ki += kWorkers;
    }
  };

  unsigned long long d_ifull = 0, d_mempty = 0, d_t = 0;
  try_issue(0);
  int mi = 0;  // items merged so far (skipped empty items excluded)
  int con_sl = 0;
  int qs = 0;
  uint32_t qph = 0;
  for (int jc = 0;; ++jc) {
    if (dts) d_t = global_timer_ns();
    mbar_wait(&i_full[qs], qph);
    if (dts) d_ifull += global_timer_ns() - d_t;
    const int item = iq[qs].item;
    const CtxItem<R> it = iq[qs].it;
    const int rbase = it.z * R;
    CtxCompute<R> cmp;
    cmp.load(smem + SM::kOffQ + qs * R * kRowBytes, smem + SM::kOffQZero, it, item, a, lane);
    // chunks below every valid row's bound need no mask: the smallest bound
    // over the item's rows is that of its first row
    const int ctx_nomask = a.causal ? it.c_r - it.m_r + rbase / a.g + 1 : it.c_r;
    const int mb = mi % kNB;
    const uint32_t mph = static_cast<uint32_t>((mi / kNB) & 1);
    // One loop, one issue site (instruction-cache footprint): the first pass
    // lets the issue cursor read this item's slot before it is released.
    int k = w;
    for (bool first = true;; first = false) {
      try_issue(jc);
      if (first) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&i_empty[qs]);
        if (++qs == kIQ) {
          qs = 0;
          qph ^= 1;
        }
        if (item < 0 || it.n_chunks == 0) break;
        cmp.init();
      }
      if (k >= it.n_chunks) break;
      // chunk `consumed` is this warp's commit group number `consumed`; the
      // groups committed after it may stay in flight
      const int newer = issued - consumed - 1;
      if (newer >= 2)
        asm volatile("cp.async.wait_group 2;" ::: "memory");
      else if (newer == 1)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();  // every lane's copies of the chunk are visible to the warp
      const bool pre = k < n_pre;
      const int key0 = (pre ? k : k - n_pre) * kChunk;
      const bool mask = key0 + kChunk > (pre ? a.s_prefix : ctx_nomask);
      cmp.chunk(ring_p + con_sl * kSlotBytes, key0, pre, it.max_lim, mask, a, lane);
      __syncwarp();  // every lane's reads precede the refill of this slot
      ++consumed;
      con_sl = (con_sl + 1 == kDepth) ? 0 : con_sl + 1;
      k += kWorkers;
    }
    if (item < 0) break;
    if (it.n_chunks == 0) continue;
    if (dts && lane == 0) dts[2 + w] = global_timer_ns();

    // ---- hand the warp's state (rows < R) to merge buffer mb
    if (dts) d_t = global_timer_ns();
    mbar_wait(&m_empty[mb], mph ^ 1);
    if (dts) d_mempty += global_timer_ns() - d_t;
    float* macc = s_acc + (mb * kWorkers + w) * R * 128;
    float* mml = s_ml + (mb * kWorkers + w) * R * 2;
    cmp.handoff(macc, mml, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&m_full[mb]);
    ++mi;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (dts && lane == 0 && w == 0) {
    dts[7] = global_timer_ns();
    dts[3072 * 8 + 3] = d_ifull;
    dts[3072 * 8 + 4] = d_mempty;
  }
  }  // workers

  // ------------------------------------------------ relay: deferred fusion
  // Rows whose system unit was not yet published when they were merged:
  // workers and merger share them once the CTA's items are done (each
  // waits for its row's unit), then the last CTA to finish rearms the
  // system-unit counters for the next step.
  if (a.ctx_part != nullptr) {
    named_bar_sync(1, 32 * (kWorkers + 1));
    const int* defer = reinterpret_cast<const int*>(smem + SM::kOffDefer);
    const int nd = defer[0];
    if (dts && warp == kMergerWarp && lane == 0) {
      dts[3072 * 8 + 6] = global_timer_ns();
      dts[3072 * 8 + 7] = static_cast<unsigned long long>(nd);
    }
    for (int e0 = (warp - 1) * 4; e0 < nd; e0 += (kWorkers + 1) * 4) {
      const int e = e0 + (lane >> 3);
      const bool valid = e < nd;
      relay_fuse_parked8(a.sys_plan, a.hq, valid ? defer[1 + e] : 0, valid, a.sys_ready, a.ctx_part,
                         a.sys_part_acc, a.sys_part_ml, a.out, a.out_fp32, a.lse_out, lane);
    }
    named_bar_sync(1, 32 * (kWorkers + 1));
    if (dts && warp == kMergerWarp && lane == 0) dts[6] = global_timer_ns();  // CTA done
    if (warp == kMergerWarp && lane == 0 && a.sched != nullptr) {
      __threadfence();
      if (atomicAdd(a.sched + 2, 1) == static_cast<int>(gridDim.x) - 1) {
        for (int u = 0; u < a.sys_plan.n_units; ++u) a.sys_ready[u] = 0;
        a.sched[2] = 0;
        __threadfence();
      }
    }
  }
}

template <int R>
static cudaError_t launch_ctx_r(const CtxArgs& a, int n_items, int n_z, cudaStream_t stream) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = CtaSmem<R>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(ctx_cta_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ctx_cta_kernel<R>, kCtxThreadsPC, smem);
  if (e != cudaSuccess) return e;
  const int grid = max(1, min(n_items, sms * max(per_sm, 1)));
  // PDL: the relay step's context kernel starts as soon as the system kernel
  // has triggered (it runs on the SMs the system kernel leaves free); the
  // other modes wait for their predecessor before the first output write.
  e = launch_pdl(ctx_cta_kernel<R>, dim3(grid), dim3(kCtxThreadsPC), smem, stream, a, n_items, n_z);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_context_attention(const CtxArgs& a, int max_rows, cudaStream_t stream) {
  // max_rows = max over requests of m_r * g
  int R = 1;
  if (max_rows >= 8) R = 8;
  else if (max_rows >= 4) R = 4;
  else if (max_rows >= 2) R = 2;
  const int n_z = (max_rows + R - 1) / R;
  const int n_items = a.b * a.hkv * n_z;
  if (n_items == 0) return cudaSuccess;
  switch (R) {
    case 1: return launch_ctx_r<1>(a, n_items, n_z, stream);
    case 2: return launch_ctx_r<2>(a, n_items, n_z, stream);
    case 4: return launch_ctx_r<4>(a, n_items, n_z, stream);
    default: return launch_ctx_r<8>(a, n_items, n_z, stream);
  }
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
// One thread per 16-byte chunk of K or V: fully parallel, coalesced.
__global__ void kv_append_kernel(const __nv_bfloat16* __restrict__ k_new,
                                 const __nv_bfloat16* __restrict__ v_new,
                                 const int* __restrict__ slots, __nv_bfloat16* k_pool,
                                 __nv_bfloat16* v_pool, int n_tok, int hkv, int block_size,
                                 long long stride_block, long long stride_tok,
                                 long long stride_head) {
  const long long n_chunks = static_cast<long long>(n_tok) * hkv * 16;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= 2 * n_chunks) return;
  const bool is_v = idx >= n_chunks;
  const long long ci = is_v ? idx - n_chunks : idx;
  const int c = static_cast<int>(ci & 15);
  const int h = static_cast<int>((ci >> 4) % hkv);
  const int t = static_cast<int>((ci >> 4) / hkv);
  const int slot = __ldg(slots + t);
  const int blk = slot / block_size, off = slot % block_size;
  const long long src = (static_cast<long long>(t) * hkv + h) * 128 + c * 8;
  const long long dst = blk * stride_block + off * stride_tok + h * stride_head + c * 8;
  if (is_v)
    *reinterpret_cast<uint4*>(v_pool + dst) = *reinterpret_cast<const uint4*>(v_new + src);
  else
    *reinterpret_cast<uint4*>(k_pool + dst) = *reinterpret_cast<const uint4*>(k_new + src);
}

cudaError_t launch_kv_append(const __nv_bfloat16* k_new, const __nv_bfloat16* v_new,
                             const int* slots, __nv_bfloat16* k_pool, __nv_bfloat16* v_pool,
                             int n_tok, int hkv, int block_size, long long stride_block,
                             long long stride_tok, long long stride_head, cudaStream_t stream) {
  if (n_tok == 0) return cudaSuccess;
  const long long total = 2LL * n_tok * hkv * 16;
  const int threads = 256;
  kv_append_kernel<<<static_cast<unsigned>((total + threads - 1) / threads), threads, 0, stream>>>(
      k_new, v_new, slots, k_pool, v_pool, n_tok, hkv, block_size, stride_block, stride_tok,
      stride_head);
  return cudaGetLastError();
}

}  // namespace rb
