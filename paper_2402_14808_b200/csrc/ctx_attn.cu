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
  int sp, grp, nsplit, k0;  // split index, (r, h, z) group, valid splits of it, first chunk
  int bt0;                  // block-table index of the item's bt[0] window
  long long roff;           // ragged mode: first token of request r
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

// The common case of the chunk copy: 16 valid rows, 256 B apart (a paged
// block's rows of one head, the [blocks][heads][block][128] layout): every
// address is a base register plus an immediate, no predicates.
__device__ __forceinline__ void cp_async_16_full(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
               "l"(reinterpret_cast<uint64_t>(gsrc))
               : "memory");
}
__device__ __forceinline__ void chunk_cp_async_full(uint8_t* slot, const __nv_bfloat16* kb,
                                                    const __nv_bfloat16* vb, int lane) {
  const int row0 = lane >> 4, c16 = lane & 15;
  const int cx = c16 ^ row0;
  uint8_t* d = slot + row0 * kRowBytes;
  const char* ks = reinterpret_cast<const char*>(kb) + row0 * kRowBytes + c16 * 16;
  const char* vs = reinterpret_cast<const char*>(vb) + row0 * kRowBytes + c16 * 16;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t off = i * 2 * kRowBytes + ((cx ^ ((2 * i) & 6)) << 4);
    cp_async_16_full(d + off, ks + i * 2 * kRowBytes);
    cp_async_16_full(d + kChunk * kRowBytes + off, vs + i * 2 * kRowBytes);
  }
}

// Cold path of the chunk copy (blocks not a multiple of 16 tokens, or other
// row layouts): per-row addresses through the block table.  Out of line so
// the hot loop stays small (instruction-cache resident).
__device__ __noinline__ void chunk_cp_async_rows(uint8_t* dst, KvView kv, int r, int t0, int h, int n,
                                                 int lane) {
  const int row0 = lane >> 4, c16 = lane & 15;
  // (not unrolled: this path is cold and ctx_row divides by the block size)
#pragma unroll 1
  for (int i = 0; i < 8; ++i) {
    const int row = row0 + 2 * i;
    const bool ok = row < n;
    const __nv_bfloat16* ks = ok ? ctx_row(kv, kv.k, r, t0 + row, h) : kv.k;
    const __nv_bfloat16* vs = ok ? kv.v + (ks - kv.k) : kv.v;
    const uint32_t so = slot_off(row, c16);
    cp_async_16(dst + so, ks + c16 * 8, ok ? 16u : 0u);
    cp_async_16(dst + kChunk * kRowBytes + so, vs + c16 * 8, ok ? 16u : 0u);
  }
}

// Per-worker compute of one item: up to R <= 8 query rows against the
// item's 16-key chunks on the tensor cores, "swap-AB" so the keys fill the
// MMA M dimension and the (few) query rows its N = 8 dimension:
//
//   S^T [16 keys x 8 rows] = K_chunk [16 x 128] . Q^T        (8 k-steps)
//   O^T [128 d  x 8 rows] += V_chunk^T [128 x 16] . P^T      (8 m-tiles)
//
// with mma.sync m16n8k16 (bf16 in, fp32 accumulate).  A decode row (R = 1)
// wastes 7/8 of N, but one 16-key chunk is still 16 MMAs + 16 ldmatrix +
// a ~30-instruction softmax -- the CUDA-core formulation it replaces needed
// ~1000 warp-instructions per chunk (64 bf16 converts each for K and V, 32
// shuffles for the dot products), which made the kernel issue-bound at
// ~0.5 of HBM (profiles/r01g).  Lane (g = lane / 4, t = lane % 4) holds
// S^T rows (keys) g, g + 8 and columns (query rows) 2t, 2t + 1; the softmax
// reduces over keys with 3 xor-shuffles per column, and P^T goes from the
// accumulator layout to the B-operand layout with two movmatrix transposes.
// Online softmax in the log2 domain with a lazy max: the reference max of a
// row moves only when a chunk exceeds it by more than kCtxTau, so O is
// rescaled rarely and p <= 2^kCtxTau.  Row sums stay per lane and are
// reduced across the 8 key lanes once per item.
constexpr float kCtxTau = 8.f;
constexpr int kAccStride = 132;   // floats per row of the merge buffers (bank-conflict padding)

template <int R>
struct SwapCompute {
  static_assert(R >= 1 && R <= 8, "one N = 8 tile of query rows per item");
  uint32_t qb[8][2];      // Q^T B fragments, 8 k-steps
  float o[8][4];          // O^T accumulator, 8 m-tiles of 16 head dims
  float m0, m1, l0, l1;   // columns 2t, 2t + 1: reference max (log2 units), partial row sum
  int lim0, lim1;         // exclusive context-key bounds of columns 2t, 2t + 1

  __device__ __forceinline__ void load(const uint8_t* qrows, const uint8_t* qzero,
                                       const CtxItem<R>& it, int item, const CtxArgs& a, int lane) {
    // B fragments of Q^T: ldmatrix (non-transposed) of the Q rows; matrix j
    // of an x4 is k-step 2kp + (j >> 1), half (j & 1); rows >= R read zeros
    const int qr = lane & 7, j = lane >> 3;
    const uint32_t qaddr = qr < R ? smem_u32(qrows + qr * kRowBytes) : smem_u32(qzero);
#pragma unroll
    for (int kp = 0; kp < 4; ++kp) {
      uint32_t r[4];
      ldsm_x4(r, qaddr + ((4 * kp + j) << 4));
      qb[2 * kp][0] = r[0];
      qb[2 * kp][1] = r[1];
      qb[2 * kp + 1][0] = r[2];
      qb[2 * kp + 1][1] = r[3];
    }
    const int rbase = it.z * R, t = lane & 3;
    int lim[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int rr = 2 * t + c, li = rbase + rr;
      const bool ok = item >= 0 && it.n_chunks > 0 && rr < R && li < it.nrows;
      // columns past the item's rows see every key (finite, never written)
      lim[c] = ok ? (a.causal ? it.c_r - it.m_r + li / a.g + 1 : it.c_r) : it.max_lim;
    }
    lim0 = lim[0];
    lim1 = lim[1];
  }
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[mt][e] = 0.f;
    m0 = m1 = -INFINITY;
    l0 = l1 = 0.f;
  }
  // one 16-key chunk in ring slot `slot` ([K|V][16 rows][256 B], 16-byte
  // columns XOR-swizzled by row & 7); key0: the chunk's first key inside
  // its segment; mask: some key of the chunk is past some row's bound
  __device__ __forceinline__ void chunk(const uint8_t* slot_p, int key0, bool pre, int /*max_lim*/,
                                        bool mask, const CtxArgs& a, int lane) {
    const uint32_t slot = smem_u32(slot_p);
    const int g = lane >> 2, j = lane >> 3, r8 = lane & 7;
    // ---- S^T = K Q^T: two accumulators (even / odd k-steps) for ILP
    float sa[4], sb[4];
    {
      const int key = r8 + 8 * (j & 1);
      const uint32_t kaddr = slot + key * kRowBytes;
      uint32_t ka[4];
      ldsm_x4(ka, kaddr + (((0 + (j >> 1)) ^ (key & 7)) << 4));
      mma_bf16_16816_zero(sa, ka, qb[0][0], qb[0][1]);
      ldsm_x4(ka, kaddr + (((2 + (j >> 1)) ^ (key & 7)) << 4));
      mma_bf16_16816_zero(sb, ka, qb[1][0], qb[1][1]);
#pragma unroll
      for (int ks = 2; ks < 8; ks += 2) {
        ldsm_x4(ka, kaddr + (((2 * ks + (j >> 1)) ^ (key & 7)) << 4));
        mma_bf16_16816(sa, ka, qb[ks][0], qb[ks][1]);
        ldsm_x4(ka, kaddr + (((2 * ks + 2 + (j >> 1)) ^ (key & 7)) << 4));
        mma_bf16_16816(sb, ka, qb[ks + 1][0], qb[ks + 1][1]);
      }
    }
    // s[0], s[1]: key g, columns 2t, 2t+1; s[2], s[3]: key g + 8
    float s[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) s[e] = (sa[e] + sb[e]) * a.scale_log2;
    if (mask) {
      // the shared prefix (naive baseline) is visible to every row
      const int b0 = pre ? a.s_prefix : lim0, b1 = pre ? a.s_prefix : lim1;
      if (key0 + g >= b0) s[0] = -INFINITY;
      if (key0 + g >= b1) s[1] = -INFINITY;
      if (key0 + g + 8 >= b0) s[2] = -INFINITY;
      if (key0 + g + 8 >= b1) s[3] = -INFINITY;
    }
    // ---- lazy online softmax per column (reduce over the 8 key lanes)
    float cm[2] = {fmaxf(s[0], s[2]), fmaxf(s[1], s[3])};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      cm[c] = fmaxf(cm[c], __shfl_xor_sync(0xffffffffu, cm[c], 4));
      cm[c] = fmaxf(cm[c], __shfl_xor_sync(0xffffffffu, cm[c], 8));
      cm[c] = fmaxf(cm[c], __shfl_xor_sync(0xffffffffu, cm[c], 16));
    }
    const bool up0 = cm[0] > m0 + kCtxTau, up1 = cm[1] > m1 + kCtxTau;
    if (__any_sync(0xffffffffu, up0 || up1)) {
      const float al0 = up0 ? ((m0 == -INFINITY) ? 0.f : fast_exp2(m0 - cm[0])) : 1.f;
      const float al1 = up1 ? ((m1 == -INFINITY) ? 0.f : fast_exp2(m1 - cm[1])) : 1.f;
      if (up0) m0 = cm[0];
      if (up1) m1 = cm[1];
      l0 *= al0;
      l1 *= al1;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        o[mt][0] *= al0;
        o[mt][1] *= al1;
        o[mt][2] *= al0;
        o[mt][3] *= al1;
      }
    }
    const float r0 = (m0 == -INFINITY) ? 0.f : m0, r1 = (m1 == -INFINITY) ? 0.f : m1;
    const float p0 = fast_exp2(s[0] - r0), p1 = fast_exp2(s[1] - r1);
    const float p2 = fast_exp2(s[2] - r0), p3 = fast_exp2(s[3] - r1);
    // P^T (keys x rows) to the B-operand layout: the accumulator pairs
    // (key g, rows 2t..2t+1) transpose to (keys 2t..2t+1, row g)
    const uint32_t pb0 = movmatrix_trans(pack_bf16x2(p0, p1));
    const uint32_t pb1 = movmatrix_trans(pack_bf16x2(p2, p3));
    l0 += p0 + p2;
    l1 += p1 + p3;
    // ---- O^T += V^T P^T: A = V^T via transposed ldmatrix of the V rows
    {
      const int key = r8 + 8 * (j >> 1);
      const uint32_t vaddr = slot + kChunk * kRowBytes + key * kRowBytes;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t va[4];
        ldsm_x4_trans(va, vaddr + (((2 * mt + (j & 1)) ^ (key & 7)) << 4));
        mma_bf16_16816(o[mt], va, pb0, pb1);
      }
    }
  }
  // Two chunks (32 keys) in one pass: the four Q.K^T chains are
  // independent, the column max / lazy-rescale vote runs once over 32 keys,
  // and the P.V MMAs of both chunks accumulate back to back -- the latency
  // chain of one chunk now covers two (the per-chunk math was ~35% of a
  // worker's per-item time at C2, profiles/diag_ctx_trace.py).
  __device__ __forceinline__ void chunk2(const uint8_t* slot_a, const uint8_t* slot_b, int key0a,
                                         int key0b, bool pre_a, bool pre_b, bool mask_a, bool mask_b,
                                         const CtxArgs& a, int lane) {
    const uint32_t sla = smem_u32(slot_a), slb = smem_u32(slot_b);
    const int g = lane >> 2, j = lane >> 3, r8 = lane & 7;
    float sa0[4], sa1[4], sb0[4], sb1[4];
    {
      const int key = r8 + 8 * (j & 1);
      const uint32_t ka_addr = sla + key * kRowBytes, kb_addr = slb + key * kRowBytes;
      uint32_t ka[4], kb[4];
      ldsm_x4(ka, ka_addr + (((0 + (j >> 1)) ^ (key & 7)) << 4));
      ldsm_x4(kb, kb_addr + (((0 + (j >> 1)) ^ (key & 7)) << 4));
      mma_bf16_16816_zero(sa0, ka, qb[0][0], qb[0][1]);
      mma_bf16_16816_zero(sb0, kb, qb[0][0], qb[0][1]);
      ldsm_x4(ka, ka_addr + (((2 + (j >> 1)) ^ (key & 7)) << 4));
      ldsm_x4(kb, kb_addr + (((2 + (j >> 1)) ^ (key & 7)) << 4));
      mma_bf16_16816_zero(sa1, ka, qb[1][0], qb[1][1]);
      mma_bf16_16816_zero(sb1, kb, qb[1][0], qb[1][1]);
#pragma unroll
      for (int ks = 2; ks < 8; ks += 2) {
        ldsm_x4(ka, ka_addr + (((2 * ks + (j >> 1)) ^ (key & 7)) << 4));
        ldsm_x4(kb, kb_addr + (((2 * ks + (j >> 1)) ^ (key & 7)) << 4));
        mma_bf16_16816(sa0, ka, qb[ks][0], qb[ks][1]);
        mma_bf16_16816(sb0, kb, qb[ks][0], qb[ks][1]);
        ldsm_x4(ka, ka_addr + (((2 * ks + 2 + (j >> 1)) ^ (key & 7)) << 4));
        ldsm_x4(kb, kb_addr + (((2 * ks + 2 + (j >> 1)) ^ (key & 7)) << 4));
        mma_bf16_16816(sa1, ka, qb[ks + 1][0], qb[ks + 1][1]);
        mma_bf16_16816(sb1, kb, qb[ks + 1][0], qb[ks + 1][1]);
      }
    }
    float s[8];  // [0..3]: chunk a (keys g, g+8; columns 2t, 2t+1), [4..7]: chunk b
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      s[e] = (sa0[e] + sa1[e]) * a.scale_log2;
      s[4 + e] = (sb0[e] + sb1[e]) * a.scale_log2;
    }
    if (mask_a) {
      const int b0 = pre_a ? a.s_prefix : lim0, b1 = pre_a ? a.s_prefix : lim1;
      if (key0a + g >= b0) s[0] = -INFINITY;
      if (key0a + g >= b1) s[1] = -INFINITY;
      if (key0a + g + 8 >= b0) s[2] = -INFINITY;
      if (key0a + g + 8 >= b1) s[3] = -INFINITY;
    }
    if (mask_b) {
      const int b0 = pre_b ? a.s_prefix : lim0, b1 = pre_b ? a.s_prefix : lim1;
      if (key0b + g >= b0) s[4] = -INFINITY;
      if (key0b + g >= b1) s[5] = -INFINITY;
      if (key0b + g + 8 >= b0) s[6] = -INFINITY;
      if (key0b + g + 8 >= b1) s[7] = -INFINITY;
    }
    float cm[2] = {fmaxf(fmaxf(s[0], s[2]), fmaxf(s[4], s[6])), fmaxf(fmaxf(s[1], s[3]), fmaxf(s[5], s[7]))};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      cm[c] = fmaxf(cm[c], __shfl_xor_sync(0xffffffffu, cm[c], 4));
      cm[c] = fmaxf(cm[c], __shfl_xor_sync(0xffffffffu, cm[c], 8));
      cm[c] = fmaxf(cm[c], __shfl_xor_sync(0xffffffffu, cm[c], 16));
    }
    const bool up0 = cm[0] > m0 + kCtxTau, up1 = cm[1] > m1 + kCtxTau;
    if (__any_sync(0xffffffffu, up0 || up1)) {
      const float al0 = up0 ? ((m0 == -INFINITY) ? 0.f : fast_exp2(m0 - cm[0])) : 1.f;
      const float al1 = up1 ? ((m1 == -INFINITY) ? 0.f : fast_exp2(m1 - cm[1])) : 1.f;
      if (up0) m0 = cm[0];
      if (up1) m1 = cm[1];
      l0 *= al0;
      l1 *= al1;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        o[mt][0] *= al0;
        o[mt][1] *= al1;
        o[mt][2] *= al0;
        o[mt][3] *= al1;
      }
    }
    const float r0 = (m0 == -INFINITY) ? 0.f : m0, r1 = (m1 == -INFINITY) ? 0.f : m1;
    float p[8];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      p[e] = fast_exp2(s[e] - r0);
      p[e + 1] = fast_exp2(s[e + 1] - r1);
    }
    const uint32_t pa0 = movmatrix_trans(pack_bf16x2(p[0], p[1]));
    const uint32_t pa1 = movmatrix_trans(pack_bf16x2(p[2], p[3]));
    const uint32_t pb0 = movmatrix_trans(pack_bf16x2(p[4], p[5]));
    const uint32_t pb1 = movmatrix_trans(pack_bf16x2(p[6], p[7]));
    l0 += (p[0] + p[2]) + (p[4] + p[6]);
    l1 += (p[1] + p[3]) + (p[5] + p[7]);
    {
      const int key = r8 + 8 * (j >> 1);
      const uint32_t va_addr = sla + kChunk * kRowBytes + key * kRowBytes;
      const uint32_t vb_addr = slb + kChunk * kRowBytes + key * kRowBytes;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        uint32_t va[4], vb[4];
        ldsm_x4_trans(va, va_addr + (((2 * mt + (j & 1)) ^ (key & 7)) << 4));
        ldsm_x4_trans(vb, vb_addr + (((2 * mt + (j & 1)) ^ (key & 7)) << 4));
        mma_bf16_16816(o[mt], va, pa0, pa1);
        mma_bf16_16816(o[mt], vb, pb0, pb1);
      }
    }
  }
  // reduce the row sums over the key lanes, then write rows < R of this
  // worker's state: macc [R][kAccStride] (unnormalised O), mml [R][2]
  __device__ __forceinline__ void handoff(float* macc, float* mml, int lane) {
    const int g = lane >> 2, t = lane & 3;
    float ls[2] = {l0, l1};
    const float ms[2] = {m0, m1};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      ls[c] += __shfl_xor_sync(0xffffffffu, ls[c], 4);
      ls[c] += __shfl_xor_sync(0xffffffffu, ls[c], 8);
      ls[c] += __shfl_xor_sync(0xffffffffu, ls[c], 16);
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int rr = 2 * t + c;
      if (rr < R) {
        float* row = macc + rr * kAccStride;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          row[16 * mt + g] = o[mt][c];
          row[16 * mt + g + 8] = o[mt][2 + c];
        }
        if (g == 0) {
          mml[rr * 2] = ms[c];
          mml[rr * 2 + 1] = ls[c];
        }
      }
    }
  }
};

template <int R>
using CtxCompute = SwapCompute<R>;

// Relay fusion of one (row, head) pair (`relay_fusion`, attention.py:137-157):
// the context state (O unnormalised, m log2, l) merged with every stream-K
// part of the pair's system unit in slot order (deterministic), normalised
// and written.  One warp, lane = 4 head dims.  The unit must be published.
// Split in two so the merger can issue the first parts' loads before it
// waits for the workers (RelayParts carries them in registers).
// system parts per batch of loads in flight in the relay fusion (C4 split
// units have 6 parts: batch 8 = one round trip per row; C4 step 110.6 ->
// 105.2 us against batch 4)
#ifndef RB_RELAY_GROUPED
#define RB_RELAY_GROUPED 1
#endif
#ifndef RB_RELAY_BATCH
#define RB_RELAY_BATCH 8
#endif
constexpr int kRB = RB_RELAY_BATCH;  // system parts per batch of loads in flight
// One step of the slot-order part fold, o * so + a * sk, with the rounding
// spelled out so every fusion path (per row, grouped rows, parked rows)
// gives the same bits whichever of them a row takes.
__device__ __forceinline__ float relay_fold(float o, float so, float a, float sk) {
  return __fmaf_rn(o, so, __fmul_rn(a, sk));
}

template <int B>
struct RelayParts {
  long long base;
  int np, col;
  float mk[B], lk[B];
  float4 ak[B];
};

template <int B>
__device__ __forceinline__ void relay_parts_load(const rb_sys_plan& SP, const float* part_acc,
                                                 const float* part_ml, long long base, int np,
                                                 int col, int k0, int lane, float* mk, float* lk,
                                                 float4* ak) {
#pragma unroll
  for (int kk = 0; kk < B; ++kk) {
    const int k = min(k0 + kk, np - 1);
    const float* pml = part_ml + (base + k) * 2 * SP.nq;
    mk[kk] = __ldcg(pml + col);
    lk[kk] = __ldcg(pml + SP.nq + col);
    ak[kk] = __ldcg(reinterpret_cast<const float4*>(part_acc + ((base + k) * SP.nq + col) * RB_HEAD_DIM + lane * 4));
  }
}

// A (row, head) pair of the relay step: output index, its system unit and
// its row within the unit (from the item geometry, no runtime divisions by
// hq / nq -- they were a few hundred instructions on the merger's per-row path)
struct RowRef {
  long long oidx;
  int u, col;
};

template <int B>
__device__ __forceinline__ RelayParts<B> relay_parts_begin(const rb_sys_plan& SP, const RowRef& rr,
                                                           const float* part_acc, const float* part_ml,
                                                           int lane) {
  RelayParts<B> P;
  P.col = rr.col;
  const int u = rr.u;
  P.np = rb_unit_parts(&SP, u);
  P.base = static_cast<long long>(u) * SP.max_parts;
  relay_parts_load<B>(SP, part_acc, part_ml, P.base, P.np, P.col, 0, lane, P.mk, P.lk, P.ak);
  return P;
}

template <int B>
__device__ __forceinline__ void relay_fuse_finish(const rb_sys_plan& SP, RelayParts<B>& P, long long pair,
                                                  const float* part_acc, const float* part_ml,
                                                  float4 O, float mt, float lt, void* out, int out_fp32,
                                                  float* lse_out, int lane) {
  const int d0 = lane * 4;
  for (int k0 = 0; k0 < P.np; k0 += B) {
    if (k0 > 0) relay_parts_load<B>(SP, part_acc, part_ml, P.base, P.np, P.col, k0, lane, P.mk, P.lk, P.ak);
#pragma unroll
    for (int kk = 0; kk < B; ++kk) {
      if (k0 + kk >= P.np) break;
      const float mn = fmaxf(mt, P.mk[kk]);
      const float so = (mt == -INFINITY) ? 0.f : fast_exp2(mt - mn);
      const float sk = fast_exp2(P.mk[kk] - mn);
      lt = relay_fold(lt, so, P.lk[kk], sk);
      O.x = relay_fold(O.x, so, P.ak[kk].x, sk);
      O.y = relay_fold(O.y, so, P.ak[kk].y, sk);
      O.z = relay_fold(O.z, so, P.ak[kk].z, sk);
      O.w = relay_fold(O.w, so, P.ak[kk].w, sk);
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

template <int B>
__device__ __forceinline__ void relay_fuse_pair(const rb_sys_plan& SP, const RowRef& rr,
                                                const float* part_acc, const float* part_ml,
                                                float4 O, float mt, float lt, void* out, int out_fp32,
                                                float* lse_out, int lane) {
  RelayParts<B> P = relay_parts_begin<B>(SP, rr, part_acc, part_ml, lane);
  relay_fuse_finish<B>(SP, P, rr.oidx, part_acc, part_ml, O, mt, lt, out, out_fp32, lse_out, lane);
}

// Relay fusion of all R rows of an item at once, when they share one published
// system unit (a row's unit: its KV head and query tile; an item's rows are
// consecutive flattened rows).  Lane group rg = lane / LPR owns row rg, lane
// li of the group head dims [li DPL, (li + 1) DPL): the row's context state
// is combined from the workers' merge buffers, then the unit's parts are
// folded in slot order with KB parts' loads in flight -- one L2 round trip
// per KB parts for the whole item instead of one per row (R = 8 at C5: the
// per-row fusion made the merger the bottleneck once the system units were
// published).  Same arithmetic per element as relay_fuse_finish.
template <int R>
__device__ __forceinline__ void relay_fuse_rows(const rb_sys_plan& SP, const RowRef& rr,
                                                const float* bacc, const float* bml,
                                                const float* part_acc, const float* part_ml,
                                                void* out, int out_fp32, float* lse_out, int lane) {
  constexpr int LPR = 32 / R, DPL = RB_HEAD_DIM / LPR, NV = DPL / 4;
  constexpr int KB = R >= 8 ? 2 : 8 / R;
  const int rg = lane / LPR, li = lane % LPR;
  float M = -INFINITY;
#pragma unroll
  for (int k = 0; k < 4; ++k) M = fmaxf(M, bml[(k * R + rg) * 2]);
  float Ls = 0.f;
  float4 O[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) O[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (M != -INFINITY) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float mk = bml[(k * R + rg) * 2];
      const float wt = (mk == -INFINITY) ? 0.f : fast_exp2(mk - M);
      Ls = fmaf(bml[(k * R + rg) * 2 + 1], wt, Ls);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const float4 av = *reinterpret_cast<const float4*>(bacc + (k * R + rg) * kAccStride + li * DPL + 4 * v);
        O[v].x = fmaf(av.x, wt, O[v].x);
        O[v].y = fmaf(av.y, wt, O[v].y);
        O[v].z = fmaf(av.z, wt, O[v].z);
        O[v].w = fmaf(av.w, wt, O[v].w);
      }
    }
  }
  const long long pair = rr.oidx;
  const int col = rr.col, u = rr.u;
  const int np = rb_unit_parts(&SP, u);
  const long long base = static_cast<long long>(u) * SP.max_parts;
  float mt = M, lt = Ls;
  for (int k0 = 0; k0 < np; k0 += KB) {
    float mk[KB], lk[KB];
    float4 ak[KB][NV];
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      const int k = min(k0 + kk, np - 1);
      const float* pml = part_ml + (base + k) * 2 * SP.nq;
      mk[kk] = __ldcg(pml + col);
      lk[kk] = __ldcg(pml + SP.nq + col);
      const float* pa = part_acc + ((base + k) * SP.nq + col) * RB_HEAD_DIM + li * DPL;
#pragma unroll
      for (int v = 0; v < NV; ++v) ak[kk][v] = __ldcg(reinterpret_cast<const float4*>(pa + 4 * v));
    }
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      if (k0 + kk >= np) break;
      const float mn = fmaxf(mt, mk[kk]);
      const float so = (mt == -INFINITY) ? 0.f : fast_exp2(mt - mn);
      const float sk = fast_exp2(mk[kk] - mn);
      lt = relay_fold(lt, so, lk[kk], sk);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        O[v].x = relay_fold(O[v].x, so, ak[kk][v].x, sk);
        O[v].y = relay_fold(O[v].y, so, ak[kk][v].y, sk);
        O[v].z = relay_fold(O[v].z, so, ak[kk][v].z, sk);
        O[v].w = relay_fold(O[v].w, so, ak[kk][v].w, sk);
      }
      mt = mn;
    }
  }
  const float inv = 1.f / lt;
  if (out_fp32) {
    float* o = reinterpret_cast<float*>(out) + pair * 128 + li * DPL;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      reinterpret_cast<float4*>(o)[v] = make_float4(O[v].x * inv, O[v].y * inv, O[v].z * inv, O[v].w * inv);
  } else {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + pair * 128 + li * DPL;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      uint2 pk;
      pk.x = pack_bf16x2(O[v].x * inv, O[v].y * inv);
      pk.y = pack_bf16x2(O[v].z * inv, O[v].w * inv);
      reinterpret_cast<uint2*>(o)[v] = pk;
    }
  }
  if (lse_out != nullptr && li == 0) lse_out[pair] = (mt + __log2f(lt)) * kLn2;
}

// Is system unit u published (all its parts written)?  Lane 0 probes with
// acquire semantics; the answer is broadcast to the warp.
__device__ __forceinline__ bool relay_unit_ready(const rb_sys_plan& SP, int u, const int* ready, int lane,
                                                 bool block) {
  if (u >= SP.n_units) return false;  // outside the plan (bad q_start): parked, then dropped
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
// Published-unit bitmask of the merger's background poll: lane l holds bit
// k for unit l + 32 k (k < kPollSlots); warp-uniform call.
constexpr int kPollSlots = 8;   // polls up to 256 system units
__device__ __forceinline__ bool relay_unit_published(int u, uint32_t pub) {
  const uint32_t bits = __shfl_sync(0xffffffffu, pub, u & 31);
  return u < 32 * kPollSlots && ((bits >> (u >> 5)) & 1);
}

constexpr int kWorkers = 4;
// Per-row-count configuration.  Two CTAs must fit an SM (<= ~113 KB of
// shared memory each) so that 8 worker warps keep their rings of K+V chunks
// in flight per SM: the merge buffers grow with R, so R = 2 / 4 keep fewer
// merge buffers (their items are long, the merger keeps up with one or two)
// and R = 8 a 2-deep ring.
template <int R>
#ifndef RB_CTX_PAIRS
#define RB_CTX_PAIRS 0   /* 1: a worker's two next chunks in one softmax pass (SwapCompute::chunk2); measured neutral */
#endif
#ifndef RB_CTX_MINB
#define RB_CTX_MINB 2   /* resident CTAs per SM the register budget is sized for */
#endif
// 1-row items (C2 / C3 decode): 2 chunks in flight per worker -- with the
// smaller kernel, C2 s=2048 47.0 -> 45.1 us, s=1024 40.9 -> 38.9 us against 3
#ifndef RB_CTX_DEPTH1
#define RB_CTX_DEPTH1 2
#endif
// chunks in flight per worker for 4- and 8-row items (C4 / C5 GQA shapes):
// measured C4 step 110.3 us at depth 3, 104.8 at 2, 136 at 1; C5 with the
// grouped relay fusion 625 us at depth 2, 659 at 1 -- fewer context bytes
// in flight leave HBM to the concurrent system kernel, too few starve the
// context side
#ifndef RB_CTX_DEPTH4
#define RB_CTX_DEPTH4 2
#endif
#ifndef RB_CTX_NB4
#define RB_CTX_NB4 1
#endif
#ifndef RB_CTX_DEPTH8
#define RB_CTX_DEPTH8 2
#endif
struct CtxCfg {
  static constexpr int kDepth = R >= 8 ? RB_CTX_DEPTH8 : (R == 1 ? RB_CTX_DEPTH1 : R == 4 ? RB_CTX_DEPTH4 : 3);  // chunks in flight per worker
  static constexpr int kNB = R == 1 ? 3 : R == 2 ? 2 : R == 4 ? RB_CTX_NB4 : 2;  // merge buffers
  // relay rows a CTA can park while their system unit is unpublished; when
  // the list is full the merger blocks on the unit.  At C5 every unit is
  // published only when the system kernel ends (~470 us), so the context
  // CTAs beside it block after ~8 items -- and that measured faster than
  // letting them run on (1022 / 4094 slots: C5 625 -> 659 us with depth 2;
  // the extra context traffic slows the tensor-bound system kernel more
  // than it saves, and their parked rows make a 20 us end-phase tail)
#ifdef RB_CTX_MAXDEFER
  static constexpr int kMaxDefer = RB_CTX_MAXDEFER;
#else
  static constexpr int kMaxDefer = 62;
#endif
};
#ifndef RB_CTX_IQ
#define RB_CTX_IQ 3
#endif
constexpr int kIQ = RB_CTX_IQ;
#ifndef RB_CLAIM_LAZY
#define RB_CLAIM_LAZY 1
#endif                         // item queue depth (claim-ahead bound)
constexpr int kCtxThreadsPC = 32 * (2 + kWorkers);  // scheduler + workers + merger
constexpr int kMergerWarp = 1 + kWorkers;
constexpr int kPartStride = 132;               // floats per relay context partial: O[128], m, l

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
    const int row = static_cast<int>(pair) / hq, hh = static_cast<int>(pair) % hq;
    const int f = row * SP.g + hh % SP.g;
    col = f % SP.nq;
    u = (hh / SP.g) * SP.n_qt + f / SP.nq;
    valid = u < SP.n_units;  // a row outside the plan (bad q_start) is dropped, never awaited
    np = valid ? rb_unit_parts(&SP, u) : 0;
    if (sub == 0 && valid)
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
  // parts in batches of 4 with all their loads in flight (the first batch's
  // with the context part's): C4's 6-part units took 6 dependent round trips
  constexpr int KB = 4;
  for (int k0 = 0; k0 < np; k0 += KB) {
    float mk[KB], lk[KB];
    float4 ak[KB][4];
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      const int k = min(k0 + kk, np - 1);
      const float* pml = part_ml + (base + k) * 2 * SP.nq;
      mk[kk] = __ldcg(pml + col);
      lk[kk] = __ldcg(pml + SP.nq + col);
      const float* pa = part_acc + ((base + k) * SP.nq + col) * RB_HEAD_DIM + d0;
#pragma unroll
      for (int v = 0; v < 4; ++v) ak[kk][v] = __ldcg(reinterpret_cast<const float4*>(pa + 4 * v));
    }
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      if (k0 + kk >= np) break;
      const float mn = fmaxf(mt, mk[kk]);
      const float so = (mt == -INFINITY) ? 0.f : fast_exp2(mt - mn);
      const float sk = fast_exp2(mk[kk] - mn);
      lt = relay_fold(lt, so, lk[kk], sk);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        O[v].x = relay_fold(O[v].x, so, ak[kk][v].x, sk);
        O[v].y = relay_fold(O[v].y, so, ak[kk][v].y, sk);
        O[v].z = relay_fold(O[v].z, so, ak[kk][v].z, sk);
        O[v].w = relay_fold(O[v].w, so, ak[kk][v].w, sk);
      }
      mt = mn;
    }
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
  int bt[32];                                  // block ids of context blocks it.bt0 .. it.bt0 + 31
};

template <int R>
struct CtaSmem {
  static constexpr int kDepth = CtxCfg<R>::kDepth;
  static constexpr int kNB = CtxCfg<R>::kNB;
  // [kIQ][R][128] bf16 query rows, then one zero row (MMA rows past R)
  static constexpr int kOffQ = kWorkers * kDepth * kSlotBytes;
  static constexpr int kOffQZero = kOffQ + kIQ * R * kRowBytes;
  static constexpr int kOffAcc = kOffQZero + kRowBytes;  // [kNB][kWorkers][R][kAccStride] f32
  static constexpr int kOffML = kOffAcc + kNB * kWorkers * R * kAccStride * 4;  // [kNB][kWorkers][R][2]
  static constexpr int kOffItems = (kOffML + kNB * kWorkers * R * 8 + 15) & ~15;  // [kIQ] ItemSlot
  static constexpr int kOffBar = (kOffItems + kIQ * static_cast<int>(sizeof(ItemSlot<R>)) + 7) & ~7;
  static constexpr int kMaxDefer = CtxCfg<R>::kMaxDefer;
  static constexpr int kOffDefer = kOffBar + (3 * kIQ + 2 * kNB) * 8;  // [1 + kMaxDefer] int
  // [R][kAccStride] f32: rows of a split combine (merger only)
  static constexpr int kOffComb = (kOffDefer + (1 + kMaxDefer) * 4 + 15) & ~15;
  static constexpr int kBytes = kOffComb + R * kAccStride * 4;
  static_assert(kBytes <= 113 * 1024, "two context CTAs must fit one SM");
};

// Diagnostics build only: per-warp event trace of CTAs 0 and 1 (clock64,
// 256 events per warp) at debug_ts + 6144 * 8, read by
// profiles/diag_ctx_trace.py.
struct WarpTrace {
  unsigned long long* p;
  int n;
  __device__ __forceinline__ void init(unsigned long long* dts_ctx, int warp, int lane) {
    p = nullptr;
    n = 0;
    if (RB_DIAG && dts_ctx != nullptr && blockIdx.x < 2 && lane == 0)
      p = dts_ctx - static_cast<long long>(blockIdx.x) * 8 + 6144 * 8 + (blockIdx.x * 6 + warp) * 512;
  }
  __device__ __forceinline__ void ev(int code) {
    if (RB_DIAG && p != nullptr && n < 256) {
      p[2 * n] = clock64();
      p[2 * n + 1] = static_cast<unsigned long long>(code);
    }
    ++n;
  }
};

template <int R, bool LAZY>
__global__ void __launch_bounds__(kCtxThreadsPC, RB_CTX_MINB)
    ctx_cta_kernel(const CtxArgs a, int n_items, int n_z) {
  using SM = CtaSmem<R>;
  constexpr int kDepth = SM::kDepth, kNB = SM::kNB;
  // relay fusion: system parts per batch of loads (C4's 6-part units with
  // 4-row items want 8; the 1-2-row items of C2 / C3 see <= 4 parts, and the
  // smaller batch keeps the merger's per-item code short)
  constexpr int kRBr = R >= 4 ? kRB : (kRB < 4 ? kRB : 4);
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_pre = (a.s_prefix + kChunk - 1) / kChunk;
  const int n_split = a.n_split;
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
      mbar_init(&i_full[i], 32);   // every scheduler lane: cp.async arrive (query rows)
      mbar_init(&i_empty[i], kWorkers + 1);  // workers + merger
    }
    for (int i = 0; i < kNB; ++i) {
      mbar_init(&m_full[i], kWorkers);
      mbar_init(&m_empty[i], 1);
    }
    fence_mbar_init();
  }
  // the zero query row stands in for MMA rows past R
  if (threadIdx.x < kRowBytes / 16)
    reinterpret_cast<uint4*>(smem + SM::kOffQZero)[threadIdx.x] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  pdl_launch_dependents();
  unsigned long long* dts = (RB_DIAG && a.debug_ts) ? a.debug_ts + blockIdx.x * 8 : nullptr;
  if (dts && threadIdx.x == 0) {
    dts[0] = global_timer_ns();
    dts[1] = smid();
  }

  WarpTrace tr;
  tr.init(dts, warp, lane);
  if (warp == 0) {
    // ----------------------------------------------------------- scheduler
    // Software pipeline: publish item j, load item j+1's metadata, claim
    // item j+3 (the atomic resolves while the scheduler waits for a free
    // queue slot).  With `sched` every item is claimed from the global
    // counter (the first three in one atomic), so CTAs that start late --
    // after the concurrent system kernel frees their SM -- still share the
    // remaining work; without it the order is static (b + k * grid).
    // Item = ((request * hkv + head) * n_z + row tile) * n_split + split.
    int* sched = a.sched;
    const bool paged = a.ctx.block_table != nullptr;
    const int per_req = n_z * a.hkv * n_split;
    struct Raw {
      int item, qs0, qs1, clen, bte, bt0;
      long long roff;
    };
    auto load_raw = [&](int item) {
      Raw w;
      w.item = item;
      w.qs0 = w.qs1 = w.clen = w.bte = w.bt0 = 0;
      w.roff = 0;
      if (item < n_items) {
        int r = item / per_req;
        if (a.req_order != nullptr) {
          // a permutation of the requests (an out-of-range entry falls back to
          // the position itself: never an out-of-bounds read)
          const int ro = __ldg(a.req_order + r);
          r = static_cast<unsigned>(ro) < static_cast<unsigned>(a.b) ? ro : r;
        }
        const int sp = item % n_split;
        w.qs0 = __ldg(a.q_start + r);
        w.qs1 = __ldg(a.q_start + r + 1);
        w.clen = __ldg(a.ctx_lens + r);
        if (a.ctx.req_offset != nullptr) w.roff = __ldg(a.ctx.req_offset + r);
        if (paged) {
          // the split's first context block (splits start on chunk
          // boundaries; a chunk never straddles blocks when block_size % 16
          // == 0, the only case the table window is used for)
          const int c0 = max(0, sp * a.split_chunks - n_pre) * kChunk;
          w.bt0 = c0 / a.ctx.block_size;
          // rows of the table are bt_stride long: entries past it are never read
          if (w.bt0 + lane < a.ctx.bt_stride)
            w.bte = __ldg(a.ctx.block_table + static_cast<long long>(r) * a.ctx.bt_stride + w.bt0 + lane);
        }
      }
      return w;
    };
    const int G = static_cast<int>(gridDim.x);
    // Long items (a.claim_lazy): claim one item at a time, the next only
    // once the one before the current is done, so a CTA never holds more
    // than two unfinished items -- claiming three ahead let the CTAs that
    // started early hoard the pool's last long items (C4: their tail ran
    // ~10 us past the others').
    // (a compile-time variant: the lazy loop's code in every kernel cost the
    // short-item decode steps ~2 us -- instruction footprint)
    const bool lazy = LAZY && sched != nullptr;
    int id0 = blockIdx.x, id1 = blockIdx.x + G, id2 = blockIdx.x + 2 * G;
    if (sched != nullptr) {
      int base = 0;
      if (lane == 0) base = atomicAdd(sched, lazy ? 1 : 3);
      base = __shfl_sync(0xffffffffu, base, 0);
      id0 = base;
      id1 = base + 1;
      id2 = base + 2;
    }
    // publish item `item` (metadata `cur`) into queue slot qs (the slot is free)
    auto publish = [&](const Raw& cur, int item, int qs) {
      ItemSlot<R>& slot = iq[qs];
      CtxItem<R> it;
      it.bt0 = cur.bt0;
      it.roff = cur.roff;
      {
        it.sp = item % n_split;
        const int grp = item / n_split;
        it.grp = grp;
        it.z = grp % n_z;
        it.h = (grp / n_z) % a.hkv;
        it.r = grp / (n_z * a.hkv);
        if (a.req_order != nullptr) {
          const int ro = __ldg(a.req_order + it.r);
          it.r = static_cast<unsigned>(ro) < static_cast<unsigned>(a.b) ? ro : it.r;
        }
        it.row0 = cur.qs0;
        it.m_r = cur.qs1 - cur.qs0;
        it.nrows = it.m_r * a.g;
        it.c_r = cur.clen;
        const int rb = it.z * R;
        it.k0 = 0;
        it.nsplit = 1;
        if (rb >= it.nrows) {
          it.max_lim = 0;
          it.n_chunks = 0;
        } else {
          const int t_last = (min(rb + R, it.nrows) - 1) / a.g;
          it.max_lim = a.causal ? it.c_r - it.m_r + t_last + 1 : it.c_r;
          const int total = n_pre + (it.max_lim + kChunk - 1) / kChunk;
          it.n_chunks = total;
          if (n_split > 1) {
            // split sp: chunks [sp L, (sp+1) L), the last valid split takes the rest
            const int L = a.split_chunks;
            it.nsplit = min(n_split, max(1, (total + L - 1) / L));
            it.k0 = it.sp * L;
            it.n_chunks = it.sp >= it.nsplit ? 0
                          : (it.sp == it.nsplit - 1 ? total - it.sp * L : L);
          }
        }
      }
      const int rbase = it.z * R;
      const int nvalid = it.n_chunks > 0 ? max(0, min(R, it.nrows - rbase)) : 0;
      slot.bt[lane] = cur.bte;
      if (lane == 0) {
        slot.it = it;
        slot.item = item;
      }
      __syncwarp();
      if (a.k_new != nullptr && it.n_chunks > 0 && it.m_r > 0) {
        // fused append: the item whose chunk range covers the request's new
        // tokens (context positions c_r - m_r .. c_r - 1) writes their K / V
        // rows of head h into the pool first; the i_meta arrive below
        // releases the stores to the CTA's workers (items of other row tiles
        // covering the same tokens write identical bytes)
        const int first_new = n_pre + (it.c_r - it.m_r) / kChunk;
        const int last_new = n_pre + (it.c_r - 1) / kChunk;
        if (it.k0 <= last_new && first_new < it.k0 + it.n_chunks) {
          for (int e = lane; e < it.m_r * 32; e += 32) {
            const int row = it.row0 + (e >> 5), c16 = e & 15;
            const bool is_v = (e & 16) != 0;
            const long long src = (static_cast<long long>(row) * a.hkv + it.h) * RB_HEAD_DIM + c16 * 8;
            const uint4 val = *reinterpret_cast<const uint4*>((is_v ? a.v_new : a.k_new) + src);
            const int slot = __ldg(a.slot_mapping + row);
            const int bs = a.ctx.block_size;
            const long long dst = static_cast<long long>(slot / bs) * a.ctx.stride_block +
                                  static_cast<long long>(slot % bs) * a.ctx.stride_tok +
                                  static_cast<long long>(it.h) * a.ctx.stride_head + c16 * 8;
            *reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(is_v ? a.ctx.v : a.ctx.k) + dst) = val;
          }
          __syncwarp();
        }
      }
      if (lane == 0) mbar_arrive(&i_meta[qs]);
      __syncwarp();
      // query rows of the item: 16-byte cp.async by all lanes (the LSU path
      // also reads queries straight from pinned host memory, the zero-copy
      // e2e step), then every lane arrives on i_full once its copies land
      for (int c = lane; c < nvalid * 16; c += 32) {
        const int li = rbase + (c >> 4);
        const int t = li / a.g, jj = li % a.g;
        const __nv_bfloat16* qp = a.q + static_cast<long long>(it.row0 + t) * a.q_row_stride +
                                  static_cast<long long>(it.h * a.g + jj) * a.q_head_stride + (c & 15) * 8;
        cp_async_16(smem + SM::kOffQ + (qs * R + (c >> 4)) * kRowBytes + (c & 15) * 16, qp, 16u);
      }
      cp_async_mbar_arrive(&i_full[qs]);
    };
    auto publish_end = [&](int qs) {
      ItemSlot<R>& slot = iq[qs];
      if (lane == 0) {
        slot.item = -1;
        mbar_arrive(&i_meta[qs]);
      }
      __syncwarp();
      mbar_arrive(&i_full[qs]);
    };
    if (lazy) {
      // at most two unfinished items: claim item j+1 once item j-1 is done
      Raw cur = load_raw(id0);
      for (int j = 0;; ++j) {
        const int qs = j % kIQ;
        mbar_wait(&i_empty[qs], ((j / kIQ) & 1) ^ 1);
        if (cur.item >= n_items) {
          publish_end(qs);
          break;
        }
        publish(cur, cur.item, qs);
        if (j >= 1) mbar_wait(&i_empty[(j - 1) % kIQ], static_cast<uint32_t>(((j - 1) / kIQ) & 1));
        int pn = 0;
        if (lane == 0) pn = atomicAdd(sched, 1);
        pn = __shfl_sync(0xffffffffu, pn, 0);
        tr.ev(620000 + pn);
        cur = load_raw(pn);
      }
    } else {
      Raw cur = load_raw(id0);
      for (int j = 0;; ++j) {
        const int item = cur.item;
        const int qs = j % kIQ;
        // claim item j+3 and load item j+1 while this one is published
        int p = id2 + G;
        tr.ev(600000 + item);
        if (sched != nullptr && lane == 0) p = atomicAdd(sched, 1);
        const Raw nxt = load_raw(id1);
        mbar_wait(&i_empty[qs], ((j / kIQ) & 1) ^ 1);
        tr.ev(610000 + item);
        if (item >= n_items) {
          publish_end(qs);
          break;
        }
        publish(cur, item, qs);
        cur = nxt;
        id1 = id2;
        id2 = (sched != nullptr) ? __shfl_sync(0xffffffffu, p, 0) : p;
        tr.ev(620000 + id2);
      }
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
    // dims) and finishes each row: split items park their partial in the
    // split workspace and the last split of the item combines all of them
    // in split order; then either the relay fusion with the system parts
    // (or parking the context partial until its system unit is published),
    // or the final output (+ optional fusion with a given o_sys / lse_sys).
    bool waited = false;
    int jp = 0;  // queue cursor
    // diagnostics (debug timestamps only): waits and work of the merger
    unsigned long long d_mfull = 0, d_work = 0, d_imeta = 0, d_t = 0;
    // relay with <= 256 system units: the publication counters are polled in
    // the background (lane l: units l, l + 32; loads issued one item ahead,
    // consumed at the next) into a bitmask of published units, so deciding
    // fuse-or-park costs no round trip on the merger's critical path
    const bool poll = a.ctx_part != nullptr && a.sys_plan.n_units <= 32 * kPollSlots;
    uint32_t pub = 0;
    int pv[kPollSlots], np[kPollSlots];
#pragma unroll
    for (int k = 0; k < kPollSlots; ++k) {
      const int u = lane + 32 * k;
      np[k] = (poll && u < a.sys_plan.n_units) ? rb_unit_parts(&a.sys_plan, u) : 0x7fffffff;
      pv[k] = np[k] != 0x7fffffff ? ld_acquire_gpu(a.sys_ready + u) : 0;
    }
    const int d0 = lane * 4;
    int* defer = reinterpret_cast<int*>(smem + SM::kOffDefer);
    // (row, head) pair of item row li (rows of an item: request row0 + li / g,
    // group member li % g); system units are power-of-two row tiles
    const int nq_sh = __ffs(a.sys_plan.nq) - 1;
    auto item_row_ref = [&](const CtxItem<R>& itm, int li) -> RowRef {
      const int t = a.g == 1 ? li : li / a.g, jj = li - t * a.g;
      const int row = itm.row0 + t;
      const int f = row * a.g + jj;
      RowRef rr;
      rr.oidx = static_cast<long long>(row) * a.hq + itm.h * a.g + jj;
      rr.u = itm.h * a.sys_plan.n_qt + (f >> nq_sh);
      rr.col = f & (a.sys_plan.nq - 1);
      return rr;
    };
    // the last step of a (row, head): relay fusion / park, or output
    auto finish = [&](float4 O, float M, float Ls, const RowRef& rr, bool use_pre, RelayParts<kRBr>& pp) {
      const long long oidx = rr.oidx;
      if (a.ctx_part != nullptr) {
        const bool full = defer[0] >= SM::kMaxDefer;
        if (use_pre) {
          relay_fuse_finish<kRBr>(a.sys_plan, pp, oidx, a.sys_part_acc, a.sys_part_ml, O, M, Ls, a.out,
                            a.out_fp32, a.lse_out, lane);
        } else if (poll ? (relay_unit_published(rr.u, pub) ||
                           (full && relay_unit_ready(a.sys_plan, rr.u, a.sys_ready, lane, true)))
                        : relay_unit_ready(a.sys_plan, rr.u, a.sys_ready, lane, full)) {
          relay_fuse_pair<kRBr>(a.sys_plan, rr, a.sys_part_acc, a.sys_part_ml, O, M, Ls, a.out,
                          a.out_fp32, a.lse_out, lane);
        } else {
          float* dst = a.ctx_part + oidx * kPartStride;
          __stcg(reinterpret_cast<float4*>(dst + d0), O);
          if (lane == 0) __stcg(reinterpret_cast<float2*>(dst + 128), make_float2(M, Ls));
          __syncwarp();
          if (lane == 0) defer[1 + defer[0]++] = static_cast<int>(oidx);
          __syncwarp();
        }
        return;
      }
      float o[4] = {O.x, O.y, O.z, O.w};
      float lse2;
      {
        const float inv = (Ls > 0.f) ? 1.f / Ls : 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) o[e] *= inv;
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
    };

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
      const bool split = it.nsplit > 1;
      const int nslots = n_split;
      // relay: if row 0's system unit is already published, issue its
      // parts' loads now so they land while the workers finish the item
      bool pre = false;
      RelayParts<kRBr> pp;
      if (poll) {
        // fold in the previous poll, then issue the next one
#pragma unroll
        for (int k = 0; k < kPollSlots; ++k)
          if (pv[k] >= np[k]) pub |= 1u << k;
        __syncwarp();  // the acquiring lanes' loads precede every lane's part reads
#pragma unroll
        for (int k = 0; k < kPollSlots; ++k)
          if (np[k] != 0x7fffffff && !((pub >> k) & 1)) pv[k] = ld_acquire_gpu(a.sys_ready + lane + 32 * k);
      }
      if (a.ctx_part != nullptr && !split && it.z * R < it.nrows) {
        const RowRef r0 = item_row_ref(it, it.z * R);
        pre = poll ? relay_unit_published(r0.u, pub)
                   : relay_unit_ready(a.sys_plan, r0.u, a.sys_ready, lane, false);
        if (pre) pp = relay_parts_begin<kRBr>(a.sys_plan, r0, a.sys_part_acc, a.sys_part_ml, lane);
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
      tr.ev(700000 + item);
      mbar_wait(&m_full[mb], mph);
      tr.ev(710000 + item);
      if (dts) {
        const unsigned long long t1 = global_timer_ns();
        d_mfull += t1 - d_t;
        d_t = t1;
      }
      const float* bacc = s_acc + mb * kWorkers * R * kAccStride;
      const float* bml = s_ml + mb * kWorkers * R * 2;
      const int rbase = it.z * R;
      const int nrow = min(R, it.nrows - rbase);
      // output row of item row i: request row0 + t, group member jj
      auto row_oidx = [&](int i) -> long long {
        const int li = rbase + i;
        const int t = li / a.g, jj = li % a.g;
        return static_cast<long long>(it.row0 + t) * a.hq + it.h * a.g + jj;
      };
      // all rows of the item in one published system unit: grouped fusion
      bool grouped = false;
      if (RB_RELAY_GROUPED && R > 1 && !split && poll && nrow == R) {
        const int u0 = item_row_ref(it, rbase).u;
        grouped = u0 == item_row_ref(it, rbase + R - 1).u && relay_unit_published(u0, pub);
      }
      if (grouped)
        relay_fuse_rows<R>(a.sys_plan, item_row_ref(it, rbase + lane / (32 / R)), bacc, bml, a.sys_part_acc,
                           a.sys_part_ml, a.out, a.out_fp32, a.lse_out, lane);
#pragma unroll 1
      for (int i = 0; i < (grouped ? 0 : nrow); ++i) {
        const long long oidx = row_oidx(i);
        float M = -INFINITY;
#pragma unroll
        for (int k = 0; k < kWorkers; ++k) M = fmaxf(M, bml[(k * R + i) * 2]);
        float Ls = 0.f;
        float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
        if (M != -INFINITY) {
#pragma unroll
          for (int k = 0; k < kWorkers; ++k) {
            const float mk = bml[(k * R + i) * 2];
            const float wt = (mk == -INFINITY) ? 0.f : fast_exp2(mk - M);
            Ls = fmaf(bml[(k * R + i) * 2 + 1], wt, Ls);
            const float4 av = *reinterpret_cast<const float4*>(bacc + (k * R + i) * kAccStride + d0);
            O.x = fmaf(av.x, wt, O.x);
            O.y = fmaf(av.y, wt, O.y);
            O.z = fmaf(av.z, wt, O.z);
            O.w = fmaf(av.w, wt, O.w);
          }
        }
        if (split) {
          float* dst = a.split_part + (oidx * nslots + it.sp) * kPartStride;
          __stcg(reinterpret_cast<float4*>(dst + d0), O);
          if (lane == 0) __stcg(reinterpret_cast<float2*>(dst + 128), make_float2(M, Ls));
        } else {
          finish(O, M, Ls, item_row_ref(it, rbase + i), i == 0 && pre, pp);
        }
      }
      __syncwarp();
      tr.ev(720000 + item);
      if (lane == 0) mbar_arrive(&m_empty[mb]);
      if (split) {
        // the last split of the item to finish combines every split's
        // partial in split order (bitwise independent of the arrival order)
        int last = 0;
        if (lane == 0) {
          __threadfence();
          last = atomicAdd(a.split_cnt + it.grp, 1) == it.nsplit - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          __threadfence();
          // The R rows combine in parallel: lane group rg = lane / LPR owns
          // row rg, lane li of the group dims [li DPL, (li + 1) DPL).  Per
          // row: the reference max over the splits (the group's lanes take
          // every LPR-th split), then O and l as exp2-weighted sums in split
          // order with KB partials' loads in flight -- deterministic (fixed
          // order and grouping) and no longer one L2 round trip per split
          // per row (b = 2, c = 32k: ~37 splits x 4 rows).
          {
            constexpr int LPR = 32 / R, DPL = RB_HEAD_DIM / LPR, NV = DPL / 4;
            constexpr int KB = R >= 8 ? 1 : 8 / R;
            float* comb = reinterpret_cast<float*>(smem + SM::kOffComb);
            const int rg = lane / LPR, li = lane % LPR;
            const bool rv = rg < nrow;
            const float* src = a.split_part + row_oidx(rv ? rg : 0) * nslots * kPartStride;
            float mloc = -INFINITY;
            for (int k = li; k < it.nsplit; k += LPR) mloc = fmaxf(mloc, __ldcg(src + k * kPartStride + 128));
#pragma unroll
            for (int off = LPR / 2; off > 0; off >>= 1)
              mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, off));
            const float M = mloc;
            float4 acc[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            float Ls = 0.f;
            for (int k0 = 0; k0 < it.nsplit; k0 += KB) {
              float4 Ok[KB][NV];
              float2 mlk[KB];
#pragma unroll
              for (int kk = 0; kk < KB; ++kk) {
                const float* sk = src + min(k0 + kk, it.nsplit - 1) * kPartStride;
#pragma unroll
                for (int v = 0; v < NV; ++v)
                  Ok[kk][v] = __ldcg(reinterpret_cast<const float4*>(sk + li * DPL + 4 * v));
                mlk[kk] = __ldcg(reinterpret_cast<const float2*>(sk + 128));
              }
#pragma unroll
              for (int kk = 0; kk < KB; ++kk) {
                if (k0 + kk >= it.nsplit) break;
                const float w = (mlk[kk].x == -INFINITY) ? 0.f : fast_exp2(mlk[kk].x - M);
                Ls = fmaf(mlk[kk].y, w, Ls);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                  acc[v].x = fmaf(Ok[kk][v].x, w, acc[v].x);
                  acc[v].y = fmaf(Ok[kk][v].y, w, acc[v].y);
                  acc[v].z = fmaf(Ok[kk][v].z, w, acc[v].z);
                  acc[v].w = fmaf(Ok[kk][v].w, w, acc[v].w);
                }
              }
            }
            if (rv) {
#pragma unroll
              for (int v = 0; v < NV; ++v)
                *reinterpret_cast<float4*>(comb + rg * kAccStride + li * DPL + 4 * v) = acc[v];
              if (li == 0) {
                comb[rg * kAccStride + 128] = M;
                comb[rg * kAccStride + 129] = Ls;
              }
            }
            __syncwarp();
#pragma unroll 1
            for (int i = 0; i < nrow; ++i) {
              const float4 O = *reinterpret_cast<const float4*>(comb + i * kAccStride + d0);
              finish(O, comb[i * kAccStride + 128], comb[i * kAccStride + 129], item_row_ref(it, rbase + i), false,
                     pp);
            }
          }
          __syncwarp();
          if (lane == 0) a.split_cnt[it.grp] = 0;  // rearm for the next launch
        }
      }
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
  uint8_t* ring_p = smem + w * kDepth * kSlotBytes;

  // issue cursor: queue item ji, next chunk ki (= w mod kWorkers), local to
  // the item's split; the global chunk index is iss_k0 + ki
  int ji = 0, ki = w, iss_item = 0, iss_bte = 0, iss_bt0 = 0;
  int iss_r = 0, iss_h = 0, iss_lim = 0, iss_nch = 0, iss_k0 = 0;
  long long iss_roff = 0;
  bool have_iss = false;
  int issued = 0, consumed = 0, iss_sl = 0;
  // Fast issue mode (paged, blocks of a multiple of 16 tokens whose rows are
  // 256 B apart, no prefix segment, <= 32 chunks of this worker in the
  // item): when the cursor enters an item, lane l resolves the K address of
  // the worker's l-th chunk of it (block-table window or a direct load, all
  // lanes in parallel); issuing a chunk is then one 64-bit shuffle and 16
  // immediate-offset copies.  V sits at a fixed distance from K.
  bool iss_fast = false;
  const __nv_bfloat16* lane_kaddr = a.ctx.k;
  const long long vdiff = a.ctx.v - a.ctx.k;
  const bool fast_ok = a.ctx.block_table != nullptr && a.ctx.block_size % kChunk == 0 &&
                       a.ctx.stride_tok == RB_HEAD_DIM && n_pre == 0;

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
        iss_k0 = iq[qs].it.k0;
        iss_bt0 = iq[qs].it.bt0;
        iss_roff = iq[qs].it.roff;
        iss_bte = iq[qs].bt[lane];
        have_iss = true;
        ki = w;
        iss_fast = fast_ok && iss_item >= 0 && iss_nch <= w + 4 * 32;
        if (iss_fast) {
          const int kk = w + 4 * lane;                 // this lane's chunk of the worker
          const int kc = iss_k0 + min(kk, iss_nch - 1);  // context chunk (n_pre == 0)
          const int bi = a.ctx.block_size == kChunk ? kc : kc * kChunk / a.ctx.block_size;
          const int rel = bi - iss_bt0;
          int blk = __shfl_sync(0xffffffffu, iss_bte, rel & 31);
          if (rel < 0 || rel >= 32)
            blk = __ldg(a.ctx.block_table + static_cast<long long>(iss_r) * a.ctx.bt_stride + bi);
          lane_kaddr = a.ctx.k + static_cast<long long>(blk) * a.ctx.stride_block +
                       static_cast<long long>(kc * kChunk - bi * a.ctx.block_size) * RB_HEAD_DIM +
                       static_cast<long long>(iss_h) * a.ctx.stride_head;
        }
      }
      if (iss_item < 0) return;
      if (ki >= iss_nch) {
        ++ji;
        have_iss = false;
        continue;
      }
      uint8_t* dst = ring_p + iss_sl * kSlotBytes;
      if (iss_fast) {
        const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(__shfl_sync(
            0xffffffffu, reinterpret_cast<unsigned long long>(lane_kaddr), ki >> 2));
        const int n = iss_lim - (iss_k0 + ki) * kChunk;
        if (n >= kChunk)
          chunk_cp_async_full(dst, kb, kb + vdiff, lane);
        else
          chunk_cp_async(dst, kb, kb + vdiff, RB_HEAD_DIM, n, lane);
        asm volatile("cp.async.commit_group;" ::: "memory");
        ++issued;
        iss_sl = (iss_sl + 1 == kDepth) ? 0 : iss_sl + 1;
        ki += kWorkers;
        continue;
      }
      const int k = iss_k0 + ki;
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
          const int bi = a.ctx.block_size == kChunk ? k - n_pre : t0 / a.ctx.block_size;
          const int v0 = __shfl_sync(0xffffffffu, iss_bte, (bi - iss_bt0) & 31);
          const int blk = (bi - iss_bt0 >= 0 && bi - iss_bt0 < 32)
                              ? v0
                              : __ldg(a.ctx.block_table +
                                      static_cast<long long>(iss_r) * a.ctx.bt_stride + bi);
          off = static_cast<long long>(blk) * a.ctx.stride_block +
                static_cast<long long>(t0 - bi * a.ctx.block_size) * a.ctx.stride_tok;
        } else {
          off = 0;
          rows_ok = false;
        }
        off += iss_h * a.ctx.stride_head;
        kb += off;
        vb += off;
        if (!rows_ok) chunk_cp_async_rows(dst, a.ctx, iss_r, t0, iss_h, n, lane);
      }
      if (rows_ok) {
        if (n == kChunk && tok_stride == RB_HEAD_DIM)
          chunk_cp_async_full(dst, kb, vb, lane);
        else
          chunk_cp_async(dst, kb, vb, tok_stride, n, lane);
      }
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
    tr.ev(400000 + jc);
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
      tr.ev(100000 + issued);
      try_issue(jc);
      tr.ev(110000 + issued);
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
#if RB_CTX_PAIRS
      if (k + kWorkers < it.n_chunks && issued - consumed >= 2) {
        // two of this worker's chunks (rings slots con_sl, con_sl + 1) in one pass
        const int newer2 = issued - consumed - 2;
        if (kDepth >= 3 && newer2 >= 1)
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        else
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        const int kga = it.k0 + k, kgb = kga + kWorkers;
        const bool pa = kga < n_pre, pb = kgb < n_pre;
        const int k0a = (pa ? kga : kga - n_pre) * kChunk, k0b = (pb ? kgb : kgb - n_pre) * kChunk;
        const bool ma = k0a + kChunk > (pa ? a.s_prefix : ctx_nomask);
        const bool mbk = k0b + kChunk > (pb ? a.s_prefix : ctx_nomask);
        const int sl2 = (con_sl + 1 == kDepth) ? 0 : con_sl + 1;
        cmp.chunk2(ring_p + con_sl * kSlotBytes, ring_p + sl2 * kSlotBytes, k0a, k0b, pa, pb, ma, mbk,
                   a, lane);
        __syncwarp();
        consumed += 2;
        con_sl = (sl2 + 1 == kDepth) ? 0 : sl2 + 1;
        k += 2 * kWorkers;
        continue;
      }
#endif
      // chunk `consumed` is this warp's commit group number `consumed`; the
      // groups committed after it may stay in flight
      const int newer = issued - consumed - 1;
      if (kDepth >= 3 && newer >= 2)
        asm volatile("cp.async.wait_group 2;" ::: "memory");
      else if (newer >= 1)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();  // every lane's copies of the chunk are visible to the warp
      tr.ev(210000 + consumed);
      const int kg = it.k0 + k;
      const bool pre = kg < n_pre;
      const int key0 = (pre ? kg : kg - n_pre) * kChunk;
      const bool mask = key0 + kChunk > (pre ? a.s_prefix : ctx_nomask);
#ifndef RB_CTX_NOCOMPUTE
      cmp.chunk(ring_p + con_sl * kSlotBytes, key0, pre, it.max_lim, mask, a, lane);
#else
      (void)key0;  // diagnostics variant: the data path alone (wrong results)
#endif
      __syncwarp();  // every lane's reads precede the refill of this slot
      tr.ev(300000 + consumed);
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
    float* macc = s_acc + (mb * kWorkers + w) * R * kAccStride;
    float* mml = s_ml + (mb * kWorkers + w) * R * 2;
    cmp.handoff(macc, mml, lane);
    __syncwarp();
    tr.ev(500000 + mi);
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
  cudaError_t e = cudaFuncSetAttribute(ctx_cta_kernel<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(ctx_cta_kernel<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ctx_cta_kernel<R, false>, kCtxThreadsPC, smem);
  if (e != cudaSuccess) return e;
  const int grid = max(1, min(n_items, sms * max(per_sm, 1)));
  // fewer than three items per CTA: claiming three at once would leave most
  // CTAs without work (C1: 128 items, 43 CTAs busy) -- claim one at a time
  CtxArgs la = a;
  if (RB_CLAIM_LAZY && n_items < 3 * grid) la.claim_lazy = 1;
  // PDL: the relay step's context kernel starts as soon as the system kernel
  // has triggered (it runs on the SMs the system kernel leaves free); the
  // other modes wait for their predecessor before the first output write.
  e = la.claim_lazy
          ? launch_pdl(ctx_cta_kernel<R, true>, dim3(grid), dim3(kCtxThreadsPC), smem, stream, la, n_items, n_z)
          : launch_pdl(ctx_cta_kernel<R, false>, dim3(grid), dim3(kCtxThreadsPC), smem, stream, la, n_items, n_z);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int ctx_resident_ctas(int sms) { return 2 * sms; }

cudaError_t launch_context_attention(const CtxArgs& a, int max_rows, cudaStream_t stream) {
  // max_rows = max over requests of m_r * g
  const int R = rb_ctx_rows(max_rows);
  const int n_z = (max_rows + R - 1) / R;
  const long long n_items = static_cast<long long>(a.b) * a.hkv * n_z * a.n_split;
  if (n_items == 0) return cudaSuccess;
  if (n_items > 0x7fffffffLL) return cudaErrorInvalidValue;
  switch (R) {
    case 1: return launch_ctx_r<1>(a, static_cast<int>(n_items), n_z, stream);
    case 2: return launch_ctx_r<2>(a, static_cast<int>(n_items), n_z, stream);
    case 4: return launch_ctx_r<4>(a, static_cast<int>(n_items), n_z, stream);
    default: return launch_ctx_r<8>(a, static_cast<int>(n_items), n_z, stream);
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

// Zero-copy relay step with the queries in pinned host memory: one pass
// copies them into device memory ([rows][hq][128], 16 B per thread per
// iteration, as many loads in flight as the SMs hold) before the system and
// context kernels read them -- both kernels used to read the host rows
// themselves, the system kernel once per stream-K part of a unit, so ~1.5 MB
// crossed PCIe for 0.43 MB of queries at C2.  The system kernel launches as a
// PDL dependent at once and prefetches its K/V tiles; its query loader waits
// for this grid.
__global__ void __launch_bounds__(256) q_stage_kernel(const __nv_bfloat16* __restrict__ q,
                                                      long long row_stride, long long head_stride,
                                                      int n_rows, int hq,
                                                      __nv_bfloat16* __restrict__ dst) {
  pdl_launch_dependents();
  const long long chunks = static_cast<long long>(n_rows) * hq * 16;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < chunks; i += 256LL * gridDim.x) {
    const int c = static_cast<int>(i & 15);
    const long long rh = i >> 4;
    const int row = static_cast<int>(rh / hq), h = static_cast<int>(rh % hq);
    reinterpret_cast<uint4*>(dst)[i] =
        *reinterpret_cast<const uint4*>(q + row * row_stride + h * head_stride + c * 8);
  }
}

cudaError_t launch_q_stage(const __nv_bfloat16* q, long long row_stride, long long head_stride,
                           int n_rows, int hq, __nv_bfloat16* dst, int sms, cudaStream_t stream) {
  const long long chunks = static_cast<long long>(n_rows) * hq * 16;
  if (chunks == 0) return cudaSuccess;
  const long long want = (chunks + 255) / 256;
  const int grid = static_cast<int>(want < 4LL * sms ? want : 4LL * sms);
  cudaError_t e = launch_pdl(q_stage_kernel, dim3(grid), dim3(256), 0, stream, q, row_stride, head_stride,
                             n_rows, hq, dst);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
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
