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
// kv head, row tile); 4 warps stride over 16-token chunks.  Each warp owns a
// private 2-slot smem ring filled by cp.async.bulk (one 4 KB copy per paged
// (block, head) run of K and of V, completing on an mbarrier), so a whole
// 128-token context is in flight at once without costing registers.  A
// half-warp reads one 256-byte key row from smem (16 B per lane), dot
// products reduce with 4 xor-shuffles, online softmax in the log2 domain per
// half-warp, then an smem merge of the 8 partial states, the fusion, and one
// coalesced store per row.
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

template <int R>
struct RowState {
  float m[R], l[R], acc[R][8];
};

// One 16-key chunk for a half-warp: keys key0 + 2p + hw, p = 0..7, K/V rows
// already in registers.  `lim[i]` is the exclusive key bound of row i inside
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
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) s = fmaf(qf[i][e], kf[e], s);
      x[i][p] = s;
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

// Work item = (request r, kv head h, row tile z).  Geometry of one item.
template <int R>
struct CtxItem {
  int r, h, z, row0, m_r, nrows, c_r, max_lim, n_chunks;
  long long roff;  // ragged mode: first token of request r
};

template <int R>
__device__ __forceinline__ CtxItem<R> ctx_item(const CtxArgs& a, int item, int n_z, int n_pre) {
  CtxItem<R> it;
  it.z = item % n_z;
  it.h = (item / n_z) % a.hkv;
  it.r = item / (n_z * a.hkv);
  it.row0 = __ldg(a.q_start + it.r);
  it.m_r = __ldg(a.q_start + it.r + 1) - it.row0;
  it.nrows = it.m_r * a.g;
  it.c_r = __ldg(a.ctx_lens + it.r);
  it.roff = a.ctx.req_offset != nullptr ? __ldg(a.ctx.req_offset + it.r) : 0;
  const int rbase = it.z * R;
  if (rbase >= it.nrows) {
    it.max_lim = 0;
    it.n_chunks = 0;
    return it;
  }
  const int t_last = (min(rbase + R, it.nrows) - 1) / a.g;
  it.max_lim = a.causal ? it.c_r - it.m_r + t_last + 1 : it.c_r;
  it.n_chunks = n_pre + (it.max_lim + kChunk - 1) / kChunk;
  return it;
}

// Everything a warp needs to start an item, loaded lane-parallel one item
// ahead: geometry, this lane's 8 query dims per row, and (lanes j, j+32) the
// block-table entries of context chunks j and j + 32.
template <int R>
struct ItemPrefetch {
  CtxItem<R> it;
  float qf[R][8];
  int bt0, bt1;
};

template <int R>
__device__ __forceinline__ void prefetch_item(const CtxArgs& a, int item, int n_z, int n_pre,
                                              int lane, ItemPrefetch<R>& pf) {
  pf.it = ctx_item<R>(a, item, n_z, n_pre);
  const CtxItem<R>& it = pf.it;
  const int l16 = lane & 15;
  const int rbase = it.z * R;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int li = rbase + i;
    if (li < it.nrows) {
      const int t = li / a.g, jj = li % a.g;
      const __nv_bfloat16* qp = a.q + static_cast<long long>(it.row0 + t) * a.q_row_stride +
                                static_cast<long long>(it.h * a.g + jj) * a.q_head_stride + l16 * 8;
      const uint4 u = *reinterpret_cast<const uint4*>(qp);
      pf.qf[i][0] = bf16_lo(u.x); pf.qf[i][1] = bf16_hi(u.x);
      pf.qf[i][2] = bf16_lo(u.y); pf.qf[i][3] = bf16_hi(u.y);
      pf.qf[i][4] = bf16_lo(u.z); pf.qf[i][5] = bf16_hi(u.z);
      pf.qf[i][6] = bf16_lo(u.w); pf.qf[i][7] = bf16_hi(u.w);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) pf.qf[i][e] = 0.f;
    }
  }
  pf.bt0 = pf.bt1 = 0;
  if (a.ctx.block_table != nullptr && it.n_chunks > 0) {
    const int nb = (it.max_lim + a.ctx.block_size - 1) / a.ctx.block_size;
    const int* row = a.ctx.block_table + static_cast<long long>(it.r) * a.ctx.bt_stride;
    if (lane < nb) pf.bt0 = __ldg(row + lane);
    if (lane + 32 < nb) pf.bt1 = __ldg(row + lane + 32);
  }
}

// Issue the bulk copies of chunk k of `it` into `slot` (warp-uniform call).
// Paged K/V of one (block, head) run is contiguous: one 4 KB copy for K and
// one for V; other layouts use one 256-byte copy per token, spread over lanes.
template <int R>
__device__ __forceinline__ void issue_chunk(const CtxArgs& a, const ItemPrefetch<R>& pf, int k,
                                            int n_pre, uint8_t* slot, uint64_t* bar, int lane) {
  const CtxItem<R>& it = pf.it;
  const __nv_bfloat16 *kb, *vb;
  int n;
  long long tok_stride;
  bool contiguous;
  int blk = 0;
  if (k >= n_pre && a.ctx.block_table != nullptr) {
    // block id of this chunk's first token: from the lane-parallel prefetch
    const int t0 = (k - n_pre) * kChunk;
    const int bi = t0 / a.ctx.block_size;
    const int v0 = __shfl_sync(0xffffffffu, pf.bt0, bi & 31);
    const int v1 = __shfl_sync(0xffffffffu, pf.bt1, bi & 31);
    blk = bi < 32 ? v0 : bi < 64 ? v1
                   : __ldg(a.ctx.block_table + static_cast<long long>(it.r) * a.ctx.bt_stride + bi);
  }
  if (k < n_pre) {
    const int t0 = k * kChunk;
    n = min(kChunk, a.s_prefix - t0);
    const long long off = static_cast<long long>(it.h) * a.p_stride_head + t0 * a.p_stride_tok;
    kb = a.pk + off;
    vb = a.pv + off;
    tok_stride = a.p_stride_tok;
    contiguous = (a.p_stride_tok == RB_HEAD_DIM);
  } else {
    const int t0 = (k - n_pre) * kChunk;
    n = min(kChunk, it.max_lim - t0);
    long long off;
    if (a.ctx.block_table != nullptr)
      off = static_cast<long long>(blk) * a.ctx.stride_block +
            static_cast<long long>(t0 % a.ctx.block_size) * a.ctx.stride_tok;
    else
      off = (it.roff + t0) * a.ctx.stride_tok;
    off += it.h * a.ctx.stride_head;
    kb = a.ctx.k + off;
    vb = a.ctx.v + off;
    tok_stride = a.ctx.stride_tok;
    contiguous = (a.ctx.stride_tok == RB_HEAD_DIM) &&
                 (a.ctx.block_table == nullptr || (a.ctx.block_size % kChunk) == 0);
  }
  if (lane == 0) mbar_arrive_expect_tx(bar, 2 * n * kRowBytes);
  __syncwarp();
  if (contiguous) {
    if (lane == 0) {
      bulk_copy_g2s(slot, kb, n * kRowBytes, bar);
      bulk_copy_g2s(slot + kChunk * kRowBytes, vb, n * kRowBytes, bar);
    }
  } else if (lane < 2 * n) {
    const int t = lane % n, which = lane / n;
    const __nv_bfloat16* src;
    if (k < n_pre || a.ctx.block_table == nullptr) {
      src = (which ? vb : kb) + t * tok_stride;
    } else {
      const int tt = (k - n_pre) * kChunk + t;
      const int bi = tt / a.ctx.block_size;
      const int b2 = __ldg(a.ctx.block_table + static_cast<long long>(it.r) * a.ctx.bt_stride + bi);
      src = (which ? a.ctx.v : a.ctx.k) + static_cast<long long>(b2) * a.ctx.stride_block +
            static_cast<long long>(tt % a.ctx.block_size) * a.ctx.stride_tok +
            it.h * a.ctx.stride_head;
    }
    bulk_copy_g2s(slot + which * kChunk * kRowBytes + t * kRowBytes, src, kRowBytes, bar);
  }
}

// Warp-per-item persistent kernel.  Global warp gw processes items gw,
// gw + W, ... (W = all warps of the grid).  Each warp streams its items'
// chunks through a private ring of kWarpSlots bulk-copy slots; chunks of the
// next item are issued while the current one finishes, and the next item's
// metadata / queries / block-table entries are prefetched one item ahead, so
// no global round trip sits on the per-item critical path.  Half-warp hw
// handles keys 2p + hw of each chunk; the two half states merge with shuffles.
constexpr int kWarpSlots = 2;
constexpr int kCtxWarps = 4;

template <int R>
__global__ void __launch_bounds__(kCtxWarps * 32, (R <= 2) ? 3 : 1)
    ctx_attn_kernel(const CtxArgs a, int n_items, int n_z) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hw = lane >> 4, l16 = lane & 15;
  const int n_pre = (a.s_prefix + kChunk - 1) / kChunk;
  const int W = gridDim.x * kCtxWarps;
  const int gw = blockIdx.x * kCtxWarps + warp;
  uint8_t* slots = smem + warp * kWarpSlots * kSlotBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kCtxWarps * kWarpSlots * kSlotBytes) +
                  warp * kWarpSlots;
  if (lane == 0) {
    for (int i = 0; i < kWarpSlots; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  pdl_launch_dependents();
  if (gw >= n_items) return;

  // issue cursor (item + chunk) runs up to kWarpSlots chunks ahead of compute
  ItemPrefetch<R> iss;
  prefetch_item<R>(a, gw, n_z, n_pre, lane, iss);
  int iss_item = gw, iss_k = 0;
  long long issued = 0;
  ItemPrefetch<R> nxt;  // next item's prefetch for the issue cursor
  bool have_nxt = false;
  auto advance_issue = [&]() {
    // move the issue cursor past exhausted items (warp-uniform)
    while (iss_item < n_items && iss_k >= iss.it.n_chunks) {
      iss_item += W;
      iss_k = 0;
      if (iss_item >= n_items) break;
      if (have_nxt) {
        iss = nxt;
        have_nxt = false;
      } else {
        prefetch_item<R>(a, iss_item, n_z, n_pre, lane, iss);
      }
    }
  };
  auto issue_one = [&]() {
    advance_issue();
    if (iss_item >= n_items) return;
    const int sl = static_cast<int>(issued % kWarpSlots);
    issue_chunk<R>(a, iss, iss_k, n_pre, slots + sl * kSlotBytes, &bar[sl], lane);
    ++issued;
    ++iss_k;
    // start fetching the following item's metadata as soon as this one is issued
    if (iss_k == iss.it.n_chunks && !have_nxt && iss_item + W < n_items) {
      prefetch_item<R>(a, iss_item + W, n_z, n_pre, lane, nxt);
      have_nxt = true;
    }
  };

  ItemPrefetch<R> cur = iss;  // compute cursor starts on the same item
  for (int s = 0; s < kWarpSlots; ++s) issue_one();

  long long consumed = 0;
  bool waited = false;
  for (int item = gw; item < n_items; item += W) {
    if (item != gw) {
      // the issue cursor has already prefetched this item (it runs ahead)
      cur = (iss_item == item) ? iss : cur;
      if (cur.it.r != item / (n_z * a.hkv) || cur.it.h != (item / n_z) % a.hkv ||
          cur.it.z != item % n_z)
        prefetch_item<R>(a, item, n_z, n_pre, lane, cur);
    }
    const CtxItem<R>& it = cur.it;
    if (it.n_chunks == 0) continue;
    const int rbase = it.z * R;
    int lim_ctx[R], lim_pre[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int li = rbase + i;
      if (li < it.nrows) {
        const int t = li / a.g;
        lim_ctx[i] = a.causal ? it.c_r - it.m_r + t + 1 : it.c_r;
        lim_pre[i] = a.s_prefix;
      } else {
        lim_ctx[i] = 0;
        lim_pre[i] = 0;
      }
    }
    RowState<R> st;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      st.m[i] = -INFINITY;
      st.l[i] = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) st.acc[i][e] = 0.f;
    }
    for (int k = 0; k < it.n_chunks; ++k, ++consumed) {
      const int sl = static_cast<int>(consumed % kWarpSlots);
      const uint8_t* src = slots + sl * kSlotBytes;
      mbar_wait(&bar[sl], static_cast<uint32_t>((consumed / kWarpSlots) & 1));
      uint4 kr[8], vr[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        kr[p] = *reinterpret_cast<const uint4*>(src + (2 * p + hw) * kRowBytes + l16 * 16);
        vr[p] = *reinterpret_cast<const uint4*>(src + kChunk * kRowBytes + (2 * p + hw) * kRowBytes +
                                                l16 * 16);
      }
      fence_proxy_async_smem();
      __syncwarp();
      issue_one();  // refill the slot just read
      if (k < n_pre)
        chunk_update<R>(st, cur.qf, kr, vr, k * kChunk, hw, lim_pre, a.scale_log2, a.s_prefix);
      else
        chunk_update<R>(st, cur.qf, kr, vr, (k - n_pre) * kChunk, hw, lim_ctx, a.scale_log2,
                        it.max_lim);
    }

    // ---- merge the two half-warp states (keys 2p and 2p+1) with shuffles
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
      st.l[i] = st.l[i] * ws + lo * wo;
      st.m[i] = M;
    }
    if (!waited) {  // before the first global write / system-output read
      pdl_wait_primary();
      waited = true;
    }
    // ---- epilogue: half-warp 0 owns 8 head dims per lane
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int li = rbase + i;
      if (li >= it.nrows) continue;
      const int t = li / a.g, jj = li % a.g;
      const long long oidx = static_cast<long long>(it.row0 + t) * a.hq + it.h * a.g + jj;
      const float M = st.m[i], Ls = st.l[i];
      float o[8], lse2;
      if (a.sys_part_acc != nullptr) {
        // relay fusion: merge every system stream-K part of this (row, head)
        const rb_sys_plan& SP = a.sys_plan;
        const long long f = static_cast<long long>(it.row0 + t) * SP.g + jj;
        const int qt = static_cast<int>(f / SP.nq), col = static_cast<int>(f % SP.nq);
        const int u = it.h * SP.n_qt + qt;
        const int np = rb_unit_parts(&SP, u);
        const long long base = static_cast<long long>(u) * SP.max_parts;
        float mt = M, lt = Ls;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = st.acc[i][e];
        for (int k0 = 0; k0 < np; k0 += 2) {
          float mk[2], lk[2];
          float4 ak[2][2];
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int k = min(k0 + kk, np - 1);
            const float* ml = a.sys_part_ml + (base + k) * 2 * SP.nq;
            mk[kk] = __ldcg(ml + col);
            lk[kk] = __ldcg(ml + SP.nq + col);
            const float4* ap = reinterpret_cast<const float4*>(
                a.sys_part_acc + ((base + k) * SP.nq + col) * RB_HEAD_DIM + l16 * 8);
            ak[kk][0] = __ldcg(ap);
            ak[kk][1] = __ldcg(ap + 1);
          }
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            if (k0 + kk >= np) break;
            const float mn = fmaxf(mt, mk[kk]);
            const float so = (mt == -INFINITY) ? 0.f : fast_exp2(mt - mn);
            const float sk = fast_exp2(mk[kk] - mn);
            lt = lt * so + lk[kk] * sk;
            const float av[8] = {ak[kk][0].x, ak[kk][0].y, ak[kk][0].z, ak[kk][0].w,
                                 ak[kk][1].x, ak[kk][1].y, ak[kk][1].z, ak[kk][1].w};
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = o[e] * so + av[e] * sk;
            mt = mn;
          }
        }
        const float inv = 1.f / lt;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] *= inv;
        lse2 = mt + __log2f(lt);
      } else {
        const float inv = (Ls > 0.f) ? 1.f / Ls : 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = st.acc[i][e] * inv;
        lse2 = (Ls > 0.f) ? M + __log2f(Ls) : -INFINITY;
      }
      if (a.o_sys != nullptr) {
        const float ls2 = __ldcg(a.lse_sys + oidx) * kLog2e;
        const float4* op = reinterpret_cast<const float4*>(a.o_sys + oidx * 128 + l16 * 8);
        const float4 s0 = __ldcg(op), s1 = __ldcg(op + 1);
        const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        const float mx = fmaxf(ls2, lse2);
        const float wc = (lse2 == -INFINITY) ? 0.f : fast_exp2(lse2 - mx);
        const float ws = (ls2 == -INFINITY) ? 0.f : fast_exp2(ls2 - mx);
        const float inv = 1.f / (wc + ws);
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (wc * o[e] + ws * sv[e]) * inv;
        lse2 = mx + __log2f(wc + ws);
      }
      if (hw == 0) {
        if (a.out_fp32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + oidx * 128 + l16 * 8);
          dst[0] = make_float4(o[0], o[1], o[2], o[3]);
          dst[1] = make_float4(o[4], o[5], o[6], o[7]);
        } else {
          uint4 pk;
          pk.x = pack_bf16x2(o[0], o[1]);
          pk.y = pack_bf16x2(o[2], o[3]);
          pk.z = pack_bf16x2(o[4], o[5]);
          pk.w = pack_bf16x2(o[6], o[7]);
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) + oidx * 128 + l16 * 8) = pk;
        }
        if (a.lse_out != nullptr && l16 == 0) a.lse_out[oidx] = lse2 * kLn2;
      }
    }
  }
}

// Long items (the naive baseline's shared prefix: hundreds of chunks per
// request): CTA-per-item producer/consumer kernel.  CTA b processes items b,
// b + grid, ...; their chunks form one sequence.  Warp 0 is the producer: its lanes
// resolve block-table entries and issue the bulk copies of up to kRing chunks
// at once into a CTA-wide ring of kRing slots (waiting on each slot's empty
// barrier), so the copies run far ahead of the math.  Warps 1..4 consume
// chunk k of an item in warp 1 + (k % 4), then merge their partial states at
// the end of the item and run the fusion epilogue (thread = head dim).
constexpr int kRing = 12;                      // 12 x 8 KB = 96 KB of K/V in flight per CTA
constexpr int kCtxThreadsPC = 160;             // producer + 4 consumers
template <int R>
__global__ void __launch_bounds__(kCtxThreadsPC)
    ctx_cta_kernel(const CtxArgs a, int n_items, int n_z) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_pre = (a.s_prefix + kChunk - 1) / kChunk;
  uint8_t* ring = smem;
  float* s_acc = reinterpret_cast<float*>(smem + kRing * kSlotBytes);  // [8][R][128]
  float* s_m = s_acc + 8 * R * 128;                                    // [8][R]
  float* s_l = s_m + 8 * R;                                            // [8][R]
  uint64_t* full = reinterpret_cast<uint64_t*>(s_l + 8 * R);
  uint64_t* empty = full + kRing;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    long long seq = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const CtxItem<R> it = ctx_item<R>(a, item, n_z, n_pre);
      // a batch never spans more than one ring round, so every lane's slot was
      // last used by a chunk issued in an earlier batch and the empty-barrier
      // parity it waits on is unambiguous
      for (int k0 = 0; k0 < it.n_chunks; k0 += kRing) {
        const int k = k0 + lane;
        if (lane < kRing && k < it.n_chunks) {
          const long long sq = seq + k;
          const int slot = static_cast<int>(sq % kRing);
          mbar_wait(&empty[slot], static_cast<uint32_t>(((sq / kRing) & 1) ^ 1));
          const __nv_bfloat16 *kb, *vb;
          int n;
          bool contiguous;
          long long tok_stride;
          if (k < n_pre) {
            const int t0 = k * kChunk;
            n = min(kChunk, a.s_prefix - t0);
            const long long off = static_cast<long long>(it.h) * a.p_stride_head + t0 * a.p_stride_tok;
            kb = a.pk + off;
            vb = a.pv + off;
            tok_stride = a.p_stride_tok;
            contiguous = (a.p_stride_tok == RB_HEAD_DIM);
          } else {
            const int t0 = (k - n_pre) * kChunk;
            n = min(kChunk, it.max_lim - t0);
            kb = ctx_row(a.ctx, a.ctx.k, it.r, t0, it.h);
            vb = ctx_row(a.ctx, a.ctx.v, it.r, t0, it.h);
            tok_stride = a.ctx.stride_tok;
            contiguous = (a.ctx.stride_tok == RB_HEAD_DIM) &&
                         (a.ctx.block_table == nullptr || (a.ctx.block_size % kChunk) == 0);
          }
          uint8_t* dst = ring + slot * kSlotBytes;
          mbar_arrive_expect_tx(&full[slot], 2 * n * kRowBytes);
          if (contiguous) {
            bulk_copy_g2s(dst, kb, n * kRowBytes, &full[slot]);
            bulk_copy_g2s(dst + kChunk * kRowBytes, vb, n * kRowBytes, &full[slot]);
          } else {
            for (int t = 0; t < n; ++t) {
              const __nv_bfloat16 *ks, *vs;
              if (k < n_pre) {
                ks = kb + t * tok_stride;
                vs = vb + t * tok_stride;
              } else {
                const int tt = (k - n_pre) * kChunk + t;
                ks = ctx_row(a.ctx, a.ctx.k, it.r, tt, it.h);
                vs = ctx_row(a.ctx, a.ctx.v, it.r, tt, it.h);
              }
              bulk_copy_g2s(dst + t * kRowBytes, ks, kRowBytes, &full[slot]);
              bulk_copy_g2s(dst + kChunk * kRowBytes + t * kRowBytes, vs, kRowBytes, &full[slot]);
            }
          }
        }
        __syncwarp();
      }
      seq += it.n_chunks;
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int cw = warp - 1;                      // 0..3
  const int hw = lane >> 4, l16 = lane & 15;
  long long seq = 0;
  bool waited = false;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const CtxItem<R> it = ctx_item<R>(a, item, n_z, n_pre);
    if (it.n_chunks == 0) continue;
    const int rbase = it.z * R;
    float qf[R][8];
    int lim_ctx[R], lim_pre[R];
    float os_pref[R], ls_pref[R];
    long long oidx[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int li = rbase + i;
      os_pref[i] = 0.f;
      ls_pref[i] = -INFINITY;
      oidx[i] = -1;
      if (li < it.nrows) {
        const int t = li / a.g, jj = li % a.g;
        oidx[i] = static_cast<long long>(it.row0 + t) * a.hq + it.h * a.g + jj;
        const __nv_bfloat16* qp = a.q + static_cast<long long>(it.row0 + t) * a.q_row_stride +
                                  static_cast<long long>(it.h * a.g + jj) * a.q_head_stride + l16 * 8;
        const uint4 u = *reinterpret_cast<const uint4*>(qp);
        qf[i][0] = bf16_lo(u.x); qf[i][1] = bf16_hi(u.x);
        qf[i][2] = bf16_lo(u.y); qf[i][3] = bf16_hi(u.y);
        qf[i][4] = bf16_lo(u.z); qf[i][5] = bf16_hi(u.z);
        qf[i][6] = bf16_lo(u.w); qf[i][7] = bf16_hi(u.w);
        lim_ctx[i] = a.causal ? it.c_r - it.m_r + t + 1 : it.c_r;
        lim_pre[i] = a.s_prefix;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) qf[i][e] = 0.f;
        lim_ctx[i] = 0;
        lim_pre[i] = 0;
      }
    }
    RowState<R> st;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      st.m[i] = -INFINITY;
      st.l[i] = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) st.acc[i][e] = 0.f;
    }
    for (int k = cw; k < it.n_chunks; k += 4) {
      const long long sq = seq + k;
      const int slot = static_cast<int>(sq % kRing);
      mbar_wait(&full[slot], static_cast<uint32_t>((sq / kRing) & 1));
      const uint8_t* src = ring + slot * kSlotBytes;
      uint4 kr[8], vr[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        kr[p] = *reinterpret_cast<const uint4*>(src + (2 * p + hw) * kRowBytes + l16 * 16);
        vr[p] = *reinterpret_cast<const uint4*>(src + kChunk * kRowBytes + (2 * p + hw) * kRowBytes +
                                                l16 * 16);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (k < n_pre)
        chunk_update<R>(st, qf, kr, vr, k * kChunk, hw, lim_pre, a.scale_log2, a.s_prefix);
      else
        chunk_update<R>(st, qf, kr, vr, (k - n_pre) * kChunk, hw, lim_ctx, a.scale_log2,
                        it.max_lim);
    }
    seq += it.n_chunks;

    if (!waited) {  // before the first global write / system-output read
      pdl_wait_primary();
      waited = true;
    }
    if (a.o_sys != nullptr) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (oidx[i] >= 0) {
          os_pref[i] = __ldcg(a.o_sys + oidx[i] * 128 + (threadIdx.x - 32));
          ls_pref[i] = __ldcg(a.lse_sys + oidx[i]);
        }
      }
    }
    // ---- merge the 8 (warp, half) partial states per row through smem
    const int wh = cw * 2 + hw;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      float* dst = s_acc + (wh * R + i) * 128 + l16 * 8;
      *reinterpret_cast<float4*>(dst) =
          make_float4(st.acc[i][0], st.acc[i][1], st.acc[i][2], st.acc[i][3]);
      *reinterpret_cast<float4*>(dst + 4) =
          make_float4(st.acc[i][4], st.acc[i][5], st.acc[i][6], st.acc[i][7]);
      if (l16 == 0) {
        s_m[wh * R + i] = st.m[i];
        s_l[wh * R + i] = st.l[i];
      }
    }
    named_bar_sync(1, 128);
    const int dcol = threadIdx.x - 32;  // 128 consumer threads = 128 head dims
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (oidx[i] < 0) continue;
      float M = -INFINITY;
#pragma unroll
      for (int k = 0; k < 8; ++k) M = fmaxf(M, s_m[k * R + i]);
      float Ls = 0.f, O = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float mk = s_m[k * R + i];
          const float w = (mk == -INFINITY) ? 0.f : fast_exp2(mk - M);
          Ls = fmaf(s_l[k * R + i], w, Ls);
          O = fmaf(s_acc[(k * R + i) * 128 + dcol], w, O);
        }
      }
      float o, lse2;
      if (a.sys_part_acc != nullptr) {
        // one LSE-weighted combine of the system kernel's stream-K parts of
        // this (row, head) and the context state (M, Ls, O): relay fusion.
        const rb_sys_plan& SP = a.sys_plan;
        const long long row = oidx[i] / a.hq;
        const int hh = static_cast<int>(oidx[i] % a.hq);
        const long long f = row * SP.g + hh % SP.g;
        const int qt = static_cast<int>(f / SP.nq), col = static_cast<int>(f % SP.nq);
        const int u = (hh / SP.g) * SP.n_qt + qt;
        const int np = rb_unit_parts(&SP, u);
        const long long base = static_cast<long long>(u) * SP.max_parts;
        float mt = M, lt = Ls, ot = O;
        for (int k0 = 0; k0 < np; k0 += 4) {  // 4 parts' loads in flight at once
          float mk[4], lk[4], ak[4];
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int k = min(k0 + kk, np - 1);
            const float* ml = a.sys_part_ml + (base + k) * 2 * SP.nq;
            mk[kk] = __ldcg(ml + col);
            lk[kk] = __ldcg(ml + SP.nq + col);
            ak[kk] = __ldcg(a.sys_part_acc + ((base + k) * SP.nq + col) * RB_HEAD_DIM + dcol);
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (k0 + kk >= np) break;
            const float mn = fmaxf(mt, mk[kk]);
            const float so = (mt == -INFINITY) ? 0.f : fast_exp2(mt - mn);
            const float sk = fast_exp2(mk[kk] - mn);
            lt = lt * so + lk[kk] * sk;
            ot = ot * so + ak[kk] * sk;
            mt = mn;
          }
        }
        o = ot / lt;
        lse2 = mt + __log2f(lt);
      } else {
        o = (Ls > 0.f) ? O / Ls : 0.f;
        lse2 = (Ls > 0.f) ? M + __log2f(Ls) : -INFINITY;
      }
      if (a.o_sys != nullptr) {
        const float ls2 = ls_pref[i] * kLog2e;
        const float mx = fmaxf(ls2, lse2);
        const float wc = (lse2 == -INFINITY) ? 0.f : fast_exp2(lse2 - mx);
        const float ws = (ls2 == -INFINITY) ? 0.f : fast_exp2(ls2 - mx);
        const float inv = 1.f / (wc + ws);
        o = (wc * o + ws * os_pref[i]) * inv;
        lse2 = mx + __log2f(wc + ws);
      }
      if (a.out_fp32)
        reinterpret_cast<float*>(a.out)[oidx[i] * 128 + dcol] = o;
      else
        reinterpret_cast<__nv_bfloat16*>(a.out)[oidx[i] * 128 + dcol] = __float2bfloat16_rn(o);
      if (a.lse_out != nullptr && dcol == 0) a.lse_out[oidx[i]] = lse2 * kLn2;
    }
    named_bar_sync(1, 128);  // merge buffer free for the next item
  }
}

template <int R>
static cudaError_t launch_ctx_r(const CtxArgs& a, int n_items, int n_z, cudaStream_t stream) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool pdl = a.o_sys != nullptr || a.sys_part_acc != nullptr;
  cudaError_t e;
  if (a.s_prefix > 0) {
    // naive baseline: long per-request key sequences -> 4 consumer warps per item
    const int smem = kRing * kSlotBytes + (8 * R * 128 + 16 * R) * 4 + 2 * kRing * 8;
    e = cudaFuncSetAttribute(ctx_cta_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ctx_cta_kernel<R>, kCtxThreadsPC, smem);
    if (e != cudaSuccess) return e;
    const int grid = max(1, min(n_items, sms * max(per_sm, 1)));
    ctx_cta_kernel<R><<<grid, kCtxThreadsPC, smem, stream>>>(a, n_items, n_z);
    return cudaGetLastError();
  }
  const int smem = kCtxWarps * kWarpSlots * kSlotBytes + kCtxWarps * kWarpSlots * 8;
  e = cudaFuncSetAttribute(ctx_attn_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ctx_attn_kernel<R>, kCtxWarps * 32, smem);
  if (e != cudaSuccess) return e;
  const int grid = max(1, min((n_items + kCtxWarps - 1) / kCtxWarps, sms * max(per_sm, 1)));
  // Relay mode follows the system kernel, which triggers early: launch with
  // PDL so this kernel streams context K/V on SMs the system kernel has
  // already released (it waits for the system grid before reading its
  // outputs).  Other modes are ordinary stream-ordered launches.
  if (pdl)
    e = launch_pdl(ctx_attn_kernel<R>, dim3(grid), dim3(kCtxWarps * 32), smem, stream, a, n_items, n_z);
  else
    ctx_attn_kernel<R><<<grid, kCtxWarps * 32, smem, stream>>>(a, n_items, n_z);
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
