// Kernel argument structs shared by the kernel translation units and the
// C-ABI layer (capi.cu).
#pragma once
#include <cuda_bf16.h>
#include "rb_plan.h"

namespace rb {

struct SysArgs {
  rb_sys_plan plan;
  const __nv_bfloat16* q;  // row r, head h at q + r*q_row_stride + h*q_head_stride
  long long q_row_stride;
  long long q_head_stride;
  float scale_log2;        // (1/sqrt(d)) * log2(e)
  float* o_sys;            // fp32 [n_rows][hq][128], normalised
  float* lse_sys;          // fp32 [n_rows][hq], natural log
  float* part_acc;         // fp32 [n_units][max_parts][nq][128] (unnormalised)
  float* part_ml;          // fp32 [n_units][max_parts][2][nq]   (m log2, l)
  int* counters;           // int  [n_units], zero between launches
  unsigned long long* debug_ts;  // optional per-CTA %globaltimer stamps [grid][8]
  int defer_merge;         // 1: write every unit part to its slot, no merge, no o_sys
  int q_tma;               // 1: the system kernels load query tiles with TMA (tmap_q):
                           //    q in device memory, g divides the tile rows
};

struct KvView {
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  const int* block_table;        // paged mode if non-null: [b][bt_stride]
  int bt_stride;
  int block_size;
  const long long* req_offset;   // ragged mode: first token index of request r
  long long stride_block;        // elements (paged)
  long long stride_tok;          // elements
  long long stride_head;         // elements
};

struct CtxArgs {
  int b, hq, hkv, g;
  const int* q_start;            // [b+1] flat row offsets (m_r = q_start[r+1]-q_start[r])
  const __nv_bfloat16* q;
  long long q_row_stride, q_head_stride;
  KvView ctx;
  const int* ctx_lens;           // [b]
  int causal;                    // 1: row t sees keys < c_r - m_r + t + 1; 0: all c_r
  // optional shared prefix (naive baseline), contiguous per head
  const __nv_bfloat16* pk;
  const __nv_bfloat16* pv;
  long long p_stride_tok, p_stride_head;
  int s_prefix;
  // relay step: the system kernel's stream-K parts (published per unit on
  // sys_ready) are fused here; rows whose unit is not yet published park an
  // unnormalised context partial, [n_rows * hq][132] floats (O[128], m
  // log2, l), and are fused at the end of the CTA
  float* ctx_part;
  const float* sys_part_acc;     // [n_units][max_parts][nq][128]
  const float* sys_part_ml;      // [n_units][max_parts][2][nq]
  int* sys_ready;                // [n_units] parts published per unit
  rb_sys_plan sys_plan;
  // optional system partial (relay)
  const float* o_sys;            // [n_rows][hq][128]
  const float* lse_sys;          // [n_rows][hq] natural log
  // outputs
  void* out;                     // [n_rows][hq][128] bf16 or fp32
  int out_fp32;
  float* lse_out;                // [n_rows][hq] natural log (may be null)
  float scale_log2;
  unsigned long long* debug_ts;  // optional per-CTA stamps [grid][8] (diagnostics)
  int* sched;                    // optional [2] zeroed counters: item claims, CTA exits (dynamic claims)
  // split-K over long contexts (rb_ctx_split): split_chunks 16-token chunks
  // per split (0: no split), n_split splits per (request, kv head, row tile)
  int split_chunks, n_split;
  float* split_part;             // [n_rows * hq][n_split][132] f32 partials (O, m log2, l)
  int* split_cnt;                // [b * hkv * n_z] zeroed counters, rearmed by the last split
  // optional fused append (relay step): the step's new tokens' K / V rows,
  // [n_rows][hkv][128] in q's row order (device or pinned host memory), are
  // written into the paged pool at slot_mapping[row] by the context item
  // that streams them, before its workers read them.  Null: no append.
  const __nv_bfloat16* k_new;
  const __nv_bfloat16* v_new;
  const int* slot_mapping;
  // optional claim order of the requests (a permutation of 0..b-1, e.g. the
  // longest context first): items are claimed in this order, so the last
  // claims -- the ones whose queued items make a CTA's tail -- are short
  const int* req_order;
  // 1: the items are long (>= 16 chunks): claim one item at a time instead of
  // three ahead (set by the host from the context-length bound)
  int claim_lazy;
};

#ifdef __CUDACC__
// cp.async the query rows f0 .. f0 + ROWS - 1 of KV head h (flattened row f =
// request f / g, group member f % g; rows past rows_per_head zero-filled)
// into ROWS / T K-major SW128 tiles of T rows ([2 kblocks][T rows][128 B]
// each), one warp: lane (half = lane / 16, ch = lane % 16) copies 16-byte
// chunk ch of rows 2 it + half.  The (request, member) pair is walked
// incrementally -- a runtime division per chunk made this loop a 10+ us
// prologue of the 256-row kernel.
template <int T, int ROWS>
__device__ __forceinline__ void load_unit_q(uint8_t* dst, const SysArgs& args, int h, int f0,
                                            int lane) {
  const rb_sys_plan& P = args.plan;
  const int half = lane >> 4, ch = lane & 15;
  int f = f0 + half;
  int row = f / P.g, jj = f % P.g;
#pragma unroll 4
  for (int it = 0; it < ROWS / 2; ++it) {
    const int c = 2 * it + half;
    const bool ok = f < P.rows_per_head;
    const __nv_bfloat16* src = args.q + static_cast<long long>(row) * args.q_row_stride +
                               static_cast<long long>(h * P.g + jj) * args.q_head_stride + ch * 8;
    const int sub = c / T, rr = c % T;
    cp_async_16(dst + sub * (T * 256) + (ch >> 3) * (T * 128) + sw128_offset(rr, (ch & 7) * 8),
                ok ? src : args.q, ok ? 16u : 0u);
    f += 2;
    jj += 2;
    while (jj >= P.g) {
      jj -= P.g;
      ++row;
    }
  }
}
#endif

}  // namespace rb
