/*
 * relay_b200 -- C-ABI of the B200 (sm_100a) RelayAttention decode path.
 *
 * The reference's kernel boundary is the Python module `relayserve.kernels`
 * (/root/reference/pkg/src/relayserve/kernels.py:14-37), which re-exports
 * per-head float64 loops (matmul_nt, softmax_lse_rows, softmax_lse_prefix:
 * _kernels_cy.pyx:13-77) that `relayserve.attention` calls inside a Python
 * (batch, head) loop (attention.py:122-133).  On B200 that per-head boundary
 * is the wrong granularity, so this library exports the operator one level
 * up -- one call per attention segment -- and the host package
 * paper_2402_14808_b200 re-exposes the reference's operator API
 * (attention_with_lse, relay_fusion, relay_attention(_ragged),
 * baseline_attention(_ragged)) on top of it.  INTEGRATION.md shows the
 * ctypes binding a relayserve maintainer would add.
 *
 * Conventions
 *  - plain pointers and sizes; tensors are device pointers (bf16 inputs,
 *    fp32 partials/LSE); strides are in ELEMENTS.
 *  - the caller allocates every output and the workspace; nothing is
 *    allocated inside a call.
 *  - launches are asynchronous and ordered on `stream` (a cudaStream_t,
 *    NULL = legacy default stream); calls are reentrant on distinct
 *    buffers.
 *  - return 0 (RB_OK) or an RB_ERR_* code; rb_last_error() has the message
 *    (thread-local).  RB_ERR_DIMENSION / RB_ERR_CONTRACT correspond to the
 *    reference's DimensionError / ContractError (errors.py:4-9).
 *  - head_dim must be 128 (the shapes BASELINE.json names); the Python
 *    layer zero-pads smaller head dims (exact: zero dims add nothing to
 *    q.k and produce zero output columns).
 *  - LSEs are natural-log, like the reference (_kernels_cy.pyx:50).
 */
#ifndef RELAY_B200_H
#define RELAY_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RB_ABI_VERSION 3

enum {
  RB_OK = 0,
  RB_ERR_DIMENSION = 1, /* relayserve.errors.DimensionError */
  RB_ERR_CONTRACT = 2,  /* relayserve.errors.ContractError  */
  RB_ERR_CUDA = 3,      /* launch / driver failure           */
};

const char* rb_last_error(void);
int rb_abi_version(void);
int rb_device_sm_count(int device, int* out);

/*
 * Work plan of the relay step's system tiles (stream-K over kv head x query
 * tile x 128-key tile; paper_2402_14808_b200/csrc/rb_plan.h).  fields[7] =
 * {nq, n_qtiles, tiles_per_unit, n_units, total_tiles, grid, max_parts};
 * *workspace_bytes = the workspace every attention entry point below needs for
 * this shape (ZERO-FILLED once before first use; the kernel leaves its grid
 * barrier in the zero state, so the buffer is reusable).  s = 0: no shared
 * prefix (context-only launches).
 */
int rb_step_plan_query(int n_rows, int hq, int hkv, int s, int grid_cap, long long* fields,
                       size_t* workspace_bytes);

/* 1 when the relay step supports the shape: hq/hkv divides the query tile
 * (g in 1,2,4,8,16), b small enough for the per-CTA request metadata, and a
 * paged block size of 16, 32 or 64 tokens. */
int rb_relay_step_supported(int n_rows, int hq, int hkv, int b, int block_size, int paged);

/*
 * The relay decode step as ONE persistent kernel (relay_step_sm100.cu) --
 * `relay_attention_ragged` (attention.py:203-243): system tiles (stream-K over
 * the shared prefix, read once) and context tiles (whole (request, kv head)
 * units) run through one TMA + tcgen05 pipeline; after a grid barrier every
 * CTA merges its share of the outputs: context partial + system parts, the
 * relay fusion (attention.py:137-157).  Writes `out` ([n_rows][hq][128], fp32
 * when out_fp32 else bf16) and the fused natural-log LSE ([n_rows][hq]).
 *
 * q: bf16 row t, head h at q + t*q_row_stride + h*q_head_stride; q_start[b+1]
 *   flat row offsets (m_r = q_start[r+1] - q_start[r]); max_rows = max m_r * g.
 * sys_k/sys_v: bf16 shared prefix, token i of kv head h at i*sys_stride_tok +
 *   h*sys_stride_head (the reference's (s, h, d) or SystemKvCache (h, s, d)).
 * context, paged (block_table != NULL): k/v are one layer's PagedKvCache pool,
 *   block i of kv head h at (i*stride_block + h*stride_head) elements, each
 *   block a [128 d][block_size] operand with the UMMA swizzle applied
 *   (kvcache.py documents the layout; rb_kv_append writes it); ctx_extent =
 *   number of blocks; block_table int32 [b][bt_stride].
 * context, ragged (req_offset != NULL): token i of kv head h at
 *   i*stride_tok + h*stride_head; request r starts at token req_offset[r];
 *   ctx_extent = number of tokens.
 * ctx_lens int32 [b] (context INCLUDING the current tokens); causal: query
 *   row t of request r sees keys < c_r - m_r + t + 1 (attention.py:120-121).
 * prefix_mode 1: no system units; every context unit first re-reads the
 *   prefix (the per-request baseline, attention.py:266-296 / vLLM-PS).
 * phases: 3 = full step; 1 / 2 = system / context tiles only (profiling; the
 *   output is then that segment's own attention).
 */
int rb_relay_step(const void* q, long long q_row_stride, long long q_head_stride,
                  const int* q_start, int b, int n_rows, int max_rows, int hq, int hkv, int d,
                  const void* sys_k, const void* sys_v, int s, long long sys_stride_tok,
                  long long sys_stride_head, const void* k, const void* v, long long ctx_extent,
                  const int* block_table, int bt_stride, int block_size,
                  const long long* req_offset, long long stride_block, long long stride_tok,
                  long long stride_head, const int* ctx_lens, int causal, int prefix_mode,
                  float scale, int grid_cap, void* out, int out_fp32, float* lse_out,
                  void* workspace, size_t workspace_bytes, int phases, void* stream);

/*
 * `_system_attention` (attention.py:177-200): every query row against the
 * shared prefix, unmasked -> o_sys fp32 [n_rows][hq][128] (normalised) and
 * natural-log lse_sys [n_rows][hq].  = rb_relay_step with phases 1.
 */
int rb_system_attention(const void* q, long long q_row_stride, long long q_head_stride,
                        int n_rows, int hq, int hkv, int d, const void* sys_k, const void* sys_v,
                        int s, long long kv_stride_tok, long long kv_stride_head, float scale,
                        int grid_cap, float* o_sys, float* lse_sys, void* workspace,
                        size_t workspace_bytes, void* stream);

/*
 * `_context_attention` / `attention_with_lse` per request (attention.py:96-174)
 * over paged or ragged context K/V (as rb_relay_step), causal or not.  With
 * s_prefix > 0, every request first attends the prefix (prefix_k/prefix_v,
 * strides as sys_k) -- the reference's `baseline_attention` over
 * [sys || ctx] (attention.py:266-296), the naive per-request baseline that
 * re-reads the shared prefix for every request.  = rb_relay_step with phases 2.
 */
int rb_context_attention(const void* q, long long q_row_stride, long long q_head_stride,
                         const int* q_start, int b, int n_rows, int max_rows, int hq, int hkv,
                         int d, const void* k, const void* v, long long ctx_extent,
                         const int* block_table, int bt_stride, int block_size,
                         const long long* req_offset, long long stride_block, long long stride_tok,
                         long long stride_head, const int* ctx_lens, int causal,
                         const void* prefix_k, const void* prefix_v, int s_prefix,
                         long long p_stride_tok, long long p_stride_head, float scale,
                         int grid_cap, void* out, int out_fp32, float* lse_out, void* workspace,
                         size_t workspace_bytes, void* stream);

/*
 * Standalone relay fusion (attention.py:137-157) over n_vec vectors of d
 * fp32 values: out = a*o_sys + (1-a)*o_ctx, a = 1/(1+exp(lse_ctx-lse_sys)),
 * evaluated with max-subtracted weights; lse_out (optional) = logaddexp.
 */
int rb_relay_fusion(const float* o_sys, const float* lse_sys, const float* o_ctx,
                    const float* lse_ctx, float* out, float* lse_out, long long n_vec, int d,
                    void* stream);

/*
 * Paged KV append (PagedKvCache.append, kvcache.py:207-235): token i of
 * k_new/v_new ([n_tok][hkv][128] bf16) goes to slot slot_mapping[i] =
 * block_id*block_size + offset of one layer's pool (block stride / head
 * stride in elements), written into the swizzled [128 d][block_size] block
 * layout rb_relay_step reads.
 */
int rb_kv_append(const void* k_new, const void* v_new, const int* slot_mapping, int n_tok,
                 void* k_pool, void* v_pool, int hkv, int d, int block_size,
                 long long stride_block, long long stride_head, void* stream);

/*
 * Debug probe of the tcgen05 operand layouts of the system tiles
 * (one CTA): S^T = K.Q^T and O^T = V^T.P^T for K,V [128][128], Q [nq][128],
 * P [nq][128] bf16 -> s_out, o_out fp32 [128][nq].  For tests only.
 */
int rb_debug_umma_probe(const void* k, const void* q, const void* v, const void* p, int nq,
                        float* s_out, float* o_out, void* stream);

/*
 * Debug probe of the paged-context operand layouts of rb_relay_step (one CTA):
 * k, v [128 keys][128 d] bf16 are laid out as PagedKvCache blocks of
 * block_size (16/32/64) tokens, q, p [32][128]; s_out = K.Q^T and
 * o_out = V^T.P^T, fp32 [128][32].  For tests only.
 */
int rb_debug_ctx_probe(const void* k, const void* q, const void* v, const void* p, int block_size,
                       float* s_out, float* o_out, void* stream);

/*
 * Debug: when `buf` (device) is non-NULL, subsequent
 * rb_relay_step launches record per-CTA %globaltimer stamps into it ([grid][512]
 * u64; layout in profiles/diag_step_timeline.py).  NULL disables.  For
 * profiling only.
 */
int rb_debug_set_timestamps(void* buf);

#ifdef __cplusplus
}
#endif
#endif /* RELAY_B200_H */
