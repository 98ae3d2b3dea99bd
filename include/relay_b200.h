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

#define RB_ABI_VERSION 4

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
 * Work plan of rb_system_attention (stream-K split over kv head x query
 * tile x 128-key tile, or whole units dealt round-robin when a KV head has
 * several query tiles; paper_2402_14808_b200/csrc/rb_plan.h).  fields[8] =
 * {nq, n_qtiles, tiles_per_unit, n_units, total_tiles, grid, max_parts, rr};
 * *workspace_bytes = bytes rb_system_attention needs (zero-filled before the
 * first use; the kernel leaves its semaphores zeroed).
 */
int rb_sys_plan_query(int n_rows, int hq, int hkv, int s, int grid_cap, long long* fields,
                      size_t* workspace_bytes);

/*
 * System-prompt attention: every flattened query row (all requests' new
 * tokens) against the shared prefix K/V, unmasked, with LSE.
 * Replaces `_system_attention` (attention.py:177-200), i.e.
 * `attention_with_lse(q_flat[None], sys_k[None], sys_v[None], causal=False)`
 * (attention.py:183-185, 96-134).
 *   q:      bf16, row r / head h at q + r*q_row_stride + h*q_head_stride
 *   sys_k/v bf16, key t / kv head h at base + t*kv_stride_tok + h*kv_stride_head
 *           ([hkv][s][d]: (d, s*d); the reference's (s, h, d): (h*d, d))
 *   o_sys:  fp32 [n_rows][hq][128] (normalised), lse_sys: fp32 [n_rows][hq]
 *   grid_cap: CTAs to use (normally the SM count; one CTA per SM).
 * Errors: s < 1 -> RB_ERR_CONTRACT (attention.py:219-222); hq % hkv -> DIMENSION.
 */
int rb_system_attention(const void* q, long long q_row_stride, long long q_head_stride,
                        int n_rows, int hq, int hkv, int d, const void* sys_k, const void* sys_v,
                        int s, long long kv_stride_tok, long long kv_stride_head, float scale,
                        int grid_cap, float* o_sys, float* lse_sys, void* workspace,
                        size_t workspace_bytes, void* stream);

/*
 * Request-context attention over paged (or ragged-contiguous) KV.  With
 * causal=1, row t of request r (m_r = q_start[r+1] - q_start[r] rows)
 * attends context keys 0 .. ctx_lens[r] - m_r + t  -- `_context_attention`
 * (attention.py:160-174) / `attention_with_lse(causal=True)`
 * (attention.py:120-121); causal=0 attends all ctx_lens[r] keys.
 *   KV addressing, key t of request r, kv head h:
 *     paged  (block_table != NULL): base + block_table[r*bt_stride + t/block_size]*stride_block
 *                                        + (t % block_size)*stride_tok + h*stride_head
 *            pool layout [num_blocks][hkv][block_size][128]: (hkv*bs*128, 128, bs*128)
 *     ragged (req_offset != NULL):  base + (req_offset[r] + t)*stride_tok + h*stride_head
 *   n_rows = q_start[b]; max_rows: max_r m_r * (hq / hkv).
 * Relay epilogue: when o_sys/lse_sys (rb_system_attention's outputs) are
 *   given, the result is fused with them (`relay_fusion`, attention.py:137-157)
 *   and lse_out receives the fused LSE = logaddexp(lse_sys, lse_ctx).
 * Naive baseline: when s_prefix > 0, each request first attends the whole
 *   shared prefix prefix_k/prefix_v (re-read per request, like the
 *   reference's `baseline_attention`, attention.py:266-296).
 * out: [n_rows][hq][128], fp32 when out_fp32 else bf16; lse_out: fp32
 *   [n_rows][hq] or NULL.
 * Split-K: max_ctx_len (an upper bound of ctx_lens, <= 0: unknown) lets the
 *   kernel cut long contexts into splits spread over the SMs (few requests x
 *   heads, long contexts), combined in a fixed order (deterministic).  The
 *   splits need `workspace` of rb_context_workspace_bytes(...) bytes,
 *   zero-filled before first use (the kernel leaves it zeroed); workspace
 *   NULL runs unsplit; a non-NULL workspace that is too small is an error.
 */
int rb_context_workspace_bytes(int b, int n_rows, int max_rows, int hq, int hkv, int s_prefix,
                               int max_ctx_len, int sm_count, size_t* bytes);
int rb_context_attention(const void* q, long long q_row_stride, long long q_head_stride,
                         const int* q_start, int b, int n_rows, int max_rows, int hq, int hkv, int d,
                         const void* k, const void* v, const int* block_table, int bt_stride,
                         int block_size, const long long* req_offset, long long stride_block,
                         long long stride_tok, long long stride_head, const int* ctx_lens,
                         int causal, const void* prefix_k, const void* prefix_v, int s_prefix,
                         long long p_stride_tok, long long p_stride_head, const float* o_sys,
                         const float* lse_sys, float scale, void* out, int out_fp32,
                         float* lse_out, int max_ctx_len, void* workspace, size_t workspace_bytes,
                         void* stream);

/*
 * The whole relay decode step in one call -- `relay_attention_ragged`
 * (attention.py:203-243) over a shared prefix and paged (or ragged) context:
 * the tcgen05 system kernel (grid_cap CTAs, see rb_relay_sys_grid) writes
 * its stream-K partial slots into `workspace` without merging them and
 * publishes each unit on a counter; the context kernel (programmatic
 * dependent launch: it starts right away on the SMs the system kernel does
 * not use and streams context K/V concurrently) merges every system slot of
 * a (row, head) with its own context state, once that unit is published, in
 * ONE LSE-weighted combine -- the relay fusion (attention.py:137-157) --
 * writing `out` (bf16 or fp32) and the fused LSE.
 * Arguments are those of rb_system_attention + rb_context_attention (causal).
 * workspace: rb_relay_workspace_bytes(...) bytes (sm_count = the device's SM
 * count), zero-filled before first use; the kernels leave it zeroed (its
 * header holds the context kernel's work counters), so one buffer serves
 * every step on a stream.  max_ctx_len: an upper bound of ctx_lens (e.g. the
 * block table's width x block_size) for the context split-K.
 * k_new, v_new, slot_mapping (all NULL, or all set; paged layout only): the
 * fused append -- the step's new tokens' K / V rows, [n_rows][hkv][128] bf16
 * in q's row order (device or pinned host memory), are written into the
 * paged pool at slot_mapping[row] (as rb_kv_append would) by the context
 * item that streams them, before its workers read them; ctx_lens already
 * count the new tokens.  One launch pair then covers append + attention.
 * q and out may be pinned host memory (the zero-copy step): host queries are
 * first copied into a staging region of the workspace by one small kernel
 * (both kernels then read device memory; the system kernel's K/V prefetch
 * overlaps the copy), and output rows are written to host memory directly.
 * req_order (optional, int32 [b], a permutation of 0..b-1; an entry out of range falls
 * back to its own position): the order in which
 * the context kernel claims the requests' work -- longest context first
 * keeps the last claims short when the contexts vary (each CTA claims a few
 * items ahead, and a long queued item at the end is a tail).  Results do not
 * depend on it.
 * phases: 3 = the full step; 1 / 2 launch only the system / context kernel
 * (2 | 4: the context kernel of a step whose system kernel was launched by an
 * earlier phase-1 call, e.g. with stream work in between; the units are
 * published by that system kernel as it runs)
 * (profiling: phase 2 consumes the slots a previous phase-1 call wrote).
 */
int rb_relay_workspace_bytes(int n_rows, int hq, int hkv, int s, int grid_cap, int b,
                             int max_rows, int max_ctx_len, int sm_count, size_t* bytes);
/*
 * System-kernel CTA count for rb_relay_attention's grid_cap: the two kernels
 * run concurrently, the system kernel on a share of the SMs proportional to
 * its HBM bytes (ctx_tokens = total context tokens of the batch), the
 * context kernel on the rest and on every SM the system kernel releases
 * (the share follows the two kernels' measured per-SM streaming rates and
 * the context length per request).  Always >= 1.
 */
int rb_relay_sys_grid(int n_rows, int hq, int hkv, int s, long long ctx_tokens, int sm_count,
                      int* grid);
int rb_relay_attention(const void* q, long long q_row_stride, long long q_head_stride,
                       const int* q_start, int b, int n_rows, int max_rows, int hq, int hkv, int d,
                       const void* sys_k, const void* sys_v, int s, long long sys_stride_tok,
                       long long sys_stride_head, const void* k, const void* v,
                       const int* block_table, int bt_stride, int block_size,
                       const long long* req_offset, long long stride_block, long long stride_tok,
                       long long stride_head, const int* ctx_lens, float scale, int grid_cap,
                       void* out, int out_fp32, float* lse_out, int max_ctx_len, void* workspace,
                       size_t workspace_bytes, int phases, const void* k_new, const void* v_new,
                       const int* slot_mapping, const int* req_order, void* stream);

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
 * block_id*block_size + offset of the pool.
 */
int rb_kv_append(const void* k_new, const void* v_new, const int* slot_mapping, int n_tok,
                 void* k_pool, void* v_pool, int hkv, int d, int block_size,
                 long long stride_block, long long stride_tok, long long stride_head,
                 void* stream);

/*
 * Rotary position embedding of fp32 rows (the reference kernel boundary's
 * `rope_rows(x, positions, base)`, _kernels_cy.pyx:80-102, called through
 * numerics.rope_rows / rope_apply, numerics.py:81-108): row i's consecutive
 * pairs (2j, 2j+1) rotated by positions[i] * base^(-2j/d), angles and
 * rotation in fp64.  x, out: fp32 [n][d] (may alias); positions int64 [n].
 */
int rb_rope_rows(const float* x, float* out, const long long* positions, long long n, int d,
                 double base, void* stream);

/*
 * Decode-step prologue in one launch: the new tokens' query and key rows
 * rotated to their positions (model.py:292-293, rope_rows above) and K / V
 * appended to the paged pool (PagedKvCache.append, kvcache.py:207-235).
 *   q_in / q_out: bf16 [n_tok][hq][128] (may alias); k_new, v_new: bf16
 *   [n_tok][hkv][128]; positions int64 [n_tok] (a context token's position
 *   is its index in the context + s, kvcache.context_position, kvcache.py:25-33);
 *   slot_mapping int32 [n_tok] as for rb_kv_append.  K is stored rotated.
 */
int rb_rope_append(const void* q_in, void* q_out, const void* k_new, const void* v_new,
                   const long long* positions, const int* slot_mapping, int n_tok, int hq, int hkv,
                   int d, double base, void* k_pool, void* v_pool, int block_size,
                   long long stride_block, long long stride_tok, long long stride_head,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RELAY_B200_H */
