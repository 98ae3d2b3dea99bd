// C-ABI boundary of librelay_b200.so (declared in include/relay_b200.h).
//
// Replaces the reference's kernel boundary, the `relayserve.kernels` module
// (/root/reference/pkg/src/relayserve/kernels.py:14-37), one level up: the
// entry points take whole attention segments instead of per-head matmul /
// softmax calls.  Conventions: plain pointers and sizes, caller-allocated
// outputs and workspace, stream-ordered asynchronous launches, int status
// (0 = ok) with the message in rb_last_error(); RB_ERR_DIMENSION and
// RB_ERR_CONTRACT mirror relayserve.errors.DimensionError / ContractError
// (errors.py:4-9).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/relay_b200.h"
#if RB_DIAG
#include "../../include/relay_b200_diag.h"
#endif
#include "rb_common.cuh"
#include "rb_plan.h"
#include "rb_args.cuh"

namespace rb {
cudaError_t launch_system_attention(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                                    const SysArgs&, cudaStream_t);
cudaError_t launch_sys_merge_parts(const SysArgs&, cudaStream_t);
cudaError_t launch_q_stage(const __nv_bfloat16*, long long, long long, int, int, __nv_bfloat16*, int,
                           cudaStream_t);
cudaError_t launch_context_attention(const CtxArgs&, int, cudaStream_t);
int ctx_resident_ctas(int sms);
cudaError_t launch_relay_fusion(const float*, const float*, const float*, const float*, float*,
                                float*, long long, int, cudaStream_t);
cudaError_t launch_umma_probe(const __nv_bfloat16*, const __nv_bfloat16*, const __nv_bfloat16*,
                              const __nv_bfloat16*, int, float*, float*, cudaStream_t);
cudaError_t launch_kv_append(const __nv_bfloat16*, const __nv_bfloat16*, const int*,
                             __nv_bfloat16*, __nv_bfloat16*, int, int, int, long long, long long,
                             long long, cudaStream_t);
cudaError_t launch_rope_append(const __nv_bfloat16*, __nv_bfloat16*, const __nv_bfloat16*,
                               const __nv_bfloat16*, const long long*, const int*, int, int, int,
                               double, __nv_bfloat16*, __nv_bfloat16*, int, long long, long long,
                               long long, cudaStream_t);
cudaError_t launch_rope_rows(const float*, float*, const long long*, long long, int, double,
                             cudaStream_t);
}  // namespace rb


static thread_local std::string g_err;
#if RB_DIAG
static unsigned long long* g_debug_ts = nullptr;  // diagnostics build only
#else
static constexpr unsigned long long* g_debug_ts = nullptr;
#endif
// context-kernel stamps start after 1024 system CTAs x 8 slots
static constexpr long long kCtxTsOffset = 1024 * 8;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

static int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return RB_OK;
  return fail(RB_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

extern "C" {

const char* rb_last_error(void) { return g_err.c_str(); }

int rb_abi_version(void) { return RB_ABI_VERSION; }

int rb_device_sm_count(int device, int* out) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  *out = v;
  return RB_OK;
}

int rb_sys_plan_query(int n_rows, int hq, int hkv, int s, int grid_cap, long long* fields,
                      size_t* workspace_bytes) {
  if (n_rows < 1 || hq < 1 || hkv < 1) return fail(RB_ERR_DIMENSION, "empty query set");
  if (hq % hkv != 0) return fail(RB_ERR_DIMENSION, "hq=%d not a multiple of hkv=%d", hq, hkv);
  if (s < 1)
    return fail(RB_ERR_CONTRACT,
                "relay attention requires a non-empty system segment; use the baseline path "
                "when there is no shared prefix");
  rb_sys_plan p;
  {
    // the stream-K index math is 32-bit (rb_plan.h): bound total x grid
    const long long total = (long long)hkv * ((long long)n_rows * (hq / hkv) + 15) / 16 *
                            (((long long)s + RB_KEY_TILE - 1) / RB_KEY_TILE);
    if (total * (grid_cap < 1 ? 1 : grid_cap) > RB_PLAN_MAX_PRODUCT || (long long)n_rows * hq > 0x7fffffffLL)
      return fail(RB_ERR_DIMENSION, "problem too large for one stream-K plan (%d rows x %d heads, s=%d)",
                  n_rows, hq, s);
  }
  rb_make_sys_plan(&p, n_rows, hq, hkv, s, grid_cap);
  if ((long long)p.total * p.grid > RB_PLAN_MAX_PRODUCT)
    return fail(RB_ERR_DIMENSION, "problem too large for one stream-K plan");
  if (fields) {
    fields[0] = p.nq;
    fields[1] = p.n_qt;
    fields[2] = p.tpu;
    fields[3] = p.n_units;
    fields[4] = p.total;
    fields[5] = p.grid;
    fields[6] = p.max_parts;
    fields[7] = p.rr;
  }
  if (workspace_bytes) {
    size_t cnt = ((size_t)p.n_units * sizeof(int) + 255) & ~(size_t)255;
    size_t ml = p.max_parts > 1 ? (size_t)p.n_units * p.max_parts * 2 * p.nq * sizeof(float) : 0;
    ml = (ml + 255) & ~(size_t)255;
    size_t acc = p.max_parts > 1
                     ? (size_t)p.n_units * p.max_parts * p.nq * RB_HEAD_DIM * sizeof(float)
                     : 0;
    *workspace_bytes = cnt + ml + acc;
  }
  return RB_OK;
}

// ------------------------------------------------------------ TMA maps
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

static int make_kv_map(CUtensorMap* map, const void* base, int s, int hkv, long long stride_tok,
                       long long stride_head) {
  auto enc = get_encode();
  if (!enc) return fail(RB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return fail(RB_ERR_CONTRACT, "system K/V base must be 16-byte aligned");
  if ((stride_tok * 2) % 16 != 0 || (stride_head * 2) % 16 != 0)
    return fail(RB_ERR_CONTRACT, "system K/V strides must be multiples of 8 elements");
  cuuint64_t dims[3] = {RB_HEAD_DIM, (cuuint64_t)s, (cuuint64_t)hkv};
  cuuint64_t strides[2] = {(cuuint64_t)(stride_tok * 2), (cuuint64_t)(stride_head * 2)};
  cuuint32_t box[3] = {64, RB_KEY_TILE, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return RB_OK;
}

// Query tiles of the 256-row GQA kernel by TMA: [n_rows][hq][128] bf16 as a 3-D
// map (d, head, row) with a (64, g, 128 / g) box = one 128-row K-major SW128
// half tile of KV head h.  Only for q in device memory (TMA does not read
// pinned host memory -- the zero-copy step keeps the cp.async loader) and g
// dividing 128; otherwise a.q_tma stays 0.
static void maybe_q_map(CUtensorMap* map, rb::SysArgs* a, const void* q, int n_rows, int hq,
                        int hkv) {
  a->q_tma = 0;
  std::memset(map, 0, sizeof(*map));
  const int g = hq / hkv;
  // query tile rows per TMA box pair: the 256-row kernel loads two 128-row
  // tiles, the others one nq-row tile
  const int tile_rows = a->plan.nq == 256 ? 128 : a->plan.nq;
  if (tile_rows % g != 0) return;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, q) != cudaSuccess || attr.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return;
  }
  auto enc = get_encode();
  if (!enc) return;
  cuuint64_t dims[3] = {RB_HEAD_DIM, (cuuint64_t)hq, (cuuint64_t)n_rows};
  cuuint64_t strides[2] = {(cuuint64_t)(a->q_head_stride * 2), (cuuint64_t)(a->q_row_stride * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)g, (cuuint32_t)(tile_rows / g)};
  cuuint32_t estr[3] = {1, 1, 1};
  if (enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
    a->q_tma = 1;
}

// ------------------------------------------------------ system attention
int rb_system_attention(const void* q, long long q_row_stride, long long q_head_stride,
                        int n_rows, int hq, int hkv, int d, const void* sys_k, const void* sys_v,
                        int s, long long kv_stride_tok, long long kv_stride_head, float scale,
                        int grid_cap, float* o_sys, float* lse_sys, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (d != RB_HEAD_DIM) return fail(RB_ERR_DIMENSION, "head_dim %d unsupported (kernels are d=128)", d);
  size_t need = 0;
  long long f[8];
  int st = rb_sys_plan_query(n_rows, hq, hkv, s, grid_cap, f, &need);
  if (st != RB_OK) return st;
  if (workspace_bytes < need)
    return fail(RB_ERR_CONTRACT, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  if ((q_head_stride * 2) % 16 != 0 || (q_row_stride * 2) % 16 != 0 ||
      (reinterpret_cast<uintptr_t>(q) & 15))
    return fail(RB_ERR_CONTRACT, "q rows must be 16-byte aligned");
  rb::SysArgs a;
  rb_make_sys_plan(&a.plan, n_rows, hq, hkv, s, grid_cap);
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.q_row_stride = q_row_stride;
  a.q_head_stride = q_head_stride;
  a.scale_log2 = scale * rb::kLog2e;
  a.o_sys = o_sys;
  a.lse_sys = lse_sys;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  size_t cnt = ((size_t)a.plan.n_units * sizeof(int) + 255) & ~(size_t)255;
  size_t ml = a.plan.max_parts > 1
                  ? (size_t)a.plan.n_units * a.plan.max_parts * 2 * a.plan.nq * sizeof(float)
                  : 0;
  ml = (ml + 255) & ~(size_t)255;
  a.counters = reinterpret_cast<int*>(ws);
  a.part_ml = reinterpret_cast<float*>(ws + cnt);
  a.part_acc = reinterpret_cast<float*>(ws + cnt + ml);
  a.debug_ts = g_debug_ts;
  // split units: every part to its slot, then one merge launch over all
  // (unit, row) pairs (the in-kernel last-CTA merge serialised a unit's rows
  // on one SM: 60-90 us at C4 shapes)
  a.defer_merge = a.plan.max_parts > 1 ? 1 : 0;
  a.counters = nullptr;
  CUtensorMap tk, tv, tq;
  st = make_kv_map(&tk, sys_k, s, hkv, kv_stride_tok, kv_stride_head);
  if (st != RB_OK) return st;
  st = make_kv_map(&tv, sys_v, s, hkv, kv_stride_tok, kv_stride_head);
  if (st != RB_OK) return st;
  maybe_q_map(&tq, &a, q, n_rows, hq, hkv);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  st = cuda_status(rb::launch_system_attention(tk, tv, tq, a, cs), "system attention launch");
  if (st != RB_OK || !a.defer_merge) return st;
  return cuda_status(rb::launch_sys_merge_parts(a, cs), "system part merge launch");
}

// ----------------------------------------------------- context attention
// ------------------------------------------------------ context split-K
static int device_sms() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return sms;
}

static void ctx_split_plan(int b, int hkv, int max_rows, int s_prefix, int max_ctx_len, int sms,
                           int* chunks, int* n_split) {
  *chunks = 0;
  *n_split = 1;
  if (max_ctx_len <= 0 || max_rows < 1 || sms < 1) return;
  const int R = rb_ctx_rows(max_rows);
  const long long base = (long long)b * hkv * ((max_rows + R - 1) / R);
  const int max_chunks = (s_prefix + RB_CTX_CHUNK - 1) / RB_CTX_CHUNK +
                         (max_ctx_len + RB_CTX_CHUNK - 1) / RB_CTX_CHUNK;
  rb_ctx_split(base, max_chunks, rb::ctx_resident_ctas(sms), chunks, n_split);
}

int rb_context_workspace_bytes(int b, int n_rows, int max_rows, int hq, int hkv, int s_prefix,
                               int max_ctx_len, int sm_count, size_t* bytes) {
  if (b < 0 || n_rows < 0 || hq < 1 || hkv < 1 || hq % hkv != 0)
    return fail(RB_ERR_DIMENSION, "bad context workspace shape");
  int L, ns;
  ctx_split_plan(b, hkv, max_rows, s_prefix, max_ctx_len, sm_count, &L, &ns);
  *bytes = (size_t)rb_ctx_split_bytes(b, n_rows, hq, hkv, max_rows, ns);
  return RB_OK;
}

// split fields of `a` from the workspace section `ws` (NULL: no split)
static int ctx_split_args(rb::CtxArgs& a, int n_rows, int max_rows, int max_ctx_len, void* ws,
                          size_t ws_bytes) {
  a.split_chunks = 0;
  a.n_split = 1;
  a.split_part = nullptr;
  a.split_cnt = nullptr;
  // items of >= 16 chunks (context bound, or the split length below): the
  // context scheduler claims them one at a time (rb_args.cuh claim_lazy)
#ifndef RB_CLAIM_LAZY
#define RB_CLAIM_LAZY 1
#endif
#ifndef RB_CLAIM_LAZY_MIN
#define RB_CLAIM_LAZY_MIN 16
#endif
  a.claim_lazy = RB_CLAIM_LAZY && (max_ctx_len + RB_CTX_CHUNK - 1) / RB_CTX_CHUNK >= RB_CLAIM_LAZY_MIN ? 1 : 0;
  if (ws == nullptr) return RB_OK;
  int L, ns;
  ctx_split_plan(a.b, a.hkv, max_rows, a.s_prefix, max_ctx_len, device_sms(), &L, &ns);
  if (ns < 2) return RB_OK;
  const size_t need = (size_t)rb_ctx_split_bytes(a.b, n_rows, a.hq, a.hkv, max_rows, ns);
  if (ws_bytes < need)
    return fail(RB_ERR_CONTRACT, "context split workspace too small: %zu < %zu bytes", ws_bytes, need);
  const size_t part = ((size_t)n_rows * a.hq * ns * 132 * 4 + 255) & ~(size_t)255;
  a.split_chunks = L;
  a.n_split = ns;
  a.claim_lazy = RB_CLAIM_LAZY && L >= RB_CLAIM_LAZY_MIN ? 1 : 0;
  a.split_part = static_cast<float*>(ws);
  a.split_cnt = reinterpret_cast<int*>(static_cast<uint8_t*>(ws) + part);
  return RB_OK;
}

int rb_context_attention(const void* q, long long q_row_stride, long long q_head_stride,
                         const int* q_start, int b, int n_rows, int max_rows, int hq, int hkv, int d,
                         const void* k, const void* v, const int* block_table, int bt_stride,
                         int block_size, const long long* req_offset, long long stride_block,
                         long long stride_tok, long long stride_head, const int* ctx_lens,
                         int causal, const void* prefix_k, const void* prefix_v, int s_prefix,
                         long long p_stride_tok, long long p_stride_head, const float* o_sys,
                         const float* lse_sys, float scale, void* out, int out_fp32,
                         float* lse_out, int max_ctx_len, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (d != RB_HEAD_DIM) return fail(RB_ERR_DIMENSION, "head_dim %d unsupported (kernels are d=128)", d);
  if (b < 1) return RB_OK;
  if (hq < 1 || hkv < 1 || hq % hkv != 0)
    return fail(RB_ERR_DIMENSION, "hq=%d must be a positive multiple of hkv=%d", hq, hkv);
  if (block_table == nullptr && req_offset == nullptr)
    return fail(RB_ERR_CONTRACT, "either block_table (paged) or req_offset (ragged) is required");
  if (block_table != nullptr && block_size < 1)
    return fail(RB_ERR_CONTRACT, "block_size must be >= 1");
  if ((o_sys == nullptr) != (lse_sys == nullptr))
    return fail(RB_ERR_CONTRACT, "o_sys and lse_sys go together");
  if (s_prefix > 0 && (prefix_k == nullptr || prefix_v == nullptr))
    return fail(RB_ERR_CONTRACT, "prefix K/V required when s_prefix > 0");
  rb::CtxArgs a;
  a.b = b;
  a.hq = hq;
  a.hkv = hkv;
  a.g = hq / hkv;
  a.q_start = q_start;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.q_row_stride = q_row_stride;
  a.q_head_stride = q_head_stride;
  a.ctx.k = static_cast<const __nv_bfloat16*>(k);
  a.ctx.v = static_cast<const __nv_bfloat16*>(v);
  a.ctx.block_table = block_table;
  a.ctx.bt_stride = bt_stride;
  a.ctx.block_size = block_size;
  a.ctx.req_offset = req_offset;
  a.ctx.stride_block = stride_block;
  a.ctx.stride_tok = stride_tok;
  a.ctx.stride_head = stride_head;
  a.ctx_lens = ctx_lens;
  a.causal = causal;
  a.pk = static_cast<const __nv_bfloat16*>(prefix_k);
  a.pv = static_cast<const __nv_bfloat16*>(prefix_v);
  a.p_stride_tok = p_stride_tok;
  a.p_stride_head = p_stride_head;
  a.s_prefix = s_prefix;
  a.ctx_part = nullptr;
  a.sys_part_acc = a.sys_part_ml = nullptr;
  a.sys_ready = nullptr;
  a.o_sys = o_sys;
  a.lse_sys = lse_sys;
  a.out = out;
  a.out_fp32 = out_fp32;
  a.lse_out = lse_out;
  a.scale_log2 = scale * rb::kLog2e;
  a.debug_ts = g_debug_ts ? g_debug_ts + kCtxTsOffset : nullptr;
  a.sched = nullptr;  // static item order
  a.k_new = a.v_new = nullptr;
  a.slot_mapping = nullptr;
  a.req_order = nullptr;
  int st = ctx_split_args(a, n_rows, max_rows, max_ctx_len, workspace, workspace_bytes);
  if (st != RB_OK) return st;
  return cuda_status(rb::launch_context_attention(a, max_rows, static_cast<cudaStream_t>(stream)),
                     "context attention launch");
}

// ------------------------------------------------- fused relay decode step
// Relay workspace: [256 B header: context claim / exit counters, fuse exit
// counter][n_units system-unit publication counters, 256-aligned][context
// partials, n_rows * hq * 132 floats][part m/l][part acc].
static void relay_ws_layout(const rb_sys_plan& p, size_t* cnt_bytes, size_t* cpart_bytes,
                            size_t* ml_bytes, size_t* acc_bytes) {
  *cnt_bytes = ((size_t)p.n_units * sizeof(int) + 255) & ~(size_t)255;
  *cpart_bytes = ((size_t)p.n_rows * p.hq * 132 * sizeof(float) + 255) & ~(size_t)255;
  *ml_bytes = ((size_t)p.n_units * p.max_parts * 2 * p.nq * sizeof(float) + 255) & ~(size_t)255;
  *acc_bytes = (size_t)p.n_units * p.max_parts * p.nq * RB_HEAD_DIM * sizeof(float);
}

// staging copy of the queries when the caller passes them in host memory
static size_t q_stage_bytes(int n_rows, int hq) {
  return ((size_t)n_rows * hq * RB_HEAD_DIM * 2 + 255) & ~(size_t)255;
}

static bool is_host_memory(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

int rb_relay_workspace_bytes(int n_rows, int hq, int hkv, int s, int grid_cap, int b,
                             int max_rows, int max_ctx_len, int sm_count, size_t* bytes) {
  long long f[8];
  size_t dummy = 0;
  int st = rb_sys_plan_query(n_rows, hq, hkv, s, grid_cap, f, &dummy);
  if (st != RB_OK) return st;
  rb_sys_plan p;
  rb_make_sys_plan(&p, n_rows, hq, hkv, s, grid_cap);
  size_t cnt, cpart, ml, acc;
  relay_ws_layout(p, &cnt, &cpart, &ml, &acc);
  int L, ns;
  ctx_split_plan(b, hkv, max_rows, 0, max_ctx_len, sm_count, &L, &ns);
  const size_t split = (size_t)rb_ctx_split_bytes(b, n_rows, hq, hkv, max_rows, ns);
  *bytes = 256 + cnt + cpart + ml + ((acc + 255) & ~(size_t)255) + q_stage_bytes(n_rows, hq) + split;
  return RB_OK;
}

int rb_relay_sys_grid(int n_rows, int hq, int hkv, int s, long long ctx_tokens, int sm_count,
                      int* grid) {
  if (n_rows < 1 || hq < 1 || hkv < 1 || hq % hkv != 0 || s < 1 || sm_count < 1 || ctx_tokens < 0)
    return fail(RB_ERR_DIMENSION, "bad relay split arguments");
  *grid = rb_relay_split(n_rows, hq, hkv, s, ctx_tokens, sm_count);
  return RB_OK;
}

int rb_relay_attention(const void* q, long long q_row_stride, long long q_head_stride,
                       const int* q_start, int b, int n_rows, int max_rows, int hq, int hkv, int d,
                       const void* sys_k, const void* sys_v, int s, long long sys_stride_tok,
                       long long sys_stride_head, const void* k, const void* v,
                       const int* block_table, int bt_stride, int block_size,
                       const long long* req_offset, long long stride_block, long long stride_tok,
                       long long stride_head, const int* ctx_lens, float scale, int grid_cap,
                       void* out, int out_fp32, float* lse_out, int max_ctx_len, void* workspace,
                       size_t workspace_bytes, int phases, const void* k_new, const void* v_new,
                       const int* slot_mapping, const int* req_order, void* stream) {
  if (d != RB_HEAD_DIM) return fail(RB_ERR_DIMENSION, "head_dim %d unsupported (kernels are d=128)", d);
  if ((k_new == nullptr) != (v_new == nullptr) || (k_new != nullptr) != (slot_mapping != nullptr))
    return fail(RB_ERR_CONTRACT, "k_new, v_new and slot_mapping go together");
  if (k_new != nullptr && block_table == nullptr)
    return fail(RB_ERR_CONTRACT, "the fused append needs the paged layout (block_table)");
  if ((reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new)) & 15)
    return fail(RB_ERR_CONTRACT, "k_new / v_new rows must be 16-byte aligned");
  size_t need = 0;
  const int sms = device_sms();
  int st = rb_relay_workspace_bytes(n_rows, hq, hkv, s, grid_cap, b, max_rows, max_ctx_len, sms,
                                    &need);
  if (st != RB_OK) return st;
  if (workspace_bytes < need)
    return fail(RB_ERR_CONTRACT, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  if (block_table == nullptr && req_offset == nullptr)
    return fail(RB_ERR_CONTRACT, "either block_table (paged) or req_offset (ragged) is required");
  if ((q_head_stride * 2) % 16 != 0 || (q_row_stride * 2) % 16 != 0 ||
      (reinterpret_cast<uintptr_t>(q) & 15))
    return fail(RB_ERR_CONTRACT, "q rows must be 16-byte aligned");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  rb::SysArgs sa;
  rb_make_sys_plan(&sa.plan, n_rows, hq, hkv, s, grid_cap);
  size_t cnt, cpart, ml, acc_b;
  relay_ws_layout(sa.plan, &cnt, &cpart, &ml, &acc_b);
  const size_t q_off = 256 + cnt + cpart + ml + ((acc_b + 255) & ~(size_t)255);
  const size_t split_off = q_off + q_stage_bytes(n_rows, hq);
  if ((phases & 1) && is_host_memory(q)) {
    // queries in pinned host memory (the zero-copy step): staged once into
    // the workspace; both kernels read the device copy
    __nv_bfloat16* qd = reinterpret_cast<__nv_bfloat16*>(ws + q_off);
    st = cuda_status(rb::launch_q_stage(static_cast<const __nv_bfloat16*>(q), q_row_stride,
                                        q_head_stride, n_rows, hq, qd, sms, cs),
                     "query staging launch");
    if (st != RB_OK) return st;
    q = qd;
    q_row_stride = (long long)hq * RB_HEAD_DIM;
    q_head_stride = RB_HEAD_DIM;
  }
  sa.q = static_cast<const __nv_bfloat16*>(q);
  sa.q_row_stride = q_row_stride;
  sa.q_head_stride = q_head_stride;
  sa.scale_log2 = scale * rb::kLog2e;
  sa.o_sys = nullptr;
  sa.lse_sys = nullptr;
  int* header = reinterpret_cast<int*>(ws);
  float* ctx_part = reinterpret_cast<float*>(ws + 256 + cnt);
  sa.counters = reinterpret_cast<int*>(ws + 256);
  sa.part_ml = reinterpret_cast<float*>(ws + 256 + cnt + cpart);
  sa.part_acc = reinterpret_cast<float*>(ws + 256 + cnt + cpart + ml);
  sa.debug_ts = g_debug_ts;
  sa.defer_merge = 1;
  CUtensorMap tk, tv, tq;
  st = make_kv_map(&tk, sys_k, s, hkv, sys_stride_tok, sys_stride_head);
  if (st != RB_OK) return st;
  st = make_kv_map(&tv, sys_v, s, hkv, sys_stride_tok, sys_stride_head);
  if (st != RB_OK) return st;
  maybe_q_map(&tq, &sa, q, n_rows, hq, hkv);
  if (phases & 1) {
    st = cuda_status(rb::launch_system_attention(tk, tv, tq, sa, cs), "system attention launch");
    if (st != RB_OK) return st;
  }
  if (b < 1 || !(phases & 2)) return RB_OK;
  rb::CtxArgs a;
  a.b = b;
  a.hq = hq;
  a.hkv = hkv;
  a.g = hq / hkv;
  a.q_start = q_start;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.q_row_stride = q_row_stride;
  a.q_head_stride = q_head_stride;
  a.ctx.k = static_cast<const __nv_bfloat16*>(k);
  a.ctx.v = static_cast<const __nv_bfloat16*>(v);
  a.ctx.block_table = block_table;
  a.ctx.bt_stride = bt_stride;
  a.ctx.block_size = block_size;
  a.ctx.req_offset = req_offset;
  a.ctx.stride_block = stride_block;
  a.ctx.stride_tok = stride_tok;
  a.ctx.stride_head = stride_head;
  a.ctx_lens = ctx_lens;
  a.causal = 1;
  a.pk = a.pv = nullptr;
  a.p_stride_tok = a.p_stride_head = 0;
  a.s_prefix = 0;
  a.ctx_part = ctx_part;
  a.sys_part_acc = sa.part_acc;
  a.sys_part_ml = sa.part_ml;
  a.sys_ready = sa.counters;
  a.sys_plan = sa.plan;
  a.o_sys = nullptr;
  a.lse_sys = nullptr;
  a.out = out;
  a.out_fp32 = out_fp32;
  a.lse_out = lse_out;
  a.scale_log2 = scale * rb::kLog2e;
  a.debug_ts = g_debug_ts ? g_debug_ts + kCtxTsOffset : nullptr;
  a.sched = header;  // workspace header: dynamic item counters
  a.k_new = static_cast<const __nv_bfloat16*>(k_new);
  a.v_new = static_cast<const __nv_bfloat16*>(v_new);
  a.slot_mapping = slot_mapping;
  a.req_order = req_order;
  {
    // (the context split-K plan covers the context chunks only)
    st = ctx_split_args(a, n_rows, max_rows, max_ctx_len, ws + split_off, workspace_bytes - split_off);
    if (st != RB_OK) return st;
  }
  if (!(phases & 1) && !(phases & 4)) {
    // context phase alone (profiling): the slots of an earlier phase-1 call
    // are complete; mark every unit published (the kernel rearms them)
    cudaError_t me = cudaMemsetAsync(sa.counters, 0x3f, (size_t)sa.plan.n_units * sizeof(int), cs);
    if (me != cudaSuccess) return cuda_status(me, "relay counters");
  }
  return cuda_status(rb::launch_context_attention(a, max_rows, cs),
                     "context attention launch");
}

int rb_relay_fusion(const float* o_sys, const float* lse_sys, const float* o_ctx,
                    const float* lse_ctx, float* out, float* lse_out, long long n_vec, int d,
                    void* stream) {
  if (n_vec < 0 || d < 1) return fail(RB_ERR_DIMENSION, "bad fusion shape");
  return cuda_status(rb::launch_relay_fusion(o_sys, lse_sys, o_ctx, lse_ctx, out, lse_out, n_vec,
                                             d, static_cast<cudaStream_t>(stream)),
                     "relay fusion launch");
}

int rb_kv_append(const void* k_new, const void* v_new, const int* slot_mapping, int n_tok,
                 void* k_pool, void* v_pool, int hkv, int d, int block_size,
                 long long stride_block, long long stride_tok, long long stride_head,
                 void* stream) {
  if (d != RB_HEAD_DIM) return fail(RB_ERR_DIMENSION, "head_dim %d unsupported", d);
  return cuda_status(
      rb::launch_kv_append(static_cast<const __nv_bfloat16*>(k_new),
                           static_cast<const __nv_bfloat16*>(v_new), slot_mapping,
                           static_cast<__nv_bfloat16*>(k_pool), static_cast<__nv_bfloat16*>(v_pool),
                           n_tok, hkv, block_size, stride_block, stride_tok, stride_head,
                           static_cast<cudaStream_t>(stream)),
      "kv append launch");
}

int rb_rope_rows(const float* x, float* out, const long long* positions, long long n, int d,
                 double base, void* stream) {
  if (n < 0 || d < 2 || d % 2 != 0 || d > 1024)
    return fail(RB_ERR_DIMENSION, "rope_rows requires an even dimension <= 1024, got %d", d);
  return cuda_status(rb::launch_rope_rows(x, out, positions, n, d, base,
                                          static_cast<cudaStream_t>(stream)),
                     "rope rows launch");
}

int rb_rope_append(const void* q_in, void* q_out, const void* k_new, const void* v_new,
                   const long long* positions, const int* slot_mapping, int n_tok, int hq, int hkv,
                   int d, double base, void* k_pool, void* v_pool, int block_size,
                   long long stride_block, long long stride_tok, long long stride_head,
                   void* stream) {
  if (d != RB_HEAD_DIM) return fail(RB_ERR_DIMENSION, "head_dim %d unsupported", d);
  if (n_tok < 0 || hq < 1 || hkv < 1 || hq % hkv != 0)
    return fail(RB_ERR_DIMENSION, "bad rope/append shape (n_tok=%d hq=%d hkv=%d)", n_tok, hq, hkv);
  return cuda_status(
      rb::launch_rope_append(static_cast<const __nv_bfloat16*>(q_in), static_cast<__nv_bfloat16*>(q_out),
                             static_cast<const __nv_bfloat16*>(k_new),
                             static_cast<const __nv_bfloat16*>(v_new), positions, slot_mapping,
                             n_tok, hq, hkv, base, static_cast<__nv_bfloat16*>(k_pool),
                             static_cast<__nv_bfloat16*>(v_pool), block_size, stride_block,
                             stride_tok, stride_head, static_cast<cudaStream_t>(stream)),
      "rope append launch");
}

#if RB_DIAG
int rb_debug_set_timestamps(void* buf) {
  g_debug_ts = static_cast<unsigned long long*>(buf);
  return RB_OK;
}

int rb_debug_umma_probe(const void* k, const void* q, const void* v, const void* p, int nq,
                        float* s_out, float* o_out, void* stream) {
  return cuda_status(
      rb::launch_umma_probe(static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(q),
                            static_cast<const __nv_bfloat16*>(v), static_cast<const __nv_bfloat16*>(p),
                            nq, s_out, o_out, static_cast<cudaStream_t>(stream)),
      "umma probe launch");
}
#endif  // RB_DIAG

}  // extern "C"
