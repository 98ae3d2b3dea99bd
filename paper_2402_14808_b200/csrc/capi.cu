// C-ABI boundary of librelay_b200.so (declared in include/relay_b200.h).
//
// Replaces the reference's kernel boundary, the `relayserve.kernels` module
// (/root/reference/pkg/src/relayserve/kernels.py:14-37), one level up: the
// entry points take whole attention segments instead of per-head matmul /
// softmax calls, and every attention entry point runs the ONE persistent
// relay-step kernel (relay_step_sm100.cu) in the matching mode:
//   rb_relay_step          system + context tiles + fusion (relay_attention)
//   rb_system_attention    system tiles only (_system_attention)
//   rb_context_attention   context tiles only (_context_attention /
//                          attention_with_lse), or with a per-request prefix
//                          re-read (baseline_attention, the naive baseline)
// Conventions: plain pointers and sizes, caller-allocated outputs and
// workspace, stream-ordered asynchronous launches, int status (0 = ok) with
// the message in rb_last_error(); RB_ERR_DIMENSION and RB_ERR_CONTRACT mirror
// relayserve.errors.DimensionError / ContractError (errors.py:4-9).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/relay_b200.h"
#include "rb_common.cuh"
#include "rb_plan.h"
#include "rb_args.cuh"

namespace rb {
cudaError_t launch_relay_step(const CUtensorMap*, const StepArgs&, int, cudaStream_t);
int relay_step_max_b(int nq);
cudaError_t launch_relay_fusion(const float*, const float*, const float*, const float*, float*,
                                float*, long long, int, cudaStream_t);
cudaError_t launch_kv_append(const __nv_bfloat16*, const __nv_bfloat16*, const int*, void*, void*,
                             int, int, int, long long, long long, cudaStream_t);
cudaError_t launch_umma_probe(const __nv_bfloat16*, const __nv_bfloat16*, const __nv_bfloat16*,
                              const __nv_bfloat16*, int, float*, float*, cudaStream_t);
cudaError_t launch_ctx_probe(const __nv_bfloat16*, const __nv_bfloat16*, const __nv_bfloat16*,
                             const __nv_bfloat16*, int, float*, float*, cudaStream_t);
}  // namespace rb

static thread_local std::string g_err;
static unsigned long long* g_debug_ts = nullptr;  // test-only instrumentation

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

// bf16 tensor map with 128-byte-swizzled boxes (inner box = 64 elements).
static int tmap_encode(CUtensorMap* map, int rank, const void* base, const cuuint64_t* dims,
                       const cuuint64_t* strides_bytes, const cuuint32_t* box, const char* what) {
  auto enc = get_encode();
  if (!enc) return fail(RB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return fail(RB_ERR_CONTRACT, "%s base must be 16-byte aligned", what);
  for (int i = 0; i < rank - 1; ++i)
    if (strides_bytes[i] % 16 != 0)
      return fail(RB_ERR_CONTRACT, "%s strides must be multiples of 8 elements", what);
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                   strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RB_ERR_CUDA, "cuTensorMapEncodeTiled(%s) failed (%d)", what, (int)r);
  return RB_OK;
}

// [rows][hkv][128] K or V with a (tokens, heads) stride pair: 3-D map
// {128, tokens, hkv} (or {128, hkv, tokens}), box of 128 tokens x 64 dims.
static int make_kv_map(CUtensorMap* map, const void* base, long long tokens, int hkv,
                       long long stride_tok, long long stride_head, bool tokens_outer,
                       const char* what) {
  if (tokens_outer) {
    cuuint64_t dims[3] = {RB_HEAD_DIM, (cuuint64_t)hkv, (cuuint64_t)tokens};
    cuuint64_t str[2] = {(cuuint64_t)(stride_head * 2), (cuuint64_t)(stride_tok * 2)};
    cuuint32_t box[3] = {64, 1, RB_KEY_TILE};
    return tmap_encode(map, 3, base, dims, str, box, what);
  }
  cuuint64_t dims[3] = {RB_HEAD_DIM, (cuuint64_t)tokens, (cuuint64_t)hkv};
  cuuint64_t str[2] = {(cuuint64_t)(stride_tok * 2), (cuuint64_t)(stride_head * 2)};
  cuuint32_t box[3] = {64, RB_KEY_TILE, 1};
  return tmap_encode(map, 3, base, dims, str, box, what);
}

// ------------------------------------------------------------------ plan
static int step_nq(int rows_per_head) { return rows_per_head <= 16 ? 16 : 32; }

// The stream-K plan of the system tiles (rb_plan.h) with the query tile the
// relay step uses.  s < 1 (no shared prefix in this launch) gives an empty plan.
static void make_step_plan(rb_sys_plan* p, int n_rows, int hq, int hkv, int s, int grid_cap) {
  memset(p, 0, sizeof(*p));
  p->n_rows = n_rows;
  p->hq = hq;
  p->hkv = hkv;
  p->g = hq / hkv;
  p->s = s > 0 ? s : 0;
  p->rows_per_head = n_rows * p->g;
  p->nq = step_nq(p->rows_per_head);
  p->n_qt = (p->rows_per_head + p->nq - 1) / p->nq;
  p->tpu = (p->s + RB_KEY_TILE - 1) / RB_KEY_TILE;
  p->n_units = hkv * p->n_qt;
  p->total = (long long)p->n_units * p->tpu;
  const long long gcap = grid_cap < 1 ? 1 : grid_cap;
  p->grid = (int)(p->total < gcap ? p->total : gcap);
  p->max_parts = 1;
  if (p->total > 0) {
    for (int u = 0; u < p->n_units; ++u) {
      const int c = rb_unit_parts(p, u);
      if (c > p->max_parts) p->max_parts = c;
    }
  }
}

struct StepWs {
  size_t cnt, sys_ml, sys_acc, ctx_ml, ctx_acc, total;
};
static StepWs step_ws(const rb_sys_plan& p) {
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  StepWs w;
  w.cnt = 0;
  w.sys_ml = up(64);
  // two partial slots per (system unit, CTA) and per context row: one per
  // softmax group of the relay step
  const size_t slots = (size_t)p.n_units * 2 * p.max_parts;
  w.sys_acc = w.sys_ml + up(slots * 2 * p.nq * sizeof(float));
  w.ctx_ml = w.sys_acc + up(slots * p.nq * RB_HEAD_DIM * sizeof(float));
  w.ctx_acc = w.ctx_ml + up((size_t)2 * p.n_rows * p.hq * 2 * sizeof(float));
  w.total = w.ctx_acc + up((size_t)2 * p.n_rows * p.hq * RB_HEAD_DIM * sizeof(float));
  return w;
}

static int check_heads(int n_rows, int hq, int hkv) {
  if (n_rows < 1 || hq < 1 || hkv < 1) return fail(RB_ERR_DIMENSION, "empty query set");
  if (hq % hkv != 0) return fail(RB_ERR_DIMENSION, "hq=%d not a multiple of hkv=%d", hq, hkv);
  return RB_OK;
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

int rb_step_plan_query(int n_rows, int hq, int hkv, int s, int grid_cap, long long* fields,
                       size_t* workspace_bytes) {
  int st = check_heads(n_rows, hq, hkv);
  if (st != RB_OK) return st;
  rb_sys_plan p;
  make_step_plan(&p, n_rows, hq, hkv, s, grid_cap);
  if (fields) {
    fields[0] = p.nq;
    fields[1] = p.n_qt;
    fields[2] = p.tpu;
    fields[3] = p.n_units;
    fields[4] = p.total;
    fields[5] = p.grid;
    fields[6] = p.max_parts;
  }
  if (workspace_bytes) *workspace_bytes = step_ws(p).total;
  return RB_OK;
}

int rb_relay_step_supported(int n_rows, int hq, int hkv, int b, int block_size, int paged) {
  if (n_rows < 1 || hq < 1 || hkv < 1 || hq % hkv != 0) return 0;
  const int g = hq / hkv;
  const int nq = step_nq(n_rows * g);
  if (nq % g != 0) return 0;
  if (b > rb::relay_step_max_b(nq)) return 0;
  if (paged && block_size != 16 && block_size != 32 && block_size != 64) return 0;
  return 1;
}

int rb_relay_step(const void* q, long long q_row_stride, long long q_head_stride,
                  const int* q_start, int b, int n_rows, int max_rows, int hq, int hkv, int d,
                  const void* sys_k, const void* sys_v, int s, long long sys_stride_tok,
                  long long sys_stride_head, const void* k, const void* v, long long ctx_extent,
                  const int* block_table, int bt_stride, int block_size,
                  const long long* req_offset, long long stride_block, long long stride_tok,
                  long long stride_head, const int* ctx_lens, int causal, int prefix_mode,
                  float scale, int grid_cap, void* out, int out_fp32, float* lse_out,
                  void* workspace, size_t workspace_bytes, int phases, void* stream) {
  if (d != RB_HEAD_DIM) return fail(RB_ERR_DIMENSION, "head_dim %d unsupported (kernels are d=128)", d);
  int st = check_heads(n_rows, hq, hkv);
  if (st != RB_OK) return st;
  const bool want_sys = (phases & 1) && !prefix_mode;
  const bool want_ctx = (phases & 2) && b > 0;
  if ((want_sys || prefix_mode) && s < 1)
    return fail(RB_ERR_CONTRACT,
                "relay attention requires a non-empty system segment; use the baseline path "
                "when there is no shared prefix");
  const int paged = block_table != nullptr;
  if (want_ctx && !paged && req_offset == nullptr)
    return fail(RB_ERR_CONTRACT, "either block_table (paged) or req_offset (ragged) is required");
  if (!rb_relay_step_supported(n_rows, hq, hkv, want_ctx ? b : 0, block_size, want_ctx && paged))
    return fail(RB_ERR_CONTRACT,
                "shape not supported: GQA group must divide the query tile (g in 1,2,4,8,16), "
                "b <= %d, paged block size 16/32/64", rb::relay_step_max_b(32));
  rb::StepArgs a;
  memset(&a, 0, sizeof(a));
  make_step_plan(&a.sp, n_rows, hq, hkv, want_sys ? s : 0, grid_cap);
  a.sp.s = s > 0 ? s : 0;  // prefix length also bounds the naive mode's prefix tiles
  size_t need = step_ws(a.sp).total;
  if (workspace_bytes < need)
    return fail(RB_ERR_CONTRACT, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  const int g = a.sp.g, nq = a.sp.nq;
  a.has_sys = want_sys ? 1 : 0;
  a.has_ctx = want_ctx ? 1 : 0;
  a.b = want_ctx ? b : 0;
  const int max_m = (max_rows + g - 1) / g;
  a.ctx_rows_box = max_m < nq / g ? max_m : nq / g;
  if (a.ctx_rows_box < 1) a.ctx_rows_box = 1;
  a.paged = paged;
  a.block_size = paged ? block_size : RB_KEY_TILE;
  a.causal = causal ? 1 : 0;
  a.prefix_tiles = prefix_mode ? (s + RB_KEY_TILE - 1) / RB_KEY_TILE : 0;
  a.k_pool = static_cast<const unsigned char*>(k);
  a.v_pool = static_cast<const unsigned char*>(v);
  a.pool_block_bytes = stride_block * 2;
  a.pool_head_bytes = stride_head * 2;
  a.q_start = q_start;
  a.ctx_lens = ctx_lens;
  a.block_table = block_table;
  a.bt_stride = bt_stride;
  a.req_offset = req_offset;
  a.scale_log2 = scale * rb::kLog2e;
  const StepWs w = step_ws(a.sp);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  a.counters = reinterpret_cast<int*>(ws + w.cnt);
  a.sys_ml = reinterpret_cast<float*>(ws + w.sys_ml);
  a.sys_acc = reinterpret_cast<float*>(ws + w.sys_acc);
  a.ctx_ml = reinterpret_cast<float*>(ws + w.ctx_ml);
  a.ctx_acc = reinterpret_cast<float*>(ws + w.ctx_acc);
  a.out = out;
  a.out_fp32 = out_fp32;
  a.lse_out = lse_out;
  a.debug_ts = g_debug_ts;
  if (a.paged && a.has_ctx) {
    if ((reinterpret_cast<uintptr_t>(k) & 15) || (reinterpret_cast<uintptr_t>(v) & 15) ||
        (a.pool_block_bytes & 15) || (a.pool_head_bytes & 15))
      return fail(RB_ERR_CONTRACT, "paged pool blocks must be 16-byte aligned");
  }

  // maps: q (system box), q (context box), prefix k, prefix v, ragged ctx k, v
  CUtensorMap maps[6];
  {
    if ((q_head_stride * 2) % 16 != 0 || (q_row_stride * 2) % 16 != 0)
      return fail(RB_ERR_CONTRACT, "q rows must be 16-byte aligned");
    cuuint64_t dims[4] = {RB_HEAD_DIM, (cuuint64_t)g, (cuuint64_t)hkv, (cuuint64_t)n_rows};
    cuuint64_t str[3] = {(cuuint64_t)(q_head_stride * 2), (cuuint64_t)(g * q_head_stride * 2),
                         (cuuint64_t)(q_row_stride * 2)};
    cuuint32_t box_s[4] = {64, (cuuint32_t)g, 1, (cuuint32_t)(nq / g)};
    cuuint32_t box_c[4] = {64, (cuuint32_t)g, 1, (cuuint32_t)a.ctx_rows_box};
    if ((st = tmap_encode(&maps[0], 4, q, dims, str, box_s, "q")) != RB_OK) return st;
    if ((st = tmap_encode(&maps[1], 4, q, dims, str, box_c, "q")) != RB_OK) return st;
  }
  if (s > 0 && (a.has_sys || a.prefix_tiles > 0)) {
    if ((st = make_kv_map(&maps[2], sys_k, s, hkv, sys_stride_tok, sys_stride_head, false,
                          "system K")) != RB_OK)
      return st;
    if ((st = make_kv_map(&maps[3], sys_v, s, hkv, sys_stride_tok, sys_stride_head, false,
                          "system V")) != RB_OK)
      return st;
  } else {
    maps[2] = maps[0];
    maps[3] = maps[0];
  }
  if (a.has_ctx && !a.paged) {
    if (ctx_extent < 1) return fail(RB_ERR_CONTRACT, "context extent must be >= 1");
    if ((st = make_kv_map(&maps[4], k, ctx_extent, hkv, stride_tok, stride_head, true,
                          "context K")) != RB_OK)
      return st;
    if ((st = make_kv_map(&maps[5], v, ctx_extent, hkv, stride_tok, stride_head, true,
                          "context V")) != RB_OK)
      return st;
  } else {
    maps[4] = maps[0];
    maps[5] = maps[0];
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = grid_cap > 0 && grid_cap < sms ? grid_cap : sms;
  return cuda_status(rb::launch_relay_step(maps, a, grid, static_cast<cudaStream_t>(stream)),
                     "relay step launch");
}

int rb_system_attention(const void* q, long long q_row_stride, long long q_head_stride,
                        int n_rows, int hq, int hkv, int d, const void* sys_k, const void* sys_v,
                        int s, long long kv_stride_tok, long long kv_stride_head, float scale,
                        int grid_cap, float* o_sys, float* lse_sys, void* workspace,
                        size_t workspace_bytes, void* stream) {
  return rb_relay_step(q, q_row_stride, q_head_stride, nullptr, 0, n_rows, 1, hq, hkv, d, sys_k,
                       sys_v, s, kv_stride_tok, kv_stride_head, nullptr, nullptr, 0, nullptr, 0, 0,
                       nullptr, 0, 0, 0, nullptr, 0, 0, scale, grid_cap, o_sys, 1, lse_sys,
                       workspace, workspace_bytes, 1, stream);
}

int rb_context_attention(const void* q, long long q_row_stride, long long q_head_stride,
                         const int* q_start, int b, int n_rows, int max_rows, int hq, int hkv,
                         int d, const void* k, const void* v, long long ctx_extent,
                         const int* block_table, int bt_stride, int block_size,
                         const long long* req_offset, long long stride_block, long long stride_tok,
                         long long stride_head, const int* ctx_lens, int causal,
                         const void* prefix_k, const void* prefix_v, int s_prefix,
                         long long p_stride_tok, long long p_stride_head, float scale,
                         int grid_cap, void* out, int out_fp32, float* lse_out, void* workspace,
                         size_t workspace_bytes, void* stream) {
  if (s_prefix > 0 && (prefix_k == nullptr || prefix_v == nullptr))
    return fail(RB_ERR_CONTRACT, "prefix K/V required when s_prefix > 0");
  return rb_relay_step(q, q_row_stride, q_head_stride, q_start, b, n_rows, max_rows, hq, hkv, d,
                       prefix_k, prefix_v, s_prefix, p_stride_tok, p_stride_head, k, v,
                       ctx_extent, block_table, bt_stride, block_size, req_offset, stride_block,
                       stride_tok, stride_head, ctx_lens, causal, s_prefix > 0 ? 1 : 0, scale,
                       grid_cap, out, out_fp32, lse_out, workspace, workspace_bytes, 2, stream);
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
                 long long stride_block, long long stride_head, void* stream) {
  if (d != RB_HEAD_DIM) return fail(RB_ERR_DIMENSION, "head_dim %d unsupported", d);
  if (block_size != 16 && block_size != 32 && block_size != 64)
    return fail(RB_ERR_CONTRACT, "paged block size must be 16, 32 or 64");
  return cuda_status(
      rb::launch_kv_append(static_cast<const __nv_bfloat16*>(k_new),
                           static_cast<const __nv_bfloat16*>(v_new), slot_mapping, k_pool, v_pool,
                           n_tok, hkv, block_size, stride_block * 2, stride_head * 2,
                           static_cast<cudaStream_t>(stream)),
      "kv append launch");
}

int rb_debug_umma_probe(const void* k, const void* q, const void* v, const void* p, int nq,
                        float* s_out, float* o_out, void* stream) {
  return cuda_status(
      rb::launch_umma_probe(static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(q),
                            static_cast<const __nv_bfloat16*>(v), static_cast<const __nv_bfloat16*>(p),
                            nq, s_out, o_out, static_cast<cudaStream_t>(stream)),
      "umma probe launch");
}

int rb_debug_ctx_probe(const void* k, const void* q, const void* v, const void* p, int block_size,
                       float* s_out, float* o_out, void* stream) {
  return cuda_status(
      rb::launch_ctx_probe(static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(q),
                           static_cast<const __nv_bfloat16*>(v), static_cast<const __nv_bfloat16*>(p),
                           block_size, s_out, o_out, static_cast<cudaStream_t>(stream)),
      "ctx probe launch");
}

int rb_debug_set_timestamps(void* buf) {
  g_debug_ts = static_cast<unsigned long long*>(buf);
  return RB_OK;
}

}  // extern "C"
