// One relay decode step in ONE persistent sm_100a kernel: system-prompt
// attention, request-context attention and the relay fusion.
//
// Reference path (/root/reference/pkg/src/relayserve/attention.py):
//   relay_attention_ragged (:203-243) = _system_attention (:177-200, one
//   unmasked attention_with_lse over the shared prefix for the whole batch)
//   + _context_attention (:160-174, causal attention_with_lse per request)
//   + relay_fusion (:137-157, LSE-weighted merge of the two partials).
//
// B200 design:
//  * Work = a stream of 128-key tiles.  System tiles: unit (kv head h, query
//    tile qt) x key tile kt of the shared prefix, split stream-K over the CTAs
//    (every shared byte read once per step).  Context tiles: unit (request r,
//    kv head h, q-tile z) x key tile kt of r's own context, units kept whole
//    and balanced over the CTAs by tile count (prefix sum over ctx_lens,
//    computed on the device so the step is CUDA-graph capturable).  CTA c
//    runs its system range, then its context range.
//  * Every tile goes through the same pipeline (swap-AB, the 128 keys are the
//    MMA M dimension, the unit's <= NQ query rows are N):
//        S^T[128 x NQ] = K_tile . Q^T        (tcgen05, TMEM accumulator)
//        O^T[128 x NQ] += V_tile^T . P^T     (tcgen05, O stays in TMEM)
//    K, V and Q tiles arrive by TMA (3-D map of the prefix, 4-D map of the
//    paged pool read in place through the block table, 4-D map of the
//    queries that picks a KV head's GQA group).
//  * Softmax: one 4-warp group, thread = key lane, NQ columns per thread,
//    log2 domain.  Lazy rescaling: the running max of a column only moves
//    when a tile exceeds it by more than kTau (P <= 2^kTau), so O is
//    accumulated by the tensor core across the whole part and is rescaled in
//    TMEM only on those rare moves; row sums stay per-lane until the part ends.
//  * Epilogue group (4 warps, thread = head dim): drains a finished part's O
//    from TMEM (double-buffered per part) and writes the partial (acc, m, l)
//    -- no synchronisation per part.  When a CTA's parts are all written it
//    joins a grid barrier (one CTA per SM, all resident); then every CTA
//    merges its share of the output vectors: context partial + system
//    stream-K parts, the relay fusion.  Partials live in L2 (a few MB), they
//    never take an HBM round trip of their own.
//  * Warp roles (12 warps): 0 K/Q TMA producer, 1 QK^T issuer (TMEM owner),
//    2 V TMA producer, 3 metadata scan then P.V issuer, 4-7 softmax,
//    8-11 epilogue.
#include "rb_common.cuh"
#include "rb_plan.h"
#include "rb_args.cuh"

namespace rb {

constexpr float kTau = 8.0f;  // lazy-rescale threshold (log2 units)

template <int NQ>
struct StepCfg {
  static constexpr int KS = 2, VS = 3, QS = 4;
  static constexpr int kTile = RB_KEY_TILE * RB_HEAD_DIM * 2;  // 32 KB K or V tile
  static constexpr int kQBytes = NQ * 256;                     // [2 kblocks][NQ][128 B]
  static constexpr int kThreads = 12 * 32;
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + KS * kTile;
  static constexpr int kOffQ = kOffV + VS * kTile;
  static constexpr int kOffP = kOffQ + QS * kQBytes;
  static constexpr int kOffRed = kOffP + 2 * kQBytes;   // float [2][4][NQ] tile max per quadrant
  static constexpr int kOffRed2 = kOffRed + 2 * 4 * NQ * 4;  // float [4][NQ] row sums
  static constexpr int kOffMu = kOffRed2 + 4 * NQ * 4;       // float [4 warps][NQ] reference max
  static constexpr int kOffAl = kOffMu + 4 * NQ * 4;         // float [4 warps][NQ] rescale factor
  static constexpr int kOffHand = kOffAl + 4 * NQ * 4;       // float [2][2][NQ] part (m, l)
  static constexpr int kOffMisc = kOffHand + 2 * 2 * NQ * 4; // int [16]
  static constexpr int kIdAhead = 4;                          // block-id lookahead (tiles)
  static constexpr int kOffIds = kOffMisc + 64;               // int [2 producers][kIdAhead][32]
  static constexpr int kOffBar = kOffIds + 2 * kIdAhead * 32 * 4;
  static constexpr int kNumBars = 2 * KS + 2 * VS + 2 * QS + 18;  // rings + s,p,o,h pairs + meta + v_go
  static constexpr int kOffMeta = kOffBar + kNumBars * 8;  // int P[b+1], lens[b], qs[b+1]
  static constexpr int kTmemCols = (4 * NQ <= 32) ? 32 : (4 * NQ <= 64) ? 64 : 128;
  static int smem_bytes(int b) { return kOffMeta + 4 * (3 * b + 2) + 16; }
};

// One tile of this CTA's work sequence.
struct Tile {
  int kind;         // 0 = system, 1 = context
  int u;            // system unit (also the output group of a system tile)
  int r, h, z;      // context unit
  int kt;           // key tile inside the unit
  int first, last;  // first / last tile of this CTA's part of the unit
};

// Query tiles of request r's context units: ceil(m_r * g / NQ).
__device__ __forceinline__ int ctx_nz(const StepArgs& a, const int* qs, int r) {
  return ((qs[r + 1] - qs[r]) * a.sp.g + a.sp.nq - 1) / a.sp.nq;
}

// Walks a CTA's sequence: system tiles [x0, xe) then context tiles [cx, ce).
struct Walker {
  long long x0, x, xe;
  int cx, ce, r;
  int ctx_ready;
  __device__ __forceinline__ void init(const StepArgs& a, int cta) {
    x0 = x = xe = 0;
    if (a.has_sys && cta < a.sp.grid) {
      x0 = x = rb_cta_begin(&a.sp, cta);
      xe = rb_cta_begin(&a.sp, cta + 1);
    }
    cx = ce = r = 0;
    ctx_ready = 0;
  }
  __device__ __forceinline__ bool next(const StepArgs& a, const int* P, const int* lens,
                                       const int* qs, const int* misc, uint64_t* meta_bar,
                                       Tile& t) {
    if (x < xe) {
      const rb_sys_plan& p = a.sp;
      t.kind = 0;
      t.u = static_cast<int>(x / p.tpu);
      t.kt = static_cast<int>(x % p.tpu);
      t.first = (x == x0) || t.kt == 0;
      t.last = (x == xe - 1) || t.kt == p.tpu - 1;
      t.r = t.h = t.z = 0;
      ++x;
      return true;
    }
    if (!a.has_ctx) return false;
    if (!ctx_ready) {
      mbar_wait(meta_bar, 0);
      cx = misc[2];
      ce = misc[3];
      r = 0;
      ctx_ready = 1;
    }
    if (cx >= ce) return false;
    while (P[r + 1] <= cx) ++r;
    const int tr = (lens[r] + RB_KEY_TILE - 1) / RB_KEY_TILE;
    const int local = cx - P[r];
    const int ui = local / tr;
    const int nz = ctx_nz(a, qs, r);
    t.kind = 1;
    t.r = r;
    t.h = ui / nz;
    t.z = ui % nz;
    t.kt = local % tr;
    t.first = t.kt == 0;
    t.last = t.kt == tr - 1;
    t.u = 0;
    ++cx;
    return true;
  }
};

template <int H, bool IS_MAX>
__device__ __forceinline__ float warp_reduce_cols(float (&v)[H], int lane) {
  // reduce-scatter over the 32 lanes: afterwards lane l holds the reduction of
  // column reduced_col<H>(l) = l / (32 / H) over all 32 lanes.
#pragma unroll
  for (int n = H, mask = 16; n > 1; n >>= 1, mask >>= 1) {
    const bool upper = (lane & mask) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float send = upper ? v[i] : v[i + n / 2];
      const float keep = upper ? v[i + n / 2] : v[i];
      const float recv = __shfl_xor_sync(0xffffffffu, send, mask);
      v[i] = IS_MAX ? fmaxf(keep, recv) : keep + recv;
    }
  }
  float r = v[0];
#pragma unroll
  for (int mask = 16 / H; mask >= 1; mask >>= 1) {
    const float o = __shfl_xor_sync(0xffffffffu, r, mask);
    r = IS_MAX ? fmaxf(r, o) : r + o;
  }
  return r;
}
template <int H>
__device__ __forceinline__ int reduced_col(int lane) { return lane / (32 / H); }
template <int H>
__device__ __forceinline__ bool reduced_writer(int lane) { return (lane % (32 / H)) == 0; }

// OR-reduction of a predicate over `n` threads at named barrier `id`.
__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t n, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "barrier.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(pred)), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

constexpr float kNegBig = -1.0e30f;  // "no key yet" reference max (exp2 of -inf - kNegBig = 0)

// Shared-memory / TMEM context of the softmax group.
struct SmxCtx {
  float* red;       // [2][4][NQ] tile maxima per quadrant
  float* red2;      // [4][NQ] row sums
  float* my_mu;     // [NQ] this warp's copy of the reference max per column
  float* my_al;     // [NQ] this warp's copy of the rescale factors
  float* hand;      // [2][2][NQ] part (m, l) -> epilogue
  uint8_t* pbase;   // P tile of this thread's key half (add sb * kQBytes)
  uint32_t poff[8];
  uint32_t lane_addr;  // TMEM address of this warp's lane quadrant
  int qd, lane;
};

// One tile of the softmax group for HC <= NQ live columns (HC = 8 for context
// units with few query rows, HC = NQ otherwise).  x: masked, log2-scaled
// scores of this thread's key lane.  Lazy rescaling: the common path is one
// OR-barrier (does any score exceed its column's reference max by > kTau?),
// exp2, row-sum accumulation and the P store; the reference maxima and the
// O accumulator in TMEM only change on the rare path.
template <int HC, int NQ>
__device__ __forceinline__ void softmax_tile(const SmxCtx& C, float (&x)[HC], float (&mr)[NQ],
                                             float (&l_part)[NQ], bool first, int j, int n,
                                             uint64_t* p_empty, uint64_t* p_full, int qbytes) {
  if (first) {
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      mr[c] = kNegBig;
      l_part[c] = 0.f;
    }
    if (reduced_writer<HC>(C.lane)) C.my_mu[reduced_col<HC>(C.lane)] = kNegBig;
  }
  bool ex = false;
#pragma unroll
  for (int c = 0; c < HC; ++c) ex |= x[c] > mr[c] + kTau;
  if (bar_red_or(1, 128, ex)) {
    // ---- rare path: per-column tile max over the 128 key lanes
    float tmp[HC];
#pragma unroll
    for (int c = 0; c < HC; ++c) tmp[c] = x[c];
    const float wmax = warp_reduce_cols<HC, true>(tmp, C.lane);
    const int rc = reduced_col<HC>(C.lane);
    const bool rw = reduced_writer<HC>(C.lane);
    float* rb = C.red + (j & 1) * 4 * NQ;
    if (rw) rb[C.qd * NQ + rc] = wmax;
    named_bar_sync(1, 128);
    const float tm = fmaxf(fmaxf(rb[rc], rb[NQ + rc]), fmaxf(rb[2 * NQ + rc], rb[3 * NQ + rc]));
    const float mold = C.my_mu[rc];
    const bool mv = tm > mold + kTau;
    const float alpha = mv ? fast_exp2(mold - tm) : 1.f;  // 0 when mold is kNegBig
    const bool from_finite = mv && mold > 0.5f * kNegBig;
    __syncwarp();
    if (rw) {
      if (mv) C.my_mu[rc] = tm;
      C.my_al[rc] = alpha;
    }
    const bool need_o = __any_sync(0xffffffffu, from_finite) && !first;
    __syncwarp();
#pragma unroll
    for (int c = 0; c < HC; ++c) mr[c] = C.my_mu[c];
    if (need_o) {
      // rescale the row sums and O (after the previous P.V has landed in TMEM)
#pragma unroll
      for (int c = 0; c < HC; ++c) l_part[c] *= C.my_al[c];
      mbar_wait(&p_empty[(j - 1) & 1], ((j - 1) >> 1) & 1);
      tc_fence_after();
      const uint32_t oaddr = C.lane_addr + 2 * NQ + (n & 1) * NQ;
#pragma unroll
      for (int c0 = 0; c0 < HC; c0 += 8) {
        float o[8];
        tmem_ld_32x32b<8>(oaddr + c0, o);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 8; ++c) o[c] *= C.my_al[c0 + c];
        tmem_st_32x32b<8>(oaddr + c0, o);
      }
      tmem_wait_st();
    }
  }
  // ---- P = 2^(x - m) (bf16) into the K-major SW128 [NQ][128 keys] tile
#pragma unroll
  for (int c = 0; c < HC; ++c) {
    x[c] = fast_exp2(x[c] - mr[c]);
    l_part[c] += x[c];
  }
  const int sb = j & 1;
  mbar_wait(&p_empty[sb], ((j >> 1) & 1) ^ 1);
  uint8_t* pdst = C.pbase + sb * qbytes;
#pragma unroll
  for (int c = 0; c < HC; ++c)
    *reinterpret_cast<__nv_bfloat16*>(pdst + (c >> 3) * 1024 + C.poff[c & 7]) =
        __float2bfloat16_rn(x[c]);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncwarp();
  if (C.lane == 0) mbar_arrive(&p_full[sb]);
}

// Part end: row sums over the 128 key lanes and the reference maxima go to the
// epilogue through `hand` (columns < HC).
template <int HC, int NQ>
__device__ __forceinline__ void softmax_part_end(const SmxCtx& C, const float (&l_part)[NQ], int n,
                                                 uint64_t* h_empty, uint64_t* h_full) {
  float tmp[HC];
#pragma unroll
  for (int c = 0; c < HC; ++c) tmp[c] = l_part[c];
  const float wsum = warp_reduce_cols<HC, false>(tmp, C.lane);
  const int rc = reduced_col<HC>(C.lane);
  const bool rw = reduced_writer<HC>(C.lane);
  if (rw) C.red2[C.qd * NQ + rc] = wsum;
  named_bar_sync(1, 128);
  if (C.qd == 0) {
    const int ob = n & 1;
    mbar_wait(&h_empty[ob], ((n >> 1) & 1) ^ 1);
    if (rw) {
      C.hand[ob * 2 * NQ + rc] = C.my_mu[rc];
      C.hand[ob * 2 * NQ + NQ + rc] =
          C.red2[rc] + C.red2[NQ + rc] + C.red2[2 * NQ + rc] + C.red2[3 * NQ + rc];
    }
    __syncwarp();
    if (C.lane == 0) mbar_arrive(&h_full[ob]);
  }
}

// Final merge, after the grid barrier: output vector (row t, query head hh)
// = LSE-weighted combine of its context partial (if the request has a
// context) and the system stream-K parts of its group u = (hh / g, f / NQ),
// in a fixed order (context, then parts by slot): the relay fusion of
// attention.py:137-157 with max-subtracted weights.  One warp per vector,
// lane = 4 head dims.
template <int NQ>
__device__ __forceinline__ void merge_vector(const StepArgs& a, const int* qs, const int* lens,
                                             long long v, int lane) {
  const rb_sys_plan& p = a.sp;
  const int t = static_cast<int>(v / p.hq), hh = static_cast<int>(v % p.hq);
  const int h = hh / p.g, j = hh % p.g;
  const int f = t * p.g + j;
  const int u = h * p.n_qt + f / NQ, col = f % NQ;
  const int np = a.has_sys ? rb_unit_parts(&p, u) : 0;
  bool hasc = false;
  if (a.has_ctx) {
    int lo = 0, hi = a.b - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (qs[mid] <= t) lo = mid; else hi = mid - 1;
    }
    hasc = lens[lo] > 0;
  }
  const long long ubase = static_cast<long long>(u) * p.max_parts;
  // pass 1: the common max (context partial and every part's m)
  float mc = -INFINITY, lc = 0.f;
  float4 xc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (hasc) {
    const float2 ml = __ldcg(reinterpret_cast<const float2*>(a.ctx_ml) + v);
    mc = ml.x;
    lc = ml.y;
    xc = __ldcg(reinterpret_cast<const float4*>(a.ctx_acc + v * RB_HEAD_DIM) + lane);
  }
  float M = mc;
#pragma unroll 4
  for (int k = 0; k < np; ++k) M = fmaxf(M, __ldcg(a.sys_ml + (ubase + k) * 2 * NQ + col));
  // pass 2: weighted sums in fixed order (context, then parts by slot)
  float L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  if (mc != -INFINITY) {
    const float w = fast_exp2(mc - M);
    L = lc * w;
    O = make_float4(xc.x * w, xc.y * w, xc.z * w, xc.w * w);
  }
#pragma unroll 4
  for (int k = 0; k < np; ++k) {
    const float* ml = a.sys_ml + (ubase + k) * 2 * NQ;
    const float mk = __ldcg(ml + col), lk = __ldcg(ml + NQ + col);
    const float4 xk = __ldcg(reinterpret_cast<const float4*>(
                                 a.sys_acc + ((ubase + k) * NQ + col) * RB_HEAD_DIM) + lane);
    if (mk != -INFINITY) {
      const float w = fast_exp2(mk - M);
      L += lk * w;
      O.x += xk.x * w; O.y += xk.y * w; O.z += xk.z * w; O.w += xk.w * w;
    }
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  O.x *= inv; O.y *= inv; O.z *= inv; O.w *= inv;
  if (a.out_fp32) {
    reinterpret_cast<float4*>(static_cast<float*>(a.out) + v * RB_HEAD_DIM)[lane] = O;
  } else {
    uint2 pk;
    pk.x = pack_bf16x2(O.x, O.y);
    pk.y = pack_bf16x2(O.z, O.w);
    reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + v * RB_HEAD_DIM)[lane] = pk;
  }
  if (a.lse_out != nullptr && lane == 0)
    a.lse_out[v] = L > 0.f ? (M + __log2f(L)) * kLn2 : -INFINITY;
}

// Sense-reversing grid barrier over all CTAs of the launch (all resident:
// one CTA per SM, cooperative launch).  bar[0] = arrivals, bar[1] = generation.
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nctas) {
  unsigned int gen;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
  fence_acq_rel_gpu();  // release this CTA's partials (cumulative over the CTA barrier)
  const unsigned int prev = atomicAdd(bar, 1u);
  if (prev == nctas - 1) {
    bar[0] = 0;
    fence_acq_rel_gpu();
    atomicAdd(bar + 1, 1u);
  } else {
    unsigned int cur;
    do {
      __nanosleep(64);
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
    } while (cur == gen);
  }
  fence_acq_rel_gpu();  // acquire every CTA's partials
}

template <int NQ>
__global__ void __launch_bounds__(StepCfg<NQ>::kThreads, 1)
    relay_step_kernel(const __grid_constant__ CUtensorMap tm_qs,
                      const __grid_constant__ CUtensorMap tm_qc,
                      const __grid_constant__ CUtensorMap tm_sk,
                      const __grid_constant__ CUtensorMap tm_sv,
                      const __grid_constant__ CUtensorMap tm_ck,
                      const __grid_constant__ CUtensorMap tm_cv, const StepArgs a) {
  using L = StepCfg<NQ>;
  constexpr int H = NQ;
  constexpr int KS = L::KS, VS = L::VS, QS = L::QS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;
  uint64_t* v_empty = v_full + VS;
  uint64_t* q_full = v_empty + VS;
  uint64_t* q_empty = q_full + QS;
  uint64_t* s_full = q_empty + QS;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 2;
  uint64_t* o_full = p_empty + 2;
  uint64_t* o_free = o_full + 2;
  uint64_t* meta_bar = o_free + 2;
  // handoff softmax -> epilogue (m, l of a finished part)
  uint64_t* h_full = meta_bar + 1;
  uint64_t* h_empty = h_full + 2;
  uint64_t* v_go = h_empty + 2;  // first K tile landed: V streaming may start
  static_assert(2 * KS + 2 * VS + 2 * QS + 18 == L::kNumBars, "barrier count");
  int* misc = reinterpret_cast<int*>(smem + L::kOffMisc);
  int* P = reinterpret_cast<int*>(smem + L::kOffMeta);
  int* lens = P + (a.b + 1);
  int* qs = lens + a.b;
  float* red = reinterpret_cast<float*>(smem + L::kOffRed);
  float* red2 = reinterpret_cast<float*>(smem + L::kOffRed2);
  float* mu = reinterpret_cast<float*>(smem + L::kOffMu);
  float* al = reinterpret_cast<float*>(smem + L::kOffAl);
  float* hand = reinterpret_cast<float*>(smem + L::kOffHand);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* dts = a.debug_ts ? a.debug_ts + blockIdx.x * 512 : nullptr;
  if (dts && threadIdx.x == 0) dts[0] = global_timer_ns();

  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023) != 0) __trap();  // SW128 tiles need 1 KB alignment
    for (int i = 0; i < KS; ++i) { mbar_init(&k_full[i], 1); mbar_init(&k_empty[i], 1); }
    for (int i = 0; i < VS; ++i) { mbar_init(&v_full[i], 1); mbar_init(&v_empty[i], 1); }
    for (int i = 0; i < QS; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_empty[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 4);
      mbar_init(&h_full[i], 1);
      mbar_init(&h_empty[i], 4);
    }
    mbar_init(meta_bar, 1);
    mbar_init(v_go, 1);
    fence_mbar_init();
  } else if (warp == 0 && lane == 1) {
    tma_prefetch_desc(&tm_qs);
    tma_prefetch_desc(&tm_sk);
    tma_prefetch_desc(&tm_sv);
  } else if (warp == 2 && lane == 1) {
    tma_prefetch_desc(&tm_qc);
    tma_prefetch_desc(&tm_ck);
    tma_prefetch_desc(&tm_cv);
  }
  if (warp == 1) tmem_alloc(reinterpret_cast<uint32_t*>(&misc[0]), L::kTmemCols);
  if (warp >= 4) {
    // V and Q rings start zeroed: rows a partial tile never loads must be
    // finite (P is 0 there, and 0 * NaN would poison O).
    const int tid = threadIdx.x - 128;
    uint4 z = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < (VS * L::kTile) / 16; i += 256)
      reinterpret_cast<uint4*>(smem + L::kOffV)[i] = z;
    for (int i = tid; i < (QS * L::kQBytes) / 16; i += 256)
      reinterpret_cast<uint4*>(smem + L::kOffQ)[i] = z;
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = static_cast<uint32_t>(misc[0]);
  // everything below reads data earlier kernels in the stream may produce
  pdl_wait_primary();
  if (dts && threadIdx.x == 0) dts[1] = global_timer_ns();

  const uint32_t smem_k = smem_u32(smem + L::kOffK);
  const uint32_t smem_v = smem_u32(smem + L::kOffV);
  const uint32_t smem_q = smem_u32(smem + L::kOffQ);
  const uint32_t smem_p = smem_u32(smem + L::kOffP);
  const int g = a.sp.g;
  const int bpt = a.paged ? RB_KEY_TILE / a.block_size : 1;  // blocks per context tile

  Walker w;
  w.init(a, blockIdx.x);
  Tile t;

  if (warp == 0 || warp == 2) {
    // ------------------------------------------------ TMA producers (K+Q / V)
    const bool is_k = warp == 0;
    const uint64_t pol = l2_policy_evict_first();
    const uint64_t pol_q = l2_policy_evict_last();
    const CUtensorMap* sysmap = is_k ? &tm_sk : &tm_sv;
    const CUtensorMap* ctxmap = is_k ? &tm_ck : &tm_cv;
    const int NS = is_k ? KS : VS;
    uint64_t* full = is_k ? k_full : v_full;
    uint64_t* empty = is_k ? k_empty : v_empty;
    const uint32_t ring = is_k ? L::kOffK : L::kOffV;
    int j = 0, n = 0;
    bool first_tile = true;
    // Block ids of context tiles are staged kIdAhead tiles ahead with 4-byte
    // cp.async (one lane per block) so no block-table round trip sits on the
    // issue path: a walker copy runs ahead, one commit group per tile.
    int* ids = reinterpret_cast<int*>(smem + L::kOffIds) + (is_k ? 0 : L::kIdAhead * 32);
    Walker wa = w;
    Tile ta;
    auto stage_ids = [&](int slot) {
      if (wa.next(a, P, lens, qs, misc, meta_bar, ta) && ta.kind == 1 && a.paged) {
        const int nv = min(RB_KEY_TILE, lens[ta.r] - ta.kt * RB_KEY_TILE);
        if (lane < bpt && lane * a.block_size < nv)
          cp_async_4(ids + slot * 32 + lane, a.block_table +
                     static_cast<long long>(ta.r) * a.bt_stride + ta.kt * bpt + lane);
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int k = 0; k < L::kIdAhead; ++k) stage_ids(k);
    while (w.next(a, P, lens, qs, misc, meta_bar, t)) {
      if (!is_k && first_tile) {
        // K first at start-up: every SM fires its rings at once and the first
        // Q.K^T must not queue behind the V tiles.
        if (lane == 0) mbar_wait(v_go, 0);
        __syncwarp();
      }
      first_tile = false;
      if (dts && is_k && lane == 0 && j < 32) dts[360 + j] = global_timer_ns();
      // context block ids of this tile, one lane per block
      cp_async_wait_group<L::kIdAhead - 1>();
      if (dts && is_k && lane == 0 && j < 32) dts[392 + j] = global_timer_ns();
      int blk = 0, nvalid = 0;
      if (t.kind == 1) {
        nvalid = min(RB_KEY_TILE, lens[t.r] - t.kt * RB_KEY_TILE);  // keys of this tile that exist
        if (a.paged) blk = ids[(j % L::kIdAhead) * 32 + lane];
      }
      __syncwarp();
      stage_ids(j % L::kIdAhead);  // slot read above is refilled for tile j + kIdAhead
      if (dts && is_k && lane == 0 && j < 32) dts[424 + j] = global_timer_ns();
      if (is_k && t.first) {
        const int qsl = n % QS;
        if (lane == 0) {
          mbar_wait(&q_empty[qsl], ((n / QS) & 1) ^ 1);
          uint8_t* dst = smem + L::kOffQ + qsl * L::kQBytes;
          if (t.kind == 0) {
            const int h = t.u / a.sp.n_qt, qt = t.u % a.sp.n_qt;
            const int t0 = qt * NQ / g;
            mbar_arrive_expect_tx(&q_full[qsl], NQ * 256);
            tma_load_4d(dst, &tm_qs, &q_full[qsl], 0, 0, h, t0, pol_q);
            tma_load_4d(dst + NQ * 128, &tm_qs, &q_full[qsl], 64, 0, h, t0, pol_q);
          } else {
            const int t0 = qs[t.r] + t.z * NQ / g;
            mbar_arrive_expect_tx(&q_full[qsl], g * a.ctx_rows_box * 256);
            tma_load_4d(dst, &tm_qc, &q_full[qsl], 0, 0, t.h, t0, pol_q);
            tma_load_4d(dst + NQ * 128, &tm_qc, &q_full[qsl], 64, 0, t.h, t0, pol_q);
          }
        }
        ++n;
      }
      if (dts && is_k && lane == 0 && j < 32) dts[456 + j] = global_timer_ns();
      const int st = j % NS;
      if (dts && is_k && lane == 0 && j < 32) dts[168 + j] = global_timer_ns();
      if (lane == 0) mbar_wait(&empty[st], ((j / NS) & 1) ^ 1);
      if (dts && lane == 0 && j < 32) dts[(is_k ? 136 : 232) + j] = global_timer_ns();
      __syncwarp();
      uint8_t* dst = smem + ring + st * L::kTile;
      if (t.kind == 0) {
        if (lane == 0) {
          const int h = t.u / a.sp.n_qt;
          mbar_arrive_expect_tx(&full[st], L::kTile);
          tma_load_3d(dst, sysmap, &full[st], 0, t.kt * RB_KEY_TILE, h, pol);
          tma_load_3d(dst + L::kTile / 2, sysmap, &full[st], 64, t.kt * RB_KEY_TILE, h, pol);
        }
      } else if (a.paged) {
        const int nb = (nvalid + a.block_size - 1) / a.block_size;
        if (lane == 0) mbar_arrive_expect_tx(&full[st], nb * a.block_size * 256);
        __syncwarp();
        if (lane < nb) {
          const uint32_t off = lane * a.block_size * 128;
          tma_load_4d(dst + off, ctxmap, &full[st], 0, 0, t.h, blk, pol);
          tma_load_4d(dst + L::kTile / 2 + off, ctxmap, &full[st], 64, 0, t.h, blk, pol);
        }
      } else {
        if (lane == 0) {
          const int tok = static_cast<int>(a.req_offset[t.r]) + t.kt * RB_KEY_TILE;
          mbar_arrive_expect_tx(&full[st], L::kTile);
          tma_load_3d(dst, ctxmap, &full[st], 0, t.h, tok, pol);
          tma_load_3d(dst + L::kTile / 2, ctxmap, &full[st], 64, t.h, tok, pol);
        }
      }
      __syncwarp();
      ++j;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ S^T = K . Q^T
    int j = 0, n = 0;
    constexpr uint32_t idesc_qk = make_idesc_bf16_f32(128, NQ, 0, 0);
    while (w.next(a, P, lens, qs, misc, meta_bar, t)) {
      if (lane == 0) {
        const int qsl = n % QS;
        if (t.first) mbar_wait(&q_full[qsl], (n / QS) & 1);
        const int st = j % KS, sb = j & 1;
        mbar_wait(&k_full[st], (j / KS) & 1);
        if (j == 0) mbar_arrive(v_go);
        mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
        if (dts && j < 32) dts[264 + j] = global_timer_ns();
        tc_fence_after();
        const uint32_t k_base = smem_k + st * L::kTile;
        const uint32_t q_base = smem_q + qsl * L::kQBytes;
        const uint32_t d_tmem = tmem_base + sb * NQ;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk & 3) * 32;
          const uint64_t ad = make_smem_desc_sw128(k_base + (kk >> 2) * (L::kTile / 2) + koff, 16, 1024);
          const uint64_t bd = make_smem_desc_sw128(q_base + (kk >> 2) * (NQ * 128) + koff, 16, 1024);
          umma_f16_ss(d_tmem, ad, bd, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        umma_commit(&k_empty[st]);
        if (t.last) umma_commit(&q_empty[qsl]);
      }
      if (t.last) ++n;
      ++j;
    }
    __syncwarp();
  } else if (warp == 3) {
    // -------------------------------- metadata: context tile prefix + range
    if (a.has_ctx) {
      const int b = a.b;
      for (int i = lane; i <= b; i += 32) qs[i] = __ldg(a.q_start + i);
      const int per = (b + 31) / 32;
      const int lo = min(lane * per, b), hi = min(lo + per, b);
      __syncwarp();
      int sum = 0;
      for (int i = lo; i < hi; ++i) {
        const int c = __ldg(a.ctx_lens + i);
        lens[i] = c;
        sum += a.sp.hkv * ctx_nz(a, qs, i) * ((max(c, 0) + RB_KEY_TILE - 1) / RB_KEY_TILE);
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int run = incl - sum;
      for (int i = lo; i < hi; ++i) {
        P[i] = run;
        run += a.sp.hkv * ctx_nz(a, qs, i) * ((max(lens[i], 0) + RB_KEY_TILE - 1) / RB_KEY_TILE);
      }
      const int Tc = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 0) P[b] = Tc;
      __syncwarp();
      if (lane < 2) {
        // range boundary of CTA (blockIdx.x + lane), moved to a unit start
        const long long B = static_cast<long long>(blockIdx.x + lane) * Tc / gridDim.x;
        int res = Tc;
        if (B < Tc) {
          int l2 = 0, h2 = b - 1;
          while (l2 < h2) {
            const int mid = (l2 + h2 + 1) >> 1;
            if (P[mid] <= B) l2 = mid; else h2 = mid - 1;
          }
          const int tr = (lens[l2] + RB_KEY_TILE - 1) / RB_KEY_TILE;
          const int local = static_cast<int>(B) - P[l2];
          res = P[l2] + ((local + tr - 1) / tr) * tr;
        }
        misc[2 + lane] = res;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(meta_bar);
    }
    // ------------------------------------------------ O^T += V^T . P^T
    int j = 0, n = 0;
    constexpr uint32_t idesc_pv = make_idesc_bf16_f32(128, NQ, 1, 0);
    while (w.next(a, P, lens, qs, misc, meta_bar, t)) {
      if (lane == 0) {
        const int st = j % VS, pb = j & 1, ob = n & 1;
        mbar_wait(&v_full[st], (j / VS) & 1);
        mbar_wait(&p_full[pb], (j >> 1) & 1);
        if (t.first) mbar_wait(&o_free[ob], ((n >> 1) & 1) ^ 1);
        if (dts && j < 32) dts[296 + j] = global_timer_ns();
        tc_fence_after();
        const uint32_t v_base = smem_v + st * L::kTile;
        const uint32_t p_base = smem_p + pb * L::kQBytes;
        const uint32_t d_tmem = tmem_base + 2 * NQ + ob * NQ;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = make_smem_desc_sw128(v_base + kk * 2048, L::kTile / 2, 1024);
          const uint64_t bd =
              make_smem_desc_sw128(p_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
          umma_f16_ss(d_tmem, ad, bd, idesc_pv, (t.first && kk == 0) ? 0u : 1u);
        }
        umma_commit(&p_empty[pb]);
        umma_commit(&v_empty[st]);
        if (t.last) umma_commit(&o_full[ob]);
      }
      if (t.last) ++n;
      ++j;
    }
    __syncwarp();
  } else if (warp < 8) {
    // --------------------------------------------------------- softmax
    SmxCtx C;
    C.qd = warp & 3;                          // TMEM lane quadrant
    C.lane = lane;
    const int kl = C.qd * 32 + lane;          // key lane of the tile
    C.red = red;
    C.red2 = red2;
    C.my_mu = mu + C.qd * NQ;
    C.my_al = al + C.qd * NQ;
    C.hand = hand;
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) C.poff[r8] = sw128_offset(r8, kl & 63);
    C.pbase = smem + L::kOffP + (kl >> 6) * (NQ * 128);
    C.lane_addr = tmem_base + (static_cast<uint32_t>(C.qd * 32) << 16);
    float l_part[NQ], mr[NQ];
    int j = 0, n = 0, small = 0;
    while (w.next(a, P, lens, qs, misc, meta_bar, t)) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      if (dts && threadIdx.x == 128) {
        if (j == 0) dts[2] = global_timer_ns();
        if (j < 32) dts[8 + j] = global_timer_ns();
      }
      tc_fence_after();
      const int key = t.kt * RB_KEY_TILE + kl;
      if (t.kind == 0) {
        float x[NQ];
        tmem_ld_32x32b<NQ>(C.lane_addr + sb * NQ, x);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        const bool valid = key < a.sp.s;
#pragma unroll
        for (int c = 0; c < NQ; ++c) x[c] = valid ? x[c] * a.scale_log2 : -INFINITY;
        softmax_tile<NQ, NQ>(C, x, mr, l_part, t.first, j, n, p_empty, p_full, L::kQBytes);
        if (t.last) softmax_part_end<NQ, NQ>(C, l_part, n, h_empty, h_full);
      } else {
        // column c (local row li = z*NQ + c, query t = li / g) sees key iff
        // key < c_r - m_r + t + 1 (attention.py:120-121), i.e. c >= cmin, and
        // c < cmax (the unit's rows): two compares per column, no division.
        const int m_r = qs[t.r + 1] - qs[t.r];
        const int cmax = m_r * g - t.z * NQ;
        const int cmin = (key - (lens[t.r] - m_r)) * g - t.z * NQ;
        if (t.first) small = cmax <= 8;
        if (small) {
          float x[8];
          tmem_ld_32x32b<8>(C.lane_addr + sb * NQ, x);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[sb]);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            x[c] = (c >= cmin && c < cmax) ? x[c] * a.scale_log2 : -INFINITY;
          softmax_tile<8, NQ>(C, x, mr, l_part, t.first, j, n, p_empty, p_full, L::kQBytes);
          if (t.last) softmax_part_end<8, NQ>(C, l_part, n, h_empty, h_full);
        } else {
          float x[NQ];
          tmem_ld_32x32b<NQ>(C.lane_addr + sb * NQ, x);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[sb]);
#pragma unroll
          for (int c = 0; c < NQ; ++c)
            x[c] = (c >= cmin && c < cmax) ? x[c] * a.scale_log2 : -INFINITY;
          softmax_tile<NQ, NQ>(C, x, mr, l_part, t.first, j, n, p_empty, p_full, L::kQBytes);
          if (t.last) softmax_part_end<NQ, NQ>(C, l_part, n, h_empty, h_full);
        }
      }
      if (dts && threadIdx.x == 128 && j < 32) dts[328 + j] = global_timer_ns();
      if (t.last) ++n;
      ++j;
    }
    if (dts && threadIdx.x == 128) dts[3] = global_timer_ns();
  } else {
    // -------------------------------------------------------- epilogue
    const int tid = threadIdx.x - 256;      // 0..127
    const int qd = warp & 3;
    const int d = qd * 32 + lane;           // TMEM lane = head dim
    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(qd * 32) << 16);
    // group bookkeeping reads the request metadata even for system parts
    if (a.has_ctx) mbar_wait(meta_bar, 0);
    int n = 0;
    while (w.next(a, P, lens, qs, misc, meta_bar, t)) {
      if (!t.last) continue;
      const int ob = n & 1;
      mbar_wait(&h_full[ob], (n >> 1) & 1);
      mbar_wait(&o_full[ob], (n >> 1) & 1);
      if (dts && tid == 0 && n < 32) dts[40 + n] = global_timer_ns();
      tc_fence_after();
      float o[H];
      tmem_ld_32x32b<H>(lane_addr + 2 * NQ + ob * NQ, o);
      tmem_wait_ld();
      if (dts && tid == 0 && n < 32) {
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < H; ++c) acc += o[c];
        dts[72 + n] = global_timer_ns() + (acc == 1.2345f ? 1 : 0);
      }
      const float* hm = hand + ob * 2 * NQ;  // this part's (m, l), freed after the writes
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[ob]);
      if (dts && tid == 0 && n < 32) dts[200 + n] = global_timer_ns();
      // ---- write this part's partial state
      const rb_sys_plan& p = a.sp;
      if (t.kind == 0) {
        const int owner0 = rb_tile_owner(&p, static_cast<long long>(t.u) * p.tpu);
        const long long pb = static_cast<long long>(t.u) * p.max_parts + (blockIdx.x - owner0);
        float* pacc = a.sys_acc + pb * NQ * RB_HEAD_DIM;
#pragma unroll
        for (int c = 0; c < H; ++c) pacc[c * RB_HEAD_DIM + d] = o[c];
        if (tid < NQ) {
          a.sys_ml[pb * 2 * NQ + tid] = hm[tid];
          a.sys_ml[pb * 2 * NQ + NQ + tid] = hm[NQ + tid];
        }
      } else {
        // valid columns c < ncol: local row li = z*NQ + c -> query row
        // qs[r] + li / g, head h*g + li % g.  Runtime loop (compact code: this
        // runs once per context unit and must stay i-cache resident).
        const int ncol = min((qs[t.r + 1] - qs[t.r]) * g - t.z * NQ, NQ);
        for (int c = 0; c < ncol; ++c) {
          float val = o[0];
#pragma unroll
          for (int cc = 1; cc < H; ++cc) val = (cc == c) ? o[cc] : val;
          const int li = t.z * NQ + c;
          const long long oi = static_cast<long long>(qs[t.r] + li / g) * p.hq + t.h * g + li % g;
          a.ctx_acc[oi * RB_HEAD_DIM + d] = val;
          if (d == 0) reinterpret_cast<float2*>(a.ctx_ml)[oi] = make_float2(hm[c], hm[NQ + c]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&h_empty[ob]);
      if (dts && tid == 0 && n < 32) dts[104 + n] = global_timer_ns();
      ++n;
    }
    if (dts && threadIdx.x == 256) dts[4] = global_timer_ns();
  }

  if (warp >= 4) {
    // ---- every part of every CTA written: grid barrier, then each CTA merges
    // its share of the output vectors (8 warps, one vector per warp)
    named_bar_sync(3, 256);
    if (threadIdx.x == 256) {
      grid_barrier(reinterpret_cast<unsigned int*>(a.counters), gridDim.x);
      if (dts) dts[6] = global_timer_ns();
    }
    named_bar_sync(3, 256);
    // all CTAs are resident now: the next kernel in the stream may launch
    // (never earlier: a dependent grid holding SMs could starve the barrier)
    pdl_launch_dependents();
    const long long V = static_cast<long long>(a.sp.n_rows) * a.sp.hq;
    const long long vb = V * blockIdx.x / gridDim.x, ve = V * (blockIdx.x + 1) / gridDim.x;
    for (long long v = vb + (warp - 4); v < ve; v += 8) merge_vector<NQ>(a, qs, lens, v, lane);
  }
  if (dts && threadIdx.x == 0) dts[5] = global_timer_ns();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, L::kTmemCols);
  }
  if (dts && threadIdx.x == 0) dts[7] = global_timer_ns();
}

// ------------------------------------------------------------------- host

template <int NQ>
static cudaError_t launch_step(const CUtensorMap* maps, const StepArgs& a, int grid,
                               cudaStream_t stream) {
  using L = StepCfg<NQ>;
  const int smem = L::smem_bytes(a.b);
  if (smem > 232448) return cudaErrorInvalidValue;
  auto kern = relay_step_kernel<NQ>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, dim3(grid), dim3(L::kThreads), smem, stream, maps[0], maps[1], maps[2],
                 maps[3], maps[4], maps[5], a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int relay_step_max_b(int nq) {
  const int base = nq == 16 ? StepCfg<16>::smem_bytes(0) : StepCfg<32>::smem_bytes(0);
  return (232448 - base) / 12;
}

cudaError_t launch_relay_step(const CUtensorMap* maps, const StepArgs& a, int grid,
                              cudaStream_t stream) {
  switch (a.sp.nq) {
    case 16: return launch_step<16>(maps, a, grid, stream);
    case 32: return launch_step<32>(maps, a, grid, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rb
