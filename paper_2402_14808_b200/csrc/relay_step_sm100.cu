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
//    Operands arrive by TMA (3-D map of the prefix, 4-D map of the queries
//    that picks a KV head's GQA group) or, for paged context, ONE 4 KB bulk
//    copy per (block, kv head): PagedKvCache stores each block as the
//    [128 d][bs] swizzled UMMA operand (K MN-major, V^T K-major).
//  * Two softmax groups (4 warps each, thread = key lane, NQ columns per
//    thread, log2 domain) take alternate tiles, so one group's tile latency
//    overlaps the other's.  Lazy rescaling: a column's reference max only
//    moves when a tile exceeds it by more than kTau (P <= 2^kTau), so O is
//    accumulated by the tensor core in the group's TMEM buffer across the
//    whole part and rescaled only on those rare moves; row sums stay per lane
//    until the group's last tile of the part, when the group drains O from
//    TMEM and writes its partial (acc, m, l).  No per-part synchronisation
//    with other CTAs.
//  * When every part of every CTA is written, a grid barrier (one CTA per SM,
//    all resident), then every CTA merges its share of the output vectors:
//    context partials + system stream-K parts = the relay fusion.  Partials
//    live in L2 (a few MB); they never take an HBM round trip of their own.
//  * Warp roles (12 warps): 0 K/Q producer, 1 QK^T issuer (TMEM owner),
//    2 V producer, 3 metadata scan then P.V issuer, 4-7 softmax group 0,
//    8-11 softmax group 1.
#include "rb_common.cuh"
#include "rb_plan.h"
#include "rb_args.cuh"

namespace rb {

constexpr float kTau = 8.0f;         // lazy-rescale threshold (log2 units)
constexpr float kNegBig = -1.0e30f;  // "no key yet" reference max (exp2(-inf - kNegBig) = 0)

// Per-tile %globaltimer trace -- compiled in only with -DRB_STEP_TRACE=1: the
// stamps cost instruction-cache footprint.
#ifndef RB_STEP_TRACE
#define RB_STEP_TRACE 0
#endif
#if RB_STEP_TRACE
#define RB_TRACE(cond, idx) \
  do {                      \
    if (dts && (cond)) dts[idx] = global_timer_ns(); \
  } while (0)
#else
#define RB_TRACE(cond, idx) \
  do {                      \
  } while (0)
#endif

template <int NQ>
struct StepCfg {
  static constexpr int KS = 2, VS = 3, QS = 4;
  static constexpr int kTile = RB_KEY_TILE * RB_HEAD_DIM * 2;  // 32 KB K or V tile
  static constexpr int kQBytes = NQ * 256;                     // [2 kblocks][NQ][128 B]
  static constexpr int kThreads = 13 * 32;  // 12 pipeline warps + the scheduler
  static constexpr int IQ = 8;                // work-item ring depth
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + KS * kTile;
  static constexpr int kOffQ = kOffV + VS * kTile;
  static constexpr int kOffP = kOffQ + QS * kQBytes;            // [2 groups] P tiles
  static constexpr int kOffRed = kOffP + 2 * kQBytes;           // float [2 grp][2][4][NQ] tile max
  static constexpr int kOffRed2 = kOffRed + 2 * 2 * 4 * NQ * 4;  // float [2 grp][4][NQ] row sums
  static constexpr int kOffMu = kOffRed2 + 2 * 4 * NQ * 4;       // float [8 warps][NQ] reference max
  static constexpr int kOffAl = kOffMu + 8 * NQ * 4;             // float [8 warps][NQ] rescale
  static constexpr int kOffMisc = kOffAl + 8 * NQ * 4;           // int [16]
  static constexpr int kOffItems = kOffMisc + 64;                // int [IQ] work-item ring
  static constexpr int kIdAhead = 4;                             // block-id lookahead (tiles)
  static constexpr int kOffIds = kOffItems + 64;                 // int [2 producers][kIdAhead][32]
  static constexpr int kOffBar = kOffIds + 2 * kIdAhead * 32 * 4;
  static constexpr int kNumBars = 2 * KS + 2 * VS + 2 * QS + 2 * IQ + 14;  // rings + s,p,o + meta + v_go
  static constexpr int kOffMeta = kOffBar + kNumBars * 8;  // int U[b+1], lens[b], qs[b+1]
  // TMEM per group: S and O accumulators of NQ columns each
  static constexpr int kTmemCols = (4 * NQ <= 32) ? 32 : (4 * NQ <= 64) ? 64 : 128;
  static int smem_bytes(int b) { return kOffMeta + 4 * (3 * b + 2) + 16; }
};

// One tile of this CTA's work sequence.
struct Tile {
  int kind;         // 0 = system, 1 = context
  int u;            // system unit
  int r, h, z;      // context unit
  int kt;           // key tile inside the unit (context tiles: inside the context)
  int pre;          // naive mode: this context-unit tile re-reads the shared prefix
  int first, last;  // first / last tile of this CTA's part of the unit
  int pidx, rem;    // index of the tile in the part / tiles left in the part (incl. this)
};

// Query tiles of request r's context units: ceil(m_r * g / NQ).
__device__ __forceinline__ int ctx_nz(const StepArgs& a, const int* qs, int r) {
  const int lg = __ffs(a.sp.nq) - 1;  // nq is 16 or 32
  return ((qs[r + 1] - qs[r]) * a.sp.g + a.sp.nq - 1) >> lg;
}

// Tiles of one context unit of a request with c_r context keys.
__device__ __forceinline__ int ctx_unit_tiles(const StepArgs& a, int c_r) {
  return a.prefix_tiles + (max(c_r, 0) + RB_KEY_TILE - 1) / RB_KEY_TILE;
}

// Work items of a CTA: first its static stream-K share of the system tiles
// (item u = the part of system unit u inside the CTA's tile range, rb_plan.h),
// then context units handed out dynamically (item n_units + v = context unit
// v in (request, kv head, q-tile) order, decoded through the per-request unit
// prefix U).  The scheduler warp publishes item ids in a ring every role reads
// in the same order; a CTA whose system share ran fast simply takes more of
// the small context units, so the step ends without a tail imbalance.

// Walks this CTA's items tile by tile.  Every role warp (all lanes) runs its
// own copy; lane 0 frees a ring slot once the warp has read it.
template <int IQ>
struct Walker {
  int qi;              // items read from the ring
  int kind;            // current item: -1 none, 0 system part, 1 context unit
  int item;            // its id
  int u, kb, ke;       // system part: unit, key tile range [kb, ke)
  int r, h, z, tr;     // context unit: request, kv head, q-tile, tiles
  int kt;              // cursor inside the item
  long long xb, xe;    // this CTA's system tile range (stream-K)
  __device__ __forceinline__ void init(const StepArgs& a, int cta) {
    qi = 0;
    kind = -1;
    kt = ke = tr = 0;
    xb = xe = 0;
    if (a.has_sys && cta < a.sp.grid) {
      xb = rb_cta_begin(&a.sp, cta);
      xe = rb_cta_begin(&a.sp, cta + 1);
    }
  }
  __device__ __forceinline__ bool next(const StepArgs& a, const int* U, const int* lens,
                                       const int* qs, const int* itq, uint64_t* itq_full,
                                       uint64_t* itq_empty, int lane, Tile& t) {
    if (kind < 0 || (kind == 0 && kt >= ke) || (kind == 1 && kt >= tr)) {
      const int slot = qi % IQ;
      mbar_wait(&itq_full[slot], (qi / IQ) & 1);
      item = itq[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&itq_empty[slot]);
      ++qi;
      const int n_sc = a.has_sys ? a.sp.n_units : 0;
      if (item < n_sc) {
        const long long ub = static_cast<long long>(item) * a.sp.tpu;
        kind = 0;
        u = item;
        kb = static_cast<int>((xb > ub ? xb : ub) - ub);
        ke = static_cast<int>((xe < ub + a.sp.tpu ? xe : ub + a.sp.tpu) - ub);
        kt = kb;
      } else if (a.has_ctx && item - n_sc < U[a.b]) {
        const int v = item - n_sc;
        int lo = 0, hi = a.b - 1;  // request r: U[r] <= v < U[r+1]
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (U[mid] <= v) lo = mid; else hi = mid - 1;
        }
        r = lo;
        const int nz = ctx_nz(a, qs, r);
        h = (v - U[r]) / nz;
        z = (v - U[r]) % nz;
        tr = ctx_unit_tiles(a, lens[r]);
        kind = 1;
        kt = 0;
      } else {
        kind = 2;  // sentinel: no more work
        kt = ke = tr = 0;
        return false;
      }
    }
    t.kind = kind;
    if (kind == 0) {
      t.u = u;
      t.kt = kt;
      t.pidx = kt - kb;
      t.rem = ke - kt;
      t.r = t.h = t.z = 0;
      t.pre = 0;
    } else {
      t.u = 0;
      t.r = r;
      t.h = h;
      t.z = z;
      t.pre = kt < a.prefix_tiles;
      t.kt = t.pre ? kt : kt - a.prefix_tiles;
      t.pidx = kt;
      t.rem = tr - kt;
    }
    t.first = t.pidx == 0;
    t.last = t.rem == 1;
    ++kt;
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

// Per-thread context of a softmax group.
struct SmxCtx {
  float* red;       // [2][4][NQ] this group's tile maxima per quadrant
  float* red2;      // [4][NQ] this group's row sums
  float* my_mu;     // [NQ] this warp's copy of the reference max per column
  float* my_al;     // [NQ] this warp's copy of the rescale factors
  uint8_t* pbase;   // this group's P tile, this thread's key half
  uint32_t poff[8];
  uint32_t s_addr;  // TMEM: this group's S buffer, this warp's lane quadrant
  uint32_t o_addr;  // TMEM: this group's O buffer, this warp's lane quadrant
  uint32_t bar;     // named barrier of the group (128 threads)
  int qd, lane;
};

// Mask of one tile: column c of the tile sees this thread's key iff
// cmin <= c < cmax (system / prefix tiles: cmin = -1 or NQ by key < s).
struct TileMask {
  int cmin, cmax;
};

// Chunk of 8 score columns [c0, c0+8) of this thread's key lane: TMEM -> masked,
// log2-scaled registers.
__device__ __forceinline__ void load_scores8(uint32_t s_addr, int c0, const TileMask& mk,
                                             float scale, float (&y)[8]) {
  float x[8];
  tmem_ld_32x32b<8>(s_addr + c0, x);
  tmem_wait_ld();
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int c = c0 + e;
    y[e] = (c >= mk.cmin && c < mk.cmax) ? x[e] * scale : -INFINITY;
  }
}

// Rare path of a tile: per-column tile max over the group's 128 key
// lanes, move the reference max of every column that grew by more than kTau,
// and rescale that column's O accumulator in TMEM; returns whether the row
// sums must be rescaled too (factors in my_al).
__device__ __forceinline__ bool softmax_rare(const SmxCtx& C, int ncol, int NQ, bool first,
                                             const TileMask& mk, float scale, int k,
                                             uint64_t* p_empty) {
  float* rb = C.red + (k & 1) * 4 * NQ;
#pragma unroll 1
  for (int c0 = 0; c0 < ncol; c0 += 8) {
    float y[8];
    load_scores8(C.s_addr, c0, mk, scale, y);
    const float wmax = warp_reduce_cols<8, true>(y, C.lane);  // lane l: column c0 + l / 4
    if (reduced_writer<8>(C.lane)) rb[C.qd * NQ + c0 + reduced_col<8>(C.lane)] = wmax;
  }
  named_bar_sync(C.bar, 128);
  bool from_finite = false;
  __syncwarp();
  if (C.lane < ncol) {
    const int c = C.lane;
    const float tm = fmaxf(fmaxf(rb[c], rb[NQ + c]), fmaxf(rb[2 * NQ + c], rb[3 * NQ + c]));
    const float mold = C.my_mu[c];
    const bool mv = tm > mold + kTau;
    C.my_al[c] = mv ? fast_exp2(mold - tm) : 1.f;  // 0 when mold is kNegBig
    if (mv) C.my_mu[c] = tm;
    from_finite = mv && mold > 0.5f * kNegBig;
  }
  const bool need_o = __any_sync(0xffffffffu, from_finite) && !first;
  __syncwarp();
  if (need_o) {
    // rescale O (after this group's previous P.V landed)
    mbar_wait(p_empty, ((k - 1) & 1));
    tc_fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < ncol; c0 += 8) {
      float o[8];
      tmem_ld_32x32b<8>(C.o_addr + c0, o);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] *= C.my_al[c0 + e];
      tmem_st_32x32b<8>(C.o_addr + c0, o);
    }
    tmem_wait_st();
    tc_fence_before();
  }
  return need_o;
}

// One tile of a softmax group over `ncol` (8 or NQ) live columns, processed
// in chunks of 8 read straight from TMEM (the loop bodies must stay small:
// the instruction cache is shared by two softmax warps and a role warp per
// SMSP, and a miss goes to L2 behind the TMA stream):
//   pass 1: does any score exceed its column's reference max by > kTau?
//           (one OR-barrier over the group; the rare path moves the maxima)
//   pass 2: P = 2^(y - m) (bf16) into the K-major SW128 [NQ][128 keys] tile,
//           fp32 row sums per key lane in l_part (reduced at the part end).
template <int NQ>
__device__ __forceinline__ void softmax_tile(const SmxCtx& C, float (&l_part)[NQ], int ncol,
                                             bool first, int k, const TileMask& mk, float scale,
                                             uint64_t* s_empty, uint64_t* p_empty,
                                             uint64_t* p_full, unsigned long long* dts, int j) {
  if (first) {
    __syncwarp();
    if (C.lane < NQ) C.my_mu[C.lane] = kNegBig;
    __syncwarp();
#pragma unroll
    for (int c = 0; c < NQ; ++c) l_part[c] = 0.f;
  }
  bool ex = false;
#pragma unroll 1
  for (int c0 = 0; c0 < ncol; c0 += 8) {
    float y[8];
    load_scores8(C.s_addr, c0, mk, scale, y);
    const float4 m0 = *reinterpret_cast<const float4*>(C.my_mu + c0);
    const float4 m1 = *reinterpret_cast<const float4*>(C.my_mu + c0 + 4);
    ex |= (y[0] > m0.x + kTau) | (y[1] > m0.y + kTau) | (y[2] > m0.z + kTau) |
          (y[3] > m0.w + kTau) | (y[4] > m1.x + kTau) | (y[5] > m1.y + kTau) |
          (y[6] > m1.z + kTau) | (y[7] > m1.w + kTau);
  }
  RB_TRACE((threadIdx.x == 128 && j < 32), 360 + j);
  const bool any_ex = bar_red_or(C.bar, 128, ex);
  RB_TRACE((threadIdx.x == 128 && j < 32), 392 + j);
  if (any_ex) {
    const bool resc = softmax_rare(C, ncol, NQ, first, mk, scale, k, p_empty);
    if (resc) {
#pragma unroll
      for (int c = 0; c < NQ; ++c) l_part[c] *= C.my_al[c];
    }
  }
  RB_TRACE((threadIdx.x == 128 && j < 32), 424 + j);
  mbar_wait(p_empty, (k & 1) ^ 1);  // this group's previous P.V has read P
  RB_TRACE((threadIdx.x == 128 && j < 32), 456 + j);
#pragma unroll
  for (int c0 = 0; c0 < NQ; c0 += 8) {
    if (c0 < ncol) {
      float y[8];
      load_scores8(C.s_addr, c0, mk, scale, y);
      const float4 m0 = *reinterpret_cast<const float4*>(C.my_mu + c0);
      const float4 m1 = *reinterpret_cast<const float4*>(C.my_mu + c0 + 4);
      const float m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
      uint8_t* row = C.pbase + (c0 >> 3) * 1024;  // 8 P rows = one SW128 atom
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float pv = fast_exp2(y[e] - m[e]);
        l_part[c0 + e] += pv;
        *reinterpret_cast<__nv_bfloat16*>(row + C.poff[e]) = __float2bfloat16_rn(pv);
      }
    }
  }
  tc_fence_before();
  fence_proxy_async_smem();
  __syncwarp();
  if (C.lane == 0) {
    mbar_arrive(s_empty);  // S fully read
    mbar_arrive(p_full);
  }
}

// The group's last tile of a part: row sums over the 128 key lanes (lane c of
// quadrant 0 ends up with column c), drain O from TMEM (thread = head dim) and
// write the group's partial (acc, m, l).  sys parts: slot (CTA - first owner)
// * 2 + group of unit u; context units: ctx partial set `grp` of each of the
// unit's query rows.  A part with one tile in this CTA also marks the other
// group's slot empty (m = kNegBig).
template <int NQ>
__device__ __forceinline__ void softmax_part_end(const SmxCtx& C, const StepArgs& a, const Tile& t,
                                                 const int* qs, const float (&l_part)[NQ],
                                                 int ncol, int grp, int kp, uint64_t* o_full,
                                                 uint64_t* o_free, unsigned long long* dts, int j) {
  // row sums: per chunk of 8 columns a warp reduce-scatter, then the 4
  // quadrants through smem
#pragma unroll
  for (int c0 = 0; c0 < NQ; c0 += 8) {
    if (c0 < ncol) {
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = l_part[c0 + e];
      const float ws = warp_reduce_cols<8, false>(v, C.lane);
      if (reduced_writer<8>(C.lane)) C.red2[C.qd * NQ + c0 + reduced_col<8>(C.lane)] = ws;
    }
  }
  RB_TRACE((threadIdx.x == 128 && j < 32), 136 + j);
  named_bar_sync(C.bar, 128);
  RB_TRACE((threadIdx.x == 128 && j < 32), 168 + j);
  const int d = C.qd * 32 + C.lane;  // TMEM lane of O = head dim
  mbar_wait(o_full, kp & 1);
  RB_TRACE((threadIdx.x == 128 && j < 32), 200 + j);
  tc_fence_after();
  const rb_sys_plan& p = a.sp;
  const bool single = t.pidx == 0 && t.rem == 1;
  long long s0 = 0;
  const long long nv = static_cast<long long>(p.n_rows) * p.hq;
  const int g = p.g;
  int nrow = ncol;  // columns with a real query row
  // the group's tiles of a part are those with pidx of this parity: its
  // partial goes to slot `half`, whichever group (and CTA) processed it, so
  // the merge order is independent of the dynamic schedule (deterministic)
  const int half = t.pidx & 1;
  if (t.kind == 0) {
    const int owner0 = rb_tile_owner(&p, static_cast<long long>(t.u) * p.tpu);
    s0 = static_cast<long long>(t.u) * 2 * p.max_parts + 2 * (blockIdx.x - owner0);
  } else {
    nrow = min((qs[t.r + 1] - qs[t.r]) * g - t.z * NQ, ncol);
  }
#pragma unroll 1
  for (int c0 = 0; c0 < ncol; c0 += 8) {
    float o[8];
    tmem_ld_32x32b<8>(C.o_addr + c0, o);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = c0 + e;
      const float lsum = C.red2[c] + C.red2[NQ + c] + C.red2[2 * NQ + c] + C.red2[3 * NQ + c];
      if (t.kind == 0) {
        const long long pb = s0 + half;
        a.sys_acc[(pb * NQ + c) * RB_HEAD_DIM + d] = o[e];
        if (d == 0) {
          a.sys_ml[pb * 2 * NQ + c] = C.my_mu[c];
          a.sys_ml[pb * 2 * NQ + NQ + c] = lsum;
          if (single) a.sys_ml[(s0 + 1) * 2 * NQ + c] = kNegBig;
        }
      } else if (c < nrow) {
        // local row li = z*NQ + c -> query row qs[r] + li / g, head h*g + li % g
        const int li = t.z * NQ + c;
        const long long oi = static_cast<long long>(qs[t.r] + li / g) * p.hq + t.h * g + li % g;
        a.ctx_acc[(half * nv + oi) * RB_HEAD_DIM + d] = o[e];
        if (d == 0) {
          reinterpret_cast<float2*>(a.ctx_ml)[half * nv + oi] = make_float2(C.my_mu[c], lsum);
          if (single) reinterpret_cast<float2*>(a.ctx_ml)[nv + oi] = make_float2(kNegBig, 0.f);
        }
      }
    }
  }
  tc_fence_before();
  __syncwarp();
  if (C.lane == 0) mbar_arrive(o_free);
}

// Final merge, after the grid barrier: output vector (row t, query head hh)
// = LSE-weighted combine of its two context partials (if the request has a
// context) and the system stream-K slots of its group u = (hh / g, f / NQ),
// in a fixed order (context, then slots): the relay fusion of
// attention.py:137-157 with max-subtracted weights.  One warp per vector
// (4 head dims per lane); all loads of a vector are issued in one round (up
// to kMergeSlots system slots in registers, more in a second loop).  Empty
// partials (m = kNegBig) are skipped.
constexpr int kMergeSlots = 8;

template <int NQ>
__device__ __forceinline__ void merge_vector(const StepArgs& a, const int* qs, const int* lens,
                                             long long v, int lane) {
  const rb_sys_plan& p = a.sp;
  const int t = static_cast<int>(v / p.hq), hh = static_cast<int>(v % p.hq);
  const int h = hh / p.g, j = hh % p.g;
  const int f = t * p.g + j;
  const int u = h * p.n_qt + f / NQ, col = f % NQ;
  const int ns = a.has_sys ? 2 * rb_unit_parts(&p, u) : 0;
  bool hasc = false;
  if (a.has_ctx) {
    int lo = 0, hi = a.b - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (qs[mid] <= t) lo = mid; else hi = mid - 1;
    }
    hasc = lens[lo] > 0;
  }
  const long long nv = static_cast<long long>(p.n_rows) * p.hq;
  const long long ubase = static_cast<long long>(u) * 2 * p.max_parts;
  // ---- one round of loads (lane = 4 head dims)
  float2 mlc[2];
  float4 xc[2];
#pragma unroll
  for (int gg = 0; gg < 2; ++gg) {
    mlc[gg] = make_float2(kNegBig, 0.f);
    xc[gg] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (hasc) {
      mlc[gg] = __ldcg(reinterpret_cast<const float2*>(a.ctx_ml) + gg * nv + v);
      xc[gg] = __ldcg(reinterpret_cast<const float4*>(a.ctx_acc + (gg * nv + v) * RB_HEAD_DIM) + lane);
    }
  }
  float ms[kMergeSlots], ls[kMergeSlots];
  float4 xs[kMergeSlots];
#pragma unroll
  for (int k = 0; k < kMergeSlots; ++k) {
    ms[k] = kNegBig;
    ls[k] = 0.f;
    xs[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < ns) {
      const float* ml = a.sys_ml + (ubase + k) * 2 * NQ;
      ms[k] = __ldcg(ml + col);
      ls[k] = __ldcg(ml + NQ + col);
      xs[k] = __ldcg(reinterpret_cast<const float4*>(
                         a.sys_acc + ((ubase + k) * NQ + col) * RB_HEAD_DIM) + lane);
    }
  }
  float M = fmaxf(mlc[0].x, mlc[1].x);
#pragma unroll
  for (int k = 0; k < kMergeSlots; ++k) M = fmaxf(M, ms[k]);
  for (int k = kMergeSlots; k < ns; ++k) M = fmaxf(M, __ldcg(a.sys_ml + (ubase + k) * 2 * NQ + col));
  // ---- weighted sums in fixed order (context, then slots)
  float L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  auto add = [&](float m, float l, const float4& x) {
    if (m > 0.5f * kNegBig) {
      const float w = fast_exp2(m - M);
      L += l * w;
      O.x += x.x * w; O.y += x.y * w; O.z += x.z * w; O.w += x.w * w;
    }
  };
#pragma unroll
  for (int gg = 0; gg < 2; ++gg) add(mlc[gg].x, mlc[gg].y, xc[gg]);
#pragma unroll
  for (int k = 0; k < kMergeSlots; ++k) add(ms[k], ls[k], xs[k]);
  for (int k = kMergeSlots; k < ns; ++k) {
    const float* ml = a.sys_ml + (ubase + k) * 2 * NQ;
    add(__ldcg(ml + col), __ldcg(ml + NQ + col),
        __ldcg(reinterpret_cast<const float4*>(a.sys_acc + ((ubase + k) * NQ + col) * RB_HEAD_DIM) +
               lane));
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
// one CTA per SM).  bar[0] = arrivals, bar[1] = generation; the last arriver
// also re-arms the scheduler's item counters bar[2], bar[3].
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nctas) {
  unsigned int gen;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
  fence_acq_rel_gpu();  // release this CTA's partials (cumulative over the CTA barrier)
  const unsigned int prev = atomicAdd(bar, 1u);
  if (prev == nctas - 1) {
    bar[0] = 0;
    bar[2] = 0;  // work-item counters of the scheduler: every CTA is done grabbing
    bar[3] = 0;
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
                      const __grid_constant__ CUtensorMap tm_rk,
                      const __grid_constant__ CUtensorMap tm_rv, const StepArgs a) {
  using L = StepCfg<NQ>;
  constexpr int KS = L::KS, VS = L::VS, QS = L::QS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;
  uint64_t* v_empty = v_full + VS;
  uint64_t* q_full = v_empty + VS;
  uint64_t* q_empty = q_full + QS;
  uint64_t* s_full = q_empty + QS;   // [group]
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 2;
  uint64_t* o_full = p_empty + 2;
  uint64_t* o_free = o_full + 2;
  uint64_t* meta_bar = o_free + 2;
  uint64_t* v_go = meta_bar + 1;     // first K tile landed: V streaming may start
  uint64_t* itq_full = v_go + 1;     // work-item ring
  uint64_t* itq_empty = itq_full + L::IQ;
  static_assert(2 * KS + 2 * VS + 2 * QS + 2 * L::IQ + 14 == L::kNumBars, "barrier count");
  // readers of every ring slot: K and V producers (main + lookahead walkers),
  // QK and PV issuers, the 8 softmax warps
  constexpr int kItemReaders = 14;
  int* misc = reinterpret_cast<int*>(smem + L::kOffMisc);
  int* itq = reinterpret_cast<int*>(smem + L::kOffItems);
  int* U = reinterpret_cast<int*>(smem + L::kOffMeta);  // context units before request r
  int* lens = U + (a.b + 1);
  int* qs = lens + a.b;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* dts = a.debug_ts ? a.debug_ts + blockIdx.x * 512 : nullptr;
  if (dts && threadIdx.x == 0) {
    dts[0] = global_timer_ns();
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    dts[480] = smid;
  }

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
    }
    mbar_init(meta_bar, 1);
    mbar_init(v_go, 1);
    for (int i = 0; i < L::IQ; ++i) {
      mbar_init(&itq_full[i], 1);
      mbar_init(&itq_empty[i], kItemReaders);
    }
    fence_mbar_init();
  } else if (warp == 0 && lane == 1) {
    tma_prefetch_desc(&tm_qs);
    tma_prefetch_desc(&tm_sk);
    tma_prefetch_desc(&tm_sv);
  } else if (warp == 2 && lane == 1) {
    tma_prefetch_desc(&tm_qc);
    tma_prefetch_desc(&tm_rk);
    tma_prefetch_desc(&tm_rv);
  }
  if (warp == 1) tmem_alloc(reinterpret_cast<uint32_t*>(&misc[0]), L::kTmemCols);
  if (warp >= 4 && warp < 12) {
    // V and Q rings start zeroed: rows a partial tile never loads must be
    // finite (P is 0 there, and 0 * NaN would poison O).
    const int tid = threadIdx.x - 128;
    uint4 zz = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < (VS * L::kTile) / 16; i += 256)
      reinterpret_cast<uint4*>(smem + L::kOffV)[i] = zz;
    for (int i = tid; i < (QS * L::kQBytes) / 16; i += 256)
      reinterpret_cast<uint4*>(smem + L::kOffQ)[i] = zz;
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

  Walker<L::IQ> w;
  w.init(a, blockIdx.x);
  Tile t;
#define RB_NEXT(W, T) W.next(a, U, lens, qs, itq, itq_full, itq_empty, lane, T)

  if (warp == 0 || warp == 2) {
    // ------------------------------------------------ TMA producers (K+Q / V)
    const bool is_k = warp == 0;
    const uint64_t pol = l2_policy_evict_first();
    const uint64_t pol_q = l2_policy_evict_last();
    const CUtensorMap* sysmap = is_k ? &tm_sk : &tm_sv;
    const CUtensorMap* ctxmap = is_k ? &tm_rk : &tm_rv;  // ragged context
    const unsigned char* pool = is_k ? a.k_pool : a.v_pool;
    const uint32_t blk_bytes = a.block_size * 256;
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
    Walker<L::IQ> wa = w;
    Tile ta;
    auto stage_ids = [&](int slot) {
      if (RB_NEXT(wa, ta) && ta.kind == 1 && !ta.pre && a.paged) {
        const int nv = min(RB_KEY_TILE, lens[ta.r] - ta.kt * RB_KEY_TILE);
        if (lane < bpt && lane * a.block_size < nv)
          cp_async_4(ids + slot * 32 + lane, a.block_table +
                     static_cast<long long>(ta.r) * a.bt_stride + ta.kt * bpt + lane);
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int k = 0; k < L::kIdAhead; ++k) stage_ids(k);
    while (RB_NEXT(w, t)) {
      if (!is_k && first_tile) {
        // K first at start-up: every SM fires its rings at once and the first
        // Q.K^T must not queue behind the V tiles.
        if (lane == 0) mbar_wait(v_go, 0);
        __syncwarp();
      }
      first_tile = false;
      // context block ids of this tile, one lane per block
      cp_async_wait_group<L::kIdAhead - 1>();
      int blk = 0, nvalid = 0;
      if (t.kind == 1 && !t.pre) {
        nvalid = min(RB_KEY_TILE, lens[t.r] - t.kt * RB_KEY_TILE);  // keys of this tile that exist
        if (a.paged) blk = ids[(j % L::kIdAhead) * 32 + lane];
      }
      __syncwarp();
      stage_ids(j % L::kIdAhead);  // slot read above is refilled for tile j + kIdAhead
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
      const int st = j % NS;
      if (lane == 0) mbar_wait(&empty[st], ((j / NS) & 1) ^ 1);
      __syncwarp();
      uint8_t* dst = smem + ring + st * L::kTile;
      if (t.kind == 0 || t.pre) {
        // shared prefix tile (system unit, or the naive baseline's re-read)
        if (lane == 0) {
          const int h = t.kind == 0 ? t.u / a.sp.n_qt : t.h;
          mbar_arrive_expect_tx(&full[st], L::kTile);
          tma_load_3d(dst, sysmap, &full[st], 0, t.kt * RB_KEY_TILE, h, pol);
          tma_load_3d(dst + L::kTile / 2, sysmap, &full[st], 64, t.kt * RB_KEY_TILE, h, pol);
        }
      } else if (a.paged) {
        // one bulk copy per (block, kv head): the pool stores each block as
        // the [128 d][bs] swizzled UMMA operand, so the bytes land as-is
        const int nb = (nvalid + a.block_size - 1) / a.block_size;
        if (lane == 0) mbar_arrive_expect_tx(&full[st], nb * blk_bytes);
        __syncwarp();
        if (lane < nb)
          bulk_copy_g2s(dst + lane * blk_bytes,
                        pool + blk * a.pool_block_bytes + t.h * a.pool_head_bytes, blk_bytes,
                        &full[st]);
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
    constexpr uint32_t idesc_qk_pg = make_idesc_bf16_f32(128, NQ, 1, 0);
    while (RB_NEXT(w, t)) {
      if (lane == 0) {
        const int qsl = n % QS;
        if (t.first) mbar_wait(&q_full[qsl], (n / QS) & 1);
        const int st = j % KS, gb = j & 1;  // group of this tile = S buffer
        mbar_wait(&k_full[st], (j / KS) & 1);
        if (j == 0) mbar_arrive(v_go);
        mbar_wait(&s_empty[gb], ((j >> 1) & 1) ^ 1);
        RB_TRACE((j < 32), 264 + j);
        tc_fence_after();
        const uint32_t k_base = smem_k + st * L::kTile;
        const uint32_t q_base = smem_q + qsl * L::kQBytes;
        const uint32_t d_tmem = tmem_base + gb * NQ;
        const bool pl = t.kind == 1 && !t.pre && a.paged;  // paged block layout (K MN-major)
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk & 3) * 32;
          const uint64_t ad =
              pl ? ctx_k_desc(k_base, kk, a.block_size)
                 : make_smem_desc_sw128(k_base + (kk >> 2) * (L::kTile / 2) + koff, 16, 1024);
          const uint64_t bd = make_smem_desc_sw128(q_base + (kk >> 2) * (NQ * 128) + koff, 16, 1024);
          umma_f16_ss(d_tmem, ad, bd, pl ? idesc_qk_pg : idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[gb]);
        umma_commit(&k_empty[st]);
        if (t.last) umma_commit(&q_empty[qsl]);
      }
      if (t.last) ++n;
      ++j;
    }
    __syncwarp();
  } else if (warp == 3) {
    // -------------------------------- metadata: context unit prefix U
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
        sum += a.sp.hkv * ctx_nz(a, qs, i);  // units of request i (none without queries)
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int run = incl - sum;
      for (int i = lo; i < hi; ++i) {
        U[i] = run;
        run += a.sp.hkv * ctx_nz(a, qs, i);
      }
      if (lane == 0) U[b] = __shfl_sync(0xffffffffu, incl, 31);
      else __shfl_sync(0xffffffffu, incl, 31);
      __syncwarp();
      if (lane == 0) mbar_arrive(meta_bar);
    }
    // ------------------------------------------------ O^T += V^T . P^T
    int j = 0;
    int kp[2] = {0, 0};  // parts each group has finished (o_full / o_free phases)
    constexpr uint32_t idesc_pv = make_idesc_bf16_f32(128, NQ, 1, 0);
    constexpr uint32_t idesc_pv_pg = make_idesc_bf16_f32(128, NQ, 0, 0);
    while (RB_NEXT(w, t)) {
      const int gb = j & 1;
      const bool gfirst = t.pidx < 2;  // the group's first tile of this part
      const bool glast = t.rem <= 2;   // the group's last tile of this part
      if (lane == 0) {
        const int st = j % VS;
        mbar_wait(&v_full[st], (j / VS) & 1);
        mbar_wait(&p_full[gb], (j >> 1) & 1);
        if (gfirst) mbar_wait(&o_free[gb], (kp[gb] & 1) ^ 1);
        RB_TRACE((j < 32), 296 + j);
        tc_fence_after();
        const uint32_t v_base = smem_v + st * L::kTile;
        const uint32_t p_base = smem_p + gb * L::kQBytes;
        const uint32_t d_tmem = tmem_base + 2 * NQ + gb * NQ;
        const bool pl = t.kind == 1 && !t.pre && a.paged;  // paged block layout (V^T K-major)
#pragma unroll 1
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = pl ? ctx_v_desc(v_base, kk, a.block_size)
                                 : make_smem_desc_sw128(v_base + kk * 2048, L::kTile / 2, 1024);
          const uint64_t bd =
              make_smem_desc_sw128(p_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
          umma_f16_ss(d_tmem, ad, bd, pl ? idesc_pv_pg : idesc_pv, (gfirst && kk == 0) ? 0u : 1u);
        }
        umma_commit(&p_empty[gb]);
        umma_commit(&v_empty[st]);
        if (glast) umma_commit(&o_full[gb]);
      }
      if (glast) ++kp[gb];
      ++j;
    }
    __syncwarp();
  } else if (warp == 12) {
    // ----------------------------------------------------------- scheduler
    // publishes this CTA's system parts (static stream-K share), then grabs
    // context units two at a time from the global counter; a sentinel ends
    // the walk
    if (lane == 0) {
      unsigned int* ctr = reinterpret_cast<unsigned int*>(a.counters);
      const int n_sc = a.has_sys ? a.sp.n_units : 0;
      int qi = 0;
      auto push = [&](int item) {
        const int slot = qi % L::IQ;
        mbar_wait(&itq_empty[slot], ((qi / L::IQ) & 1) ^ 1);
        itq[slot] = item;
        mbar_arrive(&itq_full[slot]);
        ++qi;
      };
      if (w.xe > w.xb) {
        const int u0 = static_cast<int>(w.xb / a.sp.tpu);
        const int u1 = static_cast<int>((w.xe - 1) / a.sp.tpu);
        for (int u = u0; u <= u1; ++u) push(u);
      }
      // the context unit count needs the metadata (ready long before the
      // system share has been streamed)
      if (a.has_ctx) mbar_wait(meta_bar, 0);
      const int n_cu = a.has_ctx ? U[a.b] : 0;
      while (n_cu > 0) {
        const int i = static_cast<int>(atomicAdd(ctr + 3, 2u));
        if (i >= n_cu) break;
        push(n_sc + i);
        if (i + 1 < n_cu) push(n_sc + i + 1);
      }
      push(n_sc + n_cu);  // sentinel
    }
    __syncwarp();
  } else {
    // ------------------------------------------------- softmax groups
    const int grp = (warp - 4) >> 2;
    SmxCtx C;
    C.qd = warp & 3;                          // TMEM lane quadrant
    C.lane = lane;
    const int kl = C.qd * 32 + lane;          // key lane of the tile
    C.red = reinterpret_cast<float*>(smem + L::kOffRed) + grp * 2 * 4 * NQ;
    C.red2 = reinterpret_cast<float*>(smem + L::kOffRed2) + grp * 4 * NQ;
    C.my_mu = reinterpret_cast<float*>(smem + L::kOffMu) + (warp - 4) * NQ;
    C.my_al = reinterpret_cast<float*>(smem + L::kOffAl) + (warp - 4) * NQ;
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) C.poff[r8] = sw128_offset(r8, kl & 63);
    C.pbase = smem + L::kOffP + grp * L::kQBytes + (kl >> 6) * (NQ * 128);
    const uint32_t lq = static_cast<uint32_t>(C.qd * 32) << 16;
    C.s_addr = tmem_base + lq + grp * NQ;
    C.o_addr = tmem_base + lq + 2 * NQ + grp * NQ;
    C.bar = 1 + grp;
    if (a.has_ctx) mbar_wait(meta_bar, 0);  // part ends read the request metadata
    float l_part[NQ];
    int j = 0, kp = 0, ncol = NQ;
    while (RB_NEXT(w, t)) {
      if ((j & 1) != grp) {
        ++j;
        continue;
      }
      const int k = j >> 1;  // this group's tile count
      const bool gfirst = t.pidx < 2;
      const bool glast = t.rem <= 2;
      mbar_wait(&s_full[grp], k & 1);
      if (dts && threadIdx.x == 128 && j == 0) dts[2] = global_timer_ns();
      RB_TRACE((threadIdx.x == 128 && j < 32), 8 + j);
      tc_fence_after();
      const int key = t.kt * RB_KEY_TILE + kl;
      // Column c of the tile sees this key iff cmin <= c < cmax.
      //   system / prefix tile: every column, key < s;
      //   context tile: column c = local row li = z*NQ + c of request r
      //   (query t = li / g) sees key iff key < c_r - m_r + t + 1
      //   (attention.py:120-121), i.e. c >= cmin, and c < cmax (unit rows).
      TileMask mk;
      mk.cmax = NQ;
      if (t.kind == 1) {
        const int m_r = qs[t.r + 1] - qs[t.r];
        mk.cmax = m_r * g - t.z * NQ;
        if (gfirst) ncol = mk.cmax <= 8 ? 8 : NQ;  // decode with g <= 8: one chunk
      } else {
        ncol = NQ;
      }
      if (t.kind == 0 || t.pre) mk.cmin = key < a.sp.s ? -1 : NQ;
      else if (a.causal) mk.cmin = (key - (lens[t.r] - (qs[t.r + 1] - qs[t.r]))) * g - t.z * NQ;
      else mk.cmin = key < lens[t.r] ? -1 : NQ;
      softmax_tile<NQ>(C, l_part, ncol, gfirst, k, mk, a.scale_log2, &s_empty[grp], &p_empty[grp],
                       &p_full[grp], dts, j);
      RB_TRACE((threadIdx.x == 128 && j < 32), 40 + j);
      if (glast)
        softmax_part_end<NQ>(C, a, t, qs, l_part, ncol, grp, kp, &o_full[grp], &o_free[grp], dts,
                             j);
      RB_TRACE((threadIdx.x == 128 && j < 32), 328 + j);
      if (glast) ++kp;
      ++j;
    }
    if (dts && (threadIdx.x == 128 || threadIdx.x == 256)) dts[3 + grp] = global_timer_ns();

    // ---- every part of every CTA written: grid barrier, then each CTA merges
    // its share of the output vectors (8 warps, one vector per warp)
    named_bar_sync(3, 256);
    if (threadIdx.x == 128) {
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
