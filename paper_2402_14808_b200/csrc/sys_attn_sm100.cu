// System-prompt attention on sm_100a: tcgen05 + TMA + TMEM.
//
// Computes, for every query row of the batch (all requests' new tokens
// flattened, as in /root/reference/pkg/src/relayserve/attention.py:183-185)
// and every query head, one UNMASKED attention pass over the shared prefix
// K/V with natural-log LSE -- the reference's `_system_attention`
// (attention.py:177-200) / `attention_with_lse(causal=False)`
// (attention.py:96-134, kernels _kernels_cy.pyx:13-51).
//
// Design:
//  * swap-AB: the MMA M dimension is the 128 keys of a tile, N is the
//    (request x GQA-group) query rows of one KV head (nq = 16/32), so a
//    batch of 32 decode rows still fills M = 128:
//        S^T[128 keys x nq] = K_tile[128 x d] . Q^T        (both K-major)
//        O^T[d x nq]       = V_tile^T[d x 128] . P^T       (A MN-major)
//    accumulators in TMEM (2 S buffers + 2 O buffers = 4*nq columns).
//  * K and V tiles (128 keys x 128 d bf16 = 32 KB each) are TMA-loaded with
//    the 128B swizzle through two mbarrier rings: K slots are released as soon
//    as S^T = K.Q^T completes, V slots after O^T = V^T.P^T, so the shallow K
//    ring and the deeper V ring keep ~4 tiles of HBM reads in flight per SM.
//    Every shared-prefix byte crosses HBM exactly once per step.
//  * warp roles: warp 0 K producer (+ Q rows via cp.async), warp 1 QK^T
//    issuer (one thread) + TMEM owner, warp 2 V producer, warp 3 PV issuer,
//    then two compute groups that alternate key tiles, each with its own
//    online-softmax state (merged at the end of a unit through TMEM).
//    Thread t of a compute warp owns TMEM lane t of its quadrant = key t of
//    the tile for S, = head-dim index t for O.
//  * online softmax in the log2 domain: per-query max / sum across the 128
//    key lanes via a warp reduce-scatter butterfly + a 4-warp smem combine;
//    O accumulates in registers (acc = acc*alpha + O_tile), so the tensor
//    core never waits for a rescale.
//  * persistent stream-K over (kv head, query tile, key tile): one CTA per
//    SM, contiguous equal tile ranges, per-unit semaphore merge of partial
//    (acc, m, l) in fixed slot order -> deterministic output.
#include "rb_common.cuh"
#include "rb_plan.h"
#include "rb_args.cuh"

namespace rb {


#ifndef RB_SYS_KS
#define RB_SYS_KS 2
#endif
constexpr int kKvTileBytes = RB_KEY_TILE * RB_HEAD_DIM * 2;  // 32 KB
// lazy max: the running max of a query column moves only when a score
// exceeds it by more than kTau (log2 units), so p <= 2^kTau stays exact in
// fp32 / bf16 and most tiles skip the cross-warp max reduction
constexpr float kTau = 8.f;

// Shared-memory / thread layout for a query tile of NQ rows.  Two compute
// groups alternate key tiles (even / odd local tile index), each with its own
// online-softmax state; a group has NHALF slices of 4 warps (one per TMEM
// lane quadrant), each thread handling H query columns.
template <int NQ>
struct SysCfg {
  static constexpr int H = 16;
  static constexpr int NHALF = NQ / H;
  static constexpr int WPG = 4 * NHALF;                 // compute warps (one group)
  static constexpr int NCW = WPG;
  static constexpr int kRoleWarps = 4;                  // K producer, QK issuer, V producer, PV issuer
  static constexpr int kThreads = (kRoleWarps + NCW) * 32;

  static constexpr int KS = RB_SYS_KS;                 // K ring (freed after Q.K^T)
  static constexpr int VS = 6 - RB_SYS_KS;             // V ring (freed after P.V)
  static constexpr int kTileBytes = kKvTileBytes;       // 32 KB per K or V tile
  static constexpr int kQBytes = NQ * 256;              // [2 kblocks][NQ][128 B]
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + KS * kTileBytes;
  static constexpr int kOffQ = kOffV + VS * kTileBytes;
  static constexpr int kOffP = kOffQ + 2 * kQBytes;
  static constexpr int kRedBytes = 2 * NHALF * 4 * H * 4;  // [group][half][quadrant][H]
  static constexpr int kOffRedMax = kOffP + 2 * kQBytes;
  static constexpr int kOffRedSum = kOffRedMax;          // unit-end row sums reuse it
  static constexpr int kOffL = kOffRedMax + kRedBytes;   // [group][NQ]
  static constexpr int kOffX = kOffL + 2 * NQ * 4;       // handover m, l: [2][NQ]
  static constexpr int kOffFlag = kOffX + 2 * NQ * 4;    // lazy-max flags [group][half][2][4]
  static constexpr int kOffMs = kOffFlag + 2 * NHALF * 2 * 4 * 4;  // running max [grp][half][H]
  static constexpr int kOffBar = kOffMs + 2 * NHALF * H * 4;
  static constexpr int kNumBars = 2 * KS + 2 * VS + 18;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kBytes = kOffMisc + 64;
  static constexpr int kTmemCols = (3 * NQ <= 128) ? 128 : 256;  // S x2, O
};

template <int H>
__device__ __forceinline__ int reduce_scatter_col(int lane) {
  constexpr int S = (H == 8) ? 3 : (H == 16) ? 4 : 5;
  return lane >> (5 - S);
}

// Reduce-scatter H per-lane values over the 32 lanes of a warp: afterwards
// the returned value is the reduction of column reduce_scatter_col<H>(lane)
// over all 32 lanes.  H - 1 + (5 - log2 H) shuffles.
template <int H, bool IS_MAX>
__device__ __forceinline__ float warp_reduce_scatter(float (&v)[H], int lane) {
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
  constexpr int S = (H == 8) ? 3 : (H == 16) ? 4 : 5;
#pragma unroll
  for (int mask = (16 >> S); mask >= 1; mask >>= 1) {
    const float o = __shfl_xor_sync(0xffffffffu, r, mask);
    r = IS_MAX ? fmaxf(r, o) : r + o;
  }
  return r;
}

// Incremental (unit, key tile) walk over a CTA's tile range: no integer
// division per tile (the per-tile path of every warp role is latency-bound).
struct TileWalker {
  int kt, u, h, qt;
  __device__ __forceinline__ void start(const rb_sys_plan& P, int cta, long long t_begin) {
    u = rb_tile_unit(&P, cta, t_begin);
    kt = static_cast<int>(t_begin % P.tpu) - 1;  // the first next() lands on t_begin
    h = u / P.n_qt;
    qt = u % P.n_qt;
  }
  __device__ __forceinline__ void next(const rb_sys_plan& P) {
    if (++kt == P.tpu) {
      kt = 0;
      u = P.rr ? u + P.grid : u + 1;
      h = u / P.n_qt;
      qt = u % P.n_qt;
    }
  }
};

// Diagnostics build only: per-role event trace of CTA 0 (clock64, 256 events
// per warp, 12 warps) at debug_ts + 3072 * 8 (profiles/diag_sys_trace.py).
struct SysTrace {
  unsigned long long* p;
  int n;
  __device__ __forceinline__ void init(const SysArgs& a, int warp, int lane) {
    p = nullptr;
    n = 0;
    if (RB_DIAG && a.debug_ts != nullptr && blockIdx.x == 0 && lane == 0 && warp < 12)
      p = a.debug_ts + 3072 * 8 + warp * 512;
  }
  __device__ __forceinline__ void ev(int code) {
    if (RB_DIAG && p != nullptr && n < 256) {
      p[2 * n] = clock64();
      p[2 * n + 1] = static_cast<unsigned long long>(code);
    }
    ++n;
  }
};

template <int NQ>
__global__ void __launch_bounds__(SysCfg<NQ>::kThreads, 1)
    sys_attn_sm100_kernel(const __grid_constant__ CUtensorMap tmap_k,
                          const __grid_constant__ CUtensorMap tmap_v,
                          const __grid_constant__ CUtensorMap tmap_q, const SysArgs args) {
  using L = SysCfg<NQ>;
  constexpr int H = L::H;
  constexpr int KS = L::KS, VS = L::VS;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
  uint64_t* k_full = bars;
  uint64_t* k_empty = bars + KS;
  uint64_t* v_full = bars + 2 * KS;
  uint64_t* v_empty = bars + 2 * KS + VS;
  uint64_t* s_full = bars + 2 * KS + 2 * VS;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_full + 4;
  uint64_t* p_empty = s_full + 6;
  uint64_t* o_full = s_full + 8;
  uint64_t* o_empty = s_full + 10;
  uint64_t* q_full = s_full + 12;
  uint64_t* q_empty = s_full + 14;
  uint64_t* x_full = s_full + 16;
  uint64_t* x_empty = s_full + 17;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);
  float* red_max = reinterpret_cast<float*>(smem + L::kOffRedMax);
  float* red_sum = reinterpret_cast<float*>(smem + L::kOffRedSum);
  float* l_s = reinterpret_cast<float*>(smem + L::kOffL);
  float* x_ml = reinterpret_cast<float*>(smem + L::kOffX);
  int* rflag = reinterpret_cast<int*>(smem + L::kOffFlag);
  float* m_sm = reinterpret_cast<float*>(smem + L::kOffMs);

  const rb_sys_plan& P = args.plan;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  long long t_begin, t_end;
  rb_cta_range(&P, blockIdx.x, &t_begin, &t_end);

  unsigned long long* dts = (RB_DIAG && args.debug_ts) ? args.debug_ts + blockIdx.x * 8 : nullptr;
  if (dts && threadIdx.x == 0) dts[0] = global_timer_ns();
  if (warp == 0) {
    // q may be produced by the previous kernel in the stream (the K/V tiles
    // are not).  Once it is complete the next kernel (the context kernel of
    // the relay step) may be scheduled on the SMs this grid leaves free:
    // everything this grid waited for is visible to it too, and it polls
    // this grid's per-unit counters before reading the partials.
    pdl_wait_primary();
    pdl_launch_dependents();
  }
  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023) != 0) __trap();  // SW128 tiles need 1 KB alignment
    tma_prefetch_desc(&tmap_k);
    tma_prefetch_desc(&tmap_v);
    if (args.q_tma) tma_prefetch_desc(&tmap_q);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], L::WPG);
      mbar_init(&p_full[i], L::WPG);
      mbar_init(&p_empty[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], L::WPG);
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(x_full, L::WPG);
    mbar_init(x_empty, L::WPG);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&misc[0], L::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = misc[0];
  if (dts && threadIdx.x == 0) dts[1] = smid();
  // extended startup stamps (diagnostics): prologue, K issue, Q ready, K0 full,
  // first MMA, V issue
  unsigned long long* dtx = dts ? args.debug_ts + 2048 * 8 + blockIdx.x * 8 : nullptr;
  if (dtx && threadIdx.x == 0) dtx[0] = global_timer_ns();

  SysTrace tr;
  tr.init(args, warp, lane);
  const uint32_t smem_k = smem_u32(smem + L::kOffK);
  const uint32_t smem_v = smem_u32(smem + L::kOffV);
  const uint32_t smem_q = smem_u32(smem + L::kOffQ);
  const uint32_t smem_p = smem_u32(smem + L::kOffP);

  if (warp == 0) {
    // ------------------------------------------------- K producer (+ Q rows)
    const uint64_t pol = l2_policy_evict_first();
    int j = 0, uq = 0;
    TileWalker tw;
    tw.start(P, blockIdx.x, t_begin);
    for (long long i = t_begin; i < t_end; ++i, ++j) {
      tw.next(P);
      const int kt = tw.kt, h = tw.h, qt = tw.qt;
      const int st = j % KS;
      mbar_wait(&k_empty[st], ((j / KS) & 1) ^ 1);
      tr.ev(100000 + j);
      if (lane == 0) {
        uint8_t* dst = smem + L::kOffK + st * L::kTileBytes;
        mbar_arrive_expect_tx(&k_full[st], L::kTileBytes);
        tma_load_3d(dst, &tmap_k, &k_full[st], 0, kt * RB_KEY_TILE, h, pol);
        tma_load_3d(dst + L::kTileBytes / 2, &tmap_k, &k_full[st], 64, kt * RB_KEY_TILE, h, pol);
        if (dtx && j == 0) dtx[1] = global_timer_ns();
      }
      __syncwarp();
      if (i == t_begin || kt == 0) {
        // query rows of unit u (after this tile's K is already in flight);
        // q may be produced by the previous kernel in the stream.
        const int qb = uq & 1;
        mbar_wait(&q_empty[qb], ((uq >> 1) & 1) ^ 1);
        uint8_t* qdst = smem + L::kOffQ + qb * L::kQBytes;
        if (args.q_tma) {
          // q in device memory, g | NQ: two TMA boxes of (64 d, g heads, NQ / g
          // requests) = the unit's K-major SW128 tile (rows past the batch
          // zero-filled)
          if (lane == 0) {
            mbar_arrive_expect_tx(&q_full[qb], L::kQBytes);
            tma_load_3d(qdst, &tmap_q, &q_full[qb], 0, h * P.g, qt * NQ / P.g, pol);
            tma_load_3d(qdst + NQ * 128, &tmap_q, &q_full[qb], 64, h * P.g, qt * NQ / P.g, pol);
          }
          __syncwarp();
        } else {
          // all of the tile's 16-byte chunks in flight at once (zero-fill past the rows)
          load_unit_q<NQ, NQ>(qdst, args, h, qt * NQ, lane);
          cp_async_wait_all();
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&q_full[qb]);
        }
        if (dtx && lane == 0 && uq == 0) dtx[2] = global_timer_ns();
        ++uq;
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ V producer
    const uint64_t pol = l2_policy_evict_first();
    if (lane == 0) {
      // Start streaming V only once this CTA's first K tile and its query
      // rows have landed: at launch every SM fires its rings at once, and the
      // first Q.K^T must not queue behind four V tiles per SM.
#ifndef RB_SYS_V_EARLY
      if (t_begin < t_end) {
        mbar_wait(&k_full[0], 0);
        mbar_wait(&q_full[0], 0);  // Q rows must not queue behind the V burst either
      }
#endif
      int j = 0;
      TileWalker tw;
      tw.start(P, blockIdx.x, t_begin);
      for (long long i = t_begin; i < t_end; ++i, ++j) {
        tw.next(P);
        const int kt = tw.kt, h = tw.h;
        const int st = j % VS;
        mbar_wait(&v_empty[st], ((j / VS) & 1) ^ 1);
        tr.ev(200000 + j);
        uint8_t* dst = smem + L::kOffV + st * L::kTileBytes;
        mbar_arrive_expect_tx(&v_full[st], L::kTileBytes);
        tma_load_3d(dst, &tmap_v, &v_full[st], 0, kt * RB_KEY_TILE, h, pol);
        tma_load_3d(dst + L::kTileBytes / 2, &tmap_v, &v_full[st], 64, kt * RB_KEY_TILE, h, pol);
        if (dtx && j == 0) dtx[5] = global_timer_ns();
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ----------------------------------------------- S^T = K . Q^T issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16_f32(128, NQ, 0, 0);
      int j = 0, uq = 0;
      TileWalker tw;
      tw.start(P, blockIdx.x, t_begin);
      for (long long i = t_begin; i < t_end; ++i, ++j) {
        tw.next(P);
        const int kt = tw.kt;
        const bool new_unit = (i == t_begin) || kt == 0;
        const bool last_of_unit = (i == t_end - 1) || kt == P.tpu - 1;
        const int qb = uq & 1;
        if (new_unit) mbar_wait(&q_full[qb], (uq >> 1) & 1);
        const int st = j % KS, sb = j & 1;
        mbar_wait(&k_full[st], (j / KS) & 1);
        tr.ev(300000 + j);
        if (dtx && j == 0) dtx[3] = global_timer_ns();
        mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
        tr.ev(310000 + j);
        tc_fence_after();
        const uint32_t k_base = smem_k + st * L::kTileBytes;
        const uint32_t q_base = smem_q + qb * L::kQBytes;
        const uint32_t d_tmem = tmem_base + sb * NQ;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk & 3) * 32;
          const uint64_t a =
              make_smem_desc_sw128(k_base + (kk >> 2) * (L::kTileBytes / 2) + koff, 16, 1024);
          const uint64_t b = make_smem_desc_sw128(q_base + (kk >> 2) * (NQ * 128) + koff, 16, 1024);
          umma_f16_ss(d_tmem, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        if (dtx && j == 0) dtx[4] = global_timer_ns();
        umma_commit(&k_empty[st]);
        if (last_of_unit) {
          umma_commit(&q_empty[qb]);
          ++uq;
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // ------------------------------------------------- O^T = V^T . P^T issuer
    if (lane == 0) {
      constexpr uint32_t idesc_pv = make_idesc_bf16_f32(128, NQ, 1, 0);
      int j = 0;
      TileWalker tw;
      tw.start(P, blockIdx.x, t_begin);
      for (long long i = t_begin; i < t_end; ++i, ++j) {
        tw.next(P);
        const int st = j % VS, pb = j & 1;
        // O accumulates over the tiles of a unit; its first tile starts fresh
        const uint32_t acc0 = (i > t_begin && tw.kt != 0) ? 1u : 0u;
        mbar_wait(&v_full[st], (j / VS) & 1);
        tr.ev(400000 + j);
        mbar_wait(&p_full[pb], (j >> 1) & 1);
        tr.ev(410000 + j);
        tc_fence_after();
        const uint32_t v_base = smem_v + st * L::kTileBytes;
        const uint32_t p_base = smem_p + pb * L::kQBytes;
        const uint32_t d_tmem = tmem_base + 2 * NQ;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          // A = V^T (M = d, MN-major): 16 keys = two 8-row swizzle atoms.
          const uint64_t a = make_smem_desc_sw128(v_base + kk * 2048, L::kTileBytes / 2, 1024);
          const uint64_t b =
              make_smem_desc_sw128(p_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
          umma_f16_ss(d_tmem, a, b, idesc_pv, kk > 0 ? 1u : acc0);
        }
        umma_commit(&o_full[pb]);  // alternating by tile: see the waits below
        umma_commit(&v_empty[st]);
        umma_commit(&p_empty[pb]);
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------- softmax / O accumulation
    // One compute group: NHALF column slices x 4 TMEM lane quadrants.  Tiles
    // go through it in order; S and P are double-buffered so Q.K^T of tile
    // j+1 and P.V of tile j-1 overlap the softmax of tile j, and O
    // accumulates in TMEM across a unit (the P.V MMAs chain).
    const int cw = warp - L::kRoleWarps;
    const int hf = cw / 4;                       // column slice
    const int qd = warp & 3;                     // TMEM lane quadrant (hardware: warp % 4)
    const int col0 = hf * H;
    const bool designated = (qd == 0) && lane < H;
    const uint32_t bar_red = 1 + hf;
    const uint32_t bar_grp = 1 + L::NHALF;
    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(qd * 32) << 16);
    const uint32_t o_addr = lane_addr + 2 * NQ + col0;
    float* rmax = red_max + hf * 4 * H;
    float* rsum = rmax;  // unit-end row sums reuse the max scratch
    float* lg = l_s;
    const int rcol = reduce_scatter_col<H>(lane);
    const bool rwriter = (lane & ((32 / H) - 1)) == 0;
    const int key_lane = qd * 32 + lane;
    // swizzled P column of this key lane: chunk (key & 63) / 8, byte (key & 7) * 2
    const uint32_t pkch = static_cast<uint32_t>((key_lane & 63) >> 3);
    const uint32_t pkby = static_cast<uint32_t>((key_lane & 7) << 1);
    const uint32_t pkb = (key_lane >> 6) * (NQ * 128);

    float m_run[H], acc[H], l_part[H];
    // diagnostics build only: epilogue time split (o_full wait, through the
    // row-sum exchange, through the part write / publish) and unit count
    unsigned long long d_t0 = 0, d_e1 = 0, d_e2 = 0, d_e3 = 0;
    int d_nu = 0;
    int pend_u = -1;  // relay: unit whose part is written but not yet published
    pdl_wait_primary();  // o_sys / partials may still be read by the previous kernel
    long long i = t_begin;
    while (i < t_end) {
      const int u = rb_tile_unit(&P, blockIdx.x, i);
      const long long unit_end = min(t_end, (i / P.tpu + 1) * P.tpu);  // local unit end
      const long long ia = i, ib = unit_end - 1;
#pragma unroll
      for (int c = 0; c < H; ++c) {
        m_run[c] = -INFINITY;
        l_part[c] = 0.f;
      }
      int kt = static_cast<int>(ia % P.tpu) - 1;
      for (long long it = ia; it <= ib; ++it) {
        const int j = static_cast<int>(it - t_begin);
        ++kt;
        const int gb = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        // ---- S tile -> scores (log2 domain)
        mbar_wait(&s_full[gb], ph);
        tr.ev(500000 + j);
        if (dts && j == 0 && threadIdx.x == L::kRoleWarps * 32) dts[2] = global_timer_ns();
        tc_fence_after();
        float x[H];
        tmem_ld_32x32b<H>(lane_addr + gb * NQ + col0, x);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[gb]);
        const bool valid = kt * RB_KEY_TILE + key_lane < P.s;
        bool over = false;
#pragma unroll
        for (int c = 0; c < H; ++c) {
          x[c] = valid ? x[c] * args.scale_log2 : -INFINITY;
          over |= x[c] > m_run[c] + kTau;
        }
        // ---- lazy max: the running max moves only when some score of the
        // column exceeds it by more than kTau (always on a unit's first tile);
        // the 4 quadrant warps agree through one flag exchange
        int* fl = rflag + (hf * 2 + gb) * 4;
        over = __any_sync(0xffffffffu, over);
        if (lane == 0) fl[qd] = over ? 1 : 0;
        named_bar_sync(bar_red, 128);
        tr.ev(510000 + j);
        const int4 fv = *reinterpret_cast<const int4*>(fl);
        if (fv.x | fv.y | fv.z | fv.w) {
          float tmp[H];
#pragma unroll
          for (int c = 0; c < H; ++c) tmp[c] = x[c];
          const float wmax = warp_reduce_scatter<H, true>(tmp, lane);
          if (rwriter) rmax[qd * H + rcol] = wmax;
          named_bar_sync(bar_red, 128);
          float al[H];
#pragma unroll
          for (int c4 = 0; c4 < H; c4 += 4) {
            const float4 a0 = *reinterpret_cast<const float4*>(rmax + 0 * H + c4);
            const float4 a1 = *reinterpret_cast<const float4*>(rmax + 1 * H + c4);
            const float4 a2 = *reinterpret_cast<const float4*>(rmax + 2 * H + c4);
            const float4 a3 = *reinterpret_cast<const float4*>(rmax + 3 * H + c4);
            const float tm[4] = {fmaxf(fmaxf(a0.x, a1.x), fmaxf(a2.x, a3.x)),
                                 fmaxf(fmaxf(a0.y, a1.y), fmaxf(a2.y, a3.y)),
                                 fmaxf(fmaxf(a0.z, a1.z), fmaxf(a2.z, a3.z)),
                                 fmaxf(fmaxf(a0.w, a1.w), fmaxf(a2.w, a3.w))};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = c4 + e;
              const float mn = fmaxf(m_run[c], tm[e]);
              al[c] = (m_run[c] == -INFINITY) ? 0.f : fast_exp2(m_run[c] - mn);
              m_run[c] = mn;
              l_part[c] *= al[c];
            }
          }
          if (it > ia) {
            // rescale the O accumulator once the previous P.V has landed.
            // o_full alternates by tile, so this parity wait is unambiguous:
            // P.V(j-3) is known complete (p_empty of tile j-1).
            mbar_wait(&o_full[(j - 1) & 1], static_cast<uint32_t>(((j - 1) >> 1) & 1));
            tc_fence_after();
            float o[H];
            tmem_ld_32x32b<H>(o_addr, o);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < H; ++c) o[c] *= al[c];
            tmem_st_32x32b<H>(o_addr, o);
            tmem_wait_st();
            tc_fence_before();
          }
        }
#pragma unroll
        for (int c = 0; c < H; ++c) {
          const float mu = (m_run[c] == -INFINITY) ? 0.f : m_run[c];
          x[c] = fast_exp2(x[c] - mu);  // p; exactly 0 for masked keys
          l_part[c] += x[c];
        }
        // ---- P (bf16) -> smem, K-major SW128 [NQ rows][128 keys]
        tr.ev(520000 + j);
        mbar_wait(&p_empty[gb], ph ^ 1);
        tr.ev(530000 + j);
        {
          uint8_t* pdst = smem + L::kOffP + gb * L::kQBytes + pkb;
#pragma unroll
          for (int c = 0; c < H; ++c) {
            const int row = col0 + c;  // row & 7 == c & 7 (col0 is a multiple of 16)
            const uint32_t off = (row >> 3) * 1024 + (c & 7) * 128 + ((pkch ^ (c & 7)) << 4) + pkby;
            *reinterpret_cast<__nv_bfloat16*>(pdst + off) = __float2bfloat16_rn(x[c]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[gb]);
        tr.ev(540000 + j);
        if (pend_u >= 0 && (it > ia || it == ib)) {
          // publish the previous unit's part now that its stores have had a
          // tile's time to drain: the fence no longer stalls the group
          if (cw == 0 && lane == 0) {
            __threadfence();
            atomicAdd(&args.counters[pend_u], 1);
          }
          pend_u = -1;
        }
      }

      // ---- unit end: O from TMEM (after the unit's last P.V), row sums
      // reduced over the 128 key lanes once per unit, then write / merge
      {
        const int jl = static_cast<int>(ib - t_begin);
        if (dts) d_t0 = global_timer_ns();
        // P.V(jl) complete implies every earlier MMA complete
        mbar_wait(&o_full[jl & 1], static_cast<uint32_t>((jl >> 1) & 1));
        if (dts) d_e1 += global_timer_ns() - d_t0;
        tc_fence_after();
        tmem_ld_32x32b<H>(o_addr, acc);
        tmem_wait_ld();
        tc_fence_before();
        const float wsum = warp_reduce_scatter<H, false>(l_part, lane);
        named_bar_sync(bar_red, 128);  // rsum aliases rmax: last tile's max reads done
        if (rwriter) rsum[qd * H + rcol] = wsum;
        named_bar_sync(bar_red, 128);
        if (designated)
          lg[col0 + lane] = rsum[0 * H + lane] + rsum[1 * H + lane] + rsum[2 * H + lane] +
                            rsum[3 * H + lane];
        named_bar_sync(bar_grp, L::NCW * 32);  // lg complete; rsum reads done
      }
      {
        float lrow[H];
#pragma unroll
        for (int c = 0; c < H; ++c) lrow[c] = lg[col0 + c];
        named_bar_sync(bar_grp, L::NCW * 32);  // lg reads done before the next unit's writes
        if (dts) d_e2 += global_timer_ns() - d_t0;
        const int h = u / P.n_qt, qt = u % P.n_qt;
        const int owner0 = rb_unit_owner0(&P, u);
        const int nparts = rb_unit_parts(&P, u);
        const int dcol = key_lane;  // O lane = head-dim index
        if (args.defer_merge) {
          // relay path: hand the (unnormalised) part to the fusion epilogue
          const int slot = blockIdx.x - owner0;
          const long long pbase = static_cast<long long>(u) * P.max_parts + slot;
          float* pacc = args.part_acc + pbase * NQ * RB_HEAD_DIM;
          float* pml = args.part_ml + pbase * 2 * NQ;
#pragma unroll
          for (int c = 0; c < H; ++c) {
            const int col = col0 + c;
            pacc[col * RB_HEAD_DIM + dcol] = acc[c];
            if (qd == 0 && lane == 0) {
              pml[col] = m_run[c];
              pml[NQ + col] = lrow[c];
            }
          }
          if (args.counters != nullptr) {
            // publish the part (the context kernel, running concurrently,
            // polls the unit's counter): the barrier orders every warp's
            // writes before thread (0, 0)'s fence + increment, which come one
            // tile into the next unit (or at the end of the CTA's range)
            named_bar_sync(bar_grp, L::NCW * 32);
            pend_u = u;
          }
        } else if (nparts == 1) {
#pragma unroll
          for (int c = 0; c < H; ++c) {
            const int f = qt * NQ + col0 + c;
            if (f < P.rows_per_head) {
              const int row = f / P.g, hh = h * P.g + f % P.g;
              const long long o_idx = static_cast<long long>(row) * P.hq + hh;
              args.o_sys[o_idx * RB_HEAD_DIM + dcol] = acc[c] / lrow[c];
              if (qd == 0 && lane == 0)
                args.lse_sys[o_idx] = (m_run[c] + __log2f(lrow[c])) * kLn2;
            }
          }
        }
        // (split units always defer: rb_system_attention merges their parts in
        // a separate launch, sys_merge_parts_kernel)
      }
      if (dts) {
        d_e3 += global_timer_ns() - d_t0;
        ++d_nu;
      }
      i = unit_end;
    }
    if (pend_u >= 0 && cw == 0 && lane == 0) {
      __threadfence();
      atomicAdd(&args.counters[pend_u], 1);
    }
    if (dts && threadIdx.x == L::kRoleWarps * 32) {
      dts[3] = global_timer_ns();
      dts[4] = d_nu;
      dtx[6] = d_e1;
      dtx[7] = d_e2;
      dtx[3] = d_e3;  // replaces the k0_full stamp
    }
  }

  if (dts && threadIdx.x == 0) dts[5] = global_timer_ns();
  if (dts && threadIdx.x == 64) dts[6] = global_timer_ns();
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
static cudaError_t launch_sys(const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& tq,
                              const SysArgs& a, cudaStream_t stream) {
  using L = SysCfg<NQ>;
  static_assert(L::kBytes <= 232448, "system kernel shared memory over the 227 KB limit");
  static_assert(L::kThreads <= 1024, "too many warps");
  auto kern = sys_attn_sm100_kernel<NQ>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, dim3(a.plan.grid), dim3(L::kThreads), L::kBytes, stream, tk, tv, tq, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_system_attention_gqa(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                                        const SysArgs&, cudaStream_t);
cudaError_t launch_system_attention_gqa2(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                                         const SysArgs&, cudaStream_t);

// Standalone system attention with split units: every CTA wrote its part of
// a unit (defer_merge); one warp per (unit, row) merges the unit's parts in
// slot order -- max of the parts' m, weights exp2(m_k - M), O and l as
// weighted sums in slot order (deterministic) -- normalises and writes o_sys
// / lse_sys.  Spread over the whole GPU instead of one CTA per unit.
__global__ void __launch_bounds__(256) sys_merge_parts_kernel(const SysArgs args) {
  const rb_sys_plan& P = args.plan;
  const int lane = threadIdx.x & 31;
  const long long pr = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  pdl_wait_primary();
  if (pr >= static_cast<long long>(P.n_units) * P.nq) return;
  const int u = static_cast<int>(pr / P.nq), ur = static_cast<int>(pr % P.nq);
  const int h = u / P.n_qt, qt = u % P.n_qt;
  const int f = qt * P.nq + ur;
  if (f >= P.rows_per_head) return;
  const long long o_idx = static_cast<long long>(f / P.g) * P.hq + h * P.g + f % P.g;
  const int np = rb_unit_parts(&P, u);
  const long long base = static_cast<long long>(u) * P.max_parts;
  float M = -INFINITY;
  for (int k = lane; k < np; k += 32) M = fmaxf(M, __ldcg(args.part_ml + (base + k) * 2 * P.nq + ur));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  float L = 0.f;
  for (int k0 = 0; k0 < np; k0 += 32) {
    // lane j holds part k0 + j's weight and l; the O rows stream 8 at a time
    float wj = 0.f, lj = 0.f;
    if (k0 + lane < np) {
      const float* ml = args.part_ml + (base + k0 + lane) * 2 * P.nq;
      const float mk = __ldcg(ml + ur);
      lj = __ldcg(ml + P.nq + ur);
      wj = (mk == -INFINITY) ? 0.f : fast_exp2(mk - M);
    }
    const int nk = min(32, np - k0);
    for (int kb = 0; kb < nk; kb += 8) {
      float4 a8[8];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int k = k0 + min(kb + kk, nk - 1);
        a8[kk] = __ldcg(reinterpret_cast<const float4*>(args.part_acc + ((base + k) * P.nq + ur) * RB_HEAD_DIM) + lane);
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const float w = __shfl_sync(0xffffffffu, wj, min(kb + kk, 31));
        const float l = __shfl_sync(0xffffffffu, lj, min(kb + kk, 31));
        if (kb + kk < nk) {
          L = fmaf(l, w, L);
          O.x = fmaf(a8[kk].x, w, O.x);
          O.y = fmaf(a8[kk].y, w, O.y);
          O.z = fmaf(a8[kk].z, w, O.z);
          O.w = fmaf(a8[kk].w, w, O.w);
        }
      }
    }
  }
  const float inv = 1.f / L;
  reinterpret_cast<float4*>(args.o_sys + o_idx * RB_HEAD_DIM)[lane] =
      make_float4(O.x * inv, O.y * inv, O.z * inv, O.w * inv);
  if (lane == 0) args.lse_sys[o_idx] = (M + __log2f(L)) * kLn2;
}

cudaError_t launch_sys_merge_parts(const SysArgs& a, cudaStream_t stream) {
  const long long pairs = static_cast<long long>(a.plan.n_units) * a.plan.nq;
  const long long blocks = (pairs + 7) / 8;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  cudaError_t e = launch_pdl(sys_merge_parts_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0,
                             stream, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_system_attention(const CUtensorMap& tk, const CUtensorMap& tv,
                                    const CUtensorMap& tq, const SysArgs& a, cudaStream_t stream) {
  switch (a.plan.nq) {
    case 16: return launch_sys<16>(tk, tv, tq, a, stream);
    case 32: return launch_sys<32>(tk, tv, tq, a, stream);
    case 128: return launch_system_attention_gqa(tk, tv, tq, a, stream);
    case 256: return launch_system_attention_gqa2(tk, tv, tq, a, stream);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------ layout probe
// One-CTA check of the exact operand layouts / descriptors the system kernel
// uses (K, V in the TMA SW128 box layout; Q, P in the K-major SW128 layout).
template <int NQ>
__global__ void umma_probe_kernel(const __nv_bfloat16* k, const __nv_bfloat16* q,
                                  const __nv_bfloat16* v, const __nv_bfloat16* p, float* s_out,
                                  float* o_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sk = smem;
  uint8_t* sv = smem + kKvTileBytes;
  uint8_t* sq = smem + 2 * kKvTileBytes;
  uint8_t* sp = sq + NQ * 256;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sp + NQ * 256);
  uint32_t* tm = reinterpret_cast<uint32_t*>(bar + 2);
  for (int idx = threadIdx.x; idx < 128 * 128; idx += blockDim.x) {
    const int row = idx / 128, col = idx % 128;
    const uint32_t off = (col >> 6) * (kKvTileBytes / 2) + sw128_offset(row, col & 63);
    *reinterpret_cast<__nv_bfloat16*>(sk + off) = k[idx];
    *reinterpret_cast<__nv_bfloat16*>(sv + off) = v[idx];
  }
  for (int idx = threadIdx.x; idx < NQ * 128; idx += blockDim.x) {
    const int row = idx / 128, col = idx % 128;
    const uint32_t off = (col >> 6) * (NQ * 128) + sw128_offset(row, col & 63);
    *reinterpret_cast<__nv_bfloat16*>(sq + off) = q[idx];
    *reinterpret_cast<__nv_bfloat16*>(sp + off) = p[idx];
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(tm, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tm;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc_qk = make_idesc_bf16_f32(128, NQ, 0, 0);
    constexpr uint32_t idesc_pv = make_idesc_bf16_f32(128, NQ, 1, 0);
    const uint32_t k_base = smem_u32(sk), v_base = smem_u32(sv);
    const uint32_t q_base = smem_u32(sq), p_base = smem_u32(sp);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a =
          make_smem_desc_sw128(k_base + (kk >> 2) * (kKvTileBytes / 2) + (kk & 3) * 32, 16, 1024);
      const uint64_t b = make_smem_desc_sw128(q_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
      umma_f16_ss(tbase, a, b, idesc_qk, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar[0]);
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t a = make_smem_desc_sw128(v_base + kk * 2048, kKvTileBytes / 2, 1024);
      const uint64_t b = make_smem_desc_sw128(p_base + (kk >> 2) * (NQ * 128) + (kk & 3) * 32, 16, 1024);
      umma_f16_ss(tbase + 64, a, b, idesc_pv, kk > 0 ? 1u : 0u);
    }
    umma_commit(&bar[1]);
  }
  __syncwarp();
  mbar_wait(&bar[0], 0);
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t laddr = tbase + (static_cast<uint32_t>(warp * 32) << 16);
  for (int c0 = 0; c0 < NQ; c0 += 8) {
    float s[8], o[8];
    tmem_ld_32x32b<8>(laddr + c0, s);
    tmem_ld_32x32b<8>(laddr + 64 + c0, o);
    tmem_wait_ld();
    for (int c = 0; c < 8; ++c) {
      s_out[(warp * 32 + lane) * NQ + c0 + c] = s[c];
      o_out[(warp * 32 + lane) * NQ + c0 + c] = o[c];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tbase, 128);
  }
}

template <int N>
static cudaError_t launch_probe_n(const __nv_bfloat16* k, const __nv_bfloat16* q,
                                  const __nv_bfloat16* v, const __nv_bfloat16* p, float* s_out,
                                  float* o_out, cudaStream_t stream) {
  const int smem = 2 * kKvTileBytes + 2 * 64 * 256 + 64;
  cudaError_t e =
      cudaFuncSetAttribute(umma_probe_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  umma_probe_kernel<N><<<1, 128, smem, stream>>>(k, q, v, p, s_out, o_out);
  return cudaGetLastError();
}

cudaError_t launch_umma_probe(const __nv_bfloat16* k, const __nv_bfloat16* q,
                              const __nv_bfloat16* v, const __nv_bfloat16* p, int nq,
                              float* s_out, float* o_out, cudaStream_t stream) {
  switch (nq) {
    case 16: return launch_probe_n<16>(k, q, v, p, s_out, o_out, stream);
    case 32: return launch_probe_n<32>(k, q, v, p, s_out, o_out, stream);
    case 64: return launch_probe_n<64>(k, q, v, p, s_out, o_out, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rb
