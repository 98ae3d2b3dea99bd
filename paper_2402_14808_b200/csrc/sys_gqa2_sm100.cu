// System-prompt attention for >= 256 query rows per KV head (GQA groups x
// large batches: C4 has 512, C5 2048 rows per KV head) on sm_100a.
//
// The reference's `_system_attention` (attention.py:177-200): one unmasked
// attention pass of every flattened query row over the shared prefix, with
// natural-log LSE.  A unit is 256 query rows of one KV head = two 128-row
// query tiles that share every K/V tile the CTA loads:
//     S_i[128 q x 128 keys] = Q_i . K^T            (SS: Q_i, K K-major SW128)
//     O_i[128 q x 128 d]   += P_i[128 x 128] . V   (TS: P_i in TMEM, V MN-major)
// for i = 0, 1.  Two softmax warpgroups (one per query tile, thread r = TMEM
// lane r = query row r) ping-pong with the tensor core: while warpgroup 0
// turns S_0(j) into probabilities, the tensor core runs P_1(j-1).V and
// Q_1.K(j)^T, and the other way round.  P_i goes back into TMEM over S_i as
// packed bf16 (tcgen05.st, 64 columns) and feeds the P.V MMA directly from
// tensor memory, so neither S nor P ever touches shared memory.  The
// tcgen05 MMAs of the issuing thread execute in order, so S_i(j+1) -- which
// overwrites P_i(j) -- is issued only after P_i(j).V.
//
// TMEM (512 columns): S_0 [0,128), O_0 [128,256), S_1 [256,384), O_1 [384,512).
// Shared memory: K ring 2 x 32 KB, V ring 2 x 32 KB, Q_0 | Q_1 2 x 32 KB.
// Roles (384 threads): warp 0 K TMA producer, warp 1 MMA issuer + TMEM
// owner, warp 2 Q rows (cp.async, SW128), warp 3 V TMA producer, warps 4-7 /
// 8-11 softmax + epilogue of query tile 0 / 1.
// Lazy max (tau = 8, log2 units) per row: the O row in TMEM is rescaled only
// when its reference moves, after the previous P.V has landed.
// Work split, parts, relay publication: as the other system kernels
// (rb_plan.h with nq = 256).
#include "rb_common.cuh"
#include "rb_plan.h"
#include "rb_args.cuh"

namespace rb {

namespace g2 {

constexpr int kRows = 128;                 // query rows per tile (MMA M)
constexpr int kSub = 2;                    // query tiles per unit
constexpr int kUnitRows = kRows * kSub;    // plan nq
constexpr int kTile = RB_KEY_TILE * RB_HEAD_DIM * 2;  // 32 KB K or V tile
#ifndef G2_KS
#define G2_KS 3
#endif
#ifndef G2_VS
#define G2_VS 2
#endif
constexpr int KS = G2_KS, VS = G2_VS;
// diagnostics experiments (variant builds only): G2_NO_SOFTMAX=1 skips the
// softmax (warps hand P back at once), G2_NO_MMA=1 issues no MMAs
#ifndef G2_NO_SOFTMAX
#define G2_NO_SOFTMAX 0
#endif
#ifndef G2_NO_MMA
#define G2_NO_MMA 0
#endif
// timing experiments only (wrong results): G2_PV_KMAJOR=1 reads the V tile
// as a K-major B operand, G2_PV_SS=1 takes the P.V A operand from smem (Q)
#ifndef G2_PV_KMAJOR
#define G2_PV_KMAJOR 0
#endif
#ifndef G2_PV_SS
#define G2_PV_SS 0
#endif
// G2_POLY=n > 0: one score pair in every n takes exp2 on the FMA pipe
// (exp2_poly2) instead of MUFU.EX2 (0: all on MUFU).  Measured per-tile
// period (C4 shape, CTA 0): n=0 3364 cycles, 2: 3432, 3: 3053, 4: 2989,
// 6: 3095, 8: 3056 -- one in four relieves the MUFU without loading the FMA
// pipe past it
#ifndef G2_POLY
#define G2_POLY 4
#endif
// G2_KV_EVICT_LAST=1: K/V tiles with the L2 evict-last hint -- the CTAs of a
// head's units read them in lockstep (C5 626 -> 623 us, C4 108.6 -> 108.2
// against evict-first)
#ifndef G2_KV_EVICT_LAST
#define G2_KV_EVICT_LAST 1
#endif
// G2_NO_QTMA=1 (diagnostics variant): query tiles always by the cp.async loader
#ifndef G2_NO_QTMA
#define G2_NO_QTMA 0
#endif
constexpr int kQBytes = kRows * 256;       // one query tile: [2 kblocks][128 rows][128 B]
constexpr int kOffK = 0;
constexpr int kOffV = kOffK + KS * kTile;
constexpr int kOffQ = kOffV + VS * kTile;
constexpr int kOffBar = kOffQ + kSub * kQBytes;
constexpr int kNumBars = 2 * KS + 2 * VS + 3 * kSub + 2;
constexpr int kOffMisc = kOffBar + kNumBars * 8;
constexpr int kBytes = kOffMisc + 64;
constexpr int kThreads = 384;
constexpr int kSmWarp0 = 4;                // first softmax warp
constexpr uint32_t kTmemCols = 512;
constexpr float kTau = 8.f;

// Incremental (unit, key tile) walk over a CTA's tile range (rb_plan.h).
struct Walk {
  int kt, u;
  __device__ __forceinline__ void start(const rb_sys_plan& P, int cta, long long t_begin) {
    u = rb_tile_unit(&P, cta, t_begin);
    kt = static_cast<int>(t_begin % P.tpu) - 1;
  }
  __device__ __forceinline__ void next(const rb_sys_plan& P) {
    if (++kt == P.tpu) {
      kt = 0;
      u = P.rr ? u + P.grid : u + 1;
    }
  }
};

}  // namespace g2

__global__ void __launch_bounds__(g2::kThreads, 1)
    sys_gqa2_sm100_kernel(const __grid_constant__ CUtensorMap tmap_k,
                          const __grid_constant__ CUtensorMap tmap_v,
                          const __grid_constant__ CUtensorMap tmap_q, const SysArgs args) {
  using namespace g2;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* k_full = bars;
  uint64_t* k_empty = bars + KS;
  uint64_t* v_full = bars + 2 * KS;
  uint64_t* v_empty = bars + 2 * KS + VS;
  uint64_t* s_full = bars + 2 * KS + 2 * VS;  // [kSub] S_i(j) computed
  uint64_t* p_full = s_full + kSub;           // [kSub] P_i(j) in TMEM (4 softmax warps)
  uint64_t* o_full = p_full + kSub;           // [kSub] P_i(j).V landed
  uint64_t* q_full = o_full + kSub;
  uint64_t* q_empty = q_full + 1;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kOffMisc);

  const rb_sys_plan& P = args.plan;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  long long t_begin, t_end;
  rb_cta_range(&P, blockIdx.x, &t_begin, &t_end);
  // diagnostics build: CTA 0 records clock64 at 8 events x 128 tiles
  // (WG0 S ready / P done, WG1 S ready / P done, MMA: P0 seen, S0 issued,
  // P1 seen, S1 issued)
  unsigned long long* evt =
      (RB_DIAG && args.debug_ts && blockIdx.x == 0) ? args.debug_ts + 6144 * 8 : nullptr;
  // per-CTA %globaltimer stamps (same slots as the other system kernels):
  // [0] entry, [1] smid, [2] first S ready (WG0), [3] last unit's epilogue
  // start, [4] its part / row written, [5] its merge done (merging CTA), [6]
  // first unit's query rows in smem, [7] exit
  unsigned long long* dts = (RB_DIAG && args.debug_ts) ? args.debug_ts + blockIdx.x * 8 : nullptr;
  if (dts && threadIdx.x == 0) {
    dts[0] = global_timer_ns();
    dts[1] = smid();
  }
#define G2_EVT(e, jj) \
  do {                \
    if (evt && (jj) < 128) evt[(e) * 128 + (jj)] = clock64(); \
  } while (0)

  if (warp == 2) {
    pdl_wait_primary();       // q may come from the previous kernel
    pdl_launch_dependents();  // the relay step's context kernel may start
  }
  if (threadIdx.x == 0) {
    if ((smem_u32(smem) & 1023) != 0) __trap();
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
    for (int i = 0; i < kSub; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_full[i], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&misc[0], kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = misc[0];
  const uint32_t smem_k = smem_u32(smem + kOffK);
  const uint32_t smem_v = smem_u32(smem + kOffV);
  const uint32_t smem_q = smem_u32(smem + kOffQ);

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------- K / V TMA producers
    const bool is_k = warp == 0;
    if (lane == 0) {
      const uint64_t pol = G2_KV_EVICT_LAST ? l2_policy_evict_last() : l2_policy_evict_first();
      const int ns = is_k ? KS : VS;
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      const CUtensorMap* map = is_k ? &tmap_k : &tmap_v;
      uint8_t* base = smem + (is_k ? kOffK : kOffV);
      int j = 0;
      Walk w;
      w.start(P, blockIdx.x, t_begin);
      for (long long i = t_begin; i < t_end; ++i, ++j) {
        w.next(P);
        const int h = w.u / P.n_qt;
        const int st = j % ns;
        mbar_wait(&empty[st], ((j / ns) & 1) ^ 1);
        uint8_t* dst = base + st * kTile;
        mbar_arrive_expect_tx(&full[st], kTile);
        tma_load_3d(dst, map, &full[st], 0, w.kt * RB_KEY_TILE, h, pol);
        tma_load_3d(dst + kTile / 2, map, &full[st], 64, w.kt * RB_KEY_TILE, h, pol);
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ------------------------------------- query rows of each unit (2 tiles)
    int uq = 0;
    for (long long i = t_begin; i < t_end;) {
      const int u = rb_tile_unit(&P, blockIdx.x, i);
      const int h = u / P.n_qt, qt = u % P.n_qt;
      mbar_wait(q_empty, (uq & 1) ^ 1);
      uint8_t* qdst = smem + kOffQ;
      if (args.q_tma && !G2_NO_QTMA) {
        // 4 boxes of (64 d, g heads, 128 / g requests): rows f = request * g
        // + member in the K-major SW128 order the MMA reads; rows past
        // rows_per_head are requests past n_rows, zero-filled by the TMA
        if (lane == 0) {
          mbar_arrive_expect_tx(q_full, kSub * kQBytes);
#pragma unroll
          for (int sb = 0; sb < kSub; ++sb)
#pragma unroll
            for (int kb = 0; kb < 2; ++kb)
              tma_load_3d(qdst + sb * kQBytes + kb * (kRows * 128), &tmap_q, q_full, kb * 64, h * P.g,
                          (qt * kUnitRows + sb * kRows) / P.g, l2_policy_evict_first());
        }
        __syncwarp();
      } else {
        load_unit_q<kRows, kUnitRows>(qdst, args, h, qt * kUnitRows, lane);
        cp_async_wait_all();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(q_full);
      }
      if (dts && lane == 0 && uq == 0) dts[6] = global_timer_ns();
      ++uq;
      i = P.rr ? (i / P.tpu + 1) * P.tpu : min(t_end, (i / P.tpu + 1) * P.tpu);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Order per key tile j: P_0(j).V, Q_0.K(j+1)^T, P_1(j).V, Q_1.K(j+1)^T --
    // each S_i(j+1) right behind the P.V that frees its TMEM, so the softmax
    // of one query tile overlaps the other tile's MMAs.  The whole warp runs
    // the loop (warp-uniform descriptors, built once and offset by adding to
    // the start-address field); one elected lane issues each MMA / commit.
    {
      constexpr uint32_t idesc_qk = make_idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16_f32(128, 128, 0, G2_PV_KMAJOR ? 0 : 1);
      const int n = static_cast<int>(t_end - t_begin);
      Walk wk, wv;
      wk.start(P, blockIdx.x, t_begin);
      wv.start(P, blockIdx.x, t_begin);
      int uq = 0;
      bool k_last = false;  // tile of the current S issue ends its unit
      auto begin_k = [&](int j) {
        wk.next(P);
        const bool first = (j == 0) || wk.kt == 0;
        k_last = (j == n - 1) || wk.kt == P.tpu - 1;
        if (first) mbar_wait(q_full, uq & 1);
        mbar_wait(&k_full[j % KS], (j / KS) & 1);
        tc_fence_after();
        G2_EVT(8, j);
      };
      // descriptor start-address field = byte address >> 4 (bits [0,14))
      const uint64_t q_desc0 = make_smem_desc_sw128(smem_q, 16, 1024);
      const uint64_t k_desc0 = make_smem_desc_sw128(smem_k, 16, 1024);
      const uint64_t v_desc0 = G2_PV_KMAJOR ? make_smem_desc_sw128(smem_v, 16, 1024)
                                            : make_smem_desc_sw128(smem_v, kTile / 2, 1024);
      auto issue_s = [&](int j, int sub) {
        const uint64_t kd = k_desc0 + (((j % KS) * kTile) >> 4);
        const uint64_t qd = q_desc0 + ((sub * kQBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * (kRows * 128) + (kk & 3) * 32) >> 4;
          const uint32_t offk = ((kk >> 2) * (kTile / 2) + (kk & 3) * 32) >> 4;
          if (!G2_NO_MMA) umma_f16_ss_elect(tmem_base + sub * 256, qd + off, kd + offk, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit_elect(&s_full[sub]);
      };
      auto end_k = [&](int j) {
        umma_commit_elect(&k_empty[j % KS]);
        if (k_last) {
          umma_commit_elect(q_empty);
          ++uq;
        }
      };
      if (n > 0) {
        begin_k(0);
        issue_s(0, 0);
        issue_s(0, 1);
        end_k(0);
      }
      for (int j = 0; j < n; ++j) {
        wv.next(P);
        const uint32_t acc0 = (j > 0 && wv.kt != 0) ? 1u : 0u;
        const int st = j % VS;
        mbar_wait(&v_full[st], (j / VS) & 1);
        G2_EVT(9, j);
        const uint64_t vd = v_desc0 + ((st * kTile) >> 4);
        for (int sub = 0; sub < kSub; ++sub) {
          mbar_wait(&p_full[sub], static_cast<uint32_t>(j & 1));
          tc_fence_after();
          G2_EVT(4 + 2 * sub, j);
          const uint32_t p_tmem = tmem_base + sub * 256;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            // A = P_i (TMEM, 16 keys = 8 columns); B = V tile, MN-major: 16 keys
            // = two 8-key swizzle atoms, the two 64-wide d halves kTile / 2 apart
            const uint64_t b = vd + ((G2_PV_KMAJOR ? (kk >> 2) * (kTile / 2) + (kk & 3) * 32 : kk * 2048) >> 4);
            if (G2_PV_SS) {
              const uint64_t a = make_smem_desc_sw128(
                  smem_q + sub * kQBytes + (kk >> 2) * (kRows * 128) + (kk & 3) * 32, 16, 1024);
              umma_f16_ss_elect(tmem_base + sub * 256 + 128, a, b, idesc_pv, kk > 0 ? 1u : acc0);
            } else if (!G2_NO_MMA) {
              umma_f16_ts_elect(tmem_base + sub * 256 + 128, p_tmem + kk * 8, b, idesc_pv,
                                kk > 0 ? 1u : acc0);
            }
          }
          umma_commit_elect(&o_full[sub]);
          if (sub == kSub - 1) umma_commit_elect(&v_empty[st]);
          if (j + 1 < n) {
            if (sub == 0) begin_k(j + 1);
            issue_s(j + 1, sub);
            G2_EVT(5 + 2 * sub, j + 1);
            if (sub == kSub - 1) end_k(j + 1);
          }
        }
      }
    }
  } else {
    // ------------------------------------------- softmax / epilogue (sub)
    const int sub = (warp - kSmWarp0) >> 2;
    const int r = (warp & 3) * 32 + lane;       // query row of the tile = TMEM lane
    const int ur = sub * kRows + r;             // row within the unit
    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t s_addr = lane_addr + sub * 256;
    const uint32_t o_addr = s_addr + 128;
    const uint32_t bar_id = 1, bar_n = 32 * 4 * kSub;  // all softmax warps
    pdl_wait_primary();  // partials / o_sys may still be read by the previous kernel
    float m_run = -INFINITY, l_run = 0.f;
    long long i = t_begin;
    int j = 0;
    while (i < t_end) {
      const int u = rb_tile_unit(&P, blockIdx.x, i);
      const long long unit_end = min(t_end, (i / P.tpu + 1) * P.tpu);
      const int kt0 = static_cast<int>(i % P.tpu);
      const int nt = static_cast<int>(unit_end - i);
      m_run = -INFINITY;
      l_run = 0.f;
      for (int t = 0; t < nt; ++t, ++j) {
        const int kt = kt0 + t;
        mbar_wait(&s_full[sub], static_cast<uint32_t>(j & 1));
        tc_fence_after();
        if (r == 0) G2_EVT(2 * sub, j);
        if (dts && r == 0 && sub == 0 && j == 0) dts[2] = global_timer_ns();
        if (G2_NO_SOFTMAX) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[sub]);
          if (r == 0) G2_EVT(2 * sub + 1, j);
          continue;
        }
        float x[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld_32x32b<32>(s_addr + c * 32, v);
#pragma unroll
          for (int e = 0; e < 32; ++e) x[c * 32 + e] = v[e];
        }
        tmem_wait_ld();
        if (r == 0) G2_EVT(10 + 4 * sub, j);
        const int valid = min(RB_KEY_TILE, P.s - kt * RB_KEY_TILE);
        if (valid < RB_KEY_TILE) {
          // the prefix's last, partial tile only: masked keys get p = 0
#pragma unroll
          for (int c = 0; c < 128; ++c) x[c] = c < valid ? x[c] : -INFINITY;
        }
        // row max on the raw scores (the scale is positive), 4 chains
        float m4[4] = {x[0], x[1], x[2], x[3]};
#pragma unroll
        for (int c = 4; c < 128; c += 4) {
#pragma unroll
          for (int e = 0; e < 4; ++e) m4[e] = fmaxf(m4[e], x[c + e]);
        }
        const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * args.scale_log2;
        if (RB_DIAG && evt) asm volatile("" ::"f"(mx));
        if (r == 0) G2_EVT(11 + 4 * sub, j);
        const bool move = mx > m_run + kTau;
        const float m_new = move ? mx : m_run;
        const float al = (!move || m_run == -INFINITY) ? (move ? 0.f : 1.f) : fast_exp2(m_run - m_new);
        // P row: p = exp2(s * scale - m), one FFMA + one MUFU per score,
        // packed bf16 pairs (lower half = even key) into S's first 64 columns
        const float mu = (m_new == -INFINITY) ? 0.f : m_new;
        const float2 sl2 = make_float2(args.scale_log2, args.scale_log2);
        const float2 nmu2 = make_float2(-mu, -mu);
        float2 l2a = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float2 a2 = ffma2(make_float2(x[c * 32 + e], x[c * 32 + e + 1]), sl2, nmu2);
            float p0, p1;
            if (G2_POLY > 0 && (e >> 1) % (G2_POLY > 0 ? G2_POLY : 1) == G2_POLY - 1) {
              const float2 pp = exp2_poly2(a2);
              p0 = pp.x;
              p1 = pp.y;
            } else {
              p0 = fast_exp2(a2.x);
              p1 = fast_exp2(a2.y);
            }
            if (e & 2)
              l2b = fadd2(l2b, make_float2(p0, p1));
            else
              l2a = fadd2(l2a, make_float2(p0, p1));
            pk[e >> 1] = pack_bf16x2(p0, p1);
          }
          tmem_st16_u32(s_addr + c * 16, pk);
        }
        if (r == 0) G2_EVT(12 + 4 * sub, j);
        l_run = l_run * al + (l2a.x + l2a.y) + (l2b.x + l2b.y);
        m_run = m_new;
        if (__any_sync(0xffffffffu, move) && t > 0) {
          // O row *= al once P(j-1).V has landed (al = 1 for rows that did
          // not move); P(j).V waits for this warp's p_full arrival below
          mbar_wait(&o_full[sub], static_cast<uint32_t>((j - 1) & 1));
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float o[32];
            tmem_ld_32x32b<32>(o_addr + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= al;
            tmem_st_32x32b<32>(o_addr + c * 32, o);
          }
        }
        tmem_wait_st();
        if (r == 0) G2_EVT(13 + 4 * sub, j);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sub]);
        if (r == 0) G2_EVT(2 * sub + 1, j);
      }
      // ---- unit end: O row from TMEM after the unit's last P.V
      const int jl = j - 1;
      mbar_wait(&o_full[sub], static_cast<uint32_t>(jl & 1));
      tc_fence_after();
      if (dts && r == 0 && sub == 0) dts[3] = global_timer_ns();
      const int h = u / P.n_qt, qt = u % P.n_qt;
      const int f = qt * kUnitRows + ur;
      const bool row_ok = f < P.rows_per_head;
      const int nparts = rb_unit_parts(&P, u);
      const int slot = blockIdx.x - rb_unit_owner0(&P, u);
      const long long pbase = static_cast<long long>(u) * P.max_parts + slot;
      const bool to_part = args.defer_merge || nparts > 1;
      float* pacc = args.part_acc + (pbase * kUnitRows + ur) * RB_HEAD_DIM;
      float* pml = args.part_ml + pbase * 2 * kUnitRows;
      long long o_idx = 0;
      if (row_ok) o_idx = static_cast<long long>(f / P.g) * P.hq + h * P.g + f % P.g;
      const float inv = 1.f / l_run;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float o[32];
        tmem_ld_32x32b<32>(o_addr + c * 32, o);
        tmem_wait_ld();
        // each thread stores its own row: 32-byte stores (whole sectors);
        // float4 stores took ~4.6 us per CTA for a unit's 128 KB part
        if (to_part) {
#pragma unroll
          for (int e = 0; e < 32; e += 8)
            st_global_v8(pacc + c * 32 + e, o[e], o[e + 1], o[e + 2], o[e + 3], o[e + 4], o[e + 5], o[e + 6],
                         o[e + 7]);
        } else if (row_ok) {
#pragma unroll
          for (int e = 0; e < 32; e += 8)
            st_global_v8(args.o_sys + o_idx * RB_HEAD_DIM + c * 32 + e, o[e] * inv, o[e + 1] * inv,
                         o[e + 2] * inv, o[e + 3] * inv, o[e + 4] * inv, o[e + 5] * inv, o[e + 6] * inv,
                         o[e + 7] * inv);
        }
      }
      tc_fence_before();
      if (to_part) {
        pml[ur] = m_run;
        pml[kUnitRows + ur] = l_run;
      } else if (row_ok) {
        args.lse_sys[o_idx] = (m_run + __log2f(l_run)) * kLn2;
      }
      if (dts && r == 0 && sub == 0) dts[4] = global_timer_ns();
      if (args.defer_merge) {
        if (args.counters != nullptr) {
          named_bar_sync(bar_id, bar_n);  // every row's part written
          if (warp == kSmWarp0 && lane == 0) {
            __threadfence();
            atomicAdd(&args.counters[u], 1);
          }
        }
      }
      // (split units always defer: rb_system_attention merges their parts in
      // a separate launch, sys_merge_parts_kernel)
      i = unit_end;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
  if (dts && threadIdx.x == 0) dts[7] = global_timer_ns();
}

cudaError_t launch_system_attention_gqa2(const CUtensorMap& tk, const CUtensorMap& tv,
                                         const CUtensorMap& tq, const SysArgs& a,
                                         cudaStream_t stream) {
  static_assert(g2::kBytes <= 232448, "GQA2 system kernel shared memory over the 227 KB limit");
  cudaError_t e = cudaFuncSetAttribute(sys_gqa2_sm100_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, g2::kBytes);
  if (e != cudaSuccess) return e;
  e = launch_pdl(sys_gqa2_sm100_kernel, dim3(a.plan.grid), dim3(g2::kThreads), g2::kBytes, stream,
                 tk, tv, tq, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace rb
