// System-prompt attention for many query rows per KV head (GQA groups x large
// batches: C4 has 512, C5 2048 rows per KV head) on sm_100a.
//
// Same computation as sys_attn_sm100.cu -- the reference's `_system_attention`
// (attention.py:177-200): one unmasked attention pass of every flattened query
// row over the shared prefix, with natural-log LSE -- but in the
// non-swapped orientation, because with >= 128 rows per KV head the query
// rows fill the MMA M dimension by themselves:
//     S[128 q x 128 keys] = Q_tile . K_tile^T          (both K-major, SW128)
//     O[128 q x 128 d]   += P[128 q x 128 keys] . V_tile   (V MN-major, in place)
// so one 128x128 tile pair carries 4x the work of the swap-AB kernel's
// 128-key x 32-query tile, and the softmax is row-local: thread r of the
// softmax warpgroup owns TMEM lane r = query row r, holds its 128 scores in
// registers, and needs no cross-thread max / sum reductions.
//
// Roles (256 threads): warp 0 K TMA producer + Q rows (cp.async), warp 1 MMA
// issuer (Q.K^T of tile j+1 is issued before P.V of tile j) + TMEM owner,
// warp 2 V TMA producer, warps 4-7 softmax / epilogue.  TMEM: S x 2, O.
// Lazy max (tau = 8, log2 units) per row: the O row in TMEM is rescaled only
// when its running max moves by more than tau, after the previous P.V.
// Work split, parts, relay publication: as the swap-AB kernel (rb_plan.h,
// nq = 128).
#include "rb_common.cuh"
#include "rb_plan.h"
#include "rb_args.cuh"

namespace rb {

namespace gqa {

constexpr int kRows = 128;                 // query rows per tile (MMA M)
constexpr int kTile = RB_KEY_TILE * RB_HEAD_DIM * 2;  // 32 KB K or V tile
#ifndef GQA_KS
#define GQA_KS 2
#endif
#ifndef GQA_VS
#define GQA_VS 2
#endif
#ifndef GQA_NP
#define GQA_NP 1
#endif
#ifndef GQA_EXP_EARLY
#define GQA_EXP_EARLY 1
#endif
constexpr int KS = GQA_KS, VS = GQA_VS;
constexpr int NP = GQA_NP;                 // P buffers (1: P.V(j-1) gates the softmax of tile j)
constexpr int kQBytes = kRows * 256;       // [2 kblocks][128 rows][128 B]
constexpr int kOffK = 0;
constexpr int kOffV = kOffK + KS * kTile;
constexpr int kOffQ = kOffV + VS * kTile;
constexpr int kOffP = kOffQ + kQBytes;
constexpr int kOffBar = kOffP + NP * kQBytes;
constexpr int kNumBars = 2 * KS + 2 * VS + 10 + 2 * NP;
constexpr int kOffMisc = kOffBar + kNumBars * 8;
constexpr int kBytes = kOffMisc + 64;
constexpr int kThreads = 256;
constexpr int kSmWarp0 = 4;                // first softmax warp
constexpr uint32_t kTmemCols = 512;        // S0 [0,128), S1 [128,256), O [256,384)
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

}  // namespace gqa

__global__ void __launch_bounds__(gqa::kThreads, 1)
    sys_gqa_sm100_kernel(const __grid_constant__ CUtensorMap tmap_k,
                         const __grid_constant__ CUtensorMap tmap_v,
                         const __grid_constant__ CUtensorMap tmap_q, const SysArgs args) {
  using namespace gqa;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* k_full = bars;
  uint64_t* k_empty = bars + KS;
  uint64_t* v_full = bars + 2 * KS;
  uint64_t* v_empty = bars + 2 * KS + VS;
  uint64_t* s_full = bars + 2 * KS + 2 * VS;  // [2]
  uint64_t* s_empty = s_full + 2;             // [2]
  uint64_t* o_full = s_full + 4;              // [2], P.V(j) -> [j & 1]
  uint64_t* p_full = s_full + 6;              // [NP]
  uint64_t* p_empty = p_full + NP;            // [NP]
  uint64_t* q_full = p_empty + NP;
  uint64_t* q_empty = q_full + 1;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kOffMisc);

  const rb_sys_plan& P = args.plan;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  long long t_begin, t_end;
  rb_cta_range(&P, blockIdx.x, &t_begin, &t_end);

  if (warp == 0) {
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
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
      mbar_init(&o_full[i], 1);
    }
    for (int i = 0; i < NP; ++i) {
      mbar_init(&p_full[i], 4);
      mbar_init(&p_empty[i], 1);
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
  const uint32_t smem_p = smem_u32(smem + kOffP);

  if (warp == 0) {
    // ------------------------------------------------- K producer (+ Q rows)
    const uint64_t pol = l2_policy_evict_first();
    int j = 0, uq = 0;
    Walk w;
    w.start(P, blockIdx.x, t_begin);
    for (long long i = t_begin; i < t_end; ++i, ++j) {
      w.next(P);
      const int h = w.u / P.n_qt, qt = w.u % P.n_qt;
      const int st = j % KS;
      mbar_wait(&k_empty[st], ((j / KS) & 1) ^ 1);
      if (lane == 0) {
        uint8_t* dst = smem + kOffK + st * kTile;
        mbar_arrive_expect_tx(&k_full[st], kTile);
        tma_load_3d(dst, &tmap_k, &k_full[st], 0, w.kt * RB_KEY_TILE, h, pol);
        tma_load_3d(dst + kTile / 2, &tmap_k, &k_full[st], 64, w.kt * RB_KEY_TILE, h, pol);
      }
      __syncwarp();
      if (i == t_begin || w.kt == 0) {
        // the unit's 128 query rows (zero past the last row), K-major SW128
        mbar_wait(q_empty, (uq & 1) ^ 1);
        uint8_t* qdst = smem + kOffQ;
        if (args.q_tma) {
          // q in device memory, g | 128: two (64 d, g heads, 128 / g requests) boxes
          if (lane == 0) {
            mbar_arrive_expect_tx(q_full, kRows * 256);
            tma_load_3d(qdst, &tmap_q, q_full, 0, h * P.g, qt * kRows / P.g, pol);
            tma_load_3d(qdst + kRows * 128, &tmap_q, q_full, 64, h * P.g, qt * kRows / P.g, pol);
          }
          __syncwarp();
        } else {
          load_unit_q<kRows, kRows>(qdst, args, h, qt * kRows, lane);
          cp_async_wait_all();
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(q_full);
        }
        ++uq;
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ V producer
    const uint64_t pol = l2_policy_evict_first();
    if (lane == 0) {
      int j = 0;
      Walk w;
      w.start(P, blockIdx.x, t_begin);
      for (long long i = t_begin; i < t_end; ++i, ++j) {
        w.next(P);
        const int h = w.u / P.n_qt;
        const int st = j % VS;
        mbar_wait(&v_empty[st], ((j / VS) & 1) ^ 1);
        uint8_t* dst = smem + kOffV + st * kTile;
        mbar_arrive_expect_tx(&v_full[st], kTile);
        tma_load_3d(dst, &tmap_v, &v_full[st], 0, w.kt * RB_KEY_TILE, h, pol);
        tma_load_3d(dst + kTile / 2, &tmap_v, &v_full[st], 64, w.kt * RB_KEY_TILE, h, pol);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Q.K^T of tile j+1 goes out before P.V of tile j, so the softmax of
    // tile j+1 can start as soon as that of tile j is done.
    if (lane == 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16_f32(128, 128, 0, 1);
      const int n = static_cast<int>(t_end - t_begin);
      Walk wq, wp;
      wq.start(P, blockIdx.x, t_begin);
      wp.start(P, blockIdx.x, t_begin);
      int uq = 0;
      auto issue_qk = [&](int j) {
        wq.next(P);
        const bool first = (j == 0) || wq.kt == 0;
        const bool last = (j == n - 1) || wq.kt == P.tpu - 1;
        if (first) mbar_wait(q_full, uq & 1);
        const int st = j % KS, sb = j & 1;
        mbar_wait(&k_full[st], (j / KS) & 1);
        mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_base = smem_k + st * kTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk & 3) * 32;
          const uint64_t a = make_smem_desc_sw128(smem_q + (kk >> 2) * (kRows * 128) + koff, 16, 1024);
          const uint64_t b = make_smem_desc_sw128(k_base + (kk >> 2) * (kTile / 2) + koff, 16, 1024);
          umma_f16_ss(tmem_base + sb * 128, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        umma_commit(&k_empty[st]);
        if (last) {
          umma_commit(q_empty);
          ++uq;
        }
      };
      if (n > 0) issue_qk(0);
      for (int j = 0; j < n; ++j) {
        if (j + 1 < n) issue_qk(j + 1);
        wp.next(P);
        const uint32_t acc0 = (j > 0 && wp.kt != 0) ? 1u : 0u;
        const int st = j % VS;
        mbar_wait(&v_full[st], (j / VS) & 1);
        mbar_wait(&p_full[j % NP], static_cast<uint32_t>((j / NP) & 1));
        tc_fence_after();
        const uint32_t v_base = smem_v + st * kTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          // A = P (K-major, 16 keys); B = V tile, MN-major: 16 keys = two
          // 8-key swizzle atoms, the two 64-wide d halves kTile / 2 apart
          const uint64_t a =
              make_smem_desc_sw128(smem_p + (j % NP) * kQBytes + (kk >> 2) * (kRows * 128) + (kk & 3) * 32, 16, 1024);
          const uint64_t b = make_smem_desc_sw128(v_base + kk * 2048, kTile / 2, 1024);
          umma_f16_ss(tmem_base + 256, a, b, idesc_pv, kk > 0 ? 1u : acc0);
        }
        umma_commit(&o_full[j & 1]);
        umma_commit(&v_empty[st]);
        umma_commit(&p_empty[j % NP]);
      }
    }
    __syncwarp();
  } else if (warp >= kSmWarp0) {
    // ----------------------------------------------------- softmax / epilogue
    const int r = (warp & 3) * 32 + lane;  // query row of the tile = TMEM lane
    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t o_addr = lane_addr + 256;
    pdl_wait_primary();  // partials / o_sys may still be read by the previous kernel
    float m_run = -INFINITY, l_run = 0.f;
    long long i = t_begin;
    int j = 0;
    int pend_u = -1;
    while (i < t_end) {
      const int u = rb_tile_unit(&P, blockIdx.x, i);
      const long long unit_end = min(t_end, (i / P.tpu + 1) * P.tpu);
      const int kt0 = static_cast<int>(i % P.tpu);
      const int nt = static_cast<int>(unit_end - i);
      m_run = -INFINITY;
      l_run = 0.f;
      for (int t = 0; t < nt; ++t, ++j) {
        const int kt = kt0 + t;
        const int sb = j & 1;
        mbar_wait(&s_full[sb], (j >> 1) & 1);
        tc_fence_after();
        float x[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float v[32];
          tmem_ld_32x32b<32>(lane_addr + sb * 128 + c * 32, v);
#pragma unroll
          for (int e = 0; e < 32; ++e) x[c * 32 + e] = v[e];
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
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
#if GQA_EXP_EARLY
        // probabilities first (packed bf16 in registers), with the reference
        // the row will have after this tile: the exponentials overlap the
        // P.V(j-1) that the P buffer and the O rescale must wait for
        const bool move = mx > m_run + kTau;
        const float m_new = move ? mx : m_run;
        const float al = (!move || m_run == -INFINITY) ? (move ? 0.f : 1.f) : fast_exp2(m_run - m_new);
        const float mu = (m_new == -INFINITY) ? 0.f : m_new;
        const float2 sl2 = make_float2(args.scale_log2, args.scale_log2);
        const float2 nmu2 = make_float2(-mu, -mu);
        float2 l2a = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
        uint32_t pk32[64];
#pragma unroll
        for (int e = 0; e < 128; e += 2) {
          const float2 a2 = ffma2(make_float2(x[e], x[e + 1]), sl2, nmu2);
          const float p0 = fast_exp2(a2.x), p1 = fast_exp2(a2.y);
          if (e & 2)
            l2b = fadd2(l2b, make_float2(p0, p1));
          else
            l2a = fadd2(l2a, make_float2(p0, p1));
          pk32[e >> 1] = pack_bf16x2(p0, p1);
        }
        const int pb = j % NP;
        mbar_wait(&p_empty[pb], static_cast<uint32_t>(((j / NP) & 1) ^ 1));
        tc_fence_after();
        if (__any_sync(0xffffffffu, move) && t > 0) {
          if (NP > 1) {
            mbar_wait(&o_full[(j - 1) & 1], static_cast<uint32_t>(((j - 1) >> 1) & 1));
            tc_fence_after();
          }
          // O row *= al (al = 1 for rows that did not move)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float o[32];
            tmem_ld_32x32b<32>(o_addr + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= al;
            tmem_st_32x32b<32>(o_addr + c * 32, o);
          }
          tmem_wait_st();
        }
        l_run *= al;
        m_run = m_new;
        uint8_t* prow = smem + kOffP + pb * kQBytes;
#pragma unroll
        for (int ch = 0; ch < 16; ++ch) {
          uint4 pk;
          pk.x = pk32[ch * 4 + 0];
          pk.y = pk32[ch * 4 + 1];
          pk.z = pk32[ch * 4 + 2];
          pk.w = pk32[ch * 4 + 3];
          *reinterpret_cast<uint4*>(prow + (ch >> 3) * (kRows * 128) + sw128_offset(r, (ch & 7) * 8)) = pk;
        }
#else
        // P buffer j % NP is free once P.V(j - NP) has read it (NP = 1: P.V(j-1)
        // has landed, so the O row may also be rescaled)
        const int pb = j % NP;
        mbar_wait(&p_empty[pb], static_cast<uint32_t>(((j / NP) & 1) ^ 1));
        tc_fence_after();
        const bool move = mx > m_run + kTau;
        if (__any_sync(0xffffffffu, move)) {
          const float mn = move ? mx : m_run;
          const float al = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - mn);
          if (t > 0) {
            if (NP > 1) {
              // rescale after P.V(j-1): o_full alternates by tile and
              // P.V(j-3) is known complete, so the parity wait is unambiguous
              mbar_wait(&o_full[(j - 1) & 1], static_cast<uint32_t>(((j - 1) >> 1) & 1));
              tc_fence_after();
            }
            // O row *= al (rows that did not move use al = 1)
            const float a = move ? al : 1.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              float o[32];
              tmem_ld_32x32b<32>(o_addr + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] *= a;
              tmem_st_32x32b<32>(o_addr + c * 32, o);
            }
            tmem_wait_st();
          }
          if (move) {
            l_run *= al;
            m_run = mn;
          }
        }
        // P row (bf16, K-major SW128: row r, two 64-key halves):
        // p = exp2(s * scale - m), one FFMA + one MUFU per score
        const float mu = (m_run == -INFINITY) ? 0.f : m_run;
        const float2 sl2 = make_float2(args.scale_log2, args.scale_log2);
        const float2 nmu2 = make_float2(-mu, -mu);
        float2 l2a = make_float2(0.f, 0.f), l2b = make_float2(0.f, 0.f);
        uint8_t* prow = smem + kOffP + pb * kQBytes;
#pragma unroll
        for (int ch = 0; ch < 16; ++ch) {
          float p[8];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const float2 a = ffma2(make_float2(x[ch * 8 + e], x[ch * 8 + e + 1]), sl2, nmu2);
            p[e] = fast_exp2(a.x);
            p[e + 1] = fast_exp2(a.y);
            if (e & 2)
              l2b = fadd2(l2b, make_float2(p[e], p[e + 1]));
            else
              l2a = fadd2(l2a, make_float2(p[e], p[e + 1]));
          }
          uint4 pk;
          pk.x = pack_bf16x2(p[0], p[1]);
          pk.y = pack_bf16x2(p[2], p[3]);
          pk.z = pack_bf16x2(p[4], p[5]);
          pk.w = pack_bf16x2(p[6], p[7]);
          *reinterpret_cast<uint4*>(prow + (ch >> 3) * (kRows * 128) + sw128_offset(r, (ch & 7) * 8)) = pk;
        }
#endif
        const float ls = (l2a.x + l2a.y) + (l2b.x + l2b.y);
        l_run += ls;
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
        if (pend_u >= 0 && (t > 0 || t == nt - 1)) {
          // publish the previous unit's part once its stores have drained
          if (warp == kSmWarp0 && lane == 0) {
            __threadfence();
            atomicAdd(&args.counters[pend_u], 1);
          }
          pend_u = -1;
        }
      }
      // ---- unit end: O row from TMEM after the unit's last P.V
      const int jl = j - 1;
      mbar_wait(&o_full[jl & 1], static_cast<uint32_t>((jl >> 1) & 1));
      tc_fence_after();
      const int h = u / P.n_qt, qt = u % P.n_qt;
      const int f = qt * kRows + r;
      const bool row_ok = f < P.rows_per_head;
      const int nparts = rb_unit_parts(&P, u);
      const int slot = blockIdx.x - rb_unit_owner0(&P, u);
      const long long pbase = static_cast<long long>(u) * P.max_parts + slot;
      const bool to_part = args.defer_merge || nparts > 1;
      float* pacc = args.part_acc + (pbase * kRows + r) * RB_HEAD_DIM;
      float* pml = args.part_ml + pbase * 2 * kRows;
      long long o_idx = 0;
      if (row_ok) o_idx = static_cast<long long>(f / P.g) * P.hq + h * P.g + f % P.g;
      const float inv = 1.f / l_run;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float o[32];
        tmem_ld_32x32b<32>(o_addr + c * 32, o);
        tmem_wait_ld();
        // each thread stores its own row: 32-byte stores (whole sectors)
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
        pml[r] = m_run;
        pml[kRows + r] = l_run;
      } else if (row_ok) {
        args.lse_sys[o_idx] = (m_run + __log2f(l_run)) * kLn2;
      }
      if (args.defer_merge) {
        if (args.counters != nullptr) {
          named_bar_sync(1, 128);  // every row's part written
          pend_u = u;
        }
      }
      // (split units always defer: rb_system_attention merges their parts in
      // a separate launch, sys_merge_parts_kernel)
      i = unit_end;
    }
    if (pend_u >= 0 && warp == kSmWarp0 && lane == 0) {
      __threadfence();
      atomicAdd(&args.counters[pend_u], 1);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

cudaError_t launch_system_attention_gqa(const CUtensorMap& tk, const CUtensorMap& tv,
                                        const CUtensorMap& tq, const SysArgs& a, cudaStream_t stream) {
  static_assert(gqa::kBytes <= 232448, "GQA system kernel shared memory over the 227 KB limit");
  cudaError_t e = cudaFuncSetAttribute(sys_gqa_sm100_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, gqa::kBytes);
  if (e != cudaSuccess) return e;
  e = launch_pdl(sys_gqa_sm100_kernel, dim3(a.plan.grid), dim3(gqa::kThreads), gqa::kBytes, stream,
                 tk, tv, tq, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace rb
