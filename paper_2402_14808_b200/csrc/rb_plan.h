// Work decomposition of the system-prompt attention kernel, shared by host
// and device (and mirrored in Python by paper_2402_14808_b200/plan.py).
//
// Units.  One unit = (kv head h, query tile qt): the query rows of KV head h
// are the n_rows * g (request-row, group-member) pairs, cut into tiles of
// `nq` rows.  Each unit streams the whole shared prefix of its head in key
// tiles of 128 keys, so the flattened iteration space is
//     global tile i  ->  unit u = i / tpu, key tile kt = i % tpu,
//     total = n_units * tpu.
// Stream-K split.  CTA c of `grid` CTAs owns the contiguous global tile range
// [c*total/grid, (c+1)*total/grid).  A unit cut by CTA boundaries is
// finished by several CTAs; CTA c writes partial slot c - owner(first tile
// of u), and the last CTA to finish (per-unit semaphore) merges the slots in
// slot order, so the result is deterministic.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define RB_HD __host__ __device__ __forceinline__
#else
#define RB_HD static inline
#endif

#define RB_KEY_TILE 128
#define RB_HEAD_DIM 128

typedef struct {
  int n_rows;         // flattened query rows (sum of m_r over requests)
  int hq, hkv, g;     // query heads, kv heads, group size hq / hkv
  int s;              // shared prefix length (keys)
  int nq;             // query rows per unit (16, 32, 128 or 256)
  int rows_per_head;  // n_rows * g
  int n_qt;           // ceil(rows_per_head / nq)
  int tpu;            // key tiles per unit, ceil(s / 128)
  int n_units;        // hkv * n_qt
  long long total;    // n_units * tpu
  int grid;           // CTAs launched
  int max_parts;      // max partial slots over all units
  int rr;             // 1: whole units dealt round-robin (CTA c: units c, c+grid, ...)
  unsigned long long total_magic;  // ceil(2^64 / total) (0 when total == 1): owner by multiply-high
} rb_sys_plan;

// The stream-K index math runs in 32-bit unsigned arithmetic: plans keep
// total * grid < 2^32 (RB_PLAN_MAX_PRODUCT; rb_sys_plan_query rejects larger
// ones -- e.g. 64 units x 8192 key tiles x 148 CTAs is 7.8e7).  The 64-bit
// divisions it replaces were ~1400 instructions of the context kernel's code
// (inlined at every relay site), whose per-item path is sensitive to its
// instruction footprint.
#define RB_PLAN_MAX_PRODUCT 4294967295LL
RB_HD long long rb_cta_begin(const rb_sys_plan* p, int c) {
  return (long long)(((unsigned)c * (unsigned)p->total) / (unsigned)p->grid);
}
// CTA owning global tile x (stream-K mode): floor(((x + 1) grid - 1) / total)
// -- on the device as a multiply-high by ceil(2^64 / total), exact for
// numerators below 2^32 (the relay sites inline it several times; a 32-bit
// division is ~20 instructions, this is ~4)
RB_HD int rb_tile_owner(const rb_sys_plan* p, long long x) {
  const unsigned n = (unsigned)(x + 1) * (unsigned)p->grid - 1u;
#ifdef __CUDA_ARCH__
  return p->total_magic ? (int)__umul64hi((unsigned long long)n, p->total_magic) : (int)n;
#else
  return (int)(n / (unsigned)p->total);
#endif
}
RB_HD int rb_unit_parts(const rb_sys_plan* p, int u) {
  if (p->rr) return 1;
  long long first = (long long)u * p->tpu;
  long long last = first + p->tpu - 1;
  return rb_tile_owner(p, last) - rb_tile_owner(p, first) + 1;
}
// Tiles of CTA c, as a local index range [*b, *e): stream-K mode uses global
// tile indices; round-robin mode numbers the CTA's own units' tiles from 0.
// Both are unit-aligned: a unit starts wherever i % tpu == 0 (or at *b).
RB_HD void rb_cta_range(const rb_sys_plan* p, int c, long long* b, long long* e) {
  if (p->rr) {
    const int mine = c < p->n_units ? (p->n_units - 1 - c) / p->grid + 1 : 0;
    *b = 0;
    *e = (long long)mine * p->tpu;
  } else {
    *b = rb_cta_begin(p, c);
    *e = rb_cta_begin(p, c + 1);
  }
}
// Unit of tile i of CTA c (i from rb_cta_range).
RB_HD int rb_tile_unit(const rb_sys_plan* p, int c, long long i) {
  return p->rr ? c + (int)((unsigned)i / (unsigned)p->tpu) * p->grid : (int)((unsigned)i / (unsigned)p->tpu);
}
// First CTA holding a part of unit u (its part slot is 0).
RB_HD int rb_unit_owner0(const rb_sys_plan* p, int u) {
  return p->rr ? u % p->grid : rb_tile_owner(p, (long long)u * p->tpu);
}

// Query rows per tile: the swap-AB kernel takes 16 / 32 (N of the MMA); from
// 128 rows per KV head on, the non-swapped kernel (sys_gqa_sm100.cu) takes
// 128-row tiles (M of the MMA); from 256 on, sys_gqa2_sm100.cu takes units of
// two 128-row tiles that share each K/V tile (two softmax warpgroups).
RB_HD int rb_pick_nq(int rows_per_head) {
  return rows_per_head <= 16 ? 16 : rows_per_head < 128 ? 32 : rows_per_head < 256 ? 128 : 256;
}

// Fill a plan. grid_cap = number of CTAs the device can hold at once
// (SM count for this one-CTA-per-SM kernel).
RB_HD void rb_make_sys_plan(rb_sys_plan* p, int n_rows, int hq, int hkv, int s,
                            int grid_cap) {
  p->n_rows = n_rows;
  p->hq = hq;
  p->hkv = hkv;
  p->g = hq / hkv;
  p->s = s;
  p->rows_per_head = n_rows * p->g;
  p->nq = rb_pick_nq(p->rows_per_head);
  p->n_qt = (p->rows_per_head + p->nq - 1) / p->nq;
  p->tpu = (s + RB_KEY_TILE - 1) / RB_KEY_TILE;
  p->n_units = hkv * p->n_qt;
  p->total = (long long)p->n_units * p->tpu;
  p->total_magic = p->total > 1 ? ~0ULL / (unsigned long long)p->total + 1ULL : 0ULL;
  long long gcap = grid_cap < 1 ? 1 : grid_cap;
  // Several query tiles per KV head (large GQA batches): deal whole units
  // round-robin, so the CTAs working on a head's query tiles at the same
  // moment walk its key tiles in lockstep and every re-read of a tile comes
  // from L2 instead of HBM.  Otherwise stream-K over the flattened tiles.
  // Only when whole units fill the CTAs in even waves (>= 85% busy):
  // otherwise a few CTAs would run one unit more than the rest.
  const long long waves = (p->n_units + gcap - 1) / gcap;
  p->rr = (p->n_qt >= 2 && 100LL * p->n_units >= 85LL * waves * gcap) ? 1 : 0;
  if (p->rr) {
    p->grid = (int)((p->n_units + waves - 1) / waves);
  } else if (p->n_qt >= 2 && p->n_units <= gcap &&
             100LL * p->n_units * (gcap / p->n_units) >= 85LL * gcap) {
    // several query tiles per KV head, fewer units than CTAs: an equal
    // number of CTAs per unit (if that keeps >= 85% of them), so each CTA
    // holds one aligned key range of one unit and the CTAs on a head's query
    // tiles stream the same key tiles at the same time (re-reads from L2)
    p->grid = (int)(p->n_units * (gcap / p->n_units));
    if ((long long)p->grid > p->total) p->grid = (int)p->total;
  } else {
    p->grid = (int)(p->total < gcap ? p->total : gcap);
  }
  int mp = 1;
  for (int u = 0; u < p->n_units; ++u) {
    int c = rb_unit_parts(p, u);
    if (c > mp) mp = c;
  }
  p->max_parts = mp;
}

// SM split of the concurrent relay step (rb_relay_attention): the system
// kernel gets a share of the SMs proportional to its HBM bytes weighted by
// the per-SM streaming rates of the two kernels (each query tile of a KV
// head streams the whole prefix), the context kernel the rest plus every SM
// the system kernel releases, so both finish together.
// RB_RELAY_RATE_RATIO = (system bytes/s per SM) / (context bytes/s per SM),
// fit on B200 with profiles/sweep_split.py to the best splits at s = 4k..32k
// (profiles/r02/sweep_split.txt: 60 / 90 / ~106 / ~115 system CTAs).
#define RB_RELAY_RATE_RATIO 1.3
#define RB_GQA2_TILE_US 2.0   /* sys_gqa2: one 128-key tile for 256 query rows */
#define RB_CTX_SM_GBS 38.0    /* context kernel streaming rate per SM (1-2 rows per item) */
#define RB_CTX_SM_GBS_GQA 50.0 /* ... with >= 4 rows per item (C4 measured 52) */
RB_HD int rb_relay_split(int n_rows, int hq, int hkv, int s, long long ctx_tokens, int sms) {
  rb_sys_plan p;
  rb_make_sys_plan(&p, n_rows, hq, hkv, s, sms);
  const double sys_bytes = (double)p.n_qt * hkv * (double)s * 512.0;
  const double ctx_bytes = (double)ctx_tokens * hkv * 512.0;
  // the context kernel streams long per-request contexts faster per SM than
  // short ones (each (request, head) item pays a fixed latency chain): the
  // rate ratio falls from RB_RELAY_RATE_RATIO at <= 8 chunks of 16 tokens per
  // item to ~0.94 at >= 32 (C3, c ~ U[64, 768]: best split measured 36 CTAs
  // vs 29 with the flat ratio, 125 -> 108 us per layer; profiles/r02)
  const double avg_chunks = n_rows > 0 ? (double)ctx_tokens / n_rows / 16.0 : 0.0;
  double lf = (avg_chunks - 8.0) / 24.0;
  lf = lf < 0.0 ? 0.0 : (lf > 1.0 ? 1.0 : lf);
  const double ratio = RB_RELAY_RATE_RATIO / (1.0 + 0.39 * lf);
  int g = (int)(sms * sys_bytes / (sys_bytes + ratio * ctx_bytes) + 0.5);
  // 8-24 key tiles per system CTA: its fixed per-CTA cost (first S,
  // epilogues) weighs on its rate, so it gets a larger share (C2 s = 2048:
  // 41 -> 48 CTAs, 45.1 -> 43.0 us measured by profiles/sweep_split.py;
  // s = 4096 and up keep the byte balance; below 8 tiles per CTA -- C1 --
  // more CTAs measured no better)
  if (g > 0 && (double)p.total / g < 24.0 && (double)p.total / g >= 8.0) {
    const double r2 = 0.8 * ratio;
    g = (int)(sms * sys_bytes / (sys_bytes + r2 * ctx_bytes) + 0.5);
  }
  if (p.nq == 256 && p.n_units <= sms) {
    // the 256-row GQA kernel is tensor-bound: balance measured time, not
    // bytes -- RB_GQA2_TILE_US per key tile per CTA against the context
    // kernel's RB_CTX_SM_GBS(_GQA) per SM (profiles/r02), rounded to whole
    // multiples of the unit count (CTAs on a head's units share K/V in L2;
    // measured C4: 64 / 80 / 96 / 112 CTAs -> 157 / 137 / 134 / 212 us;
    // C5: 64 / 96 / 128 / 144 -> 1091 / 878 / 728 / 726 us)
    const double sys_work = (double)p.total * RB_GQA2_TILE_US;
    // context items of >= 4 query rows (GQA groups) share each K/V chunk
    // across the rows and stream faster per SM
    const double ctx_rate = p.g >= 4 ? RB_CTX_SM_GBS_GQA : RB_CTX_SM_GBS;
    const double ctx_work = ctx_bytes / (ctx_rate * 1e3);
    const double gt = sms * sys_work / (sys_work + ctx_work);
    int k = (int)(gt / p.n_units + 0.5);
    if (k < 1) k = 1;
    if (k * p.n_units > sms) k = sms / p.n_units;
    return k * p.n_units;
  }
  if (p.nq >= 128 && p.n_units <= sms) {
    // 128-row GQA kernel: whole multiples of the unit count, rounded down
    // (at least one CTA per unit), so the CTAs on a head's query tiles stay
    // aligned and share K/V in L2 (measured: C4 best at 2 CTAs per unit,
    // C5 at 1; misaligned splits lose 10-20%)
    const int k = g / p.n_units;
    g = (k < 1 ? 1 : k) * p.n_units;
    return g;
  }
  {
    // Round-robin plans (several query tiles per KV head, whole units per
    // CTA) can only take n_units / waves CTAs: rounding the byte balance to
    // one of them leaves the two kernels unbalanced.  Pick the wave count
    // with the shortest estimated step instead: the system kernel takes
    // waves x tpu key tiles per CTA; the context kernel streams on the other
    // SMs meanwhile and on all of them after.  (C3, c ~ U[64, 768], with the
    // context claimed longest first: 32 CTAs (2 waves) 3223 us per 32-layer
    // stack, 64 CTAs (1 wave) 3064 us; profiles/diag_c3_stack.py)
    rb_sys_plan pg;
    rb_make_sys_plan(&pg, n_rows, hq, hkv, s, g < 1 ? 1 : g);
    if (pg.rr) {
      const double rc = RB_CTX_SM_GBS * 1e3;  // context bytes per us per SM
      const double rs = ratio * rc;           // system bytes per us per SM
      const double tile_bytes = RB_KEY_TILE * 512.0;
      double best = 1e300;
      int bg = pg.grid;
      for (int w = 1; w <= 8 && w <= p.n_units; ++w) {
        const int gw = (p.n_units + w - 1) / w;
        if (gw >= sms) continue;
        rb_sys_plan pw;
        rb_make_sys_plan(&pw, n_rows, hq, hkv, s, gw);
        if (!pw.rr || pw.grid != gw) continue;
        const double t_sys = (double)w * p.tpu * tile_bytes / rs;
        const double done = (double)(sms - gw) * rc * t_sys;
        const double t = done >= ctx_bytes ? t_sys : t_sys + (ctx_bytes - done) / (sms * rc);
        if (t < best) {
          best = t;
          bg = gw;
        }
      }
      g = bg;
    }
  }
  // latency floor: with few key tiles per CTA the system kernel is bound by
  // its per-CTA pipeline (prologue + ~1.5 us per tile), not by bytes; the
  // measured optimum at s <= 2k keeps ~20% of the SMs on it
  const int floor_g = sms * 20 / 100;
  if (g < floor_g) g = floor_g;
  if ((long long)g > p.total) g = (int)p.total;
  if (g < 1) g = 1;
  if (g > sms) g = sms;
  return g;
}

// Context split-K (rb_context_attention / rb_relay_attention): the context
// kernel's work items are (request, kv head, row tile); with few of them
// (small batches, long contexts) one item would be streamed by one CTA while
// most SMs idle, so each item's 16-token chunks are cut into splits of
// `chunks` chunks (the last split of a request takes the remainder), combined
// in split order by the last split to finish (deterministic).
// max_chunks = prefix chunks + ceil(max context tokens / 16); resident =
// CTAs the context kernel keeps resident (2 per SM).  chunks == 0: no split.
#define RB_CTX_CHUNK 16
#define RB_CTX_SPLIT_MIN_CHUNKS 8   /* >= 2 chunks per worker warp */
RB_HD void rb_ctx_split(long long base_items, int max_chunks, int resident, int* chunks,
                        int* n_split) {
  *chunks = 0;
  *n_split = 1;
  if (base_items < 1 || max_chunks < 2 * RB_CTX_SPLIT_MIN_CHUNKS) return;
  if (base_items >= 2LL * resident) return;
  const long long want = (2LL * resident + base_items - 1) / base_items;   // splits per item
  int L = (int)((max_chunks + want - 1) / want);
  if (L < RB_CTX_SPLIT_MIN_CHUNKS) L = RB_CTX_SPLIT_MIN_CHUNKS;
  const int ns = (max_chunks + L - 1) / L;
  if (ns < 2) return;
  *chunks = L;
  *n_split = ns;
}

// rows per work item (R) and row tiles per (request, kv head) for a batch
// whose largest request has max_rows = m_r * g query rows per kv head
RB_HD int rb_ctx_rows(int max_rows) {
  return max_rows >= 8 ? 8 : max_rows >= 4 ? 4 : max_rows >= 2 ? 2 : 1;
}

// workspace bytes of the context split: partials [n_rows * hq][n_split][132]
// f32 + one counter per (request, kv head, row tile), 256-aligned sections
RB_HD long long rb_ctx_split_bytes(int b, int n_rows, int hq, int hkv, int max_rows, int n_split) {
  if (n_split < 2) return 0;
  const int R = rb_ctx_rows(max_rows);
  const long long n_z = (max_rows + R - 1) / R;
  const long long part = ((long long)n_rows * hq * n_split * 132 * 4 + 255) & ~255LL;
  const long long cnt = ((long long)b * hkv * n_z * 4 + 255) & ~255LL;
  return part + cnt;
}
