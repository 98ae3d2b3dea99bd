// Work decomposition of the relay step's system tiles, shared by host and
// device (and mirrored in Python by paper_2402_14808_b200/plan.py).
//
// Units.  One unit = (kv head h, query tile qt): the query rows of KV head h
// are the n_rows * g (request-row, group-member) pairs, cut into tiles of
// `nq` rows.  Each unit streams the whole shared prefix of its head in key
// tiles of 128 keys, so the flattened system tile space is
//     global tile i  ->  unit u = i / tpu, key tile kt = i % tpu,
//     total = n_units * tpu.
// Stream-K split (static, balanced to one tile).  CTA c of `grid` CTAs owns
// the system tiles [c*total/grid, (c+1)*total/grid); a unit cut by CTA
// boundaries is finished by several CTAs (its "parts"); CTA c writes part
// slot c - owner(first tile of u), and the merge reads the slots in order,
// so the result is deterministic.  The context units that follow are handed
// out dynamically by each CTA's scheduler warp (relay_step_sm100.cu), which
// absorbs whatever imbalance the static system split leaves.
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
  int nq;             // query rows per tile (16 or 32)
  int rows_per_head;  // n_rows * g
  int n_qt;           // ceil(rows_per_head / nq)
  int tpu;            // key tiles per unit, ceil(s / 128)
  int n_units;        // hkv * n_qt
  long long total;    // n_units * tpu
  int grid;           // CTAs sharing the system tiles
  int max_parts;      // max parts (CTAs) over all units
} rb_sys_plan;

RB_HD long long rb_cta_begin(const rb_sys_plan* p, int c) {
  return (long long)c * p->total / p->grid;
}
// CTA owning global tile x.
RB_HD int rb_tile_owner(const rb_sys_plan* p, long long x) {
  return (int)(((x + 1) * (long long)p->grid - 1) / p->total);
}
RB_HD int rb_unit_parts(const rb_sys_plan* p, int u) {
  long long first = (long long)u * p->tpu;
  long long last = first + p->tpu - 1;
  return rb_tile_owner(p, last) - rb_tile_owner(p, first) + 1;
}
