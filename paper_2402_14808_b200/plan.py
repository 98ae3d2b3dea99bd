"""Python mirror of the relay step's stream-K plan of the system tiles
(csrc/rb_plan.h) and of its context-unit numbering.

Used by host-logic tests (no GPU needed) and by DESIGN.md's worked
examples; the kernels compute the same integers on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

KEY_TILE = 128


def pick_nq(rows_per_head: int) -> int:
    return 16 if rows_per_head <= 16 else 32


@dataclass(frozen=True)
class SysPlan:
    n_rows: int
    hq: int
    hkv: int
    s: int
    grid_cap: int

    @property
    def g(self):
        return self.hq // self.hkv

    @property
    def rows_per_head(self):
        return self.n_rows * self.g

    @property
    def nq(self):
        return pick_nq(self.rows_per_head)

    @property
    def n_qt(self):
        return -(-self.rows_per_head // self.nq)

    @property
    def tpu(self):
        return -(-self.s // KEY_TILE)

    @property
    def n_units(self):
        return self.hkv * self.n_qt

    @property
    def total(self):
        return self.n_units * self.tpu

    @property
    def grid(self):
        return max(1, min(self.total, self.grid_cap))

    def cta_begin(self, c):
        return c * self.total // self.grid

    def owner(self, x):
        return ((x + 1) * self.grid - 1) // self.total

    def unit_parts(self, u):
        first = u * self.tpu
        return self.owner(first + self.tpu - 1) - self.owner(first) + 1

    @property
    def max_parts(self):
        return max(self.unit_parts(u) for u in range(self.n_units))

    def cta_ranges(self):
        return [(self.cta_begin(c), self.cta_begin(c + 1)) for c in range(self.grid)]


def context_units(q_rows, g, hkv, nq):
    """Per-request unit prefix U (U[r] = context units before request r) for
    query counts q_rows[r]: hkv * ceil(m_r * g / nq) units per request.
    Context unit v of the relay step is (request r, kv head, q-tile) with
    U[r] <= v < U[r+1]; each CTA's scheduler hands them out dynamically."""
    U = [0]
    for m in q_rows:
        U.append(U[-1] + hkv * (-(-m * g // nq)))
    return U
