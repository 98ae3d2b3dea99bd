"""Python mirror of the system kernel's stream-K work plan (csrc/rb_plan.h).

Used by host-logic tests (no GPU needed) and by DESIGN.md's worked
examples; the kernels compute the same integers on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

KEY_TILE = 128


def pick_nq(rows_per_head: int) -> int:
    if rows_per_head <= 16:
        return 16
    if rows_per_head < 128:
        return 32
    return 128 if rows_per_head < 256 else 256


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
    def rr(self):
        """Whole units dealt round-robin (several query tiles per KV head, and
        whole units fill the CTAs in even waves, >= 85% busy): CTAs on a
        head's query tiles walk its key tiles in lockstep, so re-reads hit L2."""
        gcap = max(1, self.grid_cap)
        waves = -(-self.n_units // gcap)
        return self.n_qt >= 2 and 100 * self.n_units >= 85 * waves * gcap

    @property
    def grid(self):
        gcap = max(1, self.grid_cap)
        if self.rr:
            waves = -(-self.n_units // gcap)
            return -(-self.n_units // waves)
        if (self.n_qt >= 2 and self.n_units <= gcap
                and 100 * self.n_units * (gcap // self.n_units) >= 85 * gcap):
            # aligned split: gcap // n_units CTAs per unit (L2 lockstep)
            return min(self.n_units * (gcap // self.n_units), self.total)
        return max(1, min(self.total, gcap))

    def cta_begin(self, c):
        return c * self.total // self.grid

    def owner(self, x):
        return ((x + 1) * self.grid - 1) // self.total

    def unit_parts(self, u):
        if self.rr:
            return 1
        first = u * self.tpu
        return self.owner(first + self.tpu - 1) - self.owner(first) + 1

    @property
    def max_parts(self):
        return max(self.unit_parts(u) for u in range(self.n_units))

    def cta_units(self, c):
        """Round-robin mode: the units of CTA c, in processing order."""
        return list(range(c, self.n_units, self.grid))

    def cta_ranges(self):
        return [(self.cta_begin(c), self.cta_begin(c + 1)) for c in range(self.grid)]
