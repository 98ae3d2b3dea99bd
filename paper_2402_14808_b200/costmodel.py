"""Traffic / roofline model of the relay decode step.

The reference's analytic cost model (costmodel.py:21-163: element-count
closed forms, traffic report, GEMM intensity, ridge / roofline helpers,
speedup-curve CSV), kept for API compatibility, plus the physical byte model
the B200 roofline uses:

  B_alg   = e*2*H_kv*d*(s + sum_c) + e*2*b*H_q*d    shared KV once + context KV + Q + O
  B_naive = e*2*H_kv*d*(b*s + sum_c) + e*2*b*H_q*d  shared KV re-read per request
  F_sys   = 4*b*H_q*s*d,  F_ctx = 4*H_q*d*sum_c

Intermediates (fp32 system partials, LSEs, block tables) are NOT in B_alg;
`overhead_bytes` reports them separately.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

from .errors import ContractError, DimensionError


def _check(b, s, c, d):
    if b < 1 or d < 1 or s < 0 or c < 0:
        raise ContractError(f"need b >= 1, d >= 1, s >= 0, c >= 0; got b={b} s={s} c={c} d={d}")


def traffic_baseline(b, s, c, d):
    """costmodel.py:85-89: b*d*(s + c + 2) elements."""
    _check(b, s, c, d)
    return b * d * (s + c + 2)


def traffic_relay(b, s, c, d):
    """costmodel.py:92-96: d*(s + b*c + 7b) elements."""
    _check(b, s, c, d)
    return d * (s + b * c + 7 * b)


def theoretical_speedup(b, s, c):
    """costmodel.py:105-112: p = (s + c + 2) / (s/b + c + 7)."""
    _check(b, s, c, 1)
    return (s + c + 2) / (s / b + c + 7)


@dataclass(frozen=True)
class TrafficReport:
    """Element traffic of one decode step on both paths (costmodel.py:43-53)."""

    n_baseline: int
    n_relay: int
    speedup: float
    b: int
    s: int
    c: int
    d: int


def traffic_report(b, s, c, d):
    """costmodel.py:115-119: both closed forms and their ratio."""
    base, relay = traffic_baseline(b, s, c, d), traffic_relay(b, s, c, d)
    return TrafficReport(base, relay, base / relay, b, s, c, d)


@dataclass(frozen=True)
class GemmShape:
    """C = A @ B.T with A (m, k), B (n, k) (numerics.py:24-33)."""

    m: int
    n: int
    k: int

    def __post_init__(self):
        if min(self.m, self.n, self.k) < 1:
            raise DimensionError(f"GemmShape dimensions must be >= 1, got {self}")


def arithmetic_intensity_gemm(shape):
    """flop per byte of a bf16 GEMM with every operand moved once
    (costmodel.py:56-61): mnk / (mk + nk + mn)."""
    m, n, k = shape.m, shape.n, shape.k
    return (m * n * k) / (m * k + n * k + m * n)


def gemm_intensity_bound(shape):
    """min(m, n, k) bounds the GEMM intensity from above (costmodel.py:64-66)."""
    return min(shape.m, shape.n, shape.k)


@dataclass(frozen=True)
class DecodeShape:
    b: int
    hq: int
    hkv: int
    s: int
    ctx_total: int     # sum of context lengths
    d: int = 128
    e: int = 2         # bytes per element (bf16)
    m: int = 1         # new tokens per request

    @property
    def rows(self):
        return self.b * self.m

    @property
    def bytes_sys(self):
        return self.e * 2 * self.hkv * self.d * self.s

    @property
    def bytes_ctx(self):
        return self.e * 2 * self.hkv * self.d * self.ctx_total

    @property
    def bytes_qo(self):
        return self.e * 2 * self.rows * self.hq * self.d

    @property
    def bytes_alg(self):
        return self.bytes_sys + self.bytes_ctx + self.bytes_qo

    @property
    def bytes_naive(self):
        return self.e * 2 * self.hkv * self.d * (self.b * self.s + self.ctx_total) + self.bytes_qo

    @property
    def flops_sys(self):
        return 4 * self.rows * self.hq * self.s * self.d

    @property
    def flops_ctx(self):
        return 4 * self.m * self.hq * self.d * self.ctx_total

    @property
    def overhead_bytes(self):
        """fp32 system output written + read, LSEs, fused LSE."""
        return 2 * 4 * self.rows * self.hq * self.d + 4 * 3 * self.rows * self.hq

    def roofline_s(self, hbm_bytes_per_s, tensor_flops_per_s):
        """t* = max(B_alg/BW, F_sys/P_tc) (overlapped)."""
        return max(self.bytes_alg / hbm_bytes_per_s, self.flops_sys / tensor_flops_per_s)

    def shard(self, hkv_local, hq_local):
        return DecodeShape(self.b, hq_local, hkv_local, self.s, self.ctx_total, self.d, self.e,
                           self.m)


# ---------------------------------------------------------------- hardware
@dataclass(frozen=True)
class HardwareProfile:
    """Bandwidth / compute envelope of one accelerator (costmodel.py:21-33)."""

    name: str
    mem_bandwidth: float  # bytes / s
    peak_flops: float     # flop / s
    bytes_per_element: int = 2

    def __post_init__(self):
        if min(self.mem_bandwidth, self.peak_flops, self.bytes_per_element) <= 0:
            raise ContractError(f"profile fields must be positive: {self}")


# The reference's profiles (costmodel.py:36-40) plus B200 at the measured
# copy bandwidth and dense bf16 throughput of this pool (MEASURED_PEAKS.json).
HARDWARE_PROFILES = {
    "A40": HardwareProfile("A40", 696e9, 37.4e12),
    "A100-PCIE-40GB": HardwareProfile("A100-PCIE-40GB", 1555e9, 77.9e12),
    "A100-SXM4-80GB": HardwareProfile("A100-SXM4-80GB", 2039e9, 77.9e12),
    "B200": HardwareProfile("B200", 6539.9e9, 1647.2e12),
}

# Measured cost of this repository's relay decode step on one B200 (one
# layer, CUDA-graph replay, L2 flushed; profiles/r01g/r01g_bench.json): above
# ~2k prefix tokens the step is an affine function of its algorithmic bytes,
# t = B200_STEP_FIXED_S + B_alg / B200_STEP_MARGINAL_BPS (fit through the
# s = 8k and 32k points: 21.1 us + 6.9 TB/s); below, a latency floor.
B200_STEP_FIXED_S = 21.1e-6
B200_STEP_MARGINAL_BPS = 6.9e12
B200_STEP_FLOOR_S = 45.0e-6


def balance_ratio(profile):
    """Ridge intensity peak_flops / bandwidth (costmodel.py:69-72)."""
    return profile.peak_flops / profile.mem_bandwidth


def compute_time_ratio(intensity, profile):
    """intensity / ridge: compute time over memory time of an overlapped
    operator (costmodel.py:75-80); below 1 it is memory-bound."""
    return intensity / balance_ratio(profile)


def is_memory_bound(intensity, profile):
    return compute_time_ratio(intensity, profile) < 1.0


def memory_time(elements, profile):
    """Seconds to move `elements` at full bandwidth (costmodel.py:122-124)."""
    return elements * profile.bytes_per_element / profile.mem_bandwidth


def compute_time(flops, profile):
    return flops / profile.peak_flops


def roofline_time(flops, elements, profile):
    """max(memory time, compute time) (costmodel.py:131-135)."""
    return max(memory_time(elements, profile), compute_time(flops, profile))


def emit_speedup_curves(path, batch_sizes=(4, 8, 16, 32), context_lens=(128, 256),
                        s_values=(64, 128, 256, 512, 1024, 2048, 4096), measured=None):
    """The theoretical-speedup grid as CSV rows (b, c, s, p_theoretical,
    p_measured_traffic) -- the reference's CSV columns (costmodel.py:
    138-163); `measured(b, c, s)`, if given, fills the last column."""
    rows = [{"b": b, "c": c, "s": s, "p_theoretical": repr(theoretical_speedup(b, s, c)),
             "p_measured_traffic": "" if measured is None else repr(measured(b, c, s))}
            for b in batch_sizes for c in context_lens for s in s_values]
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0]) if rows else
                           ["b", "c", "s", "p_theoretical", "p_measured_traffic"])
        w.writeheader()
        w.writerows(rows)
    return rows


def b200_relay_step_seconds(shape: "DecodeShape") -> float:
    """Measured-model wall time of one HBM-bound relay decode step (for the
    engine's step-cost hook, engine.py:77-85); tensor-bound shapes (large GQA
    batches) are bounded below by their roofline at the measured peaks."""
    prof = HARDWARE_PROFILES["B200"]
    t = B200_STEP_FIXED_S + shape.bytes_alg / B200_STEP_MARGINAL_BPS
    return max(B200_STEP_FLOOR_S, t, shape.roofline_s(prof.mem_bandwidth, prof.peak_flops))
