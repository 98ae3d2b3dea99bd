"""Traffic / roofline model of the relay decode step.

Reference element-count closed forms (costmodel.py:85-112), kept for API
compatibility, plus the physical byte model the B200 roofline uses
(SURVEY.md section 8d):

  B_alg   = e*2*H_kv*d*(s + sum_c) + e*2*b*H_q*d    shared KV once + context KV + Q + O
  B_naive = e*2*H_kv*d*(b*s + sum_c) + e*2*b*H_q*d  shared KV re-read per request
  F_sys   = 4*b*H_q*s*d,  F_ctx = 4*H_q*d*sum_c

Intermediates (fp32 system partials, LSEs, block tables) are NOT in B_alg;
`overhead_bytes` reports them separately.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ContractError


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
