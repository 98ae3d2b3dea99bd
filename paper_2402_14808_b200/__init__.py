"""paper_2402_14808_b200 -- B200-native RelayAttention decode path.

Drop-in for the hot path of the reference package `relayserve`
(/root/reference/pkg/src/relayserve/attention.py): system-prompt attention
over the shared prefix KV (tcgen05 + TMA + TMEM, read once per batch),
request-context attention over paged KV with the LSE relay fusion fused into
its epilogue, and KV-head sharding across the GPUs of one node.

The only compute backend is librelay_b200.so (sm_100a); importing the
operator modules fails loudly if it is not built.
"""

__version__ = "0.1.0"

__all__ = [
    "TrafficCounter", "LseAttentionOutput", "attention_with_lse", "naive_causal_attention",
    "relay_fusion", "relay_attention", "relay_attention_ragged", "baseline_attention",
    "baseline_attention_ragged", "RelayDecodeStep", "RelayDecodeStack", "NaiveDecodeStep",
    "SystemKvCache",
    "PagedKvCache", "BlockAllocator", "theoretical_speedup", "kernel_backend",
]


def kernel_backend():
    """Name of the active kernel backend (there is exactly one)."""
    from .kernels import BACKEND
    return BACKEND


def __getattr__(name):
    if name in ("TrafficCounter", "LseAttentionOutput", "attention_with_lse",
                "naive_causal_attention", "relay_fusion", "relay_attention",
                "relay_attention_ragged", "baseline_attention", "baseline_attention_ragged",
                "RelayDecodeStep", "RelayDecodeStack", "NaiveDecodeStep"):
        from . import attention
        return getattr(attention, name)
    if name in ("SystemKvCache", "PagedKvCache", "BlockAllocator", "context_position"):
        from . import kvcache
        return getattr(kvcache, name)
    if name in ("theoretical_speedup", "traffic_relay", "traffic_baseline", "DecodeShape"):
        from . import costmodel
        return getattr(costmodel, name)
    raise AttributeError(f"module 'paper_2402_14808_b200' has no attribute {name!r}")
