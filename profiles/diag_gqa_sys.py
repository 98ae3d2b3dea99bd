"""One launch of the system kernel at a GQA-large shape (C4 by default:
b=128, 32q/8kv, s=32k) for ncu captures.  Diagnostics.

    python profiles/diag_gqa_sys.py [b hq hkv s]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14808_b200 import kernels  # noqa: E402


def main():
    b, hq, hkv, s = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (128, 32, 8, 32768)))
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(b, hq, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(hkv, s, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(hkv, s, 128, device="cuda", generator=g).to(torch.bfloat16)
    for _ in range(3):
        kernels.system_attention(q, k, v, kv_layout="hsd")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        kernels.system_attention(q, k, v, kv_layout="hsd")
    e1.record()
    torch.cuda.synchronize()
    print(f"system kernel b={b} hq={hq} hkv={hkv} s={s}: {e0.elapsed_time(e1) / 5 * 1e3:.1f} us")


if __name__ == "__main__":
    main()
