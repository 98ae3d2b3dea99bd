"""Generate tests/golden/*.npz by running the REFERENCE itself.

Run in the authoring container (where /root/reference exists):
    python tests/golden/make_golden.py
The reference package is imported from /root/reference/pkg/src (its
pure-Python kernel backend, bitwise identical to its Cython build per
/root/reference/pkg/tests/test_backends.py).  The fixtures are small and
committed; nothing on the GPU box reads /root/reference.
"""

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    os.environ.setdefault("RELAYSERVE_BACKEND", "pure")
    sys.path.insert(0, REF)
    from relayserve import attention, costmodel, numerics  # noqa: E402

    out = {}

    # known answers (test_numerics.py:49-63, test_attention.py:60-156)
    for i, row in enumerate([[0.0, 0.0], [1000.0, 1000.0], [0.0, math.log(3.0)]]):
        p, l = numerics.softmax_lse([row])
        out[f"softmax_in_{i}"] = np.asarray([row])
        out[f"softmax_probs_{i}"] = p
        out[f"softmax_lse_{i}"] = l

    rng = np.random.default_rng(2)
    q = rng.standard_normal((1, 1, 1, 8)); k = rng.standard_normal((1, 1, 1, 8))
    v = rng.standard_normal((1, 1, 1, 8))
    r = attention.attention_with_lse(q, k, v, causal=False)
    out.update(single_q=q, single_k=k, single_v=v, single_o=r.output, single_lse=r.lse)

    lse_sys = np.asarray([[[0.0, 50.0, 0.0, 3.0]]])
    lse_ctx = np.asarray([[[math.log(3.0), 0.0, 0.0, -2.0]]])
    o_sys = rng.standard_normal((1, 1, 4, 8)); o_ctx = rng.standard_normal((1, 1, 4, 8))
    out.update(fusion_o_sys=o_sys, fusion_lse_sys=lse_sys, fusion_o_ctx=o_ctx,
               fusion_lse_ctx=lse_ctx,
               fusion_out=attention.relay_fusion(o_sys, lse_sys, o_ctx, lse_ctx))

    # attention_with_lse random cases, causal and not
    rng = np.random.default_rng(4)
    for causal in (0, 1):
        q = rng.standard_normal((2, 3, 2, 16)); k = rng.standard_normal((2, 7, 2, 16))
        v = rng.standard_normal((2, 7, 2, 16))
        r = attention.attention_with_lse(q, k, v, causal=bool(causal))
        out.update({f"awl{causal}_q": q, f"awl{causal}_k": k, f"awl{causal}_v": v,
                    f"awl{causal}_o": r.output, f"awl{causal}_lse": r.lse})

    # relay decode + prompt-phase cases (test_attention.py:190-200 shapes, d=16)
    cases = {"decode": (4, 8, [1, 3, 5, 7], 1, 2, 16),
             "prompt": (2, 4, [6, 6], 6, 2, 16),
             "bf16dec": (4, 64, [16, 9, 1, 33], 1, 4, 128)}
    for name, (b, s, lens, m, h, d) in cases.items():
        rng = np.random.default_rng(10 + len(name))
        sk = rng.standard_normal((s, h, d)); sv = rng.standard_normal((s, h, d))
        ck = [rng.standard_normal((c, h, d)) for c in lens]
        cv = [rng.standard_normal((c, h, d)) for c in lens]
        qq = rng.standard_normal((b, m, h, d))
        if name.startswith("bf16"):
            # inputs representable in bf16 so the GPU sees the same values
            def rb(x):
                f = np.ascontiguousarray(x, dtype=np.float32)
                u = f.view(np.uint32).astype(np.uint64)
                u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
                return u.astype(np.uint32).view(np.float32).astype(np.float64)
            sk, sv, qq = rb(sk), rb(sv), rb(qq)
            ck = [rb(x) for x in ck]; cv = [rb(x) for x in cv]
        o = attention.relay_attention(qq, sk, sv, ck, cv)
        # fused lse via the reference's own segment LSEs
        q_flat = np.concatenate([qq[i] for i in range(b)], axis=0)
        rs = attention.attention_with_lse(q_flat[None], sk[None], sv[None], causal=False)
        lse_f = []
        for i in range(b):
            rc = attention.attention_with_lse(qq[i][None], ck[i][None], cv[i][None], causal=True)
            lse_f.append(np.logaddexp(rs.lse[0, i * m:(i + 1) * m], rc.lse[0]))
        pre = f"relay_{name}_"
        out[pre + "q"] = qq; out[pre + "sys_k"] = sk; out[pre + "sys_v"] = sv
        out[pre + "lens"] = np.asarray(lens, dtype=np.int64)
        out[pre + "ctx_k"] = np.concatenate(ck, axis=0)
        out[pre + "ctx_v"] = np.concatenate(cv, axis=0)
        out[pre + "out"] = o
        out[pre + "lse"] = np.stack(lse_f, axis=0)
        cnt = attention.TrafficCounter()
        attention.relay_attention(qq, sk, sv, ck, cv, counter=cnt)
        out[pre + "traffic"] = np.asarray([cnt.elements_read, cnt.elements_written,
                                           cnt.lse_elements], dtype=np.int64)
        fk = [np.concatenate([sk, x]) for x in ck]; fv = [np.concatenate([sv, x]) for x in cv]
        cnt.reset()
        ob = attention.baseline_attention(qq, fk, fv, counter=cnt)
        out[pre + "baseline_out"] = ob
        out[pre + "baseline_traffic"] = np.asarray(
            [cnt.elements_read, cnt.elements_written], dtype=np.int64)

    tuples = []
    for b in (1, 2, 4, 32):
        for s in (1, 64, 2048):
            for c in (1, 128):
                for d in (4, 6656):
                    tuples.append((b, s, c, d, costmodel.traffic_relay(b, s, c, d),
                                   costmodel.traffic_baseline(b, s, c, d)))
    out["traffic_tuples"] = np.asarray(tuples, dtype=np.int64)
    out["speedup_32_2048_128"] = np.asarray([costmodel.theoretical_speedup(32, 2048, 128)])

    # RoPE (decode prologue): numerics.rope_rows / rope_apply
    # (numerics.py:81-108 -> kernels.rope_rows, _kernels_cy.pyx:80-102) at
    # context positions token_index + s (kvcache.context_position, kvcache.py:25-33)
    from relayserve import kvcache  # noqa: E402
    rng = np.random.default_rng(5)
    xr = rng.standard_normal((12, 128))
    pos = np.asarray([kvcache.context_position(t, s) for t, s in
                      [(0, 0), (1, 0), (0, 1), (5, 512), (127, 8192), (3, 32768), (1023, 65536),
                       (0, 65535), (17, 4096), (2, 7), (100, 100), (64, 131072)]], dtype=np.int64)
    out["rope_x"] = xr
    out["rope_pos"] = pos
    out["rope_out"] = numerics.rope_rows(xr, pos)
    v8 = rng.standard_normal(8)
    out["rope_apply_v"] = v8
    out["rope_apply_out"] = np.stack([numerics.rope_apply(v8, p) for p in (0, 1, 2, 1000)])

    # RELAYKV system-cache files written by the reference (kvcache.py:66-82)
    rng = np.random.default_rng(6)
    ks = [rng.standard_normal((7, 3, 16)) for _ in range(2)]
    vs = [rng.standard_normal((7, 3, 16)) for _ in range(2)]
    for bits in (32, 16):
        cache = kvcache.SystemKvCache(keys=tuple(k.astype(f"<f{bits // 8}") for k in ks),
                                      values=tuple(v.astype(f"<f{bits // 8}") for v in vs),
                                      system_len=7, prompt_id="golden")
        kvcache.save_system_cache(cache, os.path.join(HERE, f"system_f{bits}.relaykv"))
        back = kvcache.load_system_cache(os.path.join(HERE, f"system_f{bits}.relaykv"))
        out[f"relaykv_f{bits}_keys"] = np.stack(back.keys)
        out[f"relaykv_f{bits}_values"] = np.stack(back.values)

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {len(out)} arrays to {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
