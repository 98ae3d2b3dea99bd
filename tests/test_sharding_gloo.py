"""World-size-2 coverage of the KV-head-sharded path on CPU (gloo).

Each rank computes the relay output of its KV-head shard (with the float64
oracle standing in for the per-rank GPU kernels, which need a B200), then
`sharding.gather_heads` all-gathers and reassembles.  The gathered result
must equal the unsharded computation bitwise: per-head math is unchanged by
sharding.
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(hq, hkv):
    rng = np.random.default_rng(3)
    b, s, d = 4, 24, 16
    q = rng.standard_normal((b, 1, hq, d))
    sk = rng.standard_normal((s, hkv, d)); sv = rng.standard_normal((s, hkv, d))
    lens = [3, 8, 1, 5]
    ck = [rng.standard_normal((c, hkv, d)) for c in lens]
    cv = [rng.standard_normal((c, hkv, d)) for c in lens]
    return q, sk, sv, ck, cv


def _worker(rank, world, port, hq, hkv, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import relay_oracle as orc
        from paper_2402_14808_b200 import sharding
        q, sk, sv, ck, cv = _inputs(hq, hkv)
        g = hq // hkv
        ka, kb, qa, qb = sharding.local_heads(hkv, hq, world, rank)
        ex = lambda x: orc.expand_kv(x[:, ka:kb], g)  # noqa: E731
        local = orc.relay_attention(q[:, :, qa:qb], ex(sk), ex(sv), [ex(x) for x in ck],
                                    [ex(x) for x in cv], threads=1)
        local_t = torch.from_numpy(np.ascontiguousarray(local[:, 0]))
        full = sharding.gather_heads(local_t, hq, hkv)
        if rank == 0:
            np.save(result_path, full.numpy())
    finally:
        dist.destroy_process_group()


def _run(hq, hkv, world, tmp_path):
    path = str(tmp_path / f"gathered_{hq}_{hkv}.npy")
    mp.start_processes(_worker, args=(world, _free_port(), hq, hkv, path), nprocs=world,
                       join=True, start_method="spawn")
    from oracle import relay_oracle as orc
    q, sk, sv, ck, cv = _inputs(hq, hkv)
    g = hq // hkv
    full = orc.relay_attention(q, orc.expand_kv(sk, g), orc.expand_kv(sv, g),
                               [orc.expand_kv(x, g) for x in ck], [orc.expand_kv(x, g) for x in cv],
                               threads=1)
    got = np.load(path)
    assert got.shape == full[:, 0].shape
    assert (got == full[:, 0]).all()


def test_head_sharded_gather_mha_uneven(tmp_path):
    _run(hq=5, hkv=5, world=2, tmp_path=tmp_path)       # 3 + 2 heads, padded gather


def test_head_sharded_gather_gqa(tmp_path):
    _run(hq=8, hkv=2, world=2, tmp_path=tmp_path)       # one KV head (4 q heads) per rank
