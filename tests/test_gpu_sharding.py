"""KV-head sharding of the PRODUCT kernels, world size 2 on one GPU.

Two processes (gloo, both on cuda:0: the mode bench.py runs under
BENCH_SAME_GPU=1) each hold one rank's KV heads -- that slice of the system
cache, of the paged context pool and of the query heads (sharding.local_heads)
-- run RelayDecodeStep on it, and `sharding.gather_heads` all-gathers the
per-rank outputs.  Rank 0 compares with the unsharded step on the full heads.

Bitwise equality holds when every rank cuts its
system units where the unsharded step does: with a system grid of k CTAs
per unit on both sides, each unit is split at the same key tiles (rb_plan.h:
CTA c starts at floor(c * tiles / grid)), the context kernel's per-item math
does not depend on the grid, and the relay merge runs in slot order.  With
the production split (each rank sizes its own grid from its bytes) the cut
points move, and the results agree within the bf16 envelope instead.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(b, hq, hkv, s, seed):
    from gpu_util import synth_paged_problem
    lens = [int(x) for x in np.random.default_rng(seed).integers(1, 300, size=b)]
    return synth_paged_problem(b, hq, hkv, s, lens, seed)


def _slice(q, sys_cache, paged, ka, kb, qa, qb):
    """This rank's heads: a new SystemKvCache / PagedKvCache over the slice
    (same block ids, same block tables)."""
    from paper_2402_14808_b200.kvcache import PagedKvCache, SystemKvCache
    sc = SystemKvCache([k[ka:kb] for k in sys_cache.keys], [v[ka:kb] for v in sys_cache.values])
    pc = PagedKvCache(paged.layers, kb - ka, paged.allocator.num_blocks, paged.block_size)
    pc.k_pool.copy_(paged.k_pool[:, :, ka:kb])
    pc.v_pool.copy_(paged.v_pool[:, :, ka:kb])
    return q[:, qa:qb].contiguous(), sc, pc


def _worker(rank, world, port, b, hq, hkv, s, seed, k_per_unit, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2402_14808_b200 import _lib, sharding
        from paper_2402_14808_b200.attention import RelayDecodeStep
        q, sys_cache, paged, bt, cl = _problem(b, hq, hkv, s, seed)
        ka, kb, qa, qb = sharding.local_heads(hkv, hq, world, rank)
        ql, sl, pl = _slice(q, sys_cache, paged, ka, kb, qa, qb)
        n_units = _lib.sys_plan(b, qb - qa, kb - ka, s, 148)[0]["n_units"]
        grid = k_per_unit * n_units if k_per_unit else None
        out, lse = RelayDecodeStep(sl, pl, bt, cl, qb - qa, grid=grid, out_dtype=torch.float32)(ql)
        torch.cuda.synchronize()
        full = sharding.gather_heads(out.cpu(), hq, hkv)
        full_lse = sharding.gather_heads(lse.cpu()[..., None], hq, hkv)[..., 0]
        if rank == 0:
            torch.save({"out": full, "lse": full_lse}, os.path.join(out_dir, "gathered.pt"))
    finally:
        dist.destroy_process_group()


def _run(tmp_path, b, hq, hkv, s, seed, k_per_unit):
    import torch.multiprocessing as mp
    from paper_2402_14808_b200 import _lib
    from paper_2402_14808_b200.attention import RelayDecodeStep
    mp.start_processes(_worker, args=(2, _free_port(), b, hq, hkv, s, seed, k_per_unit,
                                      str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    got = torch.load(os.path.join(tmp_path, "gathered.pt"))
    q, sys_cache, paged, bt, cl = _problem(b, hq, hkv, s, seed)
    n_units = _lib.sys_plan(b, hq, hkv, s, 148)[0]["n_units"]
    grid = k_per_unit * n_units if k_per_unit else None
    out, lse = RelayDecodeStep(sys_cache, paged, bt, cl, hq, grid=grid, out_dtype=torch.float32)(q)
    torch.cuda.synchronize()
    return got["out"], got["lse"], out.cpu(), lse.cpu()


@pytest.mark.parametrize("b,hq,hkv,s", [(16, 8, 8, 1000), (40, 16, 4, 700), (12, 10, 5, 400)])
def test_sharded_step_bitwise_with_aligned_split(tmp_path, b, hq, hkv, s):
    g_out, g_lse, out, lse = _run(tmp_path, b, hq, hkv, s, seed=b + s, k_per_unit=2)
    assert torch.equal(g_out, out) and torch.equal(g_lse, lse), \
        f"max diff {(g_out - out).abs().max().item()}"


def test_sharded_step_production_split(tmp_path):
    from gpu_util import assert_close
    g_out, g_lse, out, lse = _run(tmp_path, 32, 12, 12, 2048, seed=5, k_per_unit=0)
    assert_close(g_out.numpy(), out.numpy(), "sharded (own SM split per rank) vs unsharded")
    assert_close(g_lse.numpy(), lse.numpy(), "sharded lse", lse=True)
