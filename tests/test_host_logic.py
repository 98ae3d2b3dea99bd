"""Host-side logic: stream-K plan (Python mirror == C), tile coverage,
head sharding, cost model, block pool (no GPU)."""

import itertools
import os

import numpy as np
import pytest

from paper_2402_14808_b200 import _lib, costmodel, sharding
from paper_2402_14808_b200.kvcache import BlockAllocator
from paper_2402_14808_b200.plan import SysPlan


@pytest.mark.parametrize("n_rows,hq,hkv,s,grid", [
    (32, 52, 52, 8192, 148), (32, 52, 52, 512, 148), (4, 32, 32, 512, 148),
    (64, 32, 32, 4096, 148), (128, 32, 8, 32768, 148), (256, 64, 8, 65536, 148),
    (32, 7, 7, 8192, 148), (1, 1, 1, 1, 148), (32, 4, 4, 1000, 5),
    (64, 2, 2, 384, 3), (24, 8, 2, 300, 7),
    (128, 32, 8, 32768, 82), (128, 32, 8, 32768, 64), (40, 8, 2, 300, 5), (64, 32, 32, 4096, 39),
])
def test_plan_matches_c_and_covers_tiles(n_rows, hq, hkv, s, grid):
    p = SysPlan(n_rows, hq, hkv, s, grid)
    f, _ = _lib.sys_plan(n_rows, hq, hkv, s, grid)
    assert (p.nq, p.n_qt, p.tpu, p.n_units, p.total, p.grid, p.max_parts, int(p.rr)) == \
        (f["nq"], f["n_qt"], f["tpu"], f["n_units"], f["total"], f["grid"], f["max_parts"], f["rr"])
    if p.rr:
        # whole units dealt round-robin: every unit once, balanced to one unit
        units = [p.cta_units(c) for c in range(p.grid)]
        assert sorted(u for us in units for u in us) == list(range(p.n_units))
        assert max(map(len, units)) - min(map(len, units)) <= 1
        assert p.max_parts == 1
        return
    ranges = p.cta_ranges()
    assert ranges[0][0] == 0 and ranges[-1][1] == p.total
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1            # balanced to one tile
    for x in range(0, p.total, max(1, p.total // 97)):
        c = p.owner(x)
        assert ranges[c][0] <= x < ranges[c][1]
    for u in range(p.n_units):
        first = u * p.tpu
        owners = {p.owner(x) for x in range(first, first + p.tpu)}
        assert len(owners) == p.unit_parts(u) <= p.max_parts


def test_head_ranges():
    assert [b - a for a, b in sharding.head_ranges(52, 8)] == [7, 7, 7, 7, 6, 6, 6, 6]
    assert [b - a for a, b in sharding.head_ranges(52, 4)] == [13] * 4
    for h, w in itertools.product([1, 7, 8, 52, 64], [1, 2, 4, 8]):
        if h < w:
            continue
        r = sharding.head_ranges(h, w)
        assert r[0][0] == 0 and r[-1][1] == h
        assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1
    assert sharding.local_heads(8, 64, 8, 3) == (3, 4, 24, 32)


def test_costmodel_reference_forms():
    assert costmodel.traffic_baseline(2, 3, 1, 4) == 48
    assert costmodel.traffic_relay(2, 3, 1, 4) == 76
    assert abs(costmodel.theoretical_speedup(32, 2048, 128) - 2178 / 199) < 1e-9
    g = np.load(__file__.replace("test_host_logic.py", "golden/reference_golden.npz"))
    for b, s, c, d, nr, nb in g["traffic_tuples"]:
        assert costmodel.traffic_relay(b, s, c, d) == nr
        assert costmodel.traffic_baseline(b, s, c, d) == nb


def test_byte_model_c2():
    sh = costmodel.DecodeShape(b=32, hq=52, hkv=52, s=8192, ctx_total=32 * 128)
    assert sh.bytes_alg == 2 * 2 * 52 * 128 * (8192 + 4096) + 2 * 2 * 32 * 52 * 128
    assert abs(sh.bytes_alg / 1e6 - 328.0) < 1.0       # 328 MB
    assert sh.flops_sys == 4 * 32 * 52 * 8192 * 128
    assert 21 < sh.bytes_naive / sh.bytes_alg < 22.5   # 21.6x


def test_block_pool_conservation():
    rng = np.random.default_rng(808)
    pool = BlockAllocator(num_blocks=64, block_size=4)
    pool.shuffle(3)
    live, nid = {}, 0
    from paper_2402_14808_b200.errors import CapacityError
    for _ in range(3000):
        if live and rng.random() < 0.45:
            rid = list(live)[int(rng.integers(len(live)))]
            assert pool.close(rid) == len(live.pop(rid))
        else:
            rid = f"r{nid}"
            nid += 1
            pool.open(rid)
            try:
                pool.reserve(rid, int(rng.integers(1, 10)))
                pool.reserve(rid, int(rng.integers(1, 20)))
                live[rid] = list(pool.blocks(rid))
            except CapacityError:
                pool.close(rid)
        assert pool.used_blocks + pool.free_blocks == pool.num_blocks
        owned = [b for t in live.values() for b in t]
        assert len(owned) == len(set(owned)) == pool.used_blocks   # no block owned twice
        assert all(0 <= b < 64 for b in owned)


def test_relay_sm_split():
    """rb_relay_sys_grid: within [1, sms], never below the latency floor,
    non-decreasing in s."""
    sms = 148
    ctx = 32 * 128
    prev = 0
    for s in (64, 512, 2048, 4096, 8192, 32768, 131072):
        g = _lib.relay_sys_grid(32, 52, 52, s, ctx, sms)
        assert 1 <= g <= sms
        assert g >= min(sms * 20 // 100, SysPlan(32, 52, 52, s, sms).total)
        assert g >= prev
        prev = g
    assert _lib.relay_sys_grid(30, 24, 8, 512, 30 * 4096, sms) >= 1
    # no context at all: the system kernel takes every SM
    assert _lib.relay_sys_grid(32, 52, 52, 8192, 0, sms) == sms


def test_plan_tile_sizes_and_aligned_split():
    """nq: 16 / 32 for the swap-AB kernel, 128 (non-swapped kernel) from 128
    rows per KV head, 256 (two query tiles per unit) from 256; several units
    per head with fewer units than CTAs get an equal number of CTAs per unit
    when that keeps >= 85% of them."""
    assert SysPlan(16, 1, 1, 100, 148).nq == 16
    assert SysPlan(127, 1, 1, 100, 148).nq == 32
    assert SysPlan(128, 1, 1, 100, 148).nq == 128
    assert SysPlan(255, 1, 1, 100, 148).nq == 128
    assert SysPlan(256, 1, 1, 100, 148).nq == 256
    c4 = SysPlan(128, 32, 8, 32768, 148)
    assert (c4.nq, c4.n_qt, c4.n_units, c4.grid) == (256, 2, 16, 144)
    # 9 CTAs per unit: every CTA's key range lies inside one unit, and the
    # units are cut at the same key tiles
    ranges = c4.cta_ranges()
    assert all(a // c4.tpu == (b - 1) // c4.tpu for a, b in ranges)
    cuts = [[a % c4.tpu for a, _ in ranges[u * 9:(u + 1) * 9]] for u in range(16)]
    assert all(c == cuts[0] for c in cuts)
    assert SysPlan(128, 32, 8, 32768, 82).grid == 80      # 5 per unit (82 would misalign)
    old = SysPlan(40, 8, 2, 300, 148)                     # 160 rows per head: 128-row kernel
    assert (old.nq, old.n_qt) == (128, 2)
    c3 = SysPlan(64, 32, 32, 4096, 148)
    assert (c3.nq, c3.n_qt, c3.n_units, c3.grid) == (32, 2, 64, 128)


def test_relay_split_gqa_large_whole_units():
    """The relay split gives the 128-row GQA kernel whole multiples of its
    unit count (at least one CTA per unit)."""
    sms = 148
    g4 = _lib.relay_sys_grid(128, 32, 8, 32768, 128 * 512, sms)
    assert g4 % 16 == 0 and 16 <= g4 <= sms
    g5 = _lib.relay_sys_grid(256, 64, 8, 65536, 256 * 1024, sms)
    assert g5 == 128


def _bf16(x):
    import torch
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("bits", [32, 16])
def test_relaykv_load_reference_files(bits):
    """SystemKvCache.load reads the reference's RELAYKV files
    (save_system_cache, kvcache.py:66-82) into bf16 [h][s][128] (head dims
    zero-padded past d), the same values the reference loads, bf16-rounded."""
    import os
    from paper_2402_14808_b200.kvcache import SystemKvCache
    here = os.path.dirname(os.path.abspath(__file__))
    g = np.load(os.path.join(here, "golden", "reference_golden.npz"))
    cache = SystemKvCache.load(os.path.join(here, "golden", f"system_f{bits}.relaykv"), device="cpu")
    assert (cache.layers, cache.kv_heads, cache.system_len) == (2, 3, 7)
    for layer in range(2):
        for got, ref in ((cache.keys[layer], g[f"relaykv_f{bits}_keys"][layer]),
                         (cache.values[layer], g[f"relaykv_f{bits}_values"][layer])):
            t = got.float().numpy()
            assert (t[:, :, :16] == _bf16(ref).transpose(1, 0, 2)).all()
            assert (t[:, :, 16:] == 0).all()


def test_relaykv_round_trip_and_errors(tmp_path):
    import torch
    from paper_2402_14808_b200.errors import ContractError
    from paper_2402_14808_b200.kvcache import SystemKvCache
    g = torch.Generator().manual_seed(3)
    cache = SystemKvCache.random(2, 4, 9, device="cpu", generator=g)
    path = tmp_path / "c.relaykv"
    cache.save(path)
    back = SystemKvCache.load(path, device="cpu")
    for a, b in zip(cache.keys + cache.values, back.keys + back.values):
        assert torch.equal(a, b)
    raw = path.read_bytes()
    (tmp_path / "bad_magic").write_bytes(b"NOTRELAY" + raw[8:])
    (tmp_path / "bad_version").write_bytes(raw[:8] + (7).to_bytes(4, "little") + raw[12:])
    (tmp_path / "truncated").write_bytes(raw[:-4])
    for name in ("bad_magic", "bad_version", "truncated"):
        with pytest.raises(ContractError):
            SystemKvCache.load(tmp_path / name, device="cpu")


def test_relaykv_written_file_loads_in_reference(tmp_path):
    """A file written by SystemKvCache.save is read back by the reference's
    own load_system_cache (oracle/_ref, the compiled reference modules)."""
    import os
    import sys
    import torch
    from paper_2402_14808_b200.kvcache import SystemKvCache
    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "relayserve")):
        pytest.skip("oracle/_ref not built")
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    from relayserve import kvcache as ref_kvcache
    g = torch.Generator().manual_seed(4)
    cache = SystemKvCache.random(2, 3, 5, device="cpu", generator=g)
    cache.save(tmp_path / "ours.relaykv")
    ref = ref_kvcache.load_system_cache(tmp_path / "ours.relaykv")
    assert ref.layers == 2 and ref.system_len == 5
    for layer in range(2):
        assert (ref.keys[layer] == cache.keys[layer].float().permute(1, 0, 2).numpy()).all()
        assert (ref.values[layer] == cache.values[layer].float().permute(1, 0, 2).numpy()).all()


def test_b200_profile_and_step_model():
    """B200 HardwareProfile and the measured step model reproduce the
    round's measured C2 sweep within 10% for s >= 2k."""
    from paper_2402_14808_b200.errors import ContractError
    assert costmodel.HARDWARE_PROFILES["B200"].mem_bandwidth == 6539.9e9
    with pytest.raises(ContractError):
        costmodel.HardwareProfile("bad", 0, 1)
    measured = {2048: 46.4e-6, 4096: 53.7e-6, 8192: 68.7e-6, 16384: 100.6e-6, 32768: 163.5e-6}
    for s, t in measured.items():
        sh = costmodel.DecodeShape(b=32, hq=52, hkv=52, s=s, ctx_total=32 * 128)
        assert abs(costmodel.b200_relay_step_seconds(sh) - t) / t < 0.10


def test_costmodel_matches_reference_module(tmp_path):
    """The ported cost-model helpers (traffic report, GEMM intensity, ridge /
    roofline, speedup-curve CSV) against the reference's own costmodel
    compiled into oracle/_ref."""
    import os
    import sys
    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "relayserve")):
        pytest.skip("oracle/_ref not built")
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import relayserve.costmodel as ref
    from relayserve.numerics import GemmShape as RefShape
    for b, s, c, d in [(1, 0, 0, 1), (32, 2048, 128, 4096), (4, 64, 256, 16), (8, 8, 1, 32)]:
        a, o = ref.traffic_report(b, s, c, d), costmodel.traffic_report(b, s, c, d)
        assert (a.n_baseline, a.n_relay, a.speedup) == (o.n_baseline, o.n_relay, o.speedup)
    for m, n, k in [(1, 1, 1), (32, 8192, 128), (7, 3, 5)]:
        assert ref.arithmetic_intensity_gemm(RefShape(m, n, k)) == pytest.approx(
            costmodel.arithmetic_intensity_gemm(costmodel.GemmShape(m, n, k)), rel=1e-14)
        assert ref.gemm_intensity_bound(RefShape(m, n, k)) == \
            costmodel.gemm_intensity_bound(costmodel.GemmShape(m, n, k))
    for name, prof in ref.HARDWARE_PROFILES.items():
        ours = costmodel.HARDWARE_PROFILES[name]
        assert ref.balance_ratio(prof) == pytest.approx(costmodel.balance_ratio(ours), rel=1e-14)
        for inten in (1.0, 38.2, 300.0):
            assert ref.is_memory_bound(inten, prof) == costmodel.is_memory_bound(inten, ours)
        assert ref.roofline_time(1e12, 10 ** 9, prof) == pytest.approx(
            costmodel.roofline_time(1e12, 10 ** 9, ours), rel=1e-14)
    ref.emit_speedup_curves(tmp_path / "ref.csv")
    costmodel.emit_speedup_curves(tmp_path / "ours.csv")
    assert (tmp_path / "ref.csv").read_text() == (tmp_path / "ours.csv").read_text()


def test_engine_traffic_convention_matches_reference():
    """The B200 engine's per-step attention element count is the reference
    engine's (relayserve/engine.py:43-53, compiled into oracle/_ref)."""
    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "relayserve")):
        pytest.skip("oracle/_ref not built")
    import sys
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import relayserve.engine as ref_engine
    from paper_2402_14808_b200.engine import attention_step_elements
    rng = np.random.default_rng(4)
    for _ in range(50):
        b = int(rng.integers(1, 9))
        new = [int(x) for x in rng.integers(1, 40, b)]
        lens = [n + int(x) for n, x in zip(new, rng.integers(0, 500, b))]
        s, d = int(rng.integers(1, 5000)), int(rng.integers(1, 1024))
        for mode in ("relay", "baseline"):
            assert attention_step_elements(mode, s, new, lens, d) == \
                ref_engine.attention_step_elements(mode, s, new, lens, d)
