"""World-size-2 gloo tests of the multi-GPU plumbing on CPU.

The CUDA kernels are not involved: each rank transforms its shard with the fp64 oracle as a
stand-in, so these tests check the sharding arithmetic, band-row mapping, the LL gather and the
max-over-ranks timing reduction — the host logic bench.py runs under torchrun.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle as o
from paper_1002_2184_b200 import dist as fdist

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, fn_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        q.put((rank, globals()[fn_name](rank)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, fn_name, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    return res


# ------------------------------------------------------------------ rank bodies
H, W, L = 512, 256, 5


def _c5_like_rank(rank):
    r0, r1 = fdist.row_band(H, WORLD, rank, L)
    band = datagen.c5_rows(r0, r1, size=512)[:, :W]
    coeffs = o.analyze_2d(band, L)
    ll = torch.from_numpy(np.ascontiguousarray(coeffs[:(r1 - r0) >> L, :W >> L]))
    gathered = fdist.gather_coarse_ll(ll)
    t = fdist.max_over_ranks(1.5 + rank)
    return {"r0": r0, "r1": r1, "coeffs": coeffs, "ll_all": gathered.numpy(), "tmax": t}


N1, J1 = 8192, 7


def _segment_rank(rank):
    s0, s1 = fdist.segment_1d(N1, WORLD, rank, J1)
    x = datagen.c2_signal(0, n=N1)[s0:s1]
    c = o.decompose_1d(x, J1)
    a = torch.from_numpy(np.ascontiguousarray(c[:(s1 - s0) >> J1]))
    return {"s0": s0, "s1": s1, "coeffs": c, "a_all": fdist.gather_coarse_ll(a[None]).numpy()}


def _weak_rank(rank):
    first, count = fdist.unit_shard(3, rank)
    x = datagen.c4_batch(first, count, size=64)
    return {"first": first, "count": count, "coeffs": o.analyze_2d(x, 4)}


def _strong_rank(rank):
    """bench.py's strong-scaling split at world 2: c4's 256 images -> 128 per rank, c2's 4096
    signals -> 2048, c5's rows -> two 16384-row bands; plus a reduced c4-like batch transformed
    per rank (oracle stand-in) and the whole-job sample count bench reports (all-reduced)."""
    import bench
    sh = {k: bench.shard_of(bench.WORKLOADS[k], WORLD, rank) for k in ("c2", "c4", "c5")}
    first, count = fdist.unit_range(6, WORLD, rank)
    x = datagen.c4_batch(first, count, size=64)
    total = bench.fdist_total(bench.WORKLOADS["c4"], WORLD, None, x.size, "cpu")
    return {"shards": sh, "first": first, "count": count, "coeffs": o.analyze_2d(x, 4), "total": total}


# ------------------------------------------------------------------ tests
@pytest.mark.timeout(300)
def test_strong_scaling_unit_split():
    """BASELINE configs[3]: c4 is sharded by image index across the GPUs (strong scaling, a fixed
    global batch of 256); c2 likewise by signal."""
    res = _run("_strong_rank")
    for r in range(WORLD):
        assert isinstance(res[r], dict), res[r]
    c4 = [res[r]["shards"]["c4"] for r in range(WORLD)]
    assert [(s["first"], s["count"]) for s in c4] == [(0, 128), (128, 128)]
    assert all(s["global_batch"] == 256 and s["scaling"] == "strong" for s in c4)
    c2 = [res[r]["shards"]["c2"] for r in range(WORLD)]
    assert [(s["first"], s["count"]) for s in c2] == [(0, 2048), (2048, 2048)]
    c5 = [res[r]["shards"]["c5"] for r in range(WORLD)]
    assert [(s["r0"], s["r1"]) for s in c5] == [(0, 16384), (16384, 32768)]
    allx = datagen.c4_batch(0, 6, size=64)
    ref = o.analyze_2d(allx, 4)
    for r in range(WORLD):
        f, c = res[r]["first"], res[r]["count"]
        np.testing.assert_allclose(res[r]["coeffs"], ref[f:f + c], atol=1e-12)
        assert res[r]["total"] == allx.size


def test_unit_range_partitions():
    for total in (1, 5, 6, 256, 4096, 257):
        for world in (1, 2, 3, 4, 8):
            if total < world:
                with pytest.raises(ValueError):
                    fdist.unit_range(total, world, 0)
                continue
            parts = [fdist.unit_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and sum(c for _, c in parts) == total
            assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    assert fdist.unit_range(256, 8, 7) == (224, 32)
    with pytest.raises(ValueError):
        fdist.unit_range(8, 2, 2)


@pytest.mark.timeout(300)
def test_row_band_sharding_and_ll_gather():
    res = _run("_c5_like_rank")
    full = datagen.c5_rows(0, H, size=512)[:, :W]
    ref = o.analyze_2d(full, L)
    for r in range(WORLD):
        assert isinstance(res[r], dict), res[r]
        d = res[r]
        assert (d["r0"], d["r1"]) == (r * H // WORLD, (r + 1) * H // WORLD)
        bh = d["r1"] - d["r0"]
        for j in range(1, L + 1):
            g0, g1 = fdist.band_rows(d["r0"], d["r1"], j)
            hj, wj, bj = H >> j, W >> j, bh >> j
            # band-local Mallat output == the corresponding rows of every global band (pin C8)
            np.testing.assert_allclose(d["coeffs"][:bj, wj:2 * wj], ref[g0:g1, wj:2 * wj], atol=1e-12)
            np.testing.assert_allclose(d["coeffs"][bj:2 * bj, :wj], ref[hj + g0:hj + g1, :wj], atol=1e-12)
            np.testing.assert_allclose(d["coeffs"][bj:2 * bj, wj:2 * wj], ref[hj + g0:hj + g1, wj:2 * wj], atol=1e-12)
        # every rank ends with the same, complete coarsest LL
        np.testing.assert_allclose(d["ll_all"], ref[:H >> L, :W >> L], atol=1e-12)
        assert d["tmax"] == 1.5 + WORLD - 1


@pytest.mark.timeout(300)
def test_weak_scaling_unit_shards():
    res = _run("_weak_rank")
    firsts = sorted((res[r]["first"], res[r]["count"]) for r in range(WORLD))
    assert firsts == [(0, 3), (3, 3)]
    allx = datagen.c4_batch(0, 6, size=64)
    ref = o.analyze_2d(allx, 4)
    for r in range(WORLD):
        f, c = res[r]["first"], res[r]["count"]
        np.testing.assert_allclose(res[r]["coeffs"], ref[f:f + c], atol=1e-12)


@pytest.mark.timeout(300)
def test_long_signal_segments():
    """§8(f) f2: one long signal split into 2^J-aligned segments; every band of every segment lands
    at its global Mallat offset, and the gathered coarse approximation is the global a_J."""
    res = _run("_segment_rank")
    ref = o.decompose_1d(datagen.c2_signal(0, n=N1), J1)
    for r in range(WORLD):
        d = res[r]
        assert isinstance(d, dict), d
        for band, (lo, go, ln) in fdist.segment_bands_1d(d["s0"], d["s1"], N1, J1).items():
            np.testing.assert_allclose(d["coeffs"][lo:lo + ln], ref[go:go + ln], atol=1e-12, err_msg=band)
        np.testing.assert_allclose(d["a_all"].reshape(-1), ref[:N1 >> J1], atol=1e-12)


def test_row_band_validation():
    assert fdist.row_band(32768, 8, 7, 8) == (28672, 32768)
    with pytest.raises(ValueError):
        fdist.row_band(32768, 3, 0, 8)          # not an equal split
    with pytest.raises(ValueError):
        fdist.row_band(1024, 8, 0, 8)           # 128-row band < 2^8: would need a halo
    assert fdist.band_rows(4096, 8192, 8) == (16, 32)
