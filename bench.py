#!/usr/bin/env python
"""Benchmark of the Fast Haar DWT+IDWT hot path on B200 (BASELINE.json metric:
"Fast Haar DWT+IDWT GB/s and Gsamples/s vs B200 HBM roofline at 1/2/4/8 GPUs").

One step = one multi-level analysis (fhwt_plan_analyze) + one synthesis (fhwt_plan_synthesize)
of the whole workload, inputs resident in HBM.  Default workload: BASELINE configs[3] (c4,
256 images 2048x2048 fp32, L=5) — the largest single-GPU 2-D config.  At N GPUs the fixed
workload is split (strong scaling, as BASELINE configs[3]/[4] say): c4 256/N images per rank, c2
4096/N signals, c5 32768/N-row bands + the coarsest-LL all-gather.  The per-rank step is replayed
as CUDA graphs.
Algorithmic bytes per step = 16 B/sample (fp32 read + write, twice).  A JSON line is printed by
rank 0.  ``--impl reference`` times the fp64 CPU oracle on the same workload instead.

Launch: python bench.py --gpus N --steps K --warmup W   (N>1 under torch.distributed.run)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Fast Haar DWT+IDWT GB/s and Gsamples/s vs B200 HBM roofline at 1/2/4/8 GPUs"
FALLBACK_HBM_GBS = 6650.0

WORKLOADS = {
    "c2": dict(kind="1d", n=65536, batch=4096, levels=10, shard="signal",
               desc="c2: 1-D batched 4096 x 65536 fp32 (3 sinusoids + N(0,0.1)), J=10, DWT+IDWT"),
    "c4": dict(kind="2d", h=2048, w=2048, batch=256, levels=5, shard="image",
               desc="c4: 2-D batched 256 x 2048x2048 fp32 (G()/255 images), L=5, DWT+IDWT"),
    "c5": dict(kind="2d", h=32768, w=32768, batch=1, levels=8, shard="rowband",
               desc="c5: 2-D 32768x32768 fp32 (G()/255), L=8, row bands + NCCL LL all-gather, DWT+IDWT"),
}


KERNEL_NAMES = {
    ("2d", "analysis"): "fhwt_plan_analyze (K1 ana2d_lean_kernel<true> + the coarse levels in the same launch)",
    ("2d", "synthesis"): "fhwt_plan_synthesize (K4 syn2d_prod_kernel<true> + the coarse levels in the same launch)",
    ("1d", "analysis"): "fhwt::ana1d_kernel",
    ("1d", "synthesis"): "fhwt::syn1d_kernel",
}


# ---------------------------------------------------------------------------------- helpers
def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md, no MEASURED_PEAKS.json)"


def ncu_traffic(workload, kernel):
    """dram read+write bytes per launch from a committed ncu --set full capture (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[workload][kernel]["dram_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        return None


class ClockSampler:
    """SM clock, board power and clock-event (throttle) reasons sampled through NVML every ~0.5 ms
    (plus the ~0.7 ms the four NVML queries take) by a background thread while the timed region runs
    (the c4 region is ~50 ms at --steps 20: nvidia-smi's 200 ms polling saw 3 mostly idle samples in
    round 1, a 2 ms period 18).  Falls back to nvidia-smi if NVML is missing."""
    PERIOD_S = 0.0005
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, device_index):
        self.dev = device_index
        self.samples = []
        self.max_mhz = None
        self._stop = None
        self._th = None
        self.err = None

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.dev]) if vis and vis.split(",")[0].isdigit() else self.dev
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001
            self.err = f"NVML unavailable: {e}"
            return self
        self._stop = threading.Event()

        def poll():
            while not self._stop.is_set():
                try:
                    self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                         nv.nvmlDeviceGetPowerUsage(h) / 1e3,
                                         nv.nvmlDeviceGetCurrentClocksEventReasons(h),
                                         nv.nvmlDeviceGetUtilizationRates(h).gpu))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(self.PERIOD_S)

        self._th = threading.Thread(target=poll, daemon=True)
        self._th.start()
        time.sleep(0.01)
        return self

    def __exit__(self, *exc):
        if self._th is not None:
            self._stop.set()
            self._th.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [self.err or "no samples"]}
        loaded = [s for s in self.samples if s[3] > 0] or self.samples
        reasons = 0
        for s in loaded:
            reasons |= int(s[2])
        return {"sm_mhz": statistics.median(s[0] for s in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(v for k, v in self.REASONS.items() if reasons & k),
                "power_w_max": max(s[1] for s in loaded), "samples": len(self.samples),
                "samples_under_load": sum(1 for s in self.samples if s[3] > 0),
                "sampler": f"NVML every {self.PERIOD_S * 1e3:.1f} ms + query time during the timed region"}


# ---------------------------------------------------------------------------------- data
def shard_of(cfg, ws, rank, weak=False):
    """This rank's share of the workload: c4 / c2 split their fixed global batch
    of images / signals into contiguous blocks of batch/N units (strong scaling; --weak gives every
    rank a full batch instead), c5 splits its rows into 2^L-aligned bands of h/N rows."""
    from paper_1002_2184_b200 import dist as fdist
    if cfg["shard"] in ("image", "signal"):
        if weak:
            first, count = fdist.unit_shard(cfg["batch"], rank)
            global_batch = cfg["batch"] * ws
        else:
            first, count = fdist.unit_range(cfg["batch"], ws, rank)
            global_batch = cfg["batch"]
        return {"kind": "units", "first": first, "count": count, "global_batch": global_batch,
                "scaling": "weak" if weak else "strong"}
    r0, r1 = fdist.row_band(cfg["h"], ws, rank, cfg["levels"])
    return {"kind": "rows", "r0": r0, "r1": r1, "global_batch": 1, "scaling": "strong"}


def make_inputs(name, cfg, ws, rank, weak=False):
    """This rank's shard of the workload as a pinned host array (datagen, seeded per unit)."""
    import torch

    import datagen
    sh = shard_of(cfg, ws, rank, weak)
    if sh["kind"] == "units":
        first, count = sh["first"], sh["count"]
        shape = (count, cfg["h"], cfg["w"]) if cfg["shard"] == "image" else (count, cfg["n"])
        host = torch.empty(shape, dtype=torch.float32).pin_memory()
        datagen.generate("c4" if cfg["shard"] == "image" else "c2", first=first, count=count, size=shape[-1],
                         out=host.numpy())
        units = f"{cfg['shard']}s [{first}, {first + count})"
    else:
        r0, r1 = sh["r0"], sh["r1"]
        host = torch.empty((r1 - r0, cfg["w"]), dtype=torch.float32).pin_memory()
        datagen.generate("c5", r0=r0, r1=r1, size=cfg["h"], out=host.numpy())
        units = f"rows [{r0}, {r1})"
    return host, units, sh


# ---------------------------------------------------------------------------------- GPU arm
def measure(name, cfg, args, ws, rank, local, pg, timed=True):
    import torch
    import torch.distributed as dist

    import paper_1002_2184_b200 as fhwt
    from paper_1002_2184_b200 import dist as fdist
    dev = torch.device("cuda", local)
    t0 = time.time()
    host, units, shard = make_inputs(name, cfg, ws, rank, weak=getattr(args, "weak", False))
    log(f"[rank {rank}] {name}: generated {tuple(host.shape)} ({units}) in {time.time() - t0:.1f}s")
    d = host.to(dev)
    coeffs = torch.empty_like(d)
    rec = torch.empty_like(d)
    L = cfg["levels"]
    if cfg["kind"] == "2d":
        plan = fhwt.Plan2d(d.shape[-2], d.shape[-1], d.numel() // (d.shape[-2] * d.shape[-1]), L, device=local)
    else:
        plan = fhwt.Plan1d(d.shape[-1], d.numel() // d.shape[-1], L, device=local)
    wsb = torch.empty(max(plan.workspace_bytes, 1), dtype=torch.uint8, device=dev)
    rowband = cfg["shard"] == "rowband"
    gather = rowband and (ws > 1 or getattr(args, "force_gather", False))
    p2p = None
    if rowband:
        ll_rows, ll_cols = d.shape[0] >> L, d.shape[1] >> L
        ll_local = torch.empty((ll_rows, ll_cols), dtype=torch.float32, device=dev)
        ll_all = torch.empty((ll_rows * ws, ll_cols), dtype=torch.float32, device=dev)
        if getattr(args, "ll_gather", "nccl") == "p2p" and dist.is_initialized():
            # pack fused with the all-gather over NVLink peer memory (one kernel + a device barrier)
            p2p = fdist.PeerLLGather(ll_rows, ll_cols, group=pg, device=dev)
    side = torch.cuda.Stream(dev)     # c5: LL pack + all-gather, overlapped with the synthesis pass
    ana_done = torch.cuda.Event()

    def ana():
        plan.analyze(d, out=coeffs, workspace=wsb)

    def rest(stream, mid_evs=None):
        """Everything after the analysis: (c5) pack + all-gather of the coarsest LL on the side
        stream — synthesis needs only the band's own coefficients — and synthesis."""
        if rowband:
            ana_done.record(stream)
            side.wait_event(ana_done)
            with torch.cuda.stream(side):
                if mid_evs:
                    mid_evs[0].record(side)
                if p2p is not None:
                    p2p(coeffs, L, stream=side)
                else:
                    fhwt.pack_ll_2d(coeffs, L, out=ll_local, stream=side)
                    if gather:
                        fdist.gather_coarse_ll(ll_local, group=pg, out=ll_all)
                if mid_evs:
                    mid_evs[1].record(side)
        plan.synthesize(coeffs, out=rec, workspace=wsb)
        if rowband:
            stream.wait_stream(side)      # the step ends when the gathered LL is in place too

    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):      # eager warm-up (allocations, TMA descriptors, NCCL setup)
        ana()
        rest(stream)
    torch.cuda.synchronize(dev)

    # The per-rank step as CUDA graphs (one for the analysis, one for the rest), so the K timed
    # steps replay them back to back; a CUDA event between the two replays times the analysis.
    # Not capturable: the gloo plumbing backend (host-side gather) and the peer-memory gather.
    graphs = None
    graph_note = "eager"
    n_per_step = None
    if not getattr(args, "no_graph", False) and p2p is None and not (gather and dist.get_backend(pg) != "nccl"):
        try:
            cs = torch.cuda.Stream(dev)
            cs.wait_stream(stream)
            g_ana, g_rest = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            n0 = fhwt.launch_count()
            with torch.cuda.stream(cs):
                with torch.cuda.graph(g_ana, stream=cs):
                    ana()
                with torch.cuda.graph(g_rest, stream=cs):
                    rest(cs)
            n_per_step = fhwt.launch_count() - n0
            stream.wait_stream(cs)
            for _ in range(2):
                g_ana.replay()
                g_rest.replay()
            torch.cuda.synchronize(dev)
            graphs = (g_ana, g_rest)
            graph_note = "CUDA graphs (analysis | pack + gather + synthesis), replayed"
        except Exception as e:  # noqa: BLE001
            log(f"[rank {rank}] graph capture failed ({e!r}); timing eager launches")
            graph_note = f"eager (capture failed: {type(e).__name__})"
            torch.cuda.synchronize(dev)

    def step(evs=None):
        if evs:
            evs[0].record(stream)
        if graphs:
            graphs[0].replay()
        else:
            ana()
        if evs:
            evs[1].record(stream)
        if graphs:
            graphs[1].replay()
        else:
            rest(stream)
        if evs:
            evs[2].record(stream)

    step()
    torch.cuda.synchronize(dev)
    # properties of this run's own output (not timed), on every rank
    checks = run_checks(name, cfg, host, d, coeffs, rec, plan, shard, L, rank, ws, pg, dev,
                        ll_local if rowband else None, (p2p.buf if p2p is not None else ll_all) if gather else None)

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    if ws > 1:
        dist.barrier(group=pg)
    torch.cuda.synchronize(dev)
    n0 = fhwt.launch_count()
    with ClockSampler(local) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for k in range(K):
            step(evs[k])
        end.record(stream)
        torch.cuda.synchronize(dev)
    launches = fhwt.launch_count() - n0 if graphs is None else n_per_step * K
    if ws > 1:
        dist.barrier(group=pg)
    total_ms = start.elapsed_time(end)
    # the side-stream pack + gather, timed in eager steps outside the timed region (graph replays
    # cannot hold events on the side stream)
    mid = []
    if rowband:
        for _ in range(min(K, 10)):
            me = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ana()
            rest(stream, me)
            torch.cuda.synchronize(dev)
            mid.append(me[0].elapsed_time(me[1]))
    sustained = None
    if getattr(args, "sustained", 0) > 0 and name == args.workload and timed:
        def eager_step():   # the variants are chosen per launch (env knobs), so no graph replays here
            ana()
            rest(stream)
        sustained = measure_sustained(eager_step, stream, local, total_ms / K, args.sustained,
                                      16.0 * d.numel() * ws)
    ana_t = [e[0].elapsed_time(e[1]) for e in evs]
    syn_t = [e[1].elapsed_time(e[2]) for e in evs]      # synthesis (+ the gather's tail, if any)
    vals = [total_ms, statistics.mean(ana_t), statistics.mean(syn_t), statistics.mean(mid) if mid else 0.0]
    if ws > 1:
        vals = fdist.max_over_ranks(vals, device=dev, group=pg)
    total_ms, ana_ms, syn_ms, mid_ms = vals
    samples_rank = d.numel()
    samples_all = samples_rank * ws if shard["scaling"] == "weak" or rowband else fdist_total(cfg, ws, pg, samples_rank, dev)
    ms_step = total_ms / K
    bytes_step = 16.0 * samples_all
    peak, peak_src = measured_peak()
    kern = "analysis" if ana_ms >= syn_ms else "synthesis"
    kern_ms = max(ana_ms, syn_ms)
    achieved = 8.0 * samples_rank / (kern_ms * 1e-3) / 1e9
    steps_ms = [e[0].elapsed_time(e[2]) for e in evs]

    def mmm(xs):   # median with min / max (this rank's per-step CUDA-event times, ms)
        return {"median": statistics.median(xs), "min": min(xs), "max": max(xs)} if xs else None

    res = {
        "per_step_ms": {"analysis": mmm(ana_t), "synthesis": mmm(syn_t), "pack_gather_eager": mmm(mid),
                        "step": mmm(steps_ms)},
        "gsamples_per_s_analysis": samples_rank / (ana_ms * 1e-3) / 1e9,
        "gsamples_per_s_synthesis": samples_rank / (syn_ms * 1e-3) / 1e9,
        "value": bytes_step / (ms_step * 1e-3) / 1e9,
        "gsamples_per_s": samples_all / (ms_step * 1e-3) / 1e9,
        "ms_per_step": ms_step,
        "analysis_ms": ana_ms, "synthesis_ms": syn_ms, "gather_ms": mid_ms,
        "analysis_gbs": 8.0 * samples_rank / (ana_ms * 1e-3) / 1e9,
        "synthesis_gbs": 8.0 * samples_rank / (syn_ms * 1e-3) / 1e9,
        "gpu_launches": launches,
        "launch_mode": graph_note,
        "clocks": clk.summary(),
        "roofline": {
            "bound": "hbm", "kernel": KERNEL_NAMES[(cfg["kind"], kern)],
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": peak_src,
            "algorithmic_bytes_per_launch": 8 * samples_rank,
            "traffic": ncu_traffic(name, kern),
        },
        "samples_per_rank": samples_rank,
        "samples_all": samples_all,
        "units": units,
        "shard": shard,
        "parity": checks,
        "sustained": sustained,
    }
    del d, coeffs, rec, wsb
    torch.cuda.empty_cache()
    return res, (plan, host)


def fdist_total(cfg, ws, pg, samples_rank, dev):
    """Strong scaling: the samples all ranks processed (shares can differ by one unit)."""
    if ws == 1:
        return samples_rank
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(samples_rank)], dtype=torch.float64,
                     device=dev if dist.get_backend(pg) == "nccl" else "cpu")
    dist.all_reduce(t, group=pg)
    return int(t.item())


def run_checks(name, cfg, host, d, coeffs, rec, plan, shard, L, rank, ws, pg, dev, ll_local, ll_gathered):
    """Properties of this run's own output that hold at any size, on the device, on EVERY rank,
    reduced to rank 0 (max of errors, min of booleans).  The oracle comparisons live in
    tests/test_gpu_fullsize.py and tests/test_gpu_parity.py; bench executes oracle/ only in its
    cpu_baseline and --impl reference legs.
    * per unit: round trip |d_R - d| / max|d| and the energy defect of the orthonormal transform
      (fp64 on the device);
    * P-invariance: the rank's first unit transformed alone (c2 / c4), or each
      half of the rank's row band transformed on its own (c5), equals bitwise the corresponding
      coefficients of the rank's batch / band output — so a split into 2N ranks gives the bits of a
      split into N, and by induction of N = 1;
    * (c5, N > 1) the all-gathered coarsest LL on this rank against a rank-local reference of every
      band, 2^L * avg_pool(band, 2^L) in fp64 (each rank's reference all-gathered the same way), and
      identical on all ranks (checksum min == max)."""
    import torch
    import torch.distributed as dist

    import paper_1002_2184_b200 as fhwt
    from paper_1002_2184_b200 import dist as fdist
    rowband = shard["kind"] == "rows"
    dims = tuple(range(1, host.dim())) if not rowband else (0, 1)
    rts, ens = [], []
    n = host.shape[0] if not rowband else 1
    stepn = max(1, n // 8)
    for i0 in range(0, n, stepn):   # a few units at a time keeps the fp64 temporaries small
        sl = slice(i0, min(n, i0 + stepn)) if not rowband else slice(None)
        x = d[sl].double()
        scale = x.abs().amax(dim=dims)
        rts.append(float(((rec[sl].double() - x).abs().amax(dim=dims) / scale).max()))
        e_in = (x * x).sum(dim=dims)
        ens.append(float((((coeffs[sl].double() ** 2).sum(dim=dims) - e_in).abs() / e_in).max()))
        del x
    torch.cuda.empty_cache()
    # P-invariance
    if not rowband:
        one = (fhwt.analyze_2d(d[:1].contiguous(), L) if cfg["kind"] == "2d" else fhwt.analyze_1d(d[:1].contiguous(), L))
        p_inv = bool(torch.equal(one, coeffs[:1]))
        del one
    else:
        H, W = d.shape
        p_inv = True
        if H % (2 << L) == 0:
            for r0, r1 in ((0, H // 2), (H // 2, H)):
                half = fhwt.analyze_2d(d[r0:r1], L)
                hb = r1 - r0
                for j in range(1, L + 1):
                    g0, g1 = fdist.band_rows(r0, r1, j)
                    hj, wj, bj = H >> j, W >> j, hb >> j
                    p_inv &= bool(torch.equal(half[:bj, wj:2 * wj], coeffs[g0:g1, wj:2 * wj]))
                    p_inv &= bool(torch.equal(half[bj:2 * bj, :wj], coeffs[hj + g0:hj + g1, :wj]))
                    p_inv &= bool(torch.equal(half[bj:2 * bj, wj:2 * wj], coeffs[hj + g0:hj + g1, wj:2 * wj]))
                p_inv &= bool(torch.equal(half[:hb >> L, :W >> L], coeffs[g0:g1, :W >> L]))
                del half
        torch.cuda.empty_cache()
    out = {"check": "every unit: round trip and energy (fp64 on device); P-invariance; gathered LL (c5, N>1)",
           "roundtrip_err_rel": max(rts), "energy_defect_rel": max(ens), "tol": 1e-5, "p_invariant": p_inv}
    if rowband:
        # the band's own packed LL against 2^L * avg_pool of its input (fp64, rank-local reference)
        x = d.double()[None, None]
        ref_local = (torch.nn.functional.avg_pool2d(x, 1 << L) * float(1 << L))[0, 0]
        scale_local = float(d.abs().max())
        out["packed_ll_err_rel"] = float((ll_local.double() - ref_local).abs().max()) / scale_local
        if ll_gathered is not None:
            nccl = dist.get_backend(pg) == "nccl"
            dv = dev if nccl else "cpu"
            ref_all = torch.empty((ws * ref_local.shape[0], ref_local.shape[1]), dtype=torch.float64, device=dv)
            if nccl:
                dist.all_gather_into_tensor(ref_all, ref_local.contiguous(), group=pg)
            else:
                parts = [torch.empty_like(ref_local.cpu()) for _ in range(ws)]
                dist.all_gather(parts, ref_local.cpu().contiguous(), group=pg)
                ref_all.copy_(torch.cat(parts, 0))
            sc = fdist.max_over_ranks(scale_local, device=dev, group=pg)
            g = ll_gathered.double().to(dv)
            err = float((g - ref_all).abs().max()) / sc
            ck = float(g.sum())
            out["gathered_ll_err_rel"] = err
            out["gathered_ll_identical_on_all_ranks"] = (fdist.max_over_ranks(ck, device=dev, group=pg) ==
                                                         -fdist.max_over_ranks(-ck, device=dev, group=pg))
        del x, ref_local
    if ws > 1:   # reduce to rank 0: max of errors, min (AND) of booleans
        keys = [k for k, v in out.items() if isinstance(v, float)]
        vals = fdist.max_over_ranks([out[k] for k in keys], device=dev, group=pg)
        out.update(zip(keys, vals))
        bkeys = [k for k, v in out.items() if isinstance(v, bool)]
        bvals = fdist.max_over_ranks([0.0 if out[k] else 1.0 for k in bkeys], device=dev, group=pg)
        out.update({k: v == 0.0 for k, v in zip(bkeys, bvals)})
        out["ranks_checked"] = ws
    return out


# Tile-order variants compared under sustained load (profiles/r02_dynamic_tiles.md):
# the default hands K1's and K4's tiles out in global order from a counter; "static_order" is the
# round-1 persistent assignment (CTA i takes tiles i, i + grid, ...) with the round-1 K4.
SUSTAINED_VARIANTS = {"default": {},
                      "static_order": {"FHWT_TUNING": "1", "FHWT_ANA_DYN": "0", "FHWT_SYN_PROD": "0"}}


def measure_sustained(step, stream, local, ms_per_step, seconds, bytes_per_step):
    """Back-to-back steps for `seconds` of warm load, then `seconds` timed (CUDA events), per
    analysis variant, with NVML SM clock / board power / clock-event reasons sampled during the
    timed part: the regime of a long streaming job, where the board power cap lowers SM clocks."""
    import threading

    import torch
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(local)
    except Exception:  # noqa: BLE001
        nv = h = None
    n = max(10, int(seconds * 1e3 / max(ms_per_step, 1e-3)))
    out = {}
    saved = {k: os.environ.get(k) for v in SUSTAINED_VARIANTS.values() for k in v}
    for name, env in SUSTAINED_VARIANTS.items():
        for k in saved:
            os.environ.pop(k, None)
        os.environ.update(env)
        for _ in range(n):
            step()
        samples, stop = [], threading.Event()

        def poll():
            while not stop.is_set() and h is not None:
                try:
                    samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(h) / 1e3,
                                    nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(0.02)

        th = threading.Thread(target=poll, daemon=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        th.start()
        e0.record(stream)
        for _ in range(n):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = e0.elapsed_time(e1) / n
        reasons = 0
        for x in samples:
            reasons |= x[2]
        out[name] = {"env": env, "value": bytes_per_step / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
                     "steps": n, "sm_mhz_median": statistics.median(x[0] for x in samples) if samples else None,
                     "power_w_median": statistics.median(x[1] for x in samples) if samples else None,
                     "clock_event_reasons": hex(reasons), "sw_power_cap": bool(reasons & 0x4)}
    for k, v in saved.items():
        os.environ.pop(k, None)
        if v is not None:
            os.environ[k] = v
    return out


def measure_direct(name, cfg, d_host, steps=5):
    """§8(f) f3: the paper's original structure (Figs. 2 and 5, full-rate filtering, materialised
    intermediates, level by level) on the same GPU and workload, next to static op counts."""
    import torch

    import paper_1002_2184_b200 as fhwt
    d = d_host.to("cuda")
    c = torch.empty_like(d)
    r = torch.empty_like(d)
    L = cfg["levels"]
    if cfg["kind"] == "2d":
        shape, batch = (cfg["h"], cfg["w"]), d.shape[0]
        ws = torch.empty(fhwt.direct_workspace_bytes(2, shape[0], shape[1], batch), dtype=torch.uint8, device="cuda")
        ana = lambda: fhwt.direct_analyze_2d(d, L, out=c, workspace=ws)  # noqa: E731
        syn = lambda: fhwt.direct_synthesize_2d(c, L, out=r, workspace=ws)  # noqa: E731
    else:
        shape, batch = (cfg["n"],), d.shape[0]
        ws = torch.empty(fhwt.direct_workspace_bytes(1, shape[0], 0, batch), dtype=torch.uint8, device="cuda")
        ana = lambda: fhwt.direct_analyze_1d(d, L, out=c, workspace=ws)  # noqa: E731
        syn = lambda: fhwt.direct_synthesize_1d(c, L, out=r, workspace=ws)  # noqa: E731
    for _ in range(2):
        ana()
        syn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(steps):
        ana()
    e[1].record()
    for _ in range(steps):
        syn()
    e[2].record()
    torch.cuda.synchronize()
    ta, ts = e[0].elapsed_time(e[1]) / steps, e[1].elapsed_time(e[2]) / steps
    err = float((r - d).abs().max() / d.abs().max())
    S = d.numel()
    ops = {}
    for st in ("direct", "fast", "kernel"):
        ma, aa = fhwt.op_counts(shape, L, st, batch=batch)
        ms, as_ = fhwt.op_counts(shape, L, st, synthesis=True, batch=batch)
        ops[st] = {"analysis_mul": ma, "analysis_add": aa, "synthesis_mul": ms, "synthesis_add": as_}
    del d, c, r, ws
    torch.cuda.empty_cache()
    return {"structure": "Fig. 2 / Fig. 5 direct form, level by level, intermediates in HBM",
            "analysis_ms": ta, "synthesis_ms": ts, "ms_per_step": ta + ts,
            "value": 16.0 * S / ((ta + ts) * 1e-3) / 1e9, "unit": "GB/s (same 16 B/sample algorithmic bytes)",
            "roundtrip_err_rel": err, "op_counts": ops,
            "mul_ratio_fast_over_direct": ops["fast"]["analysis_mul"] / ops["direct"]["analysis_mul"]}


def measure_latency(iters=200):
    """c1 (1 x 1024, J=1) and c3 (512^2, L=3) are latency-bound: microseconds per
    DWT+IDWT, eager launches vs one CUDA graph replay of the two launches; parity of the output."""
    import torch

    import datagen
    import paper_1002_2184_b200 as fhwt
    out = {}
    cases = {"c1": (datagen.c1_signal()[None], fhwt.Plan1d(1024, 1, 1), 1),
             "c3": (datagen.c3_image()[None], fhwt.Plan2d(512, 512, 1, 3), 3)}
    for name, (x_np, plan, L) in cases.items():
        x = torch.from_numpy(x_np).cuda()
        c = torch.empty_like(x)
        r = torch.empty_like(x)

        def step():
            plan.analyze(x, out=c)
            plan.synthesize(c, out=r)

        for _ in range(20):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            step()
        e1.record()
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / iters * 1e3
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            step()
        for _ in range(20):
            g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / iters * 1e3
        rt = float((r - x).abs().max() / x.abs().max())
        out[name] = {"eager_us_per_dwt_idwt": eager, "graph_us_per_dwt_idwt": graph, "samples": x.numel(),
                     "roundtrip_err_rel": rt}
    return out


def measure_lowpass(steps=10):
    """§8(f) f1: LL-only lowpass of the c4 images in their native uint8 form (Fig. 12):
    reads 1 B/pixel, writes LL_5 only.  Algorithmic bytes per launch = S (uint8 in) + 4 S / 4^5."""
    import torch

    import datagen
    import paper_1002_2184_b200 as fhwt
    cfg = WORKLOADS["c4"]
    host = torch.empty((cfg["batch"], cfg["h"], cfg["w"]), dtype=torch.uint8).pin_memory()
    datagen.generate("c4u8", count=cfg["batch"], out=host.numpy())
    d = host.cuda()
    L = cfg["levels"]
    out = torch.empty((cfg["batch"], cfg["h"] >> L, cfg["w"] >> L), device="cuda")
    for _ in range(3):
        fhwt.lowpass_2d_u8(d, L, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fhwt.lowpass_2d_u8(d, L, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    S = d.numel()
    alg = S + 4 * S / 4 ** L
    peak, src = measured_peak()
    full = fhwt.analyze_2d(d[7].float().contiguous(), L)[: cfg["h"] >> L, : cfg["w"] >> L]
    same = bool((full == out[7]).all())
    # bf16 input variant (same images as bf16: exact for 0..255): 2 B/pixel read
    db = d.to(torch.bfloat16)
    del d
    for _ in range(3):
        fhwt.lowpass_2d_bf16(db, L, out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        fhwt.lowpass_2d_bf16(db, L, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms16 = e0.elapsed_time(e1) / steps
    alg16 = 2 * S + 4 * S / 4 ** L
    full16 = fhwt.analyze_2d(db[7].float().contiguous(), L)[: cfg["h"] >> L, : cfg["w"] >> L]
    same16 = bool((full16 == out[7]).all())
    bf16 = {"ms": ms16, "gbs": alg16 / (ms16 * 1e-3) / 1e9, "gpix_per_s": S / (ms16 * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": alg16 / (ms16 * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg16 / (ms16 * 1e-3) / 1e9 / peak, "peak_source": src,
                         "algorithmic_bytes_per_launch": alg16},
            "parity": {"unit": "image 7", "bitwise_equal_to_fused_transform_LL": same16}}
    del db
    torch.cuda.empty_cache()
    return {"workload": "c4 images as uint8 (256 x 2048^2), LL_5 only", "ms": ms,
            "gbs": alg / (ms * 1e-3) / 1e9, "gpix_per_s": S / (ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": alg / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (ms * 1e-3) / 1e9 / peak, "peak_source": src,
                         "algorithmic_bytes_per_launch": alg},
            "parity": {"unit": "image 7", "bitwise_equal_to_fused_transform_LL": same},
            "bf16_input": bf16}


def measure_e2e(cfg, host, steps):
    """Same metric through the public host-buffer API: every step copies the pinned input H2D, runs
    DWT + IDWT and copies the step's result d_R back D2H (fhwt_roundtrip_*_host; the coefficients
    are the step's intermediate and stay on the device).  Also the PCIe copy rates seen in this
    process, for the e2e roofline."""
    import torch

    import paper_1002_2184_b200 as fhwt
    out = torch.empty_like(host).pin_memory()
    fn = fhwt.roundtrip_2d_host if cfg["kind"] == "2d" else fhwt.roundtrip_1d_host
    L = cfg["levels"]
    fn(host, L, out=out)           # warm-up (pool allocation)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        fn(host, L, out=out)
        times.append(time.perf_counter() - t0)
    s = host.numel()
    t = statistics.median(times)
    # PCIe reference: one pinned H2D and one D2H of the same bytes, concurrently on two streams
    # (separate device source and destination, best of 3; the round trip cannot beat this plus
    # one chunk of pipeline fill and drain)
    dbuf = torch.empty(host.shape, dtype=host.dtype, device="cuda")
    dsrc = torch.zeros(host.shape, dtype=host.dtype, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t_duplex = None
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            dbuf.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2):
            out.copy_(dsrc, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t_duplex = dt if t_duplex is None else min(t_duplex, dt)
    del dbuf, dsrc
    return {"value": 16.0 * s / t / 1e9, "unit": "GB/s", "gsamples_per_s": s / t / 1e9,
            "ms_per_step": t * 1e3, "steps": steps,
            "h2d_bytes_per_step": 4 * s, "d2h_bytes_per_step": 4 * s,
            "pcie_duplex_ms_same_bytes": t_duplex * 1e3,
            "frac_of_pcie_duplex": t_duplex / t,
            "api": "fhwt_roundtrip_%s_host (pinned host buffers; chunked H2D, DWT, IDWT, D2H of d_R on 3 CUDA streams)"
                   % ("2d" if cfg["kind"] == "2d" else "1d")}


# ---------------------------------------------------------------------------------- oracle arm
def _oracle_unit(args):
    kind, idx, n_or_size, levels = args
    import datagen
    import oracle
    if kind == "c4":
        x = datagen.c4_image(idx, n_or_size)
        t0 = time.perf_counter()
        r = oracle.synthesize_2d(oracle.analyze_2d(x, levels), levels)
    elif kind == "c2":
        x = datagen.c2_signal(idx, n_or_size)
        t0 = time.perf_counter()
        r = oracle.reconstruct_1d(oracle.decompose_1d(x, levels), levels)
    else:
        x = datagen.c5_rows(idx * 256, idx * 256 + 256, size=n_or_size)
        t0 = time.perf_counter()
        r = oracle.synthesize_2d(oracle.analyze_2d(x, levels), levels)
    dt = time.perf_counter() - t0
    assert np.abs(r - x).max() <= 1e-9 * max(1.0, np.abs(x).max())
    return x.size, dt


def time_oracle(name, cfg, budget_s=20.0):
    """The fp64 oracle, as it stands, on a bounded sample of the workload, one process per core."""
    from concurrent.futures import ProcessPoolExecutor
    cores = min(len(os.sched_getaffinity(0)), 64)
    if name == "c4":
        per = 1.2                               # ~seconds per 2048^2 image DWT+IDWT (one core)
        units = max(1, min(cfg["batch"], int(budget_s / per * cores)))
        tasks = [("c4", i, cfg["h"], cfg["levels"]) for i in range(units)]
        sample = f"{units} of the {cfg['batch']} c4 images (DWT+IDWT, L=5)"
    elif name == "c2":
        units = max(1, min(cfg["batch"], int(budget_s / 0.006 * cores)))
        tasks = [("c2", i, cfg["n"], cfg["levels"]) for i in range(units)]
        sample = f"{units} of the {cfg['batch']} c2 signals (DWT+IDWT, J=10)"
    else:
        units = max(1, min(cfg["h"] // 256, int(budget_s / 2.3 * cores)))
        tasks = [("c5", i, cfg["h"], min(cfg["levels"], 8)) for i in range(units)]
        sample = f"{units} of the 128 256-row bands of c5 (each band DWT+IDWT with L=8 — band-local, halo-free)"
    import multiprocessing as mp
    t0 = time.perf_counter()
    with ProcessPoolExecutor(cores, mp_context=mp.get_context("forkserver")) as ex:
        res = list(ex.map(_oracle_unit, tasks))
    wall = time.perf_counter() - t0
    samples = sum(r[0] for r in res)
    return {"value": 16.0 * samples / wall / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "gsamples_per_s": samples / wall / 1e9, "wall_s": wall,
            "sample": sample + f", fp64 numpy direct form (oracle/haar.py), {cores} worker processes"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = WORKLOADS[args.workload]
    steps = []
    per_step_budget = max(3.0, 120.0 / max(1, args.steps))
    for i in range(args.warmup + args.steps):
        r = time_oracle(args.workload, cfg, budget_s=per_step_budget if i >= args.warmup else 0.5)
        if i >= args.warmup:
            steps.append(r)
    v = statistics.median(s["value"] for s in steps)
    cb = dict(steps[0])
    cb["value"] = v
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(s["wall_s"] for s in steps),
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "levels": cfg["levels"]},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference arm is the fp64 CPU oracle (no reference implementation exists); each step is a bounded sample",
    }
    emit(out)
    return 0


# ---------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fhwt", choices=["fhwt", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--no-breakdown", action="store_true", help="skip the c2/c5 secondary measurements")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-direct", action="store_true", help="skip the direct-form (Fig. 2/5) baseline")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only for plumbing checks (FHWT_BENCH_ONE_DEVICE=1 on one GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ll-gather", default="nccl", choices=["nccl", "p2p"],
                    help="c5 coarse-LL exchange: NCCL all-gather, or pack + stores into peer symmetric memory")
    ap.add_argument("--sustained", type=float, default=1.5,
                    help="seconds of warm + timed back-to-back steps per analysis variant (0 = skip)")
    ap.add_argument("--weak", action="store_true",
                    help="c2 / c4: every rank transforms a full batch (weak scaling) instead of batch/N units")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA graph replays")
    ap.add_argument("--force-gather", action="store_true",
                    help="check of the N > 1 code path on one GPU: c5's LL all-gather through a one-rank NCCL "
                         "group, captured in the CUDA graph like at N > 1")
    ap.add_argument("--no-t1", action="store_true",
                    help="N > 1: skip rank 0's single-GPU run of the whole workload (the T(1) of the self-check)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if os.environ.get("FHWT_BENCH_ONE_DEVICE"):   # plumbing check only: all ranks share cuda:0 (gloo)
        local = 0
    torch.cuda.set_device(local)
    pg = None
    if ws > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
        pg = dist.group.WORLD
    elif args.ll_gather == "p2p" or args.force_gather:   # one GPU: a one-rank group exercises the gather path
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        pg = dist.group.WORLD
    cfg = WORKLOADS[args.workload]
    res, (plan, host) = measure(args.workload, cfg, args, ws, rank, local, pg)
    lowpass = latency = None
    if not args.no_breakdown and rank == 0:
        lowpass = measure_lowpass()
        latency = measure_latency()
    direct = None
    if not args.no_direct and rank == 0:
        direct = measure_direct(args.workload, cfg, host)
        direct["fast_speedup"] = direct["ms_per_step"] / res["ms_per_step"]
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(cfg, host, args.e2e_steps)
        if ws > 1:
            from paper_1002_2184_b200 import dist as fdist
            e2e["ms_per_step"] = fdist.max_over_ranks(e2e["ms_per_step"], device=torch.device("cuda", local), group=pg)
            e2e["value"] = 16.0 * res["samples_all"] / (e2e["ms_per_step"] * 1e-3) / 1e9
            e2e["h2d_bytes_per_step"] = e2e["d2h_bytes_per_step"] = 4 * res["samples_all"]
            e2e["note"] = "every rank round-trips its own shard; bytes are the whole job's"
    del host
    multi = None
    if ws > 1:
        # Self-check of the scaling (the driver computes the official efficiency from its own per-N
        # runs): rank 0 times the whole workload alone on its GPU, T(1), next to this run's T(N).
        multi = {"t_n_ms": res["ms_per_step"], "shard_per_rank": res["shard"],
                 "gather_ms": res["gather_ms"] if cfg["shard"] == "rowband" else None}
        if not args.no_t1 and not args.weak:
            if rank == 0:
                sub = argparse.Namespace(**vars(args))
                sub.sustained = 0
                r1, (p1, h1) = measure(args.workload, cfg, sub, 1, 0, local, None, timed=False)
                del p1, h1
                multi.update(t1_ms=r1["ms_per_step"], t1_value=r1["value"],
                             self_check_efficiency=r1["ms_per_step"] / (ws * res["ms_per_step"]),
                             note="T(1)/(N*T(N)) with T(1) timed by rank 0 alone in this run; "
                                  "the driver's own per-N runs are authoritative")
            dist.barrier(group=pg)
    breakdown = {}
    if not args.no_breakdown:
        for other in ("c2", "c5", "c4"):
            if other == args.workload:
                continue
            sub_args = argparse.Namespace(**vars(args))
            sub_args.steps = max(20, args.steps)   # >= 20 timed iterations
            r2, (p2, h2) = measure(other, WORKLOADS[other], sub_args, ws, rank, local, pg)
            del p2, h2
            breakdown[other] = {k: r2[k] for k in ("value", "gsamples_per_s", "ms_per_step", "analysis_ms",
                                                    "synthesis_ms", "gather_ms", "analysis_gbs", "synthesis_gbs",
                                                    "gsamples_per_s_analysis", "gsamples_per_s_synthesis",
                                                    "per_step_ms", "roofline", "parity", "gpu_launches", "clocks")}
            breakdown[other]["workload"] = WORKLOADS[other]["desc"]
            breakdown[other]["scaling"] = r2["shard"]["scaling"]
            breakdown[other]["launch_mode"] = r2["launch_mode"]
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = time_oracle(args.workload, cfg)
    if rank == 0:
        out = {
            "metric": METRIC, "value": res["value"], "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": res["shard"]["scaling"], "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["desc"], "levels": cfg["levels"],
                       "global_batch": res["shard"]["global_batch"],
                       "per_rank": res["units"],
                       "shape": [cfg.get("h"), cfg.get("w")] if cfg["kind"] == "2d" else [cfg["n"]],
                       "parallelism": f"dp{ws} ({cfg['shard']} shards, {res['shard']['scaling']} scaling)",
                       "launch": res["launch_mode"],
                       "l2": "no flush: every step streams >= 4 GiB in and out, >> 126 MB L2",
                       "dtype_note": "fp32 I/O and levels 1-3; fp64 butterflies from level 4 (analysis)"},
            "gsamples_per_s": res["gsamples_per_s"],
            "kernels": {k: res[k] for k in ("analysis_ms", "synthesis_ms", "gather_ms", "analysis_gbs", "synthesis_gbs",
                                            "gsamples_per_s_analysis", "gsamples_per_s_synthesis", "per_step_ms")},
            "roofline": res["roofline"],
            "sustained": res["sustained"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": res["gpu_launches"],
            "clocks": res["clocks"],
            "parity": res["parity"],
            "multi_gpu": multi,
            "workloads": breakdown,
            "direct_form": direct,
            "lowpass_u8": lowpass,
            "latency": latency,
        }
        emit(out)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _json_stdout():
    """Keep stdout to the one JSON line: library banners written to fd 1 (NCCL's version line,
    symmetric-memory notices) are sent to stderr, and the JSON line goes to a saved copy of fd 1."""
    global _OUT
    try:
        sys.stdout.flush()
        _OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    except OSError:
        _OUT = sys.stdout


_OUT = sys.stdout


def emit(obj):
    print(json.dumps(obj), file=_OUT, flush=True)


if __name__ == "__main__":
    _json_stdout()
    sys.exit(main())
