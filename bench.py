#!/usr/bin/env python
"""Benchmark of the TILES tile-wise Reslim forward (ORBIT-2) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the whole hot path (gather -> embed -> L blocks ->
head -> stitch + bilinear residual) over one batch of synthetic ERA5-shaped
input (BASELINE.json configs[1] = C2 at N=1, B = 64 samples).  Multi-GPU
(one process per GPU; `--gpus N` re-executes itself under torch.distributed.run
when WORLD_SIZE is unset): the SAME batch's tiles are partitioned over the N
GPUs (LPT), the halo exchange and the output gather run through NVLink peer
memory inside the library (strong scaling); `--mode dp`
instead gives every rank its own batch (weak scaling).  Timing: CUDA events on
the launching stream, barrier + synchronize on both sides, max over ranks.

Prints ONE JSON line on rank 0.  See DESIGN.md §Measurement for every key.
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

METRIC = "high-res pixels/s & tiled-attn TFLOP/s (% bf16 peak) at 1/2/4/8 B200"
UNIT = "high-res px/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batch", type=int, default=0, help="override the config's bench batch")
    ap.add_argument("--chunk", type=int, default=-1, help="tiles per forward call (default: auto-fit HBM)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="sp", choices=["dp", "sp", "train", "compress", "sweep"],
                    help="N > 1 only.  sp (default): the tiles of one batch spread over the ranks, halo "
                         "exchange + output gather through NVLink peer memory (strong scaling); dp: every "
                         "rank its own batch (weak scaling).  train (any N): the training step (SURVEY "
                         "§8(f) row 3): forward, Bayesian loss, backward, one gradient all-reduce per batch.  "
                         "compress (N = 1): adaptive spatial compression (§8(f) row 4) of the batch's coarse "
                         "fields: Canny + quad-tree partition, variable-size tokens, decompression.  sweep "
                         "(N = 1): the tile-count sweep T in {1, 4, 16, 36} of the config (SURVEY §8(d), the "
                         "shape of Tab. P:379-381), CUDA-graph replay of the forward beside it")
    ap.add_argument("--lam", type=float, default=1e-3, help="train: TV prior weight lambda (R34)")
    ap.add_argument("--train-tiles", action="store_true",
                    help="train, N > 1: tile-parallel training (the SAME batch, its tiles over the ranks, the "
                         "field and the gradient summed with NCCL: training.TilesTrainSP; strong scaling) instead "
                         "of data parallel")
    ap.add_argument("--delta", type=float, default=1e-3, help="train: Huber width delta (R34)")
    ap.add_argument("--sp-groups", type=int, default=0,
                    help="N > 1: sample groups per rank (default 4 when the batch allows, else 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--set", action="append", default=[], metavar="FIELD=INT",
                    help="override a workload field (experiments only, e.g. --set tiles_y=2)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return {"hbm": j["hbm_gbs"], "bf16": j["bf16_tflops"], "bf16_sus": j["bf16_tflops_sustained"],
                "src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        load = [s for s in sm if smax and s > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_init(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def _sum_over_ranks(world, v: float) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(world, v: float) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# algorithmic work per kernel class
# ---------------------------------------------------------------------------
def class_work(w, info, B):
    """Per kernel class: (bound, total algorithmic work per step) with FLOPs
    for contractions and bytes for HBM-bound kernels."""
    D, L, Din, Nh, V, K = w.embed, w.depth, w.din, w.head_out, w.V, w.K
    npad, ncore = info.tokens_per_sample, info.core_tokens_per_sample
    n2, nc = info.sum_n2_per_sample, info.sum_nc_per_sample
    sH, sW = w.scale * w.H, w.scale * w.W
    last = 1 if L >= 1 else 0
    f = {
        "embed_gemm": 2.0 * npad * Din * D,
        "qkv_gemm": (L - last) * 6.0 * npad * D * D + last * (4.0 * npad * D * D + 2.0 * ncore * D * D),
        "tile_attention": (L - last) * 4.0 * D * n2 + last * 4.0 * D * nc,
        "oproj_gemm": (L - last) * 2.0 * npad * D * D + last * 2.0 * ncore * D * D,
        "mlp_up_gemm": (L - last) * 8.0 * npad * D * D + last * 8.0 * ncore * D * D,
        "mlp_down_gemm": (L - last) * 8.0 * npad * D * D + last * 8.0 * ncore * D * D,
        "head_gemm": 2.0 * ncore * D * Nh,
    }
    f["mlp_fused"] = f["mlp_up_gemm"] + f["mlp_down_gemm"]   # one kernel does both (D = 256)
    f["block_tail"] = f["oproj_gemm"] + f["mlp_fused"]        # O-proj + LN2 + MLP in one kernel (D = 256)
    out = {k: ("tensor", v * B) for k, v in f.items()}
    # HBM kernels: unique algorithmic bytes
    out["tile_gather"] = ("hbm", B * (4.0 * V * w.H * w.W + 2.0 * npad * Din))
    out["stitch_residual"] = ("hbm", B * (2.0 * K * sH * sW + 4.0 * K * w.H * w.W + 4.0 * K * sH * sW))
    # layernorm launches: fp32 read + bf16 write of D per row.  D = 256: LN1 of block 0
    # runs in the embedding GEMM's epilogue, LN2 and the next block's LN1 in the
    # block-tail kernel, leaving the final (core rows) LN; otherwise 2L + 1 launches.
    ln_full = 0 if D == 256 else 2 * L
    out["layernorm"] = ("hbm", B * (ln_full * npad * D * 6.0 + ncore * D * 6.0))
    return out


def auto_chunk(o2, w, B):
    """Largest number of tiles per forward/stitch call whose workspace and
    tile_out, plus the resident input and output fields, fit in 85% of free HBM."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    _, info = o2.orbit2_tiles_plan(o2.config_from(w, batch=B))
    fixed = info.out_bytes + B * w.V * w.H * w.W * 4 + 4 * o2.orbit2_tiles_plan(o2.config_from(w))[1].canonical_weight_count * 2
    n = info.n_local_tiles
    for div in range(1, n + 1):
        ch = -(-n // div)
        _, ci = o2.orbit2_tiles_plan(o2.config_from(w, batch=B, chunk_tiles=ch))
        if fixed + ci.workspace_bytes + ci.tile_out_bytes < 0.85 * free:
            return 0 if ch >= n else ch
    raise RuntimeError("workload does not fit one GPU even one tile at a time")


def class_bytes_embed(w, info, B):
    """Algorithmic HBM bytes of the embedding GEMM per step: bf16 patch rows in
    (2 Din), fp32 z out (4 D) and, when LN1 of block 0 is fused (D = 256), bf16 xn
    out (2 D); weights are negligible."""
    ln = 2.0 * w.embed if (w.embed == 256 and w.depth > 0) else 0.0
    return B * info.tokens_per_sample * (2.0 * w.din + 4.0 * w.embed + ln)


def host_cpu():
    """nproc and the /proc/cpuinfo model of the host the oracle runs on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def attn_bytes(w, info, B):
    """Algorithmic HBM bytes of one attention launch: read Q,K,V (bf16) once,
    write the head outputs (bf16) once, over all padded tokens."""
    return B * info.tokens_per_sample * (3 + 1) * w.embed * 2.0


def latest_traffic():
    """Per-launch DRAM traffic measured by the latest committed ncu capture."""
    import glob
    out = {}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic_*.json"))):
        try:
            with open(path) as f:
                for k, v in json.load(f).items():
                    v = dict(v)
                    v["source"] = os.path.relpath(path, ROOT)
                    out[k] = v
        except Exception:
            pass
    return out


# ---------------------------------------------------------------------------
# the oracle as the CPU baseline / reference arm
# ---------------------------------------------------------------------------
def oracle_units(w, blob, x, seconds_budget=None, n_units=None):
    """Run the oracle over (sample, tile) units; returns (units, high-res px, seconds, threads)."""
    from oracle import reslim_tiles as O
    pr = O.Problem.from_config(w)
    tiles = pr.tiles()
    Wt = pr.weights(blob)
    px = 0
    done = 0
    t0 = time.perf_counter()
    i = 0
    while True:
        b, t = divmod(i % (x.shape[0] * len(tiles)), len(tiles))
        tile = tiles[t]
        g = O.tile_forward(x[b], tile, pr, Wt)
        ys = slice(tile.core_y0 * pr.P, tile.core_y1 * pr.P)      # the oracle's step O7 on this tile's
        xs = slice(tile.core_x0 * pr.P, tile.core_x1 * pr.P)      # output block (stitch is a placement)
        up = [O.upsample_bilinear_region(x[b][m], pr.scale, ys, xs) for m in pr.cmap()]
        _ = g.sum() + sum(u.sum() for u in up)
        px += tile.n_core * pr.P * pr.P
        done += 1
        i += 1
        el = time.perf_counter() - t0
        if n_units is not None and done >= n_units:
            break
        if seconds_budget is not None and el >= seconds_budget:
            break
    try:
        from threadpoolctl import threadpool_info
        threads = max([p.get("num_threads", 1) for p in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    return done, px, time.perf_counter() - t0, threads


def run_reference(args, w, world, rank):
    """--impl reference: the fp64 oracle as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return
    from workloads import make_input, make_weights
    x = make_input(w, batch=1)
    blob = make_weights(w)
    for _ in range(args.warmup):
        oracle_units(w, blob, x, n_units=1)
    times, pxs = [], []
    for s in range(args.steps):
        _, px, dt, threads = oracle_units(w, blob, x, n_units=1)
        times.append(dt)
        pxs.append(px)
    total_t = sum(times)
    value = sum(pxs) / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (ERA5-shaped, seeded)",
        "config": {"workload": w.name, "batch": 1, "step": "one (sample, tile) unit of the workload"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"1 (sample, tile) unit of {w.name} per step (fp64 numpy oracle)", **host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, w, world, rank, local):
    import numpy as np
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    from workloads import make_input, make_weights

    B = w.batch
    chunk = args.chunk if args.chunk >= 0 else auto_chunk(o2, w, B)
    cfg = o2.config_from(w, batch=B, precision=o2.BF16, chunk_tiles=chunk)
    ctx = o2.Context(cfg)
    info = ctx.info
    blob = make_weights(w)
    x_host = make_input(w, batch=B, seed=1000 + 97 * rank + int(w.name[1]))
    x_pin = torch.from_numpy(x_host).pin_memory()
    x_dev = x_pin.to("cuda")
    packed = ctx.prepare_weights(torch.from_numpy(blob).cuda())
    out = torch.empty((B, w.K, w.scale * w.H, w.scale * w.W), dtype=torch.float32, device="cuda")
    out_pin = torch.empty(out.shape, dtype=torch.float32).pin_memory()
    tile_out = ctx.tile_out_buffer()
    stream = torch.cuda.current_stream()

    def step():
        ctx.forward(packed, x_dev, out=out, tile_out=tile_out, stream=stream)

    for _ in range(max(3, args.warmup)):
        step()
    barrier(world)

    # ---- device-resident timed region ----
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        barrier(world)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier(world)
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = (ctx.launch_count() - l0) // args.steps
    ms = max_over_ranks(world, ms)
    clocks = clk.summary()

    # ---- end-to-end through the public API with host buffers ----
    # Context.forward_host: pinned host input -> pinned host output for the whole
    # batch, in groups of B / E2E_GROUPS samples so the PCIe copies (both
    # directions) overlap the compute of the neighbouring groups
    h2d = x_pin.numel() * 4
    d2h = out.numel() * 4
    # 2 groups: with the copies overlapped across back-to-back calls the larger per-group batch
    # wins (C2: 39.3 ms vs 39.7 / 39.9 for 4 / 8 groups, profiles/r02ao)
    groups = int(os.environ.get("ORBIT2_E2E_GROUPS", "0")) or next(g for g in (2, 1) if B % g == 0)
    ctx_h = o2.Context(o2.config_from(w, batch=B // groups, precision=o2.BF16, chunk_tiles=chunk)) \
        if groups > 1 else ctx
    packed_h = ctx_h.prepare_weights(torch.from_numpy(blob).cuda()) if groups > 1 else packed

    def e2e_step(last=True):
        if groups > 1:   # back-to-back calls overlap across steps; the last one orders its copies
            ctx_h.forward_host(packed_h, x_pin, out_pin, stream=stream, sync_out=last)
        else:   # one sample (C4 / C5): no second set of device buffers, serial copies
            x_dev.copy_(x_pin, non_blocking=True)
            step()
            out_pin.copy_(out, non_blocking=True)

    e2e_step()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_steps = max(2, args.steps // 2)
    e0.record(stream)
    for i in range(e_steps):
        e2e_step(last=i + 1 == e_steps)
    e1.record(stream)
    barrier(world)
    e2e_ms = max_over_ranks(world, e0.elapsed_time(e1) / e_steps)

    # ---- per-kernel-class times (separate profiled pass, CUDA events per launch) ----
    prof = {}
    if not args.no_profile:
        ctx.set_profiling(True)
        for _ in range(max(2, min(args.steps, 5))):
            step()
        torch.cuda.synchronize()
        prof = ctx.kernel_times()
        ctx.set_profiling(False)

    px_per_step = world * B * w.scale * w.H * w.scale * w.W
    value = px_per_step / (ms * 1e-3)
    flops_step = world * B * info.flops_per_sample
    pk = peaks()
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (ERA5-shaped seeded fields, random-init weights)",
        "config": {"workload": w.name, "batch_per_gpu": B, "coarse": [w.H, w.W, w.V], "out": [w.scale * w.H,
                   w.scale * w.W, w.K], "tiles": [w.tiles_y, w.tiles_x], "halo": w.halo,
                   "vit": [w.embed, w.depth, w.heads], "parallelism": f"dp{world} (samples sharded, tiles local)",
                   "l2": "working set > L2 (126 MB) every step; no flush needed",
                   "chunk_tiles": info.chunk_tiles},
        "tokens_per_s": world * B * info.tokens_per_sample / (ms * 1e-3),
        "core_tokens_per_s": world * B * info.core_tokens_per_sample / (ms * 1e-3),
        "path_tflops": flops_step / (ms * 1e-3) / 1e12,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": {"value": px_per_step / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "api": "Context.forward_host" if groups > 1 else "Context.forward + copies",
                "groups": groups},
    }
    if prof:
        work = class_work(w, info, B)
        total_ms = sum(v[1] for v in prof.values())
        classes = {}
        for name, (n, t) in prof.items():
            steps_prof = max(2, min(args.steps, 5))
            per_step_ms = t / steps_prof
            launches_per_step = n / steps_prof
            entry = {"share": t / total_ms, "ms_per_step": per_step_ms, "launches_per_step": launches_per_step}
            if name in work:
                bound, amount = work[name]
                if bound == "tensor":
                    entry["tflops"] = amount / (per_step_ms * 1e-3) / 1e12
                else:
                    entry["gbs"] = amount / (per_step_ms * 1e-3) / 1e9
            classes[name] = entry
        res["kernels"] = classes
        dom = max((k for k in classes if k in work), key=lambda k: classes[k]["share"])
        bound, amount = work[dom]
        launches_dom = classes[dom]["launches_per_step"]
        per_launch_ms = classes[dom]["ms_per_step"] / launches_dom
        traffic, traffic_note = None, None
        tr = latest_traffic().get(dom)
        if tr and tr.get("workload") == w.name:
            traffic = tr["dram_bytes_per_launch"] * B / tr["batch"]
            traffic_note = (f"ncu --set full dram read+write of one {dom} launch at batch {tr['batch']} "
                            f"({tr['source']}), scaled linearly to batch {B}")
        # Peak choice: the timed region is far below the 4 s over which MEASURED_PEAKS'
        # sustained figure was taken (and runs at the clocks sampled above), so a kernel
        # in it is compared with the BURST peak; the sustained ratio is reported beside it.
        region_s = ms * 1e-3 * args.steps
        peak_kind = "burst" if region_s < 4.0 else "sustained"
        if bound == "tensor":
            achieved = amount / launches_dom / (per_launch_ms * 1e-3) / 1e12
            peak = pk["bf16"] if peak_kind == "burst" else pk["bf16_sus"]
            res["roofline"] = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peak,
                               "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                               "traffic_note": traffic_note,
                               "algorithmic_bytes_per_launch": attn_bytes(w, info, B) if dom == "tile_attention" else None,
                               "peak_src": f"{pk['src']} bf16_tflops ({peak_kind}: timed region {region_s:.2f} s "
                                           f"at {clocks.get('sm_mhz')} MHz median)",
                               "frac_of_burst": achieved / pk["bf16"], "frac_of_sustained": achieved / pk["bf16_sus"]}
        else:
            achieved = amount / launches_dom / (per_launch_ms * 1e-3) / 1e9
            res["roofline"] = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": pk["hbm"],
                               "unit": "GB/s", "frac": achieved / pk["hbm"], "traffic": traffic,
                               "traffic_note": traffic_note, "peak_src": pk["src"]}
        for k, v in classes.items():      # every class against its own roofline
            if "tflops" in v:
                v["frac_of_burst"] = v["tflops"] / pk["bf16"]
            if "gbs" in v:
                v["frac_of_hbm"] = v["gbs"] / pk["hbm"]
        att = classes.get("tile_attention")
        if att and "tflops" in att:
            res["attn_tflops"] = att["tflops"]
            res["attn_frac_bf16_peak"] = att["tflops"] / pk["bf16"]
            res["attn_frac_bf16_sustained"] = att["tflops"] / pk["bf16_sus"]
        res["hbm_kernels"] = {k: {"gbs": classes[k]["gbs"], "frac_of_hbm": classes[k]["gbs"] / pk["hbm"]}
                              for k in ("tile_gather", "stitch_residual", "layernorm") if k in classes
                              and "gbs" in classes[k]}
        if "embed_gemm" in classes:   # HBM-bound at Din = 80: patches in, z (+ LN1 xn) out
            eb = class_bytes_embed(w, info, B)
            g = eb / (classes["embed_gemm"]["ms_per_step"] * 1e-3) / 1e9
            res["hbm_kernels"]["embed_gemm"] = {"gbs": g, "frac_of_hbm": g / pk["hbm"]}
        # measured tensor-core classes other than attention (GEMMs, fused MLP / block tail)
        tck = [k for k in classes if k in work and work[k][0] == "tensor" and k != "tile_attention"]
        gemm_ms = sum(classes[k]["ms_per_step"] for k in tck)
        gemm_f = sum(work[k][1] for k in tck)
        res["gemm_tflops"] = gemm_f / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None
        tc_ms = gemm_ms + (att["ms_per_step"] if att else 0)
        tc_f = gemm_f + work["tile_attention"][1]
        res["attn_gemm_tflops"] = tc_f / (tc_ms * 1e-3) / 1e12 if tc_ms else None
        res["attn_gemm_frac_bf16_peak"] = res["attn_gemm_tflops"] / pk["bf16"] if tc_ms else None
        res["attn_gemm_frac_bf16_sustained"] = res["attn_gemm_tflops"] / pk["bf16_sus"] if tc_ms else None

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        xs = x_host[:1]
        done, px, dt, threads = oracle_units(w, blob, xs, seconds_budget=15.0)
        res["cpu_baseline"] = {"value": px / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
                               "sample": f"{done} (sample, tile) units of {w.name} sample 0 in {dt:.1f} s "
                                         f"(fp64 numpy oracle, as it stands)",
                               "cores_note": "threads of the BLAS pool the oracle's matmuls ran on", **host_cpu()}
    if rank == 0:
        print(json.dumps(res), flush=True)


def run_sp(args, w, world, rank, local):
    """TILES sequence parallelism (strong scaling): ONE batch, its tiles LPT-spread
    over the N ranks; the library moves the data through NVLink peer memory
    (sequence_parallel.PeerSP): halo push + barrier, forward chunks, stitch of each
    chunk straight into rank 0's output field (side stream, overlapping the next
    chunk), end barrier.  Every rank's input field holds only its owned core pixels
    (plus what peers push)."""
    import torch
    import torch.distributed as dist
    from paper_2505_04802_b200 import orbit2 as o2
    from paper_2505_04802_b200.sequence_parallel import PeerSP
    from workloads import make_input, make_weights
    B = w.batch
    _, info0 = o2.orbit2_tiles_plan(o2.config_from(w, batch=B, world_size=world, rank=rank))
    n_local = info0.n_local_tiles
    # Work split of a rank's share: G sample groups x all its tiles (kernels keep B/G x n_local
    # tile-samples per launch; the last group's stitch, the only one not overlapped with
    # compute, carries 1/G of the rank's output), or, for small batches, <= 4 tile chunks.
    # default: the most groups (<= 4) that keep >= 4 waves of 128-row blocks per launch
    rows_min = 4 * 148 * 128
    groups = args.sp_groups if args.sp_groups > 0 else next(
        g for g in (4, 2, 1) if B % g == 0 and (g == 1 or (B // g) * info0.local_tokens >= rows_min))
    chunk = args.chunk if args.chunk > 0 else (0 if groups > 1 else max(1, -(-n_local // 4)))
    cfg = o2.config_from(w, batch=B, precision=o2.BF16, world_size=world, rank=rank, chunk_tiles=chunk)
    ctx = o2.Context(cfg)
    info = ctx.info
    wctx = o2.Context(o2.config_from(w, batch=B // groups, precision=o2.BF16, world_size=world, rank=rank,
                                     chunk_tiles=chunk)) if groups > 1 else None
    blob = make_weights(w)
    x_host = make_input(w, batch=B)
    x_pin = torch.from_numpy(x_host).pin_memory()
    full = x_pin.to("cuda")
    x = torch.full_like(full, float("nan"))
    for t in ctx.tiles:                                   # owned core pixels only
        if t.owner_rank == rank:
            sl = (slice(None), slice(None), slice(t.core_y0 * w.patch, t.core_y1 * w.patch),
                  slice(t.core_x0 * w.patch, t.core_x1 * w.patch))
            x[sl] = full[sl]
    del full
    packed = ctx.prepare_weights(torch.from_numpy(blob).cuda())
    out = torch.empty((B, w.K, w.scale * w.H, w.scale * w.W), dtype=torch.float32, device="cuda") \
        if rank == 0 else None
    sp = PeerSP(ctx, x, out, dist, gather_root=0, work_ctx=wctx)
    stream = torch.cuda.current_stream()

    for _ in range(max(3, args.warmup)):
        sp.step(packed, stream)
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lctx = [ctx] + ([wctx] if wctx is not None else [])
    l0 = sum(c.launch_count() for c in lctx)
    with ClockSampler(local) as clk:
        barrier(world)
        ev0.record(stream)
        for _ in range(args.steps):
            sp.step(packed, stream)
        ev1.record(stream)
        barrier(world)
    ms = max_over_ranks(world, ev0.elapsed_time(ev1) / args.steps)
    launches = (sum(c.launch_count() for c in lctx) - l0) // args.steps
    clocks = clk.summary()
    ctx.comm_status()

    # ---- end to end: pinned host input -> every rank (H2D of the field), SP step, root ->
    # pinned host output (D2H).  Two independent SP instances (their own contexts, fields and
    # barrier flags) alternate, so step k+1's input copy and step k's output copy run on side
    # streams while the other instance computes.  The root enters an instance's next step
    # (whose first act is the halo barrier every rank waits on) only after the output copy of
    # that instance's previous step: no rank stitches into a field still being copied out ----
    out_pin = torch.empty(tuple(out.shape), dtype=torch.float32).pin_memory() if rank == 0 else None
    ctx2 = o2.Context(cfg)
    wctx2 = o2.Context(o2.config_from(w, batch=B // groups, precision=o2.BF16, world_size=world, rank=rank,
                                      chunk_tiles=chunk)) if groups > 1 else None
    x2 = x.clone()
    out2 = torch.empty_like(out) if rank == 0 else None
    packed2 = ctx2.prepare_weights(torch.from_numpy(blob).cuda())
    sp2 = PeerSP(ctx2, x2, out2, dist, gather_root=0, work_ctx=wctx2)
    inst = [(sp, x, out, packed, ctx), (sp2, x2, out2, packed2, ctx2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    comp_done, out_done = [None, None], [None, None]
    kstep = [0]

    def e2e_step(last=False):
        b = kstep[0] & 1
        kstep[0] += 1
        spb, xb, outb, pb, _ = inst[b]
        ev_in = torch.cuda.Event()
        with torch.cuda.stream(s_in):
            if comp_done[b] is not None:
                s_in.wait_event(comp_done[b])
            xb.copy_(x_pin, non_blocking=True)
            ev_in.record(s_in)
        stream.wait_event(ev_in)
        if rank == 0 and out_done[b] is not None:
            stream.wait_event(out_done[b])
        spb.step(pb, stream)
        cd = torch.cuda.Event()
        cd.record(stream)
        comp_done[b] = cd
        if rank == 0:
            with torch.cuda.stream(s_out):
                s_out.wait_event(cd)
                out_pin.copy_(outb, non_blocking=True)
                od = torch.cuda.Event()
                od.record(s_out)
            out_done[b] = od
        if last and rank == 0:
            for e in out_done:
                if e is not None:
                    stream.wait_event(e)

    for _ in range(2):
        e2e_step(last=True)
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_steps = max(2, args.steps // 2)
    e0.record(stream)
    for i in range(e_steps):
        e2e_step(last=i + 1 == e_steps)
    e1.record(stream)
    barrier(world)
    e2e_ms = max_over_ranks(world, e0.elapsed_time(e1) / e_steps)
    ctx.comm_status()
    ctx2.comm_status()

    # ---- per-kernel-class times of this rank (profiled pass, events per launch) ----
    prof = {}
    if not args.no_profile:
        for c in lctx:
            c.set_profiling(True)
        for _ in range(3):
            sp.step(packed, stream)
        torch.cuda.synchronize()
        for c in lctx:
            for k, (n, t) in c.kernel_times().items():
                n0, t0 = prof.get(k, (0.0, 0.0))
                prof[k] = (n0 + n / 3, t0 + t / 3)
            c.set_profiling(False)
    allprof = [None] * world
    dist.all_gather_object(allprof, prof)
    px = B * w.scale * w.H * w.scale * w.W
    if rank == 0:
        pk = peaks()
        res = {
            "metric": METRIC, "value": px / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (ERA5-shaped seeded fields, random-init weights)",
            "config": {"workload": w.name, "batch": B, "coarse": [w.H, w.W, w.V], "out": [w.scale * w.H,
                       w.scale * w.W, w.K], "tiles": [w.tiles_y, w.tiles_x], "halo": w.halo,
                       "vit": [w.embed, w.depth, w.heads],
                       "parallelism": f"tiles-sp{world} (LPT tile partition; halo push + output gather through "
                                      "NVLink peer memory, stitch fused with the gather)",
                       "chunk_tiles": (wctx or ctx).info.chunk_tiles, "sample_groups": groups, "gather_root": 0,
                       "l2": "working set > L2 (126 MB) every step; no flush needed"},
            "tokens_per_s": B * info.tokens_per_sample / (ms * 1e-3),
            "core_tokens_per_s": B * info.core_tokens_per_sample / (ms * 1e-3),
            "path_tflops": B * info.flops_per_sample / (ms * 1e-3) / 1e12,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "e2e": {"value": px / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": world * x_pin.numel() * 4, "d2h_bytes_per_step": out.numel() * 4,
                    "ms_per_step": e2e_ms,
                    "api": "PeerSP.step (two instances alternating, copies on side streams) with the input "
                           "field copied from pinned host on every rank and the gathered field copied to "
                           "pinned host on rank 0"},
            "per_rank_kernels": [{k: {"launches": round(n, 2), "ms": round(t, 4)} for k, (n, t) in (pr or {}).items()}
                                 for pr in allprof],
            "note": "strong scaling: one batch over N GPUs; CUDA-event time of K back-to-back steps, max over ranks",
        }
        print(json.dumps(res), flush=True)


# ---------------------------------------------------------------------------
# the training step
# ---------------------------------------------------------------------------
def class_work_train(w, info, B):
    """Algorithmic FLOPs per step of every kernel class of the training step (all
    queries of every block; backward = input and weight gradients, attention 2.5x)."""
    D, L, Din, Nh = w.embed, w.depth, w.din, w.head_out
    n, nc, n2 = info.tokens_per_sample, info.core_tokens_per_sample, info.sum_n2_per_sample
    f = {"embed_gemm": 2.0 * n * Din * D, "head_gemm": 2.0 * nc * D * Nh,
         "qkv_gemm": L * 6.0 * n * D * D, "oproj_gemm": L * 2.0 * n * D * D,
         "mlp_up_gemm": L * 8.0 * n * D * D, "mlp_down_gemm": L * 8.0 * n * D * D,
         "tile_attention": L * 4.0 * D * n2, "attn_bwd": L * 10.0 * D * n2,
         "wgrad_w2": L * 8.0 * n * D * D, "dx_mlp_down": L * 8.0 * n * D * D,
         "wgrad_w1": L * 8.0 * n * D * D, "dx_mlp_up": L * 8.0 * n * D * D,
         "wgrad_wo": L * 2.0 * n * D * D, "dx_oproj": L * 2.0 * n * D * D,
         "wgrad_wqkv": L * 6.0 * n * D * D, "dx_qkv": L * 6.0 * n * D * D,
         "wgrad_head": 2.0 * nc * D * Nh, "dx_head": 2.0 * nc * D * Nh, "wgrad_embed": 2.0 * n * Din * D}
    return {k: v * B for k, v in f.items()}


def run_train(args, w, world, rank, local):
    """Data-parallel training step: every rank its own batch of B samples over all tiles
    (forward keeping activations, stitch, Bayesian loss, backward), then ONE NCCL
    all-reduce (average) of the gradient per batch (reading R36)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2505_04802_b200 import orbit2 as o2
    from workloads import make_input, make_weights
    B = w.batch
    tiles_sp = args.train_tiles and world > 1
    free, _ = torch.cuda.mem_get_info()
    while True:   # the largest batch (<= the config's) whose training workspace fits 85% of HBM
        cfg = o2.config_from(w, batch=B, precision=o2.BF16, world_size=world if tiles_sp else 1,
                             rank=rank if tiles_sp else 0)
        ctx = o2.Context(cfg)
        ti = ctx.train_info()
        need = ti.workspace_bytes + 4 * cfg.batch * w.K * w.scale * w.H * w.scale * w.W * 4 + ctx.info.tile_out_bytes
        if need < 0.85 * torch.cuda.mem_get_info()[0] or B == 1:
            break
        del ctx
        torch.cuda.empty_cache()
        B //= 2
    if tiles_sp:
        from paper_2505_04802_b200.training import TilesTrainSP
        sp = TilesTrainSP(ctx, dist)
    else:
        ctx.train_bind()
    info = ctx.info
    blob = torch.from_numpy(make_weights(w)).cuda()
    packed = ctx.prepare_weights(blob)
    if tiles_sp:
        sp.prepare(blob)
    else:
        ctx.train_prepare(blob)
    seed = 0 if tiles_sp else rank          # tile-parallel: the same batch on every rank
    x_host = make_input(w, batch=B, seed=2000 + 97 * seed)
    rng = np.random.default_rng(3000 + seed)
    y_host = rng.standard_normal((B, w.K, w.scale * w.H, w.scale * w.W)).astype(np.float32)
    x_pin, y_pin = torch.from_numpy(x_host).pin_memory(), torch.from_numpy(y_host).pin_memory()
    x_dev, y_dev = x_pin.cuda(), y_pin.cuda()
    bufs = ctx.train_buffers()
    grad = bufs[4]
    loss_pin = torch.empty(B, dtype=torch.float64).pin_memory()
    stream = torch.cuda.current_stream()

    # the weight update (R43: AdamW) and the re-packing of the updated weights are part of the step
    mom = torch.zeros_like(blob)
    vel = torch.zeros_like(blob)
    t_step = [0]

    def step():
        if tiles_sp:    # tiles over the ranks; field and gradient summed (training.TilesTrainSP)
            loss, g, _ = sp.step(packed, x_dev, y_dev, args.lam, args.delta, True, stream)
        else:
            loss, g, _ = ctx.train_step(packed, x_dev, y_dev, args.lam, args.delta, True, bufs, stream)
            if world > 1:
                dist.all_reduce(g, op=dist.ReduceOp.AVG)   # once per batch
        t_step[0] += 1
        o2.adamw_step(blob, g, mom, vel, t_step[0], 1e-4, 0.9, 0.95, 1e-8, 0.01, stream)
        ctx.prepare_weights(blob, stream, out=packed)
        if tiles_sp:
            sp.prepare(blob, stream)
        else:
            ctx.train_prepare(blob, stream)
        return loss

    for _ in range(max(3, args.warmup)):
        step()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        barrier(world)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier(world)
    ms = max_over_ranks(world, ev0.elapsed_time(ev1) / args.steps)
    launches = (ctx.launch_count() - l0) // args.steps
    clocks = clk.summary()

    def e2e_step():   # pinned host input and truth in, per-sample loss out
        x_dev.copy_(x_pin, non_blocking=True)
        y_dev.copy_(y_pin, non_blocking=True)
        loss = step()
        loss_pin.copy_(loss, non_blocking=True)

    e2e_step()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_steps = max(2, args.steps // 2)
    e0.record(stream)
    for _ in range(e_steps):
        e2e_step()
    e1.record(stream)
    barrier(world)
    e2e_ms = max_over_ranks(world, e0.elapsed_time(e1) / e_steps)

    prof = {}
    if not args.no_profile:
        ctx.set_profiling(True)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        prof = {k: (n / 3, t / 3) for k, (n, t) in ctx.kernel_times().items()}
        ctx.set_profiling(False)
    px = (1 if tiles_sp else world) * B * w.scale * w.H * w.scale * w.W
    # tile-parallel: the ranks' tile shares of ONE batch (train_plan counts rank-local tiles)
    flops = B * _sum_over_ranks(world, ti.flops_per_sample) if tiles_sp else world * B * ti.flops_per_sample
    pk = peaks()
    res = {
        "metric": "training high-res px/s (forward + Bayesian loss + backward + gradient all-reduce + AdamW update)",
        "value": px / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if tiles_sp else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (ERA5-shaped seeded fields and truth, random-init weights)",
        "config": {"workload": w.name, "batch_per_gpu": B, "mode": "train", "lambda": args.lam, "delta": args.delta,
                   "parallelism": (f"tiles-sp{world} (one batch, LPT tiles per rank; NCCL all-reduce of the field "
                                   "and of the gradient)") if tiles_sp else f"dp{world} (one gradient all-reduce per batch)",
                   "l2": "working set > L2 (126 MB) every step; no flush needed"},
        "train_tflops": flops / (ms * 1e-3) / 1e12,
        "train_frac_bf16_peak": flops / (ms * 1e-3) / 1e12 / pk["bf16"],
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": {"value": px / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": (x_pin.numel() + y_pin.numel()) * 4, "d2h_bytes_per_step": B * 8,
                "api": "Context.train_step with input and truth copied from pinned host, per-sample loss to host"},
    }
    if prof:
        work = class_work_train(w, info, B)
        total = sum(t for _, t in prof.values())
        classes = {}
        for k, (n, t) in prof.items():
            e = {"share": t / total, "ms_per_step": t, "launches_per_step": n}
            if k in work:
                e["tflops"] = work[k] / (t * 1e-3) / 1e12
                e["frac_of_burst"] = e["tflops"] / pk["bf16"]
            classes[k] = e
        res["kernels"] = classes
        dom = max((k for k in classes if k in work), key=lambda k: classes[k]["share"])
        ach = classes[dom]["tflops"]
        res["roofline"] = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": pk["bf16"], "unit": "TFLOP/s",
                           "frac": ach / pk["bf16"], "traffic": None, "peak_src": f"{pk['src']} bf16_tflops (burst)"}
    if rank == 0:
        print(json.dumps(res), flush=True)


# ---------------------------------------------------------------------------
# adaptive spatial compression
# ---------------------------------------------------------------------------
def run_compress(args, w, world, rank, local):
    """Partition (Canny on variable 0 + quad-tree, min_side = p, max_side = 16 p), tokenize
    the V input variables of every leaf into D-wide tokens, decompress back to V fields:
    the batch's coarse fields edge-padded to a multiple of max_side."""
    import numpy as np
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    from workloads import make_input
    B, V, D, mn = w.batch, w.V, w.embed, w.patch
    mx = 16 * mn
    x = make_input(w, batch=B)
    H, W = -(-w.H // mx) * mx, -(-w.W // mx) * mx
    x = np.pad(x, ((0, 0), (0, 0), (0, H - w.H), (0, W - w.W)), mode="edge").astype(np.float32)
    feat = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    img = feat[:, 0].contiguous()
    # sigma 2 / threshold 0.13: ~2-5x fewer tokens on these synthetic fields (the paper's runs: 4-32x)
    thr, sigma = 0.13, 2.0
    comp = o2.Compressor(batch=B, H=H, W=W, C=V, min_side=mn, max_side=mx, embed=D, threshold=thr, sigma=sigma)
    rng = np.random.default_rng(0)
    levels = int(np.log2(mx // mn)) + 1
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    Wt, bt, E = cu(0.05 * rng.standard_normal((D, V * mn * mn))), cu(rng.standard_normal(D)), \
        cu(rng.standard_normal((levels, D)))
    Wd, bd = cu(0.05 * rng.standard_normal((V * mn * mn, D))), cu(rng.standard_normal(V * mn * mn))
    Ws, bs = cu(0.05 * rng.standard_normal((V, V, 3, 3))), cu(rng.standard_normal(V))
    stream = torch.cuda.current_stream()

    def step():
        patches, _, n, _ = comp.partition(img)
        tok = comp.tokenize(feat, patches, n, Wt, bt, E)
        comp.detokenize(tok, patches, n, Wd, bd, Ws, bs)
        return n

    for _ in range(max(3, args.warmup)):
        n = step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            n = step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    uniform = B * (H // mn) * (W // mn)
    res = {"metric": "adaptive compression: coarse px/s through partition + tokenize + decompress",
           "value": B * H * W / (ms * 1e-3), "unit": "coarse px/s", "n_gpus": 1, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic ERA5-shaped fields (edge padded)",
           "config": {"workload": w.name, "batch": B, "field": [H, W], "channels": V, "embed": D,
                      "min_side": mn, "max_side": mx, "threshold": thr, "sigma": sigma, "mode": "compress"},
           "tokens": n, "uniform_tokens": uniform, "compression_ratio": uniform / max(n, 1),
           "clocks": clk.summary(), "host_s_per_step": (time.perf_counter() - t0) / args.steps}
    # the Reslim forward on compressed tokens vs the same forward uncompressed: one tile (R41,
    # the paper's compression rows run untiled, Tab. P:376-378) and the C2 tiling (R42, every
    # tile compressed on its own), C2 model, max_side 8 patches
    from workloads import make_weights
    Bf = min(B, 16)
    for key, wf in (("forward_on_compressed_tokens", w.replace(batch=Bf, tiles_y=1, tiles_x=1, halo=0)),
                    ("forward_on_compressed_tokens_tiles", w.replace(batch=Bf))):
        res[key] = _compressed_vs_uncompressed(o2, wf, Bf, D, thr, sigma, stream)
    print(json.dumps(res), flush=True)


def _compressed_vs_uncompressed(o2, wf, Bf, D, thr, sigma, stream):
    import torch
    from workloads import make_input, make_weights
    ctx = o2.Context(o2.config_from(wf, precision=o2.BF16))
    packed = ctx.prepare_weights(torch.from_numpy(make_weights(wf)).cuda())
    xf = torch.from_numpy(make_input(wf, batch=Bf)).cuda()
    Ef = torch.zeros((4, D), dtype=torch.float32, device="cuda")
    outf = torch.empty((Bf, wf.K, wf.scale * wf.H, wf.scale * wf.W), dtype=torch.float32, device="cuda")
    fwd = {}
    for name, fn in (("uncompressed", lambda: ctx.forward(packed, xf, out=outf)),
                     ("compressed", lambda: ctx.compressed_forward(packed, xf, Ef, max_side=8, threshold=thr,
                                                                   sigma=sigma, out=outf))):
        for _ in range(2):
            r = fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            r = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        fwd[name] = {"ms_per_step": e0.elapsed_time(e1) / 3}
        if name == "compressed":
            fwd[name]["tokens"] = r[2]
    fwd["uncompressed"]["tokens"] = Bf * ctx.info.local_tokens
    fwd["speedup"] = fwd["uncompressed"]["ms_per_step"] / fwd["compressed"]["ms_per_step"]
    fwd["token_reduction"] = fwd["uncompressed"]["tokens"] / max(fwd["compressed"]["tokens"], 1)
    fwd["config"] = {"batch": Bf, "tiles": [wf.tiles_y, wf.tiles_x], "halo": wf.halo, "max_side_patches": 8,
                     "threshold": thr, "sigma": sigma,
                     "note": "event time incl. the host syncs of the partition (hysteresis passes, token count)"}
    return fwd


# ---------------------------------------------------------------------------
# tile-count sweep (Tab. P:379-381) + CUDA-graph replay
# ---------------------------------------------------------------------------
def run_sweep(args, w, world, rank, local):
    import torch
    from paper_2505_04802_b200 import orbit2 as o2
    from workloads import make_input, make_weights
    B = args.batch or 16
    stream = torch.cuda.current_stream()
    rows = []
    for ty, tx in ((1, 1), (2, 2), (4, 4), (6, 6)):
        wt = w.replace(batch=B, tiles_y=ty, tiles_x=tx, halo=0 if ty * tx == 1 else w.halo)
        ctx = o2.Context(o2.config_from(wt, precision=o2.BF16))
        packed = ctx.prepare_weights(torch.from_numpy(make_weights(wt)).cuda())
        x = torch.from_numpy(make_input(wt, batch=B)).cuda()
        out = torch.empty((B, wt.K, wt.scale * wt.H, wt.scale * wt.W), dtype=torch.float32, device="cuda")
        tile_out = ctx.tile_out_buffer()
        for _ in range(max(3, args.warmup)):
            ctx.forward(packed, x, out=out, tile_out=tile_out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ctx.forward(packed, x, out=out, tile_out=tile_out)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        g = ctx.capture_forward(packed, x, out, tile_out=tile_out)
        g.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_g = e0.elapsed_time(e1) / args.steps
        info = ctx.info
        rows.append({"tiles": ty * tx, "halo": wt.halo, "ms_per_step": ms, "ms_per_step_graph": ms_g,
                     "tokens_per_sample": info.tokens_per_sample,
                     "attn_flops_per_sample": 4.0 * wt.embed * wt.depth * info.sum_n2_per_sample,
                     "path_tflops": B * info.flops_per_sample / (ms * 1e-3) / 1e12})
        del ctx, packed, x, out, tile_out, g
        torch.cuda.empty_cache()
    for r in rows:
        r["speedup_vs_T1"] = rows[0]["ms_per_step"] / r["ms_per_step"]
    px = B * w.scale * w.H * w.scale * w.W
    res = {"metric": "tile-count sweep: high-res px/s of the forward at T = 1 / 4 / 16 / 36 tiles",
           "value": px / (min(r["ms_per_step"] for r in rows) * 1e-3), "unit": UNIT, "n_gpus": 1,
           "steps": args.steps, "warmup": max(3, args.warmup), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "bf16", "data": "synthetic (ERA5-shaped seeded fields, random-init weights)",
           "config": {"workload": w.name, "batch": B, "mode": "sweep",
                      "note": "T = 1 without halo; the others with the config's halo (P:379-381 shape)"},
           "sweep": rows}
    print(json.dumps(res), flush=True)


def relaunch_if_needed(args):
    """`python bench.py --gpus N` without torchrun: re-exec under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    from workloads import get_config
    w = get_config(args.config)
    if args.batch:
        w = w.replace(batch=args.batch)
    for kv in args.set:
        k, v = kv.split("=")
        w = w.replace(**{k: int(v)})
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, w, int(os.environ.get("WORLD_SIZE", "1")), rank)
        return
    relaunch_if_needed(args)
    world, rank, local = dist_init(args.gpus)
    try:
        if args.mode == "train":
            run_train(args, w, world, rank, local)
        elif args.mode == "compress":
            run_compress(args, w, world, rank, local)
        elif args.mode == "sweep":
            run_sweep(args, w, world, rank, local)
        elif world > 1 and args.mode == "sp":
            run_sp(args, w, world, rank, local)
        else:
            run_ours(args, w, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
