"""Throughput benchmark of the B200 hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2|3|4|5]
                    [--smoother fir|iir] [--impl ours|reference]

Workloads are BASELINE.json's configs on seeded synthetic inputs (the
reference measures no public dataset):

* config 2 (default, the metric's headline): 1024x1024 f32 image (seed 1,
  5x5 box blur), 8 orientations x 4 frequencies, FIR r=3 -> 32 complex64
  outputs.  One step = one full bank.  With N GPUs every rank runs its own
  bank on its own image (seed 1 + rank): weak scaling, no collective.
* config 3: batched bank, 64 images 1024^2 sharded by image (strong).
* config 4: 2048^2 localized SDFT, 16x16 window, sigma 4, 256 bins (strong,
  sharded by conjugate u-pairs).
* config 5: 8192^2 bank, 16 orientations x 5 frequencies (strong, sharded by
  (frequency, theta/pi-theta) units, LPT).

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the
launching stream; an L2 flush (256 MiB memset, outside the events) runs
between timed steps; the reported time is the sum of the K step times, max
over ranks.  A second pass with libfgb200's live per-kernel profiling gives
the roofline of the dominant kernel.  `e2e` repeats the metric through the
host-buffer C-ABI entry (pinned host input -> H2D -> compute -> D2H of every
output) timed on the host clock.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    2: dict(kind="bank", size=1024, freqs=[math.pi / 2 ** j for j in (1, 2, 3, 4)], sigmas=[2.0, 4.0, 8.0, 16.0], n=8,
            images=1, seed=1, blur=True, workload="cfg2: 1024x1024 f32 (seed 1, 5x5 box blur), N=8 x 4 freqs, FIR r=3"),
    3: dict(kind="bank", size=1024, freqs=[math.pi / 2 ** j for j in range(1, 6)], sigmas=[2.0 ** j for j in range(1, 6)],
            n=8, images=64, seed=100, blur=False, workload="cfg3: 64 x 1024x1024 f32 (seeds 100..163), N=8 x 5 freqs, FIR r=3"),
    4: dict(kind="sdft", size=2048, m=16, sigma=4.0, seed=2, workload="cfg4: 2048x2048 f32 (seed 2), 16x16 window, sigma 4, FIR r=3, 256 bins"),
    5: dict(kind="bank", size=8192, freqs=[math.pi / 2 ** j for j in range(1, 6)], sigmas=[2.0 ** j for j in range(1, 6)],
            n=16, images=1, seed=3, blur=False, gratings=True,
            workload="cfg5: 8192x8192 f32 (seed 3 + 16 gratings), N=16 x 5 freqs, FIR r=3"),
}


def make_image(cfg, seed_offset=0, size=None):
    n = size or cfg["size"]
    rng = np.random.default_rng(cfg["seed"] + seed_offset)
    img = rng.uniform(0.0, 1.0, size=(n, n))
    if cfg.get("gratings"):
        y, x = np.mgrid[0:n, 0:n].astype(np.float64)
        for _ in range(16):
            th = rng.uniform(0, math.pi)
            per = rng.uniform(4, 64)
            amp = rng.uniform(0, 0.5)
            ph = rng.uniform(0, 2 * math.pi)
            img += amp * np.sin(2 * math.pi * (x * math.cos(th) + y * math.sin(th)) / per + ph)
    img = img.astype(np.float32)
    if cfg.get("blur"):
        import scipy.ndimage as ndi

        img = ndi.uniform_filter(img.astype(np.float64), size=5, mode="nearest").astype(np.float32)
    return img


def units_per_image(cfg):
    s = cfg["size"] * cfg["size"]
    if cfg["kind"] == "bank":
        return s * len(cfg["freqs"]) * cfg["n"]
    return s * cfg["m"] * cfg["m"]


def metric_name(cfg):
    return "gabor_bank_px_filters_per_s" if cfg["kind"] == "bank" else "sdft_px_bins_per_s"


def unit_name(cfg):
    return "px*filters/s" if cfg["kind"] == "bank" else "px*bins/s"


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clocks + throttle reasons DURING the timed region: an NVML polling
    thread (1 ms period, so even sub-second regions get samples); falls back
    to `nvidia-smi -lms 50` when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, dev):
        self.dev = dev
        self.samples = []
        self.mx = None

    def __enter__(self):
        import threading

        self.stop = threading.Event()
        self.th = None
        try:
            import pynvml
        except ImportError:  # no NVML bindings: clocks are reported as unavailable
            return self
        try:
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def run():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(sm), int(rs)))
                    except pynvml.NVMLError:  # a missed sample is not fatal
                        pass
                    self.stop.wait(0.001)

            self.th = threading.Thread(target=run, daemon=True)
            self.th.start()
        except pynvml.NVMLError:
            self.th = None
        return self

    def __exit__(self, *a):
        if self.th is not None:
            self.stop.set()
            self.th.join(2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": [], "samples": 0, "source": "nvml"}
        reasons = sorted(n for n, bit in self.REASONS.items() if any(r & bit for _, r in self.samples))
        return {"sm_mhz": float(np.median([s for s, _ in self.samples])), "sm_max_mhz": self.mx, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------------------
# CPU baseline (the oracle port; it is the checker, timed here as the baseline)
# ---------------------------------------------------------------------------
def _oracle_bank_unit(args):
    from oracle import fastgabor_oracle as O

    f, omega, k, n, sigma = args
    jr, ji = O.horizontal_stage(f, omega, k * math.pi / n, sigma, ("fir", 3.0))
    O.vertical_stage(jr, ji, omega, k * math.pi / n, sigma, ("fir", 3.0))
    nh = n // 2
    outs = 1
    if nh < n - k < n:
        O.vertical_stage(jr, ji, omega, k * math.pi / n, sigma, ("fir", 3.0), conjugate=True)
        outs = 2
    return outs


def _oracle_sdft_rows(args):
    from oracle import fastgabor_oracle as O

    f, m, sigma = args
    O.sdft_full(f, m, m, ("fir", 3.0), sigma)
    return m * m


def cpu_sample(cfg, rows, cores, pool=None):
    """Run the oracle on a `rows`-row strip; returns (units, seconds)."""
    img = make_image(cfg if cfg["kind"] == "sdft" or cfg["size"] <= 2048 else dict(cfg, size=1024), 0,
                     size=min(cfg["size"], 2048))[:rows].astype(np.float64)
    t0 = time.perf_counter()
    if cfg["kind"] == "bank":
        nh = cfg["n"] // 2
        # (frequency, direct k) units -- the reference's own parallel grain (compute_bank
        # threads=k) -- heaviest (largest sigma) first so the pool's tail is short
        jobs = [(img, w, k, cfg["n"], s) for w, s in zip(cfg["freqs"], cfg["sigmas"]) for k in range(nh + 1)]
        jobs.sort(key=lambda j: -j[4])
        outs = sum(pool.map(_oracle_bank_unit, jobs, chunksize=1)) if pool else sum(map(_oracle_bank_unit, jobs))
        units = img.shape[0] * img.shape[1] * outs
    else:
        if pool:
            strips = np.array_split(img, cores, axis=0)
            pool.map(_oracle_sdft_rows, [(s, cfg["m"], cfg["sigma"]) for s in strips])
        else:
            _oracle_sdft_rows((img, cfg["m"], cfg["sigma"]))
        units = img.shape[0] * img.shape[1] * cfg["m"] ** 2
    return units, time.perf_counter() - t0


def run_reference(args, cfg, rank, world):
    """The reference's CPU algorithm (the oracle port: NumPy fp64 restatement of
    fastgabor's hot path) on the host cores, a bounded strip per step."""
    if rank != 0:
        return
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    rows = 64 if cfg["kind"] == "bank" else 32
    with mp.get_context("fork").Pool(cores) as pool:
        for _ in range(args.warmup):
            cpu_sample(cfg, 16, cores, pool)
        tot_u, tot_s = 0, 0.0
        for _ in range(args.steps):
            u, s = cpu_sample(cfg, rows, cores, pool)
            tot_u += u
            tot_s += s
    v = tot_u / tot_s
    sample = (f"oracle port (NumPy fp64 restatement of the reference hot path, FIR r=3), {rows}-row strip of the "
              f"{cfg['workload'].split(':')[0]} image per step, pool of {cores} processes")
    line = {
        "impl": "reference", "metric": metric_name(cfg), "value": v, "unit": unit_name(cfg), "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"]},
        "cpu_baseline": {"value": v, "unit": unit_name(cfg), "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": unit_name(cfg), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1704_05231_b200 as fg
    from paper_1704_05231_b200 import _native as N
    from paper_1704_05231_b200.device import BankPlan, SdftPlan

    dev = torch.device("cuda", local_rank % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    kind = fg.ExactFIR(3.0) if args.smoother == "fir" else fg.RecursiveIIR()

    # ---- shard the workload (config 2: every rank its own image -> weak) ----
    scaling = "weak"
    bcast_ms = None

    def timed_broadcast(t):
        """The one input broadcast of the sharded configs, timed on the device
        (max over ranks); it happens once per job, outside the timed steps."""
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        dist.broadcast(t, 0)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return ms.item()

    if cfg["kind"] == "bank":
        spec = fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"]))
        if args.config == 3:
            from paper_1704_05231_b200.parallel import shard_images

            mine = shard_images(cfg["images"], world)[rank]
            scaling = "strong"
            imgs = np.stack([make_image(cfg, i) for i in mine]) if mine else np.zeros((0, 1, 1), np.float32)
            units = None
        elif args.config == 5:
            from paper_1704_05231_b200.parallel import bank_unit_costs, lpt_assign

            scaling = "strong"
            costs = bank_unit_costs(cfg["freqs"], cfg["sigmas"], cfg["n"], 3.0)
            units = lpt_assign(costs, world)[rank]
            imgs = make_image(cfg, 0)[None]
            if world > 1:
                t = torch.from_numpy(imgs).to(dev)
                bcast_ms = timed_broadcast(t)  # one NCCL broadcast of the input over NVLink
        else:
            imgs = make_image(cfg, rank)[None]
            units = None
        timg = torch.from_numpy(imgs).to(dev)
        plan = BankPlan(tuple(timg.shape), spec, kind, "f32", True, units)
        units_step = timg.shape[0] * timg.shape[1] * timg.shape[2] * plan.entries
    else:
        from paper_1704_05231_b200.parallel import sdft_heads

        spec = fg.SdftSpec(cfg["m"], cfg["m"], kind, cfg["sigma"])
        heads = sdft_heads(cfg["m"], world)[rank] if world > 1 else None
        scaling = "strong" if world > 1 else "weak"
        imgs = make_image(cfg, 0)[None]
        timg = torch.from_numpy(imgs).to(dev)
        if world > 1:
            bcast_ms = timed_broadcast(timg)
        plan = SdftPlan(tuple(timg.shape), spec, "f32", heads)
        units_step = timg.shape[1] * timg.shape[2] * plan.bins
    out = plan.new_output(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        plan(timg, out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = N.lib.fgb_launch_count()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            flush.zero_()
            starts[k].record()
            step()
            ends[k].record()
        torch.cuda.synchronize()
    launches = N.lib.fgb_launch_count() - l0
    if world > 1:
        dist.barrier()
    per_step = sorted(s.elapsed_time(e) for s, e in zip(starts, ends))
    total_ms = sum(per_step)
    step_stats = {"min": per_step[0], "p50": per_step[len(per_step) // 2],
                  "p90": per_step[min(len(per_step) - 1, (9 * len(per_step)) // 10)], "max": per_step[-1]}
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        u = torch.tensor([float(units_step)], dtype=torch.float64, device=dev)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
        units_all = u.item()
    else:
        units_all = float(units_step)
    max_ms = t.item()
    value = units_all * args.steps / (max_ms / 1e3)

    # ---- live per-kernel profile pass (CUDA events on the launching stream; the
    #      library serialises its stream lanes while profiling so each kernel is timed alone) ----
    N.lib.fgb_profile_enable(1)
    N.profile_read()
    nprof = min(20, args.steps)
    for _ in range(nprof):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    prof = N.profile_read()
    N.lib.fgb_profile_enable(0)
    fp32 = N.lib.fgb_probe_fp32_tflops()
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except (OSError, ValueError):  # absent / unreadable: fall back to the recipe's figure
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    kernels = {}
    for e in prof:
        ms = e["ms"] / e["launches"]
        kernels[e["name"]] = {
            "launches_per_step": e["launches"] / nprof, "ms_per_launch": ms,
            "share": e["ms"] / sum(x["ms"] for x in prof),
            "tflops": e["flops"] / (e["ms"] * 1e-3) / 1e12 if e["ms"] > 0 else None,
            "gbs": e["bytes"] / (e["ms"] * 1e-3) / 1e9 if e["ms"] > 0 else None,
        }
    top = max(prof, key=lambda e: e["ms"]) if prof else None
    traffic = None
    try:  # ncu-measured DRAM bytes per launch of the dominant kernel (profiles/, committed)
        with open(os.path.join(ROOT, "profiles", "r01", "traffic.json")) as fh:
            tr = json.load(fh)
        if top is not None:
            traffic = tr.get(f"cfg{args.config}/{top['name']}")
    except (OSError, ValueError):
        traffic = None
    roof = None
    if top is not None:
        if cfg["kind"] == "sdft":
            ach = top["bytes"] / (top["ms"] * 1e-3) / 1e9
            roof = {"bound": "hbm", "kernel": top["name"], "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": traffic, "algorithmic_bytes_per_launch": top["bytes"] / top["launches"],
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        else:
            ach = top["flops"] / (top["ms"] * 1e-3) / 1e12
            roof = {"bound": "fp32", "kernel": top["name"], "achieved": ach, "peak": fp32, "unit": "TFLOP/s",
                    "frac": ach / fp32 if fp32 > 0 else None, "traffic": traffic,
                    "algorithmic_flops_per_launch": top["flops"] / top["launches"],
                    "peak_source": "live FFMA probe (fgb_probe_fp32_tflops); flops = reference OpCounters M+A"}
            if top["name"] == "iir":
                roof["note"] = ("RecursiveIIR stage (iir32_sum + iir32_fin): the reference counts ~12 flops per "
                                "output and plane, the exact segment-parallel fp32 recursion issues ~36 FMA per "
                                "sample and plane in two passes; its ncu FMA-pipe utilisation (32-44%) is in "
                                "profiles/r01/ncu_full_summary.txt")
    # whole-step roofline: algorithmic work of one step (sum over every launch, from the
    # profile pass) / measured step time of the timed region
    step_roof = None
    if prof:
        per_step = {k: sum(e[k] for e in prof) / nprof for k in ("flops", "bytes")}
        step_s = max_ms / args.steps / 1e3
        if cfg["kind"] == "sdft":
            ach = per_step["bytes"] / step_s / 1e9
            step_roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
        else:
            ach = per_step["flops"] / step_s / 1e12
            step_roof = {"bound": "fp32", "achieved": ach, "peak": fp32, "unit": "TFLOP/s",
                         "frac": ach / fp32 if fp32 > 0 else None,
                         "note": "reference OpCounters flops of the whole bank / step time (all launches, lanes overlapped)"}
    # ---- e2e: host buffers through the C ABI (H2D + compute + D2H each step) ----
    e2e = None
    if True:  # every rank times its own host-buffer calls; the max over ranks is reported
        hin = torch.from_numpy(imgs).pin_memory()
        hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        desc = plan.desc
        desc.img.pitch = imgs.shape[2]
        desc.img.batch_stride = imgs.shape[1] * imgs.shape[2]
        call = N.lib.fgb_bank_host if cfg["kind"] == "bank" else N.lib.fgb_sdft_host
        ne = max(3, min(args.steps, 20))
        N.check(call(C.byref(desc), C.c_void_p(hin.data_ptr()), C.c_void_p(hout.data_ptr())))
        t0 = time.perf_counter()
        for _ in range(ne):
            N.check(call(C.byref(desc), C.c_void_p(hin.data_ptr()), C.c_void_p(hout.data_ptr())))
        e2e_s = (time.perf_counter() - t0) / ne
        # the PCIe link itself: the same H2D + D2H bytes as plain pinned copies
        # (no compute), so e2e can be read as a fraction of what the link moves
        dev_in = torch.empty(hin.shape, dtype=hin.dtype, device=dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(ne):
            dev_in.copy_(hin, non_blocking=True)
            hout.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
        link_s = (time.perf_counter() - t1) / ne
        del dev_in
        nbytes = int(hin.numel() * hin.element_size()) + int(hout.numel() * hout.element_size())
        e2e = {"value": units_step * world / e2e_s if world == 1 else None, "unit": unit_name(cfg),
               "h2d_bytes_per_step": int(hin.numel() * hin.element_size()),
               "d2h_bytes_per_step": int(hout.numel() * hout.element_size()), "ms_per_step": e2e_s * 1e3,
               "link_copy_ms": link_s * 1e3, "link_gbs": nbytes / link_s / 1e9,
               "frac_of_link": link_s / e2e_s,
               "note": "host buffers through fgb_*_host (H2D, compute, D2H per step); link_copy_ms = the same "
                       "bytes as bare pinned copies, so frac_of_link ~ 1 means the step is PCIe-bound"}
        if world > 1:
            et = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
            e2e["value"] = units_all / et.item()
    # ---- CPU baseline (rank 0, N=1): oracle port on a bounded strip ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rows = 256 if cfg["kind"] == "bank" else 24
        u, s = cpu_sample(cfg, rows, 1)
        cpu = {"value": u / s, "unit": unit_name(cfg), "cores": 1, "kind": "port",
               "sample": f"oracle port (numpy fp64), {rows}-row strip of the config image, all filters/bins, {s:.1f} s"}
    if rank == 0:
        line = {
            "metric": metric_name(cfg), "value": value, "unit": unit_name(cfg), "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE.json shapes)",
            "config": {"workload": cfg["workload"], "smoother": args.smoother, "l2": "256 MiB flush between timed steps",
                       "input_broadcast_ms": bcast_ms,
                       "parallelism": f"{'image' if args.config in (2, 3) else 'unit'}-sharded x{world}"},
            "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(), "kernels": kernels, "fp32_peak_tflops_measured": fp32,
            "step_ms_rank0": step_stats,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5])
    ap.add_argument("--smoother", default="fir", choices=["fir", "iir"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        dev = torch.device("cuda", local_rank % max(1, torch.cuda.device_count()))
        torch.cuda.set_device(dev)
        backend = os.environ.get("FGB_DIST_BACKEND", "nccl")  # gloo: host-logic test with ranks sharing a GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
