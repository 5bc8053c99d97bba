"""Throughput benchmark of the B200 hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2|3|4|5]
                    [--smoother fir|iir] [--impl ours|reference]

Workloads are BASELINE.json's configs on seeded synthetic inputs (the
reference measures no public dataset; shapes, seeds and value distributions
follow BASELINE.json / SURVEY.md section 8(d)):

* config 5 (default: the largest single-GPU BASELINE config): one 8192x8192
  f32 image (seed 3 + 16 gratings), 16 orientations x 5 frequencies, FIR r=3
  -> 80 complex64 outputs (43 GB).  One step = the whole bank.  With N GPUs
  the image is broadcast once and the (frequency, theta/pi-theta) units are
  LPT-sharded: strong scaling, no collective in the timed steps.
* config 2: 1024x1024 f32 (seed 1, 5x5 box blur), 8 orientations x 4
  frequencies.  N GPUs: every rank runs its own bank (weak scaling).
* config 3: batched bank, 64 images 1024^2, sharded by image (strong).
* config 4: 2048^2 localized SDFT, 16x16 window, sigma 4, 256 bins (strong,
  sharded by conjugate u-pairs).

`--gpus N` without torchrun's environment re-launches this script under
`torch.distributed.run` with N ranks (one per GPU, NCCL; FGB_DIST_BACKEND=gloo
for host-logic runs with ranks sharing one GPU).

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the
launching stream; an L2 flush (256 MiB memset, outside the events) runs
between timed steps; the reported time is the sum of the K step times, max
over ranks.  A second pass with libfgb200's live per-kernel profiling gives
the roofline of the dominant kernel.  `e2e` repeats the metric through the
host-buffer C-ABI entry (pinned host input -> H2D -> compute -> D2H of every
output) timed on the host clock, max over ranks.

`--impl reference` times the reference's own CPU implementation (the
unmodified `fastgabor` installed in baseline/_ref by tools/install_reference.py;
the oracle port only if that install is absent) on every host core, on the
same config: per step a bounded sample of the workload (see RefArm).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

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
DEFAULT_CONFIG = 5


def make_image(cfg, seed_offset=0, size=None):
    """Seeded synthetic input of a BASELINE config (float32).

    Gratings (config 5): a*sin(2 pi (x cos t + y sin t)/p + phi), evaluated as
    sin(A+B) = sin A cos B + cos A sin B of separable row / column factors."""
    n = size or cfg["size"]
    rng = np.random.default_rng(cfg["seed"] + seed_offset)
    img = rng.uniform(0.0, 1.0, size=(n, n))
    if cfg.get("gratings"):
        ax = np.arange(n, dtype=np.float64)
        for _ in range(16):
            th = rng.uniform(0, math.pi)
            per = rng.uniform(4, 64)
            amp = rng.uniform(0, 0.5)
            ph = rng.uniform(0, 2 * math.pi)
            a = 2 * math.pi * ax * math.cos(th) / per + ph  # along x
            b = 2 * math.pi * ax * math.sin(th) / per       # along y
            img += amp * (np.sin(a)[None, :] * np.cos(b)[:, None] + np.cos(a)[None, :] * np.sin(b)[:, None])
    img = img.astype(np.float32)
    if cfg.get("blur"):
        import scipy.ndimage as ndi

        img = ndi.uniform_filter(img.astype(np.float64), size=5, mode="nearest").astype(np.float32)
    return img


def metric_name(cfg):
    return "gabor_bank_px_filters_per_s" if cfg["kind"] == "bank" else "sdft_px_bins_per_s"


def unit_name(cfg):
    return "px*filters/s" if cfg["kind"] == "bank" else "px*bins/s"


def scaling_of(config):
    return "weak" if config == 2 else "strong"


def config_dict(args, cfg, world):
    """The `config` object of the JSON line -- identical for both arms."""
    par = {2: "image per rank (weak)", 3: "images sharded", 4: "conjugate u-pairs sharded",
           5: "(frequency, theta/pi-theta) units partitioned (partition_units)"}[args.config]
    return {"workload": cfg["workload"], "smoother": args.smoother,
            "l2": "256 MiB flush between timed steps (inputs and outputs also exceed L2)" if args.config in (4, 5)
            else "256 MiB flush between timed steps",
            "parallelism": f"{par} x{world}"}


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clocks + throttle reasons DURING the timed region (NVML polling
    thread, 1 ms period, so even sub-second regions get samples)."""

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
# reference CPU arm
# ---------------------------------------------------------------------------
_REF: dict = {}  # worker state, set in the parent before the fork


def load_reference():
    """The unmodified reference package from baseline/_ref, else None."""
    if not os.path.isdir(os.path.join(REF_DIR, "fastgabor")):
        try:  # this container: install it (never on the GPU box: /root/reference is absent there)
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from install_reference import install

            install()
        except Exception:  # noqa: BLE001 -- a failed install falls back to the port
            pass
    if not os.path.isdir(os.path.join(REF_DIR, "fastgabor")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fgb_numba_cache")  # gabor.py:24,46 cache=True
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import fastgabor

    return fastgabor


def _ref_image(i):
    cfg = _REF["cfg"]
    if cfg["kind"] == "sdft" or cfg["images"] == 1:
        return _REF["img"]
    return make_image(cfg, i).astype(np.float64)


def _ref_task(task):
    """One task of a reference step; returns the units it produced.

    bank: ("bank", image, i, k, y0, y1) -- the reference's own unit of work in
    compute_bank (bank.py:103-116: horizontal_stage, vertical_stage and, for
    k with a mirror N-k, vertical_stage_conjugate) on output rows [y0, y1),
    computed on the band with ceil(3 sigma) real context rows on each side
    (FIR r=3: the kept rows equal the full-image outputs).
    sdft: ("sdft", y0, y1) -- sdft_full (sdft.py:178-213) on the band + context."""
    F, cfg = _REF["F"], _REF["cfg"]
    if task[0] == "bank":
        _, im, i, k, y0, y1 = task
        img = _ref_image(im)
        n, omega, sigma = cfg["n"], cfg["freqs"][i], cfg["sigmas"][i]
        h = max(1, math.ceil(3.0 * sigma))
        a, b = max(0, y0 - h), min(img.shape[0], y1 + h)
        band = np.ascontiguousarray(img[a:b])
        outs = 2 if n // 2 < n - k < n else 1
        if F is not None:
            c = F.OpCounters()
            hs = F.horizontal_stage(F.RealImage.from_array(band), F.GaborParams(omega, k * math.pi / n, sigma),
                                    F.ExactFIR(3.0), c)
            F.vertical_stage(hs, c)
            if outs == 2:
                F.vertical_stage_conjugate(hs, c)
        else:
            from oracle import fastgabor_oracle as O

            jr, ji = O.horizontal_stage(band, omega, k * math.pi / n, sigma, ("fir", 3.0))
            O.vertical_stage(jr, ji, omega, k * math.pi / n, sigma, ("fir", 3.0))
            if outs == 2:
                O.vertical_stage(jr, ji, omega, k * math.pi / n, sigma, ("fir", 3.0), conjugate=True)
        return (y1 - y0) * img.shape[1] * outs
    _, y0, y1 = task
    img = _REF["img"]
    h = max(1, math.ceil(3.0 * cfg["sigma"]))
    a, b = max(0, y0 - h), min(img.shape[0], y1 + h)
    band = np.ascontiguousarray(img[a:b])
    m = cfg["m"]
    if F is not None:
        F.sdft_full(F.RealImage.from_array(band), F.SdftSpec(m, m, F.ExactFIR(3.0), cfg["sigma"]), F.OpCounters())
    else:
        from oracle import fastgabor_oracle as O

        O.sdft_full(band, m, m, ("fir", 3.0), cfg["sigma"])
    return (y1 - y0) * img.shape[1] * m * m


class RefArm:
    """The reference's CPU implementation on every host core, one bounded
    sample of the config's workload per step (a pool of processes, one per
    core, each running the reference's own stage functions single-threaded;
    heaviest tasks first):

    * config 2: the whole bank on the whole image -- its 20 (frequency,
      direct k) units (compute_bank's threads= grain, bank.py:77-87);
    * config 3: 4 whole images per step (rotating through the 64), 25 units each;
    * config 5: all 45 units on a 1024-row band (rotating through the 8192
      rows), each with its 3 sigma context rows -- the reference's stages need
      86 GB for the whole image in float64;
    * config 4: sdft_full on 16 bands of 192 rows (+ context), rotating.
    """

    def __init__(self, args, cfg):
        self.args, self.cfg = args, cfg
        self.F = load_reference()
        self.kind = "reference" if self.F is not None else "port"
        _REF.update(F=self.F, cfg=cfg)
        if cfg["kind"] == "sdft" or cfg["images"] == 1:
            _REF["img"] = make_image(cfg, 0).astype(np.float64)
        self.cores = os.cpu_count() or 1

    def tasks(self, step, warm):
        cfg = self.cfg
        nh = cfg.get("n", 0) // 2
        if self.args.config == 2:
            t = [("bank", 0, i, k, 0, cfg["size"]) for i in range(len(cfg["freqs"])) for k in range(nh + 1)]
        elif self.args.config == 3:
            ims = [(4 * step + j) % cfg["images"] for j in range(1 if warm else 4)]
            t = [("bank", im, i, k, 0, cfg["size"]) for im in ims for i in range(len(cfg["freqs"]))
                 for k in range(nh + 1)]
        elif self.args.config == 5:
            s = min(64 if warm else 1024, cfg["size"])
            y0 = (step * s) % (cfg["size"] - s + 1)
            t = [("bank", 0, i, k, y0, y0 + s) for i in range(len(cfg["freqs"])) for k in range(nh + 1)]
        else:
            s = 16 if warm else 192
            t = []
            for j in range(self.cores):
                y0 = ((step * self.cores + j) * s) % (cfg["size"] - s + 1)
                t.append(("sdft", y0, y0 + s))
        if t and t[0][0] == "bank":
            t.sort(key=lambda x: -cfg["sigmas"][x[2]])  # LPT: largest sigma first
        return t

    def sample_text(self):
        what = {2: "the whole bank on the whole image per step",
                3: "4 whole images per step (rotating over the 64), all 25 units each",
                4: f"sdft_full on {self.cores} bands of 192 rows (+12 context rows each side) per step, rotating",
                5: "all 45 (frequency, direct k) units on a 1024-row band per step (+ceil(3 sigma) context rows "
                   "each side, kept rows identical to the full-image outputs), rotating over the 8192 rows"}
        src = ("unmodified reference fastgabor (baseline/_ref) stage functions" if self.kind == "reference"
               else "oracle port (NumPy fp64 restatement; baseline/_ref absent)")
        return f"{src}, FIR r=3, float64; {what[self.args.config]}; pool of {self.cores} processes"

    def run(self, steps, warmup, pool):
        for w in range(warmup):
            list(pool.imap_unordered(_ref_task, self.tasks(w, True), chunksize=1))
        tot_u, tot_s = 0, 0.0
        for s in range(steps):
            t0 = time.perf_counter()
            tot_u += sum(pool.imap_unordered(_ref_task, self.tasks(s, False), chunksize=1))
            tot_s += time.perf_counter() - t0
        return tot_u, tot_s


def ref_pool(arm):
    import multiprocessing as mp

    if arm.F is not None:  # JIT the reference's Numba kernels once in the parent (inherited by the fork)
        _ref_task(("bank", 0, 0, 1, 0, 8) if arm.cfg["kind"] == "bank" else ("sdft", 0, 8))
    return mp.get_context("fork").Pool(arm.cores)


def run_reference(args, cfg, world):
    arm = RefArm(args, cfg)
    with ref_pool(arm) as pool:
        u, s = arm.run(args.steps, args.warmup, pool)
    v = u / s
    line = {
        "impl": "reference", "metric": metric_name(cfg), "value": v, "unit": unit_name(cfg), "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * s / args.steps, "higher_is_better": True,
        "scaling": scaling_of(args.config), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, cfg, world),
        "cpu_baseline": {"value": v, "unit": unit_name(cfg), "cores": arm.cores, "kind": arm.kind,
                         "sample": arm.sample_text()},
        "e2e": {"value": v, "unit": unit_name(cfg), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class Dist:
    """Rank plumbing: NCCL (one GPU per rank) or gloo (ranks may share a GPU;
    collectives on host tensors)."""

    def __init__(self, world, rank, dev):
        import torch
        import torch.distributed as dist

        self.world, self.rank, self.dev = world, rank, dev
        self.backend = os.environ.get("FGB_DIST_BACKEND", "nccl")
        self.dist = dist
        if world > 1:
            if self.backend == "nccl":
                if torch.cuda.device_count() < world:
                    raise SystemExit(f"bench.py --gpus {world}: NCCL needs one GPU per rank and this box shows "
                                     f"{torch.cuda.device_count()}; FGB_DIST_BACKEND=gloo lets ranks share a GPU "
                                     "(plumbing check only, not a scaling measurement)")
                dist.init_process_group("nccl", device_id=dev)
            else:
                dist.init_process_group(self.backend)
        self.cdev = dev if self.backend == "nccl" else torch.device("cpu")

    def reduce(self, x, op="max"):
        if self.world == 1:
            return float(x)
        import torch

        t = torch.tensor([float(x)], dtype=torch.float64, device=self.cdev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return t.item()

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def broadcast_image(self, host):
        """The one input broadcast of the sharded configs (outside the timed
        steps), timed on the device for NCCL (max over ranks)."""
        import torch

        if self.world == 1:
            return torch.from_numpy(host).to(self.dev), None
        if self.backend != "nccl":
            t = torch.from_numpy(host) if self.rank == 0 else torch.empty(host.shape, dtype=torch.float32)
            self.dist.broadcast(t, 0)
            return t.to(self.dev), None
        t = torch.from_numpy(host).to(self.dev) if self.rank == 0 else torch.empty(host.shape, dtype=torch.float32,
                                                                                   device=self.dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.barrier()
        torch.cuda.synchronize()
        e0.record()
        self.dist.broadcast(t, 0)
        e1.record()
        torch.cuda.synchronize()
        return t, self.reduce(e0.elapsed_time(e1))

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def build_workload(args, cfg, D):
    """(plan, device input, host input array, units of this rank per step, broadcast ms)."""
    import paper_1704_05231_b200 as fg
    from paper_1704_05231_b200.device import BankPlan, SdftPlan
    from paper_1704_05231_b200.parallel import partition_units, sdft_heads, shard_images

    kind = fg.ExactFIR(3.0) if args.smoother == "fir" else fg.RecursiveIIR()
    bcast = None
    if cfg["kind"] == "bank":
        spec = fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"]))
        units = None
        if args.config == 3:
            mine = shard_images(cfg["images"], D.world)[D.rank]
            imgs = np.stack([make_image(cfg, i) for i in mine])
            timg = __import__("torch").from_numpy(imgs).to(D.dev)
        elif args.config == 5:
            units = (partition_units(cfg["freqs"], cfg["sigmas"], cfg["n"], D.world, 3.0)[D.rank]
                     if D.world > 1 else None)
            imgs = make_image(cfg, 0)[None] if D.rank == 0 or D.backend != "nccl" else np.empty(
                (1, cfg["size"], cfg["size"]), np.float32)
            timg, bcast = D.broadcast_image(imgs)
            imgs = timg.cpu().numpy() if D.rank != 0 else imgs
        else:
            imgs = make_image(cfg, D.rank)[None]
            timg = __import__("torch").from_numpy(imgs).to(D.dev)
        plan = BankPlan(tuple(timg.shape), spec, kind, "f32", True, units)
        units_step = timg.shape[0] * timg.shape[1] * timg.shape[2] * plan.entries
    else:
        spec = fg.SdftSpec(cfg["m"], cfg["m"], kind, cfg["sigma"])
        heads = sdft_heads(cfg["m"], D.world)[D.rank] if D.world > 1 else None
        imgs = make_image(cfg, 0)[None]
        timg, bcast = D.broadcast_image(imgs)
        plan = SdftPlan(tuple(timg.shape), spec, "f32", heads)
        units_step = timg.shape[1] * timg.shape[2] * plan.bins
    return plan, timg, imgs, units_step, bcast


def fma_pipe(config, name):
    """ncu FMA-pipe utilisation (%) of a kernel family on this config (profiles/r02/fma_pipe.json, committed):
    the hardware-utilisation figure beside the reference-flop roofline (the row kernel's symmetric pairs
    issue fewer flops than the reference counts, so its reference-flop `frac` can exceed 1)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "fma_pipe.json")) as fh:
            return json.load(fh).get(f"cfg{config}/{name}")
    except (OSError, ValueError):
        return None


def roofline(args, cfg, prof, nprof, fp32, hbm):
    """Dominant kernel (longest total time in the live profile) against its bound."""
    top = max(prof, key=lambda e: e["ms"]) if prof else None
    if top is None:
        return None
    traffic = None
    for rnd in ("r02", "r01"):  # ncu DRAM bytes per launch of that kernel (profiles/, committed)
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "traffic.json")) as fh:
                traffic = json.load(fh).get(f"cfg{args.config}/{top['name']}")
        except (OSError, ValueError):
            continue
        if traffic is not None:
            break
    fma = fma_pipe(args.config, top["name"])
    if top["name"].endswith("_umma"):
        # tensor-core split-fp16 passes: bounded by HBM (J read once + outputs written);
        # the reference-counted flops they replace are reported beside, not as the bound
        ach = top["bytes"] / (top["ms"] * 1e-3) / 1e9
        return {"bound": "hbm", "kernel": top["name"], "ncu_fma_pipe_pct": None, "achieved": ach, "peak": hbm,
                "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
                "algorithmic_bytes_per_launch": top["bytes"] / top["launches"],
                "ref_flops_tflops": top["flops"] / (top["ms"] * 1e-3) / 1e12,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "note": {"bank_umma": "algorithmic bytes = the image read once + complex64 outputs written once "
                                      "(row + column passes of a frequency in one kernel, J in shared memory)",
                         "row_umma": "algorithmic bytes = the image read once + split-fp16 J planes written once "
                                     "(8 B per px and direct)"}.get(
                    top["name"], "algorithmic bytes = J planes read once (split-fp16 hi+lo, 8 B per px) + complex64 "
                                 "outputs written once")
                + "; ref_flops_tflops = the reference OpCounters flops of the stage / time"}
    if cfg["kind"] == "sdft":
        ach = top["bytes"] / (top["ms"] * 1e-3) / 1e9
        return {"bound": "hbm", "kernel": top["name"], "ncu_fma_pipe_pct": fma, "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": traffic, "algorithmic_bytes_per_launch": top["bytes"] / top["launches"],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    ach = top["flops"] / (top["ms"] * 1e-3) / 1e12
    r = {"bound": "fp32", "kernel": top["name"], "ncu_fma_pipe_pct": fma, "achieved": ach, "peak": fp32,
         "unit": "TFLOP/s",
         "frac": ach / fp32 if fp32 > 0 else None, "traffic": traffic,
         "algorithmic_flops_per_launch": top["flops"] / top["launches"],
         "peak_source": "live FFMA probe (fgb_probe_fp32_tflops); flops = reference OpCounters M+A"}
    if top["name"] == "iir":
        r["note"] = ("RecursiveIIR stage: reference flops (~12 per output and plane); the exact segment-parallel "
                     "fp32 recursion issues ~36 FMA per sample and plane in two passes (DESIGN.md section 5)")
    return r


def run_ours(args, cfg, world, rank, local_rank):
    import torch

    from paper_1704_05231_b200 import _native as N

    dev = torch.device("cuda", local_rank % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    D = Dist(world, rank, dev)
    try:
        plan, timg, imgs, units_step, bcast = build_workload(args, cfg, D)
        out = plan.new_output(dev)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

        def step():
            plan(timg, out)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        D.barrier()
        torch.cuda.synchronize()
        l0 = N.lib.fgb_launch_count()
        with ClockSampler(dev.index) as clk:
            for k in range(args.steps):
                flush.zero_()
                starts[k].record()
                step()
                ends[k].record()
            torch.cuda.synchronize()
        launches = D.reduce(N.lib.fgb_launch_count() - l0, "sum")
        D.barrier()
        per_step = sorted(s.elapsed_time(e) for s, e in zip(starts, ends))
        max_ms = D.reduce(sum(per_step))
        units_all = D.reduce(units_step, "sum")
        value = units_all * args.steps / (max_ms / 1e3)
        step_stats = {"min": per_step[0], "p50": per_step[len(per_step) // 2],
                      "p90": per_step[min(len(per_step) - 1, (9 * len(per_step)) // 10)], "max": per_step[-1]}

        # ---- live per-kernel profile (CUDA events on the launching stream; the library
        #      serialises its stream lanes while profiling so each kernel is timed alone) ----
        N.lib.fgb_profile_enable(1)
        N.profile_read()
        nprof = max(1, min(20 if args.config != 5 else 3, args.steps))
        for _ in range(nprof):
            flush.zero_()
            step()
        torch.cuda.synchronize()
        prof = N.profile_read()
        N.lib.fgb_profile_enable(0)
        fp32 = N.lib.fgb_probe_fp32_tflops()
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
                hbm = json.load(fh).get("hbm_gbs", 6650.0)
        except (OSError, ValueError):  # absent: B200_PROFILING.md's fallback copy bandwidth
            hbm = 6650.0
        tot_ms = sum(x["ms"] for x in prof) or 1.0
        kernels = {e["name"]: {"launches_per_step": e["launches"] / nprof, "ms_per_launch": e["ms"] / e["launches"],
                               "share": e["ms"] / tot_ms,
                               "tflops": e["flops"] / (e["ms"] * 1e-3) / 1e12 if e["ms"] > 0 else None,
                               "gbs": e["bytes"] / (e["ms"] * 1e-3) / 1e9 if e["ms"] > 0 else None,
                               "ncu_fma_pipe_pct": fma_pipe(args.config, e["name"])} for e in prof}
        roof = roofline(args, cfg, prof, nprof, fp32, hbm)
        step_roof = None
        if prof:
            work = {k: sum(e[k] for e in prof) / nprof for k in ("flops", "bytes")}
            step_s = max_ms / args.steps / 1e3
            if cfg["kind"] == "sdft" or (roof and roof["kernel"].endswith("_umma")):
                ach = work["bytes"] / step_s / 1e9
                step_roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
                if cfg["kind"] == "bank":
                    step_roof["ref_flops_tflops"] = work["flops"] / step_s / 1e12
                    step_roof["note"] = ("bytes of this rank's step summed over its kernels (image reads, J planes "
                                         "written and read once, outputs written) / step time (lanes overlapped)")
            else:
                ach = work["flops"] / step_s / 1e12
                step_roof = {"bound": "fp32", "achieved": ach, "peak": fp32, "unit": "TFLOP/s",
                             "frac": ach / fp32 if fp32 > 0 else None,
                             "note": "reference OpCounters flops of this rank's step / step time (lanes overlapped)"}

        # ---- e2e: host buffers through the C ABI (H2D + compute + D2H every step), max over ranks ----
        hin = torch.from_numpy(np.ascontiguousarray(imgs)).pin_memory()
        hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        desc = plan.desc
        desc.img.pitch = imgs.shape[2]
        desc.img.batch_stride = imgs.shape[1] * imgs.shape[2]
        call = N.lib.fgb_bank_host if cfg["kind"] == "bank" else N.lib.fgb_sdft_host
        ne = max(3, min(args.steps, 20 if args.config != 5 else 8))
        N.check(call(C.byref(desc), C.c_void_p(hin.data_ptr()), C.c_void_p(hout.data_ptr())))
        D.barrier()
        t0 = time.perf_counter()
        for _ in range(ne):
            N.check(call(C.byref(desc), C.c_void_p(hin.data_ptr()), C.c_void_p(hout.data_ptr())))
        e2e_s = D.reduce((time.perf_counter() - t0) / ne)
        # the PCIe link alone: the same H2D + D2H bytes as bare pinned copies
        dev_in = torch.empty(hin.shape, dtype=hin.dtype, device=dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(ne):
            dev_in.copy_(hin, non_blocking=True)
            hout.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
        link_s = (time.perf_counter() - t1) / ne
        del dev_in
        h2d, d2h = int(hin.numel() * hin.element_size()), int(hout.numel() * hout.element_size())
        e2e = {"value": units_all / e2e_s, "unit": unit_name(cfg), "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "link_copy_ms": link_s * 1e3,
               "link_gbs": (h2d + d2h) / link_s / 1e9, "frac_of_link": link_s / e2e_s,
               "note": "host buffers through fgb_*_host (H2D, compute, D2H per step; bytes of rank 0); "
                       "link_copy_ms = the same bytes as bare pinned copies"}
        del hin, hout

        # ---- CPU baseline (rank 0, N=1): one step of the reference arm ----
        cpu = None
        if rank == 0 and world == 1 and not args.no_cpu:
            arm = RefArm(args, cfg)
            with ref_pool(arm) as pool:
                u, s = arm.run(1, 0, pool)
            cpu = {"value": u / s, "unit": unit_name(cfg), "cores": arm.cores, "kind": arm.kind,
                   "sample": arm.sample_text() + f"; one step, {s:.1f} s"}
        if rank == 0:
            line = {
                "metric": metric_name(cfg), "value": value, "unit": unit_name(cfg), "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
                "higher_is_better": True, "scaling": scaling_of(args.config), "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded, BASELINE.json shapes)", "config": config_dict(args, cfg, world),
                "input_broadcast_ms": bcast, "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(), "kernels": kernels,
                "fp32_peak_tflops_measured": fp32, "step_ms_rank0": step_stats,
                "dist_backend": D.backend if world > 1 else None,
            }
            print(json.dumps(line), flush=True)
    finally:
        D.close()


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: re-run this script with N ranks."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=[2, 3, 4, 5])
    ap.add_argument("--smoother", default="fir", choices=["fir", "iir"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--size", type=int, default=None, help="test runs only: override the image size")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.size:
        cfg["size"] = args.size
        cfg["workload"] += f" [reduced to {args.size}^2: not a BASELINE measurement]"
        if cfg["kind"] == "bank":
            cfg["images"] = min(cfg["images"], 8)
    env_world = os.environ.get("WORLD_SIZE")
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:  # under torchrun only rank 0 runs the CPU arm; the others exit 0
            run_reference(args, cfg, int(env_world or args.gpus))
        return 0
    if env_world is None and args.gpus > 1:
        return relaunch(args)
    world = int(env_world or 1)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE={world}")
    run_ours(args, cfg, world, rank, int(os.environ.get("LOCAL_RANK", "0")))
    return 0


if __name__ == "__main__":
    sys.exit(main())
