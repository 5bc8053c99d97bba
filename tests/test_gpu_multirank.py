"""Multi-rank device path on ONE GPU: two gloo ranks share cuda:0 and each
computes its shard through libfgb200 -- no rank waits on another's kernels,
so this is a correctness test of the sharding, not a scaling measurement.

* config-5 style single-image bank: the image broadcast from rank 0, LPT
  (frequency, direct k) units per rank (parallel.sharded_bank, device compute);
* config-3 style batches: images sharded;
* config-4 style SDFT: conjugate u-pair heads sharded;

the union of the shards equals the 1-rank output bit for bit.  Plus
bench.py --gpus 2 end to end (it relaunches itself under torchrun)."""

import json
import math
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FREQS = tuple(math.pi / 2 ** j for j in range(1, 6))
SIGMAS = tuple(2.0 ** j for j in range(1, 6))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_1704_05231_b200 as fg
    from paper_1704_05231_b200 import parallel as P
    from paper_1704_05231_b200.device import BankPlan, SdftPlan

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    res = {}
    # (1) single-image bank, LPT units
    spec = fg.BankSpec(FREQS, 16, SIGMAS)
    img = torch.from_numpy(np.random.default_rng(3).uniform(0, 1, (320, 352)).astype(np.float32)) if rank == 0 \
        else torch.zeros((320, 352), dtype=torch.float32)

    def dev_compute(im, sp, kind, units):
        from paper_1704_05231_b200.device import compute_bank

        return compute_bank(im.cuda(), sp, kind, True, units)[0].cpu()

    out, entries = P.sharded_bank(img, spec, fg.ExactFIR(3.0), compute=dev_compute)
    res["bank"] = (entries, out.numpy())
    # (2) batched images
    spec3 = fg.BankSpec(FREQS, 8, SIGMAS)
    mine = P.shard_images(5, world)[rank]
    imgs = np.stack([np.random.default_rng(100 + i).uniform(0, 1, (192, 160)).astype(np.float32) for i in mine])
    t = torch.from_numpy(imgs).cuda()
    res["images"] = (mine, BankPlan(tuple(t.shape), spec3, fg.ExactFIR(3.0), "f32", True)(t).cpu().numpy())
    # (3) SDFT heads
    heads = P.sdft_heads(16, world)[rank]
    f = torch.from_numpy(np.random.default_rng(2).uniform(0, 1, (1, 200, 232)).astype(np.float32)).cuda()
    sspec = fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0)
    res["sdft"] = (P.head_bins(heads, 16), SdftPlan(tuple(f.shape), sspec, "f32", heads)(f)[0].cpu().numpy())
    torch.cuda.synchronize()
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_gloo_ranks_device_shards_equal_full():
    import torch
    import torch.multiprocessing as mp

    import paper_1704_05231_b200 as fg
    from paper_1704_05231_b200.device import BankPlan, SdftPlan

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=500) for _ in range(2))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0

    # 1-rank references on the same device
    img = torch.from_numpy(np.random.default_rng(3).uniform(0, 1, (1, 320, 352)).astype(np.float32)).cuda()
    full = BankPlan(tuple(img.shape), fg.BankSpec(FREQS, 16, SIGMAS), fg.ExactFIR(3.0), "f32", True)(img)[0].cpu().numpy()
    seen = set()
    for r in (0, 1):
        entries, out = got[r]["bank"]
        for (i, k), plane in zip(entries, out):
            assert np.array_equal(plane, full[i * 16 + k]), (r, i, k)
            seen.add((i, k))
    assert seen == {(i, k) for i in range(5) for k in range(16)}

    imgs = np.stack([np.random.default_rng(100 + i).uniform(0, 1, (192, 160)).astype(np.float32) for i in range(5)])
    t = torch.from_numpy(imgs).cuda()
    full3 = BankPlan(tuple(t.shape), fg.BankSpec(FREQS, 8, SIGMAS), fg.ExactFIR(3.0), "f32", True)(t).cpu().numpy()
    done = []
    for r in (0, 1):
        mine, out = got[r]["images"]
        for j, i in enumerate(mine):
            assert np.array_equal(out[j], full3[i])
            done.append(i)
    assert sorted(done) == list(range(5))

    f = torch.from_numpy(np.random.default_rng(2).uniform(0, 1, (1, 200, 232)).astype(np.float32)).cuda()
    fulls = SdftPlan(tuple(f.shape), fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0), "f32")(f)[0].cpu().numpy()
    bins = []
    for r in (0, 1):
        hb, out = got[r]["sdft"]
        for (u, v), plane in zip(hb, out):
            assert np.array_equal(plane, fulls[u * 16 + v]), (r, u, v)
            bins.append((u, v))
    assert sorted(bins) == [(u, v) for u in range(16) for v in range(16)]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("config,size", [(5, 1024), (3, 256), (4, 512)])
def test_bench_two_ranks_gloo(config, size):
    env = dict(os.environ, FGB_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", str(config),
                        "--size", str(size), "--steps", "2", "--warmup", "3", "--no-cpu"],
                       capture_output=True, text=True, timeout=800, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["dist_backend"] == "gloo"
    assert line["scaling"] == "strong" and line["e2e"]["value"] > 0


def test_library_nccl_driver_world1():
    """fgb_mgpu_* (library-owned NCCL communicator) at world size 1 on this GPU:
    the 'broadcast' is a no-op, the rank owns every unit / head, and the outputs
    equal the plain calls bit for bit.  (Multi-rank NCCL needs one GPU per rank.)"""
    import torch

    import paper_1704_05231_b200 as fg
    from paper_1704_05231_b200.device import BankPlan, SdftPlan
    from paper_1704_05231_b200 import _native as N
    from paper_1704_05231_b200.parallel import LibComm, partition_units

    comm = LibComm(1, 0, 0)
    try:
        img = torch.from_numpy(np.random.default_rng(4).uniform(0, 1, (1, 256, 288)).astype(np.float32)).cuda()
        plan = BankPlan(tuple(img.shape), fg.BankSpec(FREQS, 16, SIGMAS), fg.ExactFIR(3.0), "f32", True)
        full = plan(img)
        assert comm.units(plan.desc) == partition_units(FREQS, SIGMAS, 16, 1, 3.0)[0] == list(range(45))
        assert N.lib.fgb_mgpu_bank_entries(C_byref(plan.desc)) == 80
        out = torch.empty_like(full)
        comm.bank(plan.desc, img, out, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        # world 1 owns all 45 units: compact order = per unit direct then mirror
        from paper_1704_05231_b200.parallel import unit_entries

        for j, (i, k) in enumerate(unit_entries(list(range(45)), 16)):
            assert torch.equal(out[0, j], full[0, i * 16 + k])
        sp = SdftPlan(tuple(img.shape), fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0), "f32")
        sfull = sp(img)
        sout = torch.empty_like(sfull)
        comm.sdft(sp.desc, img, sout, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        from paper_1704_05231_b200.parallel import head_bins

        for j, (u, v) in enumerate(head_bins(list(range(9)), 16)):
            assert torch.equal(sout[0, j], sfull[0, u * 16 + v])
    finally:
        comm.close()


def C_byref(x):
    import ctypes

    return ctypes.byref(x)
