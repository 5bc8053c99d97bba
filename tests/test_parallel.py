"""Multi-GPU partitioning logic, tested on CPU with
gloo at world size 2: broadcast of the image, per-rank LPT unit shares, the
compact output order, and that the union of the shards is the full bank."""

import math
import os
import socket

import numpy as np
import pytest

from paper_1704_05231_b200 import parallel as P


def test_shard_images_cover_once():
    for world in (1, 2, 3, 4, 8):
        parts = P.shard_images(64, world)
        flat = [i for p in parts for i in p]
        assert flat == list(range(64))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_lpt_units_balanced_config5():
    freqs = [math.pi / 2 ** j for j in range(1, 6)]
    sig = [2.0 ** j for j in range(1, 6)]
    costs = P.bank_unit_costs(freqs, sig, 16, 3.0)
    assert len(costs) == 5 * 9
    for world in (2, 4, 8):
        parts = P.lpt_assign(costs, world)
        flat = sorted(u for p in parts for u in p)
        assert flat == sorted(costs)
        assert P.load_balance(parts, costs) < 1.05
        ent = [e for p in parts for e in P.unit_entries(p, 16)]
        assert sorted(ent) == sorted((i, k) for i in range(5) for k in range(16))


def test_partition_units_config5():
    """Contiguous runs per rank (shared row launches) + local search; every unit once;
    modelled efficiency at 2/4/8 ranks against the measured cost model."""
    freqs = [math.pi / 2 ** j for j in range(1, 6)]
    sig = [2.0 ** j for j in range(1, 6)]
    total = P.partition_cost([list(range(45))], sig, 16)[0]
    assert abs(total * 67.108864 - 14.9) < 1.5  # the measured config-5 step (profiles/r02/bench_c5.json: 14.25 ms)
    for world, eff in ((1, 1.0), (2, 0.98), (4, 0.95), (8, 0.93)):
        parts = P.partition_units(freqs, sig, 16, world)
        assert sorted(u for p in parts for u in p) == list(range(45))
        c = P.partition_cost(parts, sig, 16)
        assert total / world / max(c) >= eff, (world, total / world / max(c))
    # partition beats unit-LPT (which splits frequencies across ranks and loses row sharing)
    lpt = P.lpt_assign(P.bank_unit_costs(freqs, sig, 16), 8)
    assert max(P.partition_cost(P.partition_units(freqs, sig, 16, 8), sig, 16)) < max(P.partition_cost(lpt, sig, 16))


def test_run_cost_model_matches_measurements():
    """A few measured B200 points of profiles/r02/unit_costs_c5.json (kernel ms, 8192^2)."""
    mpx = 67.108864
    for sigma, ks, ms in ((32.0, range(9), 4.346), (16.0, range(9), 2.984), (8.0, [3], 0.334), (4.0, range(5), 1.301),
                          (8.0, range(9), 2.315), (16.0, [1], 0.396), (2.0, range(9), 1.984)):
        got = P.run_cost(sigma, ks, 16, 3.0, mpx)
        # the model sits above the bare kernel times: its per-unit terms carry what a rank's whole call costs
        # beyond them (cold L2, launch tails; largest for the small half-widths, parallel.py:_FIT)
        assert -0.05 < (got - ms) / ms < 0.40, (sigma, list(ks), got, ms)


def test_sdft_heads_cover_all_bins():
    for world in (1, 2, 4, 8):
        parts = P.sdft_heads(16, world)
        bins = [b for p in parts for b in P.head_bins(p, 16)]
        assert sorted(bins) == sorted((u, v) for u in range(16) for v in range(16))
    parts = P.sdft_heads(16, 8)
    assert sorted(len(P.head_bins(p, 16)) for p in parts) == [32] * 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import fastgabor_oracle as O
    import paper_1704_05231_b200 as fg

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = fg.BankSpec((math.pi / 2, math.pi / 4), 8, (2.0, 4.0))
    if rank == 0:
        img = torch.from_numpy(np.random.default_rng(9).uniform(0, 1, (20, 24)))
    else:
        img = torch.zeros((20, 24), dtype=torch.float64)

    def cpu_compute(im, sp, kind, units):  # CPU stand-in for the device kernels
        f = im.numpy()
        outs = []
        for (i, k) in P.unit_entries(units, sp.orientations_n):
            re, imag = O.gabor_filter(f, sp.frequencies[i], k * math.pi / 8, sp.sigma_for(i), ("fir", 3.0))
            outs.append(re + 1j * imag)
        return torch.from_numpy(np.stack(outs))

    out, entries = P.sharded_bank(img, spec, fg.ExactFIR(3.0), compute=cpu_compute)
    # the broadcast delivered rank 0's image everywhere
    chk = img.sum().item()
    q.put((rank, chk, entries, out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_sharded_bank_equals_full():
    import torch.multiprocessing as mp

    from oracle import fastgabor_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    assert res[0][1] == pytest.approx(res[1][1])  # same image on both ranks
    f = np.random.default_rng(9).uniform(0, 1, (20, 24))
    full = O.compute_bank(f, (math.pi / 2, math.pi / 4), 8, (2.0, 4.0), ("fir", 3.0))
    seen = set()
    for _, _, entries, out in res:
        for (i, k), plane in zip(entries, out):
            ref = full[i * 8 + k]
            assert np.max(np.abs(plane.real - ref[3])) < 1e-12 and np.max(np.abs(plane.imag - ref[4])) < 1e-12
            seen.add((i, k))
    assert seen == {(i, k) for i in range(2) for k in range(8)}


def test_c_abi_partition_equals_python():
    """fgb_mgpu_bank_units / fgb_mgpu_sdft_heads (csrc/mgpu.cu, host-only) give the
    same shards as parallel.partition_units / sdft_heads."""
    import ctypes as C

    from paper_1704_05231_b200 import _native as N
    from paper_1704_05231_b200.bank import BankSpec, bank_desc
    from paper_1704_05231_b200.gaussian import ExactFIR

    cases = [([math.pi / 2 ** j for j in range(1, 6)], [2.0 ** j for j in range(1, 6)], 16),
             ([math.pi / 2 ** j for j in range(1, 6)], [2.0 ** j for j in range(1, 6)], 8),
             ([math.pi / 2 ** j for j in (1, 2, 3, 4)], [2.0, 4.0, 8.0, 16.0], 8),
             ([0.5, 1.0, 2.0], [5.0, 1.5, 0.9], 7), ([1.0], [3.0], 1)]
    for freqs, sig, n in cases:
        d, _keep = bank_desc(64, 64, BankSpec(tuple(freqs), n, tuple(sig)), ExactFIR(3.0), "f32", True)
        for world in (1, 2, 3, 4, 8, 64):
            py = P.partition_units(freqs, sig, n, world, 3.0)
            for r in range(world):
                buf = (C.c_int32 * 512)()
                cnt = N.check(N.lib.fgb_mgpu_bank_units(C.byref(d), world, r, buf, 512), mgpu=True)
                assert list(buf[:cnt]) == (py[r] if r < len(py) else []), (freqs, n, world, r)
    for m in (1, 4, 16, 32):
        for world in (1, 2, 4, 8):
            py = P.sdft_heads(m, world)
            for r in range(world):
                buf = (C.c_int32 * 64)()
                cnt = N.check(N.lib.fgb_mgpu_sdft_heads(m, world, r, buf, 64), mgpu=True)
                assert list(buf[:cnt]) == py[r], (m, world, r)
    with pytest.raises(ValueError):
        N.check(N.lib.fgb_mgpu_sdft_heads(16, 2, 2, (C.c_int32 * 4)(), 4), mgpu=True)
