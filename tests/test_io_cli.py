"""File I/O, metrics and CLI surface: host-side tests run on CPU
against bytes/values produced by the reference; GPU-side tests (device-fed
GBNK writer, CLI end to end) are marked gpu."""

import math
import os

import numpy as np
import pytest

from .conftest import random_image


@pytest.fixture(scope="module")
def fg():
    import paper_1704_05231_b200 as m

    return m


def _entries(fg, z):
    f3 = z["f3"]
    return [(fg.GaborParams(1.0 + i, 0.3 * i, 2.0), fg.ComplexImage.from_planes(f3 * (i + 1), -f3 / (i + 2)))
            for i in range(3)]


def test_gbnk_writer_bytes_match_reference(fg, golden, tmp_path):
    z, _ = golden
    ents = _entries(fg, z)
    p = tmp_path / "b.gbnk"
    fg.write_bank_container(ents, p)
    assert np.array_equal(np.frombuffer(p.read_bytes(), dtype=np.uint8), z["io.gbnk_bytes"])
    fg.write_bank_container([((1.0, 2.0, 0.5), ents[0][1])], p, sdft=True)
    assert np.array_equal(np.frombuffer(p.read_bytes(), dtype=np.uint8), z["io.gbnk_sdft_bytes"])
    back, sdft = fg.read_bank_container(p)
    assert sdft and back[0][0] == (1.0, 2.0, 0.5)
    assert np.array_equal(back[0][1].re, ents[0][1].re)


def test_gbnk_errors(fg, tmp_path):
    p = tmp_path / "x.gbnk"
    p.write_bytes(b"NOPE" + b"\0" * 32)
    with pytest.raises(fg.ContainerFormatError):
        fg.read_bank_container(p)
    p.write_bytes(b"GBNK" + b"\1\0\0\0" + b"\4\0\0\0" * 3)
    with pytest.raises(fg.ContainerFormatError):
        fg.read_bank_container(p)
    with pytest.raises(ValueError):
        fg.write_bank_container([], p)


def test_magnitude_pgm_matches_reference_and_roundtrips(fg, golden, tmp_path):
    z, _ = golden
    ents = _entries(fg, z)
    p = tmp_path / "m.pgm"
    fg.write_magnitude(ents[1][1], p)
    assert np.array_equal(np.frombuffer(p.read_bytes(), dtype=np.uint8), z["io.magnitude_pgm_bytes"])
    img = fg.load_grayscale(p)
    assert img.data.shape == ents[1][1].re.shape and img.data.max() == 255.0


def test_pgm_16bit_and_errors(fg, tmp_path):
    data = (np.arange(12, dtype=np.uint16).reshape(3, 4) * 1000)
    p = tmp_path / "a.pgm"
    p.write_bytes(b"P5\n# comment\n4 3\n65535\n" + data.astype(">u2").tobytes())
    img = fg.load_grayscale(p)
    assert np.array_equal(img.data, data.astype(np.float64))
    p.write_bytes(b"P2\n4 3\n255\n")
    with pytest.raises(fg.ImageFormatError):
        fg.load_grayscale(p)
    p.write_bytes(b"P5\n4 3\n255\n\0\0")
    with pytest.raises(fg.ImageFormatError):
        fg.load_grayscale(p)


def test_ser_matches_reference(fg, golden):
    z, meta = golden
    ents = _entries(fg, z)
    f3 = z["f3"]
    b = fg.ComplexImage.from_planes(f3 * 1.01 + 0.3, -f3 / 2 + 0.01)
    assert fg.ser(b, ents[0][1], "real") == pytest.approx(meta["ser"]["real"], rel=1e-12)
    assert fg.ser(b, ents[0][1], "imag") == pytest.approx(meta["ser"]["imag"], rel=1e-12)
    assert fg.ser(ents[0][1], ents[0][1], "real") == math.inf


def test_cli_usage_errors():
    from paper_1704_05231_b200.cli import main

    assert main(["bank"]) == 1
    assert main(["sdft", "--input", "/nonexistent.pgm"]) == 1
    assert main(["bank", "--input", "/nonexistent.pgm", "--frequencies", ""]) == 1


def _write_pgm(path, arr):
    a = np.clip(arr, 0, 255).astype(np.uint8)
    path.write_bytes(b"P5\n%d %d\n255\n" % (a.shape[1], a.shape[0]) + a.tobytes())


@pytest.mark.gpu
def test_gpu_bruteforce_matches_reference_goldens(fg, golden):
    z, meta = golden
    f1 = fg.RealImage.from_array(z["f1"])
    for i in range(3):
        om, th, sg = meta["cases"][f"gabor.fir6.{i}"]["params"]
        out = fg.fir_gabor(f1, fg.GaborParams(om, th, sg), precision="f64")
        ref = (z[f"firgabor.{i}.re"], z[f"firgabor.{i}.im"])
        scale = max(np.abs(ref[0]).max(), np.abs(ref[1]).max())
        assert max(np.abs(out.re - ref[0]).max(), np.abs(out.im - ref[1]).max()) / scale <= 1e-12
    f3 = fg.RealImage.from_array(z["f3"])
    for kn, kind in (("fir6", fg.ExactFIR()), ("box1", fg.Box(1))):
        out = fg.localized_dft(f3, 1, 3, fg.SdftSpec(4, 4, kind), precision="f64")
        ref = (z[f"ldft.{kn}.re"], z[f"ldft.{kn}.im"])
        scale = max(np.abs(ref[0]).max(), np.abs(ref[1]).max())
        assert max(np.abs(out.re - ref[0]).max(), np.abs(out.im - ref[1]).max()) / scale <= 1e-12
    # radius 3 at sigma 16 / 32 (97^2 / 193^2 taps, wider than the 120x136 image): the banded
    # large-support path the config-3/5 full-size checks run
    f7 = fg.RealImage.from_array(z["f7"])
    for i in range(2):
        om, th, sg = meta["cases"][f"firgabor_r3.{i}"]["params"]
        ref = (z[f"firgabor_r3.{i}.re"], z[f"firgabor_r3.{i}.im"])
        scale = max(np.abs(ref[0]).max(), np.abs(ref[1]).max())
        for prec, tol in (("f64", 1e-12), ("f32", 1e-5)):
            out = fg.fir_gabor(f7, fg.GaborParams(om, th, sg), fg.OracleConfig(3.0), precision=prec)
            assert max(np.abs(out.re - ref[0]).max(), np.abs(out.im - ref[1]).max()) / scale <= tol, (i, prec)
    out = fg.localized_dft(f7, 5, 27, fg.SdftSpec(32, 32, fg.ExactFIR(3.0), 16.0), fg.OracleConfig(3.0),
                           precision="f64")
    ref = (z["ldft_r3.re"], z["ldft_r3.im"])
    scale = max(np.abs(ref[0]).max(), np.abs(ref[1]).max())
    assert max(np.abs(out.re - ref[0]).max(), np.abs(out.im - ref[1]).max()) / scale <= 1e-12


@pytest.mark.gpu
def test_gpu_device_gbnk_writer(fg, tmp_path):
    import torch

    from paper_1704_05231_b200.device import compute_bank

    f = random_image(3, 40, 0.0, 1.0, width=48)
    spec = fg.BankSpec((math.pi / 4,), 4, (2.0,))
    for prec, dt in (("f64", torch.float64), ("f32", torch.float32)):
        out = compute_bank(torch.from_numpy(f).to(dt).cuda(), spec, fg.ExactFIR(3.0))[0]
        params = [(spec.frequencies[0], k * math.pi / 4, 2.0) for k in range(4)]
        p = tmp_path / f"d_{prec}.gbnk"
        fg.write_container_from_device(out, params, p)
        torch.cuda.synchronize()
        back, sdft = fg.read_bank_container(p)
        host = out.cpu().numpy()
        assert not sdft and len(back) == 4
        for k, (tri, img) in enumerate(back):
            assert tri == params[k]
            assert np.array_equal(img.re, host[k].real.astype(np.float64))
            assert np.array_equal(img.im, host[k].imag.astype(np.float64))


@pytest.mark.gpu
def test_gpu_cli_end_to_end(fg, tmp_path):
    from paper_1704_05231_b200.cli import main

    rng = np.random.default_rng(4)
    pgm = tmp_path / "in.pgm"
    _write_pgm(pgm, rng.uniform(0, 255, (48, 56)))
    out = tmp_path / "bank.gbnk"
    assert main(["bank", "--input", str(pgm), "--output", str(out), "--smoother", "fir", "--orientations", "4",
                 "--magnitude-dir", str(tmp_path / "mag")]) == 0
    ents, _ = fg.read_bank_container(out)
    assert len(ents) == 20 and len(os.listdir(tmp_path / "mag")) == 20
    assert main(["sdft", "--input", str(pgm), "--output", str(tmp_path / "s.gbnk"), "--window", "4x4",
                 "--smoother", "fir"]) == 0
    ents, sdft = fg.read_bank_container(tmp_path / "s.gbnk")
    assert sdft and len(ents) == 16
    csvp = tmp_path / "cmp.csv"
    assert main(["compare", "--input", str(pgm), "--output", str(csvp), "--frequencies", "3.9"]) == 0
    lines = csvp.read_text().strip().splitlines()
    assert lines[0].startswith("omega,theta_deg") and len(lines) == 1 + 9
    fir_ser = [float(l.split(",")[5]) for l in lines[1:]]
    assert min(fir_ser) > 150.0  # f64 FIR decomposition vs brute force: exact to rounding
    assert main(["bench", "--size", "64", "--orientation-list", "4", "--sdft-windows", "4", "--repeats", "2",
                 "--output", str(tmp_path / "b.csv")]) == 0


@pytest.mark.gpu
def test_config2_full_vs_gpu_bruteforce(fg):
    """Every entry of BASELINE config 2 at full size (fp32 fast path) against the
    independent fp64 brute-force 2-D tap sum on the GPU, tol 1e-5."""
    import scipy.ndimage as ndi

    f64 = np.random.default_rng(1).uniform(0.0, 1.0, size=(1024, 1024)).astype(np.float32).astype(np.float64)
    f32 = ndi.uniform_filter(f64, size=5, mode="nearest").astype(np.float32)
    freqs = (math.pi / 2, math.pi / 4, math.pi / 8, math.pi / 16)
    spec = fg.BankSpec(freqs, 8, (2.0, 4.0, 8.0, 16.0))
    img = fg.RealImage.from_array(f32)
    out = fg.compute_bank(img, spec, fg.ExactFIR(3.0), fg.OpCounters(), precision="f32")
    worst = 0.0
    for p, got in out.entries:
        ref = fg.fir_gabor(img, p, fg.OracleConfig(3.0), precision="f64")
        scale = max(np.abs(ref.re).max(), np.abs(ref.im).max())
        worst = max(worst, max(np.abs(got.re - ref.re).max(), np.abs(got.im - ref.im).max()) / scale)
    assert worst <= 1e-5, worst


@pytest.mark.gpu
def test_config4_bins_vs_gpu_bruteforce(fg):
    """BASELINE config 4 (2048^2, 16x16, sigma 4) at full size: all 256 bins of the
    fused fp32 SDFT against the fp64 brute-force localized DFT on the GPU."""
    import torch

    from paper_1704_05231_b200.device import sdft_full

    f32 = np.random.default_rng(2).uniform(0.0, 1.0, size=(2048, 2048)).astype(np.float32)
    spec = fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0)
    bins = sdft_full(torch.from_numpy(f32).cuda(), spec)[0]
    img64 = torch.from_numpy(f32.astype(np.float64)).cuda()
    import ctypes as C

    from paper_1704_05231_b200 import _native as N
    from paper_1704_05231_b200.sdft import sdft_desc

    d, keep = sdft_desc(2048, 2048, spec, "f64")
    ref = torch.empty((2048, 2048), dtype=torch.complex128, device="cuda")
    worst = 0.0
    for u in range(16):
        for v in range(16):
            N.check(N.lib.fgb_localized_dft(C.byref(d), u, v, 3.0, C.c_void_p(img64.data_ptr()),
                                            C.c_void_p(ref.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
            got = bins[u * 16 + v].to(torch.complex128)
            scale = torch.maximum(ref.real.abs().max(), ref.imag.abs().max())
            err = torch.maximum((got.real - ref.real).abs().max(), (got.imag - ref.imag).abs().max()) / scale
            worst = max(worst, err.item())
    assert worst <= 1e-5, worst


def _bruteforce_worst(fg, img_t64, spec, out, entries, radius=3.0):
    """max over entries of max|got-ref|/max|ref| with the fp64 GPU brute force (on device)."""
    import ctypes as C

    import torch

    from paper_1704_05231_b200 import _native as N
    from paper_1704_05231_b200.gabor import _filter_desc

    H, W = img_t64.shape
    ref = torch.empty((H, W), dtype=torch.complex128, device="cuda")
    worst = 0.0
    for e, (i, k) in enumerate(entries):
        p = fg.GaborParams(spec.frequencies[i], k * math.pi / spec.orientations_n, spec.sigma_for(i))
        d = _filter_desc(H, W, p, fg.ExactFIR(radius), "f64")
        N.check(N.lib.fgb_fir_gabor(C.byref(d), radius, C.c_void_p(img_t64.data_ptr()), C.c_void_p(ref.data_ptr()),
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        got = out[e].to(torch.complex128)
        scale = torch.maximum(ref.real.abs().max(), ref.imag.abs().max())
        err = torch.maximum((got.real - ref.real).abs().max(), (got.imag - ref.imag).abs().max()) / scale
        worst = max(worst, err.item())
    return worst


@pytest.mark.gpu
def test_config3_images_vs_gpu_bruteforce(fg):
    """BASELINE config 3 (batched 64 x 1024^2, N=8 x 5 freqs, sigma up to 32): images
    0, 31, 63 of the batched fp32 run, all 40 entries each, vs fp64 brute force."""
    import sys

    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_1704_05231_b200.device import compute_bank

    cfg = bench.CONFIGS[3]
    imgs = np.stack([bench.make_image(cfg, i) for i in (0, 31, 63)])
    spec = fg.BankSpec(tuple(cfg["freqs"]), 8, tuple(cfg["sigmas"]))
    out = compute_bank(torch.from_numpy(imgs).cuda(), spec, fg.ExactFIR(3.0))
    ent = [(i, k) for i in range(5) for k in range(8)]
    worst = max(_bruteforce_worst(fg, torch.from_numpy(imgs[b].astype(np.float64)).cuda(), spec, out[b], ent)
                for b in range(3))
    assert worst <= 1e-5, worst


@pytest.mark.gpu
def test_config5_all_entries_vs_gpu_bruteforce(fg):
    """BASELINE config 5 (8192^2 + gratings, N=16 x 5 freqs, sigma up to 32): all 80
    entries of the fp32 bank, computed as LPT shards of 8 GPUs' unit lists (compact
    layouts), against the fp64 brute force on the GPU."""
    import sys

    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_1704_05231_b200 import parallel as P
    from paper_1704_05231_b200.device import compute_bank

    cfg = bench.CONFIGS[5]
    f = bench.make_image(cfg, 0)
    spec = fg.BankSpec(tuple(cfg["freqs"]), 16, tuple(cfg["sigmas"]))
    t32 = torch.from_numpy(f).cuda()
    t64 = torch.from_numpy(f.astype(np.float64)).cuda()

    worst = 0.0
    for units in P.partition_units(cfg["freqs"], cfg["sigmas"], 16, 8, 3.0):
        out = compute_bank(t32, spec, fg.ExactFIR(3.0), True, units)[0]
        worst = max(worst, _bruteforce_worst(fg, t64, spec, out, P.unit_entries(units, 16)))
        del out
        torch.cuda.empty_cache()
    assert worst <= 1e-5, worst


@pytest.mark.gpu
def test_gpu_ser_device_reduction(fg, golden):
    """SER (metrics.py:63-83) reduced on the device equals the reference's golden
    values and the host formula; sentinels +inf / -inf; deterministic."""
    import torch

    z, meta = golden
    f3 = z["f3"]
    a = torch.from_numpy(f3 * 1.0 - 1j * (f3 / 2)).cuda()                 # _ents[0][1] of make_golden.py
    b = torch.from_numpy((f3 * 1.01 + 0.3) + 1j * (-f3 / 2 + 0.01)).cuda()  # _b
    for part in ("real", "imag"):
        got = fg.ser(b, a, part)
        assert abs(got - meta["ser"][part]) <= 1e-9 * abs(meta["ser"][part]), (part, got)
        assert fg.ser(b, a, part) == got  # bit-identical rerun
    rng = np.random.default_rng(5)
    x = rng.normal(size=(333, 517)) + 1j * rng.normal(size=(333, 517))
    y = x + 1e-3 * (rng.normal(size=x.shape) + 1j * rng.normal(size=x.shape))
    hx, hy = fg.ComplexImage.from_planes(x.real, x.imag), fg.ComplexImage.from_planes(y.real, y.imag)
    for dt in (torch.complex128, torch.complex64):
        tx, ty = torch.from_numpy(x).to(dt).cuda(), torch.from_numpy(y).to(dt).cuda()
        hx2 = fg.ComplexImage.from_planes(tx.real.double().cpu().numpy(), tx.imag.double().cpu().numpy())
        hy2 = fg.ComplexImage.from_planes(ty.real.double().cpu().numpy(), ty.imag.double().cpu().numpy())
        for part in ("real", "imag"):
            assert abs(fg.ser(ty, tx, part) - fg.ser(hy2, hx2, part)) < 1e-9
    assert fg.ser(torch.from_numpy(x).cuda(), torch.from_numpy(x).cuda(), "real") == math.inf
    zero = torch.zeros((4, 4), dtype=torch.complex128, device="cuda")
    assert fg.ser(zero + 1, zero, "imag") == math.inf and fg.ser(zero + 1, zero, "real") == -math.inf
    with pytest.raises(ValueError):
        fg.ser(zero, zero, "both")
    with pytest.raises(ValueError):
        fg.ser(zero, torch.zeros((4, 5), dtype=torch.complex128, device="cuda"), "real")
    del hx, hy
