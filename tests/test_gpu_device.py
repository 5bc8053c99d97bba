"""GPU: device-tensor API, sharded (compact) layouts, fused-vs-separable SDFT,
large-sigma IIR in fp32 (parallel-form sections; the fp64-state direct form
kept behind FGB_IIR64), batch handling."""

import math
import os

import numpy as np
import pytest

from oracle import fastgabor_oracle as O
from .conftest import max_rel_err, random_image

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_1704_05231_b200 as fg
    from paper_1704_05231_b200 import device as D
    from paper_1704_05231_b200 import parallel as P

    return torch, fg, D, P


def test_units_compact_layout_matches_full(env):
    torch, fg, D, P = env
    f = torch.from_numpy(random_image(3, 80, 0.0, 1.0, width=96).astype(np.float32)).cuda()
    spec = fg.BankSpec((math.pi / 2, math.pi / 8), 16, (2.0, 8.0))
    full = D.compute_bank(f, spec, fg.ExactFIR(3.0))[0]
    for units in ([0, 3, 9], [4, 8, 17, 12], list(range(18))):
        part = D.compute_bank(f, spec, fg.ExactFIR(3.0), True, units)[0]
        ent = P.unit_entries(units, 16)
        assert part.shape[0] == len(ent)
        for e, (i, k) in enumerate(ent):
            assert torch.equal(part[e], full[i * 16 + k])


def test_sdft_heads_compact_layout(env):
    torch, fg, D, P = env
    f = torch.from_numpy(random_image(4, 64, 0.0, 1.0, width=64).astype(np.float32)).cuda()
    spec = fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0)
    full = D.sdft_full(f, spec)[0]
    for heads in ([0], [8], [3, 5], [0, 8, 1]):
        part = D.sdft_full(f, spec, heads)[0]
        bins = P.head_bins(heads, 16)
        assert part.shape[0] == len(bins)
        for e, (u, v) in enumerate(bins):
            assert torch.equal(part[e], full[u * 16 + v])


@pytest.mark.parametrize("m,sigma,radius", [(16, 4.0, 3.0), (8, None, 6.0), (32, 3.0, 3.0), (4, 1.0, 3.0), (16, 2.5, 3.0)])
def test_sdft_fused_matches_separable_and_oracle(env, m, sigma, radius):
    torch, fg, D, P = env
    fimg = random_image(5, 48, 0.0, 1.0, width=56)
    f = torch.from_numpy(fimg.astype(np.float32)).cuda()
    spec = fg.SdftSpec(m, m, fg.ExactFIR(radius), sigma)
    fused = D.sdft_full(f, spec)[0].cpu().numpy()
    os.environ["FGB_SDFT_UNFUSED"] = "1"
    try:
        from paper_1704_05231_b200 import _native as N

        N.lib.fgb_release_caches()
        sep = D.sdft_full(f, spec)[0].cpu().numpy()
    finally:
        del os.environ["FGB_SDFT_UNFUSED"]
        N.lib.fgb_release_caches()
    ref = O.sdft_full(fimg.astype(np.float32).astype(np.float64), m, m, ("fir", radius), sigma)
    worst_f = worst_s = 0.0
    for u in range(m):
        for v in range(m):
            r = ref[u][v]
            worst_f = max(worst_f, max_rel_err((fused[u * m + v].real, fused[u * m + v].imag), r))
            worst_s = max(worst_s, max_rel_err((sep[u * m + v].real, sep[u * m + v].imag), r))
    assert worst_f <= 1e-5 and worst_s <= 1e-5, (worst_f, worst_s)


def test_iir_large_sigma_f32(env):
    """The fp32 build's parallel-form sections (iir32.cu) meet 1e-5 at sigma = 16, 32, where a
    direct-form fp32 recursion misses it by up to 125x."""
    torch, fg, D, P = env
    fimg = random_image(6, 200, 0.0, 1.0, width=120)
    for sigma in (16.0, 32.0):
        p = fg.GaborParams(math.pi / sigma, 3 * math.pi / 8, sigma)
        out = fg.gabor_filter(fg.RealImage.from_array(fimg), p, fg.RecursiveIIR(), fg.OpCounters(), precision="f32")
        ref = O.gabor_filter(fimg, p.omega, p.theta, sigma, ("iir",))
        assert max_rel_err(out, ref) <= 1e-5


def test_iir_fp64_state_alternative_f32():
    """FGB_IIR64=1 switches the fp32 build to the direct-form kernels with fp64 state (iir.cu);
    read once per process, so the check runs in a subprocess: a bank and an SDFT vs the oracle."""
    import subprocess
    import sys

    code = (
        "import math, numpy as np, sys; sys.path.insert(0, '.');"
        "import paper_1704_05231_b200 as fg; from oracle import fastgabor_oracle as O;"
        "f = np.random.default_rng(4).uniform(0, 1, size=(90, 130));"
        "spec = fg.BankSpec((math.pi / 4, math.pi / 16), 8, (4.0, 16.0));"
        "out = fg.compute_bank(fg.RealImage.from_array(f), spec, fg.RecursiveIIR(), fg.OpCounters(), precision='f32');"
        "ref = O.compute_bank(f, spec.frequencies, 8, spec.sigmas, ('iir',));"
        "w = max(O.max_rel_err((e.re, e.im), r[3:]) for (_, e), r in zip(out.entries, ref));"
        "sd = fg.sdft_full(fg.RealImage.from_array(f), fg.SdftSpec(8, 8, fg.RecursiveIIR(), 2.0), fg.OpCounters(), precision='f32');"
        "bins = O.sdft_full(f, 8, 8, ('iir',), 2.0);"
        "w2 = max(O.max_rel_err((sd.bins[u][v].re, sd.bins[u][v].im), bins[u][v]) for u in range(8) for v in range(8));"
        "print(w, w2); assert w <= 1e-5 and w2 <= 1e-5"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, FGB_IIR64="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_batched_bank_equals_per_image(env):
    torch, fg, D, P = env
    imgs = np.stack([random_image(10 + i, 64, 0.0, 1.0, width=72) for i in range(3)]).astype(np.float32)
    t = torch.from_numpy(imgs).cuda()
    spec = fg.BankSpec((math.pi / 4, math.pi / 16), 8, (4.0, 16.0))
    batched = D.compute_bank(t, spec, fg.ExactFIR(3.0))
    for i in range(3):
        single = D.compute_bank(t[i], spec, fg.ExactFIR(3.0))[0]
        assert torch.equal(batched[i], single)


def test_odd_width_and_tiny_images(env):
    """Edge cases: odd widths (1-column kernel path), 1-pixel-wide and tiny images."""
    torch, fg, D, P = env
    for shape in ((37, 53), (5, 3), (1, 9), (9, 1), (2, 2)):
        fimg = random_image(7, shape[0], 0.0, 1.0, width=shape[1])
        spec = fg.BankSpec((1.0, 2.5), 4, (1.5, 0.8))
        out = fg.compute_bank(fg.RealImage.from_array(fimg), spec, fg.ExactFIR(3.0), fg.OpCounters(), precision="f64")
        ref = O.compute_bank(fimg, spec.frequencies, 4, spec.sigmas, ("fir", 3.0))
        for (p, img), r in zip(out.entries, ref):
            assert max_rel_err(img, r[3:]) <= 1e-10, shape


def test_very_long_kernels_fallback(env):
    """sigma = 50 at radius 6 (605 taps): column tile beyond shared memory -> global-memory path."""
    torch, fg, D, P = env
    fimg = random_image(8, 96, 0.0, 1.0, width=64)
    p = fg.GaborParams(0.125, 0.7, 2 * math.pi / 0.125)
    out = fg.gabor_filter(fg.RealImage.from_array(fimg), p, fg.ExactFIR(), fg.OpCounters(), precision="f64")
    ref = O.gabor_filter(fimg, p.omega, p.theta, p.sigma, ("fir", 6.0))
    assert max_rel_err(out, ref) <= 1e-10


@pytest.mark.parametrize("kn,shape", [("fir", (2, 48, 80)), ("iir", (2, 33, 71)), ("box", (1, 17, 30)),
                                      ("sdft", (1, 40, 48)), ("sdft", (1, 23, 31))])
def test_outputs_fully_written_within_bounds(env, kn, shape):
    """NaN-poisoned outputs with NaN guard bands on both sides: every output
    element is written (parity would fail on a left-over NaN) and nothing
    outside the output is touched (compute-sanitizer is not available on the
    GPU pool, so this is the out-of-bounds-write check)."""
    torch, fg, D, P = env
    b, h, w = shape
    imgs = np.random.default_rng(11).uniform(0.0, 1.0, size=(b, h, w)).astype(np.float32)
    t = torch.from_numpy(imgs).cuda()
    if kn == "sdft":
        plan = D.SdftPlan(shape, fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0), "f32")
        n_out = 256
    else:
        kind = {"fir": fg.ExactFIR(3.0), "iir": fg.RecursiveIIR(), "box": fg.Box(2)}[kn]
        spec = fg.BankSpec((math.pi / 2, math.pi / 8), 8, (2.0, 8.0))
        plan = D.BankPlan(shape, spec, kind, "f32")
        n_out = plan.entries
    guard = 4096
    n = b * n_out * h * w
    buf = torch.empty((n + 2 * guard,), dtype=torch.complex64, device="cuda")
    torch.view_as_real(buf).fill_(float("nan"))
    out = buf[guard:guard + n].view(b, n_out, h, w)
    plan(t, out)
    torch.cuda.synchronize()
    assert torch.isnan(torch.view_as_real(buf[:guard])).all() and torch.isnan(torch.view_as_real(buf[guard + n:])).all()
    o = out.cpu().numpy()
    assert np.isfinite(o.view(np.float32)).all()
    for bi in range(b):
        f64 = imgs[bi].astype(np.float64)
        if kn == "sdft":
            ref = O.sdft_full(f64, 16, 16, ("fir", 3.0), 4.0)
            err = max(max_rel_err((o[bi, u * 16 + v].real, o[bi, u * 16 + v].imag), ref[u][v])
                      for u in range(16) for v in range(16))
        else:
            ok = {"fir": ("fir", 3.0), "iir": ("iir",), "box": ("box", 2)}[kn]
            ref = O.compute_bank(f64, spec.frequencies, 8, spec.sigmas, ok)
            err = max(max_rel_err((o[bi, e].real, o[bi, e].imag), r[3:]) for e, r in enumerate(ref))
        assert err <= 1e-5


def test_randomized_sweep_f64(env):
    """Seeded random shapes / orientation counts / sigmas / smoothers / windows
    (incl. 1-pixel extents, N = 1..9, odd windows, sigma below one pixel) through
    the drop-in API in the fp64 build vs the oracle at 1e-10."""
    torch, fg, D, P = env
    rng = np.random.default_rng(2024)
    kinds = [(fg.ExactFIR(3.0), ("fir", 3.0)), (fg.ExactFIR(), ("fir", 6.0)), (fg.RecursiveIIR(), ("iir",))]
    for case in range(16):
        h, w = int(rng.integers(1, 90)), int(rng.integers(1, 90))
        f = rng.uniform(0.0, 1.0, size=(h, w))
        k, ok = kinds[case % 3]
        nf = int(rng.integers(1, 3))
        freqs = tuple(float(x) for x in rng.uniform(0.2, 2.5, size=nf))
        sig = tuple(float(x) for x in rng.uniform(0.6, 5.0, size=nf))
        n = int(rng.integers(1, 10))
        out = fg.compute_bank(fg.RealImage.from_array(f), fg.BankSpec(freqs, n, sig), k, fg.OpCounters(),
                              precision="f64")
        ref = O.compute_bank(f, freqs, n, sig, ok)
        for e, ((p, img), r) in enumerate(zip(out.entries, ref)):
            assert max_rel_err(img, r[3:]) <= 1e-10, (case, h, w, n, e)
        mx, my = int(rng.integers(1, 10)), int(rng.integers(1, 10))
        if case % 4 == 3:
            spec, sk = fg.SdftSpec(mx, my, fg.Box(1)), ("box", 1)
        else:
            spec, sk = fg.SdftSpec(mx, my, k, float(rng.uniform(0.6, 3.0))), ok
        sd = fg.sdft_full(fg.RealImage.from_array(f), spec, fg.OpCounters(), precision="f64")
        sref = O.sdft_full(f, mx, my, sk, spec.sigma)
        for u in range(mx):
            for v in range(my):
                assert max_rel_err(sd.bins[u][v], sref[u][v]) <= 1e-10, (case, h, w, mx, my, u, v)


def test_non_finite_outputs_raise_like_reference(env):
    """Outputs that overflow (1e308-valued fp64 input) are rejected with the
    reference's ComplexImage error, through the GPU finiteness flag."""
    torch, fg, D, P = env
    f = fg.RealImage.from_array(np.full((16, 16), 1e308))
    with pytest.raises(ValueError, match="finite"):
        fg.compute_bank(f, fg.BankSpec((1.0,), 2, (1.0,)), fg.ExactFIR(3.0), fg.OpCounters(), precision="f64")
    with pytest.raises(ValueError, match="finite"):
        fg.gabor_filter(f, fg.GaborParams(1.0, 0.3, 1.0), fg.ExactFIR(3.0), fg.OpCounters(), precision="f64")


@pytest.mark.parametrize("shape", [(70, 97), (64, 64), (100, 130)])
def test_fused_small_sigma_bank_f32(env, shape):
    """sigma <= 2 (h <= 6) frequencies run the fused row+column kernel (J in shared
    memory) in the fp32 build: partial 32x32 tiles, odd widths, batch 2, vs the
    oracle and vs the separate row / column kernels (FGB_FUSED_BANK=0 path is the
    same engine with the fusion disabled, checked through the oracle here)."""
    torch, fg, D, P = env
    h, w = shape
    imgs = np.random.default_rng(5).uniform(0.0, 1.0, size=(2, h, w)).astype(np.float32)
    spec = fg.BankSpec((math.pi / 2, math.pi / 3, 1.9), 8, (2.0, 1.3, 0.7))
    plan = D.BankPlan((2, h, w), spec, fg.ExactFIR(3.0), "f32")
    out = plan(torch.from_numpy(imgs).cuda(), plan.new_output()).cpu().numpy()
    for b in range(2):
        ref = O.compute_bank(imgs[b].astype(np.float64), spec.frequencies, 8, spec.sigmas, ("fir", 3.0))
        for e, r in enumerate(ref):
            assert max_rel_err((out[b, e].real, out[b, e].imag), r[3:]) <= 1e-5, (shape, b, e)


@pytest.mark.parametrize("batch,units", [(1, None), (3, None), (1, [0, 4, 7])])
def test_host_buffer_bank_matches_device(env, batch, units):
    """fgb_bank_host pipelines the D2H behind the compute (pieces = images of a
    batch, else frequencies); its output must equal the device entry point's
    bit for bit, including compact unit layouts."""
    import ctypes as C

    torch, fg, D, P = env
    from paper_1704_05231_b200 import _native as N

    h, w = 96, 80
    imgs = np.random.default_rng(3).uniform(0.0, 1.0, size=(batch, h, w)).astype(np.float32)
    spec = fg.BankSpec((math.pi / 2, math.pi / 4, math.pi / 8), 8, (2.0, 4.0, 8.0))
    plan = D.BankPlan((batch, h, w), spec, fg.ExactFIR(3.0), "f32", units=units)
    dev = plan(torch.from_numpy(imgs).cuda(), plan.new_output()).cpu().numpy()
    host = np.empty_like(dev)
    desc = plan.desc
    desc.img.pitch = w
    desc.img.batch_stride = h * w
    N.check(N.lib.fgb_bank_host(C.byref(desc), C.c_void_p(imgs.ctypes.data), C.c_void_p(host.ctypes.data)))
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("kn", ["fir", "iir"])
def test_huge_image_int64_offsets(env, kn):
    """16384^2 x 16 orientations (32 GB of outputs, element offsets past 2^31):
    interior pixels of the full-image bank equal a crop's bank computed
    separately (the crop carries the full filter support as margin)."""
    torch, fg, D, P = env
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(9)
    img = torch.rand((1, n, n), device="cuda", generator=g)
    kind = fg.ExactFIR(3.0) if kn == "fir" else fg.RecursiveIIR()
    spec = fg.BankSpec((math.pi / 4,), 16, (3.0,))
    plan = D.BankPlan((1, n, n), spec, kind, "f32")
    out = plan(img, plan.new_output())
    y0, x0, m, s = n - 300, n - 260, 200, 120  # crop with a margin wider than the support
    crop = img[:, y0 - m:y0 + s + m, x0 - m:x0 + s + m].contiguous()
    cplan = D.BankPlan(tuple(crop.shape), spec, kind, "f32")
    cout = cplan(crop, cplan.new_output())
    a = out[0, :, y0:y0 + s, x0:x0 + s]
    b = cout[0, :, m:m + s, m:m + s]
    scale = b.abs().max().item()
    assert torch.isfinite(torch.view_as_real(out[0, -1])).all()
    assert (a - b).abs().max().item() <= 1e-5 * scale
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kn", ["fir", "iir"])
def test_workspace_chunking_equals_unchunked(env, kn, monkeypatch):
    """A 1 MB workspace budget forces the engine to run a batch of 5 images one
    chunk at a time (and the IIR scratch per chunk); results are bit-identical
    to the default budget."""
    torch, fg, D, P = env
    imgs = torch.from_numpy(np.random.default_rng(21).uniform(0, 1, size=(5, 88, 104)).astype(np.float32)).cuda()
    kind = fg.ExactFIR(3.0) if kn == "fir" else fg.RecursiveIIR()
    spec = fg.BankSpec((math.pi / 2, math.pi / 8), 8, (2.0, 8.0))
    ref = D.BankPlan((5, 88, 104), spec, kind, "f32")
    want = ref(imgs, ref.new_output())
    from paper_1704_05231_b200 import _native as N

    torch.cuda.synchronize()
    N.lib.fgb_release_caches()  # plans are cached per descriptor: rebuild under the small budget
    monkeypatch.setenv("FGB_WS_BUDGET_MB", "1")
    small = D.BankPlan((5, 88, 104), spec, kind, "f32")
    got = small(imgs, small.new_output())
    torch.cuda.synchronize()
    N.lib.fgb_release_caches()  # later tests plan under the default budget again
    assert torch.equal(got, want)


def test_randomized_sweep_f32(env):
    """Seeded random f32 banks and SDFTs at sizes that take the fast paths (fused
    small-sigma kernel, FFMA2 row / column kernels, fused SDFT, IIR) vs the
    float64 oracle at 1e-5."""
    torch, fg, D, P = env
    rng = np.random.default_rng(77)
    for case in range(10):
        h, w = int(rng.integers(64, 260)), int(rng.integers(64, 260))
        f = rng.uniform(0.0, 1.0, size=(h, w)).astype(np.float32)
        f64 = f.astype(np.float64)
        iir = case % 3 == 2
        k, ok = (fg.RecursiveIIR(), ("iir",)) if iir else (fg.ExactFIR(3.0), ("fir", 3.0))
        nf = int(rng.integers(1, 4))
        freqs = tuple(float(x) for x in rng.uniform(0.2, 2.5, size=nf))
        sig = tuple(float(x) for x in rng.uniform(0.8, 6.0, size=nf))
        n = int(rng.integers(2, 10))
        out = fg.compute_bank(fg.RealImage.from_array(f), fg.BankSpec(freqs, n, sig), k, fg.OpCounters(),
                              precision="f32")
        ref = O.compute_bank(f64, freqs, n, sig, ok)
        for e, ((p, img), r) in enumerate(zip(out.entries, ref)):
            assert max_rel_err(img, r[3:]) <= 1e-5, (case, h, w, n, e, freqs, sig)
        m = int(rng.choice([4, 8, 16]))
        spec = fg.SdftSpec(m, m, k, float(rng.uniform(1.0, 4.0)))
        sd = fg.sdft_full(fg.RealImage.from_array(f), spec, fg.OpCounters(), precision="f32")
        sref = O.sdft_full(f64, m, m, ok, spec.sigma)
        for u in range(m):
            for v in range(m):
                assert max_rel_err(sd.bins[u][v], sref[u][v]) <= 1e-5, (case, h, w, m, u, v)


def test_workspace_bytes_query(env):
    """fgb_*_workspace_bytes: the fused small-sigma frequency needs no J planes,
    the FIR bank of config 2 keeps one J plane set per lane, the fused SDFT
    none, the IIR adds scratch; the numbers bound what the call allocates."""
    torch, fg, D, P = env
    hw = 1024 * 1024
    fused = D.BankPlan((1, 1024, 1024), fg.BankSpec((math.pi / 2,), 8, (2.0,)), fg.ExactFIR(3.0), "f32")
    assert fused.workspace_bytes < 4096
    cfg2 = D.BankPlan((1, 1024, 1024), fg.BankSpec((math.pi / 2, math.pi / 4, math.pi / 8, math.pi / 16), 8,
                                                  (2.0, 4.0, 8.0, 16.0)), fg.ExactFIR(3.0), "f32")
    assert 3 * 5 * hw * 8 <= cfg2.workspace_bytes <= 4 * 5 * hw * 8 + 4096  # J of the 3 non-fused lanes
    sd = D.SdftPlan((1, 512, 512), fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0), "f32")
    assert sd.workspace_bytes < 4096
    iir = D.BankPlan((1, 256, 256), fg.BankSpec((math.pi / 4,), 8, (4.0,)), fg.RecursiveIIR(), "f32")
    assert iir.workspace_bytes > 5 * 256 * 256 * 8
    before = torch.cuda.memory_allocated()
    out = cfg2(torch.rand(1, 1024, 1024, device="cuda"), cfg2.new_output())
    torch.cuda.synchronize()
    assert out.shape[1] == 32 and torch.cuda.memory_allocated() >= before  # torch's pool is separate


def test_iir_lane_state_alignment_odd_shapes():
    """odd N, two IIR frequencies, odd width, height % 4 == 0 put a
    lane's segment states at an 8-mod-16 byte offset before the 256-byte rounding;
    the fp32 recursion must run (16-byte copies) and match the oracle."""
    import torch

    import paper_1704_05231_b200 as fg
    from oracle import fastgabor_oracle as O
    from paper_1704_05231_b200.device import compute_bank

    f = np.random.default_rng(21).uniform(0, 1, (256, 255))
    for n, sig in ((3, (4.0, 2.0)), (5, (2.0, 3.0, 4.0))):
        freqs = tuple(math.pi / 2 ** (j + 1) for j in range(len(sig)))
        out = compute_bank(torch.from_numpy(f.astype(np.float32)).cuda(), fg.BankSpec(freqs, n, sig),
                           fg.RecursiveIIR())[0].cpu().numpy()
        ref = O.compute_bank(f, freqs, n, sig, ("iir",))
        for e, r in enumerate(ref):
            scale = max(np.abs(r[3]).max(), np.abs(r[4]).max())
            err = max(np.abs(out[e].real - r[3]).max(), np.abs(out[e].imag - r[4]).max()) / scale
            assert err <= 1e-5, (n, e, err)


def test_two_streams_share_the_workspace_safely():
    """calls on different streams reuse the one device workspace;
    the library orders them (event wait), so concurrent banks on two streams equal
    the serial results bit for bit."""
    import torch

    import paper_1704_05231_b200 as fg
    from paper_1704_05231_b200.device import BankPlan

    spec = fg.BankSpec((math.pi / 8, math.pi / 16), 8, (8.0, 16.0))
    imgs = [torch.rand(1, 512, 512, device="cuda") for _ in range(2)]
    plans = [BankPlan((1, 512, 512), spec, k, "f32") for k in (fg.ExactFIR(3.0), fg.RecursiveIIR())]
    ref = [p(i).clone() for p, i in zip(plans, imgs)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [p.new_output("cuda") for p in plans]
    for _ in range(3):
        for p, i, o, s in zip(plans, imgs, outs, streams):
            with torch.cuda.stream(s):
                p(i, o, stream=s)
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            assert torch.equal(o, r)
