"""GPU parity of the drop-in API against the reference's golden vectors and the
CPU oracle (fp64 build <= 1e-10, fp32 build <= 1e-5, max|err|/max|ref| as in
the reference conftest.py:33-36)."""

import math

import numpy as np
import pytest

from oracle import fastgabor_oracle as O
from .conftest import max_rel_err, random_image

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-5


@pytest.fixture(scope="module")
def fg():
    import paper_1704_05231_b200 as m

    return m


def kind_obj(fg, kn):
    return {"fir6": fg.ExactFIR(), "fir3": fg.ExactFIR(3.0), "iir": fg.RecursiveIIR(), "box1": fg.Box(1)}[kn]


def gold(z, name):
    return z[name + ".re"], z[name + ".im"]


def test_single_filters_golden_f64(fg, golden):
    z, meta = golden
    f1 = fg.RealImage.from_array(z["f1"])
    for kn in ("fir6", "fir3", "iir"):
        for i in range(6):
            key = f"gabor.{kn}.{i}"
            if key not in meta["cases"]:
                continue
            om, th, sg = meta["cases"][key]["params"]
            p = fg.GaborParams(om, th, sg)
            c = fg.OpCounters()
            h = fg.horizontal_stage(f1, p, kind_obj(fg, kn), c, precision="f64")
            assert max_rel_err(h.j, gold(z, f"hstage.{kn}.{i}")) <= TOL64, key
            out = fg.vertical_stage(h, c, precision="f64")
            assert max_rel_err(out, gold(z, key)) <= TOL64, key
            assert [c.multiplications, c.additions, c.smoothings_h, c.smoothings_v] == meta["cases"][key]["counters"]
            conj = fg.vertical_stage_conjugate(h, fg.OpCounters(), precision="f64")
            assert max_rel_err(conj, gold(z, f"vconj.{kn}.{i}")) <= TOL64, key
            full = fg.gabor_filter(f1, p, kind_obj(fg, kn), fg.OpCounters(), precision="f64")
            assert max_rel_err(full, gold(z, key)) <= TOL64, key


def test_banks_golden_f64(fg, golden):
    z, meta = golden
    f2 = fg.RealImage.from_array(z["f2"])
    for key, case in meta["cases"].items():
        if not key.startswith("bank."):
            continue
        _, kn, bn, tag = key.split(".")
        spec = fg.BankSpec(tuple(case["freqs"]), case["n"], None if case["sigmas"] is None else tuple(case["sigmas"]))
        fn = fg.compute_bank if tag == "reuse" else fg.compute_bank_noreuse
        c = fg.OpCounters()
        out = fn(f2, spec, kind_obj(fg, kn), c, precision="f64")
        assert [c.multiplications, c.additions, c.smoothings_h, c.smoothings_v] == case["counters"], key
        for e, (p, img) in enumerate(out.entries):
            assert [p.omega, p.theta, p.sigma] == case["entries"][e]
            assert max_rel_err(img, gold(z, f"{key}.{e}")) <= TOL64, (key, e)


def test_config1_golden_f64(fg, golden):
    """BASELINE config 1: 256x256 f64, omega=pi/4, N=4, sigma=4, FIR r=3, tol 1e-10."""
    z, _ = golden
    f = np.random.default_rng(0).uniform(0.0, 1.0, size=(256, 256))
    out = fg.compute_bank(fg.RealImage.from_array(f), fg.BankSpec((math.pi / 4,), 4, (4.0,)), fg.ExactFIR(3.0),
                          fg.OpCounters(), precision="f64")
    ref = O.compute_bank(f, (math.pi / 4,), 4, (4.0,), ("fir", 3.0))
    for e, (p, img) in enumerate(out.entries):
        assert max_rel_err(img, ref[e][3:]) <= TOL64
        for pi_, part in enumerate(("re", "im")):
            a = getattr(img, part)
            scale = max(np.abs(ref[e][3]).max(), np.abs(ref[e][4]).max())
            for sel, arr in (("sub", a[::5, ::5]), ("rows", a[[0, 1, 254, 255], :]), ("cols", a[:, [0, 1, 254, 255]])):
                assert np.max(np.abs(arr - z[f"cfg1.{e}.{part}.{sel}"])) <= TOL64 * scale


def test_sdft_golden_f64(fg, golden):
    z, meta = golden
    f3 = fg.RealImage.from_array(z["f3"])
    for key, case in meta["cases"].items():
        if not key.startswith("sdft."):
            continue
        _, kn, sn = key.split(".")
        spec = fg.SdftSpec(case["mx"], case["my"], kind_obj(fg, kn), case["sigma"])
        c = fg.OpCounters()
        out = fg.sdft_full(f3, spec, c, precision="f64")
        assert [c.multiplications, c.additions, c.smoothings_h, c.smoothings_v] == case["counters"], key
        for u in range(spec.mx):
            for v in range(spec.my):
                assert max_rel_err(out.bins[u][v], gold(z, f"{key}.{u}.{v}")) <= TOL64, (key, u, v)
        b = meta["cases"][f"sdftbin.{kn}.{sn}"]
        cb = fg.OpCounters()
        assert max_rel_err(fg.sdft_bin(f3, b["u"], b["v"], spec, cb, precision="f64"), gold(z, f"sdftbin.{kn}.{sn}")) <= TOL64
        assert [cb.multiplications, cb.additions, cb.smoothings_h, cb.smoothings_v] == b["counters"]
        h = meta["cases"][f"sdfth.{kn}.{sn}"]
        assert max_rel_err(fg.sdft_horizontal(f3, h["u"], spec, fg.OpCounters(), precision="f64"),
                           gold(z, f"sdfth.{kn}.{sn}")) <= TOL64


@pytest.mark.parametrize("kn", ["fir3", "fir6", "iir"])
def test_bank_f32_vs_oracle(fg, kn):
    f = random_image(5, 96, 0.0, 1.0, width=80)
    spec = fg.BankSpec((math.pi / 2, math.pi / 4, math.pi / 8), 8, (2.0, 4.0, 8.0))
    k = {"fir3": ("fir", 3.0), "fir6": ("fir", 6.0), "iir": ("iir",)}[kn]
    out = fg.compute_bank(fg.RealImage.from_array(f), spec, kind_obj(fg, kn), fg.OpCounters(), precision="f32")
    ref = O.compute_bank(f, spec.frequencies, 8, spec.sigmas, k)
    worst = max(max_rel_err(img, r[3:]) for (_, img), r in zip(out.entries, ref))
    assert worst <= TOL32, worst


@pytest.mark.parametrize("kn,m", [("fir3", 16), ("fir6", 8), ("iir", 8), ("box1", 8)])
def test_sdft_f32_vs_oracle(fg, kn, m):
    f = random_image(6, 64, 0.0, 1.0, width=72)
    kind = kind_obj(fg, kn)
    sigma = 4.0 if m == 16 else None
    spec = fg.SdftSpec(m, m, kind, sigma)
    k = {"fir3": ("fir", 3.0), "fir6": ("fir", 6.0), "iir": ("iir",), "box1": ("box", 1)}[kn]
    out = fg.sdft_full(fg.RealImage.from_array(f), spec, fg.OpCounters(), precision="f32")
    ref = O.sdft_full(f, m, m, k, sigma)
    worst = max(max_rel_err(out.bins[u][v], ref[u][v]) for u in range(m) for v in range(m))
    assert worst <= TOL32, worst


def test_config2_full_f32(fg):
    """BASELINE config 2 at full size: 1024^2 f32 (seed 1, 5x5 box blur), 8 orientations x 4 freqs, FIR r=3."""
    import scipy.ndimage as ndi

    f64 = np.random.default_rng(1).uniform(0.0, 1.0, size=(1024, 1024)).astype(np.float32).astype(np.float64)
    f32 = ndi.uniform_filter(f64, size=5, mode="nearest").astype(np.float32)
    freqs = (math.pi / 2, math.pi / 4, math.pi / 8, math.pi / 16)
    sig = (2.0, 4.0, 8.0, 16.0)
    out = fg.compute_bank(fg.RealImage.from_array(f32), fg.BankSpec(freqs, 8, sig), fg.ExactFIR(3.0),
                          fg.OpCounters(), precision="f32")
    # oracle on a subset of entries (theta_k and its mirror) at every frequency
    f = f32.astype(np.float64)
    worst = 0.0
    for i, (om, s) in enumerate(zip(freqs, sig)):
        for k in (0, 3, 4, 5):
            ref = O.gabor_filter(f, om, k * math.pi / 8, s, ("fir", 3.0))
            worst = max(worst, max_rel_err(out.entries[i * 8 + k][1], ref))
    assert worst <= TOL32, worst


def test_config2_full_iir_f32(fg):
    """Config 2's image and bank with RecursiveIIR (the reference CLI's default
    smoother) at full size, fp32 build (parallel-form sections) vs the oracle's
    float64 lfilter restatement: every frequency, a direct / mirror pair and the
    theta = pi/2 entry (the near-DC row pass, SURVEY App. B's worst case)."""
    import scipy.ndimage as ndi

    f64 = np.random.default_rng(1).uniform(0.0, 1.0, size=(1024, 1024)).astype(np.float32).astype(np.float64)
    f32 = ndi.uniform_filter(f64, size=5, mode="nearest").astype(np.float32)
    freqs = (math.pi / 2, math.pi / 4, math.pi / 8, math.pi / 16)
    sig = (2.0, 4.0, 8.0, 16.0)
    out = fg.compute_bank(fg.RealImage.from_array(f32), fg.BankSpec(freqs, 8, sig), fg.RecursiveIIR(),
                          fg.OpCounters(), precision="f32")
    f = f32.astype(np.float64)
    worst = 0.0
    for i, (om, s) in enumerate(zip(freqs, sig)):
        jr, ji = O.horizontal_stage(f, om, 3 * math.pi / 8, s, ("iir",))
        worst = max(worst, max_rel_err(out.entries[i * 8 + 3][1], O.vertical_stage(jr, ji, om, 3 * math.pi / 8, s, ("iir",))))
        worst = max(worst, max_rel_err(out.entries[i * 8 + 5][1],
                                       O.vertical_stage(jr, ji, om, 3 * math.pi / 8, s, ("iir",), conjugate=True)))
        worst = max(worst, max_rel_err(out.entries[i * 8 + 4][1], O.gabor_filter(f, om, math.pi / 2, s, ("iir",))))
    assert worst <= TOL32, worst


def test_iir_sigma32_full_size_f32(fg):
    """RecursiveIIR at sigma = 32 (config 3 / 5's widest filter) on a 1024^2 image, fp32 build:
    the parallel-form sections keep ~2.7x margin to 1e-5 (worst: theta = pi/2, the near-DC
    row stage; measured 1.6e-6 / 2.5e-6 / 3.7e-6 at theta = 0 / 3pi/8 / pi/2)."""
    f = np.random.default_rng(100).uniform(0.0, 1.0, size=(1024, 1024)).astype(np.float32).astype(np.float64)
    worst = 0.0
    for th in (0.0, 3 * math.pi / 8, math.pi / 2):
        p = fg.GaborParams(math.pi / 32, th, 32.0)
        out = fg.gabor_filter(fg.RealImage.from_array(f), p, fg.RecursiveIIR(), fg.OpCounters(), precision="f32")
        worst = max(worst, max_rel_err(out, O.gabor_filter(f, p.omega, p.theta, 32.0, ("iir",))))
    assert worst <= TOL32, worst


def test_config2_full_f64_validation_build(fg):
    """The fp64 validation build at config 2's full size: every frequency's
    direct / mirror pair and theta = pi/2 vs the float64 oracle at 1e-10."""
    import scipy.ndimage as ndi

    f64 = np.random.default_rng(1).uniform(0.0, 1.0, size=(1024, 1024)).astype(np.float32).astype(np.float64)
    f = ndi.uniform_filter(f64, size=5, mode="nearest").astype(np.float32).astype(np.float64)
    freqs = (math.pi / 2, math.pi / 4, math.pi / 8, math.pi / 16)
    sig = (2.0, 4.0, 8.0, 16.0)
    out = fg.compute_bank(fg.RealImage.from_array(f), fg.BankSpec(freqs, 8, sig), fg.ExactFIR(3.0),
                          fg.OpCounters(), precision="f64")
    worst = 0.0
    for i, (om, s) in enumerate(zip(freqs, sig)):
        jr, ji = O.horizontal_stage(f, om, 3 * math.pi / 8, s, ("fir", 3.0))
        worst = max(worst, max_rel_err(out.entries[i * 8 + 3][1], O.vertical_stage(jr, ji, om, 3 * math.pi / 8, s,
                                                                                   ("fir", 3.0))))
        worst = max(worst, max_rel_err(out.entries[i * 8 + 5][1], O.vertical_stage(jr, ji, om, 3 * math.pi / 8, s,
                                                                                   ("fir", 3.0), conjugate=True)))
        worst = max(worst, max_rel_err(out.entries[i * 8 + 4][1], O.gabor_filter(f, om, math.pi / 2, s, ("fir", 3.0))))
    assert worst <= TOL64, worst
