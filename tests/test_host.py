"""CPU-only checks of the host side: the C ABI library loads and exports every
symbol include/fgb200.h declares; host coefficient math and the analytic
OpCounters match the reference's golden values; parameter validation raises
the reference's exception types/messages.  No GPU work is launched here."""

import math
import os
import re

import numpy as np
import pytest

from oracle import fastgabor_oracle as O
from .conftest import ROOT


@pytest.fixture(scope="module")
def fg():
    import paper_1704_05231_b200 as m

    return m


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fgb200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fgb_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol(fg):
    from paper_1704_05231_b200 import _native as N

    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(N.lib, s), s
    assert set(syms) <= set(N.EXPORTED), set(syms) - set(N.EXPORTED)
    assert N.lib.fgb_version() >= 10000


def test_abi_struct_layouts_match_header():
    """ctypes mirrors of the descriptors have the C layout (sizes/offsets)."""
    import ctypes as C

    from paper_1704_05231_b200 import _native as N

    assert C.sizeof(N.fgb_smoother) == 16
    assert C.sizeof(N.fgb_image) == 32
    assert N.fgb_bank_desc.omegas.offset == 40
    assert N.fgb_filter_desc.smoother.offset == 56
    assert N.fgb_sdft_desc.u_heads.offset == 64


def test_iir_coefficients_match_golden(fg, golden):
    _, meta = golden
    for s, ref in meta["coeffs"].items():
        c = fg.make_coeffs(float(s))
        got = [c.B, -c.b1, -c.b2, -c.b3]
        assert np.allclose(got, ref, rtol=0, atol=2e-16), s
        assert c.b0 == 1.0
        assert c.B == pytest.approx(float(c.denominator().sum()), abs=1e-15)


def test_iir_parallel_form_sections(fg):
    """fgb_iir_sections (what the fp32 IIR kernels run, csrc/iir32.cu) against NumPy's roots
    and residues of the reference coefficients, the unit DC gain, and the impulse response of
    the direct form (gaussian.py:215-228 restated by the oracle)."""
    import ctypes as C

    from paper_1704_05231_b200 import _native as N

    for sigma in (0.6, 2.0, 4.3, 16.0, 32.0, 50.0):
        out = (C.c_double * 6)()
        assert N.lib.fgb_iir_sections(sigma, out) == 0
        qr, qc, cr, cc = out[0], complex(out[1], out[2]), out[3], complex(out[4], out[5])
        B, a1, a2, a3 = O.iir_coeffs(sigma)
        roots = np.roots([1.0, a1, a2, a3])
        assert min(abs(roots - qr)) < 1e-12 and min(abs(roots - qc)) < 1e-12 and qc.imag > 0
        assert abs(cr / (1 - qr) + 2 * (cc / (1 - qc)).real - 1.0) < 1e-10  # unit DC gain (B = sum a)
        n = np.arange(200)
        h_sec = cr * qr ** n + 2 * (cc * qc ** n).real
        x = np.zeros(200)
        x[0] = 1.0
        y, p1, p2, p3 = np.empty(200), 0.0, 0.0, 0.0
        for i in range(200):
            y[i] = B * x[i] - a1 * p1 - a2 * p2 - a3 * p3
            p3, p2, p1 = p2, p1, y[i]
        assert np.max(abs(h_sec - y)) < 1e-12 * max(1.0, sigma)
    with pytest.raises(Exception):
        fg.make_coeffs(0.25)
    assert N.lib.fgb_iir_sections(0.25, (C.c_double * 6)()) != 0  # same validation as fgb_iir_coeffs


def test_sampled_gaussian_matches_golden(fg, golden):
    z, meta = golden
    for key, h in meta["gauss"].items():
        a, b, c, d = key.split(".")
        k, hh = fg.sampled_gaussian(float(a + "." + b), float(c + "." + d))
        assert hh == h
        # same pairwise summation as numpy; exp() may differ from numpy's SIMD exp by an ulp
        assert np.allclose(k, z[f"gauss.{key}"], rtol=1e-15, atol=0.0)
        assert k.sum() == pytest.approx(1.0, abs=1e-15)


def test_pad_radius(fg):
    # gaussian.py:198-212 and the reference test test_gaussian.py:154-157
    assert fg.pad_radius(fg.ExactFIR(), 1.5) == 9
    assert fg.pad_radius(fg.RecursiveIIR(), 2.0) == 12
    assert fg.pad_radius(fg.Box(half_width=2), 2.0) == 0
    assert fg.pad_radius(fg.ExactFIR(3.0), 32.0) == 96
    from paper_1704_05231_b200 import _native as N

    for kind, s in ((fg.ExactFIR(3.0), 4.0), (fg.RecursiveIIR(), 7.3), (fg.Box(3), 1.0)):
        from paper_1704_05231_b200.gaussian import native_smoother

        sm = native_smoother(kind)
        assert N.lib.fgb_pad_radius(sm, s) == fg.pad_radius(kind, s)


def _kind(fg, kn):
    return {"fir6": fg.ExactFIR(), "fir3": fg.ExactFIR(3.0), "iir": fg.RecursiveIIR(), "box1": fg.Box(1)}[kn]


def test_counters_match_reference_golden(fg, golden):
    """Analytic OpCounters == the reference's instrumented counters (metrics.py:13-42)."""
    from paper_1704_05231_b200.bank import _charge_bank
    from paper_1704_05231_b200.metrics import charge_gabor_col, charge_gabor_row
    from paper_1704_05231_b200.sdft import _charge_full, _charge_h, _charge_v

    _, meta = golden
    n_checked = 0
    for key, case in meta["cases"].items():
        c = fg.OpCounters()
        if key.startswith("gabor."):
            _, kn, _ = key.split(".")
            om, th, sg = case["params"]
            charge_gabor_row(c, _kind(fg, kn), sg, 32, 40)
            charge_gabor_col(c, _kind(fg, kn), sg, 32, 40)
        elif key.startswith("bank."):
            _, kn, bn, tag = key.split(".")
            spec = fg.BankSpec(tuple(case["freqs"]), case["n"],
                               None if case["sigmas"] is None else tuple(case["sigmas"]))
            _charge_bank(c, spec, _kind(fg, kn), 16, 20, tag == "reuse")
        elif key == "cfg1":
            _charge_bank(c, fg.BankSpec((math.pi / 4,), 4, (4.0,)), fg.ExactFIR(3.0), 256, 256, True)
        elif key.startswith("sdft."):
            _, kn, sn = key.split(".")
            spec = fg.SdftSpec(case["mx"], case["my"], _kind(fg, kn), case["sigma"])
            _charge_full(c, spec, 10, 12)
        elif key.startswith("sdftbin."):
            _, kn, sn = key.split(".")
            base = meta["cases"]["sdft." + kn + "." + sn]
            spec = fg.SdftSpec(base["mx"], base["my"], _kind(fg, kn), base["sigma"])
            _charge_h(c, spec, 10, 12)
            _charge_v(c, spec, 10, 12)
        elif key.startswith("sdfth."):
            _, kn, sn = key.split(".")
            base = meta["cases"]["sdft." + kn + "." + sn]
            spec = fg.SdftSpec(base["mx"], base["my"], _kind(fg, kn), base["sigma"])
            _charge_h(c, spec, 10, 12)
        else:
            continue
        assert [c.multiplications, c.additions, c.smoothings_h, c.smoothings_v] == case["counters"], key
        n_checked += 1
    assert n_checked > 40


def test_bank_counter_laws(fg):
    """Smoothing-count law of test_bank.py:134-146 and the IIR 38 M / 30 A per pixel of test_gabor.py:138-148."""
    from paper_1704_05231_b200.bank import _charge_bank
    from paper_1704_05231_b200.metrics import charge_gabor_col, charge_gabor_row

    h = w = 32
    for n in (2, 3, 8, 9):
        spec = fg.BankSpec((3.0,), n)
        c = fg.OpCounters()
        _charge_bank(c, spec, fg.RecursiveIIR(), h, w, True)
        assert c.smoothings_h == 2 * h * (n // 2 + 1)
        assert c.smoothings_v == 2 * w * n
        c2 = fg.OpCounters()
        _charge_bank(c2, spec, fg.RecursiveIIR(), h, w, False)
        assert c2.smoothings_h == 2 * h * n
    c = fg.OpCounters()
    charge_gabor_row(c, fg.RecursiveIIR(), 1.0, 16, 16)
    charge_gabor_col(c, fg.RecursiveIIR(), 1.0, 16, 16)
    assert (c.multiplications, c.additions) == (38 * 256, 30 * 256)


def test_validation_matches_reference(fg):
    with pytest.raises(ValueError):
        fg.BankSpec(frequencies=(), orientations_n=4)
    with pytest.raises(ValueError):
        fg.BankSpec(frequencies=(1.0,), orientations_n=0)
    with pytest.raises(ValueError):
        fg.BankSpec(frequencies=(1.0, 2.0), orientations_n=4, sigmas=(1.0,))
    with pytest.raises(ValueError):
        fg.GaborParams(0.0, 0.0, 1.0)
    with pytest.raises(ValueError):
        fg.GaborParams(1.0, 0.0, -1.0)
    p = fg.GaborParams(1.0, math.pi + 0.3, 2.0)
    assert p.theta == pytest.approx(0.3)
    with pytest.raises(ValueError):
        fg.ExactFIR(radius=2.0)
    with pytest.raises(ValueError):
        fg.Box(half_width=-1)
    with pytest.raises(ValueError):
        fg.SdftSpec(mx=0, my=4, smoother=fg.ExactFIR())
    with pytest.raises(ValueError):
        fg.SdftSpec(mx=4, my=4, smoother=fg.ExactFIR(), sigma=-1.0)
    with pytest.raises(ValueError):
        fg.make_coeffs(0.0)
    with pytest.raises(ValueError, match="ExactFIR"):
        fg.make_coeffs(0.25)
    spec = fg.BankSpec(frequencies=(0.5, 2.0), orientations_n=4)
    assert spec.sigma_for(0) == pytest.approx(4.0 * math.pi)
    assert spec.thetas() == pytest.approx([0.0, math.pi / 4, math.pi / 2, 3 * math.pi / 4])
    s = fg.SdftSpec(mx=8, my=8, smoother=fg.ExactFIR())
    assert s.sigma_value == pytest.approx(4 / 3)
    assert s.omega0x == pytest.approx(math.pi / 4)


def test_images_and_conjugate(fg):
    img = fg.ComplexImage(1, 1, np.array([[1.0]]), np.array([[2.0]]))
    conj = fg.conjugate_image(img)
    assert conj.re[0, 0] == 1.0 and conj.im[0, 0] == -2.0
    with pytest.raises(ValueError):
        fg.RealImage.from_array(np.array([[np.nan]]))
    with pytest.raises(ValueError):
        fg.RealImage.from_array(np.zeros(3))
    for empty in (np.zeros((0, 5)), np.zeros((5, 0))):  # image_io.py:33,59
        with pytest.raises(ValueError, match="at least 1x1"):
            fg.RealImage.from_array(empty)


def test_complex_image_from_planar(fg):
    """*_host_planar results: GPU-checked planes become views without a copy;
    unchecked (non-finite) ones go through the reference constructor's check."""
    planes = np.arange(24, dtype=np.float64).reshape(2, 3, 4)
    img = fg.ComplexImage.from_planar(planes, True)
    assert (img.width, img.height) == (4, 3) and np.shares_memory(img.re, planes)
    assert np.array_equal(img.im, planes[1])
    bad = planes.copy()
    bad[1, 0, 0] = np.inf
    with pytest.raises(ValueError, match="finite"):
        fg.ComplexImage.from_planar(bad, False)


def test_entry_and_bin_counts(fg):
    """Output sizing of sharded calls (compact layouts) computed by the library."""
    import ctypes as C

    from paper_1704_05231_b200 import _native as N
    from paper_1704_05231_b200.bank import bank_desc
    from paper_1704_05231_b200.sdft import sdft_desc

    spec = fg.BankSpec((1.0, 2.0), 8, (2.0, 3.0))
    d, keep = bank_desc(16, 16, spec, fg.ExactFIR(3.0), "f32", True)
    assert N.lib.fgb_bank_entries(C.byref(d)) == 16
    d, keep = bank_desc(16, 16, spec, fg.ExactFIR(3.0), "f32", True, units=[0, 4, 5])
    # unit 0: k=0 (no mirror); unit 4: k=4 (no mirror); unit 5: i=1,k=0
    assert N.lib.fgb_bank_entries(C.byref(d)) == 3
    d, keep = bank_desc(16, 16, spec, fg.ExactFIR(3.0), "f32", True, units=[1, 2])
    assert N.lib.fgb_bank_entries(C.byref(d)) == 4
    sp = fg.SdftSpec(16, 16, fg.ExactFIR(3.0), 4.0)
    d, keep = sdft_desc(16, 16, sp, "f32")
    assert N.lib.fgb_sdft_bins(C.byref(d)) == 256
    d, keep = sdft_desc(16, 16, sp, "f32", heads=[0, 8])
    assert N.lib.fgb_sdft_bins(C.byref(d)) == 32
    d, keep = sdft_desc(16, 16, sp, "f32", heads=[3])
    assert N.lib.fgb_sdft_bins(C.byref(d)) == 32


def test_oracle_matches_reference_closed_forms():
    """The oracle itself satisfies the reference's closed forms (test_gabor.py:93-107)."""
    data = np.zeros((33, 33))
    data[16, 16] = 1.0
    om, th, sg = 2.5, 1.1, 1.3
    re, im = O.gabor_filter(data, om, th, sg, ("fir", 6.0))
    k, h = O.sampled_gaussian(sg)
    env = np.zeros(33)
    env[16 - h : 16 + h + 1] = k
    x = np.arange(33.0) - 16
    exp = np.outer(env, env) * np.exp(1j * om * (math.cos(th) * x[None, :] + math.sin(th) * x[:, None]))
    assert np.max(np.abs(re - exp.real)) <= 1e-10
    assert np.max(np.abs(im - exp.imag)) <= 1e-10
