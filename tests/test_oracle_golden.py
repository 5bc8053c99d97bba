"""Pin the CPU oracle (oracle/fastgabor_oracle.py) to golden vectors produced
by the reference itself (tests/golden/make_golden.py)."""

import math

import numpy as np
import pytest

from oracle import fastgabor_oracle as O
from .conftest import max_rel_err

KINDS = {"fir6": ("fir", 6.0), "fir3": ("fir", 3.0), "iir": ("iir",), "box1": ("box", 1)}


def g(z, name):
    return z[name + ".re"], z[name + ".im"]


def test_iir_coefficient_kats(golden):
    _, meta = golden
    for s, ref in meta["coeffs"].items():
        got = O.iir_coeffs(float(s))
        assert np.allclose(got, ref, rtol=0, atol=1e-15), s


def test_sampled_gaussian(golden):
    z, meta = golden
    for key, h in meta["gauss"].items():
        a, b, c, d = key.split(".")
        k, hh = O.sampled_gaussian(float(a + "." + b), float(c + "." + d))
        assert hh == h
        assert np.max(np.abs(k - z[f"gauss.{key}"])) <= 1e-16


def test_smooth_1d(golden):
    z, _ = golden
    sig = z["smooth.in"]
    for name, k in list(KINDS.items())[:3] + [("box2", ("box", 2))]:
        for s in (0.8, 2.0, 5.0):
            ref = z[f"smooth.{name}.{s}"]
            assert np.max(np.abs(O.smooth_1d(sig, k, s) - ref)) <= 1e-13 * max(1.0, np.abs(ref).max())


def test_single_filters(golden):
    z, meta = golden
    f1 = z["f1"]
    for kn in ("fir6", "fir3", "iir"):
        for i in range(6):
            key = f"gabor.{kn}.{i}"
            if key not in meta["cases"]:
                continue
            om, th, sg = meta["cases"][key]["params"]
            k = KINDS[kn]
            jr, ji = O.horizontal_stage(f1, om, th, sg, k)
            assert max_rel_err((jr, ji), g(z, f"hstage.{kn}.{i}")) <= 1e-13
            assert max_rel_err(O.vertical_stage(jr, ji, om, th, sg, k), g(z, key)) <= 1e-13
            assert max_rel_err(O.vertical_stage(jr, ji, om, th, sg, k, conjugate=True), g(z, f"vconj.{kn}.{i}")) <= 1e-13


def test_banks(golden):
    z, meta = golden
    f2 = z["f2"]
    for key, case in meta["cases"].items():
        if not key.startswith("bank."):
            continue
        _, kn, bn, tag = key.split(".")
        fn = O.compute_bank if tag == "reuse" else O.compute_bank_noreuse
        out = fn(f2, case["freqs"], case["n"], case["sigmas"], KINDS[kn])
        assert len(out) == len(case["entries"])
        for e, (ent, params) in enumerate(zip(out, case["entries"])):
            assert list(ent[:3]) == pytest.approx(params, abs=0, rel=0)
            assert max_rel_err(ent[3:], g(z, f"{key}.{e}")) <= 1e-12


def test_config1_golden(golden):
    z, _ = golden
    f = np.random.default_rng(0).uniform(0.0, 1.0, size=(256, 256))
    out = O.compute_bank(f, (math.pi / 4,), 4, (4.0,), ("fir", 3.0))
    for e, ent in enumerate(out):
        for pi, part in enumerate(("re", "im")):
            a = ent[3 + pi]
            for sel, arr in (("sub", a[::5, ::5]), ("rows", a[[0, 1, 254, 255], :]), ("cols", a[:, [0, 1, 254, 255]])):
                ref = z[f"cfg1.{e}.{part}.{sel}"]
                assert np.max(np.abs(arr - ref)) <= 1e-13


def test_sdft(golden):
    z, meta = golden
    f3 = z["f3"]
    for key, case in meta["cases"].items():
        if not key.startswith("sdft."):
            continue
        _, kn, sn = key.split(".")
        mx, my, sg = case["mx"], case["my"], case["sigma"]
        bins = O.sdft_full(f3, mx, my, KINDS[kn], sg)
        for u in range(mx):
            for v in range(my):
                assert max_rel_err(bins[u][v], g(z, f"{key}.{u}.{v}")) <= 1e-12, (key, u, v)
        b = meta["cases"][f"sdftbin.{kn}.{sn}"]
        assert max_rel_err(O.sdft_bin(f3, b["u"], b["v"], mx, my, KINDS[kn], sg), g(z, f"sdftbin.{kn}.{sn}")) <= 1e-12
        h = meta["cases"][f"sdfth.{kn}.{sn}"]
        assert max_rel_err(O.sdft_horizontal(f3, h["u"], mx, my, KINDS[kn], sg), g(z, f"sdfth.{kn}.{sn}")) <= 1e-12


def test_bruteforce_oracles(golden):
    z, meta = golden
    f1, f3 = z["f1"], z["f3"]
    for i in range(3):
        om, th, sg = meta["cases"][f"gabor.fir6.{i}"]["params"]
        assert max_rel_err(O.fir_gabor(f1, om, th, sg), g(z, f"firgabor.{i}")) <= 1e-14
    for kn in ("fir6", "box1"):
        assert max_rel_err(O.localized_dft(f3, 1, 3, 4, 4, KINDS[kn]), g(z, f"ldft.{kn}")) <= 1e-14
    # radius 3, supports larger than the image (sigma 16 / 32)
    f7 = z["f7"]
    for i in range(2):
        om, th, sg = meta["cases"][f"firgabor_r3.{i}"]["params"]
        assert max_rel_err(O.fir_gabor(f7, om, th, sg, radius=3.0), g(z, f"firgabor_r3.{i}")) <= 1e-13
    assert max_rel_err(O.localized_dft(f7, 5, 27, 32, 32, ("fir", 3.0), 16.0, radius=3.0), g(z, "ldft_r3")) <= 1e-13
