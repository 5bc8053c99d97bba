"""GPU parity of the 1-D smoothing entry points smooth_lines / smooth_1d /
smooth_pair_1d (gaussian.py:245-302) through fgb_smooth_lines(_host):
reference goldens (tests/golden, made by the reference itself) and the CPU
oracle (oracle.smooth_lines); fp64 <= 1e-10, fp32 <= 1e-5 of max|ref|."""

import math

import numpy as np
import pytest

from oracle import fastgabor_oracle as O

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-5


@pytest.fixture(scope="module")
def fg():
    import paper_1704_05231_b200 as m

    return m


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.abs(b).max(), 1e-300))


def kinds(fg):
    return {"fir6": (fg.ExactFIR(), ("fir", 6.0)), "fir3": (fg.ExactFIR(3.0), ("fir", 3.0)),
            "iir": (fg.RecursiveIIR(), ("iir",)), "box2": (fg.Box(2), ("box", 2)), "box1": (fg.Box(1), ("box", 1))}


def ref_charge(kind, sigma, lines, nominal):
    """gaussian.py:263-284 counter charges."""
    if kind[0] == "iir":
        return 6 * lines * nominal, 6 * lines * nominal
    if kind[0] == "fir":
        t = 2 * max(1, math.ceil(kind[1] * sigma)) + 1
        return t * lines * nominal, (t - 1) * lines * nominal
    if kind[0] == "box":
        return 0, 2 * kind[1] * lines * nominal
    return 0, (kind[2] - kind[1]) * lines * nominal


def test_smooth_1d_goldens(fg, golden):
    z, _ = golden
    sig = z["smooth.in"]
    for name in ("fir6", "fir3", "iir", "box2"):
        k, _ = kinds(fg)[name]
        for s in (0.8, 2.0, 5.0):
            ref = z[f"smooth.{name}.{s}"]
            c = fg.OpCounters()
            got = fg.smooth_1d(sig, k, s, c, precision="f64")
            assert got.dtype == np.float64 and got.shape == ref.shape
            assert rel(got, ref) <= TOL64, (name, s)
            assert rel(fg.smooth_1d(sig, k, s, fg.OpCounters(), precision="f32"), ref) <= TOL32, (name, s)
            m, a = ref_charge(kinds(fg)[name][1], s, 1, sig.size)
            assert (c.multiplications, c.additions, c.smoothings_h, c.smoothings_v) == (m, a, 1, 0)


def test_smooth_lines_vs_oracle(fg):
    rng = np.random.default_rng(11)
    for rows, n in ((1, 1), (3, 2), (17, 300), (40, 1031), (5, 8192)):
        x = rng.uniform(0, 255, size=(rows, n))
        for name, (k, ok) in kinds(fg).items():
            for s in (0.6, 3.0, 32.0):
                if ok[0] == "iir" and s < 0.5:
                    continue
                ref = O.smooth_lines(x, ok, s)
                for prec, tol in (("f64", TOL64), ("f32", TOL32)):
                    got = fg.smooth_lines(x, k, s, fg.OpCounters(), precision=prec)
                    assert rel(got, ref) <= tol, (rows, n, name, s, prec)


def test_smooth_lines_asym_box_and_assume_padded(fg):
    from paper_1704_05231_b200.gaussian import _AsymBox

    rng = np.random.default_rng(12)
    x = rng.normal(size=(9, 257))
    for lo, hi in ((-8, 7), (-3, -1), (0, 0), (2, 9)):
        c = fg.OpCounters()
        got = fg.smooth_lines(x, _AsymBox(lo, hi), 1.0, c, direction="v", precision="f64")
        assert rel(got, O.smooth_lines(x, ("abox", lo, hi), 1.0)) <= TOL64
        assert (c.additions, c.smoothings_v, c.smoothings_h) == ((hi - lo) * x.size, 9, 0)
    for s in (2.0, 16.0):
        c = fg.OpCounters()
        got = fg.smooth_lines(x, fg.RecursiveIIR(), s, c, nominal_len=100, assume_padded=True, precision="f64")
        assert rel(got, O.smooth_lines(x, ("iir",), s, assume_padded=True)) <= TOL64
        assert c.multiplications == 6 * 9 * 100  # nominal_len overrides the charged length


def test_smooth_pair_and_errors(fg):
    rng = np.random.default_rng(13)
    a, b = rng.normal(size=77), rng.normal(size=77)
    c = fg.OpCounters()
    ga, gb = fg.smooth_pair_1d(a, b, fg.ExactFIR(3.0), 2.0, c, precision="f64")
    assert rel(ga, O.smooth_1d(a, ("fir", 3.0), 2.0)) <= TOL64
    assert rel(gb, O.smooth_1d(b, ("fir", 3.0), 2.0)) <= TOL64
    assert c.smoothings_h == 2
    with pytest.raises(ValueError, match="ExactFIR"):
        fg.smooth_1d(a, fg.RecursiveIIR(), 0.3, fg.OpCounters())
    with pytest.raises(ValueError):
        fg.smooth_1d(np.zeros((2, 2)), fg.ExactFIR(3.0), 2.0, fg.OpCounters())
    with pytest.raises(TypeError):
        fg.smooth_1d(a, object(), 2.0, fg.OpCounters())


def test_device_entry_with_pitch(fg):
    import ctypes as C

    import torch

    from paper_1704_05231_b200 import _native as N
    from paper_1704_05231_b200.gaussian import _lines_desc

    rng = np.random.default_rng(14)
    x = rng.uniform(0, 1, size=(33, 500))
    dev = torch.zeros((33, 512), dtype=torch.float64, device="cuda")
    dev[:, :500] = torch.from_numpy(x).cuda()
    for k, ok, s in ((fg.ExactFIR(3.0), ("fir", 3.0), 4.0), (fg.RecursiveIIR(), ("iir",), 8.0), (fg.Box(3), ("box", 3), 1.0)):
        d = _lines_desc(33, 500, k, s, "f64", False)
        d.pitch = 512
        out = torch.empty((33, 500), dtype=torch.float64, device="cuda")
        N.check(N.lib.fgb_smooth_lines(C.byref(d), C.c_void_p(dev.data_ptr()), C.c_void_p(out.data_ptr()),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), O.smooth_lines(x, ok, s)) <= TOL64


def test_criterion_8_reproduces_reference_values(fg):
    """Acceptance criterion 8 (test_acceptance.py:278-311) is red in the reference
    itself (impulse err 7.113e-03 at sigma=1.0, pkg/test_output.txt:204); the
    drop-in must reproduce the same numbers, not 'fix' them."""
    worst, at = 0.0, None
    for sigma in (1.0, 1.5, 2.0, 3.0, 4.0, 6.0, 8.0, 10.0):
        kernel, half = fg.sampled_gaussian(sigma)
        n = 4 * half + 1
        imp = np.zeros(n)
        imp[n // 2] = 1.0
        resp = fg.smooth_1d(imp, fg.RecursiveIIR(), sigma, fg.OpCounters(), precision="f64")
        assert rel(resp, O.smooth_1d(imp, ("iir",), sigma)) <= TOL64
        exp = np.zeros(n)
        exp[n // 2 - half: n // 2 + half + 1] = kernel
        err = float(np.abs(resp - exp).max())
        if err > worst:
            worst, at = err, sigma
    assert at == 1.0 and abs(worst - 7.113e-3) < 5e-7, (worst, at)
    dc = fg.smooth_1d(np.ones(256), fg.RecursiveIIR(), 3.0, fg.OpCounters(), precision="f64")
    assert float(np.abs(dc - 1.0).max()) <= 1e-6
