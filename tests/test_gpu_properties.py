"""Size-independent properties of the full-size BASELINE workloads on the GPU
(fp32 build), complementing the oracle comparisons of test_gpu_fullsize.py:

* linearity of the bank (config 5, 8192^2): bank(f + 2 g) = bank(f) + 2 bank(g);
* conjugate symmetry of the localized DFT (config 4, 2048^2):
  F(M-u, M-v) = conj F(u, v), bit-exact for the bins sdft.py:209-212 fills
  that way (v > M/2), to rounding for pairs that are both computed;
* batch independence (config 3): a batched call equals per-image calls bit for bit;
* a constant image gives a constant response equal to the reference's DC gain of
  the filter (replicate padding keeps the constant up to the borders).
Tolerance for the float identities: max|lhs - rhs| / max|rhs| <= 1e-5."""

import math

import numpy as np
import pytest

import bench

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


@pytest.fixture(scope="module")
def fg():
    import paper_1704_05231_b200 as m

    return m


def _plan(fg, shape, cfg, kind, units=None):
    from paper_1704_05231_b200.device import BankPlan

    return BankPlan(shape, fg.BankSpec(tuple(cfg["freqs"]), cfg["n"], tuple(cfg["sigmas"])), kind, "f32", True, units)


def test_config5_bank_linearity(fg):
    import torch

    cfg = bench.CONFIGS[5]
    f = torch.from_numpy(bench.make_image(cfg, 0)[None]).cuda()
    g = torch.from_numpy(np.random.default_rng(77).uniform(0, 1, (1, 8192, 8192)).astype(np.float32)).cuda()
    h = f + 2.0 * g
    nh = cfg["n"] // 2
    for i in range(5):  # one frequency at a time (17 GB of outputs per frequency set)
        units = [i * (nh + 1) + k for k in range(nh + 1)]
        p = _plan(fg, (1, 8192, 8192), cfg, fg.ExactFIR(3.0), units)
        a, b, c = p(f), p(g), p(h)
        ref = a + 2.0 * b
        err = (c - ref).abs().amax(dim=(-2, -1)) / ref.abs().amax(dim=(-2, -1))
        assert float(err.max()) <= 1e-5, (i, float(err.max()))
        del a, b, c, ref
        torch.cuda.empty_cache()


def test_config4_conjugate_symmetry_and_batch(fg):
    import torch

    from paper_1704_05231_b200.device import SdftPlan

    cfg = bench.CONFIGS[4]
    m = cfg["m"]
    img = torch.from_numpy(bench.make_image(cfg, 0)[None]).cuda()
    for kind in (fg.ExactFIR(3.0), fg.RecursiveIIR()):
        out = SdftPlan(tuple(img.shape), fg.SdftSpec(m, m, kind, cfg["sigma"]), "f32")(img)[0]
        scale = out.abs().amax()
        for u in range(m):
            for v in range(m):
                pu, pv = (m - u) % m, (m - v) % m
                a, b = out[pu * m + pv], out[u * m + v].conj()
                if v > m // 2:  # filled as the conjugate of a computed bin (sdft.py:209-212): bit-exact
                    assert torch.equal(out[u * m + v], out[pu * m + pv].conj()), (u, v)
                else:  # both computed: equal up to rounding (self-paired bins: real up to rounding)
                    assert float((a - b).abs().amax() / scale) <= 1e-6, (u, v)
        del out
        torch.cuda.empty_cache()


def test_config3_batch_equals_single_images(fg):
    """An image's outputs do not depend on its position in a batch (bit-exact, same plan), and equal
    the single-image call's to rounding: the kernel choice may differ with the batch size (the
    persistent tensor-core kernels need enough tiles per SM), never the arithmetic semantics."""
    import torch

    cfg = bench.CONFIGS[3]
    ims = (0, 17, 63)
    imgs = torch.from_numpy(np.stack([bench.make_image(cfg, i) for i in ims])).cuda()
    plan = _plan(fg, tuple(imgs.shape), cfg, fg.ExactFIR(3.0))
    batched = plan(imgs)
    perm = plan(imgs[[2, 0, 1]].contiguous())
    for j, pj in ((0, 1), (1, 2), (2, 0)):
        assert torch.equal(batched[j], perm[pj]), j
    for j in range(len(ims)):
        one = _plan(fg, (1, 1024, 1024), cfg, fg.ExactFIR(3.0))(imgs[j:j + 1].contiguous())[0]
        scale = one.abs().amax()
        assert float((batched[j] - one).abs().amax() / scale) <= 2e-6, j


def test_constant_image_gives_the_dc_response(fg):
    """Replicate padding keeps a constant image constant through both stages, so every
    output pixel is c * K(omega cos theta) * K(omega sin theta) with K the sampled
    Gaussian's transfer function at the stage frequency (gabor.py:107-169)."""
    import torch

    cfg = bench.CONFIGS[3]
    c = 0.75
    img = torch.full((1, 256, 320), c, dtype=torch.float32, device="cuda")
    out = _plan(fg, tuple(img.shape), cfg, fg.ExactFIR(3.0))(img)[0].cpu().numpy()
    for i, (om, sg) in enumerate(zip(cfg["freqs"], cfg["sigmas"])):
        w, h = fg.sampled_gaussian(sg, 3.0)
        t = np.arange(-h, h + 1)
        for k in range(cfg["n"]):
            th = k * math.pi / cfg["n"]
            kx = np.sum(w * np.exp(-1j * om * math.cos(th) * t))
            ky = np.sum(w * np.exp(-1j * om * math.sin(th) * t))
            want = c * kx * ky
            plane = out[i * cfg["n"] + k]
            # relative to the input level c (the DC gain can be ~1e-3 at high omega * sigma)
            assert np.max(np.abs(plane - want)) / max(abs(want), c) <= 1e-5, (i, k, want, plane[0, 0])
