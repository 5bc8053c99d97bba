"""GPU: the tensor-core (tcgen05, split-fp16) row and column passes of the fp32
bank (csrc/row_umma.cu, csrc/col_umma.cu) against the CPU oracle, tolerance
max|err| / max|ref| <= 1e-5 (the reference's metric, conftest.py:33-36).

What these cases pin beyond the full-size configs (test_gpu_fullsize.py):
* both tensor-core passes (W % 8 == 0), the column pass alone (W % 8 == 4:
  FFMA rows writing split-fp16 J) and the FFMA fallback (K = 64 + 2 jpad > 256);
* tile edges: heights that are not multiples of 64 / 128, widths that are not
  multiples of 64 (partial strips), the replicate pad rows at both image edges;
* the per-image J scale 2^e (max|f| of each image of a batch, 12 decades apart),
  an all-zero image (exact zeros) and a constant image;
* the FFMA kernels behind FGB_COL_FFMA / FGB_ROW_FFMA (read once per process, so
  in a subprocess) against the same oracle."""

import math
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import fastgabor_oracle as O
from .conftest import max_rel_err, random_image

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_1704_05231_b200 as fg
    from paper_1704_05231_b200 import device as D

    return torch, fg, D


def bank_err(fg, f, N, freqs, sigmas):
    spec = fg.BankSpec(tuple(freqs), N, tuple(sigmas))
    out = fg.compute_bank(fg.RealImage.from_array(f), spec, fg.ExactFIR(3.0), fg.OpCounters(), precision="f32")
    ref = O.compute_bank(f, spec.frequencies, N, spec.sigmas, ("fir", 3.0))
    return max(max_rel_err((img.re, img.im), r[3:]) for (_, img), r in zip(out.entries, ref))


@pytest.mark.parametrize(
    "H,W,N,freqs,sigmas",
    [
        (64, 64, 4, [math.pi / 4], [4.0]),                       # one tile each way
        (131, 200, 8, [math.pi / 4, math.pi / 8], [4.0, 8.0]),   # partial strips / tiles, both passes
        (333, 320, 8, [math.pi / 8, math.pi / 16], [8.0, 16.0]),
        (260, 196, 16, [math.pi / 16, math.pi / 32], [16.0, 32.0]),  # W % 8 == 4: FFMA rows, TC columns
        (97, 136, 6, [1.3, 0.4], [5.0, 11.0]),                   # non-dyadic frequencies
        (150, 264, 8, [0.2], [40.0]),                            # K > 256: FFMA fallback for both passes
    ],
)
def test_tensor_core_bank_vs_oracle(env, H, W, N, freqs, sigmas):
    torch, fg, D = env
    f = random_image(H * 7 + W, H, 0.0, 1.0, width=W)
    assert bank_err(fg, f, N, freqs, sigmas) <= TOL


def test_tensor_core_kernels_are_the_ones_that_run(env):
    """The live per-kernel profile of an fp32 FIR bank names the tensor-core kernels."""
    torch, fg, D = env
    from paper_1704_05231_b200 import _native as N

    f = torch.rand((4, 1024, 1024), device="cuda")  # >= 16 row tiles per SM: the row pass runs on the tensor cores too
    spec = fg.BankSpec((math.pi / 8, math.pi / 32), 8, (8.0, 32.0))
    N.lib.fgb_profile_enable(1)
    try:
        D.compute_bank(f, spec, fg.ExactFIR(3.0))
        torch.cuda.synchronize()
        names = {e["name"] for e in N.profile_read()}
    finally:
        N.lib.fgb_profile_enable(0)
    assert {"row_umma", "col_umma", "bank_umma"} <= names, names  # sigma 32: two passes; sigma 8: fused


def test_per_image_scale_in_a_batch(env):
    """Images 12 decades apart in one batched call: each gets its own J scale."""
    torch, fg, D = env
    spec = fg.BankSpec((math.pi / 4, math.pi / 16), 8, (4.0, 16.0))
    imgs = [random_image(40 + i, 96, 0.0, 1.0, width=128) * s for i, s in enumerate((1e-6, 1.0, 1e6))]
    f = torch.from_numpy(np.stack(imgs).astype(np.float32)).cuda()
    out = D.compute_bank(f, spec, fg.ExactFIR(3.0)).cpu().numpy()
    for i, img in enumerate(imgs):
        ref = O.compute_bank(img.astype(np.float32).astype(np.float64), spec.frequencies, 8, spec.sigmas, ("fir", 3.0))
        for e, r in enumerate(ref):
            assert max_rel_err((out[i, e].real, out[i, e].imag), r[3:]) <= TOL, (i, e)


def test_zero_and_constant_images(env):
    torch, fg, D = env
    spec = fg.BankSpec((math.pi / 4, math.pi / 16), 8, (4.0, 16.0))
    z = torch.zeros((1, 128, 128), dtype=torch.float32, device="cuda")
    assert int((D.compute_bank(z, spec, fg.ExactFIR(3.0)).abs() != 0).sum()) == 0
    c = np.full((128, 192), 3.25)
    assert bank_err(fg, c, 8, spec.frequencies, spec.sigmas) <= TOL


def test_tensor_core_rows_on_small_images():
    """FGB_ROW_UMMA forces the tensor-core row pass below its size threshold (read once per process:
    a subprocess) -- the parity cases above again, through row_umma's tile edges."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import math, sys; sys.path.insert(0, '.');"
        "from tests.test_gpu_umma import bank_err; import paper_1704_05231_b200 as fg;"
        "from tests.conftest import random_image;"
        "cases = [(64, 64, 4, [math.pi / 4], [4.0]), (131, 200, 8, [math.pi / 4, math.pi / 8], [4.0, 8.0]),"
        " (333, 320, 8, [math.pi / 8, math.pi / 16], [8.0, 16.0]), (97, 136, 6, [1.3, 0.4], [5.0, 11.0]),"
        " (260, 264, 16, [math.pi / 16, math.pi / 32], [16.0, 32.0])];"
        "errs = [bank_err(fg, random_image(H * 7 + W, H, 0.0, 1.0, width=W), N, fr, sg) for H, W, N, fr, sg in cases];"
        "print(errs); assert max(errs) <= 1e-5"
    )
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, FGB_ROW_UMMA="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout, r.stderr[-2000:])


def test_fused_tensor_core_bank_on_small_images():
    """FGB_BANK_UMMA=2 forces the fused row + column kernel (bank_umma.cu, J in shared memory) below its
    size threshold: tile edges, partial strips, the replicate rows of the padded image planes."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import math, sys; sys.path.insert(0, '.');"
        "from tests.test_gpu_umma import bank_err; import paper_1704_05231_b200 as fg;"
        "from tests.conftest import random_image;"
        "cases = [(64, 64, 4, [math.pi / 4], [4.0]), (131, 200, 8, [math.pi / 4, math.pi / 8], [4.0, 8.0]),"
        " (333, 320, 8, [math.pi / 8, math.pi / 3], [8.0, 10.0]), (97, 136, 6, [1.3, 0.4], [5.0, 7.0]),"
        " (260, 264, 16, [math.pi / 16], [3.0]), (200, 328, 8, [math.pi / 16, math.pi / 32], [16.0, 32.0]),"
        " (131, 72, 5, [0.2], [14.5])];"
        "errs = [bank_err(fg, random_image(H * 7 + W, H, 0.0, 1.0, width=W), N, fr, sg) for H, W, N, fr, sg in cases];"
        "print(errs); assert max(errs) <= 1e-5"
    )
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, FGB_BANK_UMMA="2"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout, r.stderr[-2000:])


def test_ffma_kernels_behind_the_knobs():
    """FGB_COL_FFMA / FGB_ROW_FFMA select the FFMA kernels (A/B runs); they meet the same bar."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import math, sys; sys.path.insert(0, '.');"
        "from tests.test_gpu_umma import bank_err; import paper_1704_05231_b200 as fg;"
        "from tests.conftest import random_image;"
        "f = random_image(3, 200, 0.0, 1.0, width=256);"
        "e = bank_err(fg, f, 8, [math.pi / 8, math.pi / 32], [8.0, 32.0]);"
        "print(e); assert e <= 1e-5"
    )
    for knobs in ({"FGB_ROW_FFMA": "1"}, {"FGB_COL_FFMA": "1"}):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **knobs),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, (knobs, r.stdout, r.stderr[-2000:])
