"""Shared test plumbing.

``gpu``-marked tests need a B200 (run via gpurun); everything else runs on
the CPU build container.  Helpers mirror the reference's conftest.py:9-36.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # the library is a build artefact (git-ignored): a fresh checkout builds it
    # once here (nvcc cross-compiles for sm_100a without a GPU)
    lib = os.path.join(ROOT, "paper_1704_05231_b200", "lib", "libfgb200.so")
    if not os.path.exists(lib):
        import subprocess

        subprocess.run([sys.executable, os.path.join(ROOT, "paper_1704_05231_b200", "_build.py")], check=True)


def random_image(seed: int, size: int = 32, lo: float = 0.0, hi: float = 255.0, width=None):
    """conftest.py:9-11 of the reference (square unless ``width`` is given)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(size, size if width is None else width))


def max_rel_err(a, b) -> float:
    """conftest.py:33-36: planes as (re, im) tuples or objects with .re/.im."""
    ar, ai = (a.re, a.im) if hasattr(a, "re") else a
    br, bi = (b.re, b.im) if hasattr(b, "re") else b
    scale = max(np.abs(br).max(), np.abs(bi).max(), 1e-300)
    return max(np.abs(ar - br).max(), np.abs(ai - bi).max()) / scale


@pytest.fixture(scope="session")
def golden():
    z = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
        meta = json.load(fh)
    return z, meta


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
