"""Brute-force references on the GPU (drop-in for the reference's oracle.py:22-109).

Direct 2-D tap sums of Eq. 1 (complex Gabor, replicate boundary) and Eq. 17
(one localized-DFT bin, Gaussian/replicate or box/zero window), computed by
``fgb_fir_gabor`` / ``fgb_localized_dft`` in libfgb200.  O(support^2) per
pixel but independent of the separable decomposition, so they validate full-
size outputs (the reference guards its CPU oracle to 2^18 px, cli.py:134-140).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._precision import cplx_dtype, real_dtype, resolve
from .gabor import GaborParams, _filter_desc
from .gaussian import ExactFIR
from .image_io import ComplexImage, RealImage
from .sdft import SdftSpec, sdft_desc


@dataclass(frozen=True)
class OracleConfig:
    """Gaussian support truncation in sigmas; replicate boundary (oracle.py:22-30)."""

    radius: float = 6.0

    def __post_init__(self) -> None:
        if self.radius < 3:
            raise ValueError("truncation radius must be at least 3 sigma")


def fir_gabor(f: RealImage, p: GaborParams, cfg: OracleConfig = OracleConfig(),
              precision: str | None = None) -> ComplexImage:
    """Direct evaluation of the 2-D complex Gabor filter (oracle.py:53-66)."""
    prec = resolve(precision)
    h, w = f.data.shape
    d = _filter_desc(h, w, p, ExactFIR(cfg.radius), prec)
    src = np.ascontiguousarray(f.data, dtype=real_dtype(prec))
    out = np.empty((h, w), dtype=cplx_dtype(prec))
    N.check(N.lib.fgb_fir_gabor_host(C.byref(d), float(cfg.radius), src.ctypes.data, out.ctypes.data))
    return ComplexImage.from_interleaved(out)


def localized_dft(f: RealImage, u: int, v: int, spec: SdftSpec, cfg: OracleConfig = OracleConfig(),
                  precision: str | None = None) -> ComplexImage:
    """Direct evaluation of one localized-DFT bin (oracle.py:69-109)."""
    if not (0 <= u < spec.mx and 0 <= v < spec.my):
        raise ValueError("bin indices outside the window grid")
    prec = resolve(precision)
    h, w = f.data.shape
    d, keep = sdft_desc(h, w, spec, prec)
    src = np.ascontiguousarray(f.data, dtype=real_dtype(prec))
    out = np.empty((h, w), dtype=cplx_dtype(prec))
    N.check(N.lib.fgb_localized_dft_host(C.byref(d), int(u), int(v), float(cfg.radius), src.ctypes.data,
                                         out.ctypes.data))
    return ComplexImage.from_interleaved(out)
