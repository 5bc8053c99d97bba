"""Single-filter Gabor stages on the GPU (drop-in for gabor.py of the reference).

Same names, signatures, validation and counter charges as the reference
(gabor.py:68-176); the arithmetic runs in libfgb200 (row kernel K1 and column
kernel K2, or the fp64-state recursion K4 for RecursiveIIR).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._precision import resolve, real_dtype, cplx_dtype
from .gaussian import SmootherKind, native_smoother
from .image_io import ComplexImage, RealImage
from .metrics import OpCounters, charge_gabor_col, charge_gabor_row


@dataclass(frozen=True)
class GaborParams:
    """(omega, theta, sigma) of one filter; theta normalised into [0, pi) (gabor.py:68-90)."""

    omega: float
    theta: float
    sigma: float

    def __post_init__(self) -> None:
        if self.omega <= 0:
            raise ValueError("omega must be positive")
        if self.sigma <= 0:
            raise ValueError("sigma must be positive")
        object.__setattr__(self, "theta", self.theta % math.pi)

    @property
    def omega_c(self) -> float:
        return self.omega * math.cos(self.theta)

    @property
    def omega_s(self) -> float:
        return self.omega * math.sin(self.theta)


@dataclass
class HorizontalStage:
    """Horizontal-stage intermediate J plus the parameters that produced it (gabor.py:93-99)."""

    j: ComplexImage
    params: GaborParams
    smoother: SmootherKind


def _filter_desc(h: int, w: int, p: GaborParams, kind, prec: str) -> N.fgb_filter_desc:
    return N.fgb_filter_desc(N.make_image(h, w, prec), float(p.omega), float(p.theta), float(p.sigma),
                             native_smoother(kind))


def _as_real(f: RealImage, prec: str) -> np.ndarray:
    return np.ascontiguousarray(f.data, dtype=real_dtype(prec))


def horizontal_stage(f: RealImage, p: GaborParams, kind: SmootherKind, counters: OpCounters,
                     precision: str | None = None) -> HorizontalStage:
    """Row-wise 1-D Gabor filtering (gabor.py:107-132)."""
    prec = resolve(precision)
    h, w = f.data.shape
    d = _filter_desc(h, w, p, kind, prec)
    src = _as_real(f, prec)
    out = np.empty((h, w), dtype=cplx_dtype(prec))
    N.check(N.lib.fgb_horizontal_stage_host(C.byref(d), src.ctypes.data, out.ctypes.data))
    charge_gabor_row(counters, kind, p.sigma, h, w)
    return HorizontalStage(ComplexImage.from_interleaved(out), p, kind)


def _vertical(hs: HorizontalStage, counters: OpCounters, conjugate: bool, precision: str | None = None) -> ComplexImage:
    """Column stage; conjugate=True evaluates pi - theta (gabor.py:135-164)."""
    prec = resolve(precision)
    p = hs.params
    h, w = hs.j.re.shape
    d = _filter_desc(h, w, p, hs.smoother, prec)
    j = np.empty((h, w), dtype=cplx_dtype(prec))
    j.real = hs.j.re
    j.imag = hs.j.im
    out = np.empty((h, w), dtype=cplx_dtype(prec))
    N.check(N.lib.fgb_vertical_stage_host(C.byref(d), j.ctypes.data, out.ctypes.data, 1 if conjugate else 0))
    charge_gabor_col(counters, hs.smoother, p.sigma, h, w)
    return ComplexImage.from_interleaved(out)


def vertical_stage(h: HorizontalStage, counters: OpCounters, precision: str | None = None) -> ComplexImage:
    """Column-wise 1-D Gabor filtering of the horizontal intermediate (gabor.py:167-169)."""
    return _vertical(h, counters, False, precision)


def gabor_filter(f: RealImage, p: GaborParams, kind: SmootherKind, counters: OpCounters,
                 precision: str | None = None) -> ComplexImage:
    """Full 2-D complex Gabor filter, fused on the GPU (gabor.py:172-176)."""
    prec = resolve(precision)
    h, w = f.data.shape
    d = _filter_desc(h, w, p, kind, prec)
    src = _as_real(f, prec)
    out = np.empty((2, h, w), dtype=np.float64)
    bad = C.c_int32(0)
    N.check(N.lib.fgb_filter_host_planar(C.byref(d), src.ctypes.data, out.ctypes.data, C.byref(bad)))
    charge_gabor_row(counters, kind, p.sigma, h, w)
    charge_gabor_col(counters, kind, p.sigma, h, w)
    return ComplexImage.from_planar(out, bad.value == 0)
