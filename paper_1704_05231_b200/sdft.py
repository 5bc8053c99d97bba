"""Gaussian-windowed 2-D localized sliding DFT on the GPU (drop-in for sdft.py
of the reference, Algorithm 2 of the paper)."""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._precision import cplx_dtype, real_dtype, resolve
from .bank import conjugate_image  # noqa: F401  (re-exported like the reference)
from .gaussian import Box, SmootherKind, _AsymBox, native_smoother
from .image_io import ComplexImage, RealImage
from .metrics import OpCounters, charge_sdft_stage

_TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class SdftSpec:
    """Window extents, Gaussian sigma and smoothing engine (sdft.py:25-57)."""

    mx: int
    my: int
    smoother: SmootherKind
    sigma: float | None = None

    def __post_init__(self) -> None:
        if self.mx < 1 or self.my < 1:
            raise ValueError("window extents must be at least 1")
        if self.sigma is not None and self.sigma <= 0:
            raise ValueError("sigma must be positive")

    @property
    def sigma_value(self) -> float:
        if self.sigma is not None:
            return self.sigma
        return (min(self.mx, self.my) // 2) / 3.0

    @property
    def omega0x(self) -> float:
        return _TWO_PI / self.mx

    @property
    def omega0y(self) -> float:
        return _TWO_PI / self.my


@dataclass
class SdftOutput:
    """bins[u][v] ComplexImages plus counters (sdft.py:60-65)."""

    bins: list[list[ComplexImage]]
    counters: OpCounters


def _axis_kind(spec: SdftSpec, m: int) -> SmootherKind:
    """sdft.py:68-72."""
    if isinstance(spec.smoother, (Box, _AsymBox)):
        return _AsymBox(lo=-(m // 2), hi=m - 1 - m // 2)
    return spec.smoother


def sdft_desc(h: int, w: int, spec: SdftSpec, prec: str, batch: int = 1, heads=None):
    sm = spec.smoother
    if isinstance(sm, _AsymBox):
        sm = Box(0)  # the window comes from (mx, my) for box kinds
    hd = N.int_array(heads) if heads is not None else None
    d = N.fgb_sdft_desc(
        N.make_image(h, w, prec, batch=batch), spec.mx, spec.my, float(spec.sigma_value), native_smoother(sm),
        C.cast(hd, C.POINTER(C.c_int32)) if hd is not None else None, len(heads) if heads is not None else 0,
    )
    return d, hd


def _charge_h(c, spec, h, w):
    charge_sdft_stage(c, _axis_kind(spec, spec.mx), spec.sigma_value, h, w, False, 1)


def _charge_v(c, spec, h, w):
    charge_sdft_stage(c, _axis_kind(spec, spec.my), spec.sigma_value, w, h, True, 0)


def sdft_horizontal(f: RealImage, u: int, spec: SdftSpec, counters: OpCounters,
                    precision: str | None = None) -> ComplexImage:
    """Horizontal intermediate J_u (sdft.py:134-150)."""
    if not 0 <= u < spec.mx:
        raise ValueError(f"bin index u={u} outside [0, {spec.mx})")
    prec = resolve(precision)
    h, w = f.data.shape
    d, keep = sdft_desc(h, w, spec, prec)
    src = np.ascontiguousarray(f.data, dtype=real_dtype(prec))
    out = np.empty((h, w), dtype=cplx_dtype(prec))
    N.check(N.lib.fgb_sdft_horizontal_host(C.byref(d), u, src.ctypes.data, out.ctypes.data))
    _charge_h(counters, spec, h, w)
    return ComplexImage.from_interleaved(out)


def sdft_bin(f: RealImage, u: int, v: int, spec: SdftSpec, counters: OpCounters,
             precision: str | None = None) -> ComplexImage:
    """Single bin (u, v), computed directly without reuse (sdft.py:169-175)."""
    if not 0 <= v < spec.my:
        raise ValueError(f"bin index v={v} outside [0, {spec.my})")
    if not 0 <= u < spec.mx:
        raise ValueError(f"bin index u={u} outside [0, {spec.mx})")
    prec = resolve(precision)
    h, w = f.data.shape
    d, keep = sdft_desc(h, w, spec, prec)
    src = np.ascontiguousarray(f.data, dtype=real_dtype(prec))
    out = np.empty((h, w), dtype=cplx_dtype(prec))
    N.check(N.lib.fgb_sdft_bin_host(C.byref(d), u, v, src.ctypes.data, out.ctypes.data))
    _charge_h(counters, spec, h, w)
    _charge_v(counters, spec, h, w)
    return ComplexImage.from_interleaved(out)


def _charge_full(counters: OpCounters, spec: SdftSpec, h: int, w: int) -> None:
    if spec.my < spec.mx:  # transposed route (sdft.py:185-195)
        _charge_full(counters, SdftSpec(mx=spec.my, my=spec.mx, smoother=spec.smoother, sigma=spec.sigma), w, h)
        return
    for _ in range(spec.mx // 2 + 1):
        _charge_h(counters, spec, h, w)
    for _ in range(spec.mx * (spec.my // 2 + 1)):
        _charge_v(counters, spec, h, w)


def sdft_full(f: RealImage, spec: SdftSpec, counters: OpCounters, precision: str | None = None) -> SdftOutput:
    """All Mx*My bins with horizontal and conjugate-symmetry reuse (sdft.py:178-213)."""
    prec = resolve(precision)
    h, w = f.data.shape
    d, keep = sdft_desc(h, w, spec, prec)
    src = np.ascontiguousarray(f.data, dtype=real_dtype(prec))
    out = np.empty((spec.mx * spec.my, 2, h, w), dtype=np.float64)
    bad = C.c_int32(0)
    N.check(N.lib.fgb_sdft_host_planar(C.byref(d), src.ctypes.data, out.ctypes.data, C.byref(bad)))
    _charge_full(counters, spec, h, w)
    bins = [[ComplexImage.from_planar(out[u * spec.my + v], bad.value == 0) for v in range(spec.my)]
            for u in range(spec.mx)]
    return SdftOutput(bins, counters)
