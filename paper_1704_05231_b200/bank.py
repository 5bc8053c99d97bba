"""Gabor filter bank with theta / pi-theta conjugate reuse on the GPU
(drop-in for bank.py of the reference, Algorithm 1 of the paper).

One ``fgb_bank`` call runs, per frequency, ONE fused row launch for every
directly computed orientation k <= N/2 and ONE column launch that emits both
theta_k and pi - theta_k from the same J read (bank.py:90-129).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._precision import real_dtype, resolve
from .gabor import GaborParams, HorizontalStage, _vertical
from .gaussian import SmootherKind, native_smoother
from .image_io import ComplexImage, RealImage
from .metrics import OpCounters, charge_gabor_col, charge_gabor_row

_TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class BankSpec:
    """Frequencies, orientation count N (theta_k = k*pi/N) and sigma rule (bank.py:23-52)."""

    frequencies: tuple[float, ...]
    orientations_n: int
    sigmas: tuple[float, ...] | None = None

    def __post_init__(self) -> None:
        object.__setattr__(self, "frequencies", tuple(float(w) for w in self.frequencies))
        if self.sigmas is not None:
            object.__setattr__(self, "sigmas", tuple(float(s) for s in self.sigmas))
        if self.orientations_n < 1:
            raise ValueError("orientation count must be at least 1")
        if not self.frequencies or any(w <= 0 for w in self.frequencies):
            raise ValueError("frequencies must be a non-empty list of positive values")
        if self.sigmas is not None and len(self.sigmas) != len(self.frequencies):
            raise ValueError("explicit sigma list must match frequencies in length")

    def sigma_for(self, i: int) -> float:
        if self.sigmas is not None:
            return self.sigmas[i]
        return _TWO_PI / self.frequencies[i]

    def thetas(self) -> list[float]:
        n = self.orientations_n
        return [k * math.pi / n for k in range(n)]


@dataclass
class BankOutput:
    """Outputs ordered frequency-major then orientation, plus counters (bank.py:55-60)."""

    entries: list[tuple[GaborParams, ComplexImage]]
    counters: OpCounters


def conjugate_image(j: ComplexImage) -> ComplexImage:
    """Complex conjugate (bank.py:63-65)."""
    return ComplexImage(j.width, j.height, j.re.copy(), -j.im)


def vertical_stage_conjugate(h: HorizontalStage, counters: OpCounters, precision: str | None = None) -> ComplexImage:
    """Mirrored orientation pi - theta from J_theta (bank.py:68-74)."""
    return _vertical(h, counters, True, precision)


def bank_desc(h: int, w: int, spec: BankSpec, kind, prec: str, reuse: bool, batch: int = 1, units=None):
    """C descriptor of a bank call; returns (desc, keepalive)."""
    om = N.double_array(spec.frequencies)
    sg = N.double_array([spec.sigma_for(i) for i in range(len(spec.frequencies))])
    un = N.int_array(units) if units is not None else None
    d = N.fgb_bank_desc(
        N.make_image(h, w, prec, batch=batch), len(spec.frequencies), spec.orientations_n,
        C.cast(om, C.POINTER(C.c_double)), C.cast(sg, C.POINTER(C.c_double)), native_smoother(kind),
        1 if reuse else 0, C.cast(un, C.POINTER(C.c_int32)) if un is not None else None,
        len(units) if units is not None else 0,
    )
    return d, (om, sg, un)


def _charge_bank(counters: OpCounters, spec: BankSpec, kind, h: int, w: int, reuse: bool) -> None:
    n = spec.orientations_n
    nh = n // 2
    for i in range(len(spec.frequencies)):
        s = spec.sigma_for(i)
        if reuse:
            for k in range(nh + 1):
                charge_gabor_row(counters, kind, s, h, w)
                charge_gabor_col(counters, kind, s, h, w)
                if nh < n - k < n:
                    charge_gabor_col(counters, kind, s, h, w)
        else:
            for _ in range(n):
                charge_gabor_row(counters, kind, s, h, w)
                charge_gabor_col(counters, kind, s, h, w)


def _run_bank(f: RealImage, spec: BankSpec, kind, counters: OpCounters, reuse: bool, precision) -> BankOutput:
    prec = resolve(precision)
    h, w = f.data.shape
    d, keep = bank_desc(h, w, spec, kind, prec, reuse)
    for i in range(len(spec.frequencies)):  # same errors as the reference, before any GPU work
        if not spec.sigma_for(i) > 0:
            raise ValueError("sigma must be positive")
    src = np.ascontiguousarray(f.data, dtype=real_dtype(prec))
    n = spec.orientations_n
    # float64 re/im planes straight from the GPU (ComplexImage layout, no host conversion)
    out = np.empty((len(spec.frequencies) * n, 2, h, w), dtype=np.float64)
    bad = C.c_int32(0)
    N.check(N.lib.fgb_bank_host_planar(C.byref(d), src.ctypes.data, out.ctypes.data, C.byref(bad)))
    del keep
    _charge_bank(counters, spec, kind, h, w, reuse)
    thetas = spec.thetas()
    entries = []
    for i, omega in enumerate(spec.frequencies):
        s = spec.sigma_for(i)
        for k in range(n):
            entries.append((GaborParams(omega, thetas[k], s), ComplexImage.from_planar(out[i * n + k], bad.value == 0)))
    return BankOutput(entries, counters)


def compute_bank(f: RealImage, spec: BankSpec, kind: SmootherKind, counters: OpCounters, threads: int = 1,
                 precision: str | None = None) -> BankOutput:
    """Bank with conjugate reuse (bank.py:90-129).  ``threads`` is accepted for
    API compatibility; the GPU schedule is fixed, so results never depend on it."""
    return _run_bank(f, spec, kind, counters, True, precision)


def compute_bank_noreuse(f: RealImage, spec: BankSpec, kind: SmootherKind, counters: OpCounters, threads: int = 1,
                         precision: str | None = None) -> BankOutput:
    """Baseline scheduler, full pipeline per orientation (bank.py:132-157)."""
    return _run_bank(f, spec, kind, counters, False, precision)
