"""Smoother kinds and coefficient helpers (mirror of gaussian.py of the reference).

The kinds are the reference's frozen dataclasses (gaussian.py:36-68).  The
coefficient math (sampled Gaussian, recursion poles) runs inside libfgb200
(``fgb_sampled_gaussian`` / ``fgb_iir_coeffs``), the same code the kernels'
tap tables come from, so the host view and the device view cannot drift.
Smoothing itself only exists on the GPU (as part of the fused stages).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from functools import lru_cache
from typing import Union

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class RecursiveIIR:
    """Recursive Gaussian smoother marker (gaussian.py:36-38)."""


@dataclass(frozen=True)
class ExactFIR:
    """Truncated exact FIR smoother; support radius*sigma (gaussian.py:41-49)."""

    radius: float = 6.0

    def __post_init__(self) -> None:
        if self.radius < 3:
            raise ValueError("truncation radius must be at least 3 sigma")


@dataclass(frozen=True)
class Box:
    """Moving sum over [-half_width, half_width], zero padded (gaussian.py:52-60)."""

    half_width: int

    def __post_init__(self) -> None:
        if self.half_width < 0:
            raise ValueError("box half-width must be non-negative")


@dataclass(frozen=True)
class _AsymBox:
    # Moving sum over offsets [lo, hi] (gaussian.py:63-68).
    lo: int
    hi: int


SmootherKind = Union[RecursiveIIR, ExactFIR, Box, _AsymBox]


@dataclass(frozen=True)
class GaussianCoeffs:
    """y[n] = B x[n] + (b1 y[n-1] + b2 y[n-2] + b3 y[n-3]) / b0 (gaussian.py:108-124)."""

    sigma: float
    b0: float
    b1: float
    b2: float
    b3: float
    B: float

    def denominator(self) -> np.ndarray:
        return np.array([self.b0, -self.b1, -self.b2, -self.b3])


def native_smoother(kind) -> N.fgb_smoother:
    """Smoother kind -> C descriptor (TypeError for unknown kinds, gaussian.py:279-280)."""
    if isinstance(kind, ExactFIR):
        return N.fgb_smoother(N.FGB_SMOOTH_FIR, 0, float(kind.radius))
    if isinstance(kind, RecursiveIIR):
        return N.fgb_smoother(N.FGB_SMOOTH_IIR, 0, 0.0)
    if isinstance(kind, Box):
        return N.fgb_smoother(N.FGB_SMOOTH_BOX, int(kind.half_width), 0.0)
    raise TypeError(f"unknown smoother kind {kind!r}")


@lru_cache(maxsize=256)
def make_coeffs(sigma: float) -> GaussianCoeffs:
    """Recursion coefficients, unit DC gain per pass (gaussian.py:164-185)."""
    out = (C.c_double * 4)()
    N.check(N.lib.fgb_iir_coeffs(float(sigma), out))
    B, a1, a2, a3 = list(out)
    return GaussianCoeffs(sigma=float(sigma), b0=1.0, b1=-a1, b2=-a2, b3=-a3, B=B)


def sampled_gaussian(sigma: float, radius: float = 6.0) -> tuple[np.ndarray, int]:
    """Unit-sum sampled Gaussian and its half-support (gaussian.py:188-195)."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    half = C.c_int32()
    N.check(N.lib.fgb_sampled_gaussian(float(sigma), float(radius), None, 0, C.byref(half)))
    buf = np.empty(2 * half.value + 1, dtype=np.float64)
    N.check(N.lib.fgb_sampled_gaussian(float(sigma), float(radius),
                                       buf.ctypes.data_as(C.POINTER(C.c_double)), buf.size, C.byref(half)))
    return buf, half.value


def pad_radius(kind: SmootherKind, sigma: float) -> int:
    """Stage-level replicate padding (gaussian.py:198-212)."""
    if isinstance(kind, ExactFIR):
        return max(1, math.ceil(kind.radius * sigma))
    if isinstance(kind, RecursiveIIR):
        return math.ceil(5.0 * sigma) + 2
    return 0


# ---- 1-D smoothing entry points (gaussian.py:245-302) ------------------------

def _lines_desc(n_lines: int, length: int, kind, sigma: float, prec: str, assume_padded: bool) -> N.fgb_lines_desc:
    lo = hi = 0
    if isinstance(kind, Box):
        sm = N.fgb_smoother(N.FGB_SMOOTH_BOX, int(kind.half_width), 0.0)
        lo, hi = -int(kind.half_width), int(kind.half_width)
    elif isinstance(kind, _AsymBox):
        sm = N.fgb_smoother(N.FGB_SMOOTH_BOX, 0, 0.0)
        lo, hi = int(kind.lo), int(kind.hi)
    else:
        sm = native_smoother(kind)  # TypeError for unknown kinds (gaussian.py:279-280)
    return N.fgb_lines_desc(n_lines, length, length, N.dtype_code(prec), int(bool(assume_padded)), float(sigma), sm,
                            lo, hi)


def smooth_lines(lines: np.ndarray, kind: SmootherKind, sigma: float, counters, nominal_len: int | None = None,
                 direction: str = "h", assume_padded: bool = False, precision: str | None = None) -> np.ndarray:
    """Smooth each row of a 2-D array independently (gaussian.py:245-285).

    Same dispatch, validation and counter charges as the reference; the lines
    are smoothed on the GPU by ``fgb_smooth_lines_host`` (FIR / box: tiled
    correlation; IIR: fp64-state recursion with the reference's padding and
    steady-state init).  Returns float64 like the reference.
    """
    from ._precision import real_dtype, resolve
    from .metrics import charge_smoothing

    prec = resolve(precision)
    arr = np.asarray(lines)
    if arr.ndim != 2:
        raise ValueError("lines must be a 2-D array")
    rows, length = arr.shape
    src = np.ascontiguousarray(arr, dtype=real_dtype(prec))
    d = _lines_desc(rows, length, kind, sigma, prec, assume_padded)
    out = np.empty((rows, length), dtype=real_dtype(prec))
    if rows and length:
        N.check(N.lib.fgb_smooth_lines_host(C.byref(d), src.ctypes.data, out.ctypes.data))
    elif isinstance(kind, (ExactFIR, RecursiveIIR)):
        # empty input: still raise the reference's parameter errors (sampled_gaussian / make_coeffs)
        if isinstance(kind, RecursiveIIR):
            make_coeffs(float(sigma))
        else:
            sampled_gaussian(float(sigma), kind.radius)
    charge_smoothing(counters, kind, sigma, rows, nominal_len if nominal_len is not None else length, direction)
    return out.astype(np.float64, copy=False)


def smooth_1d(signal: np.ndarray, kind: SmootherKind, sigma: float, counters,
              precision: str | None = None) -> np.ndarray:
    """Smooth a single 1-D signal (gaussian.py:288-295)."""
    signal = np.asarray(signal, dtype=np.float64)
    if signal.ndim != 1 or signal.size < 1:
        raise ValueError("signal must be a non-empty 1-D array")
    return smooth_lines(signal[None, :], kind, sigma, counters, precision=precision)[0]


def smooth_pair_1d(a: np.ndarray, b: np.ndarray, kind: SmootherKind, sigma: float, counters,
                   precision: str | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Smooth two signals -- per-stage cost is visibly two smoothings (gaussian.py:298-302)."""
    return (smooth_1d(a, kind, sigma, counters, precision=precision),
            smooth_1d(b, kind, sigma, counters, precision=precision))
