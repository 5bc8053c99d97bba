"""Precision selection of the drop-in API.

The reference computes in float64 (image_io.py:33-35), so the drop-in
defaults to the fp64 build ("f64", parity <= 1e-10).  "f32" is the
throughput build (complex64 outputs, parity <= 1e-5).  Override per call with
``precision=...`` or globally with ``set_precision`` / ``FGB_PRECISION``.
"""

from __future__ import annotations

import os

import numpy as np

_DEFAULT = os.environ.get("FGB_PRECISION", "f64")


def set_precision(p: str) -> None:
    global _DEFAULT
    if p not in ("f32", "f64"):
        raise ValueError("precision must be 'f32' or 'f64'")
    _DEFAULT = p


def get_precision() -> str:
    return _DEFAULT


def resolve(p: str | None) -> str:
    p = _DEFAULT if p is None else p
    if p not in ("f32", "f64"):
        raise ValueError("precision must be 'f32' or 'f64'")
    return p


def real_dtype(p: str):
    return np.float32 if p == "f32" else np.float64


def cplx_dtype(p: str):
    return np.complex64 if p == "f32" else np.complex128
