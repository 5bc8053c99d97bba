"""ctypes binding of libfgb200.so (the C ABI declared in include/fgb200.h).

There is no CPU fallback: if the shared library is missing the import fails
loudly (run ``python paper_1704_05231_b200/_build.py`` or
``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FGB200_LIB", os.path.join(_HERE, "lib", "libfgb200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libfgb200.so not found at {LIB_PATH}: build it with `python paper_1704_05231_b200/_build.py` "
        "(the B200 path has no CPU fallback)"
    )

lib = C.CDLL(LIB_PATH)

FGB_OK = 0
FGB_EINVAL = -1
FGB_ECUDA = -2
FGB_ENOMEM = -3
FGB_EUNSUPPORTED = -4
FGB_ENCCL = -5
FGB_MGPU_ID_BYTES = 128
FGB_F32 = 0
FGB_F64 = 1
FGB_SMOOTH_FIR = 0
FGB_SMOOTH_IIR = 1
FGB_SMOOTH_BOX = 2


class fgb_smoother(C.Structure):
    _fields_ = [("kind", C.c_int32), ("box_half", C.c_int32), ("radius", C.c_double)]


class fgb_image(C.Structure):
    _fields_ = [
        ("height", C.c_int32),
        ("width", C.c_int32),
        ("pitch", C.c_int64),
        ("batch", C.c_int32),
        ("dtype", C.c_int32),
        ("batch_stride", C.c_int64),
    ]


class fgb_bank_desc(C.Structure):
    _fields_ = [
        ("img", fgb_image),
        ("n_freq", C.c_int32),
        ("orientations", C.c_int32),
        ("omegas", C.POINTER(C.c_double)),
        ("sigmas", C.POINTER(C.c_double)),
        ("smoother", fgb_smoother),
        ("reuse", C.c_int32),
        ("units", C.POINTER(C.c_int32)),
        ("n_units", C.c_int32),
    ]


class fgb_filter_desc(C.Structure):
    _fields_ = [
        ("img", fgb_image),
        ("omega", C.c_double),
        ("theta", C.c_double),
        ("sigma", C.c_double),
        ("smoother", fgb_smoother),
    ]


class fgb_sdft_desc(C.Structure):
    _fields_ = [
        ("img", fgb_image),
        ("mx", C.c_int32),
        ("my", C.c_int32),
        ("sigma", C.c_double),
        ("smoother", fgb_smoother),
        ("u_heads", C.POINTER(C.c_int32)),
        ("n_heads", C.c_int32),
    ]


class fgb_lines_desc(C.Structure):
    _fields_ = [
        ("n_lines", C.c_int32),
        ("len", C.c_int32),
        ("pitch", C.c_int64),
        ("dtype", C.c_int32),
        ("assume_padded", C.c_int32),
        ("sigma", C.c_double),
        ("smoother", fgb_smoother),
        ("box_lo", C.c_int32),
        ("box_hi", C.c_int32),
    ]


class fgb_prof_entry(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("launches", C.c_int64), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double)]


_vp = C.c_void_p
_P = C.POINTER
_SIGS = {
    "fgb_last_error": (C.c_char_p, []),
    "fgb_version": (C.c_int32, []),
    "fgb_device_sm_count": (C.c_int32, []),
    "fgb_pad_radius": (C.c_int32, [_P(fgb_smoother), C.c_double]),
    "fgb_sampled_gaussian": (C.c_int32, [C.c_double, C.c_double, _P(C.c_double), C.c_int32, _P(C.c_int32)]),
    "fgb_iir_coeffs": (C.c_int32, [C.c_double, _P(C.c_double)]),
    "fgb_iir_sections": (C.c_int32, [C.c_double, _P(C.c_double)]),
    "fgb_bank_entries": (C.c_int64, [_P(fgb_bank_desc)]),
    "fgb_sdft_bins": (C.c_int64, [_P(fgb_sdft_desc)]),
    "fgb_bank_workspace_bytes": (C.c_int64, [_P(fgb_bank_desc)]),
    "fgb_sdft_workspace_bytes": (C.c_int64, [_P(fgb_sdft_desc)]),
    "fgb_bank": (C.c_int32, [_P(fgb_bank_desc), _vp, _vp, _vp]),
    "fgb_filter": (C.c_int32, [_P(fgb_filter_desc), _vp, _vp, _vp]),
    "fgb_horizontal_stage": (C.c_int32, [_P(fgb_filter_desc), _vp, _vp, _vp]),
    "fgb_vertical_stage": (C.c_int32, [_P(fgb_filter_desc), _vp, _vp, C.c_int32, _vp]),
    "fgb_sdft": (C.c_int32, [_P(fgb_sdft_desc), _vp, _vp, _vp]),
    "fgb_sdft_bin": (C.c_int32, [_P(fgb_sdft_desc), C.c_int32, C.c_int32, _vp, _vp, _vp]),
    "fgb_sdft_horizontal": (C.c_int32, [_P(fgb_sdft_desc), C.c_int32, _vp, _vp, _vp]),
    "fgb_smooth_lines": (C.c_int32, [_P(fgb_lines_desc), _vp, _vp, _vp]),
    "fgb_ser_sums": (C.c_int32, [_vp, _vp, C.c_int64, C.c_int32, _P(C.c_double), _vp]),
    "fgb_smooth_lines_host": (C.c_int32, [_P(fgb_lines_desc), _vp, _vp]),
    "fgb_bank_host": (C.c_int32, [_P(fgb_bank_desc), _vp, _vp]),
    "fgb_filter_host": (C.c_int32, [_P(fgb_filter_desc), _vp, _vp]),
    "fgb_sdft_host": (C.c_int32, [_P(fgb_sdft_desc), _vp, _vp]),
    "fgb_bank_host_planar": (C.c_int32, [_P(fgb_bank_desc), _vp, _vp, _P(C.c_int32)]),
    "fgb_filter_host_planar": (C.c_int32, [_P(fgb_filter_desc), _vp, _vp, _P(C.c_int32)]),
    "fgb_sdft_host_planar": (C.c_int32, [_P(fgb_sdft_desc), _vp, _vp, _P(C.c_int32)]),
    "fgb_horizontal_stage_host": (C.c_int32, [_P(fgb_filter_desc), _vp, _vp]),
    "fgb_vertical_stage_host": (C.c_int32, [_P(fgb_filter_desc), _vp, _vp, C.c_int32]),
    "fgb_sdft_bin_host": (C.c_int32, [_P(fgb_sdft_desc), C.c_int32, C.c_int32, _vp, _vp]),
    "fgb_sdft_horizontal_host": (C.c_int32, [_P(fgb_sdft_desc), C.c_int32, _vp, _vp]),
    "fgb_fir_gabor": (C.c_int32, [_P(fgb_filter_desc), C.c_double, _vp, _vp, _vp]),
    "fgb_localized_dft": (C.c_int32, [_P(fgb_sdft_desc), C.c_int32, C.c_int32, C.c_double, _vp, _vp, _vp]),
    "fgb_fir_gabor_host": (C.c_int32, [_P(fgb_filter_desc), C.c_double, _vp, _vp]),
    "fgb_localized_dft_host": (C.c_int32, [_P(fgb_sdft_desc), C.c_int32, C.c_int32, C.c_double, _vp, _vp]),
    "fgb_gbnk_write_device": (C.c_int32, [C.c_char_p, _P(C.c_double), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                          _vp, C.c_int32, _vp]),
    "fgb_mgpu_unique_id": (C.c_int32, [_P(C.c_ubyte)]),
    "fgb_mgpu_init": (C.c_int32, [_P(C.c_ubyte), C.c_int32, C.c_int32, C.c_int32]),
    "fgb_mgpu_finalize": (C.c_int32, []),
    "fgb_mgpu_bank_units": (C.c_int32, [_P(fgb_bank_desc), C.c_int32, C.c_int32, _P(C.c_int32), C.c_int32]),
    "fgb_mgpu_sdft_heads": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32, _P(C.c_int32), C.c_int32]),
    "fgb_mgpu_bank_entries": (C.c_int32, [_P(fgb_bank_desc)]),
    "fgb_mgpu_bank": (C.c_int32, [_P(fgb_bank_desc), _vp, _vp, _vp]),
    "fgb_mgpu_sdft": (C.c_int32, [_P(fgb_sdft_desc), _vp, _vp, _vp]),
    "fgb_mgpu_last_error": (C.c_char_p, []),
    "fgb_profile_enable": (None, [C.c_int32]),
    "fgb_profile_read": (C.c_int32, [_P(fgb_prof_entry), C.c_int32]),
    "fgb_launch_count": (C.c_int64, []),
    "fgb_probe_fp32_tflops": (C.c_double, []),
    "fgb_probe_fp64_tflops": (C.c_double, []),
    "fgb_probe_fma": (C.c_double, [C.c_int32, C.c_int32]),
    "fgb_stream_synchronize": (C.c_int32, [_vp]),
    "fgb_release_caches": (None, []),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def last_error() -> str:
    return (lib.fgb_last_error() or b"").decode()


def check(rc: int, mgpu: bool = False) -> int:
    """Map a negative status to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = (lib.fgb_mgpu_last_error() or b"").decode() if mgpu else last_error()
    if rc == FGB_EINVAL:
        raise ValueError(msg)
    if rc == FGB_EUNSUPPORTED:
        raise TypeError(msg)
    if rc == FGB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libfgb200: {msg}")


def dtype_code(precision: str) -> int:
    if precision in ("f32", "float32", np.float32):
        return FGB_F32
    if precision in ("f64", "float64", np.float64):
        return FGB_F64
    raise ValueError(f"precision must be 'f32' or 'f64', got {precision!r}")


def make_image(h: int, w: int, precision: str, batch: int = 1, pitch=None, batch_stride=None) -> fgb_image:
    p = w if pitch is None else pitch
    return fgb_image(h, w, p, batch, dtype_code(precision), h * p if batch_stride is None else batch_stride)


def double_array(vals):
    arr = (C.c_double * len(vals))(*[float(v) for v in vals])
    return arr


def int_array(vals):
    return (C.c_int32 * len(vals))(*[int(v) for v in vals])


def profile_read() -> list[dict]:
    cap = 4096  # distinct step names (FGB_PROF_DETAIL names every step of a plan)
    buf = (fgb_prof_entry * cap)()
    n = check(lib.fgb_profile_read(buf, cap))
    return [dict(name=e.name.decode(), launches=e.launches, ms=e.ms, flops=e.flops, bytes=e.bytes)
            for e in buf[: min(n, cap)]]
