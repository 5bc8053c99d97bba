"""Device-tensor API (the "native" throughput path): inputs and outputs stay in
HBM, calls are stream-ordered on torch's current CUDA stream.

PyTorch is only plumbing here (device memory, streams); the arithmetic runs
in libfgb200 through the same C ABI the drop-in host API uses.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .bank import BankSpec, bank_desc
from .sdft import SdftSpec, sdft_desc


def _prec(t: torch.Tensor) -> str:
    if t.dtype == torch.float32:
        return "f32"
    if t.dtype == torch.float64:
        return "f64"
    raise TypeError(f"image must be float32 or float64, got {t.dtype}")


def _cplx(prec: str):
    return torch.complex64 if prec == "f32" else torch.complex128


def _stream(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _check_img(img: torch.Tensor):
    if not img.is_cuda:
        raise ValueError("image must be a CUDA tensor")
    if img.dim() == 2:
        img = img.unsqueeze(0)
    if img.dim() != 3 or img.stride(-1) != 1:
        raise ValueError("image must be [H, W] or [B, H, W] with unit column stride")
    return img


def _check_out(out: torch.Tensor, shape, prec: str, device) -> torch.Tensor:
    """A caller-supplied output must be exactly what the kernels write: the plan's
    shape, complex dtype of the plan precision, dense, on the image's device."""
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"out shape {tuple(out.shape)} != {tuple(shape)}")
    if out.dtype != _cplx(prec):
        raise ValueError(f"out dtype {out.dtype} != {_cplx(prec)}")
    if out.device != device:
        raise ValueError(f"out is on {out.device}, image on {device}")
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")
    return out


class BankPlan:
    """Reusable bank call: descriptor built once, output [B, E, H, W] complex."""

    def __init__(self, shape, spec: BankSpec, kind, precision: str = "f32", reuse: bool = True, units=None):
        b, h, w = shape
        self.shape = (b, h, w)
        self.prec = precision
        self.desc, self._keep = bank_desc(h, w, spec, kind, precision, reuse, batch=b, units=units)
        self.entries = int(N.check(N.lib.fgb_bank_entries(C.byref(self.desc))))

    @property
    def out_shape(self):
        b, h, w = self.shape
        return (b, self.entries, h, w)

    def new_output(self, device="cuda") -> torch.Tensor:
        return torch.empty(self.out_shape, dtype=_cplx(self.prec), device=device)

    @property
    def workspace_bytes(self) -> int:
        """Device workspace the library keeps for this call (J planes, IIR scratch)."""
        return int(N.check(N.lib.fgb_bank_workspace_bytes(C.byref(self.desc))))

    def __call__(self, img: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        img = _check_img(img)
        if tuple(img.shape) != self.shape:
            raise ValueError(f"image shape {tuple(img.shape)} != plan shape {self.shape}")
        if _prec(img) != self.prec:
            raise ValueError("image dtype does not match the plan precision")
        self.desc.img.pitch = img.stride(1)
        self.desc.img.batch_stride = img.stride(0)
        out = self.new_output(img.device) if out is None else _check_out(out, self.out_shape, self.prec, img.device)
        N.check(N.lib.fgb_bank(C.byref(self.desc), C.c_void_p(img.data_ptr()), C.c_void_p(out.data_ptr()),
                               C.c_void_p(_stream(stream))))
        return out


class SdftPlan:
    """Reusable SDFT call: output [B, bins, H, W] complex (bins u-major, or compact per pair head)."""

    def __init__(self, shape, spec: SdftSpec, precision: str = "f32", heads=None):
        b, h, w = shape
        self.shape = (b, h, w)
        self.prec = precision
        self.desc, self._keep = sdft_desc(h, w, spec, precision, batch=b, heads=heads)
        self.bins = int(N.check(N.lib.fgb_sdft_bins(C.byref(self.desc))))

    @property
    def out_shape(self):
        b, h, w = self.shape
        return (b, self.bins, h, w)

    def new_output(self, device="cuda") -> torch.Tensor:
        return torch.empty(self.out_shape, dtype=_cplx(self.prec), device=device)

    @property
    def workspace_bytes(self) -> int:
        """Device workspace the library keeps for this call (J planes, IIR scratch)."""
        return int(N.check(N.lib.fgb_sdft_workspace_bytes(C.byref(self.desc))))

    def __call__(self, img: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        img = _check_img(img)
        if tuple(img.shape) != self.shape:
            raise ValueError(f"image shape {tuple(img.shape)} != plan shape {self.shape}")
        if _prec(img) != self.prec:
            raise ValueError("image dtype does not match the plan precision")
        self.desc.img.pitch = img.stride(1)
        self.desc.img.batch_stride = img.stride(0)
        out = self.new_output(img.device) if out is None else _check_out(out, self.out_shape, self.prec, img.device)
        N.check(N.lib.fgb_sdft(C.byref(self.desc), C.c_void_p(img.data_ptr()), C.c_void_p(out.data_ptr()),
                               C.c_void_p(_stream(stream))))
        return out


def compute_bank(img: torch.Tensor, spec: BankSpec, kind, reuse: bool = True, units=None) -> torch.Tensor:
    img3 = _check_img(img)
    return BankPlan(tuple(img3.shape), spec, kind, _prec(img3), reuse, units)(img3)


def sdft_full(img: torch.Tensor, spec: SdftSpec, heads=None) -> torch.Tensor:
    img3 = _check_img(img)
    return SdftPlan(tuple(img3.shape), spec, _prec(img3), heads)(img3)


def gabor_filter(img: torch.Tensor, p, kind) -> torch.Tensor:
    """One filter on a device image [H, W] (gabor.py:172-176): complex [H, W] on the device."""
    from .gabor import _filter_desc

    img3 = _check_img(img)
    b, h, w = img3.shape
    d = _filter_desc(h, w, p, kind, _prec(img3))
    d.img.pitch, d.img.batch, d.img.batch_stride = img3.stride(1), b, img3.stride(0)
    out = torch.empty((b, h, w), dtype=_cplx(_prec(img3)), device=img3.device)
    N.check(N.lib.fgb_filter(C.byref(d), C.c_void_p(img3.data_ptr()), C.c_void_p(out.data_ptr()),
                             C.c_void_p(_stream(None))))
    return out[0] if img.dim() == 2 else out


def fir_gabor(img: torch.Tensor, p, radius: float = 6.0) -> torch.Tensor:
    """GPU brute-force 2-D tap sum (oracle.py:53-66) of a device image."""
    from .gabor import _filter_desc
    from .gaussian import ExactFIR

    img3 = _check_img(img)
    b, h, w = img3.shape
    d = _filter_desc(h, w, p, ExactFIR(radius), _prec(img3))
    d.img.pitch, d.img.batch, d.img.batch_stride = img3.stride(1), b, img3.stride(0)
    out = torch.empty((b, h, w), dtype=_cplx(_prec(img3)), device=img3.device)
    N.check(N.lib.fgb_fir_gabor(C.byref(d), float(radius), C.c_void_p(img3.data_ptr()), C.c_void_p(out.data_ptr()),
                                C.c_void_p(_stream(None))))
    return out[0] if img.dim() == 2 else out


def ser_sums(approx: torch.Tensor, truth: torch.Tensor):
    """(signal_re, error_re, signal_im, error_im) of two device complex tensors,
    reduced on the GPU in fp64 (fgb_ser_sums, deterministic)."""
    if approx.shape != truth.shape:
        raise ValueError("SER operands must share dimensions")
    if approx.dtype != truth.dtype or approx.dtype not in (torch.complex64, torch.complex128):
        raise ValueError("SER operands must be complex64 or complex128 of one dtype")
    if not (approx.is_cuda and truth.is_cuda and approx.is_contiguous() and truth.is_contiguous()):
        raise ValueError("SER operands must be contiguous CUDA tensors")
    out = (C.c_double * 4)()
    dt = N.FGB_F32 if approx.dtype == torch.complex64 else N.FGB_F64
    N.check(N.lib.fgb_ser_sums(C.c_void_p(approx.data_ptr()), C.c_void_p(truth.data_ptr()), approx.numel(), dt, out,
                               C.c_void_p(_stream(None))))
    return tuple(out)
