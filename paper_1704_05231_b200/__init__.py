"""B200-native fastgabor hot path: 2-D complex Gabor filter bank with kernel
decomposition + theta/pi-theta conjugate reuse, and the Gaussian-windowed
localized sliding DFT (arXiv 1704.05231), as sm_100a CUDA behind the
reference package's own entry points.

Drop-in surface (same names/signatures as fastgabor/__init__.py:11-80 for the
hot path): ``compute_bank``, ``compute_bank_noreuse``, ``gabor_filter``,
``horizontal_stage``, ``vertical_stage``, ``vertical_stage_conjugate``,
``sdft_full``, ``sdft_bin``, ``sdft_horizontal``, ``smooth_lines``,
``smooth_1d``, ``smooth_pair_1d`` plus their types.  Every
call crosses the C ABI of ``lib/libfgb200.so`` (include/fgb200.h); there is no
CPU fallback.  ``paper_1704_05231_b200.device`` is the device-tensor API used
for throughput runs.
"""

from ._precision import get_precision, set_precision
from .image_io import (
    ComplexImage,
    ContainerFormatError,
    ImageFormatError,
    RealImage,
    load_grayscale,
    read_bank_container,
    write_bank_container,
    write_container_from_device,
    write_magnitude,
)
from .gaussian import (
    Box,
    ExactFIR,
    GaussianCoeffs,
    RecursiveIIR,
    SmootherKind,
    make_coeffs,
    pad_radius,
    sampled_gaussian,
    smooth_1d,
    smooth_lines,
    smooth_pair_1d,
)
from .gabor import GaborParams, HorizontalStage, gabor_filter, horizontal_stage, vertical_stage
from .bank import (
    BankOutput,
    BankSpec,
    compute_bank,
    compute_bank_noreuse,
    conjugate_image,
    vertical_stage_conjugate,
)
from .sdft import SdftOutput, SdftSpec, sdft_bin, sdft_full, sdft_horizontal
from .metrics import OpCounters, SerReport, fit_affine, fit_features, per_pixel_counts, ser, ser_report
from .bruteforce import OracleConfig, fir_gabor, localized_dft

__all__ = [
    "RealImage",
    "ComplexImage",
    "RecursiveIIR",
    "ExactFIR",
    "Box",
    "GaussianCoeffs",
    "SmootherKind",
    "make_coeffs",
    "sampled_gaussian",
    "pad_radius",
    "smooth_lines",
    "smooth_1d",
    "smooth_pair_1d",
    "GaborParams",
    "HorizontalStage",
    "horizontal_stage",
    "vertical_stage",
    "gabor_filter",
    "BankSpec",
    "BankOutput",
    "conjugate_image",
    "vertical_stage_conjugate",
    "compute_bank",
    "compute_bank_noreuse",
    "SdftSpec",
    "SdftOutput",
    "sdft_horizontal",
    "sdft_bin",
    "sdft_full",
    "OpCounters",
    "per_pixel_counts",
    "SerReport",
    "ser",
    "ser_report",
    "fit_affine",
    "fit_features",
    "OracleConfig",
    "fir_gabor",
    "localized_dft",
    "load_grayscale",
    "write_magnitude",
    "write_bank_container",
    "read_bank_container",
    "write_container_from_device",
    "ImageFormatError",
    "ContainerFormatError",
    "set_precision",
    "get_precision",
]
