"""Generate golden vectors by running the REFERENCE fastgabor package.

Runs only in the build container, where the read-only reference is mounted
at /root/reference (it does not exist on the GPU box).  Output:
``tests/golden/golden.npz`` (float64 arrays) and ``tests/golden/golden.json``
(scalars: counters, coefficient KATs, case metadata).

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Every case uses seeded inputs (``np.random.default_rng(seed).uniform``, the
generator family of the reference's conftest.py:9-11).
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import fastgabor as fg  # noqa: E402  (the reference itself)

arrays: dict[str, np.ndarray] = {}
meta: dict = {"cases": {}, "coeffs": {}, "gauss": {}}


def kind_obj(k):
    if k[0] == "fir":
        return fg.ExactFIR(k[1])
    if k[0] == "iir":
        return fg.RecursiveIIR()
    if k[0] == "box":
        return fg.Box(k[1])
    raise ValueError(k)


def ctr(c: fg.OpCounters):
    return [c.multiplications, c.additions, c.smoothings_h, c.smoothings_v]


def img(seed, h, w, lo=0.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, size=(h, w))


def put(name, ci):
    arrays[name + ".re"] = np.ascontiguousarray(ci.re)
    arrays[name + ".im"] = np.ascontiguousarray(ci.im)


KINDS = {"fir6": ("fir", 6.0), "fir3": ("fir", 3.0), "iir": ("iir",)}

# 1. IIR coefficient KATs (gaussian.py:164-185) and sampled Gaussians.
for s in (0.5, 0.6, 0.8, 1.0, 1.2, 1.5, 1.61, 2.0, 2.5, 3.0, 4.0, 6.0, 8.0, 10.0, 16.0, 24.0, 32.0, 40.0, 50.0):
    c = fg.make_coeffs(s)
    meta["coeffs"][repr(s)] = [c.B, -c.b1, -c.b2, -c.b3]
for s, r in ((0.5, 6.0), (1.2, 6.0), (2.0, 3.0), (4.0, 3.0), (32.0, 3.0), (3.7, 6.0)):
    k, h = fg.sampled_gaussian(s, r)
    arrays[f"gauss.{s}.{r}"] = k
    meta["gauss"][f"{s}.{r}"] = h

# 2. smooth_1d on a raw signal for every kind (gaussian.py:288-295).
sig = np.random.default_rng(7).normal(size=61)
arrays["smooth.in"] = sig
for name, k in list(KINDS.items()) + [("box2", ("box", 2))]:
    for s in (0.8, 2.0, 5.0):
        if k[0] == "iir" and s < 0.5:
            continue
        arrays[f"smooth.{name}.{s}"] = fg.smooth_1d(sig, kind_obj(k), s, fg.OpCounters())

# 3. Single filters: horizontal stage, vertical stage (+conjugate), full filter.
f1 = img(11, 32, 40, 0.0, 255.0)
arrays["f1"] = f1
single = [(2.0, 0.3, 1.2), (0.5, 2.0, 4.0), (3.0, math.pi / 2, 2.0), (1.0, 0.0, 0.7), (5.0, 2.5, 0.6), (math.pi / 4, 3 * math.pi / 4, 4.0)]
for kn, k in KINDS.items():
    for i, (om, th, sg) in enumerate(single):
        if k[0] == "iir" and sg < 0.5:
            continue
        p = fg.GaborParams(om, th, sg)
        c = fg.OpCounters()
        h = fg.horizontal_stage(fg.RealImage.from_array(f1), p, kind_obj(k), c)
        put(f"hstage.{kn}.{i}", h.j)
        out = fg.vertical_stage(h, c)
        put(f"gabor.{kn}.{i}", out)
        conj = fg.vertical_stage_conjugate(h, fg.OpCounters())
        put(f"vconj.{kn}.{i}", conj)
        meta["cases"][f"gabor.{kn}.{i}"] = {"params": [om, th, sg], "counters": ctr(c), "theta_norm": p.theta}

# 4. Banks with reuse and without (bank.py:90-157).
f2 = img(22, 16, 20, 0.0, 255.0)
arrays["f2"] = f2
banks = {
    "b7": ((3.0, 1.0), 7, None),
    "b8": ((math.pi / 2, math.pi / 4), 8, (2.0, 4.0)),
    "b1": ((2.0,), 1, None),
    "b2": ((3.0,), 2, None),
    "b16": ((math.pi / 2,), 16, (2.0,)),
}
for kn, k in KINDS.items():
    for bn, (freqs, n, sig_) in banks.items():
        spec = fg.BankSpec(freqs, n, sig_)
        for tag, fn in (("reuse", fg.compute_bank), ("noreuse", fg.compute_bank_noreuse)):
            if tag == "noreuse" and bn not in ("b7", "b2"):
                continue
            c = fg.OpCounters()
            out = fn(fg.RealImage.from_array(f2), spec, kind_obj(k), c)
            for e, (p, ci) in enumerate(out.entries):
                put(f"bank.{kn}.{bn}.{tag}.{e}", ci)
            meta["cases"][f"bank.{kn}.{bn}.{tag}"] = {
                "freqs": list(freqs), "n": n, "sigmas": None if sig_ is None else list(sig_),
                "entries": [[p.omega, p.theta, p.sigma] for p, _ in out.entries],
                "counters": ctr(c),
            }

# 5. BASELINE config 1 exactly (256x256 f64 seed 0, omega=pi/4, N=4, sigma=4, FIR r=3),
#    stored as a strided sub-sample plus the four border lines (size budget).
f_cfg1 = np.random.default_rng(0).uniform(0.0, 1.0, size=(256, 256))
c = fg.OpCounters()
out = fg.compute_bank(fg.RealImage.from_array(f_cfg1), fg.BankSpec((math.pi / 4,), 4, (4.0,)), fg.ExactFIR(3.0), c)
for e, (p, ci) in enumerate(out.entries):
    for part in ("re", "im"):
        a = getattr(ci, part)
        arrays[f"cfg1.{e}.{part}.sub"] = a[::5, ::5].copy()
        arrays[f"cfg1.{e}.{part}.rows"] = a[[0, 1, 254, 255], :].copy()
        arrays[f"cfg1.{e}.{part}.cols"] = a[:, [0, 1, 254, 255]].copy()
meta["cases"]["cfg1"] = {"entries": [[p.omega, p.theta, p.sigma] for p, _ in out.entries], "counters": ctr(c)}

# 6. Localized SDFT (sdft.py:134-213): square, wide, tall windows, every kind.
f3 = img(33, 10, 12, 0.0, 255.0)
arrays["f3"] = f3
sdfts = {"s44": (4, 4, None), "s84": (8, 4, None), "s46": (4, 6, None), "s88": (8, 8, 1.5), "s1616": (16, 16, 4.0)}
for kn, k in list(KINDS.items()) + [("box1", ("box", 1))]:
    for sn, (mx, my, sg) in sdfts.items():
        if sn == "s1616" and kn != "fir3":
            continue
        spec = fg.SdftSpec(mx, my, kind_obj(k), sg)
        c = fg.OpCounters()
        out = fg.sdft_full(fg.RealImage.from_array(f3), spec, c)
        for u in range(mx):
            for v in range(my):
                put(f"sdft.{kn}.{sn}.{u}.{v}", out.bins[u][v])
        meta["cases"][f"sdft.{kn}.{sn}"] = {"mx": mx, "my": my, "sigma": sg, "counters": ctr(c)}
        cb = fg.OpCounters()
        put(f"sdftbin.{kn}.{sn}", fg.sdft_bin(fg.RealImage.from_array(f3), 1, my - 1, spec, cb))
        meta["cases"][f"sdftbin.{kn}.{sn}"] = {"u": 1, "v": my - 1, "counters": ctr(cb)}
        ch = fg.OpCounters()
        put(f"sdfth.{kn}.{sn}", fg.sdft_horizontal(fg.RealImage.from_array(f3), mx - 1, spec, ch))
        meta["cases"][f"sdfth.{kn}.{sn}"] = {"u": mx - 1, "counters": ctr(ch)}

# 7. Brute-force oracles (oracle.py:53-109).
for i, (om, th, sg) in enumerate(single[:3]):
    put(f"firgabor.{i}", fg.fir_gabor(fg.RealImage.from_array(f1), fg.GaborParams(om, th, sg)))
for kn, k in (("fir6", ("fir", 6.0)), ("box1", ("box", 1))):
    spec = fg.SdftSpec(4, 4, kind_obj(k))
    put(f"ldft.{kn}", fg.localized_dft(fg.RealImage.from_array(f3), 1, 3, spec))
# 7b. Large supports at the configs' radius 3 (sigma 16 / 32: 97^2 / 193^2 taps, larger
#     than the image), the case the GPU brute force runs as banded kernel rows.
f7 = img(17, 120, 136)
arrays["f7"] = f7
for i, (om, th, sg) in enumerate(((math.pi / 16, 3 * math.pi / 8, 16.0), (math.pi / 32, 13 * math.pi / 16, 32.0))):
    put(f"firgabor_r3.{i}", fg.fir_gabor(fg.RealImage.from_array(f7), fg.GaborParams(om, th, sg), fg.OracleConfig(3.0)))
    meta["cases"][f"firgabor_r3.{i}"] = {"params": [om, th, sg]}
put("ldft_r3", fg.localized_dft(fg.RealImage.from_array(f7), 5, 27, fg.SdftSpec(32, 32, fg.ExactFIR(3.0), 16.0),
                                fg.OracleConfig(3.0)))

# 8. I/O and metrics (image_io.py:136-212, metrics.py:63-83): bytes written by the
#    reference for known inputs, SER of known pairs.
import tempfile  # noqa: E402

_ents = [(fg.GaborParams(1.0 + i, 0.3 * i, 2.0), fg.ComplexImage.from_planes(f3 * (i + 1), -f3 / (i + 2)))
         for i in range(3)]
with tempfile.TemporaryDirectory() as td:
    pth = os.path.join(td, "b.gbnk")
    fg.write_bank_container(_ents, pth)
    arrays["io.gbnk_bytes"] = np.frombuffer(open(pth, "rb").read(), dtype=np.uint8).copy()
    fg.write_bank_container([((1.0, 2.0, 0.5), _ents[0][1])], pth, sdft=True)
    arrays["io.gbnk_sdft_bytes"] = np.frombuffer(open(pth, "rb").read(), dtype=np.uint8).copy()
    pg = os.path.join(td, "m.pgm")
    fg.write_magnitude(_ents[1][1], pg)
    arrays["io.magnitude_pgm_bytes"] = np.frombuffer(open(pg, "rb").read(), dtype=np.uint8).copy()
_a, _b = _ents[0][1], fg.ComplexImage.from_planes(f3 * 1.01 + 0.3, -f3 / 2 + 0.01)
meta["ser"] = {"real": fg.ser(_b, _a, "real"), "imag": fg.ser(_b, _a, "imag")}

np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
with open(os.path.join(HERE, "golden.json"), "w") as fh:
    json.dump(meta, fh, indent=1, sort_keys=True)
print(f"wrote {len(arrays)} arrays, {os.path.getsize(os.path.join(HERE, 'golden.npz')) / 1e6:.2f} MB")
