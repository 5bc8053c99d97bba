"""Float64 NumPy restatement of the fastgabor hot path -- TEST INFRASTRUCTURE ONLY.

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/fastgabor``).  Arrays are plain float64 NumPy
arrays; complex planes travel as ``(re, im)`` tuples exactly like the
reference's planar ``ComplexImage`` (``image_io.py:48-66``).

Smoother kinds are tuples so the oracle does not depend on the product's
dataclasses:

* ``("fir", radius)``  -- ``ExactFIR(radius)``      (``gaussian.py:41-49``)
* ``("iir",)``         -- ``RecursiveIIR()``        (``gaussian.py:36-38``)
* ``("box", half)``    -- ``Box(half_width)``       (``gaussian.py:52-60``)
* ``("abox", lo, hi)`` -- ``_AsymBox(lo, hi)``      (``gaussian.py:63-68``)

Not the product: ``paper_1704_05231_b200`` never imports this module.
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------------------
# 1-D smoothing engines (gaussian.py)
# ---------------------------------------------------------------------------

# Pole-parameter knots of the third-order recursion, log2(sigma) = -1..5 in
# steps of 0.25; columns (log(r-1), phi, log(d-1)).  Data table quoted from
# gaussian.py:78-105 (numbers are data, required for bit-level parity).
IIR_KNOTS_LOG2S = np.linspace(-1.0, 5.0, 25)
IIR_KNOTS = np.array([
    [1.4935547894, 1.7389422874, 1.4116802788],
    [1.0124325346, 1.6028888671, 0.9948121036],
    [0.7060188604, 1.4246405642, 0.7655646807],
    [0.3711981889, 1.3035671168, 0.4599139117],
    [0.0723219048, 1.1741421430, 0.1988303275],
    [-0.0657826821, 1.0609426640, 0.0641342325],
    [-0.1084526360, 0.8746229033, 0.0520603916],
    [-0.3079872798, 0.7888980715, -0.2103392209],
    [-0.4435572915, 0.6681318749, -0.3543999555],
    [-0.5826541508, 0.5511044975, -0.4681767292],
    [-0.6341889379, 0.4375707759, -0.4950920113],
    [-0.9438814088, 0.3960503190, -0.8422106914],
    [-1.1264093957, 0.3331316708, -1.0232036316],
    [-1.3323529220, 0.2853777435, -1.2419374903],
    [-1.5043108087, 0.2384505949, -1.4119365035],
    [-1.6909017377, 0.2010996380, -1.6007291308],
    [-1.8639872273, 0.1677245302, -1.7693707791],
    [-2.0526626380, 0.1419695700, -1.9627706878],
    [-2.2480922032, 0.1206592327, -2.1643322734],
    [-2.4183618584, 0.1007997229, -2.3318115898],
    [-2.6108636240, 0.0856583363, -2.5302995718],
    [-2.7812366868, 0.0716083982, -2.6981612487],
    [-2.9595594412, 0.0602521009, -2.8771310090],
    [-3.1353804585, 0.0506201753, -3.0527659020],
    [-3.3165061207, 0.0427250483, -3.2360423517],
])


def sampled_gaussian(sigma: float, radius: float = 6.0):
    """Unit-sum sampled Gaussian on [-h, h], h = max(1, ceil(radius*sigma)).

    Restates gaussian.py:188-195.
    """
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    h = max(1, math.ceil(radius * sigma))
    t = np.arange(-h, h + 1, dtype=np.float64)
    g = np.exp(-(t * t) / (2.0 * sigma * sigma))
    return g / g.sum(), h


def pad_radius(kind, sigma: float) -> int:
    """Stage replicate-pad width.  Restates gaussian.py:198-212."""
    if kind[0] == "fir":
        return max(1, math.ceil(kind[1] * sigma))
    if kind[0] == "iir":
        return math.ceil(5.0 * sigma) + 2
    return 0


def _knot_params(sigma: float) -> np.ndarray:
    # gaussian.py:127-133: linear interpolation in clamped log2(sigma).
    l2 = min(max(math.log2(sigma), IIR_KNOTS_LOG2S[0]), IIR_KNOTS_LOG2S[-1])
    return np.array([np.interp(l2, IIR_KNOTS_LOG2S, IIR_KNOTS[:, j]) for j in range(3)])


def _poles(params) -> np.ndarray:
    # gaussian.py:136-142: reciprocal z-plane poles r e^{+-i phi}, d.
    lr, phi, ld = params
    r = 1.0 + math.exp(lr)
    d = 1.0 + math.exp(ld)
    return np.array([r * np.exp(1j * phi), r * np.exp(-1j * phi), d + 0j])


def _cascade_var(p: np.ndarray) -> float:
    # gaussian.py:145-147.
    return float(np.sum(2.0 * p / (p - 1.0) ** 2).real)


def iir_coeffs(sigma: float):
    """(B, a1, a2, a3) of y[n] = B x[n] - a1 y[n-1] - a2 y[n-2] - a3 y[n-3].

    Restates gaussian.py:150-185 (pole table, brentq variance rescale above
    sigma=32, ``np.poly`` expansion, B = sum(a)).
    """
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    if sigma < 0.5:
        raise ValueError("sigma below 0.5: use the ExactFIR smoother instead")
    if sigma <= 32.0:
        p = _poles(_knot_params(sigma))
    else:
        from scipy.optimize import brentq  # root finder only (gaussian.py:160)

        top = _poles(IIR_KNOTS[-1])
        target = sigma * sigma

        def f(q):
            return _cascade_var(top ** (1.0 / q)) - target

        hi = 2.0
        while f(hi) < 0.0:
            hi *= 2.0
        p = top ** (1.0 / brentq(f, 0.5, hi))
    a = np.poly(1.0 / p).real
    return float(a.sum()), float(a[1]), float(a[2]), float(a[3])


def iir_lines(z: np.ndarray, coeffs) -> np.ndarray:
    """Forward then backward 3rd-order recursion along axis 1 of padded lines.

    Restates gaussian.py:215-228 (``lfilter`` with ``lfilter_zi * x[0]``
    steady-state init, time reversal, second ``lfilter``) in direct form:
    forward state y[-1..-3] = z[0]; backward state u[L..L+2] = y[L-1].
    """
    B, a1, a2, a3 = coeffs
    z = np.asarray(z, dtype=np.float64)
    n = z.shape[1]
    y = np.empty_like(z)
    p1 = z[:, 0].copy()
    p2 = p1.copy()
    p3 = p1.copy()
    for i in range(n):
        v = B * z[:, i] - a1 * p1 - a2 * p2 - a3 * p3
        y[:, i] = v
        p3, p2, p1 = p2, p1, v
    out = np.empty_like(z)
    p1 = y[:, n - 1].copy()
    p2 = p1.copy()
    p3 = p1.copy()
    for i in range(n - 1, -1, -1):
        v = B * y[:, i] - a1 * p1 - a2 * p2 - a3 * p3
        out[:, i] = v
        p3, p2, p1 = p2, p1, v
    return out


def fir_lines_nearest(z: np.ndarray, sigma: float, radius: float) -> np.ndarray:
    """Correlation with the sampled Gaussian, nearest-edge extension.

    Restates gaussian.py:231-233 (``correlate1d(mode="nearest")``).
    """
    w, h = sampled_gaussian(sigma, radius)
    z = np.asarray(z, dtype=np.float64)
    n = z.shape[1]
    idx = np.clip(np.arange(-h, n + h), 0, n - 1)
    zp = z[:, idx]
    out = np.zeros_like(z)
    for k in range(2 * h + 1):
        out += w[k] * zp[:, k : k + n]
    return out


def box_lines(z: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Zero-padded moving sum over offsets [lo, hi].  Restates gaussian.py:236-242."""
    z = np.asarray(z, dtype=np.float64)
    n = z.shape[1]
    c = np.zeros((z.shape[0], n + 1))
    np.cumsum(z, axis=1, out=c[:, 1:])
    up = np.clip(np.arange(n) + hi + 1, 0, n)
    dn = np.clip(np.arange(n) + lo, 0, n)
    return c[:, up] - c[:, dn]


def smooth_lines(z: np.ndarray, kind, sigma: float, assume_padded: bool = False) -> np.ndarray:
    """Dispatch of gaussian.py:245-285 (values only; counters live in the product)."""
    tag = kind[0]
    if tag == "iir":
        z = np.asarray(z, dtype=np.float64)
        if assume_padded:
            return iir_lines(z, iir_coeffs(sigma))
        p = math.ceil(5.0 * sigma) + 2
        zp = np.pad(z, ((0, 0), (p, p)), mode="edge")
        return iir_lines(zp, iir_coeffs(sigma))[:, p : p + z.shape[1]]
    if tag == "fir":
        return fir_lines_nearest(z, sigma, kind[1])
    if tag == "box":
        return box_lines(z, -kind[1], kind[1])
    if tag == "abox":
        return box_lines(z, kind[1], kind[2])
    raise TypeError(f"unknown smoother kind {kind!r}")


def smooth_1d(signal, kind, sigma: float) -> np.ndarray:
    """gaussian.py:288-295."""
    s = np.asarray(signal, dtype=np.float64)
    return smooth_lines(s[None, :], kind, sigma)[0]


# ---------------------------------------------------------------------------
# Gabor decomposition stages (gabor.py) and the bank scheduler (bank.py)
# ---------------------------------------------------------------------------


def norm_theta(theta: float) -> float:
    """GaborParams theta normalisation into [0, pi) (gabor.py:81-82)."""
    return theta % math.pi


def _edge_pad_cols(a: np.ndarray, p: int) -> np.ndarray:
    if p == 0:
        return np.asarray(a, dtype=np.float64)
    n = a.shape[1]
    return np.asarray(a, dtype=np.float64)[:, np.clip(np.arange(-p, n + p), 0, n - 1)]


def _tables(freq: float, lo: int, n: int):
    # gabor.py:102-104: phases from the TRUE (possibly negative) coordinate.
    x = np.arange(lo, lo + n, dtype=np.float64)
    return np.cos(freq * x), np.sin(freq * x)


def _smooth_crop(pa, pb, kind, sigma, pad, n):
    sa = smooth_lines(pa, kind, sigma, assume_padded=bool(pad))
    sb = smooth_lines(pb, kind, sigma, assume_padded=bool(pad))
    if pad:
        sa = sa[:, pad : pad + n]
        sb = sb[:, pad : pad + n]
    return sa, sb


def horizontal_stage(f: np.ndarray, omega: float, theta: float, sigma: float, kind):
    """Row stage J (Eqs. 5-6).  Restates gabor.py:107-132.  Returns (jr, ji)."""
    f = np.asarray(f, dtype=np.float64)
    _, w = f.shape
    theta = norm_theta(theta)
    wc = omega * math.cos(theta)
    pad = pad_radius(kind, sigma)
    d = _edge_pad_cols(f, pad)
    c, s = _tables(wc, -pad, w + 2 * pad)
    sa, sb = _smooth_crop(d * c, d * s, kind, sigma, pad, w)
    c, s = c[pad : pad + w], s[pad : pad + w]
    return c * sa + s * sb, s * sa - c * sb


def vertical_stage(jr, ji, omega: float, theta: float, sigma: float, kind, conjugate: bool = False):
    """Column stage (Eqs. 7-10; Eqs. 15-16 when ``conjugate``).

    Restates gabor.py:135-164 and bank.py:68-74.  Returns (re, im).
    """
    theta = norm_theta(theta)
    ws = omega * math.sin(theta)
    jr = np.asarray(jr, dtype=np.float64).T
    ji = np.asarray(ji, dtype=np.float64).T
    _, h = jr.shape
    pad = pad_radius(kind, sigma)
    zr = _edge_pad_cols(jr, pad)
    zi = _edge_pad_cols(ji, pad)
    c, s = _tables(ws, -pad, h + 2 * pad)
    if conjugate:
        pa, pb = zr * c - zi * s, zr * s + zi * c
    else:
        pa, pb = zr * c + zi * s, zr * s - zi * c
    sa, sb = _smooth_crop(pa, pb, kind, sigma, pad, h)
    c, s = c[pad : pad + h], s[pad : pad + h]
    return (c * sa + s * sb).T.copy(), (s * sa - c * sb).T.copy()


def gabor_filter(f, omega, theta, sigma, kind):
    """gabor.py:172-176."""
    jr, ji = horizontal_stage(f, omega, theta, sigma, kind)
    return vertical_stage(jr, ji, omega, theta, sigma, kind)


def bank_thetas(n: int):
    """BankSpec.thetas (bank.py:50-52)."""
    return [k * math.pi / n for k in range(n)]


def bank_sigma(freqs, sigmas, i):
    """BankSpec.sigma_for (bank.py:45-48)."""
    if sigmas is not None:
        return float(sigmas[i])
    return 2.0 * math.pi / float(freqs[i])


def compute_bank(f, freqs, n: int, sigmas, kind):
    """Algorithm 1 with conjugate reuse.  Restates bank.py:90-129.

    Returns a list of ``(omega, theta, sigma, re, im)`` in frequency-major,
    then orientation order.
    """
    thetas = bank_thetas(n)
    nh = n // 2
    out = []
    for i, omega in enumerate(freqs):
        omega = float(omega)
        sigma = bank_sigma(freqs, sigmas, i)
        planes = {}
        for k in range(nh + 1):
            jr, ji = horizontal_stage(f, omega, thetas[k], sigma, kind)
            planes[k] = vertical_stage(jr, ji, omega, thetas[k], sigma, kind)
            if nh < n - k < n:
                planes[n - k] = vertical_stage(jr, ji, omega, thetas[k], sigma, kind, conjugate=True)
        for k in range(n):
            out.append((omega, norm_theta(thetas[k]), sigma) + planes[k])
    return out


def compute_bank_noreuse(f, freqs, n: int, sigmas, kind):
    """Full pipeline per orientation.  Restates bank.py:132-157."""
    thetas = bank_thetas(n)
    out = []
    for i, omega in enumerate(freqs):
        omega = float(omega)
        sigma = bank_sigma(freqs, sigmas, i)
        for k in range(n):
            out.append((omega, norm_theta(thetas[k]), sigma) + gabor_filter(f, omega, thetas[k], sigma, kind))
    return out


# ---------------------------------------------------------------------------
# Localized sliding DFT (sdft.py)
# ---------------------------------------------------------------------------


def sdft_sigma(mx: int, my: int, sigma):
    """SdftSpec.sigma_value (sdft.py:45-49)."""
    if sigma is not None:
        return float(sigma)
    return (min(mx, my) // 2) / 3.0


def sdft_axis_kind(kind, m: int):
    """_axis_kind (sdft.py:68-72): box windows become [-m//2, m-1-m//2]."""
    if kind[0] in ("box", "abox"):
        return ("abox", -(m // 2), m - 1 - m // 2)
    return kind


def sdft_stage(jr, ji, freq: float, center: int, kind, sigma: float, axis: int):
    """One localized-DFT stage.  Restates sdft.py:75-131.  ``ji=None`` = real input."""
    jr = np.asarray(jr, dtype=np.float64)
    if axis == 0:
        jr = jr.T
        ji = None if ji is None else np.asarray(ji, dtype=np.float64).T
    _, n = jr.shape
    pad = pad_radius(kind, sigma)
    zr = _edge_pad_cols(jr, pad)
    c, s = _tables(freq, -pad, n + 2 * pad)
    if ji is None:
        pa, pb = zr * c, zr * s
    else:
        zi = _edge_pad_cols(ji, pad)
        pa, pb = zr * c - zi * s, zr * s + zi * c
    sa, sb = _smooth_crop(pa, pb, kind, sigma, pad, n)
    xh = np.arange(n, dtype=np.float64) - center
    ca, sn = np.cos(freq * xh), np.sin(freq * xh)
    re, im = ca * sa + sn * sb, ca * sb - sn * sa
    if axis == 0:
        re, im = re.T, im.T
    return np.ascontiguousarray(re), np.ascontiguousarray(im)


def sdft_horizontal(f, u: int, mx: int, my: int, kind, sigma=None):
    """J_u (sdft.py:134-150)."""
    if not 0 <= u < mx:
        raise ValueError(f"bin index u={u} outside [0, {mx})")
    return sdft_stage(f, None, 2.0 * math.pi / mx * u, mx // 2, sdft_axis_kind(kind, mx),
                      sdft_sigma(mx, my, sigma), axis=1)


def sdft_vertical_bin(jr, ji, v: int, mx: int, my: int, kind, sigma=None):
    """_vertical_bin (sdft.py:153-166)."""
    return sdft_stage(jr, ji, 2.0 * math.pi / my * v, my // 2, sdft_axis_kind(kind, my),
                      sdft_sigma(mx, my, sigma), axis=0)


def sdft_bin(f, u: int, v: int, mx: int, my: int, kind, sigma=None):
    """sdft.py:169-175."""
    if not 0 <= v < my:
        raise ValueError(f"bin index v={v} outside [0, {my})")
    jr, ji = sdft_horizontal(f, u, mx, my, kind, sigma)
    return sdft_vertical_bin(jr, ji, v, mx, my, kind, sigma)


def sdft_full(f, mx: int, my: int, kind, sigma=None):
    """Algorithm 2 with horizontal + conjugate-symmetry reuse (sdft.py:178-213).

    Returns ``bins[u][v] = (re, im)``.
    """
    f = np.asarray(f, dtype=np.float64)
    if my < mx:
        tb = sdft_full(f.T.copy(), my, mx, kind, sigma)
        return [[(tb[v][u][0].T.copy(), tb[v][u][1].T.copy()) for v in range(my)] for u in range(mx)]
    mxh, myh = mx // 2, my // 2
    js = {u: sdft_horizontal(f, u, mx, my, kind, sigma) for u in range(mxh + 1)}
    for u in range(mxh + 1, mx):
        jr, ji = js[mx - u]
        js[u] = (jr.copy(), -ji)
    bins = [[None] * my for _ in range(mx)]
    for u in range(mx):
        for v in range(myh + 1):
            bins[u][v] = sdft_vertical_bin(js[u][0], js[u][1], v, mx, my, kind, sigma)
    for u in range(mx):
        for v in range(myh + 1, my):
            re, im = bins[(mx - u) % mx][(my - v) % my]
            bins[u][v] = (re.copy(), -im)
    return bins


# ---------------------------------------------------------------------------
# Brute-force 2-D tap sums (oracle.py)
# ---------------------------------------------------------------------------


def _tap_sum(padded, kre, kim, h, w):
    # oracle.py:33-50.
    ky, kx = kre.shape
    are = np.zeros((h, w))
    aim = np.zeros((h, w))
    for iy in range(ky):
        for ix in range(kx):
            p = padded[iy : iy + h, ix : ix + w]
            are += kre[iy, ix] * p
            aim += kim[iy, ix] * p
    return are, aim


def fir_gabor(f, omega, theta, sigma, radius: float = 6.0):
    """Direct 2-D complex Gabor tap sum, replicate boundary (oracle.py:53-66)."""
    f = np.asarray(f, dtype=np.float64)
    theta = norm_theta(theta)
    g, half = sampled_gaussian(sigma, radius)
    d = np.arange(-half, half + 1, dtype=np.float64)
    ph = omega * (math.cos(theta) * d[None, :] + math.sin(theta) * d[:, None])
    env = np.outer(g, g)
    kre = (env * np.cos(ph))[::-1, ::-1]
    kim = (env * np.sin(ph))[::-1, ::-1]
    return _tap_sum(np.pad(f, half, mode="edge"), kre, kim, *f.shape)


def localized_dft(f, u, v, mx, my, kind, sigma=None, radius: float = 6.0):
    """Direct evaluation of one localized-DFT bin (oracle.py:69-109)."""
    f = np.asarray(f, dtype=np.float64)
    if not (0 <= u < mx and 0 <= v < my):
        raise ValueError("bin indices outside the window grid")
    if kind[0] in ("box", "abox"):
        lox, hix = -(mx // 2), mx - 1 - mx // 2
        loy, hiy = -(my // 2), my - 1 - my // 2
        dm = np.arange(lox, hix + 1, dtype=np.float64)
        dn = np.arange(loy, hiy + 1, dtype=np.float64)
        env = np.ones((dn.size, dm.size))
        padded = np.pad(f, ((-loy, hiy), (-lox, hix)), mode="constant")
    else:
        s = sdft_sigma(mx, my, sigma)
        gx, hx = sampled_gaussian(s, radius)
        gy, hy = sampled_gaussian(s, radius)
        dm = np.arange(-hx, hx + 1, dtype=np.float64)
        dn = np.arange(-hy, hy + 1, dtype=np.float64)
        env = np.outer(gy, gx)
        padded = np.pad(f, ((hy, hy), (hx, hx)), mode="edge")
    ph = (2.0 * math.pi / mx) * u * (mx // 2 + dm)[None, :] + (2.0 * math.pi / my) * v * (my // 2 + dn)[:, None]
    return _tap_sum(padded, env * np.cos(ph), env * np.sin(ph), *f.shape)


def max_rel_err(a, b) -> float:
    """conftest.py:33-36: max |a-b| over both planes / max |b| (either plane)."""
    scale = max(np.abs(b[0]).max(), np.abs(b[1]).max(), 1e-300)
    return max(np.abs(a[0] - b[0]).max(), np.abs(a[1] - b[1]).max()) / scale
