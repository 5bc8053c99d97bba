"""The fp32 RecursiveIIR kernels (csrc/iir32.cu) restated in NumPy float64:
parallel-form sections, segment summaries, super-segment carries and their
expansion must reproduce the reference's direct-form forward/backward
recursion (the oracle's restatement of gaussian.py:215-228) to rounding.

A separate fp32 emulation bounds what the single-precision sections cost in
accuracy at the largest sigma of the BASELINE configs (SURVEY Appendix B's
direct-form fp32 recursion missed 1e-5 by up to 125x there)."""

import math

import numpy as np
import pytest

from oracle import fastgabor_oracle as O

KM, KSY = 32, 4  # samples per segment, segments per super-segment (iir32.cu)


def sections(sigma):
    B, a1, a2, a3 = O.iir_coeffs(sigma)
    q = np.roots([1.0, a1, a2, a3])
    ir = int(np.argmin(abs(q.imag)))
    ic = [k for k in range(3) if k != ir and q[k].imag > 0][0]
    qs = np.array([q[ir].real + 0j, q[ic], np.conj(q[ic])])
    c = np.array([B / np.prod([1 - qs[j] / qs[k] for j in range(3) if j != k]) for k in range(3)])
    return (B, a1, a2, a3), qs[0].real, qs[1], c[0].real, c[1]


def run(x, qr, qc, cr, cc, s0r, s0c):
    """forward sections over axis 1 from states (s0r, s0c); returns y and end states"""
    y = np.empty_like(x)
    sr, sc = s0r.copy(), s0c.copy()
    for i in range(x.shape[1]):
        sr = qr * sr + cr * x[:, i]
        sc = qc * sc + cc * x[:, i]
        y[:, i] = sr + 2 * sc.real
    return y, sr, sc


def vec(sr, sc):
    return np.stack([sr, sc.real, sc.imag], axis=-1)


def qmul(q, v):  # (r, c re, c im) state times (q_r, q_c)
    qr, qc = q
    c = qc * (v[..., 1] + 1j * v[..., 2])
    return np.stack([qr * v[..., 0], c.real, c.imag], axis=-1)


def mb_matrix(qr, qc, cr, cc, m):
    """backward-start response of a run of m samples to a forward carry-in (iir32_params)"""
    M = np.zeros((3, 3))
    for i in range(m):
        basis = np.array([qr ** (i + 1), 2 * (qc ** (i + 1)).real, -2 * (qc ** (i + 1)).imag])
        wr, wc = cr * qr ** i, cc * qc ** i
        M[0] += wr * basis
        M[1] += wc.real * basis
        M[2] += wc.imag * basis
    return M


def segmented(z, sigma):
    """iir32.cu's two passes, super-segment carries and expansion, in float64"""
    _, qr, qc, cr, cc = sections(sigma)
    nl, L = z.shape
    nseg = -(-L // KM)
    ms = [min(KM, L - j * KM) for j in range(nseg)]
    gr, gc = cr / (1 - qr), cc / (1 - qc)
    # pass 1: local forward runs -> e (end state), b (backward-start sums)
    e, b = np.zeros((nseg, nl, 3)), np.zeros((nseg, nl, 3))
    for j in range(nseg):
        x = z[:, j * KM: j * KM + ms[j]]
        s0r, s0c = (gr * z[:, 0], gc * z[:, 0]) if j == 0 else (np.zeros(nl), np.zeros(nl, complex))
        y, sr, sc = run(x, qr, qc, cr, cc, s0r, s0c)
        e[j] = vec(sr, sc)
        w = np.arange(ms[j])
        b[j] = vec(y @ (cr * qr ** w), y @ (cc * qc ** w))
    Q = [(qr ** m, qc ** m) for m in ms]
    Mb = [mb_matrix(qr, qc, cr, cc, m) for m in ms]
    # super-segments: local chains + summaries
    nS = -(-nseg // KSY)
    sloc, tloc = np.zeros_like(e), np.zeros_like(e)
    eS, bS = np.zeros((nS, nl, 3)), np.zeros((nS, nl, 3))
    for S in range(nS):
        ks = range(S * KSY, min(nseg, (S + 1) * KSY))
        r = np.zeros((nl, 3))
        for k in ks:
            sloc[k] = r
            r = qmul(Q[k], r) + e[k]
        eS[S] = r
        t = np.zeros((nl, 3))
        for k in reversed(ks):
            tloc[k] = t
            t = qmul(Q[k], t) + b[k] + sloc[k] @ Mb[k].T
        bS[S] = t
    # carries over super-segments
    mS = [sum(ms[S * KSY:(S + 1) * KSY]) for S in range(nS)]
    QS = [(qr ** m, qc ** m) for m in mS]
    MbS = [mb_matrix(qr, qc, cr, cc, m) for m in mS]
    sS, tS = np.zeros_like(eS), np.zeros_like(bS)
    r = np.zeros((nl, 3))
    for S in range(nS):
        sS[S] = r
        r = qmul(QS[S], r) + eS[S]
    yL = r[:, 0] + 2 * r[:, 1]
    t = vec(gr * yL, gc * yL)
    for S in reversed(range(nS)):
        tS[S] = t
        t = qmul(QS[S], t) + bS[S] + sS[S] @ MbS[S].T
    # expansion (QF, QB, G as iir32_params builds them) + pass 2
    out = np.empty_like(z)
    for j in range(nseg):
        S, k = divmod(j, KSY)
        K = min(KSY, nseg - S * KSY)
        sin = qmul((qr ** (KM * k), qc ** (KM * k)), sS[S]) + sloc[j]
        P = np.eye(3)
        G = np.zeros((3, 3))
        QB = (1.0, 1.0 + 0j)
        for i in range(k + 1, K):
            jj = S * KSY + i
            F = np.array([[qr ** (KM * i), 0, 0], [0, (qc ** (KM * i)).real, -(qc ** (KM * i)).imag],
                          [0, (qc ** (KM * i)).imag, (qc ** (KM * i)).real]])
            G += P @ Mb[jj] @ F
            qm = Q[jj]
            P = P @ np.array([[qm[0], 0, 0], [0, qm[1].real, -qm[1].imag], [0, qm[1].imag, qm[1].real]])
            QB = (QB[0] * qm[0], QB[1] * qm[1])
        tin = qmul(QB, tS[S]) + tloc[j] + sS[S] @ G.T
        x = z[:, j * KM: j * KM + ms[j]]
        if j == 0:
            s0r, s0c = gr * z[:, 0], gc * z[:, 0]
        else:
            s0r, s0c = sin[:, 0], sin[:, 1] + 1j * sin[:, 2]
        y, _, _ = run(x, qr, qc, cr, cc, s0r, s0c)
        u, _, _ = run(y[:, ::-1], qr, qc, cr, cc, tin[:, 0], tin[:, 1] + 1j * tin[:, 2])
        out[:, j * KM: j * KM + ms[j]] = u[:, ::-1]
    return out


def padded_lines(sigma, n, seed, omega):
    p = int(math.ceil(5 * sigma)) + 2
    img = np.random.default_rng(seed).uniform(0, 1, size=(6, n))
    xs = np.arange(-p, n + p)
    return img[:, np.clip(xs, 0, n - 1)] * np.cos(omega * xs)


@pytest.mark.parametrize("sigma,n", [(0.8, 40), (2.0, 200), (4.0, 301), (16.0, 333), (32.0, 290), (50.0, 97)])
def test_segmented_parallel_form_equals_direct_form(sigma, n):
    z = padded_lines(sigma, n, int(sigma * 10), math.pi / max(sigma, 2.0))
    ref = O.iir_lines(z, O.iir_coeffs(sigma))
    got = segmented(z, sigma)
    assert np.max(abs(got - ref)) / np.max(abs(ref)) <= 1e-10  # the fp64-build bar (near-unit poles: ~2e-11 at sigma 50)


def test_fp32_sections_error_budget_sigma32():
    """fp32 sections with poles stored as 1 - d (one FMA per pole step) stay
    ~5x inside 1e-5 at sigma = 32 for one smoothing (two per Gabor entry)."""
    sigma, n = 32.0, 256
    coef, qr, qc, cr, cc = sections(sigma)
    z = padded_lines(sigma, n, 1, math.pi / 32 * math.cos(3 * math.pi / 8))
    ref = O.iir_lines(z, coef)
    f = np.float32
    ndr, ndc, qi = f(-(1 - qr)), f(-(1 - qc.real)), f(qc.imag)
    crf, ccr, cci = f(cr), f(cc.real), f(cc.imag)

    def fma(a, b, c):  # single rounding, fp32 operands
        return (np.float64(a) * np.asarray(b, np.float64) + np.asarray(c, np.float64)).astype(f)

    def fwd(x, s0r, s0c):
        sr, scr, sci = s0r.astype(f), s0c.real.astype(f), s0c.imag.astype(f)
        y = np.empty_like(x)
        for i in range(x.shape[1]):
            xi = x[:, i]
            sr = fma(crf, xi, fma(ndr, sr, sr))
            tr = fma(ccr, xi, fma(-qi, sci, fma(ndc, scr, scr)))
            ti = fma(cci, xi, fma(qi, scr, fma(ndc, sci, sci)))
            scr, sci = tr, ti
            y[:, i] = fma(f(2), scr, sr)
        return y

    x = z.astype(f)
    y = fwd(x, (cr / (1 - qr)) * x[:, 0].astype(np.float64), (cc / (1 - qc)) * x[:, 0].astype(np.float64))
    yl = y[:, -1].astype(np.float64)
    u = fwd(y[:, ::-1].copy(), (cr / (1 - qr)) * yl, (cc / (1 - qc)) * yl)[:, ::-1]
    err = np.max(abs(u - ref)) / np.max(abs(ref))
    assert err <= 5e-6, err
