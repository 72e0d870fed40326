"""Pins of the f1 oracle: the fidelity loss of Eq. 3 with
D-SSIM = 1 − SSIM (A39), 11×11 Gaussian window σ = 1.5, zero padding."""

import numpy as np
import pytest

import oracle

scipy_nd = pytest.importorskip("scipy.ndimage")


def _img(seed, H=20, W=27, lo=0.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, size=(3, H, W)).astype(np.float32)


def _ssim_scipy(a, b):
    """Independent windowed SSIM: scipy.ndimage.correlate, constant (zero) mode."""
    k = np.exp(-((np.arange(11) - 5) ** 2) / (2 * 1.5 ** 2))
    k /= k.sum()
    w = np.outer(k, k)
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    vals = []
    for ch in range(3):
        x, y = a[ch].astype(np.float64), b[ch].astype(np.float64)
        f = lambda z: scipy_nd.correlate(z, w, mode="constant", cval=0.0)
        m1, m2 = f(x), f(y)
        v1, v2, v12 = f(x * x) - m1 ** 2, f(y * y) - m2 ** 2, f(x * y) - m1 * m2
        s = ((2 * m1 * m2 + C1) * (2 * v12 + C2)) / ((m1 ** 2 + m2 ** 2 + C1) * (v1 + v2 + C2))
        vals.append(s)
    return float(np.mean(vals))


def test_identical_images_and_symmetry():
    a, b = _img(1), _img(2)
    L, l1, ssim, _ = oracle.fidelity_loss(a, a, 0.2)
    assert l1 == 0.0 and ssim == pytest.approx(1.0, abs=1e-12) and L == pytest.approx(0.0, abs=1e-12)
    assert oracle.fidelity_loss(a, b)[2] == pytest.approx(oracle.fidelity_loss(b, a)[2], abs=1e-12)


def test_l1_only_and_ssim_against_independent_scipy():
    a, b = _img(3), _img(4)
    L, l1, ssim, g = oracle.fidelity_loss(a, b, 0.0)
    assert l1 == pytest.approx(np.abs(a.astype(np.float64) - b).mean(), rel=1e-12)
    assert L == pytest.approx(l1, rel=1e-12)
    np.testing.assert_allclose(g, np.sign(a.astype(np.float64) - b) / a.size, atol=1e-18)
    assert ssim == pytest.approx(_ssim_scipy(a, b), rel=1e-10)
    c = np.clip(a + np.float32(0.1), 0, 2).astype(np.float32)                 # S:266 example shape
    assert oracle.fidelity_loss(a, c, 1.0)[2] == pytest.approx(_ssim_scipy(a, c), rel=1e-10)


def test_gradient_central_differences():
    a, b = _img(5, 9, 11), _img(6, 9, 11)
    lam = 0.3
    L0, _, _, g = oracle.fidelity_loss(a, b, lam)
    rng = np.random.default_rng(7)
    for _ in range(40):
        ch, y, x = rng.integers(3), rng.integers(9), rng.integers(11)
        if abs(float(a[ch, y, x]) - float(b[ch, y, x])) < 1e-2:
            continue  # |·| kink
        h = 1e-3
        ap, am = a.copy(), a.copy()
        ap[ch, y, x] += np.float32(h); am[ch, y, x] -= np.float32(h)
        dh = float(ap[ch, y, x]) - float(am[ch, y, x])
        fd = (oracle.fidelity_loss(ap, b, lam, grad=False)[0] - oracle.fidelity_loss(am, b, lam, grad=False)[0]) / dh
        assert abs(fd - g[ch, y, x]) <= 1e-5 * max(abs(g[ch, y, x]), 1e-3), (ch, y, x, fd, g[ch, y, x])


def test_spec_example_dssim_half_scale():
    """λ = 1, identical images shifted by a constant 0.1 → the loss
    equals D-SSIM = (1 − SSIM)/2 with SSIM from an independently coded windowed
    reference, to 1e-6 (dssim_scale = 0.5; A39's default 1 gives 1 − SSIM)."""
    a = _img(5, lo=0.1, hi=0.8)
    b = (a + 0.1).astype(np.float32)
    ref = _ssim_scipy(a, b)
    L_half, _, ssim, g_half = oracle.fidelity_loss(a, b, 1.0, dssim_scale=0.5)
    assert ssim == pytest.approx(ref, abs=1e-9)
    assert L_half == pytest.approx((1 - ref) / 2, abs=1e-6)
    L_one, _, _, g_one = oracle.fidelity_loss(a, b, 1.0)
    assert L_one == pytest.approx(1 - ref, abs=1e-6)
    np.testing.assert_allclose(g_half, 0.5 * g_one, rtol=1e-12, atol=0)
