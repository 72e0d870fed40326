"""Pins of the oracle's geometry (O2, O2-key) against mathematics and the
SPEC/paper examples — nothing here re-types the oracle's own formulas.

P:341 Eq. 6 (Σ = R S Sᵀ Rᵀ), Eq. 7 (EWA), P:351 (view-dependent colour),
S:42-80 (core-geometry examples), include/dass.h KEY CHAIN.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2411_14847_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _sandwich(q, v):
    """Rotate v by unit quaternion q via the quaternion sandwich q v q*,
    written with the Hamilton product as a 4x4 left-multiplication matrix."""
    def L(a):
        w, x, y, z = a
        return np.array([[w, -x, -y, -z], [x, w, -z, y], [y, z, w, -x], [z, -y, x, w]])
    qc = q * np.array([1, -1, -1, -1])
    return (L(L(q) @ np.r_[0.0, v]) @ qc)[1:]


@pytest.mark.parametrize("ex", GOLD["quat_to_rotmat"])
def test_rotmat_spec_examples(ex):
    R, _ = oracle.rotmat_cov(np.array(ex["q"], np.float32), np.ones(3, np.float32))
    np.testing.assert_allclose(R, ex["R"], atol=1e-15)


def test_rotmat_matches_sandwich_and_is_rotation():
    g = np.random.default_rng(0)
    for _ in range(50):
        q = g.normal(size=4).astype(np.float32)
        R, _ = oracle.rotmat_cov(q, np.ones(3, np.float32))
        qh = q.astype(np.float64) / np.linalg.norm(q.astype(np.float64))
        for e in np.eye(3):
            np.testing.assert_allclose(R @ e, _sandwich(qh, e), atol=1e-12)
        np.testing.assert_allclose(R.T @ R, np.eye(3), atol=1e-12)
        assert abs(np.linalg.det(R) - 1) < 1e-12


@pytest.mark.parametrize("ex", GOLD["build_covariance"])
def test_covariance_spec_examples(ex):
    _, S = oracle.rotmat_cov(np.array(ex["q"], np.float32), np.array(ex["scale"], np.float32))
    np.testing.assert_allclose(S, ex["Sigma"], atol=1e-12)


def test_covariance_eigen():
    """Eigenvalues of Σ = s² as a multiset, eigenvectors the columns of R."""
    g = np.random.default_rng(1)
    for _ in range(50):
        q = g.normal(size=4).astype(np.float32)
        s = g.uniform(0.1, 3.0, size=3).astype(np.float32)
        R, S = oracle.rotmat_cov(q, s)
        w = np.linalg.eigvalsh(S)
        np.testing.assert_allclose(np.sort(w), np.sort(s.astype(np.float64) ** 2), rtol=1e-10, atol=1e-12)
        for k in range(3):
            np.testing.assert_allclose(S @ R[:, k], float(s[k]) ** 2 * R[:, k], atol=1e-10)


def _one(pos, scale, rot=(1, 0, 0, 0), opa=0.9):
    pos_opa = np.array([[*pos, opa]], np.float32)
    sc = np.array([[*scale, 0]], np.float32)
    r = np.array([rot], np.float32)
    return pos_opa, sc, r


def test_ewa_on_axis_isotropic_exact():
    """W = I, on-axis isotropic σ²I at depth d: Σ' = diag(fx²σ²/d², fy²σ²/d²) + 0.3 I
    exactly (J's third column vanishes on axis) — Eq. 7."""
    cam = synth.Camera(640, 480, 500.0, 420.0, 319.5, 239.5,
                       np.concatenate([np.eye(3), np.zeros((3, 1))], 1).astype(np.float32))
    for d, s in [(2.0, 0.01), (5.0, 0.3), (3.0, 0.05)]:
        po, sc, r = _one((0, 0, d), (s, s, s))
        a, b, c, det = oracle.cov2d(cam, po, sc, r)[0]
        sd = float(np.float32(s))
        dd = float(np.float32(d))
        assert a == pytest.approx(500.0 ** 2 * sd ** 2 / dd ** 2 + 0.3, rel=1e-13)
        assert c == pytest.approx(420.0 ** 2 * sd ** 2 / dd ** 2 + 0.3, rel=1e-13)
        assert abs(b) < 1e-12


def test_ewa_zero_covariance_is_lowpass_floor():
    """Σ = 0 → Σ' = diag(0.3, 0.3)."""
    cam = synth.n3dv_rig()[3]
    po, sc, r = _one((0.3, -0.2, 4.0), (0, 0, 0))
    a, b, c, det = oracle.cov2d(cam, po, sc, r)[0]
    assert a == pytest.approx(0.3, abs=1e-15) and c == pytest.approx(0.3, abs=1e-15)
    assert abs(b) < 1e-15


def _fd_jacobian(cam, p):
    """Finite-difference Jacobian of the pinhole map world p → (u, v)."""
    V = cam.viewmat.astype(np.float64)

    def proj(x):
        t = V[:, :3] @ x + V[:, 3]
        fx, fy, cx, cy = (float(np.float32(x)) for x in (cam.fx, cam.fy, cam.cx, cam.cy))
        return np.array([fx * t[0] / t[2] + cx, fy * t[1] / t[2] + cy])

    J = np.zeros((2, 3))
    for k in range(3):
        h = 1e-5
        e = np.zeros(3); e[k] = h
        J[:, k] = (proj(p + e) - proj(p - e)) / (2 * h)
    return J   # this is J·W of Eq. 7 in world coordinates


def test_ewa_matches_fd_jacobian_rotated_camera():
    """Σ' = (J W) Σ (J W)ᵀ + 0.3 I with J W from finite differences of the
    pinhole projection, for points inside the guard band (Eq. 7)."""
    cams = synth.n3dv_rig()
    g = np.random.default_rng(3)
    for cam in cams[:5]:
        for _ in range(10):
            t = np.array([g.uniform(-0.4, 0.4), g.uniform(-0.3, 0.3), 1.0]) * g.uniform(2, 8)
            V = cam.viewmat.astype(np.float64)
            p = V[:, :3].T @ (t - V[:, 3])
            q = g.normal(size=4)
            s = g.uniform(0.01, 0.2, size=3)
            po, sc, r = _one(p, s, q)
            a, b, c, det = oracle.cov2d(cam, po, sc, r)[0]
            R, S = oracle.rotmat_cov(r[0], sc[0, :3])
            JW = _fd_jacobian(cam, po[0, :3].astype(np.float64))
            S2 = JW @ S @ JW.T + 0.3 * np.eye(2)
            np.testing.assert_allclose([a, b, c], [S2[0, 0], S2[0, 1], S2[1, 1]], rtol=1e-6,
                                       atol=1e-6 * abs(S2).max())
            assert det == pytest.approx(np.linalg.det(S2), rel=1e-6)


def test_project_mean_is_pinhole_and_depth_is_camera_z():
    """u, v = pinhole projection; z = camera-frame z (A02)."""
    cams = synth.n3dv_rig()
    cam = cams[11]
    sc = synth.n3dv_scene(n=2000, seed=11)
    pr = oracle.project(cam, sc)
    V = cam.viewmat.astype(np.float64)
    t = sc.pos_opa[:, :3].astype(np.float64) @ V[:, :3].T + V[:, 3]
    vis = pr["visible"] == 1
    assert vis.sum() > 1000
    np.testing.assert_allclose(pr["uvz"][vis, 2], t[vis, 2], rtol=1e-14)
    fx, fy, cx, cy = (float(np.float32(x)) for x in (cam.fx, cam.fy, cam.cx, cam.cy))
    np.testing.assert_allclose(pr["uvz"][vis, 0], fx * t[vis, 0] / t[vis, 2] + cx, rtol=1e-12)
    np.testing.assert_allclose(pr["uvz"][vis, 1], fy * t[vis, 1] / t[vis, 2] + cy, rtol=1e-12)
    # the fp32 key replica depth is the float32 rounding of the exact depth
    # up to the rounding of a 4-op fp32 chain (a few ulp)
    zf = pr["zf"][vis].astype(np.float64)
    assert np.all(np.abs(zf - t[vis, 2]) <= 4 * np.spacing(np.float32(zf)).astype(np.float64))
    assert np.array_equal(pr["zbits"][vis], pr["zf"][vis].view(np.uint32))
    # culled: behind the near plane (A09)
    assert not np.any(pr["visible"][t[:, 2] <= cam.near])


def test_project_box_and_tiles_brute_force():
    """Pixel box = integer pixels within r = ceil(3 sqrt(λ_max)) of (u, v),
    clipped to the image (A05/A06); tiles_touched = count of 16×16 tiles
    intersecting it (A04) — recomputed here from the double eigenvalues."""
    cams = synth.n3dv_rig()
    cam = cams[2]
    sc = synth.n3dv_scene(n=3000, seed=12)
    pr = oracle.project(cam, sc)
    ab = oracle.cov2d(cam, sc.pos_opa, sc.scale, sc.rot)
    vis = np.nonzero(pr["visible"])[0]
    nties = 0
    for i in vis:
        a, b, c, det = ab[i]
        lam = np.linalg.eigvalsh(np.array([[a, b], [b, c]]))[1]
        mid = 0.5 * (a + c)
        lam_r = mid + math.sqrt(max(0.1, mid * mid - det))  # = λmax unless the 0.1 floor binds
        if mid * mid - det >= 0.1:
            assert lam_r == pytest.approx(lam, rel=1e-9)
        r_exact = 3 * math.sqrt(lam_r)
        if abs(r_exact - round(r_exact)) < 1e-4:
            nties += 1
            continue
        r = math.ceil(r_exact)
        u, v = pr["uvz"][i, 0], pr["uvz"][i, 1]
        if min(abs(u - r - round(u - r)), abs(v - r - round(v - r))) < 1e-3:
            nties += 1
            continue
        x0 = max(0, math.ceil(u - r)); x1 = min(cam.width - 1, math.floor(u + r))
        y0 = max(0, math.ceil(v - r)); y1 = min(cam.height - 1, math.floor(v + r))
        assert list(pr["box"][i]) == [x0, x1, y0, y1]
        # the A50 footprint keeps a subset of the box's tiles
        assert 1 <= pr["tiles"][i] <= (x1 // 16 - x0 // 16 + 1) * (y1 // 16 - y0 // 16 + 1) or \
            pr["tiles"][i] == 0
    assert nties < 0.01 * len(vis)


def footprint_tiles(pr, i, tiles_x):
    """Decode Gaussian i's A50 row spans (include/dass.h KEY CHAIN step 13)."""
    x0, x1, y0, y1 = pr["box"][i]
    tx0, tx1, ty0, ty1 = x0 // 16, x1 // 16, y0 // 16, y1 // 16
    rows = pr["rows"][i]
    if np.all(rows == 0xFFFFFFFF):
        return {(ty, tx) for ty in range(ty0, ty1 + 1) for tx in range(tx0, tx1 + 1)}
    out = set()
    for k, ty in enumerate(range(ty0, ty1 + 1)):
        span = (int(rows[k >> 1]) >> (16 * (k & 1))) & 0xFFFF
        lo, hi = span & 0xFF, span >> 8
        out |= {(ty, tx0 + j) for j in range(lo, hi + 1)}
    return out


def test_tiles_touched_counts_the_footprint():
    """tiles_touched = the number of tiles of the A50 row spans, every one of
    them inside the box's tile rectangle; rows past the box's last tile row
    are empty."""
    cam = synth.tiny_camera(100, 70)
    sc = synth.random_scene(300, cam, seed=5, sigma_median=4.0)
    pr = oracle.project(cam, sc)
    for i in np.nonzero(pr["visible"])[0]:
        x0, x1, y0, y1 = pr["box"][i]
        tiles = footprint_tiles(pr, i, cam.tiles_x)
        assert pr["tiles"][i] == len(tiles)
        assert all(x0 // 16 <= tx <= x1 // 16 and y0 // 16 <= ty <= y1 // 16 for ty, tx in tiles)


@pytest.mark.parametrize("case", ["c1", "n3dv_crop"])
def test_footprint_holds_every_accepted_pixel(case):
    """A50's premise, by brute force: every (pixel, Gaussian) the oracle's double
    render accepts (α ≥ 1/255, Eq. 8) lies in a tile of the Gaussian's footprint,
    so the tiled per-pixel sequences equal the tile-free ones (the lemma of SURVEY
    §8(c)) and the image is the same as under A05's whole-box rule; and the
    footprint is tighter than the box (fewer pairs)."""
    if case == "c1":
        cam, sc = synth.c1()
    else:
        cam = synth.n3dv_rig(width=320, height=240)[9]
        sc = synth.n3dv_scene(n=6000, seed=23, degree=1, fx=cam.fx)
    pr = oracle.project(cam, sc)
    X, Y = np.meshgrid(np.arange(cam.width), np.arange(cam.height))
    k_box = k_fp = 0
    for i in np.nonzero(pr["visible"])[0]:
        x0, x1, y0, y1 = pr["box"][i]
        u, v = pr["uvz"][i, :2]
        A, B, C = pr["conic"][i]
        o = pr["opa"][i]
        xs, ys = X[y0:y1 + 1, x0:x1 + 1], Y[y0:y1 + 1, x0:x1 + 1]
        dx, dy = u - xs, v - ys
        power = -0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy
        acc = (power <= 0) & (np.minimum(0.99, o * np.exp(power)) >= 1 / 255)
        tiles = footprint_tiles(pr, i, cam.tiles_x)
        need = {(int(a) // 16, int(b) // 16) for a, b in zip(ys[acc], xs[acc])}
        assert need <= tiles, (i, sorted(need - tiles)[:4])
        k_box += (x1 // 16 - x0 // 16 + 1) * (y1 // 16 - y0 // 16 + 1)
        k_fp += len(tiles)
    assert k_fp < 0.9 * k_box


def test_sh_orthonormal_quadrature():
    """∫ Y_i Y_j dΩ = δ_ij (Gauss-Legendre in cos θ × uniform φ, exact for
    these polynomial degrees) — pins the SH constants up to sign (A14)."""
    xs, ws = np.polynomial.legendre.leggauss(16)
    nphi = 32
    phis = 2 * np.pi * np.arange(nphi) / nphi
    dirs, wts = [], []
    for ct, w in zip(xs, ws):
        st = math.sqrt(1 - ct * ct)
        for ph in phis:
            dirs.append([st * math.cos(ph), st * math.sin(ph), ct])
            wts.append(w * 2 * np.pi / nphi)
    Y = oracle.sh_basis(3, np.array(dirs))
    G = (Y * np.array(wts)[:, None]).T @ Y
    np.testing.assert_allclose(G, np.eye(16), atol=1e-10)
    # degree 0: col = Y_0 · sh_0 + 0.5 with Y_0 = 1/(2√π)
    assert Y[0, 0] == pytest.approx(0.5 / math.sqrt(math.pi), rel=1e-15)


def test_sh_colour_degree0_and_clamp():
    """Degree 0: col = sh0/(2√π) + 0.5, clamped at 0 with its clamp bit (A14)."""
    cam = synth.tiny_camera(64, 64)
    sc = synth.random_scene(200, cam, seed=2, degree=0)
    coeffs = sc.sh_coeffs()[:, 0, :].astype(np.float64)
    coeffs[:10] = -3.0
    sc.sh = synth.pack_sh(coeffs[:, None, :])
    pr = oracle.project(cam, sc)
    vis = pr["visible"] == 1
    col = coeffs / (2 * math.sqrt(math.pi)) + 0.5
    np.testing.assert_allclose(pr["rgb"][vis], np.maximum(col[vis], 0), rtol=1e-6, atol=1e-7)
    bits = (col < 0).astype(int) @ np.array([1, 2, 4])
    assert np.array_equal(pr["clampbits"][vis], bits[vis])


def test_degenerate_quaternion_and_masked_are_culled():
    """Zero/non-finite q culled (A15); keep_mask = 0 culls (Eq. 1 + A10)."""
    cam = synth.tiny_camera(64, 64)
    sc = synth.random_scene(50, cam, seed=3)
    sc.rot[0] = 0
    sc.rot[1] = np.nan
    keep = np.ones(50, np.uint8); keep[2] = 0
    pr = oracle.project(cam, sc, keep=keep)
    assert pr["visible"][0] == 0 and pr["visible"][1] == 0 and pr["visible"][2] == 0
    assert pr["tiles"][2] == 0
