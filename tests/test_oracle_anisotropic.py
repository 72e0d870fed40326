"""Pins of the oracle's conic cross term and of the ∇p̄ statistic's value,
both from mathematics that shares nothing with oracle.cpp:

* The image of one rotated, anisotropic Gaussian seen by a rotated camera,
  off-axis, is c·min(0.99, o·exp(−½ dᵀΣ′⁻¹d)) (Eq. 5, Eq. 7 P:345,
  Eq. 8) with Σ′ = J R_cw Σ R_cwᵀ Jᵀ + 0.3 I (A07).  Here R(q) comes from
  the quaternion sandwich product q v q*, J is the Jacobian of the pinhole map
  π(t) = (fx tx/tz + cx, fy ty/tz + cy) taken by complex-step differentiation
  (exact to rounding, no formula for J typed), and Σ′⁻¹ is numpy's inverse.
  A sign slip in the conic's B = −b/det or in the −B·dx·dy term mirrors the
  ellipse and fails by O(0.1).
* ∂L/∂u and ∂L/∂v of one Gaussian are the derivatives of L with respect to the
  camera's principal point: u = fx tx/tz + cx (P:409 pinhole, A19), and nothing
  else in the forward depends on cx, cy.  Central differences over cx and cy
  therefore pin the oracle's gradstat = ‖(∂L/∂u·W/2, ∂L/∂v·H/2)‖ (A23)
  and the 2D gradients g2d[0:2]; with W ≠ H a dropped or swapped W/2 fails.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2411_14847_b200 import synth

Y0 = 0.5 / math.sqrt(math.pi)


def _hamilton(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def _rot_sandwich(q):
    """Columns R e_k = q e_k q* (textbook rotation by a unit quaternion)."""
    q = np.asarray(q, np.float64)
    q = q / np.linalg.norm(q)
    qc = q * np.array([1, -1, -1, -1])
    cols = [_hamilton(_hamilton(q, np.r_[0.0, e]), qc)[1:] for e in np.eye(3)]
    return np.stack(cols, 1)


def _axis_angle(axis, ang):
    axis = np.asarray(axis, np.float64) / np.linalg.norm(axis)
    return np.r_[math.cos(ang / 2), math.sin(ang / 2) * axis]


def _camera(W, H, fx, fy, cx, cy, q_cam, t):
    R = _rot_sandwich(q_cam).astype(np.float32)
    vm = np.concatenate([R, np.array(t, np.float32)[:, None]], 1).astype(np.float32)
    return synth.Camera(W, H, fx, fy, cx, cy, vm)


def _scene(p, s, q, o, col):
    pos_opa = np.array([[*p, o]], np.float32)
    sc = np.array([[*s, 0.0]], np.float32)
    coeffs = np.zeros((1, 1, 3))
    coeffs[0, 0, :] = (np.array(col, np.float64) - 0.5) / Y0
    return synth.Scene(pos_opa, sc, np.array([q], np.float32), synth.pack_sh(coeffs), 0)


def _expected(cam, sc):
    """Closed-form image, T and box of the single Gaussian (double arithmetic
    on the fp32-rounded inputs)."""
    f = lambda v: np.asarray(v, np.float32).astype(np.float64)
    Rcw, tcw = f(cam.viewmat[:, :3]), f(cam.viewmat[:, 3])
    fx, fy, cx, cy = (float(np.float32(v)) for v in (cam.fx, cam.fy, cam.cx, cam.cy))
    p, s, q = f(sc.pos_opa[0, :3]), f(sc.scale[0, :3]), f(sc.rot[0])
    o = float(sc.pos_opa[0, 3])
    t = Rcw @ p + tcw

    def pinhole(tt):
        return np.array([fx * tt[0] / tt[2] + cx, fy * tt[1] / tt[2] + cy])

    h = 1e-20
    J = np.stack([np.imag(pinhole(t + 1j * h * e)) / h for e in np.eye(3)], 1)   # 2×3
    u, v = pinhole(t)
    Rq = _rot_sandwich(q)
    Sigma = Rq @ np.diag(s ** 2) @ Rq.T
    M = J @ Rcw
    Sp = M @ Sigma @ M.T + 0.3 * np.eye(2)
    Ki = np.linalg.inv(Sp)
    lam = np.linalg.eigvalsh(Sp).max()
    r = math.ceil(3 * math.sqrt(lam))
    col = np.array([float(sc.sh.reshape(-1)[c]) * Y0 + 0.5 for c in range(3)])
    X, Y = np.meshgrid(np.arange(cam.width, dtype=np.float64), np.arange(cam.height, dtype=np.float64))
    dX, dY = X - u, Y - v
    m2 = Ki[0, 0] * dX * dX + 2 * Ki[0, 1] * dX * dY + Ki[1, 1] * dY * dY
    alpha = np.minimum(0.99, o * np.exp(-0.5 * m2))
    inbox = (np.abs(dX) <= r) & (np.abs(dY) <= r)
    acc = inbox & (alpha >= 1 / 255)
    img = np.where(acc[None], col[:, None, None] * alpha[None], 0.0)
    T = np.where(acc, 1 - alpha, 1.0)
    return dict(img=img, T=T, acc=acc, u=u, v=v, r=r, lam=lam, Sp=Sp, alpha=alpha)


CASES = [
    # (W, H, fx, fy, cx, cy, camera quaternion, camera t, p, s, q, o)
    (72, 56, 60.0, 75.0, 35.2, 27.9, _axis_angle([0.3, 1.0, -0.2], 0.35), (0.1, -0.05, 0.2),
     (0.4, 0.1, 3.0), (0.35, 0.06, 0.12), _axis_angle([0.2, -0.5, 1.0], 0.9), 0.3),
    (64, 52, 58.0, 58.0, 31.5, 25.5, _axis_angle([1.0, 0.0, 0.4], -0.25), (0.0, 0.1, 0.0),
     (-0.3, 0.2, 2.5), (0.05, 0.3, 0.08), _axis_angle([1.0, 1.0, 0.0], 0.6), 0.25),
    (80, 48, 70.0, 52.0, 41.0, 22.5, _axis_angle([0.0, 0.0, 1.0], 0.5), (0.05, 0.0, 0.3),
     (0.2, -0.15, 2.8), (0.25, 0.04, 0.2), _axis_angle([0.4, 0.1, 1.0], -1.1), 0.93),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_rotated_anisotropic_gaussian_closed_form(case):
    W, H, fx, fy, cx, cy, qc, tc, p, s, q, o = CASES[case]
    cam = _camera(W, H, fx, fy, cx, cy, qc, tc)
    sc = _scene(p, s, q, o, [0.8, 0.35, 0.6])
    e = _expected(cam, sc)
    # the case is genuinely anisotropic with a strong cross term, and fully on screen
    a, b, c = e["Sp"][0, 0], e["Sp"][0, 1], e["Sp"][1, 1]
    assert abs(b) > 0.3 * math.sqrt(a * c), (a, b, c)
    assert 0.08 < 3 * math.sqrt(e["lam"]) % 1 < 0.92       # the box radius is not a rounding tie
    assert e["acc"].sum() > 50
    r = oracle.render(cam, sc, mode="literal")
    np.testing.assert_allclose(r["img"], e["img"], atol=1e-9)
    np.testing.assert_allclose(r["T"], e["T"], atol=1e-9)
    assert r["nacc"].sum() == e["acc"].sum()
    # the mirrored ellipse (cross term's sign flipped) is far from the oracle's image
    Ki = np.linalg.inv(e["Sp"] * np.array([[1, -1], [-1, 1]]))
    X, Y = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    dX, dY = X - e["u"], Y - e["v"]
    alt = np.minimum(0.99, o * np.exp(-0.5 * (Ki[0, 0] * dX * dX + 2 * Ki[0, 1] * dX * dY + Ki[1, 1] * dY * dY)))
    assert np.abs(alt - e["alpha"]).max() > 0.05


def _render_loss(cam, sc, g, bg):
    r = oracle.render(cam, sc, bg=bg, mode="literal")
    return float((r["img"] * g).sum()), r["nacc"].copy()


@pytest.mark.parametrize("case", range(len(CASES)))
def test_gradstat_value_against_principal_point_differences(case):
    W, H, fx, fy, cx, cy, qc, tc, p, s, q, o = CASES[case]
    cam = _camera(W, H, fx, fy, cx, cy, qc, tc)
    sc = _scene(p, s, q, o, [0.8, 0.35, 0.6])
    g = synth.grad_image(cam, 300 + case)
    bg = np.array([0.1, 0.2, 0.3], np.float32)
    ref = oracle.render_bwd(cam, sc, g, bg=bg, mode="literal")
    _, na0 = _render_loss(cam, sc, g, bg)
    grads = []
    for field in ("cx", "cy"):
        x = getattr(cam, field)
        for hh in (2e-3, 1.3e-3, 7e-4):     # first step whose accepted set is unchanged (A18)
            c1 = _camera(W, H, fx, fy, cx, cy, qc, tc)
            c2 = _camera(W, H, fx, fy, cx, cy, qc, tc)
            setattr(c1, field, float(np.float32(x + hh)))
            setattr(c2, field, float(np.float32(x - hh)))
            Lp, nap = _render_loss(c1, sc, g, bg)
            Lm, nam = _render_loss(c2, sc, g, bg)
            if np.array_equal(nap, na0) and np.array_equal(nam, na0):
                grads.append((Lp - Lm) / (getattr(c1, field) - getattr(c2, field)))
                break
        else:
            pytest.fail(f"accepted set changes for every probe step on {field}")
    gu, gv = grads
    assert abs(gu) > 1e-6 and abs(gv) > 1e-6
    np.testing.assert_allclose(ref["g2d"][0, 0], gu, rtol=1e-5)
    np.testing.assert_allclose(ref["g2d"][0, 1], gv, rtol=1e-5)
    stat = math.hypot(gu * W / 2, gv * H / 2)
    assert ref["gradstat_sum"][0] == pytest.approx(stat, rel=1e-5)
    assert ref["gradstat_cnt"][0] == 1
    # W ≠ H or |gu| ≠ |gv|: a dropped or swapped W/2, H/2 scaling is distinguishable
    for wrong in (math.hypot(gu, gv), math.hypot(gu * H / 2, gv * W / 2), math.hypot(gu * W, gv * H)):
        assert abs(wrong - stat) > 1e-3 * stat


def test_tie_slack_is_the_flipped_pixels_contribution():
    """A29 tie slack: with one Gaussian and exactly one pixel inside a widened
    α-threshold margin, branch B drops that pixel's entry, so the slack equals
    that pixel's own contribution (its 2D terms from a render whose dL/dC is
    that pixel alone); with default margins and no ties the slack is zero."""
    W, H = 40, 32
    cam = _camera(W, H, 50.0, 50.0, 19.3, 15.6, _axis_angle([0, 0, 1], 0.0), (0, 0, 0))
    sc = _scene((0.02, -0.01, 3.0), (0.05, 0.07, 0.06), _axis_angle([0.3, 1, 0], 0.4), 0.6,
                [0.7, 0.2, 0.5])
    g = synth.grad_image(cam, 77)
    r = oracle.render(cam, sc, mode="literal")
    pr = oracle.project(cam, sc)
    u, v = pr["uvz"][0, :2]
    A, B, C = pr["conic"][0]
    o = pr["opa"][0]
    X, Y = np.meshgrid(np.arange(W), np.arange(H))
    dx, dy = u - X, v - Y
    alpha = np.minimum(0.99, o * np.exp(-0.5 * (A * dx * dx + C * dy * dy) - B * dx * dy))
    rel = np.abs(alpha - 1 / 255) * 255
    inbox = r["nacc"] >= 0
    order = np.argsort(rel.reshape(-1))
    p0, p1 = order[0], order[1]
    margin = 0.5 * (rel.reshape(-1)[p0] + rel.reshape(-1)[p1])   # exactly one pixel inside
    assert rel.reshape(-1)[p0] < margin < rel.reshape(-1)[p1] and alpha.reshape(-1)[p0] < 0.5
    eps = np.array([margin, 1e-12, 1e-12, 1e-12])
    b = oracle.render_bwd(cam, sc, g, mode="literal", tie_eps=eps, kappa=True)
    Y0, X0 = divmod(int(p0), W)
    tie = oracle.render(cam, sc, mode="literal", tie_eps=eps)["tie"]
    assert tie.sum() == 1 and tie[Y0, X0] == 1
    # the pixel's own contribution: a render whose dL/dC is that pixel alone, where the
    # entry is accepted (α above 1/255) — else the slack's branch B is the accepting one
    one = np.zeros_like(g)
    one[:, Y0, X0] = g[:, Y0, X0]
    lo = oracle.render_bwd(cam, sc, one, mode="literal", tie_eps=eps)
    if alpha[Y0, X0] >= 1 / 255:
        gu, gv = lo["g2d"][0, 0], lo["g2d"][0, 1]
        assert b["t_gradstat"][0] == pytest.approx(abs(gu) * W / 2 + abs(gv) * H / 2, rel=1e-12)
    else:
        assert not lo["g2d"].any() and b["t_gradstat"][0] > 0
    assert b["gtie"][0] == 0
    d = oracle.render_bwd(cam, sc, g, mode="literal", kappa=True)
    assert oracle.render(cam, sc, mode="literal")["tie"].sum() == 0
    assert not d["t_pos_opa"].any() and not d["t_gradstat"].any()
