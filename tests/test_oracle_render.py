"""Pins of the oracle renderer (O4, O5, O6) against closed forms, invariants
and finite differences — Eq. 8, its derivative, S:195-206,
S:227-231 and the north star's "closed-form image of a single isotropic
Gaussian, transmittance monotonicity and early-termination invariants, and
finite-difference gradients on tiny scenes"."""
import copy
import math

import numpy as np
import pytest

import oracle
from paper_2411_14847_b200 import synth

Y0 = 0.5 / math.sqrt(math.pi)   # degree-0 real SH: 1/(2√π) (normalisation, pinned by quadrature)


def _cam(W, H, fx, fy, cx, cy, R=None, t=(0, 0, 0)):
    R = np.eye(3) if R is None else R
    vm = np.concatenate([R, np.array(t, dtype=np.float64)[:, None]], 1).astype(np.float32)
    return synth.Camera(W, H, fx, fy, cx, cy, vm)


def _scene(pos, scale, rot, opa, cols, degree=0):
    n = len(pos)
    pos_opa = np.concatenate([np.array(pos, np.float64), np.array(opa, np.float64)[:, None]], 1)
    sc = np.concatenate([np.array(scale, np.float64), np.zeros((n, 1))], 1)
    coeffs = np.zeros((n, (degree + 1) ** 2, 3))
    coeffs[:, 0, :] = (np.array(cols, np.float64) - 0.5) / Y0
    return synth.Scene(pos_opa.astype(np.float32), sc.astype(np.float32),
                       np.array(rot, np.float32), synth.pack_sh(coeffs), degree)


def test_empty_scene_is_background():
    cam = _cam(40, 30, 40, 40, 19.5, 14.5)
    sc = _scene([[0, 0, -5]], [[0.1] * 3], [[1, 0, 0, 0]], [0.9], [[1, 1, 1]])  # behind camera
    bg = np.array([0.25, 0.5, 0.75], np.float32)
    r = oracle.render(cam, sc, bg=bg, mode="literal")
    assert np.array_equal(r["img"], np.broadcast_to(bg.astype(np.float64)[:, None, None], r["img"].shape))
    assert np.all(r["T"] == 1.0) and np.all(r["nacc"] == 0)


@pytest.mark.parametrize("fx,fy,d,sigma,o", [(50.0, 70.0, 3.0, 0.1, 0.7), (64.0, 64.0, 2.5, 0.05, 0.999),
                                             (40.0, 55.0, 4.0, 0.2, 0.3)])
def test_single_isotropic_gaussian_closed_form(fx, fy, d, sigma, o):
    """SURVEY §8(c) closed form: image = c·min(0.99, o·exp(−½((X−cx)²/a + (Y−cy)²/c′)))
    on box pixels with α ≥ 1/255, T = 1 − α, with a = fx²σ²/d² + 0.3 and
    r = ⌈3√λmax⌉, λmax = max(a,c′) if |a−c′|/2 ≥ √0.1 else (a+c′)/2 + √0.1."""
    W, H, cx, cy = 64, 48, 31.3, 22.6
    cam = _cam(W, H, fx, fy, cx, cy)
    col = [0.8, 0.35, 0.6]
    sc = _scene([[0, 0, d]], [[sigma] * 3], [[0.3, 0.1, -0.5, 0.2]], [o], [col])
    r = oracle.render(cam, sc, mode="literal")
    f32 = lambda v: float(np.float32(v))
    fx_, fy_, cx_, cy_, s_, d_, o_ = map(f32, (fx, fy, cx, cy, sigma, d, o))
    a = fx_ ** 2 * s_ ** 2 / d_ ** 2 + 0.3
    c = fy_ ** 2 * s_ ** 2 / d_ ** 2 + 0.3
    lam = max(a, c) if abs(a - c) / 2 >= math.sqrt(0.1) else (a + c) / 2 + math.sqrt(0.1)
    rad = math.ceil(3 * math.sqrt(lam))
    cols = np.array([float(np.float32((cc - 0.5) / Y0)) * Y0 + 0.5 for cc in col])
    X, Y = np.meshgrid(np.arange(W), np.arange(H))
    alpha = np.minimum(0.99, o_ * np.exp(-0.5 * ((X - cx_) ** 2 / a + (Y - cy_) ** 2 / c)))
    inbox = (np.abs(X - cx_) <= rad) & (np.abs(Y - cy_) <= rad)
    acc = inbox & (alpha >= 1 / 255)
    exp_img = np.where(acc[None], cols[:, None, None] * alpha[None], 0.0)
    np.testing.assert_allclose(r["img"], exp_img, atol=1e-12)
    np.testing.assert_allclose(r["T"], np.where(acc, 1 - alpha, 1.0), atol=1e-12)
    assert r["nacc"].sum() == acc.sum()


def test_three_on_axis_gaussians_blend_front_to_back_with_termination():
    """C = c1α1 + c2α2(1−α1) (+ c3α3(1−α1)(1−α2)) at the principal pixel where
    G = 1 — Eq. 8 with ascending depth (A01) and 'stop before adding' at T<1e-4
    (A12). Input order is deliberately not depth order."""
    cam = _cam(33, 33, 40, 40, 16.0, 16.0)
    cols = [[0.9, 0.1, 0.2], [0.3, 0.8, 0.5], [0.1, 0.2, 0.95]]
    # depths 4, 2, 3 → front-to-back order: index 1, 2, 0
    pos = [[0, 0, 4.0], [0, 0, 2.0], [0, 0, 3.0]]
    sc = _scene(pos, [[0.05] * 3] * 3, [[1, 0, 0, 0]] * 3, [0.7, 0.5, 0.6], cols)
    r = oracle.render(cam, sc, mode="literal")
    c = np.array([[float(np.float32((v - 0.5) / Y0)) * Y0 + 0.5 for v in cc] for cc in cols])
    a1, a2, a3 = float(np.float32(0.5)), float(np.float32(0.6)), float(np.float32(0.7))
    expect = c[1] * a1 + c[2] * a2 * (1 - a1) + c[0] * a3 * (1 - a1) * (1 - a2)
    np.testing.assert_allclose(r["img"][:, 16, 16], expect, atol=1e-14)
    assert r["T"][16, 16] == pytest.approx((1 - a1) * (1 - a2) * (1 - a3), abs=1e-15)
    # termination: α = 0.99, 0.98, 0.9 → T = 0.01, 2e-4, (2e-5 < 1e-4: third not added)
    sc2 = _scene(pos, [[0.05] * 3] * 3, [[1, 0, 0, 0]] * 3, [0.9, 0.999, 0.98], cols)
    r2 = oracle.render(cam, sc2, mode="literal")
    b1, b2 = 0.99, float(np.float32(0.98))
    np.testing.assert_allclose(r2["img"][:, 16, 16], c[1] * b1 + c[2] * b2 * (1 - b1), atol=1e-14)
    assert r2["term"][16, 16] == 1 and r2["nacc"][16, 16] == 2
    assert r2["T"][16, 16] == pytest.approx((1 - b1) * (1 - b2), rel=1e-14)


def test_equal_depth_ties_broken_by_index():
    """Equal depth bits → lower index composites first (A03)."""
    cam = _cam(17, 17, 20, 20, 8.0, 8.0)
    cols = [[0.9, 0.05, 0.1], [0.1, 0.1, 0.9]]
    sc = _scene([[0, 0, 3.0], [0, 0, 3.0]], [[0.05] * 3] * 2, [[1, 0, 0, 0]] * 2, [0.6, 0.6], cols)
    r = oracle.render(cam, sc, mode="literal")
    a = float(np.float32(0.6))
    c = np.array([[float(np.float32((v - 0.5) / Y0)) * Y0 + 0.5 for v in cc] for cc in cols])
    np.testing.assert_allclose(r["img"][:, 8, 8], c[0] * a + c[1] * a * (1 - a), atol=1e-14)


def test_partition_of_unity_white_on_white():
    """Σ_k w_k + T_final = 1: all-white Gaussians on a white background render 1."""
    cam, sc = synth.c1()
    coeffs = sc.sh_coeffs()
    coeffs[:, 0, :] = 0.5 / Y0
    sc.sh = synth.pack_sh(coeffs)
    r = oracle.render(cam, sc, bg=np.ones(3, np.float32))
    np.testing.assert_allclose(r["img"], 1.0, atol=1e-6)


def test_invariants_c1():
    """T_final ≥ 1e-4 (A12); terminated ⇒ T_final < 1e-4/(1−0.99); pixel value
    bounded by (1−T)·max col; literal ≡ scatter bit-exact; permutation
    invariance; masked-to-zero = deleted bit-exact."""
    cam, sc = synth.c1()
    lit = oracle.render(cam, sc, mode="literal")
    sca = oracle.render(cam, sc, mode="scatter")
    for k in ("img", "T", "nacc", "last_id", "tie", "term", "pfwd", "pbwd"):
        assert np.array_equal(lit[k], sca[k]), k
    T = lit["T"]
    assert T.min() >= 1e-4 and T.max() <= 1.0
    assert np.all(T[lit["term"] == 1] < 1e-2)
    pr = oracle.project(cam, sc)
    cmax = pr["rgb"].max()
    assert np.all(lit["img"] <= (1 - T)[None] * cmax + 1e-12)
    assert np.all(lit["pbwd"] <= lit["pfwd"]) and np.all(lit["nacc"] <= lit["pbwd"])
    # permutation invariance (distinct depths)
    perm = np.random.default_rng(0).permutation(sc.n)
    sp = synth.Scene(sc.pos_opa[perm], sc.scale[perm], sc.rot[perm], sc.sh[:, perm], 0)
    rp = oracle.render(cam, sp)
    assert np.array_equal(rp["img"], lit["img"]) and np.array_equal(rp["T"], lit["T"])
    # masked = deleted
    keep = (np.arange(sc.n) % 3 != 0).astype(np.uint8)
    rm = oracle.render(cam, sc, keep=keep)
    idx = np.nonzero(keep)[0]
    sd = synth.Scene(sc.pos_opa[idx], sc.scale[idx], sc.rot[idx], sc.sh[:, idx], 0)
    rd = oracle.render(cam, sd)
    assert np.array_equal(rm["img"], rd["img"]) and np.array_equal(rm["T"], rd["T"])


def test_tie_fraction_small_c1():
    cam, sc = synth.c1()
    r = oracle.render(cam, sc)
    assert r["tie"].mean() < 1e-3


# ------------------------------------------------------------- backward ----

def _fd_scene(seed, degree=3, clamp_case=False):
    cam = _cam(16, 16, 16, 18, 7.5, 8.2,
               R=synth._rot_yaw_pitch(0.1, -0.05).T, t=(0.05, -0.02, 0.1))
    sc = synth.random_scene(8, synth.tiny_camera(16, 16), seed=seed, degree=degree, sigma_median=2.0)
    if clamp_case:
        # a large Gaussian outside the guard band (|t_x/t_z| > 1.3 W/(2 fx)) reaching into view
        sc.pos_opa[0, :3] = [3.2, 0.1, 3.0]
        sc.scale[0, :3] = [1.5, 0.6, 0.9]
        sc.pos_opa[0, 3] = 0.8
    return cam, sc


def _loss(cam, sc, g, bg):
    r = oracle.render(cam, sc, bg=bg, mode="literal")
    return float((r["img"] * g).sum()), r["nacc"].copy(), r["last_id"].copy()


@pytest.mark.parametrize("seed,clamp_case", [(7, False), (8, True), (9, False)])
def test_backward_matches_central_differences(seed, clamp_case):
    """Every analytic gradient (p, o, s, q, SH) vs central FD of the double
    forward, rel < 1e-4 (floor 1e-3), rejecting probes whose accepted set
    changes (A18) — S:205."""
    cam, sc = _fd_scene(seed, clamp_case=clamp_case)
    g = synth.grad_image(cam, seed + 100)
    bg = np.array([0.2, 0.3, 0.4], np.float32)
    ref = oracle.render_bwd(cam, sc, g, bg=bg, mode="literal")
    L0, na0, li0 = _loss(cam, sc, g, bg)
    checked = rejected = 0

    def fd(field, idx, rel=2e-4):
        s1, s2 = copy.deepcopy(sc), copy.deepcopy(sc)
        a1, a2 = getattr(s1, field), getattr(s2, field)
        x = float(a1[idx]); h = max(abs(x) * rel, 2e-5)
        a1[idx] = np.float32(x + h); a2[idx] = np.float32(x - h)
        dh = float(a1[idx]) - float(a2[idx])
        Lp, nap, lip = _loss(cam, s1, g, bg)
        Lm, nam, lim = _loss(cam, s2, g, bg)
        ok = all(np.array_equal(u, v) for u, v in ((nap, na0), (nam, na0), (lip, li0), (lim, li0)))
        return (Lp - Lm) / dh, ok

    for i in range(sc.n):
        for field, key, comps in (("pos_opa", "g_pos_opa", range(4)), ("scale", "g_scale", range(3)),
                                  ("rot", "g_rot", range(4))):
            for a in comps:
                f, ok = fd(field, (i, a))
                if not ok:
                    rejected += 1
                    continue
                an = ref[key][i, a]
                assert abs(f - an) <= 1e-4 * max(abs(an), 1e-3), (field, i, a, f, an)
                checked += 1
        for k in range(16):
            for ch in range(3):
                fl = 3 * k + ch
                f, ok = fd("sh", (fl // 4, i, fl % 4))
                if not ok:
                    rejected += 1
                    continue
                an = ref["g_sh"][i, k, ch]
                assert abs(f - an) <= 1e-4 * max(abs(an), 1e-3), ("sh", i, k, ch, f, an)
                checked += 1
    assert checked > 10 * rejected and checked > 400
    if clamp_case:
        assert np.any(ref["g_pos_opa"][0] != 0)   # the clamped-J Gaussian contributes


def test_backward_zero_in_zero_out_and_colour_sum():
    """dL/dC = 0 → all gradients 0; with dL/dC ≡ 1 per channel,
    Σ_i dL/dcol_i = Σ_px (1 − T_final) (partition of unity)."""
    cam, sc = synth.c1()
    z = oracle.render_bwd(cam, sc, np.zeros((3, 64, 64), np.float32))
    for k in ("g_pos_opa", "g_scale", "g_rot", "g_sh", "g2d"):
        assert not np.any(z[k]), k
    one = oracle.render_bwd(cam, sc, np.ones((3, 64, 64), np.float32))
    for ch in range(3):
        assert one["g2d"][:, 6 + ch].sum() == pytest.approx((1 - one["T"]).sum(), rel=1e-10)


def test_backward_literal_equals_scatter():
    cam, sc = synth.c1()
    g = synth.grad_image(cam, 5)
    a = oracle.render_bwd(cam, sc, g, bg=np.array([0.1, 0.2, 0.3], np.float32), mode="literal")
    b = oracle.render_bwd(cam, sc, g, bg=np.array([0.1, 0.2, 0.3], np.float32), mode="scatter")
    for k in ("g_pos_opa", "g_scale", "g_rot", "g_sh", "g2d", "gradstat_sum"):
        np.testing.assert_allclose(a[k], b[k], rtol=1e-9, atol=1e-12 * np.abs(a[k]).max())


def test_gradstat_counts_visible_views():
    """cnt = 1 for each Gaussian visible in the view, 0 otherwise; sum = 0 when
    invisible (A23)."""
    cam, sc = synth.c1()
    pr = oracle.project(cam, sc)
    g = synth.grad_image(cam, 5)
    b = oracle.render_bwd(cam, sc, g)
    assert np.array_equal(b["gradstat_cnt"], pr["visible"].astype(np.int32))
    assert np.all(b["gradstat_sum"][pr["visible"] == 0] == 0)
    assert np.all(b["gradstat_sum"] >= 0)


def test_kappa_bounds_gradient_magnitude():
    """κ = Σ_px |L|·|terms| ≥ |Σ_px L·terms| (triangle inequality), entrywise."""
    cam, sc = synth.c1()
    g = synth.grad_image(cam, 5)
    o = oracle.render_bwd(cam, sc, g, kappa=True)
    for gk, kk in (("g_pos_opa", "k_pos_opa"), ("g_scale", "k_scale"), ("g_rot", "k_rot"), ("g_sh", "k_sh")):
        assert np.all(o[kk] >= np.abs(o[gk]) * (1 - 1e-9) - 1e-15), gk
    assert np.all(o["k_pos_opa"] >= 0)
