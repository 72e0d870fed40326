"""Pins of the oracle's binning (O3), shift (O1) and error map / Alg. 1 (O7).

O3: brute-force enumeration is the definition (A03-A04, A50); pinned by an
independent decoding of the footprints, each inside the box's tile rectangle,
and the sort invariants (the footprints' conservativeness is pinned in
test_oracle_geometry.py).
O1: §3.3 P:128 — pinned by rotation composition (sandwich product), identity
cases, unit norm and finite differences.
O7: §3.4, Alg. 1 P:403-415 — pinned by S:213-215/S:630 examples and
the textbook pinhole projection.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2411_14847_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ O3 -----

def _check_binsort(cam, pr):
    keys, ids, ranges = oracle.bin_sort(cam, pr)
    K = len(keys)
    vis = np.nonzero(pr["visible"])[0]
    assert K == int(pr["tiles"][vis].sum())
    # independent enumeration: the decoded A50 footprints (KEY CHAIN step 13), each
    # a subset of the box's tile rectangle
    from test_oracle_geometry import footprint_tiles
    expect = set()
    for i in vis:
        x0, x1, y0, y1 = pr["box"][i]
        for ty, tx in footprint_tiles(pr, i, cam.tiles_x):
            assert tx * 16 <= x1 and tx * 16 + 15 >= x0 and ty * 16 <= y1 and ty * 16 + 15 >= y0
            expect.add((ty * cam.tiles_x + tx, int(i)))
    got = {(int(k >> np.uint64(32)), int(i)) for k, i in zip(keys, ids)}
    assert got == expect and len(got) == K
    # key low bits are the depth bits of the id
    assert np.array_equal((keys & np.uint64(0xFFFFFFFF)).astype(np.uint32), pr["zbits"][ids])
    # ranges partition [0, K) in tile order; each range sorted by (zbits, id)
    pos = 0
    for t in range(cam.num_tiles):
        s, e = ranges[t]
        if s == e:
            assert s == 0 and e == 0
            continue
        assert s == pos and e > s
        assert np.all((keys[s:e] >> np.uint64(32)) == t)
        zb = pr["zbits"][ids[s:e]].astype(np.int64)
        order = np.lexsort((ids[s:e], zb))
        assert np.array_equal(order, np.arange(e - s))
        pos = e
    assert pos == K


def test_binsort_c1():
    cam, sc = synth.c1()
    _check_binsort(cam, oracle.project(cam, sc))


def test_binsort_ragged_image_rotated_camera():
    cam = synth.n3dv_rig(width=200, height=150)[6]
    sc = synth.n3dv_scene(n=3000, seed=21, fx=cam.fx)
    _check_binsort(cam, oracle.project(cam, sc))


def test_binsort_equal_depth_plane_ties_by_index():
    """Planar scene with exactly equal depth bits: order within a tile is by index."""
    cam = synth.tiny_camera(48, 40)
    sc = synth.random_scene(200, cam, seed=4)
    sc.pos_opa[:, 2] = 3.0
    pr = oracle.project(cam, sc)
    assert len(np.unique(pr["zbits"][pr["visible"] == 1])) == 1
    keys, ids, ranges = oracle.bin_sort(cam, pr)
    for t in range(cam.num_tiles):
        s, e = ranges[t]
        assert np.all(np.diff(ids[s:e].astype(np.int64)) > 0)
    _check_binsort(cam, pr)


def test_binsort_empty():
    cam = synth.tiny_camera(32, 32)
    sc = synth.random_scene(10, cam, seed=1)
    sc.pos_opa[:, 2] = -1.0
    keys, ids, ranges = oracle.bin_sort(cam, oracle.project(cam, sc))
    assert len(keys) == 0 and not np.any(ranges)


# ------------------------------------------------------------------ O1 -----

def _L(a):
    w, x, y, z = a
    return np.array([[w, -x, -y, -z], [x, w, -z, y], [y, z, w, -x], [z, -y, x, w]])


def _rot_of(q):
    q = q / np.linalg.norm(q)
    out = np.zeros((3, 3))
    for k, e in enumerate(np.eye(3)):
        out[:, k] = (_L(_L(q) @ np.r_[0.0, e]) @ (q * np.array([1, -1, -1, -1])))[1:]
    return out


@pytest.mark.parametrize("ex", GOLD["quat_mul"])
def test_quat_mul_spec_examples(ex):
    a = np.array([ex["a"]], np.float32); b = np.array([ex["b"]], np.float32)
    _, ro = oracle.shift(np.zeros((1, 4), np.float32), a, np.zeros((1, 4), np.float32), b)
    expect = np.array(ex["ab"], np.float64) / np.linalg.norm(np.array(ex["a"], np.float64))
    np.testing.assert_allclose(ro[0], expect, atol=1e-7)


def test_shift_identity_copy_and_composition():
    cam, sc = synth.c1()
    n = sc.n
    g = np.random.default_rng(5)
    # μ = 0, σ = identity → p' = p, q' = n(q)
    po, ro = oracle.shift(sc.pos_opa, sc.rot, np.zeros((n, 4), np.float32),
                          np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)))
    np.testing.assert_array_equal(po, sc.pos_opa.astype(np.float64))
    qn = sc.rot.astype(np.float64) / np.linalg.norm(sc.rot.astype(np.float64), axis=1, keepdims=True)
    np.testing.assert_allclose(ro, qn, atol=1e-15)
    # mask = 0 → exact copy
    mu = g.normal(size=(n, 4)).astype(np.float32)
    sig = g.normal(size=(n, 4)).astype(np.float32)
    mask = (g.uniform(size=n) < 0.3).astype(np.uint8)
    po, ro = oracle.shift(sc.pos_opa, sc.rot, mu, sig, mask)
    off = mask == 0
    np.testing.assert_array_equal(po[off], sc.pos_opa[off].astype(np.float64))
    np.testing.assert_array_equal(ro[off], sc.rot[off].astype(np.float64))
    on = np.nonzero(mask)[0]
    np.testing.assert_allclose(po[on, :3], sc.pos_opa[on, :3].astype(np.float64) + mu[on, :3], atol=1e-15)
    assert np.array_equal(po[on, 3], sc.pos_opa[on, 3].astype(np.float64))
    # unit norm and rotation composition R(q ⊗ σ) = R(q) R(σ)
    np.testing.assert_allclose(np.linalg.norm(ro[on], axis=1), 1.0, atol=1e-12)
    for i in on[:50]:
        np.testing.assert_allclose(_rot_of(ro[i]), _rot_of(sc.rot[i].astype(np.float64)) @
                                   _rot_of(sig[i].astype(np.float64)), atol=1e-12)
    # ‖σ‖ < 1e-8 → identity rotation offset
    sig[on[0]] = 1e-10
    po, ro = oracle.shift(sc.pos_opa, sc.rot, mu, sig, mask)
    np.testing.assert_allclose(ro[on[0]], qn[on[0]], atol=1e-15)


def test_shift_bwd_central_differences():
    g = np.random.default_rng(6)
    n = 20
    pos = g.normal(size=(n, 4)).astype(np.float32)
    rot = g.normal(size=(n, 4)).astype(np.float32)
    mu = (g.normal(size=(n, 4)) * 0.1).astype(np.float32)
    sig = (np.array([1, 0, 0, 0]) + g.normal(size=(n, 4)) * 0.2).astype(np.float32)
    mask = (np.arange(n) % 4 != 0).astype(np.uint8)
    gp = g.normal(size=(n, 4)); gq = g.normal(size=(n, 4))
    gmu, gsig = oracle.shift_bwd(rot, sig, mask, gp, gq)

    def L(mu_, sig_):
        po, ro = oracle.shift(pos, rot, mu_, sig_, mask)
        return float((po[:, :3] * gp[:, :3]).sum() + (ro * gq).sum())

    for i in range(n):
        for a in range(4):
            for arr, grad in ((mu, gmu), (sig, gsig)):
                if arr is mu and a == 3:
                    continue
                x = float(arr[i, a]); h = 1e-3
                p1 = arr.copy(); p1[i, a] = np.float32(x + h)
                p2 = arr.copy(); p2[i, a] = np.float32(x - h)
                dh = float(p1[i, a]) - float(p2[i, a])
                f = (L(p1, sig) - L(p2, sig)) / dh if arr is mu else (L(mu, p1) - L(mu, p2)) / dh
                assert abs(f - grad[i, a]) <= 1e-5 * max(1.0, abs(grad[i, a])), (i, a, f, grad[i, a])
    assert not np.any(gmu[mask == 0]) and not np.any(gsig[mask == 0])


# ------------------------------------------------------------------ O7 -----

def test_error_map_spec_examples():
    cam = synth.tiny_camera(40, 30)
    a = synth.random_image(cam, 1)
    pos = np.array([[0, 0, 3, 1]], np.float32)
    o = oracle.error_map(cam, a, a, 0.1, pos)
    assert not np.any(o["err"]) and not np.any(o["D"])
    o = oracle.error_map(cam, np.zeros_like(a), np.ones_like(a), 0.1, pos)
    assert np.all(o["err"] == 1.0) and np.all(o["D"] == 1)
    gam = float(np.float32(0.25))
    b = np.full_like(a, np.float32(0.5)); c = np.full_like(a, np.float32(0.75))
    o = oracle.error_map(cam, b, c, gam, pos)
    assert np.all(o["err"] == 0.25) and not np.any(o["D"])                   # S:630 strict
    rnd = synth.random_image(cam, 2)
    o = oracle.error_map(cam, a, rnd, 0.3, pos)
    np.testing.assert_allclose(o["err"], np.abs(a.astype(np.float64) - rnd).mean(0), atol=1e-15)


def test_alg1_principal_point_behind_and_pinhole():
    """Alg. 1 with T from the camera: a point on the optical axis lands on
    (round cx, round cy); behind the camera is excluded; random
    visible points agree with the textbook pinhole K[R|t]p — exactly
    after round-half-away, except at rounding ties."""
    cam = synth.n3dv_rig(width=301, height=201)[8]   # odd sizes: integer principal point
    V = cam.viewmat.astype(np.float64)
    n = 4000
    g = np.random.default_rng(7)
    tcam = np.stack([g.uniform(-0.7, 0.7, n), g.uniform(-0.6, 0.6, n), np.ones(n)], 1) * \
        g.uniform(0.5, 8, n)[:, None]
    tcam[:5] = [[0, 0, 2.0], [0, 0, 5.0], [0.3, 0.1, -2.0], [0, 0, 0.1], [0, 0, 0.19]]
    p = (tcam - V[:, 3]) @ V[:, :3]   # world = Rᵀ(t_cam − t)
    pos = np.concatenate([p, np.ones((n, 1))], 1).astype(np.float32)
    img = np.zeros((3, 201, 301), np.float32)
    o = oracle.error_map(cam, img, img, 0.1, pos)
    xy = o["xy"]
    cx, cy = float(np.float32(cam.cx)), float(np.float32(cam.cy))
    assert tuple(xy[0]) == (150, 100) == (round(cx), round(cy))
    assert tuple(xy[1]) == tuple(xy[0])
    assert tuple(xy[2]) == (-1, -1) and tuple(xy[3]) == (-1, -1)  # behind / before near (0.2)
    tc = pos[:, :3].astype(np.float64) @ V[:, :3].T + V[:, 3]
    fx, fy = float(np.float32(cam.fx)), float(np.float32(cam.fy))
    u = fx * tc[:, 0] / tc[:, 2] + cx
    v = fy * tc[:, 1] / tc[:, 2] + cy
    ok = (tc[:, 2] > cam.near) & (o["tie_g"] == 0)
    rx = np.floor(np.abs(u) + 0.5) * np.sign(u)
    ry = np.floor(np.abs(v) + 0.5) * np.sign(v)
    inside = ok & (rx >= 0) & (rx < 301) & (ry >= 0) & (ry < 201)
    assert inside.sum() > 1000
    assert np.array_equal(xy[inside, 0], rx[inside].astype(np.int32))
    assert np.array_equal(xy[inside, 1], ry[inside].astype(np.int32))
    assert np.all(xy[ok & ~inside] == -1)
    assert np.all(np.abs(xy[inside] - np.stack([u, v], 1)[inside]) <= 0.5 + 1e-9)


def test_s_err_brute_force_union():
    """S_err^c = {n : D^c(x_n, y_n) = 1} over 𝒢^base; S_err = ∪_c (
    S:638-640) — checked against the pinhole pixel of every (Gaussian, view)."""
    cams = synth.n3dv_rig(width=120, height=90, num_views=3)
    sc = synth.n3dv_scene(n=3000, seed=31, fx=cams[0].fx)
    n_base = 2500
    s_err = np.zeros(sc.n, np.uint8)
    expect = np.zeros(sc.n, bool)
    for k, cam in enumerate(cams):
        a = synth.random_image(cam, 40 + k); b = synth.random_image(cam, 50 + k)
        o = oracle.error_map(cam, a, b, 0.33, sc.pos_opa, n_base=n_base, s_err=s_err)
        s_err = o["s_err"]
        V = cam.viewmat.astype(np.float64)
        tc = sc.pos_opa[:, :3].astype(np.float64) @ V[:, :3].T + V[:, 3]
        u = float(np.float32(cam.fx)) * tc[:, 0] / tc[:, 2] + float(np.float32(cam.cx))
        v = float(np.float32(cam.fy)) * tc[:, 1] / tc[:, 2] + float(np.float32(cam.cy))
        E = np.abs(a.astype(np.float64) - b).mean(0)
        for i in range(n_base):
            if tc[i, 2] <= cam.near:
                continue
            x = int(np.floor(abs(u[i]) + 0.5) * np.sign(u[i])); y = int(np.floor(abs(v[i]) + 0.5) * np.sign(v[i]))
            if 0 <= x < 120 and 0 <= y < 90 and E[y, x] > 0.33:
                expect[i] = True
    assert not np.any(s_err[n_base:])
    assert np.array_equal(s_err[:n_base].astype(bool), expect[:n_base])
