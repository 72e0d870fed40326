"""Pins of the f2 oracle: the hash-grid deformation field (§3.3 P:127-129,
supplement §B; readings A41-A43).

What pins what:
  - dense levels index the (N+1)³ lattice bijectively (a wrong stride collides);
  - trilinear interpolation equals scipy's RegularGridInterpolator on the
    lattice values (an independent library routine; wrong weights / corners fail);
  - the spatial hash is XOR-separable with π = (1, 2654435761, 805459861) (S:380s);
  - levels are concatenated in order (level-major table);
  - the MLP against a numpy forward; the zero head is the identity;
  - gradients against central differences of the double forward.
"""
import numpy as np
import pytest

import oracle
from paper_2411_14847_b200 import synth

interp = pytest.importorskip("scipy.interpolate")

LO = np.array([-1.0, -2.0, 0.5], np.float32)
HI = np.array([3.0, 2.0, 4.5], np.float32)


def field(res, log2T, F=1, seed=0, trained=True, table=None):
    f = synth.hash_field(log2T, F, (LO, HI), seed, levels=len(res), trained=trained, res=res)
    if table is not None:
        f.table = np.ascontiguousarray(table, np.float32)
    return f


def lattice_points(N):
    g = np.arange(N + 1, dtype=np.float64) / N
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    u = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    return u


def to_pos(u):
    """Unit-cube coordinates → positions exactly representable on the lattice."""
    p = np.zeros((u.shape[0], 4), np.float32)
    p[:, :3] = (LO + u * (HI - LO)).astype(np.float32)
    return p


def test_dense_level_is_a_bijection_of_the_lattice():
    N = 4                                   # 5³ = 125 ≤ 128 = T → dense
    T = 128
    tab = np.arange(T, dtype=np.float32).reshape(1, T, 1)
    f = field((N,), 7, table=tab)
    vals = oracle.hash_encode(f, to_pos(lattice_points(N)))[:, 0]
    assert np.allclose(vals, np.round(vals), atol=1e-4)        # each a single stored row
    rows = np.round(vals).astype(int)
    assert len(set(rows.tolist())) == (N + 1) ** 3              # no two lattice points collide
    assert rows.min() >= 0 and rows.max() < T


@pytest.mark.parametrize("N,log2T", [(6, 9), (9, 6)])          # dense (343 ≤ 512) and hashed
def test_trilinear_against_scipy(N, log2T):
    f = field((N,), log2T, F=2, seed=3)
    u = lattice_points(N)
    V = oracle.hash_encode(f, to_pos(u))                        # values at the lattice points
    g = np.arange(N + 1) / N
    q = np.random.default_rng(1).uniform(0, 1, size=(300, 3))
    pos = to_pos(q)
    uq = (pos[:, :3].astype(np.float64) - LO) / (HI.astype(np.float64) - LO)
    for ch in range(2):
        rgi = interp.RegularGridInterpolator((g, g, g), V[:, ch].reshape(N + 1, N + 1, N + 1))
        ref = rgi(np.clip(uq, 0, 1))
        got = oracle.hash_encode(f, pos)[:, ch]
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-5)
    # the cell centre is the mean of its 8 corners
    c = to_pos(np.array([[2.5 / N, 1.5 / N, 3.5 / N]]))
    corners = [[2, 1, 3], [3, 1, 3], [2, 2, 3], [3, 2, 3], [2, 1, 4], [3, 1, 4], [2, 2, 4], [3, 2, 4]]
    cv = np.mean([V[(a * (N + 1) + b) * (N + 1) + cc] for a, b, cc in corners], 0)
    np.testing.assert_allclose(oracle.hash_encode(f, c)[0], cv, atol=1e-5)


def test_spatial_hash_constants_and_xor_structure():
    N, log2T = 40, 10                                           # 41³ > 1024 → hashed
    T = 1 << log2T
    tab = np.arange(T, dtype=np.float32).reshape(1, T, 1)
    f = field((N,), log2T, table=tab)
    row = lambda x, y, z: int(round(oracle.hash_encode(f, to_pos(np.array([[x / N, y / N, z / N]])))[0, 0]))
    # π1 = 1: along x the row is x mod T; π2, π3 from SPEC's prime list
    assert [row(x, 0, 0) for x in range(0, 40, 7)] == [x % T for x in range(0, 40, 7)]
    assert row(0, 1, 0) == 2654435761 % T
    assert row(0, 0, 1) == 805459861 % T
    rng = np.random.default_rng(2)
    for _ in range(30):
        x, y, z = (int(v) for v in rng.integers(0, N + 1, 3))
        assert row(x, y, z) == row(x, 0, 0) ^ row(0, y, 0) ^ row(0, 0, z)


def test_levels_concatenate_in_order_and_clamp():
    res = (5, 11, 30)
    f = field(res, 8, F=2, seed=5)
    pos = to_pos(np.random.default_rng(3).uniform(-0.2, 1.2, size=(50, 3)))   # some outside
    full = oracle.hash_encode(f, pos)
    for l, N in enumerate(res):
        single = field((N,), 8, F=2, table=f.table[l:l + 1])
        np.testing.assert_array_equal(full[:, 2 * l:2 * l + 2], oracle.hash_encode(single, pos))
    clamped = pos.copy()
    clamped[:, :3] = np.clip(pos[:, :3], LO, HI)
    np.testing.assert_allclose(full, oracle.hash_encode(f, clamped), atol=1e-12)


def _np_forward(f, pos):
    x = oracle.hash_encode(f, pos)
    H, nin = synth.MLP_HIDDEN, f.inputs
    p = f.mlp.astype(np.float64)
    o = 0
    W1 = p[o:o + H * nin].reshape(H, nin); o += H * nin
    b1 = p[o:o + H]; o += H
    W2 = p[o:o + H * H].reshape(H, H); o += H * H
    b2 = p[o:o + H]; o += H
    W3 = p[o:o + 7 * H].reshape(7, H); o += 7 * H
    b3 = p[o:o + 7]
    h1 = np.maximum(x @ W1.T + b1, 0)
    h2 = np.maximum(h1 @ W2.T + b2, 0)
    return h2 @ W3.T + b3


def test_mlp_against_numpy_and_identity_at_init():
    f = field(synth.HASH_LEVEL_RES, 12, F=4, seed=7)
    pos = to_pos(np.random.default_rng(4).uniform(0, 1, size=(200, 3)))
    mu, sg, _ = oracle.deform(f, pos)
    out = _np_forward(f, pos)
    np.testing.assert_allclose(mu[:, :3], out[:, :3], rtol=1e-12, atol=1e-15)
    assert np.all(mu[:, 3] == 0)
    np.testing.assert_allclose(sg, out[:, 3:] + np.array([1.0, 0, 0, 0]), rtol=1e-12, atol=1e-15)
    assert oracle.hash_params(f.inputs) == f.mlp.size
    # freshly initialised field: μ = 0 and σ = (1,0,0,0) exactly → q' = n(q)
    f0 = field(synth.HASH_LEVEL_RES, 12, F=4, seed=8, trained=False)
    pos = to_pos(np.random.default_rng(5).uniform(0, 1, size=(1000, 3)))
    mu, sg, _ = oracle.deform(f0, pos)
    assert np.all(mu == 0) and np.all(sg == np.array([1.0, 0, 0, 0]))
    q = np.random.default_rng(6).normal(size=(1000, 4)).astype(np.float32)
    _, q2 = oracle.shift(pos, q, mu.astype(np.float32), sg.astype(np.float32))
    np.testing.assert_allclose(q2, q / np.linalg.norm(q.astype(np.float64), axis=1, keepdims=True),
                               atol=1e-7)


def test_gradients_central_differences():
    f = field((4, 9, 20), 8, F=4, seed=9)          # one dense, two hashed levels
    pos = to_pos(np.random.default_rng(7).uniform(0, 1, size=(6, 3)))
    gm, gs = synth.offset_grads(6, 10)
    gt, gp, kt, km = oracle.deform_bwd(f, pos, gm, gs, kappa=True)
    assert np.all(kt >= np.abs(gt) - 1e-15) and np.all(km >= np.abs(gp) - 1e-15)

    def loss(ff):
        mu, sg, tie = oracle.deform(ff, pos)
        assert not tie.any()
        return float((mu * gm).sum() + (sg * gs).sum())

    rng = np.random.default_rng(11)
    touched = np.flatnonzero(np.abs(gt.ravel()) > 0)
    checks = [("table", int(e)) for e in rng.choice(touched, 25, replace=False)]
    checks += [("mlp", int(e)) for e in rng.choice(f.mlp.size, 40, replace=False)]
    for kind, e in checks:
        arr = f.table if kind == "table" else f.mlp
        flat = arr.reshape(-1)
        v0 = flat[e]
        h = np.float32(1e-4 * max(abs(float(v0)), 0.1))   # small: no ReLU flips
        flat[e] = v0 + h; lp = loss(f); up = float(flat[e])
        flat[e] = v0 - h; lm = loss(f); dn = float(flat[e])
        flat[e] = v0
        fd = (lp - lm) / (up - dn)
        an = (gt if kind == "table" else gp).reshape(-1)[e]
        assert abs(fd - an) <= 1e-7 * max(abs(an), 1e-3) + 1e-12, (kind, e, fd, an)
