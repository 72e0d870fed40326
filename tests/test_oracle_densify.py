"""Pins of the f4 oracle: Eq. 4 selection, spawn densification,
and the identity-feature render of Eq. 9.  Readings A44-A47.

What pins what:
  - Eq. 4 against a literal numpy set evaluation written from the equation, plus
    its degenerate cases (S_err = ∅ and τ_err = τ_pos give the vanilla criterion)
    and monotonicity in S_err;
  - the Philox4x64-10 generator against numpy's independent implementation;
  - spawned positions: the sample mean and covariance of many children of one
    parent against p and Σ = R S Sᵀ Rᵀ from the (separately pinned)
    oracle.rotmat_cov — a transposed R or a dropped scale fails;
  - Eq. 9: with the colours as features it is Eq. 8's image (pinned by closed
    forms); all-ones features give 1 − T (partition of unity).
"""
import numpy as np

import oracle
from paper_2411_14847_b200 import synth


def literal_eq4(gsum, gcnt, s_err, tau_pos, tau_err):
    gbar = np.where(gcnt > 0, gsum.astype(np.float32) / np.maximum(gcnt, 1).astype(np.float32),
                    np.float32(0)).astype(np.float32)
    pos = set(np.flatnonzero(gbar > np.float32(tau_pos)).tolist())
    err = set(np.flatnonzero(s_err).tolist()) & set(np.flatnonzero(gbar > np.float32(tau_err)).tolist())
    return pos | err


def test_eq4_literal_degenerate_and_monotone():
    rng = np.random.default_rng(0)
    n = 5000
    gsum = (rng.exponential(2e-4, n) * rng.integers(0, 5, n)).astype(np.float32)
    gcnt = rng.integers(0, 5, n).astype(np.uint32)
    gsum[gcnt == 0] = 0
    s_err = (rng.uniform(size=n) < 0.2).astype(np.uint8)
    tp, te = 2e-4, 1e-4
    flags, c = oracle.densify_select(gsum, gcnt, s_err, tp, te)
    S = set(np.flatnonzero(flags).tolist())
    assert S == literal_eq4(gsum, gcnt, s_err, tp, te) and c == len(S)
    vanilla, _ = oracle.densify_select(gsum, gcnt, None, tp, te)
    assert set(np.flatnonzero(vanilla).tolist()) == literal_eq4(gsum, gcnt, np.zeros(n, np.uint8), tp, te)
    same, _ = oracle.densify_select(gsum, gcnt, s_err, tp, tp)        # τ_err = τ_pos collapses
    assert np.array_equal(same, vanilla)
    bigger = s_err | (rng.uniform(size=n) < 0.2).astype(np.uint8)      # enlarging S_err never shrinks S
    f2, _ = oracle.densify_select(gsum, gcnt, bigger, tp, te)
    assert np.all(f2 >= flags)
    assert oracle.densify_select(gsum, np.zeros(n, np.uint32), s_err, tp, te)[1] == 0


def test_philox_against_numpy():
    # numpy's Philox increments its 256-bit counter before each block, so the
    # block for counter c is the first output of a generator started at c − 1
    for ctr, key in [((1, 0, 0, 0), (0, 0)), ((6, 0, 0, 0), (7, 9)),
                     ((2 ** 63 + 3, 11, 2 ** 40, 1), (0x44415353, 2 ** 64 - 1))]:
        bg = np.random.Philox(counter=np.array([ctr[0] - 1] + list(ctr[1:]), np.uint64),
                              key=np.array(key, np.uint64))
        ref = bg.random_raw(4).astype(np.uint64)
        assert np.array_equal(oracle.philox4x64(ctr, key), ref), (ctr, key)


def test_spawn_statistics_and_copies():
    rng = np.random.default_rng(1)
    q = rng.normal(size=(1, 4)).astype(np.float32)
    s = np.array([[0.3, 0.05, 0.12, 0.0]], np.float32)
    p = np.array([[1.0, -2.0, 5.0, 0.7]], np.float32)
    K = 40000
    po, sc, z = oracle.spawn(np.array([0]), K, 1.6, 0.1, 1234, p, s, q, want_z=True)
    x = po[:, :3]
    _, Sigma = oracle.rotmat_cov(q[0], s[0, :3])      # Σ = R S Sᵀ Rᵀ (pinned by the geometry tests)
    sd = np.sqrt(np.diag(Sigma))
    assert np.all(np.abs(x.mean(0) - p[0, :3]) < 4 * sd / np.sqrt(K))
    cov = np.cov(x.T)
    assert np.all(np.abs(cov - Sigma) < 0.03 * np.max(np.abs(Sigma)))
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1) < 0.02
    assert np.all(po[:, 3] == 0.1)
    np.testing.assert_allclose(sc[:, :3], np.repeat(s[:, :3].astype(np.float64) / 1.6, K, 0), rtol=1e-15)
    # distinct children and parents draw distinct samples; same seed reproduces
    po2, _ = oracle.spawn(np.array([0, 0]), 3, 1.6, 0.1, 1234, p, s, q)
    assert np.array_equal(po2[:3], po[:3]) and not np.array_equal(po2[:3], po2[3:])


def test_feature_render_equals_colour_render_and_partition_of_unity():
    cam, sc = synth.c1()
    pr = oracle.project(cam, sc)
    feat = pr["rgb"].astype(np.float32)
    M, tie = oracle.render_features(cam, sc, feat)
    ref = oracle.render(cam, sc)
    np.testing.assert_allclose(M, ref["img"], atol=1e-6)
    assert np.array_equal(tie, ref["tie"])
    ones, _ = oracle.render_features(cam, sc, np.ones((sc.n, 16), np.float32))
    np.testing.assert_allclose(ones, np.broadcast_to(1 - ref["T"], ones.shape), atol=1e-12)


def test_prune_keep_definition():
    po = np.zeros((8, 4), np.float32)
    po[:, 3] = [0.001, 0.9, 0.005, 0.0049, 0.5, 0.0, 0.006, 0.004]
    keep, c = oracle.prune_keep(po, 2, 0.005)
    assert keep.tolist() == [1, 1, 1, 0, 1, 0, 1, 0] and c == 5     # base rows kept; o = τ kept
