"""Pins of the f3 oracle (Eq. 1, STE P:389-393, Eq. 2)."""
import json
import os

import numpy as np

import oracle
from paper_2411_14847_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_quant_threshold_and_masked_equals_deleted():
    m = np.array([-3.0, -1e-6, 0.0, 1e-6, 2.0], np.float32)
    assert list(oracle.inherit(m)) == [0, 0, 1, 1, 1]          # Quant(0.5) = 1
    cam, sc = synth.c1()
    mm = np.random.default_rng(0).normal(size=sc.n).astype(np.float32)
    keep = oracle.inherit(mm)
    a = oracle.render(cam, sc, keep=keep)
    idx = np.nonzero(keep)[0]
    b = oracle.render(cam, synth.Scene(sc.pos_opa[idx], sc.scale[idx], sc.rot[idx], sc.sh[:, idx], 0))
    assert np.array_equal(a["img"], b["img"])                    # Eq. 1: Quant = 0 contributes nothing


def test_ste_gradient_closed_forms():
    ex = GOLD["inheritance_quant"][0]
    m = np.array([ex["m"]], np.float32)
    po = np.array([[0, 0, 0, 1.0]], np.float32)
    sc = np.zeros((1, 4), np.float32)
    g = oracle.inherit_bwd(m, po, sc, np.array([[0, 0, 0, 1.0]]), np.zeros((1, 4)))
    assert abs(g[0] - ex["sigmoid_prime"]) < 1e-12                # σ'(3)
    # σ' by central differences of the logistic function; linear in ∂L/∂o_r, ∂L/∂s_r
    rng = np.random.default_rng(1)
    n = 50
    m = rng.normal(size=n).astype(np.float32)
    po = np.concatenate([rng.normal(size=(n, 3)), rng.uniform(0.05, 0.95, (n, 1))], 1).astype(np.float32)
    sc = np.concatenate([rng.uniform(0.01, 0.5, (n, 3)), np.zeros((n, 1))], 1).astype(np.float32)
    gpo, gs = rng.normal(size=(n, 4)), rng.normal(size=(n, 4))
    lam = 0.01
    g = oracle.inherit_bwd(m, po, sc, gpo, gs, lam)
    h = 1e-6
    sig = lambda x: 1 / (1 + np.exp(-x))
    dsig = (sig(m.astype(np.float64) + h) - sig(m.astype(np.float64) - h)) / (2 * h)
    dmop = po[:, 3] * gpo[:, 3] + (sc[:, :3] * gs[:, :3]).sum(1)
    np.testing.assert_allclose(g, (dmop + lam) * dsig, rtol=1e-8, atol=1e-12)
