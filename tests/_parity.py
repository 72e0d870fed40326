"""Shared comparison policy of the GPU parity tests (DESIGN A29/A37).

grad_compare: |Δ| ≤ tol·max(|g_ref|, 1e-2·rms_field(g_ref)); an entry over that
bound may pass only by the κ clause |Δ| ≤ eps_kappa·κ (κ = Σ_px |term| through
|Jacobian|, the fp32 accuracy limit of a cancelling sum), and at most
max_rescue of the entries may need it.  Tie pixels (A29) add the oracle's tie
slack t_* to the bound: at a pixel with one tie decision either branch is a
correct fp32 result, so the entry may differ by the two branches' difference
there; Gaussians at pixels with two or more tie points are excluded (gtie).  Every comparison's counts, and every
image comparison's tie-pixel fraction, are recorded in STATS; with
DASS_PARITY_STATS=<path> the session writes them there as JSON (conftest.py).
"""
from __future__ import annotations

import os

import numpy as np

STATS: list[dict] = []


def _test_name() -> str:
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]


def grad_compare(name, a, b, k=None, tol=1e-3, eps_kappa=1e-5, max_rescue=1e-3, slack=None):
    """slack: the oracle's A29 tie slack t_* (|branch difference| at one-tie
    pixels through |Jacobian|), an absolute allowance added to the bound."""
    a = np.asarray(a, np.float64).reshape(-1)
    b = np.asarray(b, np.float64).reshape(-1)
    rms = float(np.sqrt(np.mean(b ** 2))) if b.size else 0.0
    rel_bound = tol * np.maximum(np.abs(b), 1e-2 * rms)
    err = np.abs(a - b)
    kb = 0.0 if k is None else eps_kappa * np.asarray(k, np.float64).reshape(-1)
    tb = 0.0 if slack is None else np.asarray(slack, np.float64).reshape(-1)
    bad = err > np.maximum(rel_bound, kb) + tb
    rescued = int(((err > rel_bound) & (err <= np.maximum(rel_bound, kb))).sum())
    tie_used = int(((err > np.maximum(rel_bound, kb)) & ~bad).sum())
    worst = float((err / np.maximum(np.abs(b), 1e-2 * rms + 1e-30)).max()) if b.size else 0.0
    STATS.append(dict(test=_test_name(), kind="grad", field=name, n=int(b.size), rescued=rescued,
                      tie_slack_used=tie_used, over=int(bad.sum()), worst_rel=worst))
    assert not bad.any(), f"{name}: {bad.sum()} of {bad.size} over tolerance; worst rel {worst:.3g}"
    # at most max_rescue of the entries (floor: 3, for fields of ~1000 entries)
    assert rescued <= max(3, max_rescue * b.size), f"{name}: {rescued} of {b.size} entries need the κ clause"
    return rescued


def record_ties(where, tie_mask, excluded_gaussians=None, n_gaussians=None):
    frac = float(np.mean(tie_mask)) if np.size(tie_mask) else 0.0
    d = dict(test=_test_name(), kind="tie", where=where, pixels=int(np.size(tie_mask)),
             tie_pixels=int(np.sum(tie_mask)), tie_frac=frac)
    if excluded_gaussians is not None:
        d.update(gtie=int(excluded_gaussians), n=int(n_gaussians))
    STATS.append(d)
    return frac
