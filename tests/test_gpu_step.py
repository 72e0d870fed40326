"""GPU parity of the exact step bench.py times: C3 at full size (20 views of
1352×1014, 300k Gaussians, SH3, 30% dynamic) through ShiftStep's captured
CUDA graph — shift, multi-view projection, 20 graph-mode sorts on 20
overlapping streams, forward, list backward, multi-view preprocess, shift
backward ("at BASELINE.json's full sizes, in the launch
configuration bench.py times").

Layered as the comparison policy says: the shift against oracle.shift; then the
oracle is fed the GPU's shifted parameters (a 1e-7 difference in a position
would otherwise move depth bits) and every view's keys, sort, ranges, image
and T, and the gradients summed over the 20 views (then through the shift
backward), are compared with the oracle's.
"""
import numpy as np
import pytest

import oracle
from _parity import grad_compare, record_ties
from paper_2411_14847_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_14847_b200.pipeline import DeviceScene  # noqa: E402
from paper_2411_14847_b200.step import ShiftStep  # noqa: E402

DEV = "cuda"


def np_(t):
    return t.detach().cpu().numpy()


@pytest.mark.slow
def test_c3_captured_step_graph_matches_oracle():
    cams, sc = synth.c3()
    W, H = cams[0].width, cams[0].height
    mu, sigma = synth.shift_offsets(sc, seed=33)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    dL_host = [synth.grad_image(c, 1000 + v, 1.0 / (3 * W * H)) for v, c in enumerate(cams)]
    base = DeviceScene.from_host(sc, DEV)
    stepper = ShiftStep(cams, sc.n, 3, 1 << 22, DEV, streams=20, validate=True)   # bench.py's launch shape
    S = stepper.buffers(base, t(mu), t(sigma), torch.stack([t(d) for d in dL_host]))
    stepper.run(S)                      # warm-up, eager (as bench.py)
    torch.cuda.synchronize()
    graph = stepper.capture(S)
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    stepper.check_overflow()
    stepper.check_numerics()
    mvp = stepper.mvp
    assert mvp.S == len(cams)           # one slot per view: every view's outputs persist

    # a1: the shift
    pos_s, rot_s = np_(S.shifted.pos_opa), np_(S.shifted.rot)
    rp, rr = oracle.shift(sc.pos_opa, sc.rot, mu, sigma, sc.dynamic)
    np.testing.assert_allclose(pos_s, rp, atol=1e-6, rtol=0)
    np.testing.assert_allclose(rot_s, rr, atol=1e-6, rtol=0)
    shifted = synth.Scene(pos_s, sc.scale, rot_s, sc.sh, 3, sc.dynamic)

    K = mvp.pair_counts()
    sum_keys = ("g_pos_opa", "g_scale", "g_rot", "g_sh", "gradstat_sum", "gradstat_cnt",
                "k_pos_opa", "k_scale", "k_rot", "k_sh", "t_pos_opa", "t_scale", "t_rot", "t_sh",
                "t_gradstat")
    ref = None
    gtie = np.zeros(sc.n, bool)
    for v, cam in enumerate(cams):
        ras = mvp.slots[v]
        xy = np_(stepper.records.xy_depth[v])
        box = np_(stepper.records.box[v]).view(np.uint32)
        tiles = np_(stepper.records.tiles[v]).view(np.uint32)
        rows = np_(stepper.records.rows[v]).view(np.uint32)
        # a2 key chain, bit-exact against the oracle's fp32 replica
        o = oracle.project(cam, shifted)
        vis = o["visible"] == 1
        b4 = np.stack([box[:, 0] & 0xFFFF, box[:, 0] >> 16, box[:, 1] & 0xFFFF, box[:, 1] >> 16], 1)
        assert np.array_equal((b4[:, 0] <= b4[:, 1]).astype(np.uint8), o["visible"]), v
        assert np.array_equal(xy[:, 2].view(np.uint32)[vis], o["zbits"][vis]), v
        assert np.array_equal(b4[vis].astype(np.int32), o["box"][vis]), v
        assert np.array_equal(rows, o["rows"]) and np.array_equal(tiles, o["tiles"]), v
        # a3-a5: sorted ids and tile ranges of the graph-mode sort, bit-exact
        keys, ids, ranges = oracle.bin_sort(cam, o)
        assert K[v] == len(ids), v
        assert np.array_equal(np_(ras.sorted_ids[:K[v]]).view(np.uint32), ids), v
        assert np.array_equal(np_(ras.ranges).view(np.uint32), ranges), v
        # a6: image and T on every non-tie pixel
        r = oracle.render(cam, shifted)
        ok = r["tie"] == 0
        frac = record_ties(f"C3 view {v}", r["tie"] == 1)
        assert frac < 1e-3, (v, frac)
        d = np.abs(np_(ras.img) - r["img"])[:, ok].max()
        assert d <= 1e-4, (v, d)
        dT = np.abs(np_(ras.T) - r["T"])
        if dT[ok].max() > 1e-5:
            w = np.unravel_index(np.argmax(np.where(ok, dT, 0)), dT.shape)
            raise AssertionError(f"view {v}: max |ΔT| {dT[ok].max():.3g} at {w} (T {r['T'][w]:.6g}, "
                                 f"accepted {r['nacc'][w]}); {(dT[ok] > 1e-5).sum()} px over 1e-5, "
                                 f"{(dT[ok] > 3e-6).sum()} over 3e-6")
        # a7-a9: per-view oracle gradients, summed over the views (A27)
        b = oracle.render_bwd(cam, shifted, dL_host[v], kappa=True)
        gtie |= b["gtie"] == 1
        if ref is None:
            ref = {k: b[k].copy() for k in sum_keys}
        else:
            for k in sum_keys:
                ref[k] += b[k]
        del b, r
    ok = ~gtie
    record_ties("C3 gradients (union over 20 views)", gtie, int(gtie.sum()), sc.n)
    assert gtie.mean() < 0.01
    g = S.grads
    nc = 16
    gsh = np_(g.sh).transpose(1, 0, 2).reshape(sc.n, -1)[:, :3 * nc].reshape(sc.n, nc, 3)
    for name, a, b_, k, ts in (
            ("pos", np_(g.pos_opa)[:, :3], ref["g_pos_opa"][:, :3], ref["k_pos_opa"][:, :3], ref["t_pos_opa"][:, :3]),
            ("opa", np_(g.pos_opa)[:, 3], ref["g_pos_opa"][:, 3], ref["k_pos_opa"][:, 3], ref["t_pos_opa"][:, 3]),
            ("scale", np_(g.scale)[:, :3], ref["g_scale"][:, :3], ref["k_scale"][:, :3], ref["t_scale"][:, :3]),
            ("rot", np_(g.rot), ref["g_rot"], ref["k_rot"], ref["t_rot"]),
            ("sh", gsh, ref["g_sh"], ref["k_sh"], ref["t_sh"]),
            ("gradstat", np_(g.gradstat_sum), ref["gradstat_sum"], None, ref["t_gradstat"])):
        grad_compare(name, a[ok], b_[ok], None if k is None else k[ok], slack=ts[ok])
    assert np.array_equal(np_(g.gradstat_cnt), ref["gradstat_cnt"])
    # a1 backward: ∂L/∂μ, ∂L/∂σ from the oracle's summed ∂L/∂p′, ∂L/∂q′
    gm, gs = oracle.shift_bwd(sc.rot, sigma, sc.dynamic, ref["g_pos_opa"], ref["g_rot"])
    dyn = sc.dynamic.astype(bool)
    km = ref["k_pos_opa"][:, :3] * dyn[:, None]                 # ∂L/∂μ = mask·∂L/∂p′
    # ∂L/∂σ = P_⊥(Lᵀ(n(q)) ∂L/∂q′)/‖σ‖ with L orthogonal and P_⊥ a projection:
    # every component is bounded by ‖κ_rot‖₂/‖σ‖ (times the mask)
    ks = (np.linalg.norm(ref["k_rot"], axis=1) / np.linalg.norm(sigma.astype(np.float64), axis=1)
          * dyn)[:, None] * np.ones((1, 4))
    tm = ref["t_pos_opa"][:, :3] * dyn[:, None]
    ts_ = (np.linalg.norm(ref["t_rot"], axis=1) / np.linalg.norm(sigma.astype(np.float64), axis=1)
           * dyn)[:, None] * np.ones((1, 4))
    grad_compare("g_mu", np_(g.g_mu)[ok, :3], gm[ok, :3], km[ok], slack=tm[ok])
    grad_compare("g_sigma", np_(g.g_sigma)[ok], gs[ok], ks[ok], slack=ts_[ok])


def test_nonfinite_scan_host_and_graph_mode():
    """dass_scan_nonfinite (DASS_ERR_NUMERICAL): clean buffers pass; one NaN and one
    Inf are counted in graph mode and raise in host mode; ShiftStep.check_numerics
    raises on a poisoned parameter set."""
    from paper_2411_14847_b200 import dass
    x = torch.randn(1 << 20, device=DEV)
    bad = torch.zeros(1, dtype=torch.int32, device=DEV)
    assert dass.dass_scan_nonfinite(x, bad, host_mode=True) == 0
    x[12345] = float("nan")
    x[-1] = float("inf")
    bad.zero_()
    dass.dass_scan_nonfinite(x, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 2
    bad.zero_()
    with pytest.raises(dass.DassError) as ei:
        dass.dass_scan_nonfinite(x, bad, host_mode=True)
    assert ei.value.status == dass.DASS_ERR_NUMERICAL
    cams = [synth.n3dv_rig(width=160, height=120)[v] for v in (0, 1)]
    sc = synth.n3dv_scene(n=4000, seed=9, degree=3, fx=cams[0].fx)
    mu, sigma = synth.shift_offsets(sc, seed=33)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    base = DeviceScene.from_host(sc, DEV)
    stepper = ShiftStep(cams, sc.n, 3, 1 << 20, DEV, streams=2, validate=True)
    dls = torch.stack([t(synth.grad_image(c, 7 + v)) for v, c in enumerate(cams)])
    S = stepper.buffers(base, t(mu), t(sigma), dls)
    stepper.run(S)
    stepper.check_numerics()
    dls[0, 1, 60, 80] = float("nan")   # a NaN in ∂L/∂C reaches the gradients
    stepper.run(S)
    with pytest.raises(dass.DassError) as ei:
        stepper.check_numerics()
    assert ei.value.status == dass.DASS_ERR_NUMERICAL


@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
def test_collective_issued_before_sh_join_sees_complete_payload(graph):
    """ShiftStep.run(collective=…, collective_after_sh=False) — bench.py's shift payload
    at N>1 — issues the exchange while the preprocess's SH part is still on its side
    stream.  A stand-in collective snapshots the payload slice on the stream the
    all_reduce would use: the snapshot must equal the finished payload bit for bit
    (nothing the shift payload holds is written after it), and the SH gradients,
    joined afterwards, must equal a run with the collective after the join."""
    cams = synth.n3dv_rig(width=320, height=240, num_views=6)
    sc = synth.n3dv_scene(n=20000, seed=61, degree=3, fx=cams[0].fx)
    mu, sigma = synth.shift_offsets(sc, seed=34)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    base = DeviceScene.from_host(sc, DEV)
    dls = torch.stack([t(synth.grad_image(c, 70 + v)) for v, c in enumerate(cams)])
    out = []
    for after_sh in (True, False):
        stepper = ShiftStep(cams, sc.n, 3, 1 << 21, DEV, streams=6)
        S = stepper.buffers(base, t(mu), t(sigma), dls)
        snap = torch.empty_like(S.grads.payload("shift"))
        coll = lambda: snap.copy_(S.grads.payload("shift"))
        if graph:
            stepper.run(S)
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                stepper.run(S, collective=coll, collective_after_sh=after_sh)
            snap.zero_()
            gr.replay()
        else:
            stepper.run(S, collective=coll, collective_after_sh=after_sh)
        torch.cuda.synchronize()
        stepper.check_overflow()
        assert torch.equal(snap.view(torch.int32), S.grads.payload("shift").view(torch.int32))
        assert float(S.grads.payload("shift").abs().sum()) > 0
        out.append(S.grads.sh.clone())
    a, b = out
    assert float(b.abs().max()) > 0
    assert float((a - b).abs().max()) <= 1e-5 * float(b.abs().max())
