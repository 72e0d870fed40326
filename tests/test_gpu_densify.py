"""GPU parity of f4 (error-guided densification §3.4 P:167-175 and the
identity-feature render of Eq. 9; readings A44-A47) through the C-ABI,
against the CPU oracle on the same seeded inputs.

Bars: selection, keep flags and index lists bit-exact (the ∇p̄ decision is one
fp32 division on both sides, A44); gathered / copied rows bit-exact; spawned
positions within 1e-6·(1 + |p|) + 1e-5·max s of the oracle (fp32 Box-Muller and
rotation against fp64); the feature render within 1e-4 on non-tie pixels (the
image bar), and with the colours as features it equals dass_render_fwd's image
bit-for-bit (same α decisions, same summation order).
"""
import numpy as np
import pytest

import oracle
from paper_2411_14847_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_14847_b200 import dass  # noqa: E402
from paper_2411_14847_b200.pipeline import DeviceScene, Raster, ViewRecords  # noqa: E402

DEV = "cuda"
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
np_ = lambda x: x.detach().cpu().numpy()


def ws_for(n):
    return torch.empty(dass.dass_partition_workspace(n) // 4 + 1, dtype=torch.int32, device=DEV)


@pytest.mark.parametrize("n", [0, 1, 5000, 300_001])
def test_select_bit_exact(n):
    rng = np.random.default_rng(n + 1)
    gcnt = rng.integers(0, 6, n).astype(np.uint32)
    gsum = (rng.exponential(2e-4, n) * gcnt).astype(np.float32)
    s_err = (rng.uniform(size=n) < 0.15).astype(np.uint8)
    ref, c = oracle.densify_select(gsum, gcnt, s_err, 2e-4, 1e-4)
    m = max(n, 1)
    in_S = torch.zeros(m, dtype=torch.uint8, device=DEV)
    idx = torch.full((m,), -1, dtype=torch.int32, device=DEV)
    counts = torch.zeros(2, dtype=torch.int32, device=DEV)
    dass.dass_densify_select(t(gsum), t(gcnt), t(s_err), 2e-4, 1e-4, in_S, idx, counts, ws_for(n))
    torch.cuda.synchronize()
    assert np.array_equal(np_(in_S)[:n], ref)
    assert np_(counts).tolist() == [c, n - c]
    assert np.array_equal(np_(idx)[:c], np.flatnonzero(ref))


def test_select_from_a_rendered_view():
    """∇p̄ and S_err produced by the GPU renderer and error map themselves."""
    cam = synth.n3dv_rig(width=320, height=240)[4]
    sc = synth.n3dv_scene(n=20_000, seed=81, degree=1, fx=cam.fx)
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(1, sc.n, DEV)
    dass.dass_project(cam, sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, *rec.view(0))
    ras = Raster(cam.width, cam.height, sc.n, 1 << 21, DEV)
    ras.forward(cam, rec.view(0), host_mode=True)
    from paper_2411_14847_b200.pipeline import Grads
    g = Grads.zeros(sc.n, sc.sh_degree, DEV)
    ras.backward(cam, ds, rec.view(0), t(synth.grad_image(cam, 82, 1e-3)), g)
    gt = t(synth.random_image(cam, 83))
    err = torch.empty(cam.height, cam.width, device=DEV)
    s_err = torch.zeros(sc.n, dtype=torch.uint8, device=DEV)
    dass.dass_error_map(cam, ras.img, gt, 0.3, err, None, sc.n, ds.pos_opa, s_err)
    torch.cuda.synchronize()
    gs, gc, se = np_(g.gradstat_sum), np_(g.gradstat_cnt).view(np.uint32), np_(s_err)
    tau = float(np.quantile(gs[gc > 0] / gc[gc > 0], 0.9))
    ref, c = oracle.densify_select(gs, gc, se, tau, 0.5 * tau)
    in_S = torch.zeros(sc.n, dtype=torch.uint8, device=DEV)
    idx = torch.empty(sc.n, dtype=torch.int32, device=DEV)
    counts = torch.zeros(2, dtype=torch.int32, device=DEV)
    dass.dass_densify_select(g.gradstat_sum, g.gradstat_cnt, s_err, tau, 0.5 * tau, in_S, idx,
                             counts, ws_for(sc.n))
    torch.cuda.synchronize()
    assert 0 < c < sc.n and np.array_equal(np_(in_S), ref)
    assert np.array_equal(np_(idx)[:c], np.flatnonzero(ref))


def test_spawn_parity_and_copies():
    sc = synth.n3dv_scene(n=20_000, seed=84, degree=3)
    rng = np.random.default_rng(85)
    sel = np.sort(rng.choice(sc.n, 3001, replace=False)).astype(np.int32)
    K, shrink, o_c, seed = 2, 1.6, 0.1, 987654321
    n_out = sc.n + sel.size * K
    k4 = synth.sh_planes(3)
    out = [torch.full((n_out, 4), np.nan, device=DEV) for _ in range(3)]
    out_sh = torch.full((k4, n_out, 4), np.nan, device=DEV)
    out_dyn = torch.full((n_out,), 7, dtype=torch.uint8, device=DEV)
    dyn = sc.dynamic.astype(np.uint8)
    dass.dass_spawn(3, t(sc.pos_opa), t(sc.scale), t(sc.rot), t(sc.sh), t(dyn), sel.size, t(sel), K,
                    shrink, o_c, seed, out[0], out[1], out[2], out_sh, out_dyn)
    torch.cuda.synchronize()
    po, s, q, sh, dy = np_(out[0]), np_(out[1]), np_(out[2]), np_(out_sh), np_(out_dyn)
    n = sc.n
    assert np.array_equal(po[:n], sc.pos_opa) and np.array_equal(s[:n], sc.scale)
    assert np.array_equal(q[:n], sc.rot) and np.array_equal(sh[:, :n], sc.sh) and np.array_equal(dy[:n], dyn)
    parent = np.repeat(sel, K)
    ref_po, ref_s = oracle.spawn(sel, K, shrink, o_c, seed, sc.pos_opa, sc.scale, sc.rot)
    tol = 1e-6 * (1 + np.abs(sc.pos_opa[parent, :3])) + 1e-5 * np.max(sc.scale[parent, :3], 1, keepdims=True)
    assert np.all(np.abs(po[n:, :3] - ref_po[:, :3]) <= tol)
    assert np.all(po[n:, 3] == np.float32(o_c))
    np.testing.assert_allclose(s[n:, :3], ref_s[:, :3], rtol=1e-6)
    assert np.array_equal(q[n:], sc.rot[parent]) and np.array_equal(sh[:, n:], sc.sh[:, parent])
    assert np.array_equal(dy[n:], dyn[parent])


def test_prune_select_and_gather():
    sc = synth.n3dv_scene(n=50_000, seed=86, degree=2)
    first = 30_000
    ref, c = oracle.prune_keep(sc.pos_opa, first, 0.2)
    pos = t(sc.pos_opa)
    keep = torch.zeros(sc.n, dtype=torch.uint8, device=DEV)
    idx = torch.empty(sc.n, dtype=torch.int32, device=DEV)
    counts = torch.zeros(2, dtype=torch.int32, device=DEV)
    dass.dass_prune_select(pos, first, 0.2, keep, idx, counts, ws_for(sc.n))
    torch.cuda.synchronize()
    assert np.array_equal(np_(keep), ref) and np_(counts).tolist() == [c, sc.n - c]
    m = int(np_(counts)[0])
    k4 = synth.sh_planes(2)
    out = [torch.empty(m, 4, device=DEV) for _ in range(3)]
    out_sh = torch.empty(k4, m, 4, device=DEV)
    out_dyn = torch.empty(m, dtype=torch.uint8, device=DEV)
    dass.dass_gather(2, pos, t(sc.scale), t(sc.rot), t(sc.sh), t(sc.dynamic.astype(np.uint8)), m, idx,
                     out[0], out[1], out[2], out_sh, out_dyn)
    torch.cuda.synchronize()
    kept = np.flatnonzero(ref)
    assert np.array_equal(np_(out[0]), sc.pos_opa[kept]) and np.array_equal(np_(out[1]), sc.scale[kept])
    assert np.array_equal(np_(out[2]), sc.rot[kept]) and np.array_equal(np_(out_sh), sc.sh[:, kept])
    assert np.array_equal(np_(out_dyn), sc.dynamic.astype(np.uint8)[kept])


def render_setup(cam, sc):
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(1, sc.n, DEV)
    dass.dass_project(cam, sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, *rec.view(0))
    ras = Raster(cam.width, cam.height, sc.n, 1 << 21, DEV)
    ras.forward(cam, rec.view(0), host_mode=True)
    return rec, ras


@pytest.mark.parametrize("case", ["c1", "n3dv"])
def test_feature_render_parity(case):
    if case == "c1":
        cam, sc = synth.c1()
    else:
        cam = synth.n3dv_rig(width=301, height=201)[7]
        sc = synth.n3dv_scene(n=15_000, seed=87, degree=0, fx=cam.fx)
    rec, ras = render_setup(cam, sc)
    feat = np.random.default_rng(88).normal(size=(sc.n, 16)).astype(np.float32)
    out = torch.empty(16, cam.height, cam.width, device=DEV)
    xy, co, rgb, box, _, _ = rec.view(0)
    dass.dass_render_features(cam, ras.ranges, ras.sorted_ids, xy, co, box, t(feat), out)
    torch.cuda.synchronize()
    ref, tie = oracle.render_features(cam, sc, feat)
    ok = tie == 0
    d = np.abs(np_(out) - ref)[:, ok]
    assert d.max() <= 1e-4, d.max()
    # the colours as 4-channel features reproduce the forward image bit-for-bit
    c4 = torch.zeros(sc.n, 4, device=DEV)
    c4[:, :3] = rgb[:, :3]
    out4 = torch.empty(4, cam.height, cam.width, device=DEV)
    dass.dass_render_features(cam, ras.ranges, ras.sorted_ids, xy, co, box, c4, out4)
    torch.cuda.synchronize()
    assert torch.equal(out4[:3], ras.img)
    assert torch.count_nonzero(out4[3]) == 0


def test_spawn_edge_cases():
    """m = 0 (copy only), K = 3, SH degree 0 and no dynamics flags."""
    sc = synth.n3dv_scene(n=777, seed=93, degree=0)
    k4 = synth.sh_planes(0)
    for m, K in ((0, 2), (5, 3)):
        sel = np.arange(0, 5 * m, 5, dtype=np.int32)[:m]
        n_out = sc.n + m * K
        out = [torch.full((n_out, 4), np.nan, device=DEV) for _ in range(3)]
        out_sh = torch.full((k4, n_out, 4), np.nan, device=DEV)
        dass.dass_spawn(0, t(sc.pos_opa), t(sc.scale), t(sc.rot), t(sc.sh), None, m,
                        t(sel) if m else None, K, 2.0, 0.05, 11, out[0], out[1], out[2], out_sh)
        torch.cuda.synchronize()
        assert np.array_equal(np_(out[0])[:sc.n], sc.pos_opa)
        if m:
            ref_po, ref_s = oracle.spawn(sel, K, 2.0, 0.05, 11, sc.pos_opa, sc.scale, sc.rot)
            po = np_(out[0])[sc.n:]
            assert np.all(np.abs(po[:, :3] - ref_po[:, :3]) <= 1e-6 * (1 + np.abs(ref_po[:, :3])) + 1e-5)
            np.testing.assert_allclose(np_(out[1])[sc.n:, :3], ref_s[:, :3], rtol=1e-6)
        assert np.isfinite(np_(out_sh)).all()
