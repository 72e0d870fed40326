"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, on the
same seeded inputs (paper_2411_14847_b200/synth.py).

Bars (BASELINE.json north star; SURVEY §8(c) comparison policy):
  * keys, sort order, ranges, K, depth bits, pixel boxes, tiles: bit-exact;
  * image ≤ 1e-4 absolute on non-tie pixels, T_final ≤ 1e-5, tie pixels < 1e-3;
  * gradients |Δ| ≤ 1e-3·max(|g_ref|, 1e-2·rms_field) excluding Gaussians
    whose box holds a tie pixel;
  * shift ≤ 1e-6; error map E ≤ 1e-6, D and s_err exact off ties.
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

from paper_2411_14847_b200 import dass  # noqa: E402
from paper_2411_14847_b200.pipeline import DeviceScene, Grads, Raster, ViewRecords  # noqa: E402

DEV = "cuda"


def np_(t):
    return t.detach().cpu().numpy()


def run_view(cam, scene, dL=None, keep=None, bg=None, capacity=1 << 22, lists=True):
    """Project + bin_sort (host mode) + fwd (+ bwd) through the C-ABI.  lists:
    the backward consumes the forward's acceptance lists (else it re-derives
    the accepted set from out_last)."""
    ds = DeviceScene.from_host(scene, DEV)
    rec = ViewRecords(1, scene.n, DEV)
    kd = None if keep is None else torch.from_numpy(keep.astype(np.uint8)).to(DEV)
    dass.dass_project(cam, scene.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, kd,
                      rec.xy_depth[0], rec.conic_opa[0], rec.rgb[0], rec.box[0], rec.rows[0], rec.tiles[0])
    ras = Raster(cam.width, cam.height, scene.n, capacity, DEV, accept_lists=lists)
    keys = torch.empty(max(capacity, 1), dtype=torch.int64, device=DEV)
    K = ras.forward(cam, rec.view(0), host_mode=True, bg=bg, sorted_keys=keys)
    out = dict(rec=rec, ras=ras, K=K, keys=np_(keys[:K]).view(np.uint64), ids=np_(ras.sorted_ids[:K]).view(np.uint32),
               ranges=np_(ras.ranges).view(np.uint32), img=np_(ras.img), T=np_(ras.T),
               last=np_(ras.last).view(np.uint32))
    if dL is not None:
        g = Grads.zeros(scene.n, scene.sh_degree, DEV)
        ras.backward(cam, ds, rec.view(0), torch.from_numpy(dL).to(DEV), g, keep=kd, bg=bg)
        torch.cuda.synchronize()
        out["grads"] = g
    torch.cuda.synchronize()
    return out


def gpu_projection(rec):
    xy = np_(rec.xy_depth[0]); co = np_(rec.conic_opa[0]); rgb = np_(rec.rgb[0])
    box = np_(rec.box[0]).view(np.uint32); tiles = np_(rec.tiles[0]).view(np.uint32)
    lo = xy[:, 3].copy().view(np.uint32)
    ulo = (lo & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float64)
    vlo = (lo >> 16).astype(np.uint16).view(np.float16).astype(np.float64)
    b4 = np.stack([box[:, 0] & 0xFFFF, box[:, 0] >> 16, box[:, 1] & 0xFFFF, box[:, 1] >> 16], 1)
    # the record's conic is the Cholesky form (A, β, γ): B = A·β, C = γ + A·β² (dass.h)
    A, beta, gam = (co[:, k].astype(np.float64) for k in range(3))
    conic = np.stack([A, A * beta, gam + A * beta * beta], 1)
    rows = np_(rec.rows[0]).view(np.uint32)
    # visible = a non-empty box (a visible Gaussian's A50 footprint may still be empty)
    return dict(u=xy[:, 0].astype(np.float64) + ulo, v=xy[:, 1].astype(np.float64) + vlo,
                zbits=xy[:, 2].view(np.uint32), conic=conic, opa=co[:, 3], rgb=rgb[:, :3],
                clampbits=rgb[:, 3].astype(np.int32), box=b4.astype(np.int32), tiles=tiles,
                rows=rows, visible=(b4[:, 0] <= b4[:, 1]).astype(np.uint8))


def check_projection(cam, scene, rec, keep=None):
    o = oracle.project(cam, scene, keep=keep)
    g = gpu_projection(rec)
    vis = o["visible"] == 1
    # key chain: bit-exact
    assert np.array_equal(g["visible"], o["visible"])
    assert np.array_equal(g["zbits"][vis], o["zbits"][vis])
    assert np.array_equal(g["box"][vis], o["box"][vis])
    assert np.array_equal(g["rows"], o["rows"])      # A50 footprints (KEY CHAIN 12-13)
    assert np.array_equal(g["tiles"], o["tiles"])
    # records: fp32 rounding of the fp64 values
    np.testing.assert_allclose(g["u"][vis], o["uvz"][vis, 0], rtol=0, atol=2e-6)
    np.testing.assert_allclose(g["v"][vis], o["uvz"][vis, 1], rtol=0, atol=2e-6)
    np.testing.assert_allclose(g["conic"][vis], o["conic"][vis], rtol=1e-6, atol=1e-7 * np.abs(o["conic"][vis]).max())
    np.testing.assert_allclose(g["rgb"][vis], o["rgb"][vis], rtol=0, atol=1e-5)
    np.testing.assert_allclose(g["opa"][vis], o["opa"][vis], rtol=0, atol=0)
    near0 = np.any(np.abs(o["rgb"][vis]) < 1e-5, axis=1)
    assert np.array_equal(g["clampbits"][vis][~near0], o["clampbits"][vis][~near0])
    return o


def check_binsort(cam, out, g):
    """Layer 1 of the comparison policy: the GPU's sort of its own projection
    equals the oracle's brute-force sort of the same (visible, zbits, box, rows)."""
    keys, ids, ranges = oracle.bin_sort(cam, dict(visible=g["visible"], zbits=g["zbits"], box=g["box"],
                                                  rows=g["rows"]))
    assert out["K"] == len(keys)
    assert np.array_equal(out["keys"], keys)
    assert np.array_equal(out["ids"], ids)
    assert np.array_equal(out["ranges"], ranges)


def check_image(cam, scene, out, keep=None, bg=None, atol=1e-4, max_tie=1e-3):
    o = oracle.render(cam, scene, keep=keep, bg=bg)
    tie = o["tie"] == 1
    frac = record_ties(f"{cam.width}x{cam.height} n={scene.n}", tie)
    assert frac < max_tie, f"tie pixels {frac:.3g} ≥ {max_tie}"
    ok = ~tie
    d = np.abs(out["img"] - o["img"])
    assert d[:, ok].max() <= atol, f"max |Δimg| {d[:, ok].max():.3g} at non-tie pixels"
    assert np.abs(out["T"] - o["T"])[ok].max() <= 1e-5
    # last contributor: the id at out_last−1 is the oracle's last accepted Gaussian
    has = ok & (o["nacc"] > 0)
    li = out["last"][has].astype(np.int64) - 1
    assert np.array_equal(out["ids"][li].astype(np.int64), o["last_id"][has].astype(np.int64))
    return o


def check_grads(cam, scene, out, dL, keep=None, bg=None, tol=1e-3, eps_kappa=1e-5):
    """Every gradient field against the oracle by tests/_parity.grad_compare
    (1e-3 relative with a 1e-2·rms floor; the κ clause may rescue at most 1e-3
    of the entries; one-tie pixels add the oracle's tie slack); Gaussians whose
    box holds a pixel with two or more tie points are excluded (gtie)."""
    o = oracle.render_bwd(cam, scene, dL, keep=keep, bg=bg, kappa=True)
    g = out["grads"]
    ok = o["gtie"] == 0
    record_ties("gradients", o["gtie"] == 1, int((~ok).sum()), scene.n)
    nc = (scene.sh_degree + 1) ** 2
    gsh = np_(g.sh).transpose(1, 0, 2).reshape(scene.n, -1)[:, :3 * nc].reshape(scene.n, nc, 3)
    pairs = [("pos", np_(g.pos_opa)[:, :3], o["g_pos_opa"][:, :3], o["k_pos_opa"][:, :3], o["t_pos_opa"][:, :3]),
             ("opa", np_(g.pos_opa)[:, 3], o["g_pos_opa"][:, 3], o["k_pos_opa"][:, 3], o["t_pos_opa"][:, 3]),
             ("scale", np_(g.scale)[:, :3], o["g_scale"][:, :3], o["k_scale"][:, :3], o["t_scale"][:, :3]),
             ("rot", np_(g.rot), o["g_rot"], o["k_rot"], o["t_rot"]),
             ("sh", gsh, o["g_sh"], o["k_sh"], o["t_sh"]),
             ("gradstat", np_(g.gradstat_sum), o["gradstat_sum"], None, o["t_gradstat"])]
    for name, a, b, k, ts in pairs:
        grad_compare(name, a[ok], b[ok], None if k is None else k[ok], tol=tol, eps_kappa=eps_kappa,
                     slack=ts[ok])
    assert np.array_equal(np_(g.gradstat_cnt), o["gradstat_cnt"])
    return o


# ---------------------------------------------------------------- tests ----

@pytest.mark.parametrize("lists", [True, False])
def test_c1_full_chain_parity(lists):
    """Config C1 (64×64, 1k Gaussians, SH0): every output against the oracle."""
    cam, sc = synth.c1()
    dL = synth.grad_image(cam, 101)
    out = run_view(cam, sc, dL=dL, lists=lists)
    check_projection(cam, sc, out["rec"])
    check_binsort(cam, out, gpu_projection(out["rec"]))
    check_image(cam, sc, out)
    check_grads(cam, sc, out, dL)


@pytest.mark.parametrize("lists", [True, False])
@pytest.mark.parametrize("W,H,n,deg,seed", [(100, 70, 3000, 1, 11), (333, 177, 20000, 3, 12),
                                            (16, 16, 50, 2, 13), (1, 1, 20, 0, 14), (17, 300, 5000, 3, 15)])
def test_ragged_sizes_parity(W, H, n, deg, seed, lists):
    """Ragged tails (W, H not multiples of 16), several tiles, degrees 0-3."""
    cam = synth.n3dv_rig(width=W, height=H)[seed % 20]
    sc = synth.n3dv_scene(n=n, seed=seed, degree=deg, fx=cam.fx)
    dL = synth.grad_image(cam, seed + 1)
    bg = np.array([0.1, 0.5, 0.9], np.float32)
    out = run_view(cam, sc, dL=dL, bg=bg, lists=lists)
    check_projection(cam, sc, out["rec"])
    check_binsort(cam, out, gpu_projection(out["rec"]))
    check_image(cam, sc, out, bg=bg)
    check_grads(cam, sc, out, dL, bg=bg)


def test_empty_and_all_culled():
    cam = synth.tiny_camera(40, 24)
    sc = synth.random_scene(30, cam, seed=3)
    sc.pos_opa[:, 2] = -2.0  # all behind the camera
    bg = np.array([0.3, 0.2, 0.1], np.float32)
    out = run_view(cam, sc, dL=synth.grad_image(cam, 4), bg=bg)
    assert out["K"] == 0 and not out["ranges"].any()
    np.testing.assert_array_equal(out["img"], np.broadcast_to(bg[:, None, None], out["img"].shape))
    assert np.all(out["T"] == 1.0)
    assert not np_(out["grads"].pos_opa).any()


def test_masked_equals_deleted_bit_exact():
    """Eq. 1 with Quant = 0 ≡ deleting the Gaussian, bit-exact on GPU."""
    cam, sc = synth.c1()
    keep = (np.arange(sc.n) % 4 != 1).astype(np.uint8)
    a = run_view(cam, sc, keep=keep)
    idx = np.nonzero(keep)[0]
    sd = synth.Scene(sc.pos_opa[idx], sc.scale[idx], sc.rot[idx], sc.sh[:, idx], 0)
    b = run_view(cam, sd)
    assert np.array_equal(a["img"], b["img"]) and np.array_equal(a["T"], b["T"])
    check_image(cam, sc, a, keep=keep)


def test_equal_depth_ties_bit_exact():
    """A planar scene (all depth bits equal): order by index (A03)."""
    cam = synth.tiny_camera(80, 64)
    sc = synth.random_scene(2000, cam, seed=21)
    sc.pos_opa[:, 2] = 3.0
    out = run_view(cam, sc)
    g = gpu_projection(out["rec"])
    assert len(np.unique(g["zbits"][g["visible"] == 1])) == 1
    check_binsort(cam, out, g)
    check_image(cam, sc, out, max_tie=3e-3)   # 2000 splats on one plane: more near-threshold pixels


def test_capacity_overflow_host_and_graph_mode():
    cam, sc = synth.c1()
    with pytest.raises(dass.DassError) as ei:
        run_view(cam, sc, capacity=100)
    assert ei.value.status == dass.DASS_ERR_CAPACITY
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(1, sc.n, DEV)
    dass.dass_project(cam, 0, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, *rec.view(0))
    ras = Raster(cam.width, cam.height, sc.n, 100, DEV)
    ras.forward(cam, rec.view(0), host_mode=False)
    torch.cuda.synchronize()
    K, flag = np_(ras.num_pairs).view(np.uint32)
    assert flag == 1 and K > 100 and not np_(ras.ranges).any()


def test_project_views_equals_per_view():
    cams = synth.n3dv_rig(width=200, height=150, num_views=20)
    sc = synth.n3dv_scene(n=5000, seed=5, fx=cams[0].fx)
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(len(cams), sc.n, DEV)
    dass.dass_project_views(cams, 3, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, rec.xy_depth,
                            rec.conic_opa, rec.rgb, rec.box, rec.rows, rec.tiles)
    one = ViewRecords(1, sc.n, DEV)
    for v in (0, 7, 16, 19):
        dass.dass_project(cams[v], 3, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, *one.view(0))
        for a, b in zip(rec.view(v), one.view(0)):
            assert torch.equal(a, b)


def test_project_views_part_equals_all():
    """The split projection (keys on one stream, records on another while the
    keys' consumer could run) gives dass_project_views' bytes; the keys part alone
    already holds everything dass_bin_sort reads."""
    cams = synth.n3dv_rig(width=200, height=150, num_views=5)
    sc = synth.n3dv_scene(n=7001, seed=6, fx=cams[0].fx)
    sc.pos_opa[::97, 3] = 0.002            # some Gaussians culled by opacity
    ds = DeviceScene.from_host(sc, DEV)
    keep = torch.from_numpy((np.arange(sc.n) % 5 != 0).astype(np.uint8)).to(DEV)
    args = lambda r: (r.xy_depth, r.conic_opa, r.rgb, r.box, r.rows, r.tiles)
    ref = ViewRecords(len(cams), sc.n, DEV)
    dass.dass_project_views(cams, 3, ds.pos_opa, ds.scale, ds.rot, ds.sh, keep, *args(ref))
    rec = ViewRecords(len(cams), sc.n, DEV)
    for t in args(rec):
        t.view(torch.uint8).fill_(0xA5)     # poison: every byte must be written
    dass.dass_project_views_part(dass.DASS_PROJECT_KEYS, cams, 3, ds.pos_opa, ds.scale, ds.rot,
                                 ds.sh, keep, *args(rec))
    torch.cuda.synchronize()
    assert torch.equal(rec.xy_depth[..., 2], ref.xy_depth[..., 2])
    for a, b in zip((rec.box, rec.rows, rec.tiles), (ref.box, ref.rows, ref.tiles)):
        assert torch.equal(a, b)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        dass.dass_project_views_part(dass.DASS_PROJECT_RECORDS, cams, 3, ds.pos_opa, ds.scale,
                                     ds.rot, ds.sh, keep, *args(rec))
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    for a, b in zip(args(rec), args(ref)):
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))
    with pytest.raises(dass.DassError):
        dass.dass_project_views_part(0, cams, 3, ds.pos_opa, ds.scale, ds.rot, ds.sh, keep,
                                     *args(rec))


def test_shift_parity():
    cams, sc = synth.c3(n=20000, num_views=1)
    mu, sigma = synth.shift_offsets(sc, seed=33)
    sigma[:5] = 0  # ‖σ‖ < 1e-8 → identity
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    pos, rot, m, s, dyn = t(sc.pos_opa), t(sc.rot), t(mu), t(sigma), t(sc.dynamic)
    po, ro = torch.empty_like(pos), torch.empty_like(rot)
    dass.dass_apply_shift(pos, rot, m, s, dyn, po, ro)
    ref_p, ref_r = oracle.shift(sc.pos_opa, sc.rot, mu, sigma, sc.dynamic)
    np.testing.assert_allclose(np_(po), ref_p, atol=1e-6, rtol=0)
    np.testing.assert_allclose(np_(ro), ref_r, atol=1e-6, rtol=0)
    off = sc.dynamic == 0
    assert np.array_equal(np_(po)[off], sc.pos_opa[off]) and np.array_equal(np_(ro)[off], sc.rot[off])
    g = np.random.default_rng(2)
    gp = g.normal(size=(sc.n, 4)).astype(np.float32)
    gq = g.normal(size=(sc.n, 4)).astype(np.float32)
    gm, gs = torch.zeros_like(pos), torch.zeros_like(rot)
    dass.dass_apply_shift_bwd(rot, s, dyn, t(gp), t(gq), gm, gs)
    rm, rs = oracle.shift_bwd(sc.rot, sigma, sc.dynamic, gp.astype(np.float64), gq.astype(np.float64))
    np.testing.assert_allclose(np_(gm)[:, :3], rm[:, :3], atol=1e-6)
    np.testing.assert_allclose(np_(gs), rs, atol=1e-5, rtol=1e-5)
    # in place
    dass.dass_apply_shift(pos, rot, m, s, dyn, pos, rot)
    np.testing.assert_allclose(np_(pos), ref_p, atol=1e-6, rtol=0)


def test_error_map_parity():
    cams = synth.meetroom_rig(width=160, height=90, num_views=3)
    sc = synth.n3dv_scene(n=8000, seed=41, fx=cams[0].fx)
    n_base = 6000
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    s_err = torch.zeros(sc.n, dtype=torch.uint8, device=DEV)
    ref = np.zeros(sc.n, np.uint8)
    tie_any = np.zeros(sc.n, bool)
    for k, cam in enumerate(cams):
        a = synth.random_image(cam, 60 + k); b = synth.random_image(cam, 70 + k)
        err = torch.empty(cam.height, cam.width, device=DEV)
        dm = torch.zeros((cam.height * cam.width + 31) // 32, dtype=torch.int32, device=DEV)
        dass.dass_error_map(cam, t(a), t(b), 0.3, err, dm, n_base, t(sc.pos_opa), s_err)
        o = oracle.error_map(cam, a, b, 0.3, sc.pos_opa, n_base=n_base, s_err=ref)
        ref = o["s_err"]
        tie_any |= o["tie_g"] == 1
        np.testing.assert_allclose(np_(err), o["err"], atol=1e-6)
        bits = np.unpackbits(np_(dm).view(np.uint8), bitorder="little")[:cam.height * cam.width]
        okp = o["tie_px"].reshape(-1) == 0
        assert np.array_equal(bits[okp], o["D"].reshape(-1)[okp])
    torch.cuda.synchronize()
    got = np_(s_err)
    assert not got[n_base:].any()
    assert np.array_equal(got[~tie_any], ref[~tie_any])


@pytest.mark.parametrize("cfg", ["c1", pytest.param("c2", marks=pytest.mark.slow)])
def test_render_stats_match_oracle_counts(cfg):
    """dass_render_stats' scene statistics (P_fwd, P_bwd, accepted,
    terminated pixels, K) against the oracle's exact counts on C1 and C2; the
    tie pixels' counts are the only allowed slack."""
    if cfg == "c1":
        cam, sc = synth.c1()
    else:
        cam, sc = synth.c2()
    out = run_view(cam, sc, capacity=1 << 22)
    ras, rec = out["ras"], out["rec"]
    cnt = torch.zeros(8, dtype=torch.int64, device=DEV)
    dass.dass_render_stats(cam, ras.ranges, ras.sorted_ids, rec.xy_depth[0], rec.conic_opa[0],
                           rec.box[0], ras.T, ras.last, cnt)
    c = np_(cnt)
    o = oracle.render(cam, sc)
    ok = o["tie"] == 0
    # counts agree exactly away from tie pixels; allow the tie pixels' share
    slack = int(o["pfwd"][~ok].sum()) + 1
    assert abs(int(c[0]) - int(o["pfwd"].sum())) <= slack
    assert abs(int(c[1]) - int(o["pbwd"].sum())) <= slack
    assert abs(int(c[2]) - int(o["nacc"].sum())) <= slack
    assert abs(int(c[3]) - int(o["term"].sum())) <= (~ok).sum()
    assert int(c[4]) == out["K"]


@pytest.mark.slow
def test_c2_full_size_parity():
    """Config C2 at full size (1352×1014, 300k Gaussians, SH3) in the launch
    configuration bench.py times: image and every gradient vs the oracle's
    scatter form (identical per-pixel op sequence at O(Σ box area) cost)."""
    cam, sc = synth.c2()
    dL = synth.grad_image(cam, 202)
    out = run_view(cam, sc, dL=dL, capacity=1 << 24)
    check_projection(cam, sc, out["rec"])
    check_binsort(cam, out, gpu_projection(out["rec"]))
    check_image(cam, sc, out)
    check_grads(cam, sc, out, dL)


def test_multiview_pass_matches_oracle_sum():
    """Two-phase backward over several views on overlapping streams (the bench's
    launch configuration, streams < views so slots are reused) equals the sum of
    per-view oracle gradients (A27); every view's image against the oracle."""
    from paper_2411_14847_b200.pipeline import MultiViewPass, project_all
    cams = synth.n3dv_rig(width=160, height=120, num_views=5)
    sc = synth.n3dv_scene(n=6000, seed=55, degree=3, fx=cams[0].fx)
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(len(cams), sc.n, DEV)
    dLs = np.stack([synth.grad_image(c, 600 + v) for v, c in enumerate(cams)])
    g = Grads.zeros(sc.n, 3, DEV)
    mv = MultiViewPass(cams, sc.n, 1 << 20, DEV, streams=3)
    project_all(cams, ds, rec)
    # the images of the views that reuse a slot are overwritten: keep a copy per
    # view on the view's own stream right after its forward
    imgs = [torch.empty(3, 120, 160, device=DEV) for _ in cams]
    Ts = [torch.empty(120, 160, device=DEV) for _ in cams]

    def keep_image(v, st):
        with torch.cuda.stream(st):
            ras = mv.slots[v % mv.S]
            imgs[v].copy_(ras.img)
            Ts[v].copy_(ras.T)
    mv.before_bwd = keep_image
    mv.run(ds, rec, torch.from_numpy(dLs).to(DEV), g)
    torch.cuda.synchronize()
    assert mv.overflowed_views() == []
    ref = None
    gtie = np.zeros(sc.n, bool)
    for v, cam in enumerate(cams):
        o = oracle.render_bwd(cam, sc, dLs[v], kappa=True)
        gtie |= o["gtie"] == 1
        if ref is None:
            ref = {k: o[k].copy() for k in ("g_pos_opa", "g_scale", "g_rot", "g_sh", "gradstat_sum",
                                            "gradstat_cnt", "k_pos_opa", "k_scale", "k_rot", "k_sh",
                                            "t_pos_opa", "t_scale", "t_rot", "t_sh", "t_gradstat")}
        else:
            for k in ref:
                ref[k] += o[k]
        # the view's image and transmittance (non-tie pixels)
        r = oracle.render(cam, sc)
        ok = r["tie"] == 0
        record_ties(f"multiview view {v}", r["tie"] == 1)
        assert (~ok).mean() < 1e-3
        assert np.abs(np_(imgs[v]) - r["img"])[:, ok].max() <= 1e-4, v
        assert np.abs(np_(Ts[v]) - r["T"])[ok].max() <= 1e-5, v
    ok = ~gtie
    record_ties("multiview gradients", gtie, int(gtie.sum()), sc.n)
    nc = 16
    gsh = np_(g.sh).transpose(1, 0, 2).reshape(sc.n, -1)[:, :3 * nc].reshape(sc.n, nc, 3)
    for name, a, b, k, ts in (("pos", np_(g.pos_opa), ref["g_pos_opa"], ref["k_pos_opa"], ref["t_pos_opa"]),
                              ("scale", np_(g.scale)[:, :3], ref["g_scale"][:, :3], ref["k_scale"][:, :3],
                               ref["t_scale"][:, :3]),
                              ("rot", np_(g.rot), ref["g_rot"], ref["k_rot"], ref["t_rot"]),
                              ("sh", gsh, ref["g_sh"], ref["k_sh"], ref["t_sh"]),
                              ("gradstat", np_(g.gradstat_sum), ref["gradstat_sum"], None, ref["t_gradstat"])):
        grad_compare(name, a[ok], b[ok], None if k is None else k[ok], slack=ts[ok])
    assert np.array_equal(np_(g.gradstat_cnt), ref["gradstat_cnt"])


@pytest.mark.slow
def test_c4_full_size_render_and_error_map():
    """Config C4 (Meet-Room 1280×720, 200k Gaussians, SH3) at full size: one
    view's image and gradients, then the error map + S_err against a GT
    rendered from a perturbed scene (5% of the Gaussians moved, §8(d) C4)."""
    cams, sc = synth.c4()
    cam = cams[4]
    dL = synth.grad_image(cam, 404)
    out = run_view(cam, sc, dL=dL, capacity=1 << 23)
    check_projection(cam, sc, out["rec"])
    check_binsort(cam, out, gpu_projection(out["rec"]))
    check_image(cam, sc, out)
    check_grads(cam, sc, out, dL)
    g = np.random.default_rng(44)
    moved = synth.Scene(sc.pos_opa.copy(), sc.scale, sc.rot, sc.sh, 3)
    sel = g.uniform(size=sc.n) < 0.05
    moved.pos_opa[sel, :3] += g.normal(0, 0.05, size=(sel.sum(), 3)).astype(np.float32)
    gt = run_view(cam, moved)["img"].astype(np.float32)
    rendered = out["img"].astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    err = torch.empty(cam.height, cam.width, device=DEV)
    dm = torch.zeros((cam.height * cam.width + 31) // 32, dtype=torch.int32, device=DEV)
    s_err = torch.zeros(sc.n, dtype=torch.uint8, device=DEV)
    dass.dass_error_map(cam, t(rendered), t(gt), 0.10, err, dm, sc.n, t(sc.pos_opa), s_err)
    o = oracle.error_map(cam, rendered, gt, 0.10, sc.pos_opa)
    torch.cuda.synchronize()
    np.testing.assert_allclose(np_(err), o["err"], atol=1e-6)
    bits = np.unpackbits(np_(dm).view(np.uint8), bitorder="little")[:cam.height * cam.width]
    okp = o["tie_px"].reshape(-1) == 0
    assert np.array_equal(bits[okp], o["D"].reshape(-1)[okp])
    okg = o["tie_g"] == 0
    assert np.array_equal(np_(s_err)[okg], o["s_err"][okg])
    assert o["D"].mean() > 0.001 and o["s_err"].sum() > 100   # the perturbation is visible


@pytest.mark.slow
def test_c5_full_size_parity():
    """Config C5 (1M Gaussians, 1352×1014, SH3, smaller splats) at full size."""
    cams, sc = synth.c5()
    cam = cams[12]
    dL = synth.grad_image(cam, 505)
    out = run_view(cam, sc, dL=dL, capacity=1 << 24)
    check_projection(cam, sc, out["rec"])
    check_binsort(cam, out, gpu_projection(out["rec"]))
    check_image(cam, sc, out)
    check_grads(cam, sc, out, dL)


def test_inheritance_mask_and_ste_gradient():
    """f3 (Eq. 1 + STE + Eq. 2's mask loss): keep bit-exact; g_m from the GPU
    gradients of a masked render equals the oracle's STE chain of the oracle's
    gradients (within the gradient tolerance)."""
    cam = synth.n3dv_rig(width=200, height=150)[9]
    sc = synth.n3dv_scene(n=8000, seed=66, degree=2, fx=cam.fx)
    m = np.random.default_rng(6).normal(0.3, 1.0, size=sc.n).astype(np.float32)
    m[:4] = 0.0
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    keep = torch.empty(sc.n, dtype=torch.uint8, device=DEV)
    dass.dass_inherit_mask(t(m), keep)
    ref_keep = oracle.inherit(m)
    assert np.array_equal(np_(keep), ref_keep)
    dL = synth.grad_image(cam, 606)
    out = run_view(cam, sc, dL=dL, keep=ref_keep)
    g = out["grads"]
    gm = torch.zeros(sc.n, device=DEV)
    dass.dass_inherit_mask_bwd(t(m), t(sc.pos_opa), t(sc.scale), g.pos_opa, g.scale, 0.01, gm)
    torch.cuda.synchronize()
    o = oracle.render_bwd(cam, sc, dL, keep=ref_keep, kappa=True)
    ref = oracle.inherit_bwd(m, sc.pos_opa, sc.scale, o["g_pos_opa"], o["g_scale"], 0.01)
    kap = oracle.inherit_bwd(m, sc.pos_opa, np.abs(sc.scale), o["k_pos_opa"], o["k_scale"], 0.0)
    tsl = oracle.inherit_bwd(m, sc.pos_opa, np.abs(sc.scale), o["t_pos_opa"], o["t_scale"], 0.0)
    ok = o["gtie"] == 0
    grad_compare("g_m", np_(gm)[ok], ref[ok], np.abs(kap[ok]), slack=np.abs(tsl[ok]))
    # culled Gaussians (Quant = 0) get only the mask-loss term λ·σ'(m)
    off = ref_keep == 0
    np.testing.assert_allclose(np_(gm)[off], ref[off], rtol=1e-5, atol=1e-9)


@pytest.mark.parametrize("W,H,lam,seed,off,ds", [(100, 70, 0.2, 1, 0, 1.0), (37, 300, 0.5, 2, 0, 1.0),
                                                  (1, 1, 0.2, 3, 0, 1.0), (1352, 1014, 0.2, 4, 0, 1.0),
                                                  (64, 40, 0.3, 5, 1, 1.0), (96, 64, 1.0, 6, 0, 0.5)])
def test_fidelity_loss_parity(W, H, lam, seed, off, ds):
    """f1 (Eq. 3): loss value and ∂L/∂img against the oracle (direct windows);
    ds = 0.5 is SPEC's D-SSIM (1 − SSIM)/2, 1.0 the 3DGS code's 1 − SSIM (A39).
    W % 4 == 0 with 16-B aligned planes stages tiles by TMA (100, 1352); odd
    widths (37, 1) and a base offset by one float (off = 1) take the load path."""
    g = np.random.default_rng(seed)
    img = g.uniform(0, 1, size=(3, H, W)).astype(np.float32)
    gt = np.clip(img + g.normal(0, 0.1, size=img.shape), 0, 1).astype(np.float32)
    gt[:, : H // 3] = img[:, : H // 3]   # an identical band (sign(0) = 0, S = 1 region)

    def t(a):
        buf = torch.empty(a.size + off, dtype=torch.float32, device=DEV)
        v = buf[off:].view(a.shape)
        v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return v
    ws = torch.empty(dass.dass_fidelity_loss_workspace(W, H) // 4 + 64, dtype=torch.float32, device=DEV)
    loss = torch.zeros(3, device=DEV)
    dL = torch.empty(3, H, W, device=DEV)
    dass.dass_fidelity_loss(t(img), t(gt), lam, ws, loss, dL, dssim_scale=ds)
    torch.cuda.synchronize()
    L, l1, ssim, ref = oracle.fidelity_loss(img, gt, lam, dssim_scale=ds)
    got = np_(loss)
    assert got[0] == pytest.approx(L, rel=1e-5, abs=1e-7)
    assert got[1] == pytest.approx(l1, rel=1e-5, abs=1e-7)
    assert got[2] == pytest.approx(ssim, rel=1e-5)
    d = np_(dL)
    rms = np.sqrt(np.mean(ref ** 2))
    assert np.all(np.abs(d - ref) <= 1e-3 * np.abs(ref) + 1e-3 * rms)


def test_dense_tiles_sort_past_shared_memory():
    """Tiles with lists of thousands of pairs (onesweep blocks of 2048 keys end
    inside one tile's run): keys, ids and ranges stay bit-exact (A03/A04), and so
    does the planar equal-depth case inside one long tile."""
    cam = synth.tiny_camera(48, 48)
    sc = synth.random_scene(12000, cam, seed=77)
    g = np.random.default_rng(77)
    # squeeze every mean into the central 2×2 tiles with small footprints
    z = sc.pos_opa[:, 2]
    sc.pos_opa[:, 0] = (g.uniform(-6, 6, sc.n) * z / cam.fx).astype(np.float32)
    sc.pos_opa[:, 1] = (g.uniform(-6, 6, sc.n) * z / cam.fy).astype(np.float32)
    sc.scale[:, :3] = (np.abs(sc.scale[:, :3]) * 0.3).astype(np.float32)
    sc.pos_opa[:3000, 2] = 3.0              # a planar slice: equal depth bits, ordered by id
    out = run_view(cam, sc, capacity=1 << 20)
    r = out["ranges"]
    assert (r[:, 1] - r[:, 0]).max() > 4096
    check_binsort(cam, out, gpu_projection(out["rec"]))


@pytest.mark.parametrize("n,lo,hi", [(800, 513, 1024), (3000, 1025, 4096), (40000, 4097, 1 << 30)],
                         ids=["list_800", "list_3000", "list_40000"])
def test_long_tile_lists_bit_exact(n, lo, hi):
    """Tile lists of ~800, ~3000 and ~40000 pairs next to short ones (one tile
    holds most of the pairs: the onesweep blocks of 2048 keys end inside it), with
    a planar slice of equal depth bits so the id order inside a tile is checked
    too (A03/A04)."""
    cam = synth.tiny_camera(48, 48)
    sc = synth.random_scene(n, cam, seed=78)
    g = np.random.default_rng(78)
    z = sc.pos_opa[:, 2]
    sc.pos_opa[:, 0] = (g.uniform(-5, 5, sc.n) * z / cam.fx).astype(np.float32)
    sc.pos_opa[:, 1] = (g.uniform(-5, 5, sc.n) * z / cam.fy).astype(np.float32)
    sc.scale[:, :3] = (np.abs(sc.scale[:, :3]) * 0.3).astype(np.float32)
    sc.pos_opa[: n // 4, 2] = 3.0
    out = run_view(cam, sc, capacity=1 << 21)
    c = out["ranges"][:, 1] - out["ranges"][:, 0]
    assert lo <= c.max() <= hi
    check_binsort(cam, out, gpu_projection(out["rec"]))


@pytest.mark.parametrize("W,H,n", [(1352, 1014, 30000), (4096, 4096, 70000)],
                         ids=["c3_image", "image_4096"])
def test_sort_many_tiles_bit_exact(W, H, n):
    """dass_bin_sort with 5440 and 65536 tiles (2 tile-digit passes, the second
    one full at 4096²) against the oracle's brute-force sort (A03/A04)."""
    cam = synth.tiny_camera(W, H)
    sc = synth.random_scene(n, cam, seed=79)
    sc.scale[:, :3] = (np.abs(sc.scale[:, :3]) * 0.5).astype(np.float32)
    out = run_view(cam, sc, capacity=1 << 22)
    assert out["K"] > n
    check_binsort(cam, out, gpu_projection(out["rec"]))


@pytest.mark.parametrize("case", ["c3_view", "dense_tiles", "overflow"])
def test_bin_sort_shared_equals_bin_sort(case):
    """dass_bin_sort_shared (the fixed, looping pair-pass grid the multi-view step uses)
    gives bit for bit dass_bin_sort's keys, ids, ranges and (K, overflow): a C3-size view
    (~1.3M pairs, hundreds of key tiles per block), a dense-tile scene with tile lists past
    4096 pairs, and a capacity overflow (graph mode: flag set, every range empty)."""
    if case == "dense_tiles":
        cam = synth.tiny_camera(48, 48)
        sc = synth.random_scene(40000, cam, seed=78)
        g = np.random.default_rng(78)
        z = sc.pos_opa[:, 2]
        sc.pos_opa[:, 0] = (g.uniform(-5, 5, sc.n) * z / cam.fx).astype(np.float32)
        sc.pos_opa[:, 1] = (g.uniform(-5, 5, sc.n) * z / cam.fy).astype(np.float32)
        sc.scale[:, :3] = (np.abs(sc.scale[:, :3]) * 0.3).astype(np.float32)
        sc.pos_opa[:10000, 2] = 3.0
    else:
        cams, sc = synth.c3()
        cam = cams[3]
    cap = 1 << 16 if case == "overflow" else 1 << 22
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(1, sc.n, DEV)
    dass.dass_project(cam, sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None,
                      rec.xy_depth[0], rec.conic_opa[0], rec.rgb[0], rec.box[0], rec.rows[0], rec.tiles[0])
    out = []
    for shared in (False, True):
        ras = Raster(cam.width, cam.height, sc.n, cap, DEV)
        keys = torch.zeros(cap, dtype=torch.int64, device=DEV)
        ras.sorted_ids.fill_(-1)
        ras.ranges.fill_(-1)
        ras.sort(cam, rec.view(0), sorted_keys=keys, shared=shared)
        torch.cuda.synchronize()
        out.append((np_(ras.num_pairs), np_(keys), np_(ras.sorted_ids), np_(ras.ranges)))
    (na, ka, ia, ra), (nb, kb, ib, rb) = out
    assert np.array_equal(na, nb)
    assert np.array_equal(ra, rb)
    if case == "overflow":
        assert na[1] == 1 and na[0] > cap and not ra.any()
        return
    K = int(na[0])
    assert na[1] == 0 and K > (100000 if case == "c3_view" else 4096)
    assert np.array_equal(ka[:K], kb[:K]) and np.array_equal(ia[:K], ib[:K])
