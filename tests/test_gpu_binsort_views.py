"""dass_bin_sort_views (a3-a5 batched over the views of one timestep) against
the oracle's brute-force sort of each view (small multi-view scenes, ragged
sizes, equal-depth ties) and against per-view dass_bin_sort at BASELINE.json's
full C3 size (20 views × 300k Gaussians); capacity overflow per view.
Bit-exact throughout (integer work)."""
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


def np_(t):
    return t.detach().cpu().numpy()


def batched(cams, rec, n, cap):
    V = len(cams)
    T = ((cams[0].width + 15) // 16) * ((cams[0].height + 15) // 16)
    ws = torch.empty(max(dass.dass_bin_sort_views_workspace(V, n, cap), 16), dtype=torch.uint8, device=DEV)
    ids = torch.full((V, max(cap, 1)), -1, dtype=torch.int32, device=DEV)
    ranges = torch.full((V, T, 2), 7, dtype=torch.int32, device=DEV)
    npairs = torch.zeros(V, 2, dtype=torch.int32, device=DEV)
    dass.dass_bin_sort_views(cams, n, rec.xy_depth, rec.box, rec.rows, rec.tiles, ws, cap, ids, ranges, npairs)
    torch.cuda.synchronize()
    return np_(ids).view(np.uint32), np_(ranges).view(np.uint32), np_(npairs).view(np.uint32)


def project(cams, sc):
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(len(cams), sc.n, DEV)
    dass.dass_project_views(cams, sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None,
                            rec.xy_depth, rec.conic_opa, rec.rgb, rec.box, rec.rows, rec.tiles)
    return rec


def oracle_view(cam, rec, v):
    xy = np_(rec.xy_depth[v])
    box = np_(rec.box[v]).view(np.uint32)
    rows = np_(rec.rows[v]).view(np.uint32)
    zb = xy[:, 2].copy().view(np.uint32)
    b4 = np.stack([box[:, 0] & 0xFFFF, box[:, 0] >> 16, box[:, 1] & 0xFFFF, box[:, 1] >> 16], 1)
    vis = (b4[:, 0] <= b4[:, 1]).astype(np.uint8)
    return oracle.bin_sort(cam, dict(visible=vis, zbits=zb, box=b4.astype(np.int32), rows=rows))


def tiny_rig(num, W, H, seed):
    """num identity-pose cameras of W×H with jittered principal points."""
    g = np.random.default_rng(seed)
    base = synth.tiny_camera(W, H)
    return [synth.Camera(W, H, base.fx, base.fy, base.cx + g.uniform(-4, 4), base.cy + g.uniform(-4, 4),
                         base.viewmat) for _ in range(num)]


@pytest.mark.parametrize("V,W,H,n,deg,seed", [(3, 100, 70, 3000, 1, 11), (5, 333, 177, 20000, 3, 12),
                                              (2, 17, 300, 5000, 0, 15), (1, 1, 1, 20, 0, 14)])
def test_views_equal_oracle_per_view(V, W, H, n, deg, seed):
    """Ragged sizes, several views of one N3DV-shaped rig, vs the oracle's brute-force sort."""
    cams = synth.n3dv_rig(width=W, height=H)[:V]
    sc = synth.n3dv_scene(n=n, seed=seed, degree=deg, fx=cams[0].fx)
    rec = project(cams, sc)
    ids, ranges, npairs = batched(cams, rec, sc.n, 1 << 18)
    for v, cam in enumerate(cams):
        keys, oids, oranges = oracle_view(cam, rec, v)
        K = len(keys)
        assert npairs[v, 0] == K and npairs[v, 1] == 0
        assert np.array_equal(ids[v, :K], oids)
        assert np.array_equal(ranges[v], oranges)


def test_views_equal_per_view_bin_sort_full_c3():
    """BASELINE.json's C3 at full size, in the launch configuration bench.py times."""
    cams, sc = synth.c3()
    rec = project(cams, sc)
    cap = 1 << 22
    ids, ranges, npairs = batched(cams, rec, sc.n, cap)
    ras = Raster(cams[0].width, cams[0].height, sc.n, cap, DEV)
    for v, cam in enumerate(cams):
        K = ras.sort(cam, rec.view(v), host_mode=True)
        assert npairs[v, 0] == K and npairs[v, 1] == 0
        assert np.array_equal(ids[v, :K], np_(ras.sorted_ids[:K]).view(np.uint32))
        assert np.array_equal(ranges[v], np_(ras.ranges).view(np.uint32))


def test_views_capacity_overflow_flags_only_that_view():
    cams = tiny_rig(2, 64, 64, 7)
    sc = synth.random_scene(1000, cams[0], seed=1)
    sc.pos_opa[500:, 0] += 50.0            # half the Gaussians leave view 1 ...
    cams[1] = synth.Camera(64, 64, cams[1].fx, cams[1].fy, cams[1].cx - 2000.0, cams[1].cy,
                           cams[1].viewmat)  # ... which looks far to the side
    rec = project(cams, sc)
    K = [len(oracle_view(c, rec, v)[0]) for v, c in enumerate(cams)]
    assert K[1] < K[0]
    ids, ranges, npairs = batched(cams, rec, sc.n, K[0] - 1)
    assert npairs[0, 1] == 1 and npairs[0, 0] == K[0] and not ranges[0].any()
    keys, oids, oranges = oracle_view(cams[1], rec, 1)
    assert npairs[1, 0] == K[1] and npairs[1, 1] == 0
    assert np.array_equal(ids[1, :K[1]], oids) and np.array_equal(ranges[1], oranges)


def test_views_equal_depth_ties():
    """A planar scene: every Gaussian at the same depth, so the order within a tile is
    decided by the index alone (A03), in every view."""
    cams = tiny_rig(3, 80, 64, 21)
    sc = synth.random_scene(2000, cams[0], seed=21)
    sc.pos_opa[:, 2] = 3.0
    rec = project(cams, sc)
    ids, ranges, npairs = batched(cams, rec, sc.n, 1 << 16)
    for v, cam in enumerate(cams):
        keys, oids, oranges = oracle_view(cam, rec, v)
        assert npairs[v, 0] == len(keys)
        assert np.array_equal(ids[v, :len(keys)], oids) and np.array_equal(ranges[v], oranges)
