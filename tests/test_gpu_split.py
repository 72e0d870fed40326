"""Split views (dist.view_plan): rendering a view as two
interleaved tile halves on different "ranks" and summing their gradient
buffers (what the all_reduce does) gives the single-GPU gradients — every
gradient by linearity, and ∇p̄ exactly through the reduced uv partials
(dass_gradstat_from_uv).  The ranks are emulated one after another on one GPU;
the NCCL all_reduce is the plain sum done here.
"""
import numpy as np
import pytest

from paper_2411_14847_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_14847_b200 import dass  # noqa: E402
from paper_2411_14847_b200.dist import FlatGrads, view_plan  # noqa: E402
from paper_2411_14847_b200.pipeline import DeviceScene, MultiViewPass, ViewRecords  # noqa: E402

DEV = "cuda"


def rank_grads(cams, scene, ds, dLs, plan, capacity=1 << 21):
    k4 = synth.sh_planes(scene.sh_degree)
    g = FlatGrads.allocate(scene.n, k4, DEV, num_split=plan.num_split)
    my = [cams[v] for v in plan.views]
    rec = ViewRecords(len(my), scene.n, DEV)
    dass.dass_project_views(my, scene.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None,
                            rec.xy_depth, rec.conic_opa, rec.rgb, rec.box, rec.rows, rec.tiles)
    uv = [None if s < 0 else g.uv[s] for s in plan.split]
    mvp = MultiViewPass(my, scene.n, capacity, DEV, streams=2, tiles=plan.tiles, uv_out=uv)
    mvp.run(ds, rec, dLs[plan.views], g)
    torch.cuda.synchronize()
    return g


@pytest.mark.parametrize("V,world", [(2, 4), (3, 2), (5, 2)])
def test_split_views_sum_to_the_single_gpu_gradients(V, world):
    cams = synth.n3dv_rig(width=301, height=203)[:V]
    scene = synth.n3dv_scene(n=20_000, seed=95, degree=3, fx=cams[0].fx)
    ds = DeviceScene.from_host(scene, DEV)
    W, H = cams[0].width, cams[0].height
    T = ((W + 15) // 16) * ((H + 15) // 16)
    dLs = torch.stack([torch.from_numpy(synth.grad_image(c, 300 + k)).to(DEV)
                       for k, c in enumerate(cams)])
    full = rank_grads(cams, scene, ds, dLs, view_plan(V, 0, 1, T))
    plans = [view_plan(V, r, world, T) for r in range(world)]
    assert plans[0].num_split > 0
    parts = [rank_grads(cams, scene, ds, dLs, p) for p in plans]
    acc = FlatGrads.allocate(scene.n, synth.sh_planes(3), DEV, num_split=plans[0].num_split)
    for p in parts:                       # the all_reduce
        acc.flat += p.flat
        acc.gradstat_cnt += p.gradstat_cnt
    dass.dass_gradstat_from_uv(acc.uv, acc.gradstat_sum)
    torch.cuda.synchronize()
    for name in ("pos_opa", "scale", "rot", "sh", "gradstat_sum"):
        a = getattr(acc, name).cpu().numpy().astype(np.float64)
        b = getattr(full, name).cpu().numpy().astype(np.float64)
        tol = 1e-5 * np.abs(b).max() + 1e-4 * np.abs(b)
        assert np.all(np.abs(a - b) <= tol), (name, float(np.abs(a - b).max()), float(np.abs(b).max()))
    assert torch.equal(acc.gradstat_cnt, full.gradstat_cnt)
