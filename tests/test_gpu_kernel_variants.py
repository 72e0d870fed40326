"""The pass's selectable schedules stay parity-green: the batched multi-view sort
(PassOptions.batch_sort), the chained sorts (PassOptions.sort_chains), and the
one-stream and chunked projections inside the overlapped pass, against the oracle's per-view sums."""
import numpy as np
import pytest

import oracle
from _parity import grad_compare
from paper_2411_14847_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_14847_b200 import dass  # noqa: E402
from paper_2411_14847_b200.pipeline import (DeviceScene, Grads, MultiViewPass,  # noqa: E402
                                            PassOptions, ViewRecords)

DEV = "cuda"


@pytest.mark.parametrize("opts", [PassOptions(batch_sort=True, sort_batch_chunks=2),
                                  PassOptions(sort_chains=2), PassOptions(pre_chunks=1, proj_chunks=1),
                                  PassOptions(split_project=False),
                                  PassOptions(proj_chunks=2), PassOptions(split_preprocess=False)],
                         ids=["batch_sort", "sort_chains", "single_preprocess", "unsplit_projection",
                              "chunked_split_projection", "one_stream_preprocess"])
def test_pass_options_parity(opts):
    cams = synth.n3dv_rig(width=160, height=120, num_views=4)
    sc = synth.n3dv_scene(n=5000, seed=57, degree=2, fx=cams[0].fx)
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(len(cams), sc.n, DEV)
    dLs = np.stack([synth.grad_image(c, 700 + v) for v, c in enumerate(cams)])
    g = Grads.zeros(sc.n, 2, DEV)
    mv = MultiViewPass(cams, sc.n, 1 << 20, DEV, streams=2,
                       options=opts)

    def project(v0, v1, part=dass.DASS_PROJECT_ALL):   # the step's callback (step.py)
        dass.dass_project_views_part(part, cams[v0:v1], sc.sh_degree, ds.pos_opa, ds.scale, ds.rot,
                                     ds.sh, None, rec.xy_depth[v0:v1], rec.conic_opa[v0:v1],
                                     rec.rgb[v0:v1], rec.box[v0:v1], rec.rows[v0:v1],
                                     rec.tiles[v0:v1])
    mv.run(ds, rec, torch.from_numpy(dLs).to(DEV), g, project=project)
    torch.cuda.synchronize()
    assert mv.overflowed_views() == []
    keys = ("g_pos_opa", "g_scale", "g_rot", "k_pos_opa", "k_scale", "k_rot", "t_pos_opa",
            "t_scale", "t_rot", "gradstat_cnt")
    ref = None
    gtie = np.zeros(sc.n, bool)
    for v, cam in enumerate(cams):
        o = oracle.render_bwd(cam, sc, dLs[v], kappa=True)
        gtie |= o["gtie"] == 1
        ref = {k: o[k].copy() for k in keys} if ref is None else {k: ref[k] + o[k] for k in keys}
    ok = ~gtie
    np_ = lambda t: t.detach().cpu().numpy()
    grad_compare("pos", np_(g.pos_opa)[ok], ref["g_pos_opa"][ok], ref["k_pos_opa"][ok], slack=ref["t_pos_opa"][ok])
    grad_compare("scale", np_(g.scale)[ok, :3], ref["g_scale"][ok, :3], ref["k_scale"][ok, :3],
                 slack=ref["t_scale"][ok, :3])
    grad_compare("rot", np_(g.rot)[ok], ref["g_rot"][ok], ref["k_rot"][ok], slack=ref["t_rot"][ok])
    assert np.array_equal(np_(g.gradstat_cnt), ref["gradstat_cnt"])


def test_split_schedules_match_one_stream():
    """The two-stream projection and preprocess (PassOptions.split_project /
    split_preprocess, the defaults) write disjoint outputs with the same kernels as
    the one-stream schedule: the records are bitwise the same and every gradient
    agrees to fp32 summation order (the backward's per-tile atomics), the counts
    exactly."""
    cams = synth.n3dv_rig(width=160, height=120, num_views=4)
    sc = synth.n3dv_scene(n=5000, seed=58, degree=3, fx=cams[0].fx)
    ds = DeviceScene.from_host(sc, DEV)
    dLs = torch.from_numpy(np.stack([synth.grad_image(c, 800 + v) for v, c in enumerate(cams)])).to(DEV)
    out = []
    for opts in (PassOptions(), PassOptions(split_project=False, split_preprocess=False)):
        rec = ViewRecords(len(cams), sc.n, DEV)
        g = Grads.zeros(sc.n, 3, DEV)
        mv = MultiViewPass(cams, sc.n, 1 << 20, DEV, streams=4, options=opts)

        def project(v0, v1, part=dass.DASS_PROJECT_ALL, rec=rec):
            dass.dass_project_views_part(part, cams[v0:v1], 3, ds.pos_opa, ds.scale, ds.rot, ds.sh,
                                         None, rec.xy_depth[v0:v1], rec.conic_opa[v0:v1],
                                         rec.rgb[v0:v1], rec.box[v0:v1], rec.rows[v0:v1],
                                         rec.tiles[v0:v1])
        mv.run(ds, rec, dLs, g, project=project)
        torch.cuda.synchronize()
        o = {k: getattr(g, k).clone() for k in ("pos_opa", "scale", "rot", "sh", "gradstat_sum",
                                                "gradstat_cnt")}
        o.update({"rec_" + k: getattr(rec, k).clone() for k in ("xy_depth", "conic_opa", "rgb", "box",
                                                              "rows", "tiles")})
        out.append(o)
    for k in out[0]:
        a, b = out[0][k], out[1][k]
        if k.startswith("rec_") or k == "gradstat_cnt":
            assert torch.equal(a.view(torch.uint8), b.view(torch.uint8)), k
        else:
            tol = 1e-5 * float(b.abs().max()) + 1e-30
            assert float((a - b).abs().max()) <= tol, k
