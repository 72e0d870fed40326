"""One small pass over every libdass export, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize.py

C1 (64×64, 1k Gaussians, SH0) and a 200×150 N3DV-shaped crop (6k Gaussians,
SH3, 3 views) through the step bench.py times (ShiftStep: shift, multi-view
projection, graph-mode sorts on overlapping streams, forward with acceptance
lists, list backward, multi-view preprocess, shift backward), the no-list
forward/backward, host-mode sort, the batched sort, error map, fidelity loss,
deformation fields, densification, feature render, statistics and the
non-finite scan.  Exits non-zero on any library error; the sanitizer reports
memory / race / barrier errors itself.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_14847_b200 import dass, synth  # noqa: E402
from paper_2411_14847_b200.pipeline import (DeformFields, DeviceScene, Grads, Raster,  # noqa: E402
                                            ViewRecords)
from paper_2411_14847_b200.step import ShiftStep  # noqa: E402

DEV = "cuda"
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def single_view(cam, sc, lists):
    ds = DeviceScene.from_host(sc, DEV)
    rec = ViewRecords(1, sc.n, DEV)
    dass.dass_project(cam, sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, *rec.view(0))
    ras = Raster(cam.width, cam.height, sc.n, 1 << 18, DEV, accept_lists=lists)
    keys = torch.empty(1 << 18, dtype=torch.int64, device=DEV)
    ras.forward(cam, rec.view(0), host_mode=True, sorted_keys=keys, bg=(0.1, 0.2, 0.3))
    g = Grads.zeros(sc.n, sc.sh_degree, DEV)
    ras.backward(cam, ds, rec.view(0), t(synth.grad_image(cam, 3)), g, bg=(0.1, 0.2, 0.3))
    cnt = torch.zeros(8, dtype=torch.int64, device=DEV)
    dass.dass_render_stats(cam, ras.ranges, ras.sorted_ids, rec.xy_depth[0], rec.conic_opa[0],
                           rec.box[0], ras.T, ras.last, cnt)
    return ds, rec, ras, g


def main():
    torch.cuda.set_device(0)
    cam, sc = synth.c1()
    for lists in (True, False):
        ds, rec, ras, g = single_view(cam, sc, lists)
    # f1 loss, f3 inheritance, error map, feature render, non-finite scan on C1
    gt = t(synth.random_image(cam, 5))
    ws = torch.empty(dass.dass_fidelity_loss_workspace(cam.width, cam.height) // 4 + 64, device=DEV)
    loss = torch.zeros(3, device=DEV)
    dass.dass_fidelity_loss(ras.img, gt, 0.2, ws, loss, torch.empty_like(ras.img))
    m = t(np.random.default_rng(1).normal(size=sc.n).astype(np.float32))
    keep = torch.empty(sc.n, dtype=torch.uint8, device=DEV)
    dass.dass_inherit_mask(m, keep)
    gm = torch.zeros(sc.n, device=DEV)
    dass.dass_inherit_mask_bwd(m, ds.pos_opa, ds.scale, g.pos_opa, g.scale, 0.01, gm)
    err = torch.empty(cam.height, cam.width, device=DEV)
    dm = torch.zeros((cam.height * cam.width + 31) // 32, dtype=torch.int32, device=DEV)
    s_err = torch.zeros(sc.n, dtype=torch.uint8, device=DEV)
    dass.dass_error_map(cam, ras.img, gt, 0.1, err, dm, sc.n, ds.pos_opa, s_err)
    feat = t(np.random.default_rng(2).normal(size=(sc.n, 16)).astype(np.float32))
    M = torch.empty(16, cam.height, cam.width, device=DEV)
    xy, co, _, box, _, _ = rec.view(0)
    dass.dass_render_features(cam, ras.ranges, ras.sorted_ids, xy, co, box, feat, M)
    bad = torch.zeros(1, dtype=torch.int32, device=DEV)
    dass.dass_scan_nonfinite(g.pos_opa, bad, host_mode=True)
    # f2 deformation and f4 densification
    dyn = (np.arange(sc.n) % 3 == 0).astype(np.uint8)
    fd, fs = synth.dual_fields(synth.Scene(sc.pos_opa, sc.scale, sc.rot, sc.sh, 0, dyn), "n3dv", seed=3)
    fields = DeformFields((fd, fs), sc.n, DEV)
    fields.partition(t(dyn))
    mu = torch.empty(sc.n, 4, device=DEV)
    sg = torch.empty(sc.n, 4, device=DEV)
    fields.forward(ds.pos_opa, mu, sg)
    fields.backward(ds.pos_opa, g.pos_opa, g.rot)
    wsp = torch.empty(dass.dass_partition_workspace(sc.n) // 4 + 1, dtype=torch.int32, device=DEV)
    in_S = torch.empty(sc.n, dtype=torch.uint8, device=DEV)
    idx = torch.empty(sc.n, dtype=torch.int32, device=DEV)
    cnt2 = torch.zeros(2, dtype=torch.int32, device=DEV)
    dass.dass_densify_select(g.gradstat_sum, g.gradstat_cnt, s_err, 1e-6, 5e-7, in_S, idx, cnt2, wsp)
    torch.cuda.synchronize()
    k = int(cnt2[0].item())
    n_out = sc.n + 2 * k
    o = [torch.empty(n_out, 4, device=DEV) for _ in range(3)]
    osh = torch.empty(1, n_out, 4, device=DEV)
    odyn = torch.empty(n_out, dtype=torch.uint8, device=DEV)
    dass.dass_spawn(0, ds.pos_opa, ds.scale, ds.rot, ds.sh, t(dyn), k, idx, 2, 1.6, 0.1, 7,
                    o[0], o[1], o[2], osh, odyn)
    kp = torch.empty(n_out, dtype=torch.uint8, device=DEV)
    kidx = torch.empty(n_out, dtype=torch.int32, device=DEV)
    wsq = torch.empty(dass.dass_partition_workspace(n_out) // 4 + 1, dtype=torch.int32, device=DEV)
    dass.dass_prune_select(o[0], sc.n, 0.05, kp, kidx, cnt2, wsq)
    torch.cuda.synchronize()
    mk = int(cnt2[0].item())
    go = [torch.empty(max(mk, 1), 4, device=DEV) for _ in range(3)]
    dass.dass_gather(0, o[0], o[1], o[2], osh, None, mk, kidx, go[0], go[1], go[2],
                     torch.empty(1, max(mk, 1), 4, device=DEV))
    # the timed step's launch shape on an N3DV crop: 3 views, graph-mode sorts
    cams = [synth.n3dv_rig(width=200, height=150)[v] for v in (2, 9, 17)]
    sc3 = synth.n3dv_scene(n=6000, seed=8, degree=3, fx=cams[0].fx)
    mu3, sg3 = synth.shift_offsets(sc3, seed=33)
    base = DeviceScene.from_host(sc3, DEV)
    stepper = ShiftStep(cams, sc3.n, 3, 1 << 19, DEV, streams=3, validate=True)
    S = stepper.buffers(base, t(mu3), t(sg3), torch.stack([t(synth.grad_image(c, v)) for v, c in enumerate(cams)]))
    stepper.run(S)
    torch.cuda.synchronize()
    stepper.check_overflow()
    stepper.check_numerics()
    # the batched multi-view sort
    nb = dass.dass_bin_sort_views_workspace(3, sc3.n, 1 << 17)
    wsb = torch.empty(nb, dtype=torch.uint8, device=DEV)
    ids = torch.empty(3, 1 << 17, dtype=torch.int32, device=DEV)
    rng = torch.empty(3, stepper.mvp.slots[0].num_tiles, 2, dtype=torch.int32, device=DEV)
    npairs = torch.zeros(3, 2, dtype=torch.int32, device=DEV)
    r = stepper.records
    dass.dass_bin_sort_views(cams, sc3.n, r.xy_depth, r.box, r.rows, r.tiles, wsb, 1 << 17, ids, rng, npairs)
    torch.cuda.synchronize()
    print("sanitize pass done; kernels launched:", dass.kernel_launches())


if __name__ == "__main__":
    main()
