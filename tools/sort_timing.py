"""Time dass_bin_sort_views (all 20 C3 views at once) against 20 dass_bin_sort calls,
isolated, CUDA events.  usage (GPU): python tools/sort_timing.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2411_14847_b200 import dass, synth  # noqa: E402
from paper_2411_14847_b200.pipeline import DeviceScene, Raster, ViewRecords  # noqa: E402

cams, sc = synth.c3()
V, n, cap = len(cams), sc.n, 1 << 22
ds = DeviceScene.from_host(sc, "cuda")
rec = ViewRecords(V, n, "cuda")
dass.dass_project_views(cams, sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None,
                        rec.xy_depth, rec.conic_opa, rec.rgb, rec.box, rec.tiles)
T = ((cams[0].width + 15) // 16) * ((cams[0].height + 15) // 16)
ws = torch.empty(dass.dass_bin_sort_views_workspace(V, n, cap), dtype=torch.uint8, device="cuda")
ids = torch.empty(V, cap, dtype=torch.int32, device="cuda")
rng = torch.empty(V, T, 2, dtype=torch.int32, device="cuda")
npairs = torch.zeros(V, 2, dtype=torch.int32, device="cuda")
ras = Raster(cams[0].width, cams[0].height, n, cap, "cuda")


def batched():
    dass.dass_bin_sort_views(cams, n, rec.xy_depth, rec.box, rec.tiles, ws, cap, ids, rng, npairs)


def per_view():
    for v, c in enumerate(cams):
        ras.sort(c, rec.view(v))


for name, f in (("batched", batched), ("per_view", per_view)):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 5:.3f} ms per 20 views")
