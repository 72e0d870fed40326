"""Measure how many acceptance-list entries the two half-tile warps share
(one C3 view): |L0 ∩ L1| / (|L0| + |L1|)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2411_14847_b200 import dass, synth  # noqa: E402
from paper_2411_14847_b200.pipeline import DeviceScene, Raster, ViewRecords  # noqa: E402

cams, sc = synth.c3(n=300_000, num_views=20)
cam = cams[7]
ds = DeviceScene.from_host(sc, "cuda")
rec = ViewRecords(1, sc.n, "cuda")
dass.dass_project(cam, sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, *rec.view(0))
ras = Raster(cam.width, cam.height, sc.n, 1 << 22, "cuda")
ras.forward(cam, rec.view(0), host_mode=True)
torch.cuda.synchronize()
nt = ras.num_tiles
al = lambda b: (b + 255) // 256 * 256
acc = ras.accept.view(torch.uint8).cpu().numpy()
cnt = acc[:2 * nt * 4].view(np.uint32)
off = al(2 * nt * 4)
cap = ras.capacity
idx = acc[off:off + 2 * cap * 4].view(np.uint32)
rng = ras.ranges.cpu().numpy().view(np.uint32)
tot = inter = 0
for t in range(nt):
    a, b = rng[t]
    ln = b - a
    if ln == 0:
        continue
    l0 = idx[2 * a: 2 * a + cnt[2 * t]]
    l1 = idx[2 * a + ln: 2 * a + ln + cnt[2 * t + 1]]
    tot += len(l0) + len(l1)
    inter += len(np.intersect1d(l0, l1, assume_unique=True))
print(f"entries {tot}, shared {inter}, union {tot - inter}, shared frac of total {inter / tot:.3f}")
