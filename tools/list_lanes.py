"""Distribution of active lanes per acceptance-list entry (one C3 view)."""
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
off_idx = al(2 * nt * 4)
cap = ras.capacity
off_b = off_idx + al(2 * cap * 4)
byts = acc[off_b:off_b + 2 * cap * 32].reshape(-1, 32)
rng = ras.ranges.cpu().numpy().view(np.uint32)
hist = np.zeros(33, np.int64)
bits_hist = np.zeros(129, np.int64)
for t in range(nt):
    a, b = rng[t]
    ln = b - a
    for w in range(2):
        base = 2 * a + w * ln
        m = cnt[2 * t + w]
        if m == 0:
            continue
        blk = byts[base:base + m]
        act = (blk != 0).sum(1)
        hist += np.bincount(act, minlength=33)[:33]
        nb = np.unpackbits(blk[:, :, None], axis=2)[:, :, 4:].sum((1, 2))
        bits_hist += np.bincount(nb, minlength=129)[:129]
tot = hist.sum()
print("entries", tot)
print("active lanes: 1:", hist[1] / tot, " ≤2:", hist[1:3].sum() / tot, " ≤4:", hist[1:5].sum() / tot,
      " mean:", (np.arange(33) * hist).sum() / tot)
print("accepted pixels per entry mean:", (np.arange(129) * bits_hist).sum() / bits_hist.sum())
