"""Time dass_deform_fwd / _bwd (both fields, N3DV profile) at C3 size with CUDA events."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2411_14847_b200 import dass, synth  # noqa: E402

sc = synth.n3dv_scene(n=300_000, seed=3, degree=0)
fd, fs = synth.dual_fields(sc, "n3dv", seed=40)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
pos = t(sc.pos_opa)
n = sc.n
idx_d = torch.empty(n, dtype=torch.int32, device="cuda"); idx_s = torch.empty_like(idx_d)
counts = torch.zeros(2, dtype=torch.int32, device="cuda")
ws = torch.empty(dass.dass_partition_workspace(n) // 4 + 1, dtype=torch.int32, device="cuda")
dass.dass_partition(t(sc.dynamic.astype(np.uint8)), idx_d, idx_s, counts, ws)
F = [(fd, t(fd.table), t(fd.mlp), idx_d, counts[0:1]), (fs, t(fs.table), t(fs.mlp), idx_s, counts[1:2])]
mu = torch.empty(n, 4, device="cuda"); sg = torch.empty(n, 4, device="cuda")
gm, gs = (t(a) for a in synth.offset_grads(n, 5, 1e-3))
gt = [torch.zeros_like(f[1]) for f in F]; gp = [torch.zeros_like(f[2]) for f in F]
res = {}
for name in ("partition", "fwd_dyn", "fwd_st", "bwd_dyn", "bwd_st"):
    def run():
        if name == "partition":
            dass.dass_partition(t(sc.dynamic.astype(np.uint8)) if False else part_mask, idx_d, idx_s, counts, ws)
            return
        k = 0 if name.endswith("dyn") else 1
        f, tab, mlp, idx, c = F[k]
        if name.startswith("fwd"):
            dass.dass_deform_fwd(f, tab, mlp, pos, mu, sg, idx=idx, count=c, n=n)
        else:
            dass.dass_deform_bwd(f, tab, mlp, pos, gm, gs, gt[k], gp[k], idx=idx, count=c, n=n)
    part_mask = t(sc.dynamic.astype(np.uint8))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    res[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 2)
res["unit"] = "us per call"
res["counts"] = counts.cpu().tolist()
print(json.dumps(res))
