"""Time dass_fidelity_loss on one 1352x1014 view (CUDA events, warm)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2411_14847_b200 import dass  # noqa: E402

W, H = 1352, 1014
g = torch.Generator(device="cuda").manual_seed(0)
img = torch.rand(3, H, W, device="cuda", generator=g)
gt = (img + 0.1 * torch.randn(3, H, W, device="cuda", generator=g)).clamp(0, 1)
ws = torch.empty(dass.dass_fidelity_loss_workspace(W, H) // 4 + 64, device="cuda")
loss = torch.zeros(3, device="cuda")
dL = torch.empty(3, H, W, device="cuda")
for _ in range(3):
    dass.dass_fidelity_loss(img, gt, 0.2, ws, loss, dL)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 50 if len(sys.argv) < 2 else int(sys.argv[1])
e0.record()
for _ in range(n):
    dass.dass_fidelity_loss(img, gt, 0.2, ws, loss, dL)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"us_per_view": round(e0.elapsed_time(e1) / n * 1e3, 2), "loss": loss.tolist()}))
