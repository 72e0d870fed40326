"""View-sharded data parallelism: one process per GPU, the V
views of a timestep split into contiguous blocks, per-Gaussian gradients
summed once per step by an all_reduce of ONE flat fp32 buffer, and the S_err
flags (S_err = ∪_c S_err^c) combined by an all_reduce(MAX).

Plumbing only: the gradient values come from libdass kernels (or, in the CPU
gloo tests, from any producer with the same layout).
"""
from __future__ import annotations

from dataclasses import dataclass


def shard(num_views: int, rank: int, world: int) -> list[int]:
    """Contiguous view blocks whose sizes differ by at most one
    (20 views: 10/10 at 2 GPUs, 5×4 at 4, 3,3,3,3,2,2,2,2 at 8)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(num_views, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


@dataclass
class FlatGrads:
    """All per-Gaussian gradient outputs as views of one contiguous buffer, so
    the cross-GPU sum is a single collective: pos_opa, scale, rot [N,4];
    sh [K4,N,4]; g_mu, g_sigma [N,4] (shift offsets); gradstat_sum [N].
    gradstat_cnt (int) is reduced separately."""
    flat: "torch.Tensor"
    pos_opa: "torch.Tensor"
    scale: "torch.Tensor"
    rot: "torch.Tensor"
    sh: "torch.Tensor"
    g_mu: "torch.Tensor"
    g_sigma: "torch.Tensor"
    gradstat_sum: "torch.Tensor"
    gradstat_cnt: "torch.Tensor"

    @staticmethod
    def allocate(n: int, k4: int, device="cuda") -> "FlatGrads":
        import torch
        sizes = [n * 4, n * 4, n * 4, k4 * n * 4, n * 4, n * 4, n]
        flat = torch.zeros(sum(sizes), dtype=torch.float32, device=device)
        p = list(torch.split(flat, sizes))
        return FlatGrads(flat, p[0].view(n, 4), p[1].view(n, 4), p[2].view(n, 4),
                         p[3].view(k4, n, 4), p[4].view(n, 4), p[5].view(n, 4), p[6],
                         torch.zeros(n, dtype=torch.int32, device=device))

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * 4

    def zero_(self):
        self.flat.zero_()
        self.gradstat_cnt.zero_()


def allreduce_grads(g: FlatGrads, group=None, counts: bool = True):
    """SUM over ranks of every gradient (A27: gradients are summed over views)."""
    import torch.distributed as dist
    dist.all_reduce(g.flat, op=dist.ReduceOp.SUM, group=group)
    if counts:
        dist.all_reduce(g.gradstat_cnt, op=dist.ReduceOp.SUM, group=group)


def allreduce_s_err(s_err, group=None):
    """S_err = ∪_c S_err^c over all ranks' views (uint8 flags, MAX = OR)."""
    import torch.distributed as dist
    dist.all_reduce(s_err, op=dist.ReduceOp.MAX, group=group)
