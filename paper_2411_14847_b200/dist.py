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
class ViewPlan:
    """This rank's share of a timestep's views.

    views: global view indices rendered here; tiles[k] = None for a whole view,
    else (begin, 2, count) — one of the view's two interleaved tile halves
    (a checkerboard over tile indices, so both halves see the same content);
    split[k] = the view's index among all split views, or -1; num_split = the
    number of views split across ranks (the uv blocks of FlatGrads)."""
    views: list
    tiles: list
    split: list
    num_split: int


def view_plan(num_views: int, rank: int, world: int, num_tiles: int,
              allow_split: bool = True) -> ViewPlan:
    """Balanced view sharding.  When the views divide evenly,
    whole views in contiguous blocks (shard()).  Otherwise, when twice the views
    divide evenly, every view is cut into two interleaved tile halves and each
    rank takes a contiguous block of halves: 20 views at 8 GPUs → 5 halves each
    (2 whole views + 1 half) instead of 3,3,3,3,2,2,2,2 views.  A view whose
    halves land on two ranks is 'split'; its ∇p̄ terms are formed after the
    all-reduce (dass_gradstat_from_uv).  Anything else falls back to shard(), as
    does allow_split=False (a step whose per-view work needs whole images, e.g.
    the error maps of C4)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if (not allow_split or num_views % world == 0 or (2 * num_views) % world != 0
            or num_tiles < 2):
        v = shard(num_views, rank, world)
        return ViewPlan(v, [None] * len(v), [-1] * len(v), 0)
    per = 2 * num_views // world
    owner = [u // per for u in range(2 * num_views)]             # unit u = 2·view + half
    split_ids, nsplit = {}, 0
    for v in range(num_views):
        if owner[2 * v] != owner[2 * v + 1]:
            split_ids[v] = nsplit
            nsplit += 1
    views, tiles, split = [], [], []
    for u in range(rank * per, (rank + 1) * per):
        v, h = divmod(u, 2)
        if views and views[-1] == v:              # both halves here: the whole view
            tiles[-1], split[-1] = None, -1
            continue
        views.append(v)
        if v in split_ids:
            tiles.append((h, 2, (num_tiles - h + 1) // 2))
            split.append(split_ids[v])
        else:
            tiles.append(None)
            split.append(-1)
    return ViewPlan(views, tiles, split, nsplit)


@dataclass
class FlatGrads:
    """All per-Gaussian gradient outputs as views of one contiguous buffer, so
    the cross-GPU sum is a single collective.  Layout (float32, 16-byte aligned
    blocks), the shift-stage payload first:

        [uv (split views) | g_mu [N,4] | g_sigma [N,4] | gradstat_sum [N] |
         cnt_f [N] | pos_opa [N,4] | scale [N,4] | rot [N,4] | sh [K4,N,4]]

    The shift stage trains only the offsets μ, σ and keeps the ∇p̄
    statistics for densification, so its all_reduce covers the prefix
    up to cnt_f (36 B per Gaussian); a stage that optimises the
    Gaussians themselves reduces the whole buffer.  gradstat_cnt is the int32
    counter the kernels write; cnt_f carries it through the float collective
    (counts < 2^24 are exact in float32)."""
    flat: "torch.Tensor"
    pos_opa: "torch.Tensor"
    scale: "torch.Tensor"
    rot: "torch.Tensor"
    sh: "torch.Tensor"
    g_mu: "torch.Tensor"
    g_sigma: "torch.Tensor"
    gradstat_sum: "torch.Tensor"
    gradstat_cnt: "torch.Tensor"
    uv: "torch.Tensor | None" = None     # [S][N][2] split-view ∇p̄ partials (ViewPlan)
    cnt_f: "torch.Tensor | None" = None  # [N] float copy of gradstat_cnt for the collective
    shift_len: int = 0                   # floats in the shift-stage payload prefix

    @staticmethod
    def allocate(n: int, k4: int, device="cuda", num_split: int = 0) -> "FlatGrads":
        import torch
        pad4 = lambda x: x + (-x) % 4        # keep every block 16-byte aligned
        u = pad4(num_split * n * 2)
        sizes = [u, n * 4, n * 4, pad4(n), pad4(n), n * 4, n * 4, n * 4, k4 * n * 4]
        flat = torch.zeros(sum(sizes), dtype=torch.float32, device=device)
        p = list(torch.split(flat, sizes))
        uv = p[0][:num_split * n * 2].view(num_split, n, 2) if num_split else None
        return FlatGrads(flat, p[5].view(n, 4), p[6].view(n, 4), p[7].view(n, 4),
                         p[8].view(k4, n, 4), p[1].view(n, 4), p[2].view(n, 4), p[3][:n],
                         torch.zeros(n, dtype=torch.int32, device=device), uv, p[4][:n],
                         sum(sizes[:5]))

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * 4

    def payload(self, stage: str = "full"):
        """The contiguous slice one all_reduce sums: 'shift' = uv, g_mu, g_sigma,
        ∇p̄ sum and count; 'full' = everything."""
        if stage == "shift":
            return self.flat[:self.shift_len]
        if stage == "full":
            return self.flat
        raise ValueError(f"unknown stage {stage!r}")

    def zero_(self):
        self.flat.zero_()
        self.gradstat_cnt.zero_()


@dataclass
class FlatParams:
    """A step's per-Gaussian inputs as views of one contiguous fp32 buffer:
    pos_opa, scale, rot [N,4]; sh [K4,N,4]; mu, sigma [N,4] (the shift
    offsets).  The buffer length is padded to a multiple of 4·world floats, so
    the buffer splits into `world` equal 16-byte-aligned shards.

    End to end, every rank needs all of it, but need not upload all of it: rank
    r copies only shard r from host memory and one in-place all_gather over
    NVLink assembles the rest (`upload_shard` + `allgather`), so the
    host→device traffic per rank is 1/world of the parameters."""
    flat: "torch.Tensor"
    pos_opa: "torch.Tensor"
    scale: "torch.Tensor"
    rot: "torch.Tensor"
    sh: "torch.Tensor"
    mu: "torch.Tensor"
    sigma: "torch.Tensor"
    world: int = 1

    @staticmethod
    def sizes(n: int, k4: int) -> list[int]:
        return [n * 4, n * 4, n * 4, k4 * n * 4, n * 4, n * 4]

    @staticmethod
    def allocate(n: int, k4: int, device="cuda", world: int = 1, pin: bool = False) -> "FlatParams":
        import torch
        sizes = FlatParams.sizes(n, k4)
        total = sum(sizes)
        total += (-total) % (4 * world)
        flat = torch.zeros(total, dtype=torch.float32, device=device)
        if pin:
            flat = flat.pin_memory()
        p = list(torch.split(flat[:sum(sizes)], sizes))
        return FlatParams(flat, p[0].view(n, 4), p[1].view(n, 4), p[2].view(n, 4),
                          p[3].view(k4, n, 4), p[4].view(n, 4), p[5].view(n, 4), world)

    def shard(self, rank: int) -> "torch.Tensor":
        """Rank `rank`'s contiguous 1/world of the buffer."""
        L = self.flat.numel() // self.world
        return self.flat[rank * L:(rank + 1) * L]

    def upload_shard(self, host: "FlatParams", rank: int):
        """Copy shard `rank` of the (pinned) host buffer into this device buffer
        on the current stream; world == 1 copies everything."""
        self.shard(rank).copy_(host.shard(rank), non_blocking=True)

    def allgather(self, rank: int, group=None):
        """Assemble every rank's shard in place (no-op at world 1)."""
        if self.world > 1:
            import torch.distributed as dist
            dist.all_gather_into_tensor(self.flat, self.shard(rank), group=group)


def allreduce_grads(g: FlatGrads, group=None, counts: bool = True, finish=None,
                    stage: str = "full"):
    """SUM over ranks (A27: gradients are summed over views) of g.payload(stage) —
    ONE collective: the int32 visibility counts ride in cnt_f.  With split views
    (g.uv), `finish(g)` then adds their ∇p̄ terms from the reduced uv blocks
    (dass_gradstat_from_uv), identically on every rank."""
    import torch.distributed as dist
    if counts:
        g.cnt_f.copy_(g.gradstat_cnt)
    dist.all_reduce(g.payload(stage), op=dist.ReduceOp.SUM, group=group)
    if counts:
        g.gradstat_cnt.copy_(g.cnt_f)
    if g.uv is not None and finish is not None:
        finish(g)


def allreduce_s_err(s_err, group=None):
    """S_err = ∪_c S_err^c over all ranks' views (uint8 flags, MAX = OR)."""
    import torch.distributed as dist
    dist.all_reduce(s_err, op=dist.ReduceOp.MAX, group=group)
