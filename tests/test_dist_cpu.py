"""World-size-2 gloo tests of the view-sharded N>1 path on CPU.

The per-view gradient producer here is the oracle (CPU, test infrastructure)
because the CUDA kernels need a GPU; what is under test is the plumbing of
paper_2411_14847_b200/dist.py — view assignment, the flat gradient buffer
layout and the collectives — which is the code bench.py runs under torchrun.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2411_14847_b200 import dist as ddist  # noqa: E402
from paper_2411_14847_b200 import synth  # noqa: E402


def test_shard_partitions_views():
    for V in (1, 13, 20, 21):
        for world in (1, 2, 4, 8):
            got = [ddist.shard(V, r, world) for r in range(world)]
            flat = [v for s in got for v in s]
            assert flat == list(range(V))
            sizes = [len(s) for s in got]
            assert max(sizes) - min(sizes) <= 1
    assert [len(ddist.shard(20, r, 8)) for r in range(8)] == [3, 3, 3, 3, 2, 2, 2, 2]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    cams = synth.n3dv_rig(width=48, height=32, num_views=5)
    sc = synth.n3dv_scene(n=400, seed=77, degree=1, fx=cams[0].fx)
    return cams, sc


def _view_grads(cams, sc, v):
    import oracle
    dL = synth.grad_image(cams[v], 500 + v)
    o = oracle.render_bwd(cams[v], sc, dL)
    nc = (sc.sh_degree + 1) ** 2
    k4 = synth.sh_planes(sc.sh_degree)
    sh = np.zeros((sc.n, 4 * k4))
    sh[:, :3 * nc] = o["g_sh"].reshape(sc.n, -1)
    return dict(pos=o["g_pos_opa"], scale=o["g_scale"], rot=o["g_rot"],
                sh=sh.reshape(sc.n, k4, 4).transpose(1, 0, 2), stat=o["gradstat_sum"],
                cnt=o["gradstat_cnt"])


def _worker(rank, world, port, out_path, stage="full"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cams, sc = _scene()
    g = ddist.FlatGrads.allocate(sc.n, synth.sh_planes(sc.sh_degree), device="cpu")
    for v in ddist.shard(len(cams), rank, world):
        vg = _view_grads(cams, sc, v)
        g.pos_opa += torch.from_numpy(vg["pos"]).float()
        g.scale += torch.from_numpy(vg["scale"]).float()
        g.rot += torch.from_numpy(vg["rot"]).float()
        g.sh += torch.from_numpy(np.ascontiguousarray(vg["sh"])).float()
        g.gradstat_sum += torch.from_numpy(vg["stat"]).float()
        g.gradstat_cnt += torch.from_numpy(vg["cnt"]).int()
        g.g_mu += float(v + 1)                 # stand-ins for the shift backward's outputs
        g.g_sigma -= float(v)
    ddist.allreduce_grads(g, stage=stage)
    s_err = torch.zeros(sc.n, dtype=torch.uint8)
    s_err[rank::7] = 1
    ddist.allreduce_s_err(s_err)
    if rank == 0:
        np.savez(out_path, flat=g.flat.numpy(), cnt=g.gradstat_cnt.numpy(), s_err=s_err.numpy(),
                 shift_len=g.shift_len)
    dist.barrier()
    dist.destroy_process_group()


def _reference(views):
    cams, sc = _scene()
    ref = ddist.FlatGrads.allocate(sc.n, synth.sh_planes(sc.sh_degree), device="cpu")
    for v in views:
        vg = _view_grads(cams, sc, v)
        ref.pos_opa += torch.from_numpy(vg["pos"]).float()
        ref.scale += torch.from_numpy(vg["scale"]).float()
        ref.rot += torch.from_numpy(vg["rot"]).float()
        ref.sh += torch.from_numpy(np.ascontiguousarray(vg["sh"])).float()
        ref.gradstat_sum += torch.from_numpy(vg["stat"]).float()
        ref.gradstat_cnt += torch.from_numpy(vg["cnt"]).int()
        ref.g_mu += float(v + 1)
        ref.g_sigma -= float(v)
    ref.cnt_f.copy_(ref.gradstat_cnt)
    return sc, ref


@pytest.mark.parametrize("stage", ["full", "shift"])
def test_gloo_world2_sum_equals_single_process(tmp_path, stage):
    """One all_reduce of FlatGrads.payload(stage): 'full' sums every
    gradient, 'shift' sums the shift stage's prefix (g_mu, g_sigma, ∇p̄ sum and
    count: 36 B per Gaussian) and leaves the per-Gaussian parameter gradients
    rank-local."""
    import oracle
    oracle.build()   # once, before the workers start
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), out, stage), nprocs=2, join=True)
    r = np.load(out)
    sc, ref = _reference(range(5))
    _, r0 = _reference(ddist.shard(5, 0, 2))     # rank 0's own views
    a, b = r["flat"], ref.flat.numpy()
    L = int(r["shift_len"])
    assert L == ref.shift_len and L * 4 <= 40 * sc.n
    np.testing.assert_allclose(a[:L], b[:L], rtol=1e-5, atol=1e-6 * np.abs(b[:L]).max())
    assert np.array_equal(r["cnt"], ref.gradstat_cnt.numpy())
    rest = b[L:] if stage == "full" else r0.flat.numpy()[L:]
    np.testing.assert_allclose(a[L:], rest, rtol=1e-5, atol=1e-6 * np.abs(rest).max())
    expect = np.zeros(sc.n, np.uint8)
    expect[0::7] = 1
    expect[1::7] = 1
    assert np.array_equal(r["s_err"], expect)


def test_view_plan_balances_halves():
    """20 views at 8 ranks: 5 tile halves each (2 whole views + 1 half); every
    view's two halves covered exactly once; no splits when the views divide."""
    from paper_2411_14847_b200.dist import view_plan
    T = 85 * 64
    for world in (1, 2, 4, 5, 10, 20):
        for r in range(world):
            p = view_plan(20, r, world, T)
            assert p.num_split == 0 and all(t is None for t in p.tiles)
    plans = [view_plan(20, r, 8, T) for r in range(8)]
    halves = {}
    for r, p in enumerate(plans):
        assert p.num_split == 4
        work = sum(1.0 if t is None else 0.5 for t in p.tiles)
        assert work == 2.5
        for v, t, s in zip(p.views, p.tiles, p.split):
            if t is None:
                halves.setdefault(v, []).extend([0, 1])
                assert s == -1
            else:
                begin, stride, count = t
                assert stride == 2 and count == (T - begin + 1) // 2 and s >= 0
                halves.setdefault(v, []).append(begin)
    assert sorted(halves) == list(range(20))
    assert all(sorted(h) == [0, 1] for h in halves.values())
    split_views = sorted({v for p in plans for v, s in zip(p.views, p.split) if s >= 0})
    ids = {v: s for p in plans for v, s in zip(p.views, p.split) if s >= 0}
    assert [ids[v] for v in split_views] == list(range(4))
    # 3 ranks: 40 halves do not divide either → whole views (shard)
    p3 = [view_plan(20, r, 3, T) for r in range(3)]
    assert sum(len(p.views) for p in p3) == 20 and all(p.num_split == 0 for p in p3)


def _uv_worker(rank, world, port, out_path):
    """Each rank holds one half of a split view: its uv partial (x, y, vis) goes
    through the same all_reduce as the gradients, then `finish` forms ∇p̄."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 50
    g = ddist.FlatGrads.allocate(n, 3, device="cpu", num_split=2)
    assert g.pos_opa.data_ptr() % 16 == 0 and g.uv.shape == (2, n, 2)
    rng = np.random.default_rng(rank)
    g.uv[:] = torch.from_numpy(rng.normal(size=(2, n, 2))).float()
    g.uv[:, ::3] = 0.0                                        # not visible in the split views
    vis = torch.ones(n, dtype=torch.int32)
    vis[::3] = 0
    if rank == 0:                                             # the half-0 GPU counts the views
        g.gradstat_cnt += 2 * vis
    g.gradstat_sum += 1.0

    def finish(gg):   # the CPU form of dass_gradstat_from_uv
        u = gg.uv
        gg.gradstat_sum += torch.sqrt(u[..., 0] ** 2 + u[..., 1] ** 2).sum(0)

    ddist.allreduce_grads(g, finish=finish)
    if rank == 0:
        np.savez(out_path, stat=g.gradstat_sum.numpy(), cnt=g.gradstat_cnt.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_split_view_uv_blocks_through_allreduce(tmp_path):
    out = str(tmp_path / "uv.npz")
    mp.spawn(_uv_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    n = 50
    parts = [np.random.default_rng(k).normal(size=(2, n, 2)) for k in range(2)]
    for p in parts:
        p[:, ::3] = 0.0
    tot = (parts[0] + parts[1]).astype(np.float32)
    vis = np.ones(n, bool)
    vis[::3] = False
    want = 2.0 + np.sqrt((tot ** 2).sum(-1)).sum(0)
    np.testing.assert_allclose(r["stat"], want, rtol=1e-5)
    assert np.array_equal(r["cnt"], 2 * vis.astype(np.int32))


def _params_worker(rank, world, port, out_path):
    """Each rank uploads only its shard of the flat parameter buffer; the
    in-place all_gather gives every rank the whole buffer (bench.py e2e)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, k4 = 37, 3
    host = ddist.FlatParams.allocate(n, k4, "cpu", world=world)
    host.flat[:] = torch.arange(host.flat.numel(), dtype=torch.float32)
    dev = ddist.FlatParams.allocate(n, k4, "cpu", world=world)
    dev.upload_shard(host, rank)
    other = dev.shard(1 - rank)
    assert torch.count_nonzero(other) == 0              # not uploaded here
    dev.allgather(rank)
    if rank == 0:
        np.savez(out_path, flat=dev.flat.numpy(), sh=dev.sh.numpy(), mu=dev.mu.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_flat_params_shard_upload_allgather(tmp_path):
    n, k4, world = 37, 3, 2
    p = ddist.FlatParams.allocate(n, k4, "cpu", world=world)
    L = p.flat.numel()
    assert L % (4 * world) == 0 and L >= sum(ddist.FlatParams.sizes(n, k4))
    assert p.shard(0).numel() == p.shard(1).numel() == L // world
    # the views tile the buffer in order, 16-byte aligned
    offs = [t.data_ptr() - p.flat.data_ptr() for t in (p.pos_opa, p.scale, p.rot, p.sh, p.mu, p.sigma)]
    assert offs == [0, 16 * n, 32 * n, 48 * n, 48 * n + 16 * k4 * n, 64 * n + 16 * k4 * n]
    out = str(tmp_path / "p.npz")
    mp.spawn(_params_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    r = np.load(out)
    want = np.arange(L, dtype=np.float32)
    assert np.array_equal(r["flat"], want)
    assert np.array_equal(r["sh"].ravel(), want[12 * n:12 * n + 4 * k4 * n])
