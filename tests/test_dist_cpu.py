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


def _worker(rank, world, port, out_path):
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
    ddist.allreduce_grads(g)
    s_err = torch.zeros(sc.n, dtype=torch.uint8)
    s_err[rank::7] = 1
    ddist.allreduce_s_err(s_err)
    if rank == 0:
        np.savez(out_path, flat=g.flat.numpy(), cnt=g.gradstat_cnt.numpy(), s_err=s_err.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sum_equals_single_process(tmp_path):
    import oracle
    oracle.build()   # once, before the workers start
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    cams, sc = _scene()
    ref = ddist.FlatGrads.allocate(sc.n, synth.sh_planes(sc.sh_degree), device="cpu")
    for v in range(len(cams)):
        vg = _view_grads(cams, sc, v)
        ref.pos_opa += torch.from_numpy(vg["pos"]).float()
        ref.scale += torch.from_numpy(vg["scale"]).float()
        ref.rot += torch.from_numpy(vg["rot"]).float()
        ref.sh += torch.from_numpy(np.ascontiguousarray(vg["sh"])).float()
        ref.gradstat_sum += torch.from_numpy(vg["stat"]).float()
        ref.gradstat_cnt += torch.from_numpy(vg["cnt"]).int()
    a, b = r["flat"], ref.flat.numpy()
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6 * np.abs(b).max())
    assert np.array_equal(r["cnt"], ref.gradstat_cnt.numpy())
    expect = np.zeros(sc.n, np.uint8)
    expect[0::7] = 1
    expect[1::7] = 1
    assert np.array_equal(r["s_err"], expect)
