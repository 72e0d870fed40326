"""bench.py — fwd+bwd throughput of the DASS hot path on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[2], the metric's "300k Gaussians, 1352x1014,
1/2/4/8 B200"): an N3DV-shaped timestep — 20 views at 1352×1014, 300k
Gaussians, SH degree 3, 30% dynamic.  One STEP = one shift-stage iteration
over all 20 views:
    dass_apply_shift → dass_project_views → per view (dass_bin_sort →
    dass_render_fwd → dass_render_bwd) → dass_apply_shift_bwd
    [N>1: one NCCL all_reduce(SUM) of the flat gradient buffer]
with a fixed seeded dL/dC per view (the loss is outside the path).
Views are sharded across ranks (strong scaling: the 20-view batch is fixed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fwd+bwd views/sec (Mpix/s) at 300k Gaussians, 1352x1014, 1/2/4/8 B200"
WORKLOAD = ("C3: N3DV-shaped timestep, 20 views 1352x1014, 300k Gaussians SH3, 30% dynamic "
            "masked shift; step = one shift iteration (shift + fwd+bwd over all views)")
WORKLOADS = {
    "c1": ("C1: 1 camera 64x64, 1k random Gaussians, SH degree 0; step = one fwd+bwd "
           "(project, bin/sort, composite, raster + preprocess backward)"),
    "c2": ("C2: 1 camera 1352x1014 (N3DV rig centre view), 300k Gaussians SH3; step = one fwd+bwd "
           "(project, bin/sort, composite, raster + preprocess backward)"),
    "c3": WORKLOAD,
    "c4": ("C4: Meet-Room-shaped timestep, 13 views 1280x720, 200k Gaussians SH3 grown to 260k by "
           "error-guided densification before the timed iterations (13 error maps vs GT, Eq. 4, "
           "spawn K=2); step = one shift iteration at 260k (shift + fwd + error map + bwd over all "
           "views)"),
    "c5": ("C5: 20 views 1352x1014, 1M Gaussians SH3 (sigma_px median x sqrt(0.3)), 30% dynamic "
           "masked shift; step = one shift iteration (shift + fwd+bwd over all views)"),
}


def workload(args):
    """(cameras, scene, workload string) of --config, with --n / --views overrides."""
    from paper_2411_14847_b200 import synth
    if args.config == "c1":
        cam, scene = synth.c1()
        return [cam], scene, WORKLOADS["c1"]
    if args.config == "c2":
        cam, scene = synth.c2(n=args.n or 300_000)
        return [cam], scene, WORKLOADS["c2"]
    if args.config == "c4":
        cams, scene = synth.c4(n=args.n or 200_000, num_views=args.views or 13)
    elif args.config == "c5":
        cams, scene = synth.c5(n=args.n or 1_000_000)
        cams = cams[:args.views] if args.views else cams
    else:
        cams, scene = synth.c3(n=args.n or 300_000, num_views=args.views or 20)
    return cams, scene, WORKLOADS[args.config]
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_TAG = "r02"   # profiles/<tag>_ncu_<kernel>.txt: the committed ncu summaries of this round
SM_COUNT = 148
FP32_LANES = 128

# Algorithmic FP32 work per accepted (pixel, entry) unit of render_bwd's raster
# part (FMA = 2 flop).  Rejected in-box evaluations are not
# counted, so the reported fraction is conservative.
FLOP_BWD_ACCEPTED = 42
STEP_OPS = ("project_views", "bin_sort", "render_fwd", "render_bwd_raster",
            "render_bwd_preprocess_views")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", choices=("c1", "c2", "c3", "c4", "c5"), default="c3",
                   help="BASELINE.json workload: c3 (default, the metric's), c1 (64x64, 1k "
                        "Gaussians, one fwd+bwd), c2 (one 1352x1014 view, 300k), c4 (Meet-Room "
                        "shaped), c5 (1M Gaussians)")
    p.add_argument("--n", type=int, default=None, help="Gaussians (default: the config's)")
    p.add_argument("--views", type=int, default=None, help="views (default: the config's)")
    p.add_argument("--capacity", type=int, default=None,
                   help="pair capacity per view (default 2^22, 2^23 for c5)")
    p.add_argument("--streams", type=int, default=20, help="overlapping per-view streams")
    p.add_argument("--no-graph", action="store_true", help="do not capture the step in a CUDA graph")
    p.add_argument("--sort-chains", type=int, default=0, help="A/B: pipeline.PassOptions.sort_chains")
    p.add_argument("--batch-sort", action="store_true", help="A/B: PassOptions.batch_sort")
    p.add_argument("--sort-batch-chunks", type=int, default=4, help="A/B: PassOptions.sort_batch_chunks")
    p.add_argument("--pre-chunks", type=int, default=1, help="A/B: PassOptions.pre_chunks")
    p.add_argument("--shared-sort-min-views", type=int, default=8,
                   help="A/B: PassOptions.shared_sort_min_views")
    p.add_argument("--proj-chunks", type=int, default=1, help="A/B: PassOptions.proj_chunks")
    p.add_argument("--no-split-preprocess", action="store_true",
                   help="A/B: PassOptions.split_preprocess=False (both preprocess parts on one stream)")
    p.add_argument("--no-split-project", action="store_true",
                   help="A/B: PassOptions.split_project=False (keys and records on one stream)")
    p.add_argument("--lean", action="store_true",
                   help="only warm-up + timed steps (no stats/diagnostic passes): for ncu launch lists")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-sample-views", type=int, default=10)
    p.add_argument("--emulate", default=None, metavar="R/W",
                   help="diagnostic: run rank R's share of a W-GPU view plan on this one GPU "
                        "(no collective) — predicts per-rank step time for --gpus W")
    p.add_argument("--late-collective", action="store_true",
                   help="issue the shift payload's all_reduce after the preprocess SH part joins "
                        "(default: before, overlapping it; the payload holds no SH gradients)")
    p.add_argument("--payload", choices=("shift", "full"), default="shift",
                   help="what the per-step all_reduce sums: the shift stage's payload (g_mu, "
                        "g_sigma, grad-stat; default, the metric's step is a shift iteration) "
                        "or every gradient")
    p.add_argument("--nccl-single", action="store_true",
                   help="diagnostic: open a one-rank NCCL group so the N>1 code path (all_reduce, "
                        "split-view finish, max over ranks) runs on one GPU; with --emulate R/W it "
                        "exercises rank R's whole multi-GPU step")
    a = p.parse_args()
    if a.capacity is None:
        a.capacity = {"c1": 1 << 18, "c5": 1 << 23}.get(a.config, 1 << 22)
    if a.config in ("c1", "c2"):
        a.payload = "full"        # a plain fwd+bwd: every gradient is the step's output
    return a


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region.

    A reader thread collects the 100 ms samples as they arrive, so a timed region
    shorter than a few sampling intervals (C1, C2) can be followed by untimed
    repeats of the same step until enough samples are in (`extend`); the summary
    then says how many repeats the window held."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.rows = []
        self.repeats = 0

    def _read(self):
        for line in self.proc.stdout:
            if line.count(",") >= 7:
                self.rows.append(line.split(","))

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def extend(self, step, sync, min_samples=3, max_s=3.0):
        """Run untimed repeats of `step` until min_samples samples were taken."""
        if self.proc is None:
            return
        t0 = time.time()
        while len(self.rows) < min_samples and time.time() - t0 < max_s:
            for _ in range(8):
                step()
                self.repeats += 1
            sync()

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=5)

    def summary(self):
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k].strip() == "Active"})
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]),
               "power_w_max": max(float(r[2]) for r in rows), "reasons": reasons,
               "samples": len(rows)}
        if self.repeats:
            out["window"] = f"the timed steps + {self.repeats} untimed repeats of the same step"
        return out


def peaks():
    try:
        return json.load(open(PEAKS_PATH)), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# --------------------------------------------------------------- our arm ----

def c4_prepare(cams, scene, dev, growth=60_000, gamma_err=0.10, tau_pos=2e-4, tau_err=1e-4):
    """BASELINE configs[3] before the timed iterations of a
    Meet-Room timestep: render the ground truth (5% of the Gaussians moved + an
    emerging 10k cluster, synth.c4_ground_truth) and the base scene, the 13 error
    maps → S_err (dass_error_map, Alg. 1), Eq. 4 selection with the
    synthetic ∇p̄ (dass_densify_select) and spawn of K = 2 children per
    selected Gaussian up to +60k (dass_spawn): 200k → 260k Gaussians.
    Returns the grown scene, the ground-truth images [V,3,H,W] and the op times."""
    import torch
    from paper_2411_14847_b200 import dass, synth
    from paper_2411_14847_b200.pipeline import DeviceScene, Raster, ViewRecords
    W, H = cams[0].width, cams[0].height
    E = lambda: torch.cuda.Event(enable_timing=True)

    def render_all(sc):
        ds = DeviceScene.from_host(sc, dev)
        rec = ViewRecords(1, sc.n, dev)
        ras = Raster(W, H, sc.n, 1 << 23, dev, accept_lists=False)
        imgs = torch.empty(len(cams), 3, H, W, device=dev)
        for v, cam in enumerate(cams):
            dass.dass_project(cam, sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, *rec.view(0))
            ras.forward(cam, rec.view(0), host_mode=True)
            imgs[v].copy_(ras.img)
        return ds, imgs

    _, gts = render_all(synth.c4_ground_truth(scene))
    ds, imgs = render_all(scene)
    n = scene.n
    ms = {}
    s_err = torch.zeros(n, dtype=torch.uint8, device=dev)
    err = torch.empty(H, W, device=dev)
    dm = torch.zeros((H * W + 31) // 32, dtype=torch.int32, device=dev)
    e = [E(), E()]
    e[0].record()
    for v, cam in enumerate(cams):
        dass.dass_error_map(cam, imgs[v], gts[v], gamma_err, err, dm, n, ds.pos_opa, s_err)
    e[1].record()
    gs, gc = synth.gradstat_lognormal(n)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    in_S = torch.empty(n, dtype=torch.uint8, device=dev)
    idx = torch.empty(n, dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int32, device=dev)
    ws = torch.empty(dass.dass_partition_workspace(n) // 4 + 1, dtype=torch.int32, device=dev)
    f = [E(), E()]
    f[0].record()
    dass.dass_densify_select(t(gs), t(gc), s_err, tau_pos, tau_err, in_S, idx, cnt, ws)
    f[1].record()
    torch.cuda.synchronize()
    sel = int(cnt[0].item())
    m = min(sel, growth // 2)
    n_out = n + 2 * m
    out = [torch.empty(n_out, 4, device=dev) for _ in range(3)]
    osh = torch.empty(synth.sh_planes(scene.sh_degree), n_out, 4, device=dev)
    odyn = torch.empty(n_out, dtype=torch.uint8, device=dev)
    g = [E(), E()]
    g[0].record()
    dass.dass_spawn(scene.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, t(scene.dynamic), m, idx, 2,
                    1.6, 0.1, 7, out[0], out[1], out[2], osh, odyn)
    g[1].record()
    torch.cuda.synchronize()
    ms = {"error_maps_13_views": round(e[0].elapsed_time(e[1]), 4),
          "densify_select": round(f[0].elapsed_time(f[1]), 4), "spawn": round(g[0].elapsed_time(g[1]), 4)}
    h = lambda x: x.cpu().numpy()
    grown = synth.Scene(h(out[0]), h(out[1]), h(out[2]), h(osh), scene.sh_degree, h(odyn))
    info = {"n_before": n, "s_err": int(s_err.sum().item()), "selected": sel, "spawned": 2 * m,
            "n_after": n_out, "gamma_err": gamma_err, "tau_pos": tau_pos, "tau_err": tau_err,
            "grad_stat": "synthetic LogNormal(ln 1e-4, 1) (SURVEY §8(d) C4)", "ms": ms}
    return grown, gts, info


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2411_14847_b200 import dass, synth
    from paper_2411_14847_b200.dist import FlatGrads, FlatParams, allreduce_grads, view_plan
    from paper_2411_14847_b200.pipeline import DeformFields, DeviceScene, PassOptions, Raster
    from paper_2411_14847_b200.step import ShiftStep

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distd = world > 1 or args.nccl_single      # a process group is open
    if distd:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)

    cams, scene, wl = workload(args)
    with_shift = args.config not in ("c1", "c2")      # C1/C2: one plain fwd+bwd
    c4info = None
    if args.config == "c4":   # error-guided densification first: 200k → 260k (C4)
        n_base = scene.n
        scene, c4_gts, c4info = c4_prepare(cams, scene, dev)
    if with_shift:
        mu, sigma = synth.shift_offsets(scene, seed=33)
    else:
        mu = np.zeros((scene.n, 4), np.float32)
        sigma = np.tile(np.array([1, 0, 0, 0], np.float32), (scene.n, 1))
    W0, H0 = cams[0].width, cams[0].height
    plan_rank, plan_world = rank, world
    if args.emulate:
        plan_rank, plan_world = (int(x) for x in args.emulate.split("/"))
    plan = view_plan(len(cams), plan_rank, plan_world, ((W0 + 15) // 16) * ((H0 + 15) // 16),
                     allow_split=c4info is None)   # C4's error maps need whole views
    # views the timed job covers: all of them, or an --emulate run's own share
    job_views = len(cams) if not args.emulate else sum(1.0 if t is None else 0.5 for t in plan.tiles)
    mine = plan.views
    my_cams = [cams[v] for v in mine]
    W, H = cams[0].width, cams[0].height
    n = scene.n
    deg = scene.sh_degree
    K4 = synth.sh_planes(deg)

    # ---- device state
    base = DeviceScene.from_host(scene, dev)                 # 𝒢_{t−1}
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    mu_d, sigma_d = t(mu), t(sigma)
    dLs = torch.stack([t(synth.grad_image(cams[v], 1000 + v, 1.0 / (3 * W * H))) for v in mine]) \
        if mine else torch.empty(0, 3, H, W, device=dev)
    # the step (paper_2411_14847_b200/step.py): buffers, streams and call order
    opts = PassOptions(sort_chains=args.sort_chains, batch_sort=args.batch_sort,
                       sort_batch_chunks=args.sort_batch_chunks,
                       pre_chunks=args.pre_chunks, proj_chunks=args.proj_chunks,
                       split_project=not args.no_split_project,
                       split_preprocess=not args.no_split_preprocess,
                       shared_sort_min_views=args.shared_sort_min_views)
    stepper = ShiftStep(my_cams, n, deg, args.capacity, dev, streams=args.streams,
                        tiles=plan.tiles, split=plan.split, num_split=plan.num_split,
                        shift=with_shift, options=opts)
    records, mvp = stepper.records, stepper.mvp
    if c4info is not None:   # every view's error map inside the step (C4)
        c4_serr = torch.zeros(scene.n, dtype=torch.uint8, device=dev)
        stepper.enable_error_map(c4_gts[mine] if mine else c4_gts[:0], c4info["gamma_err"], n_base,
                                 c4_serr)
    # one flat gradient buffer = the all_reduce payload (dist.FlatGrads)
    bufs0 = stepper.buffers(base, mu_d, sigma_d, dLs)
    grads = bufs0.grads
    flat, g_mu, g_sigma = grads.flat, grads.g_mu, grads.g_sigma
    shifted = bufs0.shifted if with_shift else base          # 𝒢_t after the shift
    raster = Raster(W, H, n, args.capacity, dev)   # single-stream scratch for stats/diagnostics

    def finish_split(g):
        """∇p̄ of the views split across ranks, from their reduced uv partials."""
        dass.dass_gradstat_from_uv(g.uv, g.gradstat_sum)

    def collective(S=bufs0):
        """The one cross-GPU exchange (NCCL all_reduce of the stage's payload)."""
        allreduce_grads(S.grads, finish=finish_split, stage=args.payload)

    def step_local(S=bufs0, wait_inputs=None, coll=False):
        """The step on this GPU; coll: with its collective, which the shift payload (no SH
        gradients) issues while the preprocess's SH part still runs (ShiftStep.run)."""
        stepper.run(S, wait_inputs=wait_inputs,
                    collective=(lambda: collective(S)) if coll else None,
                    collective_after_sh=args.payload != "shift" or args.late_collective)

    coll_in_graph = {"value": False}

    def run_step(graph=None, S=bufs0):
        if graph is None:
            step_local(S, coll=distd)
        else:
            graph.replay()
            if distd and not coll_in_graph["value"]:
                collective(S)

    def step():
        run_step(None)

    def barrier():
        if distd:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- scene statistics (not timed) and overflow check
    stats = {"K": [], "P_fwd": [], "P_bwd": [], "accepted": [], "terminated_px": [],
             "tile_list_mean": [], "tile_list_max": []}
    step()
    torch.cuda.synchronize()
    stepper.check_overflow()     # a view over the pair capacity would render as background
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    stats["n_visible"] = []
    tiles_hist = []
    # this rank's raster work, per work unit: "full" = whole views (the isolated per-op pass
    # renders every view of the rank whole); "step" = weighted by the share of the view's
    # tiles the rank renders in the step (a split view's tile half: 1/2)
    work = {"full": {"P_fwd": 0.0, "P_bwd": 0.0, "accepted": 0.0, "views": 0.0},
            "step": {"P_fwd": 0.0, "P_bwd": 0.0, "accepted": 0.0, "views": 0.0}}
    ntiles = ((W + 15) // 16) * ((H + 15) // 16)
    for k, cam in enumerate([] if args.lean else my_cams):
        split_half = plan.tiles[k] is not None
        rec = records.view(k)
        K = raster.forward(cam, rec, host_mode=True)
        dass.dass_render_stats(cam, raster.ranges, raster.sorted_ids, rec[0], rec[1], rec[3],
                               raster.T, raster.last, cnt)
        c = cnt.cpu().numpy()
        wv = plan.tiles[k][2] / ntiles if split_half else 1.0
        for key, val in (("P_fwd", c[0]), ("P_bwd", c[1]), ("accepted", c[2]), ("views", 1)):
            work["full"][key] += float(val)
            work["step"][key] += wv * float(val)
        if split_half and plan.tiles[k][0] != 0:
            continue   # a split view's scene statistics are counted once, by the rank with half 0
        tt = records.tiles[k]
        vis = tt[tt > 0]
        stats["n_visible"].append(int(vis.numel()))
        tiles_hist.append(torch.bincount(vis.clamp(max=4095), minlength=4096).cpu())
        stats["K"].append(int(K)); stats["P_fwd"].append(int(c[0])); stats["P_bwd"].append(int(c[1]))
        stats["accepted"].append(int(c[2])); stats["terminated_px"].append(int(c[3]))
        stats["tile_list_mean"].append(float(c[4]) / max(int(c[6]), 1))
        stats["tile_list_max"].append(int(c[5]))

    # ---- warm-up (eager), then capture the step in a CUDA graph
    for _ in range(args.warmup):
        step()
    barrier()
    graph = None
    per_step_launches = None
    if not args.no_graph:
        l0 = dass.kernel_launches()
        graph = torch.cuda.CUDAGraph()
        try:   # the collective captured with the step: one graph launch per step
            with torch.cuda.graph(graph):
                step_local(coll=distd)
            coll_in_graph["value"] = distd
        except Exception as exc:   # NCCL capture unavailable: the collective runs after the replay
            print(f"bench: collective not captured ({exc}); running it after the graph", file=sys.stderr)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step_local()
        per_step_launches = dass.kernel_launches() - l0
        for _ in range(2):
            run_step(graph)
        barrier()

    def timed():
        run_step(graph)

    # ---- exactly K timed steps
    l0 = dass.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        barrier()
        ev0.record()
        step_ev[0].record()
        for k in range(args.steps):
            timed()
            step_ev[k + 1].record()
        ev1.record()
        barrier()
        launches = dass.kernel_launches() - l0
        if not distd:            # ranks would disagree on the repeat count (collectives)
            clk.extend(timed, torch.cuda.synchronize)
    per_step = np.array([step_ev[k].elapsed_time(step_ev[k + 1]) for k in range(args.steps)])
    stepper.check_overflow()     # the timed steps' sorts all fit (checked after the timing)
    if graph is not None:
        launches = per_step_launches * args.steps
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if distd:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_step = float(ms_t.item())

    # ---- in-step phases: the same step graph re-captured with a GPU-timer stamp on
    # every view's stream at sort start, forward start, backward start and backward end
    # (dass_timestamp), replayed after the timed region.  In the timed graph the 20
    # views' kernels overlap, so a raster kernel's in-step rate is the step's units of
    # that kernel over its phase's span (first start → last end; other kernels run
    # inside that span too, so the rate is a lower bound).
    phases = None
    if graph is not None and mvp is not None and my_cams:
        stamps = torch.zeros(4 * len(my_cams), dtype=torch.int64, device=dev)
        mvp.stamps = stamps
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            step_local(coll=distd and coll_in_graph["value"])
        mvp.stamps = None
        span = {"sort": [], "render_fwd": [], "render_bwd_raster": []}
        share = {"sort": [], "render_fwd": [], "render_bwd_raster": []}
        ends = []
        reps = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g2.replay()
            e1.record()
            if distd and not coll_in_graph["value"]:
                collective()
            torch.cuda.synchronize()
            t = stamps.view(-1, 4).cpu().numpy().astype(np.float64) / 1e6   # ms
            span["sort"].append(t[:, 1].max() - t[:, 0].min())
            span["render_fwd"].append(t[:, 2].max() - t[:, 1].min())
            span["render_bwd_raster"].append(t[:, 3].max() - t[:, 2].min())
            for k, v in fair_share(t).items():
                share[k].append(v)
            ends.append(t[:, 1:] - t[:, :1].min())
            reps.append(e0.elapsed_time(e1))
        del g2
        phases = {k: round(float(np.median(v)), 4) for k, v in span.items()}
        # fair-share attribution: each moment of the pass split evenly over the views' phases
        # running then (a straggler view's forward under 19 backward kernels gets 1/20 of it)
        phases["fair_share_ms"] = {k: round(float(np.median(v)), 4) for k, v in share.items()}
        # per view: (sort end, forward end, backward end) in ms from the first sort start
        phases["per_view_ends_ms"] = np.round(np.median(np.stack(ends), 0), 3).tolist()
        phases["stamped_step_ms"] = round(float(np.median(reps)), 4)   # the re-captured step, stamps included
        barrier()

    # ---- the collective's share of the step: the same all_reduce
    # (+ split-view ∇p̄ finish) timed alone, max over ranks
    allreduce = None
    if distd:
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a0.record()
        for _ in range(5):
            collective()
        a1.record()
        barrier()
        ar = torch.tensor([a0.elapsed_time(a1) / 5], device=dev)
        dist.all_reduce(ar, op=dist.ReduceOp.MAX)
        allreduce = {"ms": round(float(ar.item()), 4), "share_of_step": round(float(ar.item()) / ms_step, 4),
                     "bytes": int(grads.payload(args.payload).numel() * 4), "payload": args.payload,
                     "payload_what": "shift stage: g_mu, g_sigma, grad-stat sum and count (36 B/Gaussian)"
                                     if args.payload == "shift" else "every gradient (full buffer)",
                     "captured_in_step_graph": coll_in_graph["value"],
                     "timing": "the collective alone, 5 repeats, max over ranks"}

    # ---- the full training iteration: ∂L/∂C from the fused fidelity loss of
    # Eq. 3 against per-view ground truth (the render of 𝒢_{t−1} before the
    # shift), instead of a fixed ∂L/∂C.  Reported next to the metric.
    train = None
    if my_cams and not args.lean and plan.num_split == 0 and with_shift:   # SSIM needs whole views
        mvp.enable_loss(0.2)
        gts = torch.empty(len(my_cams), 3, H, W, device=dev)
        dass.dass_project_views(my_cams, deg, base.pos_opa, base.scale, base.rot, base.sh, None,
                                records.xy_depth, records.conic_opa, records.rgb, records.box,
                                records.rows, records.tiles)
        for k, cam in enumerate(my_cams):
            raster.forward(cam, records.view(k))
            gts[k].copy_(raster.img)

        # the dual deformation fields (f2) emit (μ, σ) for every Gaussian:
        # 𝓗_dyn for the dynamic group, 𝓗_st for the static one
        fields = DeformFields(synth.dual_fields(scene, "n3dv", seed=40), n, dev)
        fields.partition(base.dynamic)
        mu_f = torch.empty(n, 4, device=dev)
        sigma_f = torch.empty(n, 4, device=dev)

        def train_local():
            grads.zero_()
            fields.zero_grad()
            fields.forward(base.pos_opa, mu_f, sigma_f)
            dass.dass_apply_shift(base.pos_opa, base.rot, mu_f, sigma_f, None,
                                  shifted.pos_opa, shifted.rot)
            def project(v0, v1, part=dass.DASS_PROJECT_ALL):
                dass.dass_project_views_part(part, my_cams[v0:v1], deg, shifted.pos_opa,
                                             shifted.scale, shifted.rot, shifted.sh, None,
                                             records.xy_depth[v0:v1], records.conic_opa[v0:v1],
                                             records.rgb[v0:v1], records.box[v0:v1],
                                             records.rows[v0:v1], records.tiles[v0:v1])
            mvp.run(shifted, records, None, grads, gts=gts, project=project)
            dass.dass_apply_shift_bwd(base.rot, sigma_f, None, grads.pos_opa, grads.rot,
                                      g_mu, g_sigma)
            fields.backward(base.pos_opa, g_mu, g_sigma)

        for _ in range(2):
            train_local()
        barrier()
        tgraph = None
        if not args.no_graph:
            tgraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(tgraph):
                train_local()
            tgraph.replay()
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nt = max(3, args.steps // 2)
        t0.record()
        for _ in range(nt):
            if tgraph is None:
                train_local()
            else:
                tgraph.replay()
            if distd:
                allreduce_grads(grads, finish=finish_split, stage=args.payload)
                for x in fields.grad_tensors():
                    dist.all_reduce(x)
        t1.record()
        barrier()
        tms = torch.tensor([t0.elapsed_time(t1) / nt], device=dev)
        if distd:
            dist.all_reduce(tms, op=dist.ReduceOp.MAX)
        train = {"value": round(job_views / (float(tms.item()) / 1e3), 3), "unit": "views/s",
                 "ms_per_step": round(float(tms.item()), 4),
                 "loss_mean": float(mvp.losses[:, 0].mean().item()),
                 "what": "one full shift-stage iteration (§3.3): dual hash-grid deformation fwd (f2) → shift → fwd + fused L1/D-SSIM loss (Eq. 3, f1) + bwd over the views → shift bwd → deformation bwd (table + MLP grads)",
                 "graph": tgraph is not None}

    # ---- per-op breakdown: one extra SEQUENTIAL step, CUDA events on the
    # launching stream around each export (diagnostic; the timed step overlaps views)
    ops = {}
    if my_cams and not args.lean:
        E = lambda: torch.cuda.Event(enable_timing=True)
        e_proj = [E(), E()]
        # keep the GPU busy (≈1 ms) while the host marshals the first call, so the events
        # time the kernels and not the launch latency of the projection's 20 cameras
        torch.cuda._sleep(2_000_000)
        e_proj[0].record()
        dass.dass_project_views(my_cams, deg, shifted.pos_opa, shifted.scale, shifted.rot,
                                shifted.sh, None, records.xy_depth, records.conic_opa,
                                records.rgb, records.box, records.rows, records.tiles)
        e_proj[1].record()
        per = []
        for k, cam in enumerate(my_cams):
            xy, co, rgb, box, rows, tiles = records.view(k)
            ev = [E() for _ in range(4)]
            ev[0].record()
            dass.dass_bin_sort(cam, n, xy, box, rows, tiles, raster.sort_ws, raster.capacity, None,
                               raster.sorted_ids, raster.ranges, raster.num_pairs)
            ev[1].record()
            dass.dass_render_fwd(cam, raster.ranges, raster.sorted_ids, xy, co, rgb, box, None,
                                 raster.img, raster.T, raster.last, raster.accept, raster.capacity)
            ev[2].record()
            dass.dass_render_bwd_raster(cam, n, raster.ranges, raster.sorted_ids, xy, co, rgb, box,
                                        None, raster.T, raster.last, dLs[k], mvp.g2d[k],
                                        raster.accept, raster.capacity)
            ev[3].record()
            per.append(ev)
        e_pre = [E(), E()]
        e_pre[0].record()
        dass.dass_render_bwd_preprocess_views(
            my_cams, deg, shifted.pos_opa, shifted.scale, shifted.rot, shifted.sh, None,
            records.conic_opa[:len(my_cams)], records.rgb[:len(my_cams)], records.box[:len(my_cams)],
            mvp.g2d[:len(my_cams)], grads.pos_opa, grads.scale, grads.rot, grads.sh,
            grads.gradstat_sum, grads.gradstat_cnt)
        e_pre[1].record()
        e_loss = [E(), E()]
        if train is not None:
            e_loss[0].record()
            for k in range(len(my_cams)):
                dass.dass_fidelity_loss(raster.img, gts[k], 0.2, mvp.loss_ws[0], mvp.losses[k],
                                        mvp.loss_dL[0])
            e_loss[1].record()
        e_def = [E(), E(), E()]
        if train is not None:
            e_def[0].record()
            fields.forward(base.pos_opa, mu_f, sigma_f)
            e_def[1].record()
            fields.backward(base.pos_opa, g_mu, g_sigma)
            e_def[2].record()
        torch.cuda.synchronize()
        ops["project_views"] = e_proj[0].elapsed_time(e_proj[1])
        ops["bin_sort"] = sum(ev[0].elapsed_time(ev[1]) for ev in per)
        ops["render_fwd"] = sum(ev[1].elapsed_time(ev[2]) for ev in per)
        ops["render_bwd_raster"] = sum(ev[2].elapsed_time(ev[3]) for ev in per)
        ops["render_bwd_preprocess_views"] = e_pre[0].elapsed_time(e_pre[1])
        if train is not None:
            ops["fidelity_loss"] = e_loss[0].elapsed_time(e_loss[1])
            ops["deform_fwd"] = e_def[0].elapsed_time(e_def[1])
            ops["deform_bwd"] = e_def[1].elapsed_time(e_def[2])

    # ---- f4 (once per timestep, not in the step): error-guided densification
    # on this GPU's state — Eq. 4 selection from the step's ∇p̄ and an S_err
    # from one view's error map, spawn (K = 2), opacity prune + gather, and the
    # 16-channel identity-feature render of one view.  CUDA events per op.
    densify = None
    if my_cams and not args.lean:
        k4 = K4
        E = lambda: torch.cuda.Event(enable_timing=True)
        ws_p = torch.empty(dass.dass_partition_workspace(n) // 4 + 1, dtype=torch.int32, device=dev)
        s_err = torch.zeros(n, dtype=torch.uint8, device=dev)
        err = torch.empty(H, W, device=dev)
        raster.forward(my_cams[0], records.view(0))
        dass.dass_error_map(my_cams[0], raster.img, gts[0] if train is not None else raster.img,
                            0.05, err, None, n, shifted.pos_opa, s_err)
        in_S = torch.empty(n, dtype=torch.uint8, device=dev)
        idx = torch.empty(n, dtype=torch.int32, device=dev)
        cnt = torch.zeros(2, dtype=torch.int32, device=dev)
        gs = grads.gradstat_sum
        gcnt = grads.gradstat_cnt
        torch.cuda.synchronize()
        gbar = (gs / gcnt.clamp(min=1)).float()
        tau = float(torch.quantile(gbar[gcnt > 0][:1 << 20], 0.95).item())
        def timed(fn):
            """ms of one call on the current stream, after a warm-up call."""
            fn()
            a, b = E(), E()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b)

        ms = {}
        ms["densify_select"] = timed(lambda: dass.dass_densify_select(
            gs, gcnt, s_err, tau, 0.5 * tau, in_S, idx, cnt, ws_p))
        m = int(cnt[0].item())
        n_out = n + 2 * m
        o = [torch.empty(n_out, 4, device=dev) for _ in range(3)]
        o_sh = torch.empty(k4, n_out, 4, device=dev)
        o_dyn = torch.empty(n_out, dtype=torch.uint8, device=dev)
        ms["spawn"] = timed(lambda: dass.dass_spawn(
            deg, shifted.pos_opa, shifted.scale, shifted.rot, shifted.sh, base.dynamic, m, idx, 2,
            1.6, 0.1, 7, o[0], o[1], o[2], o_sh, o_dyn))
        keep = torch.empty(n_out, dtype=torch.uint8, device=dev)
        kidx = torch.empty(n_out, dtype=torch.int32, device=dev)
        ws_q = torch.empty(dass.dass_partition_workspace(n_out) // 4 + 1, dtype=torch.int32, device=dev)
        ms["prune_select"] = timed(lambda: dass.dass_prune_select(o[0], n, 0.05, keep, kidx, cnt, ws_q))
        mk = int(cnt[0].item())
        g_out = [torch.empty(mk, 4, device=dev) for _ in range(3)]
        g_sh = torch.empty(k4, mk, 4, device=dev)
        ms["gather"] = timed(lambda: dass.dass_gather(deg, o[0], o[1], o[2], o_sh, None, mk, kidx,
                                                      g_out[0], g_out[1], g_out[2], g_sh))
        feat = torch.randn(n, 16, device=dev)
        fout = torch.empty(16, H, W, device=dev)
        xy, co, rgb, box, _, _ = records.view(0)
        ms["render_features_16ch_one_view"] = timed(lambda: dass.dass_render_features(
            my_cams[0], raster.ranges, raster.sorted_ids, xy, co, box, feat, fout))
        ms["render_fwd_rgb_same_view"] = timed(lambda: dass.dass_render_fwd(
            my_cams[0], raster.ranges, raster.sorted_ids, xy, co, rgb, box, None, raster.img,
            raster.T, raster.last, raster.accept, raster.capacity))
        densify = {"selected": m, "spawned": 2 * m, "kept_after_prune": mk, "rows": n_out,
                   "bytes_gather_per_row": 16 * 3 + 16 * k4, "ms": ms}
        densify["ms"] = {k: round(v, 4) for k, v in densify["ms"].items()}

    # ---- end-to-end through the public API with host buffers: every step
    # uploads its inputs from pinned host memory and downloads its gradients.
    # Double-buffered: step k+1's upload (copy stream) overlaps step k's
    # compute, and step k's download overlaps step k+1; all inside the timed
    # region (first upload → last download).
    e2e = None
    if not args.no_e2e:
        # Two complete input/output buffer sets, each with its own captured step graph:
        # step k runs set k mod 2, the upload of step k+1 goes straight into the other
        # set (copy engine, pinned host → device), and step k's gradients are read
        # straight out of its set — no device-side staging copies on the compute stream.
        # Inputs: the parameters and shift offsets as one flat buffer (dist.FlatParams) — at
        # N > 1 each rank uploads only its 1/N shard and an in-place all_gather over NVLink
        # assembles the rest — plus this rank's own views' ∂L/∂C, uploaded view by view.
        shard_world = plan_world if args.emulate else world
        shard_rank = plan_rank if args.emulate else rank
        hp = FlatParams.allocate(n, K4, "cpu", world=shard_world, pin=True)
        for dst, src in ((hp.pos_opa, scene.pos_opa), (hp.scale, scene.scale), (hp.rot, scene.rot),
                         (hp.sh, scene.sh), (hp.mu, mu), (hp.sigma, sigma)):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src)))
        h_dl = dLs.cpu().pin_memory()
        dps = [FlatParams.allocate(n, K4, dev, world=shard_world) for _ in range(2)]
        for dp in dps:   # whole buffers once; under --emulate the other shards stay as gathered
            dp.flat.copy_(hp.flat)
        sets = [stepper.buffers(DeviceScene(dp.pos_opa, dp.scale, dp.rot, dp.sh, deg, base.dynamic),
                                dp.mu, dp.sigma, torch.empty_like(dLs)) for dp in dps]
        h_out = [torch.empty(flat.numel(), dtype=torch.float32).pin_memory() for _ in range(2)]
        h2d_params = hp.shard(shard_rank).numel() * 4
        h2d = h2d_params + h_dl.numel() * 4
        d2h = flat.numel() * 4
        comp = torch.cuda.current_stream()
        copy_in = torch.cuda.Stream(device=dev)
        copy_out = torch.cuda.Stream(device=dev)
        nv = len(mine)
        ev_par = [torch.cuda.Event() for _ in range(2)]     # parameters + offsets of set b landed
        ev_dl = [[torch.cuda.Event() for _ in range(nv)] for _ in range(2)]   # view v's ∂L/∂C landed
        ev_res = [torch.cuda.Event() for _ in range(2)]     # step on set b done
        ev_out = [torch.cuda.Event() for _ in range(2)]     # download from set b done
        for e in ev_par + [x for row in ev_dl for x in row]:
            e.record(copy_in)                               # create the events before capture
        torch.cuda.synchronize()
        cudart = ctypes.CDLL("libcudart.so.12")             # the runtime libdass links

        def wait_external(stream, event):
            """cudaStreamWaitEvent(…, cudaEventWaitExternal): inside a capture this becomes an
            event-wait node on the upload stream's record of the current step."""
            rc = cudart.cudaStreamWaitEvent(ctypes.c_void_p(stream.cuda_stream),
                                            ctypes.c_void_p(event.cuda_event), ctypes.c_uint(1))
            if rc != 0:
                raise RuntimeError(f"cudaStreamWaitEvent failed: {rc}")

        # Each set's step graph waits inside itself: for the parameters before the shift, and on
        # view v's stream for its ∂L/∂C right before its backward, so a step starts as soon as its
        # 105 MB of parameters have landed while the 20 views' 16 MB gradients images still stream in.
        graphs = [None, None]

        def hook(b, capture=True):
            # cudaEventWaitExternal is valid only under capture; eagerly it is a plain wait
            w = wait_external if capture else (lambda st, e: st.wait_event(e))
            if mvp is not None:
                mvp.before_bwd = None if b is None else (lambda v, st: w(st, ev_dl[b][v]))

        for b in range(2):
            if graph is not None:
                hook(b)
                graphs[b] = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graphs[b]):
                    # as the timed step: the collective in the graph
                    step_local(sets[b], wait_inputs=lambda b=b: wait_external(
                        torch.cuda.current_stream(), ev_par[b]), coll=coll_in_graph["value"])
        hook(None)

        def upload(k):
            b = k % 2
            with torch.cuda.stream(copy_in):
                copy_in.wait_event(ev_res[b])        # the step that last read set b is done
                dps[b].upload_shard(hp, shard_rank)
                if world > 1:
                    dps[b].allgather(rank)           # NCCL, ordered on copy_in
                ev_par[b].record(copy_in)
                for v in range(nv):
                    sets[b].dLs[v].copy_(h_dl[v], non_blocking=True)
                    ev_dl[b][v].record(copy_in)

        def compute(k):
            b = k % 2
            comp.wait_event(ev_out[b])               # set b's previous gradients downloaded
            if graphs[b] is not None:
                run_step(graphs[b], sets[b])
            else:                                    # eager: the same waits, issued directly
                hook(b, capture=False)
                step_local(sets[b], wait_inputs=lambda: comp.wait_event(ev_par[b]), coll=distd)
                hook(None)
            ev_res[b].record(comp)

        def download(k):
            b = k % 2
            with torch.cuda.stream(copy_out):
                copy_out.wait_event(ev_res[b])
                h_out[b].copy_(sets[b].grads.flat, non_blocking=True)
                ev_out[b].record(copy_out)

        def run_e2e(nsteps):
            for b in range(2):
                ev_res[b].record(comp)
                ev_out[b].record(comp)
            upload(0)
            for k in range(nsteps):
                if k + 1 < nsteps:
                    upload(k + 1)
                compute(k)
                download(k)
            comp.wait_stream(copy_out)

        run_e2e(2)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_e2e(args.steps)
        e1.record()
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
        if distd:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": job_views / (float(ems.item()) / 1e3), "unit": "views/s",
               "ms_per_step": float(ems.item()), "h2d_bytes_per_step": int(h2d),
               "h2d_params_shard": f"{h2d_params} B = 1/{shard_world} of the parameters"
                                   + ("; the all_gather is not run under --emulate" if args.emulate
                                      and shard_world > 1 else ""),
               "d2h_bytes_per_step": int(d2h),
               "pipelining": "two buffer sets, one captured graph each: the upload of step k+1 "
                             "and the download of step k−1 overlap step k, with no device-side copies; "
                             "inside a step, view v's backward waits only for its own dL/dC upload"}

    # ---- gather stats to rank 0
    if distd:
        obj = [None] * world
        dist.all_gather_object(obj, stats)
        allst = {k: sum((o[k] for o in obj), []) for k in stats}
        launches_t = torch.tensor([launches], device=dev, dtype=torch.int64)
        dist.all_reduce(launches_t)
        launches = int(launches_t.item())
    else:
        allst = stats
    clocks = clk.summary()
    tiles_summary = None
    if tiles_hist:   # rank 0's views (mean, p50, p99 of tiles_touched over visible Gaussians)
        h = torch.stack(tiles_hist).sum(0).numpy().astype(np.float64)
        c = np.cumsum(h) / max(h.sum(), 1.0)
        tiles_summary = {"mean": round(float((np.arange(h.size) * h).sum() / max(h.sum(), 1.0)), 3),
                         "p50": int(np.searchsorted(c, 0.5)), "p99": int(np.searchsorted(c, 0.99))}
    result = None
    if rank == 0:
        pk, pk_kind = peaks()
        f_max = pk.get("sm_max_mhz", 1965.0) * 1e6
        peak_tflops = SM_COUNT * FP32_LANES * 2 * f_max / 1e12
        # the dominant kernel of the step (the larger of the two raster kernels in the
        # isolated per-op pass) against the FP32 roof, algorithmic flops only
        dom = dominant_roofline(ops, stats, f_max, peak_tflops, profiled=args.config == "c3",
                                phases=phases, work=work)
        views_s = job_views / (ms_step / 1e3)
        result = {
            "metric": METRIC, "value": round(views_s, 3), "unit": "views/s",
            "mpix_per_s": round(views_s * W * H / 1e6, 1),
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "ms_per_step_percentiles_rank0": {q: round(float(np.percentile(per_step, v)), 4)
                                              for q, v in (("p10", 10), ("p50", 50), ("p90", 90))},
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded N3DV-shaped scene and rig)",
            "config": {"workload": wl, "n_gaussians": n, "views": len(cams), "width": W,
                       "height": H, "sh_degree": deg, "dynamic_frac": 0.3 if with_shift else None,
                       "cuda_graph": graph is not None, "streams": args.streams,
                       "pass_options": vars(opts),
                       "emulated_share": args.emulate,
                       "parallelism": f"view-sharded dp{world}" + (
                           f" ({plan.num_split} views split into tile halves)" if plan.num_split else ""),
                       "l2": "inputs larger than L2 (≈0.5 GB of params, dL/dC and records per step)"},
            "roofline": dom,
            "ops_ms_per_step_rank0": {k: round(v, 4) for k, v in ops.items()},
            "hot_path_roofline": hot_path_roofline(ops, stats, pk, peak_tflops, n, len(my_cams), deg,
                                                   f_max, profiled=args.config == "c3"),
            "rows_roofline": rows_roofline(ops, densify, allst, pk, peak_tflops, n, W, H,
                                           len(my_cams), deg),
            "scene_stats": None if args.lean else {"K_per_view_mean": float(np.mean(allst["K"])),
                            "n_visible_per_view_mean": float(np.mean(allst["n_visible"])),
                            "tiles_per_visible_gaussian": tiles_summary,
                            "P_fwd_per_px": float(np.sum(allst["P_fwd"]) / (len(allst["K"]) * W * H)),
                            "P_bwd_per_px": float(np.sum(allst["P_bwd"]) / (len(allst["K"]) * W * H)),
                            "accepted_per_px": float(np.sum(allst["accepted"]) / (len(allst["K"]) * W * H)),
                            "early_terminated_frac": float(np.sum(allst["terminated_px"]) / (len(allst["K"]) * W * H)),
                            "tile_list_mean": float(np.mean(allst["tile_list_mean"])),
                            "tile_list_max": int(np.max(allst["tile_list_max"]))},
            "allreduce": allreduce,
            "training_step_with_loss": train,
            "densification_f4": densify,
            "densification_c4": c4info,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "e2e": e2e,
        }
    if distd:
        dist.barrier()
        dist.destroy_process_group()
    return result, (cams, scene)


# ------------------------------------------------------ oracle baseline ----

def time_oracle(cams, scene, views, seed_base=1000, shift=True, mode="scatter"):
    """Seconds of the oracle doing the step's work for `views`: the shift (O1) when
    the step has one, then fwd+bwd (O2-O6, double) per view."""
    import oracle
    from paper_2411_14847_b200 import synth
    W, H = cams[0].width, cams[0].height
    t0 = time.perf_counter()
    sc = scene
    if shift:
        mu, sigma = synth.shift_offsets(scene, seed=33)
        po, ro = oracle.shift(scene.pos_opa, scene.rot, mu, sigma, scene.dynamic)
        sc = synth.Scene(po.astype(np.float32), scene.scale, ro.astype(np.float32), scene.sh,
                         scene.sh_degree, scene.dynamic)
    for v in views:
        dL = synth.grad_image(cams[v], seed_base + v, 1.0 / (3 * W * H))
        oracle.render_bwd(cams[v], sc, dL, mode=mode)
    return time.perf_counter() - t0


def host_cpu():
    """The CPU the oracle ran on (model, affinity, logical CPUs)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "affinity": len(os.sched_getaffinity(0)), "cpu_count": os.cpu_count()}


def cpu_baseline(cams, scene, nviews, config="c3"):
    """The oracle as it stands, on the box's host cores: C1 in its
    literal form (every pixel over every depth-sorted Gaussian) and C2 in its
    scatter form, each single-threaded and on every OpenMP thread; C3-C5 on a
    bounded sample of the views, every thread."""
    import oracle
    oracle.build()
    allt = oracle.threads()
    if config in ("c1", "c2"):
        mode = "literal" if config == "c1" else "scatter"
        out = {}
        for label, k in (("all_threads", allt), ("single_thread", 1)):
            oracle.set_threads(k)
            reps, secs = 0, 0.0
            while reps < 3 or (secs < 2.0 and reps < 50):
                secs += time_oracle(cams, scene, [0], shift=False, mode=mode)
                reps += 1
            out[label] = {"seconds_per_step": round(secs / reps, 4), "threads": k, "repeats": reps}
        oracle.set_threads(allt)
        s1 = out["all_threads"]["seconds_per_step"]
        return {"value": round(1.0 / s1, 4), "unit": "views/s", "cores": allt, "kind": "oracle",
                "host": host_cpu(), "form": mode,
                "sample": f"the whole {config} step (one view fwd+bwd, {mode} form, double), repeated",
                "seconds": out}
    secs = time_oracle(cams, scene, list(range(nviews)))
    out = {"value": round(nviews / secs, 4), "unit": "views/s", "cores": allt,
           "kind": "oracle", "host": host_cpu(),
           "sample": f"{nviews} of the {len(cams)} views (fwd+bwd, scatter form, double) + the shift, "
                     f"{secs:.1f} s on {allt} OpenMP threads"}
    if config != "c5":   # C5's 1M Gaussians would take about a minute on one thread
        # and one view (+ the shift) on one thread: the oracle's serial rate
        oracle.set_threads(1)
        try:
            s1 = time_oracle(cams, scene, [0])
        finally:
            oracle.set_threads(allt)
        out["single_thread"] = {"value": round(1.0 / s1, 4), "unit": "views/s", "threads": 1,
                                "sample": f"view 0 (fwd+bwd, scatter form, double) + the shift, {s1:.1f} s"}
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    from paper_2411_14847_b200 import synth
    import oracle
    oracle.build()
    cams, scene, wl = workload(args)
    W, H = cams[0].width, cams[0].height
    shift = args.config not in ("c1", "c2")
    mode = "literal" if args.config == "c1" else "scatter"
    for k in range(args.warmup):
        time_oracle(cams, scene, [k % len(cams)], shift=shift, mode=mode)
    secs = []
    for k in range(args.steps):
        secs.append(time_oracle(cams, scene, [k % len(cams)], shift=shift, mode=mode))
    s = float(np.mean(secs))
    value = 1.0 / s
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "views/s",
            "mpix_per_s": round(value * W * H / 1e6, 3), "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(s * 1e3, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N3DV-shaped scene and rig)",
            "config": {"workload": wl, "n_gaussians": scene.n, "views": len(cams),
                       "width": W, "height": H, "sh_degree": scene.sh_degree,
                       "parallelism": "CPU oracle, OpenMP"},
            "cpu_baseline": {"value": round(value, 4), "unit": "views/s", "cores": oracle.threads(),
                             "kind": "oracle",
                             "sample": ("each step = the shift + fwd+bwd of ONE of the views (bounded sample)"
                                        if shift else f"each step = the whole {args.config} fwd+bwd ({mode} form)")},
            "e2e": {"value": round(value, 4), "unit": "views/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# Algorithmic work of the SURVEY §8(f) rows, per unit:
FLOP_SSIM_PER_PXCH = 2 * (5 * 11 * 2) + 40 + 2 * (3 * 11 * 2) + 10   # fwd + bwd stencils
BYTES_LOSS_PER_PX = 3 * 4 * 3                                           # img, gt in; ∂L/∂img out
DEFORM_IN = {"dyn": 32, "st": 16}                                       # L·F (N3DV profile)


FLOP_FWD_ACCEPTED = 15   # blend of an accepted (pixel, entry): 1 − α, T·(1 − α), w, 3 colour FMAs
FLOP_FWD_INBOX = 8       # α of an in-box (pixel, entry): dx, dy, power, exp, o·G, compare
RASTER_KERNELS = {
    "render_fwd": ("render_fwd_tw_kernel via dass_render_fwd (lists)", "P_fwd", 20,
                   f"{FLOP_FWD_ACCEPTED} flop per accepted (pixel, entry) + {FLOP_FWD_INBOX} per "
                   "in-box (pixel, entry) up to termination"),
    "render_bwd_raster": ("render_bwd_tw_kernel via dass_render_bwd_raster (accepted units only)",
                          "P_bwd", 55, f"{FLOP_BWD_ACCEPTED} flop per accepted (pixel, entry)"),
}


def issue_view(prof, ms, launches, f_max):
    """The kernel against the instruction-issue roof (148 SMs × 4 schedulers × 1 warp
    instruction per clock): executed warp instructions per launch from the committed ncu
    summary (one C3 view; the scene is fixed) × the launches, over the live time.  The
    raster kernels are issue-bound (compares, selects, shuffles, MUFU next to the FMAs),
    so this is the roof they actually meet; `frac` above counts algorithmic flops only."""
    instr = profiled_instructions(prof)
    if not instr or not ms or ms != ms:
        return None
    rate = instr * launches / (ms / 1e3)
    peak = SM_COUNT * 4 * f_max
    return {"warp_instr_per_launch": instr, "achieved_ginstr_s": round(rate / 1e9, 1),
            "peak_ginstr_s": round(peak / 1e9, 1), "frac": round(rate / peak, 4),
            "source": f"profiles/{PROFILE_TAG}_ncu_{prof}.txt (Executed Instructions)"}


def dominant_roofline(ops, stats, f_max, peak_tflops, profiled=True, phases=None, work=None):
    """Roofline object of the step's dominant kernel: whichever raster kernel (forward
    or backward) takes more of the timed step (its fair-share phase time, when the
    stamped re-capture ran; else its isolated per-op time).  achieved = the work units
    of the step's launches / their summed isolated durations."""
    cand = {k: ops.get(k, float("nan")) for k in RASTER_KERNELS}
    cand = {k: v for k, v in cand.items() if v == v and v > 0}
    if not cand or not stats.get("accepted"):
        return None
    share = (phases or {}).get("fair_share_ms") or {}
    if all(share.get(k) for k in cand):
        key = max(cand, key=lambda k: share[k])
    else:
        key = max(cand, key=cand.get)
    ms = cand[key]
    name, p_key, instr, unit = RASTER_KERNELS[key]
    full = work["full"] if work and work["full"].get("accepted") else None
    acc = full["accepted"] if full else float(sum(stats["accepted"]))
    if key == "render_fwd":
        flops = FLOP_FWD_ACCEPTED * acc + FLOP_FWD_INBOX * float(sum(stats["P_fwd"]))
        per_unit = {"accepted": FLOP_FWD_ACCEPTED, "P_fwd": FLOP_FWD_INBOX}
    else:
        flops = FLOP_BWD_ACCEPTED * acc
        per_unit = {"accepted": FLOP_BWD_ACCEPTED}
    achieved = flops / (ms / 1e3) / 1e12
    units = full[p_key] if full else float(sum(stats[p_key]))
    peak_i = SM_COUNT * FP32_LANES * f_max / 1e12
    rate = units * instr / (ms / 1e3) / 1e12
    prof = "render_fwd" if key == "render_fwd" else "render_bwd"
    # the committed ncu summaries are of a C3 view: other configs get no profiled numbers
    # Headline (SURVEY §8(d)'s unit): every evaluated (pixel, tile-list entry) — P_fwd for
    # the forward, P_bwd for the backward — × its FP32-pipe instruction count (≈20 / ≈55)
    # against the FP32 pipe's issue peak, SMs × 128 lanes × f_SM (one FP32-pipe
    # instruction per lane per clock).  The builder's algorithmic flop count is kept as a
    # secondary view.
    return {"bound": "alu", "kernel": name, "achieved": round(rate, 3), "peak": round(peak_i, 2),
            "unit": "Tinstr/s", "frac": round(rate / peak_i, 4),
            "traffic": profiled_traffic(prof) if profiled else None,
            "traffic_source": f"profiles/{PROFILE_TAG}_ncu_{prof}.txt (ncu --set full, dram read+write "
                              "per launch = one view)",
            "peak_kind": f"FP32 pipe {SM_COUNT} SMs x {FP32_LANES} lanes x 1 instr/clk at {f_max/1e6:.0f} MHz",
            "work_unit": f"SURVEY §8(d): evaluated (pixel, tile-list entry) = {p_key} (scene statistic), "
                         f"x {instr} FP32-pipe instructions per unit",
            "units_per_step": int(units), "instr_per_unit": instr,
            "algorithmic_flop_view": {"achieved_tflops": round(achieved, 2), "peak_tflops": round(peak_tflops, 1),
                                      "frac": round(achieved / peak_tflops, 4), "flop_unit": unit,
                                      "units_per_step": {"accepted": int(acc), p_key: int(units)},
                                      "flop_per_unit": per_unit,
                                      "what": "the builder's count of the flops the kernel must do on the "
                                              "pixels it accepts (FMA = 2), against 2 x the FP32 peak"},
            "issue_view": issue_view(prof, ms, full["views"] if full else len(stats["accepted"]),
                                     f_max) if profiled else None,
            "timing": "isolated launches: one sequential pass over the step's kernels (CUDA events on "
                      "the launching stream), since in the timed graph the per-view kernels of 20 "
                      "streams overlap",
            "share_of_step_kernels": round(ms / max(sum(v for k, v in ops.items() if k in STEP_OPS), 1e-9), 4),
            "ncu_share_source": f"profiles/{PROFILE_TAG}_launches.txt",
            "in_step": in_step_view(key, phases, step_units(work, p_key, units), instr, peak_i, prof,
                                    step_units(work, "views", len(stats["accepted"])), f_max,
                                    profiled),
            "other_raster_kernel": other_raster(key, stats, ops, phases, peak_i, f_max, profiled, work)}


def step_units(work, p_key, default):
    """The units the rank's step renders (split views weighted by their tile share)."""
    return work["step"][p_key] if work and work["step"].get(p_key) else default


def other_raster(key, stats, ops, phases, peak_i, f_max, profiled, work=None):
    """The other raster kernel (forward when the backward dominates, and vice versa) in the
    same survey unit, alone and inside the step, for comparison."""
    other = next(k for k in RASTER_KERNELS if k != key)
    ms = ops.get(other)
    if not ms or ms != ms:
        return None
    name, p_key, instr, _ = RASTER_KERNELS[other]
    units = (work["full"][p_key] if work and work["full"].get(p_key)
             else float(sum(stats[p_key])))
    rate = units * instr / (ms / 1e3) / 1e12
    prof = "render_fwd" if other == "render_fwd" else "render_bwd"
    return {"kernel": name, "work_unit": f"{p_key} x {instr} FP32-pipe instructions",
            "achieved": round(rate, 3), "frac": round(rate / peak_i, 4),
            "in_step": in_step_view(other, phases, step_units(work, p_key, units), instr, peak_i,
                                    prof, step_units(work, "views", len(stats["accepted"])), f_max,
                                    profiled)}


def fair_share(t):
    """t[v] = GPU-timer stamps (sort start, forward start, backward start, backward end) of
    view v.  Every interval between consecutive stamps is split evenly over the phases
    (sort, forward, backward) of the views running in it; returns the ms attributed to
    each phase over the whole pass."""
    names = ("sort", "render_fwd", "render_bwd_raster")
    ev = np.unique(t.reshape(-1))
    out = {k: 0.0 for k in names}
    for a, b in zip(ev[:-1], ev[1:]):
        mid = 0.5 * (a + b)
        act = [int(np.sum((t[:, i] <= mid) & (mid < t[:, i + 1]))) for i in range(3)]
        tot = sum(act)
        if tot:
            for i, k in enumerate(names):
                out[k] += (b - a) * act[i] / tot
    return out


def in_step_view(key, phases, units, instr, peak_i, prof, launches, f_max, profiled):
    """The same kernel inside the timed step graph: the step's units over the span of
    its phase (first launch start → last launch end, GPU-timer stamps on the view
    streams), i.e. with the overlap of the 20 views' launches that the isolated pass
    removes.  A lower bound: other kernels also run inside the span."""
    if not phases or not phases.get(key):
        return None
    phases = dict(phases)
    ms = phases["fair_share_ms"][key]
    span = phases[key]
    rate = units * instr / (ms / 1e3) / 1e12
    rate_span = units * instr / (span / 1e3) / 1e12
    out = {"phase_ms": ms, "achieved": round(rate, 3), "frac": round(rate / peak_i, 4),
           "span_ms": span, "span_frac": round(rate_span / peak_i, 4),
           "phases_ms": phases,
           "timing": "GPU-timer stamps (dass_timestamp) on every view's stream in a re-capture "
                     "of the timed step graph, median of 3 replays; phase_ms = the pass time "
                     "attributed to this kernel's phase when every moment is split evenly over "
                     "the views' phases running then; span_ms = first launch start to last "
                     "launch end (a lower bound of the rate: other kernels run in the span)"}
    if profiled:
        iv = issue_view(prof, ms, launches, f_max)
        if iv:
            out["issue_frac"] = iv["frac"]
    return out


def issue_view_parts(profs, ms, views, f_max):
    """Executed warp instructions of the committed 20-view ncu summaries of a kernel
    group's launches (profiles/<tag>_ncu_<name>.txt, one launch each for all C3 views) over
    the group's measured time, against the issue roof (148 SMs × 4 per clock).  Only for
    the 20-view C3 launch the profiles describe."""
    if views != 20 or not ms or ms != ms:
        return None
    instr = [profiled_instructions(p) for p in profs]
    if not all(instr):
        return None
    rate = sum(instr) / (ms / 1e3)
    peak = SM_COUNT * 4 * f_max
    return {"warp_instr_per_step": int(sum(instr)), "frac": round(rate / peak, 4),
            "source": ", ".join(f"profiles/{PROFILE_TAG}_ncu_{p}.txt" for p in profs)}


def hot_path_roofline(ops, stats, pk, peak_fp32, n, views, deg, f_max=1965e6, profiled=False):
    """Every §8(a) kernel group of the step against its own roof,
    from the sequential per-op pass of rank 0 and that rank's scene statistics."""
    if not ops or not stats.get("K"):
        return None
    hbm = pk.get("hbm_gbs", 6650.0)
    k4 = (3 * (deg + 1) ** 2 + 3) // 4
    K = float(sum(stats["K"]))
    acc = float(sum(stats["accepted"]))
    pfwd = float(sum(stats["P_fwd"]))
    out = {}

    def hb(name, by):
        t = ops[name] / 1e3
        out[name] = {"bound": "hbm", "bytes": int(by), "achieved_gbs": round(by / t / 1e9, 1),
                     "peak_gbs": hbm, "frac": round(by / t / 1e9 / hbm, 4)}

    # projection: parameters once per launch (48 + 16·K4 B) + 60 B of records per view
    hb("project_views", n * (48 + 16 * k4) + n * views * 60)
    out["project_views"]["note"] = "issue-bound, not HBM: fp64 record chain + the fp32 key-chain replica"
    if profiled:   # the committed 20-view summaries are of C3
        out["project_views"]["issue_view"] = issue_view_parts(
            ("project_keys_20v", "project_records_20v"), ops["project_views"], views, f_max)
    # binning + sort: per pair 8 B key written by emit, 2 onesweep passes of 16 B read + 16 B
    # written (key + id), finalize 8 B read + 4 B id + range writes; N-key presort ≈ 4 × 32 B
    hb("bin_sort", K * (8 + 2 * 32 + 12) + n * views * 4 * 32)
    out["bin_sort"]["note"] = "latency-bound launch chain (10 kernels per view), hidden under other views' raster kernels"
    # preprocess: 88 B of records + moments per Gaussian-view, parameters and gradients once
    hb("render_bwd_preprocess_views", n * views * 88 + n * 3 * (48 + 16 * k4))
    if profiled:
        out["render_bwd_preprocess_views"]["issue_view"] = issue_view_parts(
            ("preprocess_20v", "preprocess2_20v"), ops["render_bwd_preprocess_views"], views, f_max)
    t = ops["render_fwd"] / 1e3
    fl = FLOP_FWD_ACCEPTED * acc + FLOP_FWD_INBOX * pfwd   # accepted blend + every in-box α evaluation
    out["render_fwd"] = {"bound": "alu", "flop": int(fl), "achieved_tflops": round(fl / t / 1e12, 2),
                         "peak_tflops": round(peak_fp32, 1), "frac": round(fl / t / 1e12 / peak_fp32, 4),
                         "unit": "15 flop per accepted (pixel, entry) + 8 per in-box evaluation"}
    t = ops["render_bwd_raster"] / 1e3
    fl = float(FLOP_BWD_ACCEPTED) * acc
    out["render_bwd_raster"] = {"bound": "alu", "flop": int(fl),
                                "achieved_tflops": round(fl / t / 1e12, 2),
                                "peak_tflops": round(peak_fp32, 1),
                                "frac": round(fl / t / 1e12 / peak_fp32, 4),
                                "unit": f"{FLOP_BWD_ACCEPTED} flop per accepted (pixel, entry)"}
    return out


def rows_roofline(ops, densify, allst, pk, peak_fp32, n, W, H, views, deg):
    """Achieved vs peak for the §8(f) kernels timed in this run (rank 0)."""
    out = {}
    hbm = pk.get("hbm_gbs", 6650.0)
    tf32 = pk.get("bf16_tflops", 2250.0) / 2.0        # nominal dense TF32 = bf16 / 2
    if "fidelity_loss" in ops and views:
        t = ops["fidelity_loss"] / 1e3
        fl = views * 3 * W * H * FLOP_SSIM_PER_PXCH
        by = views * W * H * BYTES_LOSS_PER_PX
        out["f1_fidelity_loss"] = {"bound": "alu", "achieved_tflops": round(fl / t / 1e12, 2),
                                   "peak_tflops": round(peak_fp32, 1),
                                   "frac": round(fl / t / 1e12 / peak_fp32, 4),
                                   "hbm_gbs": round(by / t / 1e9, 1), "hbm_frac": round(by / t / 1e9 / hbm, 4),
                                   "unit": f"pixel-channel ({FLOP_SSIM_PER_PXCH} flop)"}
    if "deform_fwd" in ops:
        # 0.3 N dynamic (in 32) + 0.7 N static (in 16); 3 TF32 passes per layer
        per = lambda i: 2 * (64 * i + 64 * 64 + 16 * 64)
        fl = 3 * (0.3 * n * per(DEFORM_IN["dyn"]) + 0.7 * n * per(DEFORM_IN["st"]))
        t = ops["deform_fwd"] / 1e3
        out["f2_deform_fwd_tcgen05"] = {"bound": "tensor", "achieved_tflops": round(fl / t / 1e12, 2),
                                        "peak_tflops": round(tf32, 1),
                                        "frac": round(fl / t / 1e12 / tf32, 4),
                                        "unit": "Gaussian (3×TF32 MMA flops incl. the N = 16 padded head)"}
    if "deform_bwd" in ops:
        per = lambda i: 2 * (64 * i + 64 * 64 + 7 * 64)
        fl = 3 * (0.3 * n * per(DEFORM_IN["dyn"]) + 0.7 * n * per(DEFORM_IN["st"]))
        t = ops["deform_bwd"] / 1e3
        out["f2_deform_bwd_simt"] = {"bound": "alu", "achieved_tflops": round(fl / t / 1e12, 2),
                                     "peak_tflops": round(peak_fp32, 1),
                                     "frac": round(fl / t / 1e12 / peak_fp32, 4),
                                     "unit": "Gaussian (recompute + δ chain + weight gradients = 3× fwd flops)"}
    if densify:
        ms = densify["ms"]
        k4 = (3 * (deg + 1) ** 2 + 3) // 4
        rows = densify["kept_after_prune"]
        by = 2 * rows * (48 + 16 * k4)
        t = ms["gather"] / 1e3
        out["f4_gather"] = {"bound": "hbm", "achieved_gbs": round(by / t / 1e9, 1),
                            "peak_gbs": hbm, "frac": round(by / t / 1e9 / hbm, 4),
                            "unit": f"row ({48 + 16 * k4} B read + written)"}
        acc0 = allst["accepted"][0] if allst.get("accepted") else None
        if acc0:
            fl = acc0 * (2 * 16 + 15)
            t = ms["render_features_16ch_one_view"] / 1e3
            out["f4_render_features"] = {"bound": "alu", "achieved_tflops": round(fl / t / 1e12, 2),
                                         "peak_tflops": round(peak_fp32, 1),
                                         "frac": round(fl / t / 1e12 / peak_fp32, 4),
                                         "unit": "accepted (pixel, entry) of view 0 (2·16 + 15 flop)"}
    return out


def profiled_instructions(kernel: str):
    """Executed warp instructions per launch of `kernel` from the committed ncu summary."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        f"{PROFILE_TAG}_ncu_{kernel}.txt")
    try:
        for line in open(path):
            if line.startswith("Executed Instructions"):
                return int(float(line.split()[2].replace(",", "")))
    except (OSError, ValueError, IndexError):
        pass
    return None


def profiled_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu summary (null if absent)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        f"{PROFILE_TAG}_ncu_{kernel}.txt")
    try:
        for line in open(path):
            if line.startswith("dram_bytes_per_launch:"):
                return int(line.split()[1])
    except OSError:
        pass
    return None


def main():
    args = parse()
    # stdout carries exactly the one JSON line: anything else written to fd 1 by the
    # libraries underneath (e.g. NCCL's "NCCL version …" banner) goes to stderr
    out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    if args.impl == "reference":
        r = run_reference(args)
        if r is not None:
            print(json.dumps(r), file=out, flush=True)
        return
    result, (cams, scene) = run_ours(args)
    rank, world, _ = dist_env()
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline(cams, scene, min(args.cpu_sample_views, len(cams)),
                                                  args.config)
        print(json.dumps(result), file=out, flush=True)


if __name__ == "__main__":
    main()
