"""Device buffers and the per-view call sequence around libdass (plumbing).

PyTorch supplies device memory and streams; every arithmetic step runs in the
CUDA kernels behind `paper_2411_14847_b200.dass` (the C-ABI).  This module only
allocates the documented layouts and calls the exports in order:

  step:  [dass_apply_shift] → dass_project_views (all views, params read once)
         → per view: dass_bin_sort (graph mode) → dass_render_fwd → dass_render_bwd
         → [dass_apply_shift_bwd]
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import dass
from .synth import sh_planes


def _torch():
    import torch
    return torch


@dataclass
class DeviceScene:
    pos_opa: "torch.Tensor"   # [N,4] f32
    scale: "torch.Tensor"     # [N,4] f32
    rot: "torch.Tensor"       # [N,4] f32
    sh: "torch.Tensor"        # [K4,N,4] f32
    sh_degree: int
    dynamic: "torch.Tensor | None" = None  # [N] u8

    @property
    def n(self) -> int:
        return self.pos_opa.shape[0]

    @staticmethod
    def from_host(scene, device="cuda", pin=False) -> "DeviceScene":
        torch = _torch()
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
        dyn = None if scene.dynamic is None else t(scene.dynamic.astype(np.uint8))
        return DeviceScene(t(scene.pos_opa), t(scene.scale), t(scene.rot), t(scene.sh),
                           scene.sh_degree, dyn)


@dataclass
class Grads:
    pos_opa: "torch.Tensor"
    scale: "torch.Tensor"
    rot: "torch.Tensor"
    sh: "torch.Tensor"
    gradstat_sum: "torch.Tensor"
    gradstat_cnt: "torch.Tensor"

    @staticmethod
    def zeros(n, sh_degree, device="cuda") -> "Grads":
        torch = _torch()
        f = lambda *s: torch.zeros(*s, dtype=torch.float32, device=device)
        return Grads(f(n, 4), f(n, 4), f(n, 4), f(sh_planes(sh_degree), n, 4), f(n),
                     torch.zeros(n, dtype=torch.int32, device=device))

    def zero_(self):
        for t in (self.pos_opa, self.scale, self.rot, self.sh, self.gradstat_sum, self.gradstat_cnt):
            t.zero_()

    def flat_views(self):
        return [self.pos_opa, self.scale, self.rot, self.sh, self.gradstat_sum]


class ViewRecords:
    """Per-view projected records for V views of N Gaussians ([V,N,…] layout)."""

    def __init__(self, num_views: int, n: int, device="cuda"):
        torch = _torch()
        self.V, self.n = num_views, n
        f = lambda *s: torch.empty(*s, dtype=torch.float32, device=device)
        self.xy_depth = f(num_views, n, 4)
        self.conic_opa = f(num_views, n, 4)
        self.rgb = f(num_views, n, 4)
        self.box = torch.empty(num_views, n, 2, dtype=torch.int32, device=device)
        self.rows = torch.empty(num_views, n, 4, dtype=torch.int32, device=device)   # A50 footprints
        self.tiles = torch.empty(num_views, n, dtype=torch.int32, device=device)

    def view(self, v: int):
        """View v's records, in dass_project's output order."""
        return (self.xy_depth[v], self.conic_opa[v], self.rgb[v], self.box[v], self.rows[v],
                self.tiles[v])


class Raster:
    """Scratch for one view at a time: sorted pairs, ranges, fwd outputs, bwd workspace."""

    def __init__(self, width: int, height: int, n: int, capacity: int, device="cuda",
                 accept_lists: bool = True):
        torch = _torch()
        self.W, self.H, self.n, self.capacity = width, height, n, capacity
        self.num_tiles = ((width + 15) // 16) * ((height + 15) // 16)
        ws = dass.dass_bin_sort_workspace(n, self.num_tiles, capacity)
        self.sort_ws = torch.empty(max(ws, 16), dtype=torch.uint8, device=device)
        self.sorted_ids = torch.empty(max(capacity, 1), dtype=torch.int32, device=device)
        self.ranges = torch.empty(self.num_tiles, 2, dtype=torch.int32, device=device)
        self.num_pairs = torch.zeros(2, dtype=torch.int32, device=device)
        self.img = torch.empty(3, height, width, dtype=torch.float32, device=device)
        self.T = torch.empty(height, width, dtype=torch.float32, device=device)
        self.last = torch.empty(height, width, dtype=torch.int32, device=device)
        bws = dass.dass_render_bwd_workspace(n)
        self.bwd_ws = torch.empty(bws // 4, dtype=torch.float32, device=device)
        self.accept = None
        if accept_lists:
            # forward-recorded acceptance lists consumed by the backward
            ab = dass.dass_render_accept_workspace(self.num_tiles, capacity)
            self.accept = torch.empty(ab // 4, dtype=torch.int32, device=device)

    def sort(self, cam, rec, host_mode=False, sorted_keys=None, num_pairs=None, shared=False):
        """num_pairs: where (K, overflow flag) go (default: this slot's own pair);
        shared: dass_bin_sort_shared (other views' kernels run next to this sort)."""
        xy, co, rgb, box, rows, tt = rec
        return dass.dass_bin_sort(cam, self.n, xy, box, rows, tt, self.sort_ws, self.capacity,
                                  sorted_keys, self.sorted_ids, self.ranges,
                                  self.num_pairs if num_pairs is None else num_pairs,
                                  host_mode=host_mode, shared=shared)

    def render(self, cam, rec, bg=None, tiles=None, ranges=None, sorted_ids=None):
        """ranges/sorted_ids: a view's slices of a batched dass_bin_sort_views (else
        this slot's own sort)."""
        xy, co, rgb, box, rows, tt = rec
        dass.dass_render_fwd(cam, self.ranges if ranges is None else ranges,
                             self.sorted_ids if sorted_ids is None else sorted_ids, xy, co, rgb,
                             box, bg, self.img, self.T, self.last, self.accept, self.capacity,
                             tiles=tiles)

    def forward(self, cam, rec, host_mode=False, bg=None, sorted_keys=None, tiles=None):
        K = self.sort(cam, rec, host_mode=host_mode, sorted_keys=sorted_keys)
        self.render(cam, rec, bg=bg, tiles=tiles)
        return K

    def backward(self, cam, scene: DeviceScene, rec, dL_dimg, grads: Grads, keep=None, bg=None,
                 want=("pos", "scale", "rot", "sh", "stat")):
        xy, co, rgb, box, rows, tiles = rec
        g = lambda name, t: t if name in want else None
        dass.dass_render_bwd(cam, scene.sh_degree, scene.pos_opa, scene.scale, scene.rot,
                             scene.sh, keep, self.ranges, self.sorted_ids, xy, co, rgb, box, bg,
                             self.T, self.last, dL_dimg, self.bwd_ws, g("pos", grads.pos_opa),
                             g("scale", grads.scale), g("rot", grads.rot), g("sh", grads.sh),
                             g("stat", grads.gradstat_sum), g("stat", grads.gradstat_cnt),
                             self.accept, self.capacity)


def project_all(cams, scene: DeviceScene, records: ViewRecords, keep=None):
    dass.dass_project_views(cams, scene.sh_degree, scene.pos_opa, scene.scale, scene.rot,
                            scene.sh, keep, records.xy_depth, records.conic_opa, records.rgb,
                            records.box, records.rows, records.tiles)


def fwd_bwd_views(cams, scene: DeviceScene, records: ViewRecords, raster: Raster, dL_dimgs,
                  grads: Grads, keep=None, bg=None):
    """One fwd+bwd pass over `cams` (all §8(a) steps a2-a9): project all views
    once, then per view bin/sort → composite → backward (+= into grads)."""
    project_all(cams, scene, records, keep)
    for v, cam in enumerate(cams):
        rec = records.view(v)
        raster.forward(cam, rec, bg=bg)
        raster.backward(cam, scene, rec, dL_dimgs[v], grads, keep=keep, bg=bg)


@dataclass
class PassOptions:
    """Scheduling choices of a MultiViewPass (the defaults are the measured best,
    DESIGN.md §7; bench.py exposes them for A/B runs).

    sort_chains: 0 = every view sorts on its own stream; k > 0 = the sorts run one
      after another on k high-priority streams.
    batch_sort: dass_bin_sort_views over sort_batch_chunks chunks of the views
      instead of one dass_bin_sort per view.
    pre_chunks: the multi-view preprocess in chunks, each on a side stream as soon
      as its views are rasterised.
    proj_chunks: with a projection callback, the projection in chunks, each view
      waiting only for its own chunk.
    split_project: with a projection callback, the projection's records part
      (fp64 records + colour, DASS_PROJECT_RECORDS) on a side stream under the
      views' sorts; the sorts wait only for the keys part, the forwards for both.
    split_preprocess: the preprocess's SH-coefficient part on a side stream next to
      its geometry part (DASS_PREPROCESS_SH / _GEOMETRY).
    stream_prio: the first half of the view streams at a higher priority.
    shared_sort_min_views: dass_bin_sort_shared from this many concurrent view streams on
    (dass_bin_sort below)."""
    sort_chains: int = 0
    batch_sort: bool = False
    sort_batch_chunks: int = 4
    pre_chunks: int = 1
    proj_chunks: int = 1
    split_project: bool = True
    split_preprocess: bool = True
    stream_prio: bool = False
    shared_sort_min_views: int = 8


class MultiViewPass:
    """fwd+bwd over a fixed list of cameras with S overlapping streams."""

    def __init__(self, cams, n: int, capacity: int, device="cuda", streams: int = 4,
                 tiles=None, uv_out=None, options: PassOptions | None = None):
        """tiles[v]: None or a (begin, stride, count) tile subset of view v (a
        split view, dist.ViewPlan); uv_out[v]: None or the float2[n] block that
        view's ∇p̄ partials go to (the GPU with the view's tile half 0 counts it)."""
        torch = _torch()
        self.cams = list(cams)
        self.tiles = list(tiles) if tiles is not None else [None] * len(self.cams)
        self.uv_out = list(uv_out) if uv_out is not None else [None] * len(self.cams)
        self.V = len(self.cams)
        self.n = n
        W, H = self.cams[0].width, self.cams[0].height
        for c in self.cams:
            if (c.width, c.height) != (W, H):
                raise ValueError("all cameras of a pass must share the image size")
        self.S = max(1, min(streams, self.V))
        opt = options or PassOptions()
        self.options = opt
        self.slots = [Raster(W, H, n, capacity, device) for _ in range(self.S)]
        # stream_prio: the streams of the first half of the views get the higher
        # priority, so those views finish first and their preprocess chunk overlaps the rest
        self.streams = [torch.cuda.Stream(device=device,
                                          priority=-1 if opt.stream_prio and 2 * k < self.S else 0)
                        for k in range(self.S)]
        # bin_sort chains: with every view's sort on its own stream, the graph runs the
        # 20 latency-bound sorts in lockstep.  sort_chains > 0 runs them one after
        # another on that many high-priority streams instead, so view 0 rasterises
        # after one sort and the later sorts overlap the earlier views' raster kernels
        # (measured: not faster).
        nch = opt.sort_chains
        self.sort_streams = ([torch.cuda.Stream(device=device, priority=-5)
                              for _ in range(min(nch, self.S))] if nch > 0 else None)
        self.pre_stream = torch.cuda.Stream(device=device)
        self.sh_stream = torch.cuda.Stream(device=device) if opt.split_preprocess else None
        # leave the SH part unjoined at the end of run(); the caller joins with join_sh()
        self.defer_sh = False
        self.rec_stream = torch.cuda.Stream(device=device) if opt.split_project else None
        self.pre_chunks = opt.pre_chunks
        self.proj_chunks = opt.proj_chunks
        # optional hook(v, stream), called on view v's stream right before its backward:
        # an end-to-end caller makes the view wait there for its own ∂L/∂C upload
        self.before_bwd = None
        # optional hook(v, raster_slot), called on view v's stream right after its
        # forward (e.g. the error map of error-guided densification)
        self.after_fwd = None
        # optional int64[4V] (diagnostic, bench.py's in-step phase timing): view v's
        # stream writes the GPU timer at 4v (sort start), 4v+1 (forward start),
        # 4v+2 (backward start), 4v+3 (backward end)
        self.stamps = None
        self.g2d = torch.empty(max(self.V, 1), n, 12, dtype=torch.float32, device=device)
        # (K_v, overflow_v) of every view's graph-mode sort, kept per view so a slot
        # reused by a later view does not overwrite an earlier view's overflow flag
        self.num_pairs = torch.zeros(max(self.V, 1), 2, dtype=torch.int32, device=device)
        # batch_sort: dass_bin_sort_views over chunks of the views instead of a
        # dass_bin_sort per view.  In the graph the per-view sort chains run in lockstep,
        # but the batched sort is slower still (its 17-bit pair passes and emission are
        # instruction-bound), so the per-view sorts stay default.
        self.batch_sort = opt.batch_sort and self.V > 0
        if self.batch_sort:
            T = self.slots[0].num_tiles
            # sort chunks: chunk c + 1 sorts on the main stream while chunk c rasterises
            self.sort_chunks = max(1, min(opt.sort_batch_chunks, self.V))
            vmax = -(-self.V // self.sort_chunks)
            ws = dass.dass_bin_sort_views_workspace(vmax, n, capacity)
            self.bs_ws = torch.empty(max(ws, 16), dtype=torch.uint8, device=device)
            self.bs_ids = torch.empty(self.V, max(capacity, 1), dtype=torch.int32, device=device)
            self.bs_ranges = torch.empty(self.V, T, 2, dtype=torch.int32, device=device)
            self.bs_pairs = torch.zeros(self.V, 2, dtype=torch.int32, device=device)

    def enable_loss(self, lam: float = 0.2):
        """Allocate per-slot scratch so run(gts=...) computes dL/dC itself with the
        fused fidelity loss of Eq. 3 (dass_fidelity_loss) from ground-truth views."""
        torch = _torch()
        dev = self.g2d.device
        W, H = self.cams[0].width, self.cams[0].height
        self.lam = lam
        nb = dass.dass_fidelity_loss_workspace(W, H)
        self.loss_ws = [torch.empty(nb // 4 + 64, dtype=torch.float32, device=dev) for _ in range(self.S)]
        self.loss_dL = [torch.empty(3, H, W, dtype=torch.float32, device=dev) for _ in range(self.S)]
        self.losses = torch.zeros(self.V, 3, dtype=torch.float32, device=dev)

    def run(self, scene: DeviceScene, records: ViewRecords, dL_dimgs, grads, keep=None, bg=None,
            gts=None, project=None):
        """dL_dimgs: fixed per-view ∂L/∂C, or None with gts (per-view ground truth,
        requires enable_loss): then ∂L/∂C comes from the fidelity loss.
        project(v0, v1, part): optional; issues the projection of views [v0, v1) on
        the current stream (part: dass.DASS_PROJECT_KEYS / _RECORDS / _ALL).  The
        pass then projects in options.proj_chunks chunks and each view waits only
        for its own chunk; with options.split_project the records part of each chunk
        runs on a side stream while the views sort."""
        torch = _torch()
        main = torch.cuda.current_stream()
        V = self.V
        if self.batch_sort:   # project all views, then sort them in chunks
            if project is not None:
                project(0, V)
            pc = self.sort_chunks
        else:
            pc = max(1, min(self.proj_chunks, V)) if project is not None else 1
        pbounds = [round(c * V / pc) for c in range(pc + 1)]
        ready = []   # per chunk: the event the chunk's views wait on
        rec_ready = []   # per chunk (split projection): the records part is done
        split = self.rec_stream is not None and project is not None and not self.batch_sort
        for c in range(pc):
            a, b = pbounds[c], pbounds[c + 1]
            if self.batch_sort:
                dass.dass_bin_sort_views(self.cams[a:b], self.n, records.xy_depth[a:b],
                                         records.box[a:b], records.rows[a:b], records.tiles[a:b],
                                         self.bs_ws,
                                         self.slots[0].capacity, self.bs_ids[a:b],
                                         self.bs_ranges[a:b], self.bs_pairs[a:b])
            elif project is not None:
                project(a, b, dass.DASS_PROJECT_KEYS if split else dass.DASS_PROJECT_ALL)
            e = torch.cuda.Event()
            e.record(main)
            ready.append(e)
            if split:
                self.rec_stream.wait_event(e)
                with torch.cuda.stream(self.rec_stream):
                    project(a, b, dass.DASS_PROJECT_RECORDS)
                r = torch.cuda.Event()
                r.record(self.rec_stream)
                rec_ready.append(r)
        chunk_of = [max(c for c in range(pc) if pbounds[c] <= v) for v in range(V)]
        # preprocess in chunks: chunk c's views are chained to parameter gradients on a side
        # stream as soon as they are rasterised (HBM-bound work under the ALU-bound raster
        # kernels of later views); only the last chunk runs after the final raster kernel.
        # Chunks run in order on ONE stream: each += into the same gradient buffers.
        # (measured with one stream per view: 2 / 4 chunks 12.20 / 12.34 ms against 12.12 for
        # one — the views' backward kernels end together, so a chunk has nothing to hide under)
        nchunk = max(1, min(self.pre_chunks, V))
        bounds = [round(c * V / nchunk) for c in range(nchunk + 1)]
        ends = {bounds[c + 1] - 1: c for c in range(nchunk - 1)}
        done = [None] * V
        vr, vi, dLv = {}, {}, {}

        def slot(v):
            k = v % self.S
            return k, self.slots[k], self.streams[k]

        def stamp(v, i, q):
            if self.stamps is not None:
                dass.dass_timestamp(self.stamps, 4 * v + i, q)

        # many views sorting at once on their own streams: the shared-GPU sort variant (its
        # 74-block pair passes need the other views to fill the GPU: with the 2-3 views of an
        # 8-GPU rank it is slower, 1.68 -> 1.77 ms per step)
        shared = self.S >= self.options.shared_sort_min_views

        def part_sort(v):
            k, ras, st = slot(v)
            cam, rec = self.cams[v], records.view(v)
            st.wait_event(ready[chunk_of[v]])
            if self.batch_sort:
                vr[v], vi[v] = self.bs_ranges[v], self.bs_ids[v]
            else:
                vr[v], vi[v] = ras.ranges, ras.sorted_ids
            if self.sort_streams is not None and not self.batch_sort:
                ss = self.sort_streams[v % len(self.sort_streams)]
                ss.wait_stream(st)    # projected, and the slot's previous view is done
                with torch.cuda.stream(ss):
                    ras.sort(cam, rec, num_pairs=self.num_pairs[v], shared=shared)
                st.wait_stream(ss)
            with torch.cuda.stream(st):
                stamp(v, 0, st)
                if self.sort_streams is None and not self.batch_sort:
                    ras.sort(cam, rec, num_pairs=self.num_pairs[v], shared=shared)

        def part_fwd(v):
            k, ras, st = slot(v)
            cam, rec = self.cams[v], records.view(v)
            with torch.cuda.stream(st):
                if split:
                    st.wait_event(rec_ready[chunk_of[v]])
                stamp(v, 1, st)
                ras.render(cam, rec, bg=bg, tiles=self.tiles[v], ranges=vr[v], sorted_ids=vi[v])
                if self.after_fwd is not None:
                    self.after_fwd(v, ras)
                if gts is not None:
                    dLv[v] = self.loss_dL[k]
                    dass.dass_fidelity_loss(ras.img, gts[v], self.lam, self.loss_ws[k],
                                            self.losses[v], dLv[v])
                else:
                    dLv[v] = dL_dimgs[v]

        def part_bwd(v):
            k, ras, st = slot(v)
            cam = self.cams[v]
            xy, co, rgb, box, rows, tiles = records.view(v)
            with torch.cuda.stream(st):
                if self.before_bwd is not None:
                    self.before_bwd(v, st)
                stamp(v, 2, st)
                dass.dass_render_bwd_raster(cam, self.n, vr[v], vi[v], xy, co, rgb,
                                            box, bg, ras.T, ras.last, dLv[v], self.g2d[v],
                                            ras.accept, ras.capacity, tiles=self.tiles[v])
                stamp(v, 3, st)
                done[v] = torch.cuda.Event()
                done[v].record(st)
            if v in ends:
                c = ends[v]
                self.pre_stream.wait_stream(main)
                for u in range(bounds[c], bounds[c + 1]):
                    self.pre_stream.wait_event(done[u])
                with torch.cuda.stream(self.pre_stream):
                    self._preprocess(scene, records, grads, keep, bounds[c], bounds[c + 1])

        for v in range(V):
            part_sort(v)
            part_fwd(v)
            part_bwd(v)
        for s in self.streams:
            main.wait_stream(s)
        for s in self.sort_streams or []:
            main.wait_stream(s)
        if split:
            main.wait_stream(self.rec_stream)
        if nchunk > 1:
            main.wait_stream(self.pre_stream)
        self._preprocess(scene, records, grads, keep, bounds[nchunk - 1], V)

    def pair_counts(self):
        """K of every view's last sort (synchronises)."""
        np_ = (self.bs_pairs if self.batch_sort else self.num_pairs).cpu().numpy().view(np.uint32)
        return [int(k) for k in np_[:self.V, 0]]

    def overflowed_views(self):
        """Views whose last sort exceeded the pair capacity (synchronises).  Such a
        view's tile ranges are all [0, 0): it rendered as background and added no
        gradient, so a caller must not use that step's results."""
        np_ = (self.bs_pairs if self.batch_sort else self.num_pairs).cpu().numpy().view(np.uint32)
        return [v for v in range(self.V) if np_[v, 1]]

    def _preprocess(self, scene, records, grads, keep, v0, v1):
        torch = _torch()

        def call(part):
            dass.dass_render_bwd_preprocess_views(
                self.cams[v0:v1], scene.sh_degree, scene.pos_opa, scene.scale, scene.rot, scene.sh,
                keep, records.conic_opa[v0:v1], records.rgb[v0:v1], records.box[v0:v1],
                self.g2d[v0:v1], grads.pos_opa, grads.scale, grads.rot, grads.sh,
                grads.gradstat_sum, grads.gradstat_cnt,
                uv_out=None if all(u is None for u in self.uv_out[v0:v1]) else self.uv_out[v0:v1],
                uv_count=[t is not None and t[0] == 0 for t in self.tiles[v0:v1]], part=part)
        if self.sh_stream is None:
            call(dass.DASS_PREPROCESS_ALL)
            return
        # the SH-coefficient part on a side stream next to the geometry part (disjoint
        # outputs, both latency-bound)
        cur = torch.cuda.current_stream()
        self.sh_stream.wait_stream(cur)
        call(dass.DASS_PREPROCESS_GEOMETRY)
        with torch.cuda.stream(self.sh_stream):
            call(dass.DASS_PREPROCESS_SH)
        if not self.defer_sh:
            cur.wait_stream(self.sh_stream)

    def join_sh(self):
        """Join the SH-coefficient part deferred by defer_sh (ShiftStep: after the
        shift stage's collective, which does not carry SH gradients)."""
        if self.sh_stream is not None:
            _torch().cuda.current_stream().wait_stream(self.sh_stream)


class DeformFields:
    """The dual deformation fields 𝓗_dyn / 𝓗_st (§3.3, f2) on the device: tables,
    MLPs, their gradients and the dynamic/static partition of the Gaussians."""

    def __init__(self, fields, n: int, device="cuda"):
        torch = _torch()
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
        self.cfg = list(fields)                      # (𝓗_dyn, 𝓗_st) synth.HashField-like
        self.table = [t(f.table) for f in self.cfg]
        self.mlp = [t(f.mlp) for f in self.cfg]
        self.g_table = [torch.zeros_like(x) for x in self.table]
        self.g_mlp = [torch.zeros_like(x) for x in self.mlp]
        self.n = n
        self.idx = [torch.empty(max(n, 1), dtype=torch.int32, device=device) for _ in range(2)]
        self.counts = torch.zeros(2, dtype=torch.int32, device=device)
        nb = dass.dass_partition_workspace(n)
        self.part_ws = torch.empty(nb // 4 + 1, dtype=torch.int32, device=device)

    def partition(self, dyn_mask):
        dass.dass_partition(dyn_mask, self.idx[0], self.idx[1], self.counts, self.part_ws)

    def zero_grad(self):
        for x in self.g_table + self.g_mlp:
            x.zero_()

    def forward(self, pos_opa, mu, sigma):
        for k in range(2):
            dass.dass_deform_fwd(self.cfg[k], self.table[k], self.mlp[k], pos_opa, mu, sigma,
                                 idx=self.idx[k], count=self.counts[k:k + 1], n=self.n)

    def backward(self, pos_opa, g_mu, g_sigma):
        for k in range(2):
            dass.dass_deform_bwd(self.cfg[k], self.table[k], self.mlp[k], pos_opa, g_mu, g_sigma,
                                 self.g_table[k], self.g_mlp[k], idx=self.idx[k],
                                 count=self.counts[k:k + 1], n=self.n)

    def grad_tensors(self):
        return self.g_table + self.g_mlp
