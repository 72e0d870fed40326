"""One shift-stage iteration over a rank's views (plumbing around libdass).

The step `bench.py` times and `tests/test_gpu_step.py` checks against the
oracle:

    dass_apply_shift → dass_project_views → per view (dass_bin_sort →
    dass_render_fwd → dass_render_bwd_raster) on overlapping streams →
    dass_render_bwd_preprocess_views → dass_apply_shift_bwd

with the per-Gaussian gradients in one flat buffer (dist.FlatGrads, the
all-reduce payload).  Every arithmetic step runs in the CUDA kernels; this
module only owns buffers and call order, and is capturable as one CUDA graph
(no host synchronisation inside).
"""
from __future__ import annotations

from . import dass
from .dist import FlatGrads
from .pipeline import DeviceScene, MultiViewPass, PassOptions, ViewRecords


class StepBufs:
    """A step's inputs (𝒢_{t−1}, the shift offsets μ/σ, the views' ∂L/∂C) and
    its outputs (the flat gradients).  `shifted` is 𝒢_t after the shift: its
    position/rotation are the step's scratch, its scale/SH are the inputs'."""

    def __init__(self, base: DeviceScene, mu, sigma, dLs, grads: FlatGrads, shifted_pos, shifted_rot):
        self.base, self.mu, self.sigma, self.dLs, self.grads = base, mu, sigma, dLs, grads
        self.shifted = DeviceScene(shifted_pos, base.scale, shifted_rot, base.sh, base.sh_degree,
                                   base.dynamic)


class ShiftStep:
    """fwd+bwd of one shift iteration over `cams` (this rank's views).

    tiles[k] / split[k]: the dist.ViewPlan entries of view k (None / −1 for a
    whole view); num_split sizes the uv blocks of the flat gradient buffer."""

    def __init__(self, cams, n: int, sh_degree: int, capacity: int, device, streams: int = 20,
                 tiles=None, split=None, num_split: int = 0, validate: bool = False,
                 shift: bool = True, options: PassOptions | None = None):
        """validate: the step ends with dass_scan_nonfinite over its gradients (graph
        mode); check_numerics() then raises DASS_ERR_NUMERICAL on NaN / Inf.
        shift=False: a plain fwd+bwd of the given Gaussians (BASELINE configs C1/C2),
        no dass_apply_shift / _bwd."""
        import torch
        self.cams = list(cams)
        self.n, self.deg, self.device = n, sh_degree, device
        self.tiles = list(tiles) if tiles is not None else [None] * len(self.cams)
        self.split = list(split) if split is not None else [-1] * len(self.cams)
        self.num_split = num_split
        self.records = ViewRecords(max(len(self.cams), 1), n, device)
        self.mvp = MultiViewPass(self.cams, n, capacity, device, streams=streams,
                                 tiles=self.tiles, options=options) if self.cams else None
        self.shifted_pos = torch.empty(n, 4, dtype=torch.float32, device=device)
        self.shifted_rot = torch.empty(n, 4, dtype=torch.float32, device=device)
        self._errmap_pos = None
        self.validate = validate
        self.shift = shift
        self.bad = torch.zeros(1, dtype=torch.int32, device=device)

    def enable_error_map(self, gts, gamma_err: float, n_base: int, s_err):
        """Every view's error map against its ground truth right after its forward
        (dass_error_map: E, D and S_err |= Alg. 1 over the n_base base Gaussians;
        P:164-165) — the C4 step of BASELINE.json.  s_err (uint8[n]) is
        OR-accumulated; the caller zeroes it once per timestep."""
        import torch
        self.gts, self.gamma_err, self.n_base, self.s_err = gts, gamma_err, n_base, s_err
        W, H = self.cams[0].width, self.cams[0].height
        self.err = [torch.empty(H, W, device=self.device) for _ in range(self.mvp.S)]
        self.dmask = [torch.zeros((H * W + 31) // 32, dtype=torch.int32, device=self.device)
                      for _ in range(self.mvp.S)]
        self._errmap_pos = None

        def hook(v, ras):
            k = v % self.mvp.S
            dass.dass_error_map(self.cams[v], ras.img, self.gts[v], self.gamma_err, self.err[k],
                                self.dmask[k], self.n_base, self._errmap_pos, self.s_err)
        self.mvp.after_fwd = hook

    def buffers(self, base: DeviceScene, mu, sigma, dLs, grads: FlatGrads | None = None) -> StepBufs:
        from .synth import sh_planes
        if grads is None:
            grads = FlatGrads.allocate(self.n, sh_planes(self.deg), self.device,
                                       num_split=self.num_split)
        return StepBufs(base, mu, sigma, dLs, grads, self.shifted_pos, self.shifted_rot)

    def run(self, S: StepBufs, wait_inputs=None, collective=None, collective_after_sh=True):
        """Everything on this GPU (capturable: no host sync).
        wait_inputs(): an end-to-end caller's wait for this step's parameter upload.
        collective(): the caller's cross-GPU exchange of this step, issued on the current
        stream after the shift backward; with collective_after_sh=False (a payload without
        SH gradients, the shift stage's) it runs while the preprocess's SH-coefficient part
        is still going on its side stream."""
        g = S.grads
        g.zero_()
        if wait_inputs is not None:
            wait_inputs()
        if self.shift:
            dass.dass_apply_shift(S.base.pos_opa, S.base.rot, S.mu, S.sigma, S.base.dynamic,
                                  S.shifted.pos_opa, S.shifted.rot)
        rec, cams, sh = self.records, self.cams, (S.shifted if self.shift else S.base)

        def project(v0, v1, part=dass.DASS_PROJECT_ALL):
            dass.dass_project_views_part(part, cams[v0:v1], self.deg, sh.pos_opa, sh.scale,
                                         sh.rot, sh.sh, None, rec.xy_depth[v0:v1],
                                         rec.conic_opa[v0:v1], rec.rgb[v0:v1], rec.box[v0:v1],
                                         rec.rows[v0:v1], rec.tiles[v0:v1])
        early = collective is not None and not collective_after_sh
        if self.mvp is not None:
            self._errmap_pos = sh.pos_opa     # the error map projects 𝒢_t (Alg. 1)
            self.mvp.uv_out = [None if s < 0 else g.uv[s] for s in self.split]
            self.mvp.defer_sh = early
            self.mvp.run(sh, rec, S.dLs, g, project=project)
            self.mvp.defer_sh = False
        if self.shift:
            dass.dass_apply_shift_bwd(S.base.rot, S.sigma, S.base.dynamic, g.pos_opa, g.rot,
                                      g.g_mu, g.g_sigma)
        if early:
            collective()
        if self.mvp is not None:
            self.mvp.join_sh()
        if collective is not None and not early:
            collective()
        if self.validate:
            self.bad.zero_()
            dass.dass_scan_nonfinite(g.flat, self.bad)

    def capture(self, S: StepBufs, wait_inputs=None):
        """The step as one CUDA graph (replay() runs it)."""
        import torch
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.run(S, wait_inputs=wait_inputs)
        return graph

    def check_numerics(self):
        """Raise DASS_ERR_NUMERICAL if the last validated step's gradients held NaN /
        Inf (synchronises)."""
        if self.validate:
            bad = int(self.bad.item())
            if bad:
                raise dass.DassError(dass.DASS_ERR_NUMERICAL, "ShiftStep",
                                     f"{bad} non-finite gradient values")

    def check_overflow(self):
        """Raise if any view's pair count exceeded the capacity in the last step
        (graph-mode sorts flag it on the device instead of failing; an
        overflowed view would render as background).  Synchronises."""
        if self.mvp is not None:
            bad = self.mvp.overflowed_views()
            if bad:
                raise dass.DassError(dass.DASS_ERR_CAPACITY, "ShiftStep",
                                     f"pair capacity {self.mvp.slots[0].capacity} exceeded in "
                                     f"views {bad} (K = {self.mvp.pair_counts()})")
