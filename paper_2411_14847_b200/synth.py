"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no projection, no SH, no
compositing): it only draws random numbers and builds camera matrices, which
are *inputs* of the method (Alg. 1 takes the full projection matrix T as an
input).  Both sides — `oracle/` and the CUDA path — consume exactly the
same arrays.  All randomness is NumPy's counter-based Philox with the seeds
listed in DESIGN.md §Input recipe (SURVEY.md §8(d) "Synthetic inputs").

Shapes follow the paper's workloads: N3DV is 1352×1014 with 18-21 forward-
facing views; Meet Room is 1280×720 with 13 cameras; Fig. 3
 says most per-timestep deformations are < 0.01 and the dynamic
group carries the large ones.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

CAMERA_DTYPE = np.dtype([
    ("width", np.int32), ("height", np.int32),
    ("fx", np.float32), ("fy", np.float32), ("cx", np.float32), ("cy", np.float32),
    ("viewmat", np.float32, (12,)),
    ("near_plane", np.float32),
    ("full_proj", np.float32, (16,)),
])  # mirrors `dass_camera` in include/dass.h (packed, 4-byte fields)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def sh_coeff_count(degree: int) -> int:
    return 3 * (degree + 1) ** 2


def sh_planes(degree: int) -> int:
    return (sh_coeff_count(degree) + 3) // 4


@dataclass
class Camera:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    viewmat: np.ndarray          # float32 [3,4] world->camera [R|t]
    near: float = 0.2
    far: float = 100.0

    @property
    def full_proj(self) -> np.ndarray:
        """Alg. 1's T in the row-vector convention [p,1]·T.

        Built so that Alg. 1's pixel map 0.5((x_norm+1)W-1) lands on the
        pinhole pixel fx·x/z + cx with integer pixel centres (A19):
        clip = K4 · V4 · [p,1]^T, T = (K4 V4)^T."""
        W, H = self.width, self.height
        n, f = self.near, self.far
        K4 = np.zeros((4, 4), np.float64)
        K4[0, 0] = 2.0 * self.fx / W
        K4[0, 2] = (2.0 * self.cx + 1.0) / W - 1.0
        K4[1, 1] = 2.0 * self.fy / H
        K4[1, 2] = (2.0 * self.cy + 1.0) / H - 1.0
        K4[2, 2] = f / (f - n)
        K4[2, 3] = -f * n / (f - n)
        K4[3, 2] = 1.0
        V4 = np.eye(4)
        V4[:3, :] = self.viewmat.astype(np.float64)
        return (K4 @ V4).T.astype(np.float32)

    def to_struct(self) -> np.ndarray:
        s = np.zeros((), CAMERA_DTYPE)
        s["width"], s["height"] = self.width, self.height
        s["fx"], s["fy"], s["cx"], s["cy"] = self.fx, self.fy, self.cx, self.cy
        s["viewmat"] = self.viewmat.astype(np.float32).reshape(12)
        s["near_plane"] = self.near
        s["full_proj"] = self.full_proj.reshape(16)
        return s

    @property
    def tiles_x(self) -> int:
        return (self.width + 15) // 16

    @property
    def tiles_y(self) -> int:
        return (self.height + 15) // 16

    @property
    def num_tiles(self) -> int:
        return self.tiles_x * self.tiles_y


def cameras_to_structs(cams) -> np.ndarray:
    out = np.zeros(len(cams), CAMERA_DTYPE)
    for i, c in enumerate(cams):
        out[i] = c.to_struct()
    return out


def _rot_yaw_pitch(yaw: float, pitch: float) -> np.ndarray:
    """Camera-to-world rotation for a camera looking along +z (x right, y down)
    turned by yaw (about y) then pitch (about x)."""
    cy_, sy_ = math.cos(yaw), math.sin(yaw)
    cp, sp = math.cos(pitch), math.sin(pitch)
    Ry = np.array([[cy_, 0, sy_], [0, 1, 0], [-sy_, 0, cy_]])
    Rx = np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]])
    return Ry @ Rx


def _look_at(eye: np.ndarray, target: np.ndarray) -> np.ndarray:
    """Camera-to-world rotation whose +z axis points from eye to target, +y down."""
    z = target - eye
    z = z / np.linalg.norm(z)
    up = np.array([0.0, -1.0, 0.0])
    x = np.cross(up, z)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    return np.stack([x, y, z], axis=1)


def _viewmat(R_c2w: np.ndarray, centre: np.ndarray) -> np.ndarray:
    R = R_c2w.T
    t = -R @ centre
    return np.concatenate([R, t[:, None]], axis=1).astype(np.float32)


def n3dv_rig(seed: int = 3, width: int = 1352, height: int = 1014,
             num_views: int = 20) -> list[Camera]:
    """20 forward-facing cameras on a 5×4 grid in z=0, spacing 0.25, ±3° seeded
    yaw/pitch jitter; 60° horizontal FOV (fx = fy = 1170.9); SURVEY §8(d) C3."""
    g = rng(seed)
    fx = 0.5 * width / math.tan(math.radians(30.0))
    cams = []
    for k in range(num_views):
        gx, gy = k % 5, (k // 5) % 4
        centre = np.array([(gx - 2) * 0.25, (gy - 1.5) * 0.25, 0.0])
        yaw, pitch = np.radians(g.uniform(-3.0, 3.0, size=2))
        cams.append(Camera(width, height, fx, fx, (width - 1) / 2.0,
                           (height - 1) / 2.0, _viewmat(_rot_yaw_pitch(yaw, pitch), centre)))
    return cams


def meetroom_rig(seed: int = 4, width: int = 1280, height: int = 720,
                 num_views: int = 13) -> list[Camera]:
    """13 cameras on a 100° horizontal arc of radius 3 aimed at (0,0,3); 70° FOV."""
    fx = 0.5 * width / math.tan(math.radians(35.0))
    focus = np.array([0.0, 0.0, 3.0])
    cams = []
    for th in np.radians(np.linspace(-50.0, 50.0, num_views)):
        eye = focus + 3.0 * np.array([math.sin(th), 0.0, -math.cos(th)])
        cams.append(Camera(width, height, fx, fx, (width - 1) / 2.0,
                           (height - 1) / 2.0, _viewmat(_look_at(eye, focus), eye)))
    return cams


def tiny_camera(width: int = 64, height: int = 64, f: float | None = None) -> Camera:
    """C1 camera: identity extrinsics, fx = fy = W, centred principal point."""
    f = float(width) if f is None else f
    return Camera(width, height, f, f, (width - 1) / 2.0, (height - 1) / 2.0,
                  np.concatenate([np.eye(3), np.zeros((3, 1))], 1).astype(np.float32))


@dataclass
class Scene:
    """Field-SoA Gaussian parameters exactly as the C-ABI consumes them."""
    pos_opa: np.ndarray   # float32 [N,4]: x,y,z, opacity in (0,1)
    scale: np.ndarray     # float32 [N,4]: sx,sy,sz>0, 0
    rot: np.ndarray       # float32 [N,4]: w,x,y,z (not normalised)
    sh: np.ndarray        # float32 [K4,N,4] coefficient planes
    sh_degree: int
    dynamic: np.ndarray = field(default=None)  # uint8 [N] dynamics mask (D05)

    @property
    def n(self) -> int:
        return self.pos_opa.shape[0]

    def sh_coeffs(self) -> np.ndarray:
        """[N, (d+1)^2, 3] view of the SH coefficients (plane layout undone)."""
        nc = sh_coeff_count(self.sh_degree)
        flat = np.transpose(self.sh, (1, 0, 2)).reshape(self.n, -1)[:, :nc]
        return flat.reshape(self.n, -1, 3)


def pack_sh(coeffs: np.ndarray) -> np.ndarray:
    """[N, (d+1)^2, 3] -> float32 [K4, N, 4] planes (zero padding)."""
    n = coeffs.shape[0]
    flat = coeffs.reshape(n, -1).astype(np.float32)
    k4 = (flat.shape[1] + 3) // 4
    pad = np.zeros((n, 4 * k4), np.float32)
    pad[:, :flat.shape[1]] = flat
    return np.ascontiguousarray(pad.reshape(n, k4, 4).transpose(1, 0, 2))


def _random_quats(g, n):
    q = g.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _sh_coeffs(g, n, degree):
    c = np.zeros((n, (degree + 1) ** 2, 3))
    c[:, 0, :] = g.uniform(-1.6, 1.6, size=(n, 3))   # base colour ≈ U(0.05,0.95)
    k = 1
    for l in range(1, degree + 1):
        m = 2 * l + 1
        c[:, k:k + m, :] = g.normal(0.0, 0.15 / (l + 1), size=(n, m, 3))
        k += m
    return c


def _assemble(g, xyz, sigma_px_scale_depth, degree, fx, dynamic=None,
              sigma_median=2.5, sigma_log_sd=0.7):
    n = xyz.shape[0]
    sig_px = np.clip(np.exp(g.normal(math.log(sigma_median), sigma_log_sd, size=(n, 3))),
                     0.3, 80.0)
    s = sig_px * sigma_px_scale_depth[:, None] / fx
    o = 1.0 / (1.0 + np.exp(-g.normal(0.0, 2.0, size=n)))
    pos_opa = np.concatenate([xyz, o[:, None]], 1).astype(np.float32)
    scale = np.concatenate([s, np.zeros((n, 1))], 1).astype(np.float32)
    rot = _random_quats(g, n).astype(np.float32)
    sh = pack_sh(_sh_coeffs(g, n, degree))
    return Scene(pos_opa, scale, rot, sh, degree,
                 np.zeros(n, np.uint8) if dynamic is None else dynamic.astype(np.uint8))


def random_scene(n: int, cam: Camera, seed: int = 1, degree: int = 0,
                 zmin: float = 2.0, zmax: float = 6.0, sigma_median: float = 2.5) -> Scene:
    """C1-style scene: z ~ U(zmin, zmax) in front of `cam` (identity pose assumed
    for the frustum bounds), x,y uniform inside the frustum."""
    g = rng(seed)
    z = g.uniform(zmin, zmax, size=n)
    hx = 0.5 * cam.width / cam.fx
    hy = 0.5 * cam.height / cam.fy
    x = g.uniform(-hx, hx, size=n) * z
    y = g.uniform(-hy, hy, size=n) * z
    xyz = np.stack([x, y, z], 1)
    # bring into world coordinates through the inverse view (identity for C1)
    R, t = cam.viewmat[:, :3].astype(np.float64), cam.viewmat[:, 3].astype(np.float64)
    xyz = (xyz - t) @ R
    return _assemble(g, xyz, z, degree, cam.fx, sigma_median=sigma_median)


def n3dv_scene(n: int = 300_000, seed: int = 3, degree: int = 3, fx: float = 1170.9,
               dynamic_frac: float = 0.3, sigma_median: float = 2.5) -> Scene:
    """N3DV-shaped scene: 70% static slab z∈[4,9], |x|≤0.65z,
    |y|≤0.5z; 30% dynamic foreground in 6 clusters at z∈[1.5,3.5]; index order
    randomly permuted so mask bits are scattered."""
    g = rng(seed)
    n_dyn = int(round(n * dynamic_frac))
    n_st = n - n_dyn
    z = g.uniform(4.0, 9.0, size=n_st)
    st = np.stack([g.uniform(-0.65, 0.65, n_st) * z, g.uniform(-0.5, 0.5, n_st) * z, z], 1)
    cz = g.uniform(1.5, 3.5, size=6)
    centres = np.stack([g.uniform(-0.3, 0.3, 6) * cz, g.uniform(-0.2, 0.2, 6) * cz, cz], 1)
    lab = g.integers(0, 6, size=n_dyn)
    dy = centres[lab] + g.normal(size=(n_dyn, 3)) * np.array([0.15, 0.25, 0.1])
    xyz = np.concatenate([st, dy], 0)
    dyn = np.concatenate([np.zeros(n_st, np.uint8), np.ones(n_dyn, np.uint8)])
    perm = g.permutation(n)
    xyz, dyn = xyz[perm], dyn[perm]
    return _assemble(g, xyz, np.maximum(xyz[:, 2], 0.5), degree, fx, dynamic=dyn,
                     sigma_median=sigma_median)


def shift_offsets(scene: Scene, seed: int = 33):
    """Per-Gaussian deformation outputs (μ, σ) as the hash fields would emit
    them (Fig. 3): dynamic μ ~ N(0, 0.02²), σ = (1,0,0,0)+N(0,0.02²);
    static ones < 0.01."""
    g = rng(seed)
    n = scene.n
    dyn = scene.dynamic.astype(bool)
    sd = np.where(dyn, 0.02, 0.002)[:, None]
    mu = np.zeros((n, 4), np.float32)
    mu[:, :3] = g.normal(size=(n, 3)) * sd
    sigma = (np.array([1.0, 0, 0, 0]) + g.normal(size=(n, 4)) * sd).astype(np.float32)
    return mu, sigma


def grad_image(cam: Camera, seed: int, scale: float = 1.0) -> np.ndarray:
    """Fixed dL/dC for one view: U(-1,1)·scale, float32 [3,H,W]."""
    g = rng(seed)
    return (g.uniform(-1.0, 1.0, size=(3, cam.height, cam.width)) * scale).astype(np.float32)


def random_image(cam: Camera, seed: int) -> np.ndarray:
    g = rng(seed)
    return g.uniform(0.0, 1.0, size=(3, cam.height, cam.width)).astype(np.float32)


def c1():
    cam = tiny_camera(64, 64)
    return cam, random_scene(1000, cam, seed=1, degree=0)


def c2(n: int = 300_000):
    cams = n3dv_rig(seed=3)
    return cams[7], n3dv_scene(n=n, seed=2, degree=3, fx=cams[7].fx)


def c3(n: int = 300_000, num_views: int = 20):
    cams = n3dv_rig(seed=3, num_views=num_views)
    return cams, n3dv_scene(n=n, seed=3, degree=3, fx=cams[0].fx)


def c4(n: int = 200_000, num_views: int = 13):
    """Meet-Room-shaped timestep (BASELINE configs[3]): 13 cameras on a 100° arc
    around (0,0,3), 1280×720; the N3DV-shaped generator places the background
    4-9 units and the clusters 1.5-3.5 units in front of the central camera."""
    cams = meetroom_rig(seed=4, num_views=num_views)
    return cams, n3dv_scene(n=n, seed=4, degree=3, fx=cams[0].fx)


def c4_ground_truth(scene: Scene, seed: int = 44, moved_frac: float = 0.05,
                    n_emerging: int = 10_000, fx: float = 914.3) -> Scene:
    """SURVEY §8(d) C4's ground-truth scene: the C4 Gaussians with a random 5%
    translated by N(0, 0.05²) per axis, plus an emerging 10k-Gaussian cluster
    (N((0.3, −0.1, 2.4), 0.12²)) that the base scene lacks — what error-guided
    densification has to find."""
    g = rng(seed)
    pos = scene.pos_opa.copy()
    sel = g.uniform(size=scene.n) < moved_frac
    pos[sel, :3] += (g.normal(size=(int(sel.sum()), 3)) * 0.05).astype(np.float32)
    xyz = np.array([0.3, -0.1, 2.4]) + g.normal(size=(n_emerging, 3)) * 0.12
    em = _assemble(g, xyz, xyz[:, 2], scene.sh_degree, fx)
    cat = lambda a, b: np.concatenate([a, b], 0)
    return Scene(cat(pos, em.pos_opa), cat(scene.scale, em.scale), cat(scene.rot, em.rot),
                 np.concatenate([scene.sh, em.sh], 1), scene.sh_degree,
                 cat(scene.dynamic, np.ones(n_emerging, np.uint8)))


def gradstat_lognormal(n: int, seed: int = 46):
    """C4's synthetic ∇p̄ statistic: LogNormal(ln 1e-4, 1), one view."""
    g = rng(seed)
    return np.exp(g.normal(math.log(1e-4), 1.0, size=n)).astype(np.float32), np.ones(n, np.int32)


def c5(n: int = 1_000_000):
    cams = n3dv_rig(seed=3)
    return cams, n3dv_scene(n=n, seed=5, degree=3, fx=cams[0].fx,
                            sigma_median=2.5 * math.sqrt(0.3))


# ---- f2: hash-grid deformation fields (configuration + seeded parameters) ----
# The paper fixes only T_Hash and F_Hash per group and dataset; the
# rest is the I-NGP-style configuration of reading A41: L = 8 levels,
# geometric resolutions from 16 to 256 (listed, not computed), MLP 64-64.
HASHGRID_DTYPE = np.dtype([
    ("L", np.int32), ("log2T", np.int32), ("F", np.int32), ("pad", np.int32),
    ("res", np.int32, (16,)), ("lo", np.float32, (3,)), ("hi", np.float32, (3,)),
])
HASH_LEVEL_RES = (16, 23, 35, 52, 78, 115, 172, 256)   # ⌊16·16^(l/7)⌋, l = 0..7
HASH_PROFILES = {                                          # (log2 T, F): dyn, static
    "n3dv": ((16, 4), (14, 2)),
    "meetroom": ((15, 4), (13, 2)),
}
MLP_HIDDEN = 64


@dataclass
class HashField:
    L: int
    log2T: int
    F: int
    res: tuple
    lo: np.ndarray
    hi: np.ndarray
    table: np.ndarray      # float32 [L][T][F]
    mlp: np.ndarray        # float32 flat: W1[64][L·F] b1[64] W2[64][64] b2[64] W3[7][64] b3[7]

    @property
    def inputs(self) -> int:
        return self.L * self.F

    def to_struct(self) -> np.ndarray:
        s = np.zeros((), HASHGRID_DTYPE)
        s["L"], s["log2T"], s["F"] = self.L, self.log2T, self.F
        s["res"][:self.L] = self.res
        s["lo"], s["hi"] = self.lo, self.hi
        return s


def mlp_param_count(inputs: int, hidden: int = MLP_HIDDEN) -> int:
    return hidden * inputs + hidden + hidden * hidden + hidden + 7 * hidden + 7


def scene_aabb(pos: np.ndarray, pad: float = 0.1):
    """Input box of the fields: the positions' bounds padded by 10% of the span."""
    lo, hi = pos[:, :3].min(0), pos[:, :3].max(0)
    span = np.maximum(hi - lo, 1e-6)
    return (lo - pad * span).astype(np.float32), (hi + pad * span).astype(np.float32)


def hash_field(log2T: int, F: int, aabb, seed: int, levels: int = 8, trained: bool = True,
               res=HASH_LEVEL_RES, table_scale: float = 0.5, head_scale: float = 0.02) -> HashField:
    """Seeded field parameters.  trained=False is the initial state (table
    U(±1e-4), zero head → identity deformation); trained=True draws a table
    U(±table_scale) and a head of scale head_scale (μ of order 1e-2, Fig. 3)."""
    g = rng(seed)
    T = 1 << log2T
    inn = levels * F
    ts = table_scale if trained else 1e-4
    table = g.uniform(-ts, ts, size=(levels, T, F)).astype(np.float32)
    H = MLP_HIDDEN
    W1 = g.normal(size=(H, inn)) * np.sqrt(2.0 / inn)
    b1 = g.normal(size=H) * 0.05
    W2 = g.normal(size=(H, H)) * np.sqrt(2.0 / H)
    b2 = g.normal(size=H) * 0.05
    if trained:
        W3 = g.normal(size=(7, H)) * head_scale / np.sqrt(H)
        b3 = g.normal(size=7) * head_scale * 0.1
    else:
        W3 = np.zeros((7, H)); b3 = np.zeros(7)
    mlp = np.concatenate([W1.ravel(), b1, W2.ravel(), b2, W3.ravel(), b3]).astype(np.float32)
    lo, hi = aabb
    return HashField(levels, log2T, F, tuple(res[:levels]), np.asarray(lo, np.float32),
                     np.asarray(hi, np.float32), table, mlp)


def dual_fields(scene: Scene, profile: str = "n3dv", seed: int = 40, trained: bool = True):
    """(𝓗_dyn, 𝓗_st) for a scene."""
    (tdyn, fdyn), (tst, fst) = HASH_PROFILES[profile]
    box = scene_aabb(scene.pos_opa)
    return (hash_field(tdyn, fdyn, box, seed, trained=trained),
            hash_field(tst, fst, box, seed + 1, trained=trained))


def offset_grads(n: int, seed: int, scale: float = 1.0):
    """Fixed ∂L/∂μ, ∂L/∂σ (float32 [n][4]) for deformation-backward tests."""
    g = rng(seed)
    gm = g.normal(size=(n, 4)).astype(np.float32) * scale
    gm[:, 3] = 0
    gs = (g.normal(size=(n, 4)) * scale).astype(np.float32)
    return gm, gs
