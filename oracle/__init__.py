"""ctypes front end of the CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs — never by the product package
`paper_2411_14847_b200`.  It shares no code with the CUDA path; its only shared
dependency is the seeded input generator `paper_2411_14847_b200/synth.py`
(random numbers and camera matrices, none of the method's arithmetic).

All results are float64 NumPy arrays (the oracle computes in double; the only
float arithmetic is the fp32 key replica of include/dass.h's KEY CHAIN).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++, -ffp-contract=off so the fp32 replica
    rounds every operation once; OpenMP for the O(Σ box area) scatter form)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.{os.getpid()}.tmp"   # concurrent builders must not share a temp file
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fopenmp", "-fPIC",
               "-shared", _SRC, "-o", tmp]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        _lib.oracle_bin_sort.restype = C.c_int64
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def threads() -> int:
    return lib().oracle_threads()


def set_threads(k: int) -> None:
    """OpenMP threads of the following oracle calls."""
    lib().oracle_set_threads(int(k))


def _cam(cam):
    s = cam.to_struct() if hasattr(cam, "to_struct") else cam
    return np.ascontiguousarray(s).reshape(1)


def shift(pos_opa, rot, mu, sigma, mask=None):
    n = pos_opa.shape[0]
    po = np.zeros((n, 4)); ro = np.zeros((n, 4))
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    lib().oracle_shift(n, _p(_f32(pos_opa)), _p(_f32(rot)), _p(_f32(mu)), _p(_f32(sigma)),
                       _p(m), _p(po), _p(ro))
    return po, ro


def shift_bwd(rot, sigma, mask, g_pos_out, g_rot_out):
    n = rot.shape[0]
    gm = np.zeros((n, 4)); gs = np.zeros((n, 4))
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    lib().oracle_shift_bwd(n, _p(_f32(rot)), _p(_f32(sigma)), _p(m),
                           _p(np.ascontiguousarray(g_pos_out, np.float64)),
                           _p(np.ascontiguousarray(g_rot_out, np.float64)), _p(gm), _p(gs))
    return gm, gs


def project(cam, scene, keep=None):
    """O2 for one view.  Returns a dict of per-Gaussian arrays."""
    n = scene.n
    out = dict(uvz=np.zeros((n, 3)), conic=np.zeros((n, 3)), opa=np.zeros(n),
               rgb=np.zeros((n, 3)), clampbits=np.zeros(n, np.int32), zf=np.zeros(n, np.float32),
               zbits=np.zeros(n, np.uint32), box=np.zeros((n, 4), np.int32),
               tiles=np.zeros(n, np.uint32), visible=np.zeros(n, np.uint8),
               rows=np.zeros((n, 4), np.uint32))
    k = None if keep is None else np.ascontiguousarray(keep, np.uint8)
    c = _cam(cam)
    lib().oracle_project(_p(c), n, scene.sh_degree, _p(_f32(scene.pos_opa)), _p(_f32(scene.scale)),
                         _p(_f32(scene.rot)), _p(_f32(scene.sh)), _p(k), _p(out["uvz"]),
                         _p(out["conic"]), _p(out["opa"]), _p(out["rgb"]), _p(out["clampbits"]),
                         _p(out["zf"]), _p(out["zbits"]), _p(out["box"]), _p(out["tiles"]),
                         _p(out["visible"]), _p(out["rows"]))
    return out


def cov2d(cam, pos_opa, scale, rot):
    n = pos_opa.shape[0]
    out = np.zeros((n, 4))
    c = _cam(cam)
    lib().oracle_cov2d(_p(c), n, _p(_f32(pos_opa)), _p(_f32(scale)), _p(_f32(rot)), _p(out))
    return out  # a, b, c, det


def rotmat_cov(q, s):
    R = np.zeros(9); S = np.zeros(9)
    rc = lib().oracle_rotmat_cov(_p(_f32(q)), _p(_f32(s)), _p(R), _p(S))
    if rc != 0:
        raise ValueError("degenerate")
    return R.reshape(3, 3), S.reshape(3, 3)


def sh_basis(deg, dirs):
    dirs = np.ascontiguousarray(dirs, np.float64)
    Y = np.zeros((dirs.shape[0], 16))
    lib().oracle_sh_basis(deg, dirs.shape[0], _p(dirs), _p(Y))
    return Y


def bin_sort(cam, proj):
    """O3: brute-force pairs sorted by (key, id) and the per-tile ranges.  The
    tiles of a Gaussian follow its A50 row spans proj["rows"] (the box rule of
    A05 if absent)."""
    n = proj["visible"].shape[0]
    c = _cam(cam)
    vis = np.ascontiguousarray(proj["visible"], np.uint8)
    zb = np.ascontiguousarray(proj["zbits"], np.uint32)
    box = np.ascontiguousarray(proj["box"], np.int32)
    rows = proj.get("rows")
    rows = None if rows is None else np.ascontiguousarray(rows, np.uint32)
    K = lib().oracle_bin_sort(_p(c), n, _p(vis), _p(zb), _p(box), C.c_int64(0), None, None, None,
                              _p(rows))
    ntiles = ((int(c["width"][0]) + 15) // 16) * ((int(c["height"][0]) + 15) // 16)
    keys = np.zeros(max(K, 1), np.uint64); ids = np.zeros(max(K, 1), np.uint32)
    ranges = np.zeros((ntiles, 2), np.uint32)
    lib().oracle_bin_sort(_p(c), n, _p(vis), _p(zb), _p(box), C.c_int64(K), _p(keys), _p(ids),
                          _p(ranges), _p(rows))
    return keys[:K], ids[:K], ranges


def _tie(tie_eps):
    return None if tie_eps is None else np.ascontiguousarray(tie_eps, np.float64)


def render(cam, scene, keep=None, bg=None, mode="scatter", tie_eps=None):
    """O4: returns dict(img[3,H,W], T[H,W], nacc, last_id, tie, term, pfwd, pbwd)."""
    c = _cam(cam)
    H, W = int(c["height"][0]), int(c["width"][0])
    o = dict(img=np.zeros((3, H, W)), T=np.zeros((H, W)), nacc=np.zeros((H, W), np.int32),
             last_id=np.zeros((H, W), np.int32), tie=np.zeros((H, W), np.uint8),
             term=np.zeros((H, W), np.uint8), pfwd=np.zeros((H, W), np.int64),
             pbwd=np.zeros((H, W), np.int64))
    k = None if keep is None else np.ascontiguousarray(keep, np.uint8)
    b = None if bg is None else np.ascontiguousarray(bg, np.float32)
    lib().oracle_render(_p(c), scene.n, scene.sh_degree, _p(_f32(scene.pos_opa)),
                        _p(_f32(scene.scale)), _p(_f32(scene.rot)), _p(_f32(scene.sh)), _p(k),
                        _p(b), 0 if mode == "literal" else 1, _p(_tie(tie_eps)), _p(o["img"]),
                        _p(o["T"]), _p(o["nacc"]), _p(o["last_id"]), _p(o["tie"]), _p(o["term"]),
                        _p(o["pfwd"]), _p(o["pbwd"]))
    return o


def render_bwd(cam, scene, dL_dimg, keep=None, bg=None, mode="scatter", tie_eps=None, kappa=False):
    """O5+O6: gradients of sum(dL_dimg * render) w.r.t. all parameters.
    kappa=True also returns the conditioning κ of every gradient entry
    (k_pos_opa, k_scale, k_rot, k_sh: Σ over pixels of |term| through |Jacobian|)
    and the A29 tie slack t_* (t_gradstat for ∇p̄): at pixels with one tie
    decision point, |contribution(branch A) − contribution(branch B)| through
    |Jacobian|.  gtie flags Gaussians whose box holds a pixel with ≥ 2 tie points."""
    c = _cam(cam)
    H, W = int(c["height"][0]), int(c["width"][0])
    n = scene.n
    nc = (scene.sh_degree + 1) ** 2
    o = dict(g_pos_opa=np.zeros((n, 4)), g_scale=np.zeros((n, 4)), g_rot=np.zeros((n, 4)),
             g_sh=np.zeros((n, nc, 3)), g2d=np.zeros((n, 9)), gradstat_sum=np.zeros(n),
             gradstat_cnt=np.zeros(n, np.int32), gtie=np.zeros(n, np.uint8),
             img=np.zeros((3, H, W)), T=np.zeros((H, W)))
    if kappa:
        o.update(k_pos_opa=np.zeros((n, 4)), k_scale=np.zeros((n, 4)), k_rot=np.zeros((n, 4)),
                 k_sh=np.zeros((n, nc, 3)))
        # tie slack (A29): |branch difference| at one-tie pixels through |Jacobian|
        o.update(t_pos_opa=np.zeros((n, 4)), t_scale=np.zeros((n, 4)), t_rot=np.zeros((n, 4)),
                 t_sh=np.zeros((n, nc, 3)), t_gradstat=np.zeros(n))
    k = None if keep is None else np.ascontiguousarray(keep, np.uint8)
    b = None if bg is None else np.ascontiguousarray(bg, np.float32)
    lib().oracle_render_bwd(_p(c), n, scene.sh_degree, _p(_f32(scene.pos_opa)),
                            _p(_f32(scene.scale)), _p(_f32(scene.rot)), _p(_f32(scene.sh)), _p(k),
                            _p(b), _p(_f32(dL_dimg)), 0 if mode == "literal" else 1,
                            _p(_tie(tie_eps)), _p(o["g_pos_opa"]), _p(o["g_scale"]),
                            _p(o["g_rot"]), _p(o["g_sh"]), _p(o["g2d"]), _p(o["gradstat_sum"]),
                            _p(o["gradstat_cnt"]), _p(o["gtie"]), _p(o["img"]), _p(o["T"]),
                            _p(o.get("k_pos_opa")), _p(o.get("k_scale")), _p(o.get("k_rot")),
                            _p(o.get("k_sh")), _p(o.get("t_pos_opa")), _p(o.get("t_scale")),
                            _p(o.get("t_rot")), _p(o.get("t_sh")), _p(o.get("t_gradstat")))
    return o


def error_map(cam, rendered, gt, gamma, pos_opa, n_base=None, s_err=None):
    c = _cam(cam)
    H, W = int(c["height"][0]), int(c["width"][0])
    n = pos_opa.shape[0]
    nb = n if n_base is None else n_base
    o = dict(err=np.zeros((H, W)), D=np.zeros((H, W), np.uint8),
             s_err=np.zeros(n, np.uint8) if s_err is None else np.array(s_err, np.uint8),
             xy=np.zeros((n, 2), np.int32), tie_g=np.zeros(n, np.uint8),
             tie_px=np.zeros((H, W), np.uint8))
    lib().oracle_error_map(_p(c), _p(_f32(rendered)), _p(_f32(gt)), C.c_double(gamma), nb,
                           _p(_f32(pos_opa)), _p(o["err"]), _p(o["D"]), _p(o["s_err"]),
                           _p(o["xy"]), _p(o["tie_g"]), _p(o["tie_px"]))
    return o


def inherit(m):
    """f3: keep = Quant(sigmoid(m)) (Eq. 1)."""
    m = _f32(m)
    keep = np.zeros(m.shape[0], np.uint8)
    lib().oracle_inherit(m.shape[0], _p(m), _p(keep))
    return keep


def inherit_bwd(m, pos_opa, scale, g_pos_opa, g_scale, lambda_inher=0.0):
    """f3: STE gradient of m + the mask loss λ_inher·Σσ(m) (Eq. 2)."""
    m = _f32(m)
    g = np.zeros(m.shape[0])
    lib().oracle_inherit_bwd(m.shape[0], _p(m), _p(_f32(pos_opa)), _p(_f32(scale)),
                             _p(np.ascontiguousarray(g_pos_opa, np.float64)),
                             _p(np.ascontiguousarray(g_scale, np.float64)),
                             C.c_double(lambda_inher), _p(g))
    return g


def fidelity_loss(img, gt, lam=0.2, grad=True, dssim_scale=1.0):
    """f1 / Eq. 3: returns (L, L1, SSIM, dL/dI or None) in double; D-SSIM =
    dssim_scale·(1 − SSIM) (1: 3DGS code, A39; 0.5: SPEC S:266)."""
    img = _f32(img); gt = _f32(gt)
    H, W = img.shape[1], img.shape[2]
    out = np.zeros(3)
    g = np.zeros(img.shape) if grad else None
    lib().oracle_fidelity_loss(W, H, _p(img), _p(gt), C.c_double(lam), C.c_double(dssim_scale),
                               _p(out), _p(g))
    return out[0], out[1], out[2], g


# ---- f2: hash-grid deformation (§3.3, §B; A41-A43) ----
def _hcfg(field):
    return np.ascontiguousarray(field.to_struct()).reshape(1)


def hash_params(inputs):
    return lib().oracle_hash_params(int(inputs))


def hash_encode(field, pos_opa):
    """enc(p): double [m][L·F]."""
    po = _f32(pos_opa)
    m = po.shape[0]
    feat = np.zeros((m, field.L * field.F))
    lib().oracle_hash_encode(_p(_hcfg(field)), _p(_f32(field.table)), m, _p(po), _p(feat))
    return feat


def deform(field, pos_opa):
    """(μ, σ, tie) for every row of pos_opa: double [m][4] ×2, uint8 [m]."""
    po = _f32(pos_opa)
    m = po.shape[0]
    mu = np.zeros((m, 4)); sg = np.zeros((m, 4)); tie = np.zeros(m, np.uint8)
    lib().oracle_deform_fwd(_p(_hcfg(field)), _p(_f32(field.table)), _p(_f32(field.mlp)), m,
                            _p(po), _p(mu), _p(sg), _p(tie))
    return mu, sg, tie


def deform_bwd(field, pos_opa, g_mu, g_sigma, kappa=False):
    """(∂L/∂table [L][T][F], ∂L/∂mlp flat[, κ_table, κ_mlp]) in double."""
    po = _f32(pos_opa)
    m = po.shape[0]
    gt = np.zeros(field.table.shape); gp = np.zeros(field.mlp.shape)
    kt = np.zeros(field.table.shape) if kappa else None
    km = np.zeros(field.mlp.shape) if kappa else None
    lib().oracle_deform_bwd(_p(_hcfg(field)), _p(_f32(field.table)), _p(_f32(field.mlp)), m,
                            _p(po), _p(np.ascontiguousarray(g_mu, np.float64)),
                            _p(np.ascontiguousarray(g_sigma, np.float64)), _p(gt), _p(gp),
                            _p(kt), _p(km))
    return (gt, gp, kt, km) if kappa else (gt, gp)


# ---- f4: error-guided densification + identity-feature render (A44-A47) ----
def densify_select(gsum, gcnt, s_err, tau_pos, tau_err):
    """Eq. 4: in_S uint8[n] and |S| (decisions in fp32, A44)."""
    gsum = _f32(gsum)
    n = gsum.shape[0]
    gcnt = np.ascontiguousarray(gcnt, np.uint32)
    se = None if s_err is None else np.ascontiguousarray(s_err, np.uint8)
    out = np.zeros(n, np.uint8)
    c = lib().oracle_densify_select(n, _p(gsum), _p(gcnt), _p(se), C.c_float(tau_pos),
                                    C.c_float(tau_err), _p(out))
    return out, c


def philox4x64(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint64); k = np.ascontiguousarray(key, np.uint64)
    out = np.zeros(4, np.uint64)
    lib().oracle_philox4x64(_p(c), _p(k), _p(out))
    return out


def spawn(idx, K, shrink, child_opacity, seed, pos_opa, scale, rot, want_z=False):
    """Spawn densification (A45): child (pos_opa, scale) double [m·K][4] (+ z)."""
    idx = np.ascontiguousarray(idx, np.int32)
    m = idx.shape[0]
    po = np.zeros((m * K, 4)); sc = np.zeros((m * K, 4))
    z = np.zeros((m * K, 3)) if want_z else None
    lib().oracle_spawn(m, _p(idx), int(K), C.c_double(shrink), C.c_double(child_opacity),
                       C.c_uint64(seed), _p(_f32(pos_opa)), _p(_f32(scale)), _p(_f32(rot)),
                       _p(po), _p(sc), _p(z))
    return (po, sc, z) if want_z else (po, sc)


def render_features(cam, scene, feat, keep=None):
    """Eq. 9: M double [C][H][W] and tie flags uint8 [H][W]."""
    feat = _f32(feat)
    Cn = feat.shape[1]
    out = np.zeros((Cn, cam.height, cam.width))
    tie = np.zeros((cam.height, cam.width), np.uint8)
    k = None if keep is None else np.ascontiguousarray(keep, np.uint8)
    lib().oracle_render_features(_p(_cam(cam)), scene.n, _p(_f32(scene.pos_opa)),
                                 _p(_f32(scene.scale)), _p(_f32(scene.rot)), _p(k), Cn, _p(feat),
                                 _p(out), _p(tie))
    return out, tie


def prune_keep(pos_opa, first, min_opacity):
    """Opacity pruning (A46): keep uint8[n] and the kept count."""
    po = _f32(pos_opa)
    keep = np.zeros(po.shape[0], np.uint8)
    c = lib().oracle_prune_keep(po.shape[0], int(first), _p(po), C.c_float(min_opacity), _p(keep))
    return keep, c
