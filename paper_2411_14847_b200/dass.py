"""Thin Python binding of libdass.so (include/dass.h), same names as the C-ABI.

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of libdass.so.  Tensors must be CUDA tensors of the documented dtype
and layout; the binding passes `tensor.data_ptr()` and the current torch
stream.  There is no CPU fallback: if libdass.so is missing or a GPU is not
available, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libdass.so")

DASS_OK = 0
DASS_ERR_INVALID_ARG = 1
DASS_ERR_DATA = 2
DASS_ERR_NUMERICAL = 3
DASS_ERR_CAPACITY = 4
DASS_ERR_CUDA = 5

EXPORTS = (
    "dass_status_string", "dass_last_error", "dass_abi_version", "dass_kernel_launches",
    "dass_apply_shift", "dass_apply_shift_bwd", "dass_project", "dass_project_views",
    "dass_project_views_part",
    "dass_bin_sort_workspace", "dass_bin_sort", "dass_render_accept_workspace", "dass_render_fwd",
    "dass_render_bwd_workspace",
    "dass_render_bwd", "dass_render_bwd_raster", "dass_render_bwd_preprocess_views",
    "dass_fidelity_loss_workspace", "dass_fidelity_loss", "dass_inherit_mask",
    "dass_inherit_mask_bwd", "dass_error_map", "dass_render_stats",
    "dass_deform_param_count", "dass_deform_fwd", "dass_deform_bwd", "dass_partition_workspace",
    "dass_partition", "dass_densify_select", "dass_spawn", "dass_prune_select", "dass_gather",
    "dass_render_features", "dass_render_fwd_tiles", "dass_render_bwd_raster_tiles",
    "dass_render_bwd_preprocess_views_uv", "dass_render_bwd_preprocess_views_part",
    "dass_gradstat_from_uv", "dass_timestamp",
    "dass_scan_nonfinite",
    "dass_bin_sort_views_workspace", "dass_bin_sort_views", "dass_bin_sort_shared",
)


class DassError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: status {status}: {msg}")
        self.status = status


class dass_camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("viewmat", C.c_float * 12), ("near_plane", C.c_float),
                ("full_proj", C.c_float * 16)]


def camera_struct(cam) -> dass_camera:
    """From any object with width/height/fx/fy/cx/cy/viewmat/near/full_proj."""
    c = dass_camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    vm = np.asarray(cam.viewmat, np.float32).reshape(12)
    for i in range(12):
        c.viewmat[i] = float(vm[i])
    c.near_plane = float(getattr(cam, "near", getattr(cam, "near_plane", 0.2)))
    fp = np.asarray(cam.full_proj, np.float32).reshape(16)
    for i in range(16):
        c.full_proj[i] = float(fp[i])
    return c


class dass_hashgrid(C.Structure):
    _fields_ = [("levels", C.c_int32), ("log2_table", C.c_int32), ("features", C.c_int32),
                ("reserved", C.c_int32), ("resolution", C.c_int32 * 16),
                ("aabb_min", C.c_float * 3), ("aabb_max", C.c_float * 3)]


def hashgrid_struct(field) -> dass_hashgrid:
    """From any object with L / log2T / F / res / lo / hi (synth.HashField)."""
    if isinstance(field, dass_hashgrid):
        return field
    c = dass_hashgrid()
    c.levels, c.log2_table, c.features = int(field.L), int(field.log2T), int(field.F)
    for i, r in enumerate(field.res):
        c.resolution[i] = int(r)
    for k in range(3):
        c.aabb_min[k] = float(field.lo[k])
        c.aabb_max[k] = float(field.hi[k])
    return c


_lib = None


def lib():
    """Load libdass.so; raise loudly if it is missing (no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2411_14847_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.dass_status_string.restype = C.c_char_p
        L.dass_last_error.restype = C.c_char_p
        L.dass_kernel_launches.restype = C.c_uint64
        P = C.c_void_p
        i32, i64 = C.c_int32, C.c_int64
        L.dass_apply_shift.argtypes = [i32, P, P, P, P, P, P, P, P]
        L.dass_apply_shift_bwd.argtypes = [i32, P, P, P, P, P, P, P, P]
        L.dass_project.argtypes = [P, i32, i32, P, P, P, P, P, P, P, P, P, P, P, P]
        L.dass_project_views.argtypes = [P, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P, P]
        L.dass_project_views_part.argtypes = [i32, P, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P, P]
        L.dass_bin_sort_workspace.argtypes = [i32, i32, i64, P]
        L.dass_bin_sort.argtypes = [P, i32, P, P, P, P, P, C.c_size_t, i64, P, P, P, P, P, P]
        L.dass_bin_sort_shared.argtypes = L.dass_bin_sort.argtypes
        L.dass_bin_sort_views_workspace.argtypes = [i32, i32, i64, P]
        L.dass_bin_sort_views.argtypes = [P, i32, i32, P, P, P, P, P, C.c_size_t, i64, P, P, P, P]
        L.dass_render_accept_workspace.argtypes = [i32, i64, P]
        L.dass_render_fwd.argtypes = [P, P, P, P, P, P, P, P, P, P, P, P, C.c_size_t, i64, P]
        L.dass_render_bwd_workspace.argtypes = [i32, P]
        L.dass_render_bwd.argtypes = [P, i32, i32, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P,
                                      P, C.c_size_t, i64, P, C.c_size_t, P, P, P, P, P, P, P]
        L.dass_render_bwd_raster.argtypes = [P, i32, P, P, P, P, P, P, P, P, P, P, P, C.c_size_t,
                                             i64, P, P]
        L.dass_render_bwd_preprocess_views.argtypes = [P, i32, i32, i32, P, P, P, P, P, P, P, P, P,
                                                       P, P, P, P, P, P, P]
        L.dass_fidelity_loss_workspace.argtypes = [i32, i32, P]
        L.dass_fidelity_loss.argtypes = [i32, i32, P, P, C.c_float, C.c_float, P, C.c_size_t, P, P, P]
        L.dass_inherit_mask.argtypes = [i32, P, P, P]
        L.dass_inherit_mask_bwd.argtypes = [i32, P, P, P, P, P, C.c_float, P, P]
        L.dass_error_map.argtypes = [P, P, P, C.c_float, P, P, i32, P, P, P]
        L.dass_render_stats.argtypes = [P, P, P, P, P, P, P, P, P, P]
        L.dass_timestamp.argtypes = [P, i32, P]
        L.dass_scan_nonfinite.argtypes = [P, i64, P, P, P]
        L.dass_deform_param_count.argtypes = [P, P, P]
        L.dass_deform_fwd.argtypes = [P, P, P, i32, P, P, P, P, P, P]
        L.dass_deform_bwd.argtypes = [P, P, P, i32, P, P, P, P, P, P, P, P]
        L.dass_partition_workspace.argtypes = [i32, P]
        L.dass_partition.argtypes = [i32, P, P, P, P, P, C.c_size_t, P]
        L.dass_densify_select.argtypes = [i32, P, P, P, C.c_float, C.c_float, P, P, P, P,
                                          C.c_size_t, P]
        L.dass_spawn.argtypes = [i32, i32, P, P, P, P, P, i32, P, i32, C.c_float, C.c_float,
                                 C.c_uint64, P, P, P, P, P, P]
        L.dass_prune_select.argtypes = [i32, i32, P, C.c_float, P, P, P, P, C.c_size_t, P]
        L.dass_gather.argtypes = [i32, i32, P, P, P, P, P, i32, P, P, P, P, P, P, P]
        L.dass_render_features.argtypes = [P, P, P, P, P, P, i32, P, P, P]
        L.dass_render_fwd_tiles.argtypes = [P, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P,
                                            C.c_size_t, i64, P]
        L.dass_render_bwd_raster_tiles.argtypes = [P, i32, i32, i32, i32, P, P, P, P, P, P, P, P,
                                                   P, P, P, C.c_size_t, i64, P, P]
        L.dass_render_bwd_preprocess_views_uv.argtypes = [P, i32, i32, i32, P, P, P, P, P, P, P,
                                                          P, P, P, P, P, P, P, P, P, P, P]
        L.dass_render_bwd_preprocess_views_part.argtypes = [i32] + list(L.dass_render_bwd_preprocess_views_uv.argtypes)
        L.dass_gradstat_from_uv.argtypes = [i32, i32, P, P, P]
        _lib = L
    return _lib


def _check(status: int, where: str):
    if status != DASS_OK:
        raise DassError(status, where, lib().dass_last_error().decode())


_BAD_DTYPES = None


def _nbytes(t) -> int:
    """Size in bytes of a contiguous tensor (0 for None)."""
    return 0 if t is None else t.numel() * t.element_size()


def _ptr(t):
    """Device pointer of a contiguous CUDA tensor.  libdass computes in fp32 and
    int32/uint8/uint64 only: a float64/float16/bfloat16 tensor is refused rather
    than reinterpreted."""
    global _BAD_DTYPES
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libdass takes CUDA tensors only (no CPU path)")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    if _BAD_DTYPES is None:
        import torch
        _BAD_DTYPES = (torch.float64, torch.float16, torch.bfloat16)
    if t.dtype in _BAD_DTYPES:
        raise TypeError(f"libdass takes float32 arrays, got {t.dtype}")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _cam(cam):
    return cam if isinstance(cam, dass_camera) else camera_struct(cam)


def kernel_launches() -> int:
    return int(lib().dass_kernel_launches())


def abi_version() -> int:
    return int(lib().dass_abi_version())


def dass_apply_shift(pos_opa, rot, mu, sigma, dyn_mask, pos_opa_out, rot_out, stream=None):
    n = pos_opa.shape[0]
    _check(lib().dass_apply_shift(n, _ptr(pos_opa), _ptr(rot), _ptr(mu), _ptr(sigma),
                                  _ptr(dyn_mask), _ptr(pos_opa_out), _ptr(rot_out),
                                  _stream(stream)), "dass_apply_shift")


def dass_apply_shift_bwd(rot, sigma, dyn_mask, g_pos_out, g_rot_out, g_mu, g_sigma, stream=None):
    n = rot.shape[0]
    _check(lib().dass_apply_shift_bwd(n, _ptr(rot), _ptr(sigma), _ptr(dyn_mask), _ptr(g_pos_out),
                                      _ptr(g_rot_out), _ptr(g_mu), _ptr(g_sigma),
                                      _stream(stream)), "dass_apply_shift_bwd")


def dass_project(cam, sh_degree, pos_opa, scale, rot, sh, keep_mask, xy_depth, conic_opa, rgb,
                 box, tile_rows, tiles_touched, stream=None):
    """tile_rows: int32 [N,4], the A50 footprint row spans (KEY CHAIN step 13)."""
    c = _cam(cam)
    _check(lib().dass_project(C.byref(c), pos_opa.shape[0], sh_degree, _ptr(pos_opa), _ptr(scale),
                              _ptr(rot), _ptr(sh), _ptr(keep_mask), _ptr(xy_depth),
                              _ptr(conic_opa), _ptr(rgb), _ptr(box), _ptr(tile_rows),
                              _ptr(tiles_touched), _stream(stream)), "dass_project")


def dass_project_views(cams, sh_degree, pos_opa, scale, rot, sh, keep_mask, xy_depth, conic_opa,
                       rgb, box, tile_rows, tiles_touched, stream=None):
    arr = (dass_camera * len(cams))(*[_cam(c) for c in cams])
    _check(lib().dass_project_views(arr, len(cams), pos_opa.shape[0], sh_degree, _ptr(pos_opa),
                                    _ptr(scale), _ptr(rot), _ptr(sh), _ptr(keep_mask),
                                    _ptr(xy_depth), _ptr(conic_opa), _ptr(rgb), _ptr(box),
                                    _ptr(tile_rows), _ptr(tiles_touched), _stream(stream)),
           "dass_project_views")


DASS_PROJECT_KEYS, DASS_PROJECT_RECORDS, DASS_PROJECT_ALL = 1, 2, 3


def dass_project_views_part(part, cams, sh_degree, pos_opa, scale, rot, sh, keep_mask, xy_depth,
                            conic_opa, rgb, box, tile_rows, tiles_touched, stream=None):
    arr = (dass_camera * len(cams))(*[_cam(c) for c in cams])
    _check(lib().dass_project_views_part(part, arr, len(cams), pos_opa.shape[0], sh_degree,
                                         _ptr(pos_opa), _ptr(scale), _ptr(rot), _ptr(sh),
                                         _ptr(keep_mask), _ptr(xy_depth), _ptr(conic_opa),
                                         _ptr(rgb), _ptr(box), _ptr(tile_rows),
                                         _ptr(tiles_touched), _stream(stream)),
           "dass_project_views_part")


def dass_bin_sort_workspace(n, num_tiles, pair_capacity) -> int:
    out = C.c_size_t(0)
    _check(lib().dass_bin_sort_workspace(n, num_tiles, pair_capacity, C.byref(out)),
           "dass_bin_sort_workspace")
    return out.value


def dass_bin_sort(cam, n, xy_depth, box, tile_rows, tiles_touched, ws, pair_capacity, sorted_keys,
                  sorted_ids, tile_ranges, num_pairs_dev, host_mode=False, stream=None,
                  shared=False):
    """Returns K in host mode (raises DassError(CAPACITY) on overflow), else None.
    shared=True calls dass_bin_sort_shared (a view sorted next to other views' work)."""
    c = _cam(cam)
    k = C.c_int64(-1)
    fn = lib().dass_bin_sort_shared if shared else lib().dass_bin_sort
    st = fn(C.byref(c), n, _ptr(xy_depth), _ptr(box), _ptr(tile_rows),
            _ptr(tiles_touched),
            _ptr(ws), ws.numel() * ws.element_size(), pair_capacity,
            _ptr(sorted_keys), _ptr(sorted_ids), _ptr(tile_ranges),
            _ptr(num_pairs_dev), C.byref(k) if host_mode else None,
            _stream(stream))
    _check(st, "dass_bin_sort_shared" if shared else "dass_bin_sort")
    return k.value if host_mode else None


def dass_bin_sort_views_workspace(num_views, n, view_capacity) -> int:
    out = C.c_size_t(0)
    _check(lib().dass_bin_sort_views_workspace(num_views, n, view_capacity, C.byref(out)),
           "dass_bin_sort_views_workspace")
    return out.value


def dass_bin_sort_views(cams, n, xy_depth, box, tile_rows, tiles_touched, ws, view_capacity,
                        sorted_ids, tile_ranges, num_pairs_dev, stream=None):
    """All views of a timestep at once (graph mode): per view v, sorted_ids[v],
    tile_ranges[v] and num_pairs_dev[v] = (K_v, overflow_v) as dass_bin_sort."""
    arr = (dass_camera * len(cams))(*[_cam(c) for c in cams])
    _check(lib().dass_bin_sort_views(arr, len(cams), n, _ptr(xy_depth), _ptr(box), _ptr(tile_rows),
                                     _ptr(tiles_touched), _ptr(ws), ws.numel() * ws.element_size(),
                                     view_capacity, _ptr(sorted_ids), _ptr(tile_ranges),
                                     _ptr(num_pairs_dev), _stream(stream)),
           "dass_bin_sort_views")


def dass_render_accept_workspace(num_tiles, pair_capacity) -> int:
    out = C.c_size_t(0)
    _check(lib().dass_render_accept_workspace(num_tiles, pair_capacity, C.byref(out)),
           "dass_render_accept_workspace")
    return out.value


def dass_render_fwd(cam, tile_ranges, sorted_ids, xy_depth, conic_opa, rgb, box, bg, out_img,
                    out_T, out_last, accept=None, pair_capacity=0, stream=None, tiles=None):
    """tiles = (begin, stride, count): render only that tile subset (dass_render_fwd_tiles)."""
    c = _cam(cam)
    b = None if bg is None else (C.c_float * 3)(*[float(x) for x in bg])
    tb, ts, tc = tiles if tiles is not None else (0, 1, -1)
    _check(lib().dass_render_fwd_tiles(C.byref(c), int(tb), int(ts), int(tc), _ptr(tile_ranges),
                                       _ptr(sorted_ids), _ptr(xy_depth), _ptr(conic_opa),
                                       _ptr(rgb), _ptr(box), b, _ptr(out_img), _ptr(out_T),
                                       _ptr(out_last), _ptr(accept), _nbytes(accept),
                                       pair_capacity, _stream(stream)), "dass_render_fwd")


def dass_render_bwd_workspace(n) -> int:
    out = C.c_size_t(0)
    _check(lib().dass_render_bwd_workspace(n, C.byref(out)), "dass_render_bwd_workspace")
    return out.value


def dass_render_bwd(cam, sh_degree, pos_opa, scale, rot, sh, keep_mask, tile_ranges, sorted_ids,
                    xy_depth, conic_opa, rgb, box, bg, out_T, out_last, dL_dimg, ws, g_pos_opa,
                    g_scale, g_rot, g_sh, gradstat_sum, gradstat_cnt, accept=None,
                    pair_capacity=0, stream=None):
    c = _cam(cam)
    b = None if bg is None else (C.c_float * 3)(*[float(x) for x in bg])
    _check(lib().dass_render_bwd(C.byref(c), pos_opa.shape[0], sh_degree, _ptr(pos_opa),
                                 _ptr(scale), _ptr(rot), _ptr(sh), _ptr(keep_mask),
                                 _ptr(tile_ranges), _ptr(sorted_ids), _ptr(xy_depth),
                                 _ptr(conic_opa), _ptr(rgb), _ptr(box), b, _ptr(out_T),
                                 _ptr(out_last), _ptr(dL_dimg), _ptr(accept), _nbytes(accept),
                                 pair_capacity,
                                 _ptr(ws), ws.numel() * ws.element_size(), _ptr(g_pos_opa),
                                 _ptr(g_scale),
                                 _ptr(g_rot), _ptr(g_sh), _ptr(gradstat_sum), _ptr(gradstat_cnt),
                                 _stream(stream)), "dass_render_bwd")


def dass_render_bwd_raster(cam, n, tile_ranges, sorted_ids, xy_depth, conic_opa, rgb, box, bg,
                           out_T, out_last, dL_dimg, g2d, accept=None, pair_capacity=0,
                           stream=None, tiles=None):
    """tiles = (begin, stride, count): the tile subset's partial moments."""
    c = _cam(cam)
    b = None if bg is None else (C.c_float * 3)(*[float(x) for x in bg])
    tb, ts, tc = tiles if tiles is not None else (0, 1, -1)
    _check(lib().dass_render_bwd_raster_tiles(C.byref(c), int(tb), int(ts), int(tc), n,
                                              _ptr(tile_ranges), _ptr(sorted_ids), _ptr(xy_depth),
                                              _ptr(conic_opa), _ptr(rgb), _ptr(box), b,
                                              _ptr(out_T), _ptr(out_last), _ptr(dL_dimg),
                                              _ptr(accept), _nbytes(accept), pair_capacity,
                                              _ptr(g2d),
                                              _stream(stream)), "dass_render_bwd_raster")


DASS_PREPROCESS_GEOMETRY, DASS_PREPROCESS_SH, DASS_PREPROCESS_ALL = 1, 2, 3


def dass_render_bwd_preprocess_views(cams, sh_degree, pos_opa, scale, rot, sh, keep_mask,
                                     conic_opa, rgb, box, g2d, g_pos_opa, g_scale, g_rot, g_sh,
                                     gradstat_sum, gradstat_cnt, stream=None, uv_out=None,
                                     uv_count=None, part=DASS_PREPROCESS_ALL):
    """uv_out: per view None or a float2[n] tensor — split views add their
    (∂L/∂u·W/2, ∂L/∂v·H/2) there instead of the ∇p̄ norm; uv_count[v] truthy:
    this GPU adds the split view's visibility count (one GPU per view).
    part: DASS_PREPROCESS_GEOMETRY / _SH / _ALL (dass_render_bwd_preprocess_views_part)."""
    arr = (dass_camera * len(cams))(*[_cam(c) for c in cams])
    uv = cnt = None
    if uv_out is not None:
        if len(uv_out) != len(cams):
            raise ValueError("uv_out needs one entry per view")
        uv = (C.c_void_p * len(cams))(*[None if u is None else _ptr(u).value for u in uv_out])
        flags = uv_count if uv_count is not None else [0] * len(cams)
        cnt = (C.c_uint8 * len(cams))(*[1 if f else 0 for f in flags])
    _check(lib().dass_render_bwd_preprocess_views_part(
        part, arr, len(cams), pos_opa.shape[0], sh_degree, _ptr(pos_opa), _ptr(scale), _ptr(rot),
        _ptr(sh), _ptr(keep_mask), _ptr(conic_opa), _ptr(rgb), _ptr(box), _ptr(g2d),
        _ptr(g_pos_opa), _ptr(g_scale), _ptr(g_rot), _ptr(g_sh), _ptr(gradstat_sum),
        _ptr(gradstat_cnt), uv, cnt, _stream(stream)), "dass_render_bwd_preprocess_views")


def dass_gradstat_from_uv(uv, gradstat_sum, stream=None):
    """∇p̄ norms of split views from their reduced uv blocks (float2 [S][n])."""
    S, n = uv.shape[0], uv.shape[1]
    _check(lib().dass_gradstat_from_uv(n, S, _ptr(uv), _ptr(gradstat_sum), _stream(stream)),
           "dass_gradstat_from_uv")


def dass_fidelity_loss_workspace(width, height) -> int:
    out = C.c_size_t(0)
    _check(lib().dass_fidelity_loss_workspace(width, height, C.byref(out)),
           "dass_fidelity_loss_workspace")
    return out.value


def dass_fidelity_loss(img, gt, lam, ws, loss, dL_dimg=None, stream=None, dssim_scale=1.0):
    """Eq. 3: loss (device float[3] = L, L1, SSIM) and optionally ∂L/∂img.
    D-SSIM = dssim_scale·(1 − SSIM): 1.0 = 3DGS (A39), 0.5 = SPEC's (1 − SSIM)/2."""
    H, W = img.shape[1], img.shape[2]
    _check(lib().dass_fidelity_loss(W, H, _ptr(img), _ptr(gt), float(lam), float(dssim_scale),
                                    _ptr(ws),
                                    ws.numel() * ws.element_size(), _ptr(loss), _ptr(dL_dimg),
                                    _stream(stream)), "dass_fidelity_loss")


def dass_inherit_mask(m, keep, stream=None):
    _check(lib().dass_inherit_mask(m.shape[0], _ptr(m), _ptr(keep), _stream(stream)),
           "dass_inherit_mask")


def dass_inherit_mask_bwd(m, pos_opa, scale, g_pos_opa, g_scale, lambda_inher, g_m, stream=None):
    _check(lib().dass_inherit_mask_bwd(m.shape[0], _ptr(m), _ptr(pos_opa), _ptr(scale),
                                       _ptr(g_pos_opa), _ptr(g_scale), float(lambda_inher),
                                       _ptr(g_m), _stream(stream)), "dass_inherit_mask_bwd")


def dass_error_map(cam, rendered, gt, gamma_err, err, dmask, n_base, pos_opa, s_err, stream=None):
    c = _cam(cam)
    _check(lib().dass_error_map(C.byref(c), _ptr(rendered), _ptr(gt), gamma_err, _ptr(err),
                                _ptr(dmask), n_base, _ptr(pos_opa), _ptr(s_err), _stream(stream)),
           "dass_error_map")


def dass_render_stats(cam, tile_ranges, sorted_ids, xy_depth, conic_opa, box, out_T, out_last,
                      counters, stream=None):
    c = _cam(cam)
    _check(lib().dass_render_stats(C.byref(c), _ptr(tile_ranges), _ptr(sorted_ids),
                                   _ptr(xy_depth), _ptr(conic_opa), _ptr(box), _ptr(out_T),
                                   _ptr(out_last), _ptr(counters), _stream(stream)),
           "dass_render_stats")


def dass_scan_nonfinite(data, bad_dev, host_mode=False, stream=None):
    """bad_dev (int32[1] device) += number of NaN/Inf in data.  Host mode returns the
    count and raises DassError(NUMERICAL) when it is non-zero; graph mode returns None."""
    h = C.c_int64(0)
    _check(lib().dass_scan_nonfinite(_ptr(data), data.numel(), _ptr(bad_dev),
                                     C.byref(h) if host_mode else None, _stream(stream)),
           "dass_scan_nonfinite")
    return h.value if host_mode else None


def dass_timestamp(stamps, slot, stream=None):
    """Diagnostic: GPU global timer (ns) → stamps[slot] when the stream gets there."""
    _check(lib().dass_timestamp(_ptr(stamps), slot, _stream(stream)), "dass_timestamp")


def dass_deform_param_count(field):
    """(table floats, mlp floats) of a hash-grid field."""
    t, m = C.c_int64(0), C.c_int64(0)
    _check(lib().dass_deform_param_count(C.byref(hashgrid_struct(field)), C.byref(t), C.byref(m)),
           "dass_deform_param_count")
    return t.value, m.value


def dass_deform_fwd(field, table, mlp, pos_opa, mu, sigma, idx=None, count=None, n=None,
                    stream=None):
    """f2: (μ, σ) = 𝓗(p) for rows idx[k], k < *count (device) or n."""
    if n is None:
        n = idx.shape[0] if idx is not None else pos_opa.shape[0]
    _check(lib().dass_deform_fwd(C.byref(hashgrid_struct(field)), _ptr(table), _ptr(mlp), int(n),
                                 _ptr(idx), _ptr(count), _ptr(pos_opa), _ptr(mu), _ptr(sigma),
                                 _stream(stream)), "dass_deform_fwd")


def dass_deform_bwd(field, table, mlp, pos_opa, g_mu, g_sigma, g_table, g_mlp, idx=None,
                    count=None, n=None, stream=None):
    """f2: g_table, g_mlp += ∂L/∂(table, mlp) from ∂L/∂μ, ∂L/∂σ."""
    if n is None:
        n = idx.shape[0] if idx is not None else pos_opa.shape[0]
    _check(lib().dass_deform_bwd(C.byref(hashgrid_struct(field)), _ptr(table), _ptr(mlp), int(n),
                                 _ptr(idx), _ptr(count), _ptr(pos_opa), _ptr(g_mu), _ptr(g_sigma),
                                 _ptr(g_table), _ptr(g_mlp), _stream(stream)), "dass_deform_bwd")


def dass_partition_workspace(n) -> int:
    out = C.c_size_t(0)
    _check(lib().dass_partition_workspace(int(n), C.byref(out)), "dass_partition_workspace")
    return out.value


def dass_partition(mask, idx_dyn, idx_st, counts, ws, stream=None):
    """Stable split of range(n) by mask ≠ 0 (device counts[2] = #dyn, #st)."""
    n = mask.shape[0]
    _check(lib().dass_partition(n, _ptr(mask), _ptr(idx_dyn), _ptr(idx_st), _ptr(counts), _ptr(ws),
                                ws.numel() * ws.element_size(), _stream(stream)),
           "dass_partition")


def _ws_bytes(ws):
    return ws.numel() * ws.element_size()


def dass_densify_select(gsum, gcnt, s_err, tau_pos, tau_err, in_S, idx, counts, ws, stream=None):
    """Eq. 4: in_S flags, idx[:counts[0]] = S ascending (device counts)."""
    n = gsum.shape[0]
    _check(lib().dass_densify_select(n, _ptr(gsum), _ptr(gcnt), _ptr(s_err), float(tau_pos),
                                     float(tau_err), _ptr(in_S), _ptr(idx), _ptr(counts), _ptr(ws),
                                     _ws_bytes(ws), _stream(stream)), "dass_densify_select")


def dass_spawn(sh_degree, pos_opa, scale, rot, sh, dyn, m, idx, spawn_count, scale_shrink,
               child_opacity, seed, out_pos_opa, out_scale, out_rot, out_sh, out_dyn=None,
               stream=None):
    """Spawn densification: out = input rows + m·K children (n_out = n + m·K)."""
    n = pos_opa.shape[0]
    _check(lib().dass_spawn(n, int(sh_degree), _ptr(pos_opa), _ptr(scale), _ptr(rot), _ptr(sh),
                            _ptr(dyn), int(m), _ptr(idx), int(spawn_count), float(scale_shrink),
                            float(child_opacity), C.c_uint64(int(seed)), _ptr(out_pos_opa),
                            _ptr(out_scale), _ptr(out_rot), _ptr(out_sh), _ptr(out_dyn),
                            _stream(stream)), "dass_spawn")


def dass_prune_select(pos_opa, first, min_opacity, keep, idx, counts, ws, stream=None):
    n = pos_opa.shape[0]
    _check(lib().dass_prune_select(n, int(first), _ptr(pos_opa), float(min_opacity), _ptr(keep),
                                   _ptr(idx), _ptr(counts), _ptr(ws), _ws_bytes(ws),
                                   _stream(stream)), "dass_prune_select")


def dass_gather(sh_degree, pos_opa, scale, rot, sh, dyn, m, idx, out_pos_opa, out_scale, out_rot,
                out_sh, out_dyn=None, stream=None):
    n = pos_opa.shape[0]
    _check(lib().dass_gather(n, int(sh_degree), _ptr(pos_opa), _ptr(scale), _ptr(rot), _ptr(sh),
                             _ptr(dyn), int(m), _ptr(idx), _ptr(out_pos_opa), _ptr(out_scale),
                             _ptr(out_rot), _ptr(out_sh), _ptr(out_dyn), _stream(stream)),
           "dass_gather")


def dass_render_features(cam, ranges, sorted_ids, xy_depth, conic_opa, box, feat, out, stream=None):
    """Eq. 9: out [C][H][W] from features feat [n][C]."""
    c = _cam(cam)
    _check(lib().dass_render_features(C.byref(c), _ptr(ranges), _ptr(sorted_ids), _ptr(xy_depth),
                                      _ptr(conic_opa), _ptr(box), int(feat.shape[1]), _ptr(feat),
                                      _ptr(out), _stream(stream)), "dass_render_features")
