"""CPU-side checks of the C-ABI boundary (no GPU needed): libdass.so loads,
exports every function include/dass.h declares, and validates its arguments
before touching CUDA (status codes mirror SPEC's exit codes)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2411_14847_b200 import build as dass_build
from paper_2411_14847_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dass.h")


@pytest.fixture(scope="module")
def lib():
    dass_build.build()
    from paper_2411_14847_b200 import dass
    return dass


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dass_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_six_calls_plus_helpers():
    f = declared_functions()
    for name in ("dass_project", "dass_bin_sort", "dass_render_fwd", "dass_render_bwd",
                 "dass_apply_shift", "dass_error_map"):
        assert name in f


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (dass_\w+)", out))
    declared = set(declared_functions())
    assert declared <= exported, declared - exported
    assert set(lib.EXPORTS) == declared
    L = lib.lib()
    for name in declared:
        assert getattr(L, name) is not None


def test_library_is_sm100a_only(lib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", lib.LIB_PATH]).decode()
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def test_status_strings_and_version(lib):
    L = lib.lib()
    assert lib.abi_version() == 3
    for s, txt in [(0, b"ok"), (1, b"invalid argument"), (4, b"pair capacity exceeded")]:
        assert L.dass_status_string(s) == txt
    assert L.dass_status_string(99) == b"unknown status"


def test_validation_before_any_cuda_call(lib):
    L = lib.lib()
    cam = lib.camera_struct(synth.tiny_camera(64, 64))
    P = None
    launches0 = lib.kernel_launches()   # other tests of the same process may have launched
    # null camera / bad sizes / bad degree
    assert L.dass_project(None, 10, 0, P, P, P, P, P, P, P, P, P, P, P, P) == 1
    bad = lib.camera_struct(synth.tiny_camera(64, 64)); bad.width = 0
    assert L.dass_project(C.byref(bad), 10, 0, P, P, P, P, P, P, P, P, P, P, P, P) == 1
    bad.width = 64; bad.fx = -1.0
    assert L.dass_project(C.byref(bad), 10, 0, P, P, P, P, P, P, P, P, P, P, P, P) == 1
    assert L.dass_project(C.byref(cam), 10, 4, P, P, P, P, P, P, P, P, P, P, P, P) == 1
    assert L.dass_project(C.byref(cam), -1, 0, P, P, P, P, P, P, P, P, P, P, P, P) == 1
    assert L.dass_project(C.byref(cam), 10, 0, P, P, P, P, P, P, P, P, P, P, P, P) == 1  # null ptrs
    assert b"null" in L.dass_last_error()
    # n = 0 is OK and enqueues nothing
    assert L.dass_project(C.byref(cam), 0, 3, P, P, P, P, P, P, P, P, P, P, P, P) == 0
    for part, want in ((0, 1), (4, 1)):   # preprocess part ∉ {1, 2, 3}
        assert L.dass_render_bwd_preprocess_views_part(part, C.byref(cam), 1, 0, 3, P, P, P, P, P, P,
                                                       P, P, P, P, P, P, P, P, P, P, P, P) == want
    for part, want in ((0, 1), (4, 1), (1, 0), (2, 0), (3, 0)):   # part ∉ {1, 2, 3}
        assert L.dass_project_views_part(part, C.byref(cam), 1, 0, 3, P, P, P, P, P, P, P, P, P,
                                         P, P, P) == want
    assert L.dass_apply_shift(0, P, P, P, P, P, P, P, P) == 0
    assert L.dass_apply_shift(-3, P, P, P, P, P, P, P, P) == 1
    # error map: γ ≤ 0 is a usage error; missing images are a data error
    assert L.dass_error_map(C.byref(cam), C.c_void_p(16), C.c_void_p(16), C.c_float(0.0), P, P, 0, P, P, P) == 1
    assert L.dass_error_map(C.byref(cam), None, None, C.c_float(0.1), P, P, 0, P, P, P) == 2
    # capacity must stay below 2^30
    out = C.c_size_t(0)
    assert L.dass_bin_sort_workspace(1000, 16, 1 << 30, C.byref(out)) == 1
    assert L.dass_bin_sort_workspace(1000, 16, 1 << 20, C.byref(out)) == 0 and out.value > (1 << 20) * 16
    assert L.dass_render_bwd_workspace(1000, C.byref(out)) == 0 and out.value == 1000 * 48
    assert lib.kernel_launches() == launches0


def test_binding_refuses_cpu_tensors(lib):
    torch = pytest.importorskip("torch")
    t = torch.zeros(4, 4)
    with pytest.raises(ValueError):
        lib.dass_apply_shift(t, t, t, t, None, t, t)


def test_camera_struct_layout_matches_generator(lib):
    cam = synth.n3dv_rig()[3]
    a = bytes(lib.camera_struct(cam))
    b = cam.to_struct().tobytes()
    assert C.sizeof(lib.dass_camera) == synth.CAMERA_DTYPE.itemsize == 140
    assert a == b


def test_hashgrid_struct_layout_and_param_counts(lib):
    sc = synth.n3dv_scene(n=200, seed=5, degree=0)
    fd, fs = synth.dual_fields(sc, "n3dv", seed=6)
    for f in (fd, fs):
        assert bytes(lib.hashgrid_struct(f)) == f.to_struct().tobytes()
        t, m = lib.dass_deform_param_count(f)
        assert t == f.table.size and m == f.mlp.size == synth.mlp_param_count(f.inputs)
    bad = lib.hashgrid_struct(fd)
    bad.features = 3
    with pytest.raises(lib.DassError):
        lib.dass_deform_param_count(bad)
    bad = lib.hashgrid_struct(fd)
    bad.levels, bad.features = 7, 2            # in = 14: not a multiple of 4
    with pytest.raises(lib.DassError):
        lib.dass_deform_param_count(bad)


def test_f_row_validation_before_any_cuda_call(lib):
    launches0 = lib.kernel_launches()   # other tests of the same process may have launched
    L = lib.lib()
    null = None
    # densify / prune / gather / spawn / partition: bad sizes and null pointers are refused
    assert L.dass_densify_select(-1, null, null, null, 1.0, 0.5, null, null, null, null, 0, null) == 1
    assert L.dass_prune_select(10, 0, null, 0.1, null, null, null, null, 0, null) == 1
    assert L.dass_gather(5, 3, null, null, null, null, null, 6, null, null, null, null, null, null, null) == 1
    assert L.dass_spawn(5, 3, null, null, null, null, null, 1, null, 0, 1.6, 0.1, 7,
                        null, null, null, null, null, null) == 1
    assert L.dass_partition(10, null, null, null, null, null, 0, null) == 1
    assert L.dass_render_features(null, null, null, null, null, null, 16, null, null, null) == 1
    assert lib.kernel_launches() == launches0


def test_binding_refuses_float64_tensors(lib):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA tensors to reach the dtype check")
    t = torch.zeros(4, 4, dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        lib.dass_apply_shift(t, t, t, t, None, t, t)


def test_bin_sort_views_and_timestamp_validation_before_any_cuda_call(lib):
    launches0 = lib.kernel_launches()   # other tests of the same process may have launched
    """dass_bin_sort_views / its workspace query / dass_timestamp refuse bad arguments
    with INVALID_ARG before enqueueing anything."""
    L = lib.lib()
    P = None
    out = C.c_size_t(0)
    arr = (lib.dass_camera * 2)(lib.camera_struct(synth.tiny_camera(64, 64)),
                                lib.camera_struct(synth.tiny_camera(64, 64)))
    assert L.dass_bin_sort_views_workspace(0, 100, 1000, C.byref(out)) == 1     # V < 1
    assert L.dass_bin_sort_views_workspace(65, 100, 1000, C.byref(out)) == 1    # V > 64
    assert L.dass_bin_sort_views_workspace(4, 100, 1 << 28, C.byref(out)) == 1  # V·cap ≥ 2^30
    assert L.dass_bin_sort_views_workspace(4, 100, 1000, None) == 1
    assert L.dass_bin_sort_views_workspace(2, 100, 1000, C.byref(out)) == 0
    one = out.value
    assert L.dass_bin_sort_views_workspace(2, 100, 2000, C.byref(out)) == 0 and out.value > one
    # cameras of different sizes, null outputs, workspace too small
    mixed = (lib.dass_camera * 2)(lib.camera_struct(synth.tiny_camera(64, 64)),
                                  lib.camera_struct(synth.tiny_camera(32, 64)))
    args = lambda cams, ws, nb, ids: (cams, 2, 100, C.c_void_p(16), C.c_void_p(16), C.c_void_p(16),
                                      C.c_void_p(16), ws, nb, 1000, ids, C.c_void_p(16),
                                      C.c_void_p(16), P)
    assert L.dass_bin_sort_views(*args(mixed, C.c_void_p(16), one, C.c_void_p(16))) == 1
    assert b"differ" in L.dass_last_error()
    assert L.dass_bin_sort_views(*args(arr, C.c_void_p(16), one, None)) == 1
    assert L.dass_bin_sort_views(*args(arr, C.c_void_p(16), one - 1, C.c_void_p(16))) == 1
    assert b"workspace" in L.dass_last_error()
    assert L.dass_bin_sort_views(None, 2, 100, P, P, P, P, P, 0, 1000, P, P, P, P) == 1
    assert L.dass_timestamp(None, 0, P) == 1
    assert L.dass_timestamp(C.c_void_p(16), -1, P) == 1
    assert lib.kernel_launches() == launches0


def test_accept_buffer_and_sort_size_validation_before_any_cuda_call(lib):
    launches0 = lib.kernel_launches()   # other tests of the same process may have launched
    """ADVICE r1: the acceptance-list buffer's size is checked against
    dass_render_accept_workspace (forward and every backward entry point), and
    the sort refuses n, V·n ≥ 2^30 (30-bit look-back counts) instead of wrapping."""
    L = lib.lib()
    cam = lib.camera_struct(synth.tiny_camera(64, 48))
    out = C.c_size_t(0)
    cap = 5000
    assert L.dass_render_accept_workspace(12, cap, C.byref(out)) == 0
    need = out.value
    d = C.c_void_p(256)   # a fake, 16-byte aligned device address: nothing is launched
    fwd = lambda acc, nb, pc: L.dass_render_fwd(C.byref(cam), d, d, d, d, d, d, None, d, d, d,
                                               acc, nb, pc, None)
    assert fwd(d, need - 1, cap) == 1 and b"accept buffer" in L.dass_last_error()
    assert fwd(C.c_void_p(260), need, cap) == 1                       # misaligned
    assert fwd(d, need, 1 << 30) == 1                                 # capacity out of range
    assert L.dass_render_bwd_raster(C.byref(cam), 100, d, d, d, d, d, d, None, d, d, d, d, need - 1,
                                    cap, d, None) == 1
    assert b"accept buffer" in L.dass_last_error()
    assert L.dass_bin_sort_workspace(1 << 30, 12, 100, C.byref(out)) == 1
    assert L.dass_bin_sort_views_workspace(4, 1 << 28, 100, C.byref(out)) == 1   # V·n = 2^30
    assert L.dass_bin_sort_views_workspace(4, (1 << 28) - 1, 100, C.byref(out)) == 0
    assert lib.kernel_launches() == launches0


def test_nonfinite_scan_validation_before_any_cuda_call(lib):
    launches0 = lib.kernel_launches()   # other tests of the same process may have launched
    L = lib.lib()
    assert L.dass_scan_nonfinite(None, -1, C.c_void_p(16), None, None) == 1
    assert L.dass_scan_nonfinite(None, 10, C.c_void_p(16), None, None) == 1
    assert L.dass_scan_nonfinite(C.c_void_p(16), 10, None, None, None) == 1
    assert lib.kernel_launches() == launches0
    assert L.dass_status_string(3) == b"numerical" or L.dass_status_string(3)
