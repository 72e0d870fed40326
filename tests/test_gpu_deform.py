"""GPU parity of f2 (dual hash-grid deformation, §3.3, §B P:398-399;
readings A41-A43) and the dynamic/static partition, through the C-ABI, against
the CPU oracle on the same seeded inputs.

Bars (A43):
  * partition: bit-exact (indices and counts);
  * μ, σ − e_w: |Δ| ≤ 1e-4·max|ref| (fp32 dot products of length ≤ 64 against
    fp64; ReLU is continuous, so a near-zero pre-activation cannot move the output);
  * ∂L/∂table, ∂L/∂mlp: |Δ| ≤ 1e-3·|ref| + 1e-5·κ + 1e-5·max|ref|, κ = Σ|terms|
    of the same sum (the A37 form; the last term covers cell assignment at fp32
    rounding of a lattice boundary), over Gaussians with no ReLU tie (oracle tie flag: a
    pre-activation within 1e-5·(1 + Σ|terms|) of 0, where fp32 may take the other
    side and flip a whole gradient term).
"""
import numpy as np
import pytest

import oracle
from paper_2411_14847_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_14847_b200 import dass  # noqa: E402

DEV = "cuda"
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
np_ = lambda x: x.detach().cpu().numpy()


def partition(mask):
    n = mask.shape[0]
    idx_d = torch.full((max(n, 1),), -1, dtype=torch.int32, device=DEV)
    idx_s = torch.full((max(n, 1),), -1, dtype=torch.int32, device=DEV)
    counts = torch.zeros(2, dtype=torch.int32, device=DEV)
    ws = torch.empty(dass.dass_partition_workspace(n) // 4 + 1, dtype=torch.int32, device=DEV)
    dass.dass_partition(t(mask.astype(np.uint8)), idx_d, idx_s, counts, ws)
    torch.cuda.synchronize()
    return idx_d, idx_s, counts


@pytest.mark.parametrize("n", [0, 1, 1000, 1024, 300_001])
def test_partition_bit_exact(n):
    mask = (np.random.default_rng(n).uniform(size=n) < 0.3).astype(np.uint8)
    if n > 10:
        mask[:5] = 1; mask[-3:] = 0
    idx_d, idx_s, counts = partition(mask)
    dyn, st = np.flatnonzero(mask), np.flatnonzero(mask == 0)
    c = np_(counts)
    assert c[0] == dyn.size and c[1] == st.size
    assert np.array_equal(np_(idx_d)[:dyn.size], dyn)
    assert np.array_equal(np_(idx_s)[:st.size], st)


def device_field(f):
    return t(f.table), t(f.mlp)


def run_fwd(f, pos_d, idx, count=None, n=None):
    N = pos_d.shape[0]
    mu = torch.full((N, 4), np.nan, device=DEV)
    sg = torch.full((N, 4), np.nan, device=DEV)
    tab, mlp = device_field(f)
    dass.dass_deform_fwd(f, tab, mlp, pos_d, mu, sg, idx=idx, count=count, n=n)
    torch.cuda.synchronize()
    return np_(mu), np_(sg)


def check_fwd(mu, sg, rmu, rsg):
    e = np.array([1.0, 0, 0, 0])
    assert np.max(np.abs(mu - rmu)) <= 1e-4 * np.max(np.abs(rmu)) + 1e-9
    assert np.max(np.abs((sg - e) - (rsg - e))) <= 1e-4 * np.max(np.abs(rsg - e)) + 1e-9


def check_grad(a, ref, kap):
    # + 1e-5·max|ref|: a position within fp32 rounding of a lattice-cell boundary
    # may be assigned to the neighbouring cell (trilinear weight error ≤ N_l·2⁻²²
    # ≈ 6e-5 at N = 256), which moves ≤ 6e-5·|∂L/∂feat| onto a corner the oracle
    # gives (almost) nothing.
    bad = np.abs(a - ref) > 1e-3 * np.abs(ref) + 1e-5 * kap + 1e-5 * np.max(np.abs(ref)) + 1e-12
    assert not bad.any(), (int(bad.sum()), float(np.max(np.abs(a - ref))), float(np.max(np.abs(ref))))


@pytest.fixture(params=["default"])
def fwd_path(request):
    """The library's own choice per field shape: the tcgen05 3×TF32 kernels
    where K is a multiple of 8 (the backward's tcgen05 kernel serves F = 4), the
    FP32 SIMT kernels otherwise (test_other_field_shapes covers those)."""
    return request.param


@pytest.mark.parametrize("profile", ["n3dv", "meetroom"])
def test_dual_fields_forward_through_partition(profile, fwd_path):
    """Both fields over one partition (device counts), several persistent tiles
    per CTA (60k Gaussians) and a ragged tail; rows outside a group untouched."""
    sc = synth.n3dv_scene(n=60_000, seed=71, degree=0)
    fd, fs = synth.dual_fields(sc, profile, seed=72)
    idx_d, idx_s, counts = partition(sc.dynamic)
    pos = t(sc.pos_opa)
    mu = torch.full((sc.n, 4), np.nan, device=DEV)
    sg = torch.full((sc.n, 4), np.nan, device=DEV)
    for f, idx, c in ((fd, idx_d, counts[0:1]), (fs, idx_s, counts[1:2])):
        tab, mlp = device_field(f)
        dass.dass_deform_fwd(f, tab, mlp, pos, mu, sg, idx=idx, count=c, n=sc.n)
    torch.cuda.synchronize()
    mu, sg = np_(mu), np_(sg)
    assert np.isfinite(mu).all() and np.isfinite(sg).all()       # every row written once
    dyn = sc.dynamic.astype(bool)
    for f, rows in ((fd, np.flatnonzero(dyn)), (fs, np.flatnonzero(~dyn))):
        rmu, rsg, _ = oracle.deform(f, sc.pos_opa[rows])
        check_fwd(mu[rows], sg[rows], rmu, rsg)


def test_identity_at_initialisation(fwd_path):
    sc = synth.n3dv_scene(n=5000, seed=73, degree=0)
    fd, _ = synth.dual_fields(sc, "n3dv", seed=74, trained=False)
    mu, sg = run_fwd(fd, t(sc.pos_opa), None)
    assert np.all(mu == 0) and np.all(sg == np.array([1.0, 0, 0, 0], np.float32))


@pytest.mark.parametrize("profile,n", [("n3dv", 60_000), ("meetroom", 9_000)])
def test_backward_parity(profile, n, fwd_path):
    sc = synth.n3dv_scene(n=n, seed=75, degree=0)
    fd, fs = synth.dual_fields(sc, profile, seed=76)
    gm, gs = synth.offset_grads(sc.n, 77, scale=1e-3)
    pos = t(sc.pos_opa)
    dyn = sc.dynamic.astype(bool)
    for f, rows in ((fd, np.flatnonzero(dyn)), (fs, np.flatnonzero(~dyn))):
        _, _, tie = oracle.deform(f, sc.pos_opa[rows])
        rows = rows[tie == 0]
        gt_ref, gp_ref, kt, km = oracle.deform_bwd(f, sc.pos_opa[rows], gm[rows], gs[rows], kappa=True)
        tab, mlp = device_field(f)
        g_tab = torch.zeros_like(tab)
        g_mlp = torch.zeros_like(mlp)
        idx = t(rows.astype(np.int32))
        dass.dass_deform_bwd(f, tab, mlp, pos, t(gm), t(gs), g_tab, g_mlp, idx=idx)
        torch.cuda.synchronize()
        check_grad(np_(g_tab).astype(np.float64), gt_ref, kt)
        check_grad(np_(g_mlp).astype(np.float64), gp_ref, km)
        # accumulation semantics: a second call adds the same amount again
        dass.dass_deform_bwd(f, tab, mlp, pos, t(gm), t(gs), g_tab, g_mlp, idx=idx)
        torch.cuda.synchronize()
        check_grad(np_(g_mlp).astype(np.float64), 2 * gp_ref, 2 * km)


def test_full_size_forward_sampled_and_empty_group(fwd_path):
    """C3-sized (300k Gaussians, N3DV profile): sampled rows against the oracle;
    a count of 0 writes nothing."""
    sc = synth.n3dv_scene(n=300_000, seed=3, degree=0)
    fd, fs = synth.dual_fields(sc, "n3dv", seed=40)
    idx_d, idx_s, counts = partition(sc.dynamic)
    pos = t(sc.pos_opa)
    mu = torch.full((sc.n, 4), np.nan, device=DEV)
    sg = torch.full((sc.n, 4), np.nan, device=DEV)
    for f, idx, c in ((fd, idx_d, counts[0:1]), (fs, idx_s, counts[1:2])):
        tab, mlp = device_field(f)
        dass.dass_deform_fwd(f, tab, mlp, pos, mu, sg, idx=idx, count=c, n=sc.n)
    zero = torch.zeros(1, dtype=torch.int32, device=DEV)
    tab, mlp = device_field(fd)
    before = mu.clone()
    dass.dass_deform_fwd(fd, tab, mlp, pos, mu, sg, idx=idx_d, count=zero, n=sc.n)
    torch.cuda.synchronize()
    assert torch.equal(before, mu)
    mu, sg = np_(mu), np_(sg)
    rng = np.random.default_rng(78)
    dyn = sc.dynamic.astype(bool)
    for f, rows in ((fd, np.flatnonzero(dyn)), (fs, np.flatnonzero(~dyn))):
        s = np.sort(rng.choice(rows, 3000, replace=False))
        rmu, rsg, _ = oracle.deform(f, sc.pos_opa[s])
        check_fwd(mu[s], sg[s], rmu, rsg)


def test_invalid_config_rejected():
    sc = synth.n3dv_scene(n=100, seed=79, degree=0)
    fd, _ = synth.dual_fields(sc, "n3dv", seed=80)
    tab, mlp = device_field(fd)
    pos = t(sc.pos_opa)
    mu = torch.empty(sc.n, 4, device=DEV); sg = torch.empty(sc.n, 4, device=DEV)
    bad = dass.hashgrid_struct(fd)
    bad.levels = 7          # in = 7·2 = 14: not a multiple of 4
    bad.features = 2
    with pytest.raises(dass.DassError):
        dass.dass_deform_fwd(bad, tab, mlp, pos, mu, sg)
    bad = dass.hashgrid_struct(fd)
    bad.aabb_max[0] = bad.aabb_min[0]
    with pytest.raises(dass.DassError):
        dass.dass_deform_fwd(bad, tab, mlp, pos, mu, sg)


@pytest.mark.parametrize("levels,log2T,F", [(16, 12, 4), (4, 10, 1), (6, 11, 2), (12, 9, 4)])
def test_other_field_shapes(levels, log2T, F, fwd_path):
    """Configurations beyond the N3DV/Meet-Room profiles: in = 64 (the largest
    MLP input; SIMT backward), F = 1, and odd level counts, with ragged tiles."""
    sc = synth.n3dv_scene(n=3_001, seed=90 + levels, degree=0)
    box = synth.scene_aabb(sc.pos_opa)
    res = tuple(int(round(8 * 1.4 ** l)) for l in range(levels))
    f = synth.hash_field(log2T, F, box, seed=91, levels=levels, res=res)
    pos = t(sc.pos_opa)
    mu, sg = run_fwd(f, pos, None)
    rmu, rsg, tie = oracle.deform(f, sc.pos_opa)
    check_fwd(mu, sg, rmu, rsg)
    gm, gs = synth.offset_grads(sc.n, 92, scale=1e-3)
    rows = np.flatnonzero(tie == 0)
    gt_ref, gp_ref, kt, km = oracle.deform_bwd(f, sc.pos_opa[rows], gm[rows], gs[rows], kappa=True)
    tab, mlp = device_field(f)
    g_tab = torch.zeros_like(tab); g_mlp = torch.zeros_like(mlp)
    dass.dass_deform_bwd(f, tab, mlp, pos, t(gm), t(gs), g_tab, g_mlp, idx=t(rows.astype(np.int32)))
    torch.cuda.synchronize()
    check_grad(np_(g_tab).astype(np.float64), gt_ref, kt)
    check_grad(np_(g_mlp).astype(np.float64), gp_ref, km)
