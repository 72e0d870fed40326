"""bench.py's host-side logic (no GPU): the §8(f) roofline bookkeeping."""
import bench


def test_rows_roofline_fractions():
    ops = {"fidelity_loss": 2.5, "deform_fwd": 0.15, "deform_bwd": 0.7}
    densify = {"kept_after_prune": 300_000,
               "ms": {"gather": 0.03, "render_features_16ch_one_view": 0.6}}
    allst = {"accepted": [65_000_000]}
    pk = {"hbm_gbs": 6400.0, "bf16_tflops": 1600.0}
    out = bench.rows_roofline(ops, densify, allst, pk, 74.4, 300_000, 1352, 1014, 20, 3)
    assert set(out) == {"f1_fidelity_loss", "f2_deform_fwd_tcgen05", "f2_deform_bwd_simt",
                        "f4_gather", "f4_render_features"}
    for v in out.values():
        assert 0 < v["frac"] < 1
    # f4 gather: 2 × rows × (48 + 16·K4) bytes at SH3 (K4 = 12)
    g = out["f4_gather"]
    assert abs(g["achieved_gbs"] - 2 * 300_000 * 240 / 0.03e-3 / 1e9) < 1.0
    assert out["f2_deform_fwd_tcgen05"]["peak_tflops"] == 800.0


def test_hot_path_roofline():
    ops = {"project_views": 0.62, "bin_sort": 4.0, "render_fwd": 8.0, "render_bwd_raster": 7.9,
           "render_bwd_preprocess_views": 0.44}
    stats = {"K": [2_100_000] * 20, "accepted": [65_000_000] * 20, "P_fwd": [215_000_000] * 20}
    out = bench.hot_path_roofline(ops, stats, {"hbm_gbs": 6400.0}, 74.4, 300_000, 20, 3)
    assert set(out) == set(ops)
    for v in out.values():
        assert 0 < v["frac"] < 1
    # the backward's flop count is 42 per accepted unit
    assert out["render_bwd_raster"]["flop"] == 42 * 65_000_000 * 20
    assert bench.hot_path_roofline({}, stats, {}, 74.4, 1, 1, 0) is None


def test_dominant_roofline_picks_the_slower_raster_kernel():
    """Headline in SURVEY §8(d)'s unit: P (evaluated (pixel, entry)) × FP32-pipe
    instructions per unit (20 forward, 55 backward) over the FP32 pipe's issue
    peak 148 × 128 × f; the builder's flop count is the secondary view."""
    stats = {"accepted": [65_000_000] * 20, "P_fwd": [215_000_000] * 20, "P_bwd": [210_000_000] * 20}
    f = 1965e6
    peak = bench.SM_COUNT * bench.FP32_LANES * 2 * f / 1e12
    peak_i = bench.SM_COUNT * bench.FP32_LANES * f / 1e12
    fwd = bench.dominant_roofline({"render_fwd": 7.9, "render_bwd_raster": 6.7}, stats, f, peak)
    assert fwd["kernel"].startswith("render_fwd") and fwd["unit"] == "Tinstr/s"
    assert abs(fwd["achieved"] - 215e6 * 20 * 20 / 7.9e-3 / 1e12) < 1e-2
    assert abs(fwd["peak"] - peak_i) < 1e-2 and abs(fwd["frac"] - fwd["achieved"] / fwd["peak"]) < 1e-3
    fl = (bench.FLOP_FWD_ACCEPTED * 65e6 + bench.FLOP_FWD_INBOX * 215e6) * 20
    assert abs(fwd["algorithmic_flop_view"]["achieved_tflops"] - fl / 7.9e-3 / 1e12) < 0.01
    bwd = bench.dominant_roofline({"render_fwd": 6.0, "render_bwd_raster": 6.7}, stats, f, peak)
    assert bwd["kernel"].startswith("render_bwd")
    assert abs(bwd["achieved"] - 210e6 * 20 * 55 / 6.7e-3 / 1e12) < 1e-2
    assert abs(bwd["algorithmic_flop_view"]["achieved_tflops"]
               - bench.FLOP_BWD_ACCEPTED * 65e6 * 20 / 6.7e-3 / 1e12) < 0.01
    assert bench.dominant_roofline({}, stats, f, peak) is None


def test_issue_view_reads_the_committed_profile():
    import os
    if not os.path.exists(os.path.join(os.path.dirname(bench.__file__), "profiles",
                                       f"{bench.PROFILE_TAG}_ncu_render_fwd.txt")):
        import pytest
        pytest.skip("this round's ncu summary is not committed yet")
    v = bench.issue_view("render_fwd", 7.4, 20, 1965e6)
    instr = bench.profiled_instructions("render_fwd")
    assert instr and instr > 1e8
    assert abs(v["frac"] - instr * 20 / 7.4e-3 / (148 * 4 * 1965e6)) < 1e-3
    assert 0 < v["frac"] < 1
    assert bench.issue_view("no_such_kernel", 7.4, 20, 1965e6) is None


def test_fair_share_attribution():
    """roofline.in_step: every interval between stamps is split evenly over the views'
    phases running in it; the attributed times add up to the pass."""
    import numpy as np
    # views 0, 1: sort [0, 1), forward [1, 5), backward [5, 9); view 2's forward runs
    # late, until 8, under the other two backward kernels, and its backward until 10
    t = np.array([[0, 1, 5, 9], [0, 1, 5, 9], [0, 1, 8, 10]], dtype=np.float64)
    out = bench.fair_share(t)
    assert out["sort"] == 1.0
    assert abs(out["render_fwd"] - (4.0 + 3.0 / 3)) < 1e-12
    assert abs(out["render_bwd_raster"] - (3.0 * 2 / 3 + 1.0 + 1.0)) < 1e-12
    assert abs(sum(out.values()) - 10.0) < 1e-12
