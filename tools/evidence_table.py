"""Print the numbers BASELINE.md §3 / README / DESIGN quote from the committed bench lines.
usage: python tools/evidence_table.py [profiles/r02_bench_c1.json ...]"""
import json
import sys

files = sys.argv[1:] or [f"profiles/r02_bench_{c}.json" for c in ("c1", "c2", "c3", "c4", "c5")] + [
    "profiles/r02_bench_c3_emulate_0of8_nccl1.json"]
for f in files:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    o = r.get("other_raster_kernel") or {}
    h, st = d.get("hot_path_roofline") or {}, d.get("scene_stats") or {}
    g = lambda x, *k: (lambda v: v)(__import__("functools").reduce(lambda a, b: (a or {}).get(b), k, x))
    print(f, "| value", d["value"], "ms", d["ms_per_step"], "e2e", round((d.get("e2e") or {}).get("value", 0), 1),
          "mpix", d.get("mpix_per_s"), "| fwd", r.get("frac"), g(r, "in_step", "frac"), r.get("kernel", "")[:22],
          "| other", o.get("frac"), g(o, "in_step", "frac"), "| proj GB/s", g(h, "project_views", "achieved_gbs"),
          "pre", g(h, "render_bwd_preprocess_views", "achieved_gbs"), "| K", st.get("K_per_view_mean"),
          "Pf", st.get("P_fwd_per_px"), "Pb", st.get("P_bwd_per_px"), "| cpu", g(d, "cpu_baseline", "value"),
          "| ar", g(d, "allreduce", "ms"), "| clocks", g(d, "clocks", "sm_mhz"), g(d, "clocks", "reasons"))
