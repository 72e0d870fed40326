"""Per-view timeline of the 20-view fwd+bwd pass as bench.py runs it (one stream per
view, captured in a CUDA graph): dass_timestamp kernels on each view's stream around
bin_sort, render_fwd and render_bwd_raster, relative to the pass start.
usage (GPU): python tools/timeline.py [streams]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2411_14847_b200 import dass, synth  # noqa: E402
from paper_2411_14847_b200.pipeline import DeviceScene, Raster, ViewRecords  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 20
CH = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # sort chains (0: sort on the view streams)
SPLIT = (int(sys.argv[3]) if len(sys.argv) > 3 else 1) == 1   # records part on a side stream
cams, sc = synth.c3()
ds = DeviceScene.from_host(sc, "cuda")
V = len(cams)
rec = ViewRecords(V, sc.n, "cuda")
dLs = torch.stack([torch.from_numpy(synth.grad_image(c, 1000 + v)) for v, c in enumerate(cams)]).cuda()
slots = [Raster(c.width, c.height, sc.n, 1 << 22, "cuda") for c in cams[:S]]
streams = [torch.cuda.Stream() for _ in range(S)]
sstreams = [torch.cuda.Stream(priority=-5) for _ in range(CH)]
g2d = torch.empty(V, sc.n, 12, device="cuda")
stamps = torch.zeros(4 + 4 * V, dtype=torch.int64, device="cuda")   # [3 + 4V]: records done
rstream = torch.cuda.Stream()


def run():
    main = torch.cuda.current_stream()
    dass.dass_timestamp(stamps, 0, main)
    outs = (rec.xy_depth, rec.conic_opa, rec.rgb, rec.box, rec.rows, rec.tiles)
    dass.dass_project_views_part(dass.DASS_PROJECT_KEYS if SPLIT else dass.DASS_PROJECT_ALL, cams,
                                 sc.sh_degree, ds.pos_opa, ds.scale, ds.rot, ds.sh, None, *outs)
    dass.dass_timestamp(stamps, 1, main)
    rdone = torch.cuda.Event()
    if SPLIT:
        rstream.wait_stream(main)
        with torch.cuda.stream(rstream):
            dass.dass_project_views_part(dass.DASS_PROJECT_RECORDS, cams, sc.sh_degree, ds.pos_opa,
                                         ds.scale, ds.rot, ds.sh, None, *outs)
    dass.dass_timestamp(stamps, 3 + 4 * V, rstream if SPLIT else main)
    rdone.record(rstream if SPLIT else main)
    for v, cam in enumerate(cams):
        k = v % S
        r, st = slots[k], streams[k]
        st.wait_stream(main)
        xy, co, rgb, box, rows, tt = rec.view(v)
        ss = sstreams[v % CH] if CH else st
        if CH:
            ss.wait_stream(st)
        with torch.cuda.stream(ss):
            dass.dass_timestamp(stamps, 3 + 4 * v, ss)
            dass.dass_bin_sort(cam, sc.n, xy, box, rows, tt, r.sort_ws, r.capacity, None, r.sorted_ids,
                               r.ranges, r.num_pairs)
            dass.dass_timestamp(stamps, 4 + 4 * v, ss)
        if CH:
            st.wait_stream(ss)
        with torch.cuda.stream(st):
            st.wait_event(rdone)
            dass.dass_render_fwd(cam, r.ranges, r.sorted_ids, xy, co, rgb, box, None, r.img, r.T,
                                 r.last, r.accept, r.capacity)
            dass.dass_timestamp(stamps, 5 + 4 * v, st)
            dass.dass_render_bwd_raster(cam, sc.n, r.ranges, r.sorted_ids, xy, co, rgb, box, None,
                                        r.T, r.last, dLs[v], g2d[v], r.accept, r.capacity)
            dass.dass_timestamp(stamps, 6 + 4 * v, st)
    for st in streams + sstreams + [rstream]:
        main.wait_stream(st)
    dass.dass_timestamp(stamps, 2, main)


run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
t = stamps.cpu().numpy().astype("float64")
t0 = t[0]
ms = lambda x: (x - t0) / 1e6
print(f"project (keys{' only' if SPLIT else ' + records'}) {ms(t[1]):.3f} ms, records done "
      f"{ms(t[3 + 4 * V]):.3f} ms, pass {ms(t[2]):.3f} ms")
print(" view  sort_start  sort_end  fwd_end  bwd_end   sort_ms  fwd_ms  bwd_ms  (ms from pass start)")
for v in range(V):
    a, b, c, d = (ms(t[3 + 4 * v + i]) for i in range(4))
    print(f"  {v:3d}  {a:8.3f}  {b:8.3f}  {c:8.3f}  {d:8.3f}   {b - a:6.3f}  {c - b:6.3f}  {d - c:6.3f}")
