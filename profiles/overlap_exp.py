"""Experiment: config 5's table sets swept on separate contexts / streams at
once (the L1-bound cake beside the HBM-bound stream and exponential sweeps)
against one after the other.
    python profiles/overlap_exp.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1705_03524_b200 import swg  # noqa: E402

wl = bench.workload("c5")
data = wl["gen"](1)
ctx0 = swg.Context(0)
models = bench.make_models(ctx0, wl, data)
frame = torch.from_numpy(data.image).cuda()
sets = []
for gi, g in enumerate(wl["groups"]):
    ctx = swg.Context(0)
    st = torch.cuda.Stream()
    ctx.set_stream(st.cuda_stream)
    t = (ctx.build_decay(frame, g["decay"], wl["fmt"], wl["bins"]) if g.get("decay")
         else ctx.build(frame, wl["fmt"], wl["bins"], g["planes"]))
    reqs = [swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings)
            for (k, meth, rings, _), m in zip(g["scales"], models[gi])]
    maps = [torch.empty(t.map_shape(r.kernel), dtype=torch.float64, device="cuda") for r in reqs]
    peaks = torch.zeros(len(reqs), 3, dtype=torch.float64, device="cuda")
    sets.append((ctx, st, t, reqs, maps, peaks))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run(order, concurrent, builds):
    ts = []
    for rep in range(6):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream()
        e0.record(main)
        evs = []
        for i in order:
            ctx, st, t, reqs, maps, peaks = sets[i]
            st.wait_event(e0)
            if not concurrent and evs:
                st.wait_event(evs[-1])
            if builds:
                t.rebuild_for(frame, reqs)
            t.likelihood_maps(reqs, scores="none", scores_dev=maps, peaks_dev=peaks)
            ev = torch.cuda.Event()
            ev.record(st)
            evs.append(ev)
        for ev in evs:
            main.wait_event(ev)
        e1.record(main)
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for builds in (False, True):
    for order in ((0, 1, 2), (1, 0, 2), (1, 2, 0)):
        print("builds" if builds else "sweeps", order, "sequential %.3f ms" % run(order, False, builds),
              "concurrent %.3f ms" % run(order, True, builds), flush=True)
