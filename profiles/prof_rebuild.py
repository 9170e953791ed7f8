"""Profiling driver for config 5's model-driven rebuilds (the bench step's
builds): builds the three table sets in full once, then runs
swg_tables_rebuild_for with the step's requests -- quadratic set first,
then the decayed set, then the 16-bit plain set -- `reps` times.
    ncu -k regex:"k_build_fused<unsigned int, 8>|k_build_decay_warp" --launch-skip 4 -c 2 \\
        python profiles/prof_rebuild.py
(skips the initial decayed build's four strip launches: the capture is the
selective quadratic build and the first selective decayed orientation)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1705_03524_b200 import swg  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
wl = bench.workload("c5")
data = wl["gen"](1)
ctx = swg.Context(0)
models = bench.make_models(ctx, wl, data)
frame = torch.from_numpy(data.image).cuda()
sets = []
for gi, g in enumerate(wl["groups"]):
    t = (ctx.build_decay(frame, g["decay"], wl["fmt"], wl["bins"]) if g.get("decay")
         else ctx.build(frame, wl["fmt"], wl["bins"], g["planes"]))
    reqs = [swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings)
            for (k, meth, rings, _), m in zip(g["scales"], models[gi])]
    sets.append((g, t, reqs))
order = sorted(sets, key=lambda s: (0 if s[0]["planes"] == swg.PLANES_QUADRATIC else
                                    1 if s[0].get("decay") else 2))
for _ in range(reps):
    for g, t, reqs in order:
        t.rebuild_for(frame, reqs)
ctx.synchronize()
print("ok", [t.built_bytes() for _, t, _ in order])
