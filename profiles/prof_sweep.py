"""Profiling driver for single sweeps of a config's timed step:
    ncu ... python profiles/prof_sweep.py c5 <group> <kw,kw,...> [reps]
group: manhattan | gauss | euclid | exp (config 5's table groups) or c2 / c4.
Builds the group's tables once, then runs each listed scale's request
(device outputs, as the timed step) `reps` times (default 1), one launch
per request in order; a 5th argument "joint" sends them in one call (the
multi-scale cake groups the library forms, as in the timed step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1705_03524_b200 import swg  # noqa: E402

cfg, group = sys.argv[1], sys.argv[2]
want = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
joint = len(sys.argv) > 5 and sys.argv[5] == "joint"
wl = bench.workload(cfg)
KIND = {"manhattan": swg.MANHATTAN, "gauss": swg.GAUSS_CHEB, "euclid": swg.EUCLID_QUAD,
        "exp": swg.EXP_L1}
gi = next((i for i, g_ in enumerate(wl["groups"])
           if any(k.kind == KIND.get(group, -1) for k, _, _, _ in g_["scales"])), 0)
g = dict(wl["groups"][gi])
sel = [i for i, (k, _, _, _) in enumerate(g["scales"])
       if group not in KIND or k.kind == KIND[group]]
g["scales"] = [g["scales"][i] for i in sel]
data = wl["gen"](1)
ctx = swg.Context(0)
models = [bench.make_models(ctx, wl, data)[gi][i] for i in sel]
dev = torch.from_numpy(data.image).cuda()
if g.get("decay"):
    t = ctx.build_decay(dev, g["decay"], wl["fmt"], wl["bins"])
else:
    t = ctx.build(dev, wl["fmt"], wl["bins"], g["planes"])
reqs, maps = [], []
for (k, meth, rings, _), m in zip(g["scales"], models):
    if want and k.kw not in want:
        continue
    reqs.append(swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings))
    maps.append(torch.empty(t.map_shape(k), dtype=torch.float64, device="cuda"))
peaks = torch.zeros(len(reqs), 3, dtype=torch.float64, device="cuda")
for _ in range(reps):
    if joint:
        t.likelihood_maps(reqs, scores="none", scores_dev=maps, peaks_dev=peaks)
        continue
    for i, r in enumerate(reqs):
        t.likelihood_maps([r], scores="none", scores_dev=[maps[i]], peaks_dev=peaks[i])
ctx.synchronize()
print("ok", [r.kernel.kw for r in reqs])
