"""A/B timing of single sweeps (tuning driver, not a bench line):
    python profiles/ab_sweep.py c5 <group> VAR=v1,v2,... [VAR2=...]
For each combination of the environment overrides, times every scale of the
group's requests (device outputs, CUDA events, L2 flushed before each
launch, median of 5) and checks the maps are bit-identical across
combinations."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1705_03524_b200 import swg  # noqa: E402

cfg, group = sys.argv[1], sys.argv[2]
axes = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[3:]]
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
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
models = [bench.make_models(ctx, wl, data)[gi][i] for i in sel]
dev = torch.from_numpy(data.image).cuda()
if g.get("decay"):
    t = ctx.build_decay(dev, g["decay"], wl["fmt"], wl["bins"])
else:
    t = ctx.build(dev, wl["fmt"], wl["bins"], g["planes"])
reqs = [swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings)
        for (k, meth, rings, _), m in zip(g["scales"], models)]
maps = [torch.empty(t.map_shape(r.kernel), dtype=torch.float64, device="cuda") for r in reqs]
peaks = torch.zeros(len(reqs), 3, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref_maps = None
for combo in itertools.product(*[v for _, v in axes]):
    for (name, _), val in zip(axes, combo):
        os.environ[name] = val
    times = []
    for i, r in enumerate(reqs):
        ts = []
        for rep in range(6):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t.likelihood_maps([r], scores="none", scores_dev=[maps[i]], peaks_dev=peaks[i])
            e1.record()
            torch.cuda.synchronize()
            if rep:
                ts.append(e0.elapsed_time(e1))
        times.append(sorted(ts)[len(ts) // 2])
    cur = [m.cpu().numpy().copy() for m in maps]
    same = ref_maps is None or all((a.view("i8") == b.view("i8")).all() for a, b in zip(cur, ref_maps))
    ref_maps = ref_maps or cur
    label = " ".join(f"{n}={v}" for (n, _), v in zip(axes, combo))
    print(f"{label:40s} total {sum(times):7.3f} ms  " +
          " ".join(f"{r.kernel.kw}:{x:.3f}" for r, x in zip(reqs, times)) +
          ("" if same else "  MAPS DIFFER"), flush=True)
