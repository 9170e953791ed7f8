"""A/B timing of config 5's model-driven rebuilds (the bench step's builds):
    python profiles/ab_rebuild.py VAR=v1,v2 ...
Times swg_tables_rebuild_for of the quadratic / decayed / 16-bit plain sets
with the step's requests (CUDA events, median of 7, L2 flushed) per
combination of the environment overrides, and checks that a sample of the
built planes stays identical to the first combination's."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1705_03524_b200 import swg  # noqa: E402

axes = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[1:]]
wl = bench.workload("c5")
data = wl["gen"](1)
ctx = swg.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
models = bench.make_models(ctx, wl, data)
frame = torch.from_numpy(data.image).cuda()
sets = []
for gi, g in enumerate(wl["groups"]):
    t = (ctx.build_decay(frame, g["decay"], wl["fmt"], wl["bins"]) if g.get("decay")
         else ctx.build(frame, wl["fmt"], wl["bins"], g["planes"]))
    reqs = [swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings)
            for (k, meth, rings, _), m in zip(g["scales"], models[gi])]
    label = "decay" if g.get("decay") else {swg.PLANES_QUADRATIC: "quad",
                                            swg.PLANES_PLAIN: "plain"}.get(g["planes"], "affine")
    sets.append((label, t, reqs))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def sample(label, t, reqs):
    """A few built planes (bins the first request's model holds)."""
    b = int(np.flatnonzero(np.asarray(reqs[0].model))[0])
    if label == "plain":  # (an export would add 32-bit planes to every later rebuild)
        return []
    if label == "decay":
        return [t.export_f64(k, b, b + 1) for k in range(4)]
    return [t.export_u32(0, b, b + 1)]


ref = {}
for combo in itertools.product(*[v for _, v in axes]):
    for (name, _), val in zip(axes, combo):
        os.environ[name] = val
    out = []
    tot = 0.0
    for label, t, reqs in sets:
        ts = []
        for rep in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t.rebuild_for(frame, reqs)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                ts.append(e0.elapsed_time(e1))
        got = sample(label, t, reqs)
        if label not in ref:
            ref[label] = got
        same = all(np.array_equal(a, b) if a.dtype != np.float64 else
                   np.allclose(a, b, rtol=1e-12, atol=0) for a, b in zip(got, ref[label]))
        med = sorted(ts)[len(ts) // 2]
        tot += med
        out.append(f"{label}: {med:.4f}{'' if same else ' DIFF'}")
    print(" ".join(f"{n}={v}" for (n, _), v in zip(axes, combo)), " | ".join(out),
          f"| sum {tot:.4f}", flush=True)
