"""A/B timing of table rebuilds (tuning driver):
    python profiles/ab_build.py VAR=v1,v2 ...
Times rebuild() of config 2's plain set and config 5's plain / quadratic /
decay sets (CUDA events, median of 7, L2 flushed) per combination of the
environment overrides, and checks the u32 exports stay identical."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1705_03524_b200 import swg, synth  # noqa: E402

axes = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[1:]]
ctx = swg.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
c2 = torch.from_numpy(synth.config2(1).image).cuda()
c5 = torch.from_numpy(synth.config5(1).image).cuda()
sets = [("c2 plain", ctx.build(c2, swg.FMT_GRAY8, 32, swg.PLANES_PLAIN), c2),
        ("c5 plain", ctx.build(c5, swg.FMT_GRAY16, 64, swg.PLANES_PLAIN), c5),
        ("c5 quad", ctx.build(c5, swg.FMT_GRAY16, 64, swg.PLANES_QUADRATIC), c5),
        ("c5 decay", ctx.build_decay(c5, 15.0 / 16.0, swg.FMT_GRAY16, 64), c5)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for combo in itertools.product(*[v for _, v in axes]):
    for (name, _), val in zip(axes, combo):
        os.environ[name] = val
    out = []
    for label, t, src in sets:
        ts = []
        for rep in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t.rebuild(src)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                ts.append(e0.elapsed_time(e1))
        out.append(f"{label}: {sorted(ts)[len(ts) // 2]:.4f}")
    print(" ".join(f"{n}={v}" for (n, _), v in zip(axes, combo)), " | ".join(out), flush=True)
