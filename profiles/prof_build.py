"""Profiling driver for the IH build alone (no target models, no sweeps):
    ncu ... python profiles/prof_build.py c2|c5a|c5q|c5d
builds the config's tables once and rebuilds them 3 times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1705_03524_b200 import swg, synth  # noqa: E402

which = sys.argv[1]
ctx = swg.Context(0)
if which == "c2":
    img, fmt, bins, planes = synth.config2(1).image, swg.FMT_GRAY8, 32, swg.PLANES_PLAIN
else:
    img, fmt, bins = synth.config5(1).image, swg.FMT_GRAY16, 64
    planes = {"c5a": swg.PLANES_AFFINE, "c5q": swg.PLANES_QUADRATIC,
              "c5d": swg.PLANES_DECAY}[which]
dev = torch.from_numpy(img).cuda()
if planes == swg.PLANES_DECAY:
    t = ctx.build_decay(dev, 15.0 / 16.0, fmt, bins)
else:
    t = ctx.build(dev, fmt, bins, planes)
for _ in range(3):
    t.rebuild(dev)
ctx.synchronize()
