"""End-to-end strategies for config 5 (tuning driver, not a bench line):
    python profiles/e2e_exp.py
Times one frame through the three table sets -- pinned frame in, every map
and peak out to page-locked host memory -- as
  req+cp    : one swg_likelihood_maps call per request with a device map,
              each map copied to the host on a copy stream right behind its
              sweep (the overlap target)
  lib_sync  : swg_likelihood_maps per table set with host maps (copy path,
              host synchronisation at the end of every call)
  lib_async : swg_likelihood_maps_async per table set, one
              swg_ctx_synchronize per frame (bench.py's e2e path)
and prints, for the library paths, when each set's work ends on the
compute stream (a device-to-host copy queued on the compute stream shows
up as a set ending at its copies' end instead of its sweeps')."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1705_03524_b200 import swg  # noqa: E402
from paper_1705_03524_b200.swg import Peak, _check, lib  # noqa: E402

wl = bench.workload("c5")
data = wl["gen"](1)
ctx = swg.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
copy = torch.cuda.Stream()
models = bench.make_models(ctx, wl, data)
pin = swg.PinnedBuffer(data.image.shape, data.image.dtype)
pin.array[...] = data.image
frame = torch.from_numpy(data.image).cuda()
units = []
for gi, g in enumerate(wl["groups"]):
    t = (ctx.build_decay(frame, g["decay"], wl["fmt"], wl["bins"]) if g.get("decay")
         else ctx.build(frame, wl["fmt"], wl["bins"], g["planes"]))
    reqs = [swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings)
            for (k, meth, rings, _), m in zip(g["scales"], models[gi])]
    u = dict(t=t, reqs=reqs)
    u["dmaps"] = [torch.empty(t.map_shape(r.kernel), dtype=torch.float64, device="cuda")
                  for r in reqs]
    u["hmaps"] = [swg.PinnedBuffer(tuple(m.shape), np.float64) for m in u["dmaps"]]
    u["hmaps_t"] = [torch.from_numpy(h.array) for h in u["hmaps"]]
    u["peaks"] = torch.zeros(len(reqs), 3, dtype=torch.float64, device="cuda")
    u["creqs"], u["keep"] = swg.Tables._creqs(reqs, t.total_bins)
    u["hp"] = (C.c_void_p * len(reqs))(*[h.array.ctypes.data for h in u["hmaps"]])
    u["pkb"] = swg.PinnedBuffer((C.sizeof(Peak) * len(reqs),), np.uint8)
    u["pk"] = (Peak * len(reqs)).from_address(u["pkb"].array.ctypes.data)
    units.append(u)
marks = []


def step_req():
    for u in units:
        u["t"].rebuild_for(pin.array, u["reqs"])
        for j, r in enumerate(u["reqs"]):
            u["t"].likelihood_maps([r], scores="none", scores_dev=[u["dmaps"][j]],
                                   peaks_dev=u["peaks"][j])
            ev = torch.cuda.Event()
            ev.record(stream)
            copy.wait_event(ev)
            with torch.cuda.stream(copy):
                u["hmaps_t"][j].copy_(u["dmaps"][j], non_blocking=True)
    torch.cuda.synchronize()


def step_lib(fn_name):
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ends = []
    for u in units:
        u["t"].rebuild_for(pin.array, u["reqs"])
        _check(getattr(lib(), fn_name)(u["t"]._h, len(u["reqs"]), C.addressof(u["creqs"]),
                                       C.addressof(u["hp"]), None, C.addressof(u["pk"]), None))
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        ends.append(ev)
    ctx.synchronize()
    marks.append([round(e0.elapsed_time(e), 2) for e in ends])


for name, fn in (("req+cp", step_req),
                 ("lib_sync", lambda: step_lib("swg_likelihood_maps")),
                 ("lib_async", lambda: step_lib("swg_likelihood_maps_async"))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    line = f"{name:10s} {1e3 * sorted(ts)[len(ts) // 2]:.2f} ms per frame"
    if marks:
        line += f"   compute-stream set ends (ms): {marks[-1]}"
        marks.clear()
    print(line, flush=True)
