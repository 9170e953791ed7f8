"""End-to-end strategies for config 5 (tuning driver, not a bench line):
    python profiles/e2e_exp.py
Times one step (pinned frame in, every map + peak out to host memory) with
  zc      : mapped pinned host maps through swg_likelihood_maps (the bench's
            e2e path), unit by unit
  dev+cp  : device maps, each unit's maps copied to pinned host memory on a
            copy stream behind the unit's sweeps, one sync per step
for several unit orders."""
import itertools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1705_03524_b200 import swg  # noqa: E402

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
units = []
for gi, g in enumerate(wl["groups"]):
    if g.get("decay"):
        t = ctx.build_decay(torch.from_numpy(data.image).cuda(), g["decay"], wl["fmt"], wl["bins"])
    else:
        t = ctx.build(torch.from_numpy(data.image).cuda(), wl["fmt"], wl["bins"], g["planes"])
    reqs = [swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings)
            for (k, meth, rings, _), m in zip(g["scales"], models[gi])]
    dmaps = [torch.empty(t.map_shape(r.kernel), dtype=torch.float64, device="cuda") for r in reqs]
    hmaps = [swg.PinnedBuffer(tuple(m.shape), np.float64) for m in dmaps]
    hmaps_t = [torch.from_numpy(h.array) for h in hmaps]
    peaks = torch.zeros(len(reqs), 3, dtype=torch.float64, device="cuda")
    units.append(dict(t=t, reqs=reqs, dmaps=dmaps, hmaps=hmaps, hmaps_t=hmaps_t, peaks=peaks,
                      name=g["scales"][0][0].kind))


def step_zc(order):
    for i in order:
        u = units[i]
        u["t"].rebuild_for(pin.array, u["reqs"])
        _zc(u)


def _zc(u):
    import ctypes as C
    from paper_1705_03524_b200.swg import Peak, _check, lib
    creqs, keep = swg.Tables._creqs(u["reqs"], u["t"].total_bins)
    hp = (C.c_void_p * len(u["hmaps"]))(*[h.array.ctypes.data for h in u["hmaps"]])
    pk = (Peak * len(u["reqs"]))()
    _check(lib().swg_likelihood_maps(u["t"]._h, len(u["reqs"]), C.addressof(creqs),
                                     C.addressof(hp), None, C.addressof(pk), None))


def step_dev(order):
    for i in order:
        u = units[i]
        u["t"].rebuild_for(pin.array, u["reqs"])
        u["t"].likelihood_maps(u["reqs"], scores="none", scores_dev=u["dmaps"],
                               peaks_dev=u["peaks"])
        ev = torch.cuda.Event()
        ev.record(stream)
        copy.wait_event(ev)
        with torch.cuda.stream(copy):
            for d, h in zip(u["dmaps"], u["hmaps_t"]):
                h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()


def step_req(order):
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    evs = []
    for i in order:
        if evs is not None and i != order[0]:
            pass
        u = units[i]
        u["t"].rebuild_for(pin.array, u["reqs"])
        for j, r in enumerate(u["reqs"]):
            u["t"].likelihood_maps([r], scores="none", scores_dev=[u["dmaps"][j]],
                                   peaks_dev=u["peaks"][j])
            ev = torch.cuda.Event()
            ev.record(stream)
            copy.wait_event(ev)
            with torch.cuda.stream(copy):
                u["hmaps_t"][j].copy_(u["dmaps"][j], non_blocking=True)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        evs.append(ev)
    torch.cuda.synchronize()
    EV.append([round(e0.elapsed_time(e), 2) for e in evs])


import ctypes as C  # noqa: E402
from paper_1705_03524_b200.swg import Peak, _check, lib  # noqa: E402
for u in units:
    u["creqs"], u["keep"] = swg.Tables._creqs(u["reqs"], u["t"].total_bins)
    u["hp"] = (C.c_void_p * len(u["hmaps"]))(*[h.array.ctypes.data for h in u["hmaps"]])
    u["pkb"] = swg.PinnedBuffer((C.sizeof(Peak) * len(u["reqs"]),), np.uint8)
    u["pk"] = (Peak * len(u["reqs"])).from_address(u["pkb"].array.ctypes.data)


HT = []


EV = []


def step_lib(order, fn_name):
    t0 = time.perf_counter()
    ht = []
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    evs = [e0]
    for i in order:
        u = units[i]
        u["t"].rebuild_for(pin.array, u["reqs"])
        ht.append(time.perf_counter() - t0)
        _check(getattr(lib(), fn_name)(u["t"]._h, len(u["reqs"]), C.addressof(u["creqs"]),
                                       C.addressof(u["hp"]), None, C.addressof(u["pk"]), None))
        ht.append(time.perf_counter() - t0)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        evs.append(ev)
    ctx.synchronize()
    EV.append([round(e0.elapsed_time(e), 2) for e in evs[1:]])
    ht.append(time.perf_counter() - t0)
    HT.append(ht)


def step_libdev(order):
    for i in order:
        u = units[i]
        u["t"].rebuild_for(pin.array, u["reqs"])
        u["t"].likelihood_maps(u["reqs"], scores="none", scores_dev=u["dmaps"], peaks_dev=u["peaks"])
        for d, h in zip(u["dmaps"], u["hmaps_t"]):
            ev = torch.cuda.Event()
            ev.record(stream)
            copy.wait_event(ev)
            with torch.cuda.stream(copy):
                h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()


for u in units:
    u["creq1"] = [swg.Tables._creqs([r], u["t"].total_bins) for r in u["reqs"]]
    u["hp1"] = [(C.c_void_p * 1)(h.array.ctypes.data) for h in u["hmaps"]]


def step_lib1(order):
    for i in order:
        u = units[i]
        u["t"].rebuild_for(pin.array, u["reqs"])
        for j in range(len(u["reqs"])):
            cr, _k = u["creq1"][j]
            _check(lib().swg_likelihood_maps_async(u["t"]._h, 1, C.addressof(cr),
                                                   C.addressof(u["hp1"][j]), None, None,
                                                   ctypes_peak_dev(u, j)))
    ctx.synchronize()


def ctypes_peak_dev(u, j):
    return C.c_void_p(u["peaks"][j].data_ptr())


for name, fn in (("req+cp", step_req),
                 ("lib_sync", lambda o: step_lib(o, "swg_likelihood_maps")),
                 ("lib_async", lambda o: step_lib(o, "swg_likelihood_maps_async"))):
    for order in [(0, 1, 2)]:
        for _ in range(3):
            fn(order)
        torch.cuda.synchronize()
        ts = []
        for _ in range(8):
            t0 = time.perf_counter()
            fn(order)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(f"{name:7s} order {order}: {1e3 * sorted(ts)[len(ts) // 2]:.2f} ms", flush=True)
        if HT:
            print("   host marks (ms):", [round(1e3 * x, 2) for x in HT[-1]])
            HT.clear()
        if EV:
            print("   compute-stream unit ends (ms):", EV[-1])
            EV.clear()
