#!/usr/bin/env python3
"""bench.py — SWIH hot path on B200: IH build + multi-scale likelihood maps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1]

One step = one frame through the hot path: quantise + weighted integral
histogram build, then the full strict likelihood map + peak at every scale
(BASELINE.json configs[1] by default: 1024x1024 u8, 32 bins, Gaussian kernel
(GaussianChebyshev sigma=0.5, exact full-ring wedding cake), windows
33/65/97).  `value` = weighted windows/s over all ranks with the frame
resident in HBM; `e2e` = the same through the C-ABI with a pinned host frame
in and host maps + peaks out.  N>1 (torchrun): one frame per GPU, no
data-path collective (weak scaling); the timed region is the max over ranks.
--impl reference times the reference CPU implementation (oracle/_ref, the
unmodified reference sources) on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "weighted windows/s"
UNIT = "windows/s"


def peaks_json():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ workload
def workload(name):
    from paper_1705_03524_b200 import swg, synth
    if name == "c1":
        return dict(name="config1: 256x256 u8, 16 bins, Manhattan, window 33x33",
                    gen=synth.config1, bins=16, planes=swg.PLANES_AFFINE,
                    scales=[(swg.Kernel(swg.MANHATTAN, 33, 33), swg.SWIH, 1, 0)],
                    P=3, elem=4)
    if name == "c5m":
        ks = (17, 25, 37, 53, 79, 117, 173, 257)
        return dict(name="config5 (Manhattan subset): 2048x2048 u16, 64 bins, Manhattan, windows "
                         + "/".join(map(str, ks)),
                    gen=synth.config5, bins=64, planes=swg.PLANES_AFFINE, fmt=swg.FMT_GRAY16,
                    scales=[(swg.Kernel(swg.MANHATTAN, k, k), swg.SWIH, 1, None) for k in ks],
                    P=3, elem=4)
    scales = []
    for i, s in enumerate((32, 64, 96)):
        kw = synth.odd_window(s)
        scales.append((swg.Kernel(swg.GAUSS_CHEB, kw, kw, 0.5), swg.CAKE, kw // 2 + 1, i))
    return dict(name="config2: 1024x1024 u8, 32 bins, Gaussian (GaussianChebyshev sigma=0.5, "
                     "exact full-ring cake), windows 33/65/97",
                gen=synth.config2, bins=32, planes=swg.PLANES_PLAIN, scales=scales, P=1,
                elem=2)


def target_center(scene, ti):
    if ti is None:  # no planted target: template from a fixed interior point
        h, w = scene.image.shape[:2]
        return w // 3, h // 2
    return scene.targets[ti][:2]


def make_requests(ctx, wl, scene):
    from paper_1705_03524_b200 import api, swg, synth
    reqs = []
    for k, method, rings, ti in wl["scales"]:
        cx, cy = target_center(scene, ti)
        templ = synth.crop(scene.image, cx, cy, k.kw, k.kh)
        model = api.target_model(ctx, templ, k, fmt=wl.get("fmt", swg.FMT_GRAY8),
                                 bins=wl["bins"], method=method, rings=rings)
        reqs.append(swg.MapRequest(k, model, method, swg.BHATTACHARYYA, rings))
    return reqs


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.path = index, None, None

    def start(self):
        try:
            self.path = f"/tmp/swg_clocks_{os.getpid()}.csv"
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU reference
def cpu_reference(wl, scene, models, budget_s=12.0, threads=None):
    """Reference CPU path (best-use): one reference build_tables
    (single-threaded; the reference has no parallel build) + per-scale sweep
    of reference queries + the restated scorer on `threads` host threads, on
    a bounded band of map rows per scale; returns projected full-frame rates."""
    from oracle import oracle as O
    threads = threads or os.cpu_count()
    R = O.Ref()
    img = scene.image
    bins = wl["bins"]
    t0 = time.perf_counter()
    if img.dtype == np.uint16:  # declared uint16 quantiser (no reference counterpart)
        fi = O.Oracle().quantize_gray16(img, bins)
    else:
        fi = R.quantize(img, bins)
    tabs = R.tables(fi, bins, budget=1 << 40)
    t_build = time.perf_counter() - t0
    per_scale = []
    total_win = 0
    proj = t_build
    sample_win = 0
    for (k, method, rings, _), model in zip(wl["scales"], models):
        ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
        mw, mh = img.shape[1] - k.kw + 1, img.shape[0] - k.kh + 1
        rows = max(threads // 2, 1)
        while True:
            t0 = time.perf_counter()
            tabs.sweep_rows(model, ok, method, 0, rings, 0, threads, 0, rows)
            dt = time.perf_counter() - t0
            if dt > budget_s / (3 * len(wl["scales"])) or rows >= mh:
                break
            rows = min(mh, rows * 2)
        rate = rows * mw / dt
        per_scale.append(rate)
        total_win += mw * mh
        sample_win += rows * mw
        proj += mw * mh / rate
    return {"value": total_win / proj, "t_build_s": t_build, "scale_rates": per_scale,
            "threads": threads, "sample_windows": sample_win, "frame_windows": total_win}


def cpu_model_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c5m"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    wl = workload(args.config)

    if args.impl == "reference":
        return run_reference(args, wl, rank, world)

    import torch
    from paper_1705_03524_b200 import swg
    # SWG_BENCH_SHARE_GPU=1: test mode for the N>1 code path on a 1-GPU box
    # (every rank on cuda:0, gloo collectives; ranks never wait on each
    # other's kernels, only on host barriers).  Never used for a reported run.
    share = os.environ.get("SWG_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    scene = wl["gen"](1 + rank)
    H, W = scene.image.shape
    ctx = swg.Context(local)
    # a non-default torch stream: our launches and the CUDA events share it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    reqs = make_requests(ctx, wl, scene)
    frame_dev = torch.from_numpy(scene.image).cuda()
    fmt = wl.get("fmt", swg.FMT_GRAY8)
    tables = ctx.build(frame_dev, fmt, wl["bins"], wl["planes"])
    maps_dev = [torch.empty(tables.map_shape(r.kernel), dtype=torch.float64, device="cuda")
                for r in reqs]
    peaks_dev = torch.zeros(len(reqs), 3, dtype=torch.float64, device="cuda")
    n_win = sum(m.numel() for m in maps_dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(ev=None):
        if ev:
            ev[0].record()
        tables.rebuild(frame_dev)
        if ev:
            ev[1].record()
        for i, r in enumerate(reqs):
            tables.likelihood_maps([r], scores="none", scores_dev=[maps_dev[i]],
                                   peaks_dev=peaks_dev[i])
            if ev:
                ev[2 + i].record()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # The step as one CUDA graph (no host launch gaps between the kernels).
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()

    nev = 2 + len(reqs)
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(args.steps)]
    clocks = Clocks(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    clocks.start()
    for s in range(args.steps):
        # a ~1 ms spin lets the host enqueue the whole step before the GPU
        # reaches it, so the per-kernel events carry no host launch gaps
        torch.cuda._sleep(2_000_000)
        flush.zero_()  # evict L2 (256 MiB > 126 MB) between timed steps; not timed
        step(events[s])
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = ctx.launches - launches0
    if dist:
        dist.barrier()
    per_step = [events[s][0].elapsed_time(events[s][-1]) for s in range(args.steps)]
    # headline timing: graph replays (same kernels, no launch gaps)
    if graph is not None:
        gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)]
               for _ in range(args.steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = Clocks(local)
        clocks.start()
        # soak: keep the GPU under this load for >= 1 s so the clock sampler
        # (100 ms period) sees it; the timed steps follow immediately
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 1.0:
            for _ in range(20):
                graph.replay()
            torch.cuda.synchronize()
        for s in range(args.steps):
            flush.zero_()
            gev[s][0].record()
            graph.replay()
            gev[s][1].record()
        torch.cuda.synchronize()
        clk = clocks.stop()
        if dist:
            dist.barrier()
        per_step = [gev[s][0].elapsed_time(gev[s][1]) for s in range(args.steps)]
    build_ms = [events[s][0].elapsed_time(events[s][1]) for s in range(args.steps)]
    scale_ms = [[events[s][1 + i].elapsed_time(events[s][2 + i]) for s in range(args.steps)]
                for i in range(len(reqs))]
    total_ms = sum(per_step)
    if dist:
        t = torch.tensor([total_ms], device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * n_win * args.steps / (total_ms / 1e3)

    # correctness spot check of the timed outputs (peak on the planted target)
    pk = peaks_dev.cpu().numpy()
    ok_peaks = True
    for i, (k, _, _, ti) in enumerate(wl["scales"]):
        ints = pk[i, :2].view(np.int32)
        cxp, cyp = int(ints[2]), int(ints[3])
        tx, ty = target_center(scene, ti)
        ok_peaks &= abs(cxp - tx) <= 1 and abs(cyp - ty) <= 1

    # ---- e2e through the C-ABI with host buffers (pinned), same frame
    frame_pin = swg.PinnedBuffer(scene.image.shape, scene.image.dtype)
    frame_pin.array[...] = scene.image
    maps_pin = [swg.PinnedBuffer(tuple(m.shape), np.float64) for m in maps_dev]
    import ctypes as C
    from paper_1705_03524_b200.swg import Peak, _Req, _check, lib
    creqs = (_Req * len(reqs))()
    for i, r in enumerate(reqs):
        creqs[i] = _Req(r.kernel, r.method, r.sim, r.rings, r.ring_rule, 0, 0,
                        r.model.ctypes.data_as(C.POINTER(C.c_double)))
    host_ptrs = (C.c_void_p * len(reqs))(*[m.array.ctypes.data for m in maps_pin])
    peaks_host = (Peak * len(reqs))()

    def e2e_step():
        _check(lib().swg_tables_rebuild(tables._h, frame_pin.array.ctypes.data, 0, 0))
        _check(lib().swg_likelihood_maps(tables._h, len(reqs), C.addressof(creqs),
                                         C.addressof(host_ptrs), None, C.addressof(peaks_host),
                                         None))

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e2e_t = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()  # returns after the host maps + peaks are filled
        e2e_t.append(time.perf_counter() - t0)
    e2e_total = sum(e2e_t)
    if dist:
        t = torch.tensor([e2e_total], device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = world * n_win * args.steps / e2e_total
    for i in range(len(reqs)):
        assert (maps_pin[i].array == maps_dev[i].cpu().numpy()).all()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel and of the IH build (SURVEY §8d bytes)
    hbm, src = peaks_json()
    b, P, e = wl["bins"], wl["P"], wl["elem"]  # e: bytes per table entry
    ih_bytes = (W + 1) * (H + 1) * b * P * e
    scale_avg = [sum(x) / args.steps for x in scale_ms]
    dom = max(range(len(reqs)), key=lambda i: scale_avg[i])  # the largest share of the step
    dom_bytes = ih_bytes + 8 * maps_dev[dom].numel()
    kname = {swg.CAKE: "k_sweep_cake16" if e == 2 else "k_sweep_cake",
             swg.SWIH: "k_sweep_affine"}.get(reqs[dom].method, "sweep")
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        t = json.load(open(tp)).get(args.config)
        if t and kname in t.get("kernel", ""):
            traffic = t["dram_bytes"]
    roofline = {"bound": "hbm", "achieved": dom_bytes / (scale_avg[dom] / 1e3) / 1e9,
                "peak": hbm, "unit": "GB/s", "traffic": traffic, "peak_source": src,
                "kernel": f"{kname} at {reqs[dom].kernel.kw}x{reqs[dom].kernel.kh} "
                          f"(IH read once + 8 B/window = {dom_bytes} B per launch, "
                          f"{scale_avg[dom]:.3f} ms)"}
    roofline["frac"] = roofline["achieved"] / hbm
    build_avg = sum(build_ms) / args.steps
    build_bytes = scene.image.nbytes + ih_bytes
    build_roof = {"bound": "hbm", "achieved": build_bytes / (build_avg / 1e3) / 1e9, "peak": hbm,
                  "unit": "GB/s", "kernel": "k_quantize + k_colsum + k_bandscan + k_build",
                  "ms": build_avg}
    build_roof["frac"] = build_roof["achieved"] / hbm

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        models = [r.model for r in reqs]
        c = cpu_reference(wl, scene, models)
        cpu = {"value": c["value"], "unit": UNIT, "cores": c["threads"], "kind": "reference",
               "sample": (f"oracle/_ref (unmodified reference sources): one build_tables "
                          f"({c['t_build_s']:.2f} s, 1 thread) + WeddingCakePlan sweep of "
                          f"{c['sample_windows']} windows (row bands of each scale, "
                          f"{c['threads']} threads), projected to the full frame of "
                          f"{c['frame_windows']} windows; CPU {cpu_model_name()}")}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32+f64",
        "data": "synthetic (seeded blurred-noise frame with planted targets, config generator "
                "in paper_1705_03524_b200/synth.py)",
        "config": {"workload": wl["name"], "frames_per_gpu": 1, "width": W, "height": H,
                   "bins": wl["bins"], "windows_per_frame": n_win,
                   "l2": "flushed between timed steps (256 MiB write, untimed)",
                   "parallelism": f"frames sharded over {world} GPU(s), no collective"},
        "ih_build": {"ms": build_avg, "gbps": build_roof["achieved"], "frac": build_roof["frac"]},
        "per_scale_ms": scale_avg,
        "roofline": roofline, "build_roofline": build_roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": scene.image.nbytes,
                "d2h_bytes_per_step": 8 * n_win + 24 * len(reqs),
                "ms_per_step": e2e_total / args.steps * 1e3},
        "gpu_launches": launches, "peaks_on_targets": bool(ok_peaks),
        "cpu_baseline": cpu, "clocks": clk,
    }
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def run_reference(args, wl, rank, world):
    if rank != 0:
        return
    import ctypes as C  # noqa: F401
    from oracle import oracle as O
    from paper_1705_03524_b200 import swg, synth  # noqa: F401
    scene = wl["gen"](1)
    # models with the reference's own target_model_for_method (matching.cpp:84-106)
    R = O.Ref()
    models = []
    for k, method, rings, ti in wl["scales"]:
        cx, cy = target_center(scene, ti)
        templ = synth.crop(scene.image, cx, cy, k.kw, k.kh)
        ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
        if templ.dtype == np.uint16:
            orc = O.Oracle()
            models.append(orc.target_model(orc.quantize_gray16(templ, wl["bins"]), wl["bins"], ok,
                                           method, rings))
        else:
            models.append(R.target_model(templ, wl["bins"], ok, method, rings))
    vals = []
    for s in range(args.warmup + args.steps):
        c = cpu_reference(wl, scene, models, budget_s=max(60.0 / (args.warmup + args.steps), 1.5))
        if s >= args.warmup:
            vals.append(c)
    value = statistics.mean(v["value"] for v in vals)
    n_win = vals[0]["frame_windows"]
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": n_win / value * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "i64+f64", "impl": "reference",
        "data": "synthetic (same generator and seed as --impl ours)",
        "config": {"workload": wl["name"], "frames_per_gpu": 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": vals[0]["threads"],
                         "kind": "reference",
                         "sample": "per step: one reference build_tables (1 thread) + row-band "
                                   "sample of each scale's WeddingCakePlan sweep on all host "
                                   "threads, projected to the full frame; CPU " + cpu_model_name()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
