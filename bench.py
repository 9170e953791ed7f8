#!/usr/bin/env python3
"""bench.py — SWIH hot path on B200: IH build + multi-scale likelihood maps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5|c5m]

One step = one pass of the hot path over one batch of input: quantise +
weighted integral histogram build, then the full strict likelihood map +
peak at every scale.  Default: BASELINE.json configs[4], the config the
metric is quoted on ("windows/s and IH GB/s per kernel and scale"): one
2048x2048 u16 frame, 64 bins, Manhattan + Gaussian (GaussianChebyshev
sigma=0.5, exact full-ring wedding cake) + Euclidean (declared quadratic) +
exponential (declared, decay 15/16 per pixel) at windows 17..257 (8 scales
each).  The other configs:
  c1   256x256 u8, 16 bins, Manhattan 33x33                      (configs[0])
  c2   1024x1024 u8, 32 bins, Gaussian (exact cake), 33/65/97   (configs[1])
  c3   64 RGB 1920x1080 frames (tracking sequence), 4x4x4 bins, Euclidean
       (declared quadratic form), windows 45x59/49x65/53x71 on a 256x256
       search region around the previous ground truth           (configs[2])
  c4   3840x2160 RGB, 8x8x8 bins, exponential (decay 15/16 per pixel),
       windows 25/37/57/85/129; one row band per rank             (configs[3])
  c5m  c5's Manhattan subset
`value` = weighted windows/s over all ranks with the input resident in HBM;
`e2e` = the same through the C-ABI with pinned host input and host maps /
peaks out.  N>1 (torchrun), strong scaling throughout: one frame's
(kernel, scale) requests partitioned over ranks (c1/c2/c5: LPT by
estimated cost, the largest split by map rows, each rank building only the
table sets its requests read -- dist.plan_frame), sequence frames (c3) or
row bands (c4); no data-path collective; the timed region is the max over
ranks.
--impl reference times the reference CPU implementation (oracle/_ref, the
unmodified reference sources; the oracle restatement for the kernels the
reference lacks) on this host's cores.
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
EXP_DECAY = 15.0 / 16.0  # declared exponential kernel: weight 15/16 per pixel of L1 distance
# the one decay serves every scale (one decayed table set per frame): the
# weight falls to 1/e at 15.5 px and to 1e-2 at 71 px of L1 distance from
# the centre, so the larger windows share that support
EXP_NOTE = ("exponential w = (15/16)^(|dx|+|dy|) at every scale (one decayed table set; "
            "weight 1/e at 15.5 px, 1e-2 at 71 px L1)")
L2_NOTE = "GPU arm: L2 flushed between timed steps (256 MiB write, untimed)"


def peaks_json():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ workloads
def exp_decay_of(kw, mode):
    """Declared exponential kernel's decay per pixel: one d = 15/16 for every
    scale ("fixed", one decayed table set), or d = exp(-4/kw) per scale
    ("scale": SURVEY App. A's lambda ~ 1/kw, the weight at the window corner
    e^(-4 (kw-1)/kw) ~ 0.018 at every scale; one decayed table set per scale)."""
    import math
    return EXP_DECAY if mode == "fixed" else math.exp(-4.0 / kw)


def exp_groups(ks, mode, bin_chunks=None):
    from paper_1705_03524_b200 import swg
    K = swg.Kernel
    extra = {"bin_chunks": bin_chunks} if bin_chunks else {}
    if mode == "fixed":
        return [dict(planes=swg.PLANES_DECAY, decay=EXP_DECAY, **extra,
                     scales=[(K(swg.EXP_L1, k, k, EXP_DECAY), swg.SWIH, 1, None) for k in ks])]
    return [dict(planes=swg.PLANES_DECAY, decay=exp_decay_of(k, mode), **extra,
                 scales=[(K(swg.EXP_L1, k, k, exp_decay_of(k, mode)), swg.SWIH, 1, None)])
            for k in ks]


EXP_SCALE_NOTE = ("exponential w = d^(|dx|+|dy|) with d = exp(-4/kw) per scale (one decayed "
                  "table set per scale; corner weight ~0.018 at every scale)")


def workload(name, exp_decay="fixed"):
    """A workload = input generator + table groups; a group = one table set
    (planes / decay) and the scales (kernel, method, rings, target index)
    it serves.  exp_decay: "fixed" (one decay for every scale) or "scale"
    (exp_decay_of)."""
    from paper_1705_03524_b200 import swg, synth
    K = swg.Kernel
    enote = EXP_NOTE if exp_decay == "fixed" else EXP_SCALE_NOTE
    if name == "c1":
        return dict(name="config1: 256x256 u8, 16 bins, Manhattan, window 33x33", kind="frame",
                    gen=synth.config1, fmt=swg.FMT_GRAY8, bins=16, nbins=16, scaling="strong",
                    groups=[dict(planes=swg.PLANES_AFFINE,
                                 scales=[(K(swg.MANHATTAN, 33, 33), swg.SWIH, 1, 0)])])
    if name in ("c5", "c5m"):
        ks = (17, 25, 37, 53, 79, 117, 173, 257)
        manhattan = [(K(swg.MANHATTAN, k, k), swg.SWIH, 1, None) for k in ks]
        groups = [dict(planes=swg.PLANES_AFFINE, scales=manhattan)]
        label = "Manhattan"
        if name == "c5":
            # one integral-table set per weight-plane family: the quadratic
            # set's planes {1, x, y, x^2, y^2} include Manhattan's {1, x, y},
            # so the Manhattan and Euclidean scales share one build
            groups = [
                dict(planes=swg.PLANES_QUADRATIC,
                     scales=manhattan + [(K(swg.EUCLID_QUAD, k, k), swg.SWIH, 1, None)
                                         for k in ks]),
                dict(planes=swg.PLANES_PLAIN,
                     scales=[(K(swg.GAUSS_CHEB, k, k, 0.5), swg.CAKE, k // 2 + 1, None)
                             for k in ks]),
            ] + exp_groups(ks, exp_decay)
            label = ("Manhattan + Gaussian (exact full-ring cake) + Euclidean (quadratic) + "
                     + enote)
        return dict(name=f"config5{' (Manhattan subset)' if name == 'c5m' else ''}: 2048x2048 "
                         f"u16, 64 bins, {label}, windows " + "/".join(map(str, ks)),
                    kind="frame", gen=synth.config5, fmt=swg.FMT_GRAY16, bins=64, nbins=64,
                    scaling="strong", groups=groups)
    if name == "c3":
        scales = [(K(swg.EUCLID_QUAD, kw, kh), swg.SWIH, 1, 0)
                  for kw, kh in ((45, 59), (49, 65), (53, 71))]
        return dict(name="config3: 64 RGB 1920x1080 frames, 4x4x4 bins, Euclidean (quadratic), "
                         "windows 45x59/49x65/53x71, 256x256 search region",
                    kind="sequence", gen=synth.config3, fmt=swg.FMT_RGB8, bins=4, nbins=64,
                    scaling="strong", groups=[dict(planes=swg.PLANES_QUADRATIC, scales=scales)])
    if name == "c4":
        return dict(name="config4: 3840x2160 RGB, 8x8x8 bins, " + enote +
                         ", windows 25/37/57/85/129, row bands",
                    kind="bands", gen=synth.config4, fmt=swg.FMT_RGB8, bins=8, nbins=512,
                    scaling="strong", groups=exp_groups((25, 37, 57, 85, 129), exp_decay, 8))
    scales = []
    for i, s in enumerate((32, 64, 96)):
        kw = synth.odd_window(s)
        scales.append((K(swg.GAUSS_CHEB, kw, kw, 0.5), swg.CAKE, kw // 2 + 1, i))
    return dict(name="config2: 1024x1024 u8, 32 bins, Gaussian (GaussianChebyshev sigma=0.5, "
                     "exact full-ring cake), windows 33/65/97",
                kind="frame", gen=synth.config2, fmt=swg.FMT_GRAY8, bins=32, nbins=32,
                scaling="strong", groups=[dict(planes=swg.PLANES_PLAIN, scales=scales)])


def manhattan_mass(k):
    """Strict-window weight sum of the Manhattan kernel (kernel.cpp:68-75)."""
    hx, hy = k.hx, k.hy
    return k.kw * k.kh * (hx + hy + 1) - k.kh * hx * (hx + 1) - k.kw * hy * (hy + 1)


def engine_of(group, k, method, windows=1 << 30):
    """(sweep kernel, planes read, bytes per entry) the library picks
    (swg_abi.cu likelihood_maps engine choice) for a map of `windows`."""
    from paper_1705_03524_b200 import swg
    if group["planes"] == swg.PLANES_DECAY:
        return "k_sweep_exp", 4, 8
    if (group["planes"] in (swg.PLANES_AFFINE, swg.PLANES_QUADRATIC) and
            k.kind == swg.MANHATTAN and method in (swg.SWIH, swg.BRUTE) and
            manhattan_mass(k) < 65536 and windows >= 1 << 20 and
            os.environ.get("SWG_AFFINE16", "1") != "0"):
        return "k_sweep_affine16", 3, 2  # narrow {1, x, y} planes: H < 2^16
    if group["planes"] == swg.PLANES_QUADRATIC:
        if k.kind == swg.MANHATTAN:  # planes {1, x, y} of the quadratic set
            return "k_sweep_affine", 3, 4
        return "k_sweep_quad", 5, 4
    if method == swg.CAKE or k.kind == swg.UNIFORM:
        small = k.kw * k.kh < 65536
        if method == swg.CAKE and not small:  # full-ring plan: ring 1 box + ring 0 frame
            small = (k.kw - 2) * (k.kh - 2) < 65536 and k.kw * k.kh - (k.kw - 2) * (k.kh - 2) < 65536
        if group["planes"] == swg.PLANES_PLAIN and small:
            return "k_sweep_cake16", 1, 2
        return "k_sweep_cake", 1, 4
    return "k_sweep_affine", 3, 4


def group_build_bytes(group, w, h, nbins, narrow=None):
    """Plane bytes one rebuild writes (every plane set the tables hold);
    `narrow`: whether the tables hold the 16-bit {1, x, y} planes (None:
    estimate from the kernels)."""
    from paper_1705_03524_b200 import swg
    cells = (w + 1) * (h + 1) * nbins
    p = group["planes"]
    if narrow is None:
        narrow = any(engine_of(group, k, m, (w - k.kw + 1) * (h - k.kh + 1))[0] ==
                     "k_sweep_affine16" for k, m, _, _ in group["scales"])
    narrow = cells * 3 * 2 if narrow else 0
    if p == swg.PLANES_DECAY:
        return cells * 4 * 8
    if p == swg.PLANES_QUADRATIC:
        return cells * 5 * 4 + narrow
    if p == swg.PLANES_AFFINE:
        return cells * 3 * 4 + narrow
    b = cells * 2  # narrow 16-bit plain planes
    if any(engine_of(group, k, m)[0] == "k_sweep_cake" for k, m, _, _ in group["scales"]):
        b += cells * 4  # 32-bit plain planes for the large windows
    return b


def est_request_ms(group, k, method, rings, rows, w, h, nbins):
    """Rough sweep cost of map rows `rows` of one request (ms), for the
    multi-GPU plan only (round-1 B200 measurements: table sweeps at ~3 TB/s
    of algorithmic bytes, the cake at ~9.4e-9 ms per window-ring at 64 bins)."""
    from paper_1705_03524_b200 import swg
    mw = w - k.kw + 1
    kname, P, e = engine_of(group, k, method, (w - k.kw + 1) * (h - k.kh + 1))
    tab = min(h + 1, rows + k.kh) * (w + 1) * nbins * P * e
    if kname in ("k_sweep_cake16", "k_sweep_cake"):
        return 0.05 + 9.4e-9 * rows * mw * rings * nbins / 64 * (2 if kname == "k_sweep_cake" else 1)
    if method == swg.BRUTE:
        return 0.05 + 1e-9 * rows * mw * k.kw * k.kh
    return 0.05 + tab / 3.0e9


def model_bins_read(group, k, method, model, nbins):
    """(bins whose records a sweep reads, the selective-build units it
    needs) -- the library's rule (plan_needs): nonzero-model bin pairs for the
    exponential sweep, octets for the Manhattan / Euclidean sweeps; every bin
    (no units) for the cake and brute force."""
    import numpy as np
    from paper_1705_03524_b200 import swg
    if os.environ.get("SWG_SPARSE", "1") == "0":
        return nbins, set()
    kname = engine_of(group, k, method)[0]
    if kname == "k_sweep_exp":
        grp = 2
    elif kname in ("k_sweep_affine", "k_sweep_affine16", "k_sweep_quad") and method == swg.SWIH:
        grp = 8
    else:
        return nbins, set()
    units = {int(b) // grp for b in np.flatnonzero(np.asarray(model) != 0)}
    return min(nbins, grp * len(units)), units


def est_build_ms(group, w, h, nbins):
    return 0.1 + group_build_bytes(group, w, h, nbins) / 3.0e9


def target_center(scene, ti):
    if ti is None:  # no planted target: template from a fixed interior point
        h, w = scene.image.shape[:2]
        return w // 3, h // 2
    return scene.targets[ti][:2]


def make_models(ctx, wl, data):
    """Per group, per scale: model = target_model_for_method of the kw x kh
    template centred on the target (matching.cpp:84-106)."""
    from paper_1705_03524_b200 import api, synth
    out = []
    for g in wl["groups"]:
        ms = []
        for k, method, rings, ti in g["scales"]:
            if wl["kind"] == "sequence":
                cx, cy = data.track[0]
                img = data.frames[0]
            else:
                cx, cy = target_center(data, ti)
                img = data.image
            templ = synth.crop(img, cx, cy, k.kw, k.kh)
            ms.append(api.target_model(ctx, templ, k, fmt=wl["fmt"], bins=wl["bins"],
                                       method=method, rings=rings))
        out.append(ms)
    return out


def band_plan(H, scales, n_bands):
    """Row bands of the frame (c4): band b owns map rows [b*S, (b+1)*S) of
    every scale and is built from pixel rows [p0, p0 + BH), BH = S + the
    largest kh - 1 (the last band is shifted up to keep one table shape)."""
    kh_max = max(k.kh for k, _, _, _ in scales)
    S = -(-H // n_bands)
    BH = min(H, S + kh_max - 1)
    bands = []
    for b in range(n_bands):
        p0 = min(b * S, H - BH)
        rows = []
        for k, _, _, _ in scales:
            mh = H - k.kh + 1
            v0, v1 = min(b * S, mh), min((b + 1) * S, mh)
            rows.append((v0, v1))
        bands.append((p0, rows))
    return BH, bands


def config_dict(wl, job_win):
    """The `config` both arms print (identical keys and values)."""
    return {"workload": wl["name"], "bins": wl["nbins"], "windows_per_step": int(job_win),
            "l2": L2_NOTE}


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
def _quantize_host(wl, img):
    from oracle import oracle as O
    from paper_1705_03524_b200 import swg
    orc = O.Oracle()
    if wl["fmt"] == swg.FMT_GRAY16:  # declared uint16 quantiser (no reference counterpart)
        return orc.quantize_gray16(img, wl["nbins"])
    if wl["fmt"] == swg.FMT_RGB8:    # declared RGB quantiser (no reference counterpart)
        return orc.quantize_rgb8(img, wl["bins"])
    return O.Ref().quantize(img, wl["bins"])


def cpu_reference(wl, data, models, budget_s=12.0, threads=None, public_api=False):
    """Reference CPU path (best-use) on `threads` host threads:
    kernels the reference implements (Manhattan swih, GaussianChebyshev
    wedding cake) run the unmodified reference sources (oracle/_ref: one
    build_tables, single-threaded as in the reference, + a row-band sweep of
    reference queries and the restated scorer); the declared kernels the
    reference lacks (Euclidean, exponential) run the oracle's brute-force
    restatement (baselines.cpp:53-69 order).  Each scale is timed on a
    bounded band of map rows and projected to the step's full work."""
    from oracle import oracle as O
    from paper_1705_03524_b200 import swg, synth
    threads = threads or os.cpu_count()
    R = O.Ref()
    orc = O.Oracle()
    if wl["kind"] == "sequence":
        f = 1
        x0, y0 = synth.search_origin(data, f)
        s = data.search
        img = data.frames[f, y0:y0 + s, x0:x0 + s]
        mult = data.frames.shape[0]
    else:
        img = data.image
        mult = 1
    t0 = time.perf_counter()
    fi = _quantize_host(wl, img)
    t_q = time.perf_counter() - t0
    nb = wl["nbins"]
    H, W = fi.shape
    tabs, t_build = None, 0.0
    proj = t_q * mult
    total_win = sample_win = 0
    kinds = set()
    rates = []
    for g, ms in zip(wl["groups"], models):
        for (k, method, rings, _), model in zip(g["scales"], ms):
            ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
            mw, mh = W - k.kw + 1, H - k.kh + 1
            ref_ok = k.kind in (swg.MANHATTAN, swg.UNIFORM, swg.GAUSS_CHEB)
            if ref_ok and tabs is None:
                t0 = time.perf_counter()
                tabs = R.tables(fi, nb, budget=1 << 40)
                t_build = time.perf_counter() - t0
                proj += t_build * mult
            rows = max(threads // 2, 1)
            while True:
                t0 = time.perf_counter()
                if ref_ok:
                    tabs.sweep_rows(model, ok, method, 0, rings, 0, threads, 0, rows)
                else:
                    orc.likelihood_map(fi, nb, model, ok, O.BRUTE, 0, rows=(0, rows),
                                       threads=threads)
                dt = time.perf_counter() - t0
                if dt > budget_s / (3 * sum(len(x["scales"]) for x in wl["groups"])) or rows >= mh:
                    break
                rows = min(mh, rows * 2)
            rate = rows * mw / dt
            rates.append(rate)
            kinds.add("reference" if ref_ok else "port")
            total_win += mw * mh * mult
            sample_win += rows * mw
            proj += mw * mh * mult / rate
    # SURVEY §8d's second variant: the reference's public API as a user calls
    # it (one likelihood_map per scale, each rebuilding the tables), for the
    # gray-u8 configs whose kernels the reference implements; full maps
    public = None
    if (public_api and wl["fmt"] == swg.FMT_GRAY8 and wl["kind"] == "frame"
            and kinds == {"reference"} and img.size <= 1024 * 1024):
        t0 = time.perf_counter()
        for g, ms in zip(wl["groups"], models):
            for (k, method, rings, _), model in zip(g["scales"], ms):
                R.likelihood_map(img, wl["bins"], model, O.kernel(k.kind, k.kw, k.kh, k.sigma),
                                 method, 0, rings, 0, threads=threads, budget=1 << 40,
                                 want_scores=True)
        public = total_win / (time.perf_counter() - t0)
    return {"value": total_win / proj, "t_build_s": t_build, "scale_rates": rates,
            "threads": threads, "sample_windows": sample_win, "frame_windows": total_win,
            "kind": "reference" if kinds == {"reference"} else "port",
            "mixed": sorted(kinds), "public_api": public}


def cpu_model_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample_text(wl, c):
    parts = []
    if "reference" in c["mixed"]:
        parts.append(f"oracle/_ref (unmodified reference sources): build_tables "
                     f"({c['t_build_s']:.2f} s, 1 thread) + reference-query sweeps")
    if "port" in c["mixed"]:
        parts.append("oracle brute-force restatement for the declared kernels the reference "
                     "lacks")
    return ("; ".join(parts) + f"; {c['sample_windows']} windows sampled (row bands of each "
            f"scale, {c['threads']} threads), projected to the step's {c['frame_windows']} "
            f"windows; CPU {cpu_model_name()}")


# ------------------------------------------------------------------ main
def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "c5m"])
    ap.add_argument("--exp-decay", default="fixed", choices=["fixed", "scale"],
                    help="declared exponential kernel: one decay 15/16 for every scale "
                         "(default) or exp(-4/kw) per scale (one decayed table set each)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--bin-chunks", type=int, default=None,
                    help="config 4: walk the bins in this many ranges on each GPU, chaining "
                         "the partial sums (smaller tables stay in L2 between a window's "
                         "corners); default 8 for config 4, 1 elsewhere")
    ap.add_argument("--p2p", default="peer", choices=["peer", "nccl"],
                    help="--shard bins: running sums written by the sweep straight into the "
                         "next rank's buffer (peer memory), or sent with NCCL")
    ap.add_argument("--shard", default="rows", choices=["rows", "bins"],
                    help="config 4 over N>1 ranks: row bands per rank (default) or every "
                         "band on every rank with bin ranges chained rank to rank")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    return args


class OursArm:
    """One rank of `bench.py --impl ours`.

    A UNIT is one table set and the requests swept on it per step: dict with
    t (Tables), src (device source view), pitch, reqs, maps (device score
    outputs), peaks, g (group index), sidx (scale index per request), h2d
    (input bytes), chunks [(bin0, requests)] (one entry unless the bins are
    walked in ranges), and for the rank-to-rank bin chain pin / pout (/ token).
    """

    def __init__(self, args, wl, rank=None, world=None):
        """rank / world override the torchrun environment (tests: one rank's
        share of the plan on one GPU, no process group)."""
        import torch
        from paper_1705_03524_b200 import swg
        self.torch, self.swg = torch, swg
        self.args, self.wl = args, wl
        injected = rank is not None
        self.rank = int(os.environ.get("RANK", 0)) if rank is None else rank
        self.world = int(os.environ.get("WORLD_SIZE", 1)) if world is None else world
        self.local = int(os.environ.get("LOCAL_RANK", 0))
        # SWG_BENCH_SHARE_GPU=1: test mode for the N>1 code path on a 1-GPU box
        # (every rank on cuda:0, gloo collectives; ranks never wait on each
        # other's kernels, only on host barriers).  Never used for a reported run.
        self.share = os.environ.get("SWG_BENCH_SHARE_GPU") == "1"
        if self.share:
            self.local = 0
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1 and not injected:
            import torch.distributed as dist
            if self.share:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.dist = dist
        self.weak = wl["scaling"] == "weak"
        self.data = wl["gen"](1 + self.rank if self.weak else 1)
        self.plan = None
        self.ctx = swg.Context(self.local)
        # a non-default torch stream: our launches and the CUDA events share it
        self.stream = torch.cuda.Stream()
        torch.cuda.set_stream(self.stream)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.models = make_models(self.ctx, wl, self.data)
        self.fmt, self.nb = wl["fmt"], wl["nbins"]
        self.bins_mode = args.shard == "bins" and self.world > 1
        self.units = []
        self.batch_peaks = None
        self.build_units()

    # ------------------------------------------------------------ set-up
    def group_chunks(self, g):
        """Bin ranges one GPU walks for this group (1: all bins at once)."""
        if self.bins_mode:
            return 1
        if self.args.bin_chunks is not None:
            return self.args.bin_chunks
        if g.get("decay") and os.environ.get("SWG_DECAY_CHUNKS"):  # tuning override
            return int(os.environ["SWG_DECAY_CHUNKS"])
        return g.get("bin_chunks", 1)

    def new_tables(self, g, src, pitch=0):
        wl, ctx = self.wl, self.ctx
        if self.group_chunks(g) > 1:  # the first bin range; the rest via rebuild_bins
            from paper_1705_03524_b200 import dist as D
            b0, b1 = D.bin_ranges(self.nb, self.group_chunks(g))[0]
            return ctx.build_bins(src, b0, b1, self.fmt, wl["bins"], g["planes"],
                                  decay=g.get("decay") or 0.0, pitch=pitch)
        if g.get("decay"):
            return ctx.build_decay(src, g["decay"], self.fmt, wl["bins"], pitch=pitch)
        return ctx.build(src, self.fmt, wl["bins"], g["planes"], pitch=pitch)

    def _requests(self, g, ms):
        swg = self.swg
        return [swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings)
                for (k, meth, rings, _), m in zip(g["scales"], ms)]

    def _map_buffers(self, t, reqs):
        torch = self.torch
        return [torch.empty(t.map_shape(r.kernel), dtype=torch.float64, device="cuda")
                for r in reqs]

    def _frame_units(self):
        """c1 / c2 / c5: ONE frame; its (kernel, scale) requests partitioned
        over the ranks (dist.plan_frame: LPT by estimated cost, the largest
        split by map rows); a rank builds only the table sets its requests
        read, over the whole frame (replicated build)."""
        from paper_1705_03524_b200 import dist as D
        swg, torch = self.swg, self.torch
        data, groups = self.data, self.wl["groups"]
        frame_dev = torch.from_numpy(data.image).cuda()
        H, W = data.image.shape[:2]
        measured = self._measure_costs(groups, frame_dev) if self.dist else None
        reqs_all = []
        build = []
        for gi, g in enumerate(groups):
            union = set()
            for si, (k, meth, rings, _) in enumerate(g["scales"]):
                mh = H - k.kh + 1
                # the sweeps with a closed-form window mass read only the
                # model's nonzero octets / bin pairs (SweepArgs::act, ExpSweep::pairs)
                nb_read, units = model_bins_read(g, k, meth, self.models[gi][si], self.nb)
                union |= units
                reqs_all.append(((gi, si), gi, mh,
                                 est_request_ms(g, k, meth, rings, mh, W, H, nb_read)))
            full = est_build_ms(g, W, H, self.nb)
            # a model-driven rebuild writes only the units the requests read
            frac = len(union) / max(1, -(-self.nb // (2 if g["planes"] == swg.PLANES_DECAY else 8)))
            build.append(full if not union else 0.1 + (full - 0.1) * min(1.0, frac))
        if measured is not None:  # rank 0's timings, the same on every rank
            req_ms, build_ms = measured
            reqs_all = [(key, gi, mh, req_ms[i]) for i, (key, gi, mh, _) in enumerate(reqs_all)]
            build = build_ms
        self.plan = D.plan_frame(reqs_all, build, self.world, min_rows=8)
        # each rank's planned load (ms): its requests + the builds of its sets
        self.plan_load = [round(sum(w.cost for w in p) + sum(build[g] for g in {w.group for w in p}), 3)
                          for p in self.plan]
        self.plan_costs = "measured (rank 0, broadcast)" if measured is not None else "estimated"
        mine = self.plan[self.rank]
        for gi, (g, ms) in enumerate(zip(groups, self.models)):
            work = [w for w in mine if w.group == gi]
            if not work:
                continue
            t = self.new_tables(g, frame_dev)
            reqs, maps = [], []
            for w in work:
                k, meth, rings, _ = g["scales"][w.key[1]]
                mh = H - k.kh + 1
                reqs.append(swg.MapRequest(k, ms[w.key[1]], meth, swg.BHATTACHARYYA, rings,
                                           rows=None if w.rows == (0, mh) else w.rows))
                maps.append(torch.empty((w.rows[1] - w.rows[0], W - k.kw + 1),
                                        dtype=torch.float64, device="cuda"))
            self.units.append(dict(t=t, src=frame_dev, pitch=0, reqs=reqs, maps=maps, g=gi,
                                   sidx=[w.key[1] for w in work],
                                   rows=[w.rows for w in work], h2d=data.image.nbytes))
        self.tab_w, self.tab_h = W, H

    def _measure_costs(self, groups, frame_dev):
        """Multi-GPU plan costs measured, not estimated: rank 0 times every
        request's full map and every table set's model-driven rebuild on its
        GPU (eager, CUDA events, median of 3) and broadcasts them, so every
        rank derives the same partition (setup only, outside the timed step).
        Returns ([ms per request in group/scale order], [build ms per group])."""
        torch = self.torch
        n_req = sum(len(g["scales"]) for g in groups)
        dev = "cpu" if self.share else "cuda"
        costs = torch.zeros(n_req + len(groups), dtype=torch.float64, device=dev)
        if self.rank == 0:
            vals, builds = [], []

            def timed(fn, reps=3):
                ts = []
                for _ in range(reps + 1):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    fn()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                return sorted(ts[1:])[len(ts[1:]) // 2]

            for gi, g in enumerate(groups):
                t = self.new_tables(g, frame_dev)
                reqs = self._requests(g, self.models[gi])
                maps = self._map_buffers(t, reqs)
                peaks = torch.zeros(len(reqs), 3, dtype=torch.float64, device="cuda")
                builds.append(timed(lambda: t.rebuild_for(frame_dev, reqs)))
                for i, r in enumerate(reqs):
                    vals.append(timed(lambda: t.likelihood_maps([r], scores="none",
                                                                 scores_dev=[maps[i]],
                                                                 peaks_dev=peaks[i])))
                t.close()
            costs.copy_(torch.tensor(vals + builds, dtype=torch.float64))
        self.dist.broadcast(costs, 0)
        c = costs.cpu().tolist()
        return c[:n_req], c[n_req:]

    def _sequence_units(self):
        """c3: this rank's frames, each a search region swept on one table set."""
        from paper_1705_03524_b200 import synth
        data, rank, world = self.data, self.rank, self.world
        F, H, W = data.frames.shape[:3]
        frames_dev = self.torch.from_numpy(data.frames).cuda()
        S = data.search
        g, ms = self.wl["groups"][0], self.models[0]
        mine = [f for f in range(F) if f % world == rank]
        x0, y0 = synth.search_origin(data, mine[0])
        t = self.new_tables(g, frames_dev[mine[0], y0:y0 + S, x0:x0 + S], pitch=W * 3)
        reqs = self._requests(g, ms)
        maps = self._map_buffers(t, reqs)  # one map per scale, overwritten frame after frame
        for f in mine:
            x0, y0 = synth.search_origin(data, f)
            self.units.append(dict(t=t, src=frames_dev[f, y0:y0 + S, x0:x0 + S], pitch=W * 3,
                                   reqs=reqs, maps=maps, g=0, sidx=list(range(len(reqs))),
                                   frame=f, origin=(x0, y0), h2d=S * S * 3))
        self.tab_w = self.tab_h = S
        self.frame_hw, self.search = (H, W), S
        self.batch_peaks = self.torch.zeros(len(self.units) * len(reqs), 3,
                                            dtype=self.torch.float64, device="cuda")

    def _band_units(self):
        """c4: row bands (one per rank, or more if a band's tables do not fit);
        every table group (one decay per scale with --exp-decay scale) builds
        its own tables over the same bands."""
        torch, swg, ctx, wl = self.torch, self.swg, self.ctx, self.wl
        data, rank, world = self.data, self.rank, self.world
        H, W = data.image.shape[:2]
        frame_dev = torch.from_numpy(data.image).cuda()
        groups = wl["groups"]
        if self.bins_mode:
            assert len(groups) == 1, "--shard bins: one table group"
        scales = [sc for g in groups for sc in g["scales"]]
        full_maps = [torch.empty((H - k.kh + 1, W - k.kw + 1), dtype=torch.float64, device="cuda")
                     for k, _, _, _ in scales]
        # one row band per rank (the whole frame on one GPU: 136 GB of decay
        # tables, the band halo costs more than it saves); twice as many if a
        # band's tables do not fit
        n_bands = int(os.environ.get("SWG_C4_BANDS", 1 if not self.bins_mode else 4))
        n_bands = max(n_bands, world) if not self.bins_mode else n_bands
        while True:
            BH, plan = band_plan(H, scales, n_bands)
            mine = list(range(n_bands)) if self.bins_mode else \
                [b for b in range(n_bands) if b % world == rank]
            tabs = []
            try:
                for g in groups:
                    if self.bins_mode:  # rank g: bins [b_g, b_g+1) of every band
                        from paper_1705_03524_b200 import dist as D
                        b0, b1 = D.bin_ranges(self.nb, world)[rank]
                        tabs.append(ctx.build_bins(frame_dev[plan[0][0]:plan[0][0] + BH], b0, b1,
                                                   self.fmt, wl["bins"], g["planes"],
                                                   decay=g.get("decay") or 0.0))
                    else:
                        tabs.append(self.new_tables(
                            g, frame_dev[plan[mine[0]][0]:plan[mine[0]][0] + BH]))
                break
            except swg.CapacityError:
                for t in tabs:
                    t.close()
                if n_bands >= 64:
                    raise
                n_bands *= 2
        for b in mine:
            p0, rows = plan[b]
            off = 0
            for gi, (g, ms, t) in enumerate(zip(groups, self.models, tabs)):
                reqs, maps, sidx = [], [], []
                for si, ((k, meth, rings, _), m) in enumerate(zip(g["scales"], ms)):
                    v0, v1 = rows[off + si]
                    if v1 <= v0:
                        continue
                    reqs.append(swg.MapRequest(k, m, meth, swg.BHATTACHARYYA, rings,
                                               rows=(v0 - p0, v1 - p0)))
                    maps.append(full_maps[off + si][v0:v1])
                    sidx.append(si)
                off += len(g["scales"])
                if reqs:
                    self.units.append(dict(t=t, src=frame_dev[p0:p0 + BH], pitch=0, reqs=reqs,
                                           maps=maps, g=gi, sidx=sidx, band=b, p0=p0,
                                           h2d=BH * W * 3))
        if self.bins_mode:
            self._attach_rank_chain()
        self.tab_w, self.tab_h = W, BH

    def _attach_rank_chain(self):
        """--shard bins: running (s, mass) per window passed rank to rank."""
        torch, swg, rank, world = self.torch, self.swg, self.rank, self.world
        last = rank == world - 1
        if self.args.p2p == "peer":
            # running (s, mass) per window written by rank g's sweep STRAIGHT
            # into rank g+1's input buffer (peer memory mapped with an IPC
            # handle; NVLink stores from the kernel's epilogue); only a 4-byte
            # token per request goes through the process group, stream-ordered
            # behind the kernel
            mine_h = []
            for u in self.units:
                u["pin"] = []
                for m in u["maps"]:
                    buf = swg.device_alloc(m.numel() * 16) if rank > 0 else None
                    u["pin"].append(buf)
                    mine_h.append(swg.ipc_export(buf) if buf else None)
            every = [None] * world
            self.dist.all_gather_object(every, mine_h)
            k = 0
            for u in self.units:
                u["pout"] = []
                for i, r in enumerate(u["reqs"]):
                    peer = None if last else swg.ipc_import(every[rank + 1][k])
                    u["pout"].append(peer)
                    r.partial_in, r.partial_out = u["pin"][i], peer
                    k += 1
                if not last:
                    u["maps"] = [m[:0] for m in u["maps"]]  # no scores off the last rank
                u["token"] = torch.zeros(1, dtype=torch.float32,
                                         device="cpu" if self.share else "cuda")
            return
        # NCCL: received from rank-1, sent to rank+1
        for u in self.units:
            u["pin"] = [torch.empty(tuple(m.shape) + (2,), dtype=torch.float64,
                                    device="cuda") if rank > 0 else None for m in u["maps"]]
            u["pout"] = [None if last else torch.empty(tuple(m.shape) + (2,),
                                                       dtype=torch.float64, device="cuda")
                         for m in u["maps"]]
            for i, r in enumerate(u["reqs"]):
                r.partial_in, r.partial_out = u["pin"][i], u["pout"][i]
            if not last:
                u["maps"] = [m[:0] for m in u["maps"]]  # no scores off the last rank

    def _attach_bin_walk(self, u):
        """Bins walked in ranges on this GPU with the running sums chained range
        to range (the partial-sum chain of the multi-GPU bin split): 1/nchunk of
        the decay planes per sweep, so a window's corner rows stay in L2."""
        torch = self.torch
        nchunk = self.group_chunks(self.wl["groups"][u["g"]])
        if nchunk <= 1:
            u["chunks"] = [(None, u["reqs"])]
            return
        from dataclasses import replace
        from paper_1705_03524_b200 import dist as D
        ranges = D.bin_ranges(self.nb, nchunk)
        bufs = [[torch.empty(tuple(m.shape) + (2,), dtype=torch.float64, device="cuda")
                 for _ in range(2)] for m in u["maps"]]
        u["chunks"] = []
        for c, (b0, _) in enumerate(ranges):
            creqs = [replace(r, partial_in=bufs[i][(c - 1) % 2] if c else None,
                             partial_out=bufs[i][c % 2] if c < nchunk - 1 else None)
                     for i, r in enumerate(u["reqs"])]
            u["chunks"].append((b0, creqs))
        u["bins_per_launch"] = ranges[0][1] - ranges[0][0]

    def build_units(self):
        kind = self.wl["kind"]
        if kind == "frame":
            self._frame_units()
        elif kind == "sequence":
            self._sequence_units()
        else:
            self._band_units()
        for u in self.units:
            u["peaks"] = self.torch.zeros(len(u["reqs"]), 3, dtype=self.torch.float64,
                                          device="cuda")
            self._attach_bin_walk(u)
        if kind == "sequence":
            self.n_win = sum(m.numel() for m in self.units[0]["maps"]) * len(self.units)
        else:
            self.n_win = sum(m.numel() for u in self.units for m in u["maps"])
        self.chained = any("pin" in u for u in self.units)
        self.flush = self.torch.empty(256 << 20, dtype=self.torch.uint8, device="cuda")

    # ------------------------------------------------------------ the step
    def p2p_send(self, x, dst):  # NCCL over NVLink; gloo (shared-GPU test mode) stages on the host
        if self.share:
            self.dist.send(x.cpu(), dst=dst)
        else:
            self.dist.send(x, dst=dst)

    def p2p_recv(self, x, src):
        if self.share:
            h = self.torch.empty(x.shape, dtype=x.dtype)
            self.dist.recv(h, src=src)
            x.copy_(h)
        else:
            self.dist.recv(x, src=src)

    def _chain_sweep(self, u, i, r):
        """One request of the rank-to-rank bin chain: receive, sweep, send."""
        rank, world = self.rank, self.world
        if rank > 0:
            if "token" in u:  # the sums are already in u["pin"][i]
                self.p2p_recv(u["token"], rank - 1)
            else:
                self.p2p_recv(u["pin"][i], rank - 1)
        u["t"].likelihood_maps([r], scores="none",
                               scores_dev=None if r.partial_out is not None else [u["maps"][i]],
                               peaks_dev=u["peaks"][i])
        if rank < world - 1:
            if "token" in u:  # stream-ordered behind the sweep's peer stores
                if self.share:
                    self.torch.cuda.synchronize()
                self.p2p_send(u["token"], rank + 1)
            else:
                self.p2p_send(u["pout"][i], rank + 1)

    def step(self, ev=None):
        """One pass of the hot path.  ev: per-launch timing events (eager)."""
        units = self.units
        if ev is None and self.batch_peaks is not None:
            # the tracking batch through swg_likelihood_batch: frames round-robin
            # over the library's table sets / worker streams (build of one
            # frame overlaps the sweeps of another)
            units[0]["t"].likelihood_batch([u["src"] for u in units], units[0]["reqs"],
                                           pitch=units[0]["pitch"], peaks_dev=self.batch_peaks)
            return
        j = 0
        for u in units:
            for c, (b0, creqs) in enumerate(u["chunks"]):
                if ev:
                    ev[j].record()
                    j += 1
                if len(u["chunks"]) == 1:
                    # the frame's tables, the units its requests read (octets /
                    # bin pairs of the models' nonzero bins; swg_tables_rebuild_for)
                    u["t"].rebuild_for(u["src"], u["reqs"], u["pitch"])
                else:  # bin-range walk: the new frame with the first range, then ranges
                    u["t"].rebuild_bins(b0, u["src"] if c == 0 else None, u["pitch"])
                if ev:
                    ev[j].record()
                    j += 1
                last = c == len(u["chunks"]) - 1
                if ev is None and "pin" not in u:
                    # one call for all scales: the library overlaps their sweeps
                    # on its worker streams (the per-scale timing path below
                    # records an event between scales instead)
                    u["t"].likelihood_maps(creqs, scores="none",
                                           scores_dev=u["maps"] if last else None,
                                           peaks_dev=u["peaks"])
                    continue
                for bt in self._batches(u, c, creqs):
                    if len(bt) > 1:  # a multi-scale cake launch: its scales in one call
                        u["t"].likelihood_maps([creqs[i] for i in bt], scores="none",
                                               scores_dev=[u["maps"][i] for i in bt],
                                               peaks_dev=u["bpeaks"])
                    elif "pin" in u:
                        self._chain_sweep(u, bt[0], creqs[bt[0]])
                    else:
                        i, r = bt[0], creqs[bt[0]]
                        u["t"].likelihood_maps([r], scores="none",
                                               scores_dev=None if r.partial_out is not None
                                               else [u["maps"][i]], peaks_dev=u["peaks"][i])
                    if ev:
                        ev[j].record()
                        j += 1

    def _batches(self, u, c, creqs):
        """The per-launch timing path's calls for chunk c of unit u: one call
        per request, except the requests the library sweeps in one
        multi-scale cake launch (swg_request_groups), which share a call."""
        key = ("batches", c)
        if key not in u:
            gid = u["t"].request_groups(creqs) if "pin" not in u else [-1] * len(creqs)
            out, seen = [], {}
            for i, g in enumerate(gid):
                if g < 0:
                    out.append([i])
                elif g not in seen:
                    seen[g] = len(out)
                    out.append([i])
                else:
                    out[seen[g]].append(i)
            u[key] = out
            u["bpeaks"] = self.torch.zeros(len(creqs), 3, dtype=self.torch.float64,
                                           device="cuda")
        return u[key]

    # ------------------------------------------------------------ timing
    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def reduce_ranks(self, v, op="max"):
        if not self.dist:
            return float(v)
        t = self.torch.tensor([float(v)], device="cpu" if self.share else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def time_device(self):
        """Per-launch events over K eager steps, then (headline) K graph replays.

        Returns (per-step ms, eager events, clocks, launches over the K steps)."""
        torch, args = self.torch, self.args
        for _ in range(args.warmup):
            self.step()
        torch.cuda.synchronize()
        # the step as one CUDA graph (no host launch gaps between the kernels)
        graph = None
        if not args.no_graph and not self.chained and self.units:  # (p2p chain: eager)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=self.stream):
                self.step()
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize()

        nev = sum(2 + len(self._batches(u, c, cr)) for u in self.units
                  for c, (_, cr) in enumerate(u["chunks"]))
        events = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)]
                  for _ in range(args.steps)]
        clocks = Clocks(self.local)
        self.barrier()
        torch.cuda.synchronize()
        clocks.start()
        t_host = time.perf_counter()
        l0 = self.ctx.launches
        self.step()
        step_launches = self.ctx.launches - l0  # the step the graph replays
        torch.cuda.synchronize()
        enqueue_s = time.perf_counter() - t_host  # host time of one eager step (sizes the spin)
        launches0 = self.ctx.launches
        for s in range(args.steps):
            # a spin longer than the host's enqueue time lets the whole step queue
            # up before the GPU reaches it, so the per-kernel events carry no host
            # launch gaps
            torch.cuda._sleep(int(max(2e6, 2.5e9 * enqueue_s)))
            self.flush.zero_()  # evict L2 (256 MiB > 126 MB) between timed steps; not timed
            self.step(events[s])
        torch.cuda.synchronize()
        clk = clocks.stop()
        launches = self.ctx.launches - launches0  # over the K timed (per-launch) steps
        self.barrier()
        per_step = [events[s][0].elapsed_time(events[s][-1]) for s in range(args.steps)]
        if graph is not None:  # headline timing: graph replays (same kernels, no launch gaps)
            launches = step_launches * args.steps  # the replayed step's kernels
            gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)]
                   for _ in range(args.steps)]
            self.barrier()
            torch.cuda.synchronize()
            clocks = Clocks(self.local)
            clocks.start()
            # soak: keep the GPU under this load for >= 1 s so the clock sampler
            # (100 ms period) sees it; the timed steps follow immediately
            t_soak = time.perf_counter()
            while time.perf_counter() - t_soak < 1.0:
                for _ in range(4):
                    graph.replay()
                torch.cuda.synchronize()
            for s in range(args.steps):
                self.flush.zero_()
                gev[s][0].record()
                graph.replay()
                gev[s][1].record()
            torch.cuda.synchronize()
            clk = clocks.stop()
            self.barrier()
            per_step = [gev[s][0].elapsed_time(gev[s][1]) for s in range(args.steps)]
        return per_step, events, clk, launches

    def launch_times(self, events):
        """Per-launch ms from the eager events: builds, and sweeps per
        (unit, request index) -- one entry per timed step and bin range."""
        build_ms, sweep_ms = [], {}
        for e in events:
            j = 0
            for ui, u in enumerate(self.units):
                for c, (_, creqs) in enumerate(u["chunks"]):
                    build_ms.append(e[j].elapsed_time(e[j + 1]))
                    j += 1
                    for bt in self._batches(u, c, creqs):
                        key = (ui, bt[0]) if len(bt) == 1 else (ui, tuple(bt))
                        sweep_ms.setdefault(key, []).append(e[j].elapsed_time(e[j + 1]))
                        j += 1
                    j += 1
        return build_ms, sweep_ms

    def peaks_on_targets(self):
        """Spot check of the timed outputs: peaks on the planted targets."""
        wl, data = self.wl, self.data
        if wl["kind"] == "frame":
            # every rank's row-chunk peaks -> each request's frame peak
            # (reference tie rule), then the planted targets
            from paper_1705_03524_b200 import dist as D
            parts, widths = [], {}
            for u in self.units:
                pk = u["peaks"].cpu().numpy()
                for i, si in enumerate(u["sidx"]):
                    ints = pk[i, :2].view(np.int32)
                    mw = u["maps"][i].shape[1]
                    key = (u["g"], si)
                    parts.append((key, u["rows"][i], float(pk[i, 2]),
                                  int(ints[1]) * mw + int(ints[0]) - u["rows"][i][0] * mw))
            if self.dist:
                every = [None] * self.world
                self.dist.all_gather_object(every, parts)
                parts = [p for e in every for p in e]
            H, W = data.image.shape[:2]
            for gi, g in enumerate(wl["groups"]):
                for si, sc in enumerate(g["scales"]):
                    widths[(gi, si)] = W - sc[0].kw + 1
            best = D.combine_request_peaks(parts, widths)
            self.frame_peaks = best
            ok = len(best) == sum(len(g["scales"]) for g in wl["groups"])
            for (gi, si), (_, idx) in best.items():
                k, _, _, ti = wl["groups"][gi]["scales"][si]
                if ti is None:
                    continue
                tx, ty = target_center(data, ti)
                mw = widths[(gi, si)]
                ok &= abs(idx % mw + k.hx - tx) <= 1 and abs(idx // mw + k.hy - ty) <= 1
            return bool(ok)
        if wl["kind"] == "sequence":
            hits = tot = 0
            for u in self.units:
                pk = u["peaks"].cpu().numpy()
                gx, gy = data.track[u["frame"]]
                for i in range(len(u["reqs"])):
                    ints = pk[i, :2].view(np.int32)
                    cx, cy = int(ints[2]) + u["origin"][0], int(ints[3]) + u["origin"][1]
                    hits += abs(cx - gx) <= 2 and abs(cy - gy) <= 2
                    tot += 1
            return f"{hits}/{tot} frame-scale peaks within 2 px of ground truth"
        return None

    # ------------------------------------------------------------ e2e
    def _e2e_sequence(self):
        """c3: the frames' search regions from pinned host memory through
        swg_likelihood_batch, host peaks out."""
        import ctypes as C
        from paper_1705_03524_b200.swg import Peak, _check, lib
        swg, data, units = self.swg, self.data, self.units
        (H, W), S = self.frame_hw, self.search
        pin = swg.PinnedBuffer(data.frames.shape, np.uint8)
        pin.array[...] = data.frames
        base = pin.array.ctypes.data
        addrs = [base + ((u["frame"] * H + u["origin"][1]) * W + u["origin"][0]) * 3
                 for u in units]
        fr = (C.c_void_p * len(addrs))(*addrs)
        t = units[0]["t"]
        creqs, _keep = swg.Tables._creqs(units[0]["reqs"], self.nb)
        nreq = len(units[0]["reqs"])
        peaks_host = (Peak * (len(addrs) * nreq))()

        def e2e_step():
            _check(lib().swg_likelihood_batch(t._h, len(addrs), C.addressof(fr), 0, W * 3,
                                              nreq, C.addressof(creqs),
                                              C.addressof(peaks_host), None))
        keep = (pin, fr, creqs, _keep, peaks_host)
        return e2e_step, None, len(addrs) * S * S * 3, C.sizeof(peaks_host), keep

    def _e2e_tables(self):
        """Frames / bands: rebuild from the pinned host frame, host maps + peaks out."""
        import ctypes as C
        from paper_1705_03524_b200.swg import Peak, _check, lib
        swg, data, units, nb = self.swg, self.data, self.units, self.nb
        pin = swg.PinnedBuffer(data.image.shape, data.image.dtype)
        pin.array[...] = data.image
        pin_t = self.torch.from_numpy(pin.array)
        # the frame is uploaded ONCE per step (pinned -> device, stream
        # ordered); every table set's rebuild reads the device copy
        fdev = self.torch.empty(pin_t.shape, dtype=pin_t.dtype, device="cuda")
        row_bytes = data.image.strides[0]
        calls, maps_pin = [], []
        h2d, d2h = data.image.nbytes, 0
        for u in units:
            mp = [swg.PinnedBuffer(tuple(m.shape), np.float64) for m in u["maps"]]
            maps_pin.append(mp)
            hp = (C.c_void_p * len(mp))(*[m.array.ctypes.data for m in mp])
            # peaks in page-locked memory too: an async copy into pageable
            # memory would block the host until the sweeps are done
            pkb = swg.PinnedBuffer((C.sizeof(Peak) * len(u["reqs"]),), np.uint8)
            mp.append(pkb)
            pk = (Peak * len(u["reqs"])).from_address(pkb.array.ctypes.data)
            src = fdev.data_ptr() + u.get("p0", 0) * row_bytes
            # per bin range (one range unless the bins are walked in chunks):
            # rebuild (upload the frame on the first), requests; host maps
            # and peaks from the last range
            for c, (b0, cr) in enumerate(u["chunks"]):
                creqs, keep = swg.Tables._creqs(cr, nb)
                last = c == len(u["chunks"]) - 1
                calls.append((u["t"], src if c == 0 else None, b0, len(u["chunks"]) > 1,
                              creqs, keep, hp if last else None, pk, len(cr)))
            d2h += sum(m.nbytes for m in mp)  # the maps and the peaks

        def e2e_step():
            # the frame's table sets back to back (swg_likelihood_maps_async:
            # one set's map copies overlap the next set's sweeps), host maps
            # and peaks filled at the context synchronisation
            fdev.copy_(pin_t, non_blocking=True)
            for t, src, b0, walk, creqs, _k, hp, pk, n in calls:
                if walk:  # bin ranges: the frame with the first range, then ranges
                    _check(lib().swg_tables_rebuild_bins(t._h, src, 1 if src else 0, 0, b0))
                else:
                    _check(lib().swg_tables_rebuild_for(t._h, src, 1, 0, n, C.addressof(creqs)))
                _check(lib().swg_likelihood_maps_async(
                    t._h, n, C.addressof(creqs),
                    C.addressof(hp) if hp is not None else None, None, C.addressof(pk), None))
            self.ctx.synchronize()

        def check():
            for u, mp in zip(units, maps_pin):
                for m, mpin in zip(u["maps"], mp[:len(u["maps"])]):
                    assert (mpin.array == m.cpu().numpy()).all()
        return e2e_step, check, h2d, d2h, (pin, calls, maps_pin, fdev, pin_t)

    def e2e(self, job_win):
        """The metric through the C-ABI with pinned host input and host outputs,
        host<->device copies inside the timed region (wall clock per step)."""
        args, torch = self.args, self.torch
        if args.no_e2e or self.chained:
            return None
        if self.wl["kind"] == "sequence":
            e2e_step, check, h2d, d2h, _keep = self._e2e_sequence()
        else:
            e2e_step, check, h2d, d2h, _keep = self._e2e_tables()
        for _ in range(args.warmup):
            e2e_step()
        torch.cuda.synchronize()
        self.barrier()
        e2e_t = []
        for _ in range(args.steps):
            self.flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()  # returns after the host maps + peaks are filled
            e2e_t.append(time.perf_counter() - t0)
        e2e_total = self.reduce_ranks(sum(e2e_t))
        if check:
            check()
        return {"value": job_win * args.steps / e2e_total, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_total / args.steps * 1e3}

    # ------------------------------------------------------------ rooflines
    def _traffic_entry(self, kname, k):
        """The ncu capture of this launch (same kernel AND scale), if committed."""
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            entries = json.load(open(tp)).get(self.args.config) or []
            for tr in entries if isinstance(entries, list) else [entries]:
                if kname in tr.get("kernel", "") and f"{k.kw}x{k.kh} " in tr["kernel"] + " ":
                    return tr
        return None

    def _plan(self, u, i):
        """swg_request_plan of request i of unit u; a bin-range walk (config 4)
        asks about its last range and averages the bins read per range with
        the library's rule (records of the model's nonzero bins: pairs for the
        exponential sweep, octets for the integer stream sweeps)."""
        chunks = u.get("chunks") or []
        if len(chunks) <= 1:
            return u["t"].request_plan(u["reqs"][i])
        import numpy as np
        from paper_1705_03524_b200 import dist as D
        pl = dict(u["t"].request_plan(chunks[-1][1][i]))
        grp = {"k_sweep_exp": 2, "k_stream_affine": 8, "k_stream_affine16": 8,
               "k_stream_quad": 8, "k_sweep_affine": 8, "k_sweep_affine16": 8,
               "k_sweep_quad": 8}.get(pl["kernel"])
        if grp and os.environ.get("SWG_SPARSE", "1") != "0":
            m = np.asarray(u["reqs"][i].model)
            per = []
            for b0, b1 in D.bin_ranges(self.nb, len(chunks)):
                nz = m[b0:b1] != 0
                per.append(sum(min(grp, b1 - g) for g in range(b0, b1, grp)
                               if nz[g - b0:g - b0 + grp].any()))
            pl["bins_read"] = sum(per) / len(per)
        return pl

    def kernel_table(self, build_ms, sweep_ms):
        """Per kernel function: launches, ms and algorithmic bytes per step
        (the table rows a launch's windows read, each once, + 8 B
        per window; builds: input + every plane entry written once), and the
        per-launch list.  The dominant kernel is the one with the largest
        share of the step."""
        swg, wl, steps = self.swg, self.wl, self.args.steps
        hbm, _ = peaks_json()
        kt = {}
        W = self.tab_w
        for (ui, i), ts in sweep_ms.items():
            u = self.units[ui]
            g = wl["groups"][u["g"]]
            if isinstance(i, tuple):  # one multi-scale cake launch over these scales
                ks = sorted((g["scales"][u["sidx"][x]][0] for x in i), key=lambda k: -k.kw)
                hmin = min(k.kw for k in ks)
                bins = self.nb
                # algorithmic: the table's records once (16-bit, one plane)
                # + 8 B per window of every scale
                win = sum((self.tab_h - k.kh + 1) * (self.tab_w - k.kw + 1) for k in ks)
                byts = (self.tab_h + 1) * (W + 1) * bins * 2 + 8 * win
                ms = sum(ts) / len(ts)
                ent = kt.setdefault("k_sweep_cake16_multi", {"launches_per_step": 0,
                                                             "ms_per_step": 0.0,
                                                             "bytes_per_step": 0,
                                                             "launches": []})
                n = len(ts) // steps
                ent["launches_per_step"] += n
                ent["ms_per_step"] += ms * n
                ent["bytes_per_step"] += byts * n
                ent["launches"].append({"window": "/".join(f"{k.kw}x{k.kh}" for k in ks),
                                        "rows": int(self.tab_h - hmin + 1), "bins": int(bins),
                                        "ms": ms, "bytes": int(byts),
                                        "hbm_frac": byts / (ms / 1e3) / 1e9 / hbm})
                continue
            k, meth = g["scales"][u["sidx"][i]][:2]
            r = u["reqs"][i]
            # the library's own report of what it runs (swg_request_plan):
            # kernel, planes, entry bytes and the bins whose records it reads
            # (a model's zero bins are skipped by the closed-form-mass sweeps)
            pl = self._plan(u, i)
            kname, P, e = pl["kernel"], pl["planes"], pl["entry_bytes"]
            bins = pl["bins_read"]
            rows = r.rows[1] - r.rows[0] if r.rows else self.tab_h - k.kh + 1
            mw = self.tab_w - k.kw + 1
            win = rows * mw
            byts = min(self.tab_h + 1, rows + k.kh) * (W + 1) * bins * P * e + 8 * win
            ms = sum(ts) / len(ts)
            ent = kt.setdefault(kname, {"launches_per_step": 0, "ms_per_step": 0.0,
                                        "bytes_per_step": 0, "launches": []})
            n = len(ts) // steps
            ent["launches_per_step"] += n
            ent["ms_per_step"] += ms * n
            ent["bytes_per_step"] += byts * n
            ent["launches"].append({"window": f"{k.kw}x{k.kh}", "rows": int(rows),
                                    "bins": int(bins), "ms": ms, "bytes": int(byts),
                                    "hbm_frac": byts / (ms / 1e3) / 1e9 / hbm})
        if build_ms:
            bms = sum(build_ms) / steps
            in_bytes = sum(u["h2d"] for u in self.units)
            # plane bytes the builds wrote (the library's count: a model-driven
            # rebuild writes only the units its requests read); a bin-range
            # walk rebuilds every range's planes
            bb = in_bytes + sum(
                u["t"].built_bytes() if len(u.get("chunks") or []) <= 1 else group_build_bytes(
                    wl["groups"][u["g"]], self.tab_w, self.tab_h, self.nb,
                    narrow=any(self._plan(u, i)["kernel"].endswith("affine16")
                               for i in range(len(u["reqs"])))) for u in self.units)
            kt["ih_build"] = {"launches_per_step": len(build_ms) // steps, "ms_per_step": bms,
                              "bytes_per_step": int(bb), "launches": [],
                              "kernels": "k_quantize + k_colsum + k_bandscan + k_build / "
                                         "k_build_fused (+ decayed: k_flip, k_colsum_decay, "
                                         "k_bandscan_decay, k_build_decay_warp)"}
        for ent in kt.values():
            ent["gbps"] = ent["bytes_per_step"] / (ent["ms_per_step"] / 1e3) / 1e9
            ent["hbm_frac"] = ent["gbps"] / hbm
        return kt

    def sweep_roofline(self, kt, clk):
        """`roofline` of the kernel with the largest share of the step: its
        algorithmic bytes per launch / its average launch time (summed over
        its launches in a step), against the measured HBM copy bandwidth."""
        hbm, src = peaks_json()
        dom = max(kt, key=lambda n: kt[n]["ms_per_step"])
        ent = kt[dom]
        step_ms = sum(e["ms_per_step"] for e in kt.values())
        roofline = {"bound": "hbm", "achieved": ent["gbps"], "peak": hbm, "unit": "GB/s",
                    "frac": ent["hbm_frac"], "traffic": None, "peak_source": src,
                    "kernel": dom, "share_of_step": ent["ms_per_step"] / step_ms,
                    "launches_per_step": ent["launches_per_step"],
                    "bytes_per_step": ent["bytes_per_step"],
                    "avg_launch_ms": ent["ms_per_step"] / max(ent["launches_per_step"], 1)}
        # ncu DRAM bytes of one launch of this kernel (profiles/traffic.json,
        # this config), next to that launch's algorithmic bytes
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            entries = json.load(open(tp)).get(self.args.config) or []
            for tr in entries if isinstance(entries, list) else [entries]:
                if not tr.get("kernel", "").startswith(dom):
                    continue
                for ln in ent["launches"]:
                    if f" {ln['window']} " in " " + tr["kernel"].replace("at ", "") + " ":
                        roofline["traffic"] = tr["dram_bytes"]
                        roofline["traffic_launch"] = {"window": ln["window"],
                                                      "algorithmic_bytes": ln["bytes"],
                                                      "ncu_source": tr.get("source")}
                        break
                if roofline["traffic"] is not None:
                    break
        if dom.startswith("k_sweep_cake"):
            # the ring telescope reads 4 corner records per ring, octet and
            # window from L1 (O(rings*b) on-chip bytes per window):
            # its roofline is the L1 data pipe, measured by ncu on one launch
            # (profiles/onchip.json), not HBM
            roofline["onchip"] = {"note": "the wedding-cake sweep is bound by the L1 -> register "
                                          "data path (ring corners, O(rings*bins) per window), "
                                          "not HBM"}
            op = os.path.join(ROOT, "profiles", "onchip.json")
            if os.path.exists(op):
                oc = json.load(open(op)).get(self.args.config)
                if oc:
                    roofline["onchip"].update(oc)
        return roofline

    def cpu_baseline(self):
        if self.world != 1 or self.args.no_cpu_baseline:
            return None
        c = cpu_reference(self.wl, self.data, self.models, public_api=True)
        cpu = {"value": c["value"], "unit": UNIT, "cores": c["threads"], "kind": c["kind"],
               "sample": cpu_sample_text(self.wl, c)}
        if c["public_api"]:
            cpu["public_api_value"] = c["public_api"]
            cpu["public_api_sample"] = ("reference likelihood_map per scale (full maps, "
                                        "tables rebuilt per call, all threads)")
        return cpu

    # ------------------------------------------------------------ the run
    def run(self):
        args, wl = self.args, self.wl
        per_step, events, clk, launches = self.time_device()
        build_ms, sweep_ms = self.launch_times(events)
        total_ms = self.reduce_ranks(sum(per_step))
        job_win = self.reduce_ranks(self.n_win, op="sum")
        value = job_win * args.steps / (total_ms / 1e3)
        ok_peaks = self.peaks_on_targets()
        e2e = self.e2e(job_win)
        if self.rank != 0:
            if self.dist:
                self.dist.destroy_process_group()
            return
        kt = self.kernel_table(build_ms, sweep_ms)
        roofline = self.sweep_roofline(kt, clk)
        cpu = self.cpu_baseline()
        kinds = ["uniform", "manhattan", "chebyshev", "gauss_cheb", "euclid_quad", "exp_l1"]
        per_scale = {}
        for (ui, i), ts in sweep_ms.items():
            u = self.units[ui]
            scs = sorted((wl["groups"][u["g"]]["scales"][u["sidx"][x]]
                          for x in (i if isinstance(i, tuple) else (i,))), key=lambda sc: -sc[0].kw)
            key = kinds[scs[0][0].kind] + "/".join(f"{sc[0].kw}x{sc[0].kh}" for sc in scs)
            per_scale[key] = per_scale.get(key, 0.0) + sum(ts) / args.steps
        ih = kt.get("ih_build")
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": self.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None,
            "dtype": "u16/u32 integral tables (f64 decay tables) + f64 scores",
            "data": "synthetic (seeded generators in paper_1705_03524_b200/synth.py)",
            "config": config_dict(wl, job_win),
            "parallelism": (f"bin ranges chained over {self.world} GPU(s) (p2p partial sums)"
                            if self.chained else
                            f"one frame's (kernel, scale) requests over {self.world} GPU(s) "
                            f"(LPT, row-split; tables built per rank), no collective"
                            if wl["kind"] == "frame" else
                            f"{wl['kind']} sharded over {self.world} GPU(s), no collective"),
            "tables": {"shape": [self.tab_w, self.tab_h], "units_rank0": len(self.units)},
            "plan": ({"load_ms_per_rank": self.plan_load, "costs": self.plan_costs}
                     if getattr(self, "plan_load", None) else None),
            "ih_build": ({"ms": ih["ms_per_step"], "gbps": ih["gbps"], "frac": ih["hbm_frac"],
                          "bytes": ih["bytes_per_step"]} if ih else None),
            "per_scale_ms": per_scale,
            "kernels": {n: {k: v for k, v in e.items() if k != "launches"} | (
                {"launches": e["launches"]} if n != "ih_build" else {}) for n, e in kt.items()},
            "roofline": roofline,
            "e2e": e2e, "gpu_launches": launches, "gpu_launches_per_step": launches // args.steps,
            "peaks_on_targets": ok_peaks, "cpu_baseline": cpu, "clocks": clk,
        }
        print(json.dumps(out), flush=True)
        if self.dist:
            self.dist.destroy_process_group()


def main():
    args = parse_args()
    wl = workload(args.config, args.exp_decay)
    if args.impl == "reference":
        return run_reference(args, wl, int(os.environ.get("RANK", 0)),
                             int(os.environ.get("WORLD_SIZE", 1)))
    OursArm(args, wl).run()


def run_reference(args, wl, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1705_03524_b200 import swg, synth
    data = wl["gen"](1)
    # models with the reference's own target_model_for_method (matching.cpp:84-106)
    # where it applies; the oracle restatement for the declared formats/kernels
    R = O.Ref()
    orc = O.Oracle()
    models = []
    for g in wl["groups"]:
        ms = []
        for k, method, rings, ti in g["scales"]:
            if wl["kind"] == "sequence":
                cx, cy = data.track[0]
                img = data.frames[0]
            else:
                cx, cy = target_center(data, ti)
                img = data.image
            templ = synth.crop(img, cx, cy, k.kw, k.kh)
            ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
            if wl["fmt"] == swg.FMT_GRAY8 and k.kind in (swg.MANHATTAN, swg.UNIFORM,
                                                         swg.GAUSS_CHEB):
                ms.append(R.target_model(templ, wl["bins"], ok, method, rings))
            else:
                ms.append(orc.target_model(_quantize_host(wl, templ), wl["nbins"], ok,
                                           O.BRUTE if method == swg.SWIH and
                                           k.kind not in (swg.MANHATTAN, swg.UNIFORM)
                                           else method, rings))
        models.append(ms)
    vals = []
    for s in range(args.warmup + args.steps):
        c = cpu_reference(wl, data, models, budget_s=max(60.0 / (args.warmup + args.steps), 1.5))
        if s >= args.warmup:
            vals.append(c)
    value = statistics.mean(v["value"] for v in vals)
    n_win = vals[0]["frame_windows"]
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": n_win / value * 1e3, "higher_is_better": True,
        "scaling": wl["scaling"], "vs_baseline": None, "dtype": "i64+f64", "impl": "reference",
        "data": "synthetic (same generator and seed as --impl ours)",
        "config": config_dict(wl, n_win),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": vals[0]["threads"],
                         "kind": vals[0]["kind"], "sample": "per step: " + cpu_sample_text(wl, vals[0])},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
