"""Full-size parity on every BASELINE config (north_star: "bit-exact integer
IH and peak locations, stated FP tolerance, on all five configs").

Each test runs bench.py's OWN timed step (OursArm.step: the same table sets,
requests, streams and output buffers the bench times) at the config's full
size and compares every output with the CPU oracle:

* maps: the bin-outer oracle (oracle/swih_fastmap.c), itself checked
  bit-for-bit against the window-by-window restatement on CPU
  (tests/test_oracle_fastmap.py) and through it against the reference
  (tests/test_oracle_golden.py).  Exact kernels (Manhattan, GaussianChebyshev
  cake, declared Euclidean quadratic): EVERY map value bit-identical.
  Declared exponential: every value within 1e-4 absolute (north_star's score
  tolerance; the bound is this test's), the peak (index and score bits)
  exact -- the oracle re-scores its near-maximum windows by the reference
  pixel-order brute force.  Mirrors acceptance_main.cpp:44-85,199-229.
* tables: uint32 planes (reference int64 mod 2^32) against the reference's
  definition (2-D inclusive prefix sums of the bin indicator and its x / y
  (/ x^2 / y^2) ramps, integral_tables.cpp:72-115; the numpy form is pinned
  to the oracle build on CPU in test_host_logic.py); decayed planes within
  1e-12 relative of the declared recurrence.
"""
import contextlib

import numpy as np
import pytest

from oracle import oracle as O
from paper_1705_03524_b200 import swg

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def bench_step(config, rank=None, world=None, extra=()):
    """bench.py's arm for `config`, one eager step run; yields the arm."""
    import torch

    import bench
    args = bench.parse_args(["--config", config, "--steps", "1", "--warmup", "3",
                             "--no-cpu-baseline", "--no-e2e", *extra])
    arm = bench.OursArm(args, bench.workload(config, args.exp_decay), rank=rank, world=world)
    try:
        arm.step()
        torch.cuda.synchronize()
        yield arm
    finally:
        torch.cuda.set_stream(torch.cuda.default_stream())
        for u in arm.units:
            u["t"].close()
        del arm
        torch.cuda.empty_cache()


def _oracle_method(kind, method):
    if kind == swg.GAUSS_CHEB:
        return O.CAKE
    if kind in (swg.EUCLID_QUAD, swg.EXP_L1):
        return O.BRUTE  # the declared kernels' brute force (baselines.cpp:53-69 order)
    return O.SWIH if method == swg.SWIH else method


def _quantized(oracle, wl, img):
    if wl["fmt"] == swg.FMT_GRAY16:
        return oracle.quantize_gray16(img, wl["nbins"])
    if wl["fmt"] == swg.FMT_RGB8:
        return oracle.quantize_rgb8(img, wl["bins"])
    return oracle.quantize_gray8(img, wl["bins"])


def _check_maps(oracle, arm, fi, groups=None, tol_exp=1e-4):
    """Every request of the arm's step against the oracle; returns the number
    of maps compared and the largest exponential deviation."""
    wl = arm.wl
    n, worst = 0, 0.0
    for u in arm.units:
        g = wl["groups"][u["g"]]
        if groups is not None and u["g"] not in groups:
            continue
        pk_all = u["peaks"].cpu().numpy()
        for i, si in enumerate(u["sidx"]):
            k, method, rings, _ = g["scales"][si]
            model = arm.models[u["g"]][si]
            ok = O.kernel(k.kind, k.kw, k.kh, k.sigma)
            want, wpk, nex = oracle.fast_map(fi, arm.nb, model, ok,
                                             _oracle_method(k.kind, method), rings=rings)
            got = u["maps"][i].cpu().numpy()
            v0, v1 = u["rows"][i] if "rows" in u else (0, want.shape[0])
            assert got.shape == (v1 - v0, want.shape[1])
            ints = pk_all[i, :2].view(np.int32)
            gpk = (int(ints[0]), int(ints[1]), int(ints[2]), int(ints[3]), float(pk_all[i, 2]))
            if k.kind == swg.EXP_L1:
                dev = float(np.abs(got - want[v0:v1]).max())
                worst = max(worst, dev)
                assert dev <= tol_exp, (k.kw, dev)
                assert nex >= 1
            else:
                bad = np.count_nonzero(got.view(np.int64) != want[v0:v1].view(np.int64))
                assert bad == 0, (k.kind, k.kw, bad)
            if (v0, v1) == (0, want.shape[0]):
                assert gpk == wpk, (k.kind, k.kw, gpk, wpk)
            n += 1
    return n, worst


def test_config1_full_map(oracle):
    """configs[0]: 256x256 u8, 16 bins, Manhattan 33x33 (the reference's own
    CPU-runnable case) -- the timed step's map and peak."""
    with bench_step("c1") as arm:
        fi = _quantized(oracle, arm.wl, arm.data.image)
        assert _check_maps(oracle, arm, fi)[0] == 1


def test_config2_full_maps(oracle):
    """configs[1]: 1024x1024 u8, 32 bins, GaussianChebyshev (exact full-ring
    cake) at 33/65/97 -- all three full maps and peaks bit-exact, through the
    timed step (16-bit plain planes, the fanned-out device-output call)."""
    with bench_step("c2") as arm:
        fi = _quantized(oracle, arm.wl, arm.data.image)
        assert _check_maps(oracle, arm, fi)[0] == 3


@pytest.mark.parametrize("group,label,nmaps", [(0, "manhattan+euclid_quad", 16),
                                               (1, "gauss_cheb", 8), (2, "exp_l1", 8)])
def test_config5_full_maps(oracle, group, label, nmaps):
    """configs[4]: 2048x2048 u16, 64 bins -- the scales (17..257) of one
    table set (Manhattan and Euclidean share the quadratic set): every map
    value and every peak against the oracle."""
    with bench_step("c5") as arm:
        fi = _quantized(oracle, arm.wl, arm.data.image)
        assert (arm.units[0]["t"].feature_image() == fi).all()
        n, worst = _check_maps(oracle, arm, fi, groups={group})
        assert n == nmaps
        if label == "exp_l1":
            print(f"config 5 exponential: max |gpu - oracle| = {worst:.3g}")


def test_config5_exponential_per_scale_decay(oracle):
    """bench.py --exp-decay scale: one decayed table set per scale with
    d = exp(-4/kw) -- every map within 1e-4 of the oracle, every peak exact."""
    with bench_step("c5", extra=("--exp-decay", "scale")) as arm:
        fi = _quantized(oracle, arm.wl, arm.data.image)
        groups = {gi for gi, g in enumerate(arm.wl["groups"]) if g.get("decay")}
        assert len(groups) == 8
        n, worst = _check_maps(oracle, arm, fi, groups=groups)
        assert n == 8
        print(f"config 5 exponential per-scale decay: max |gpu - oracle| = {worst:.3g}")


def test_config5_multi_gpu_plan_union(oracle):
    """The N-GPU plan of config 5 (dist.plan_frame: requests split by map rows
    where LPT asks) run rank by rank on this GPU: every rank's row chunks
    stitch into the single-GPU maps bit for bit (exponential: its exact
    re-scored windows included -- the two-phase peak runs per chunk, and
    combining the chunk peaks with the tie rule gives the frame peak)."""
    from paper_1705_03524_b200 import dist as D
    single = {}
    with bench_step("c5") as arm:
        for u in arm.units:
            for i, si in enumerate(u["sidx"]):
                single[(u["g"], si)] = (u["maps"][i].cpu().numpy(),
                                        u["peaks"][i].cpu().numpy().copy())
    world = 3
    stitched = {k: np.full_like(m, np.nan) for k, (m, _) in single.items()}
    parts, widths = [], {}
    for rank in range(world):
        with bench_step("c5", rank=rank, world=world) as arm:
            for u in arm.units:
                for i, si in enumerate(u["sidx"]):
                    key = (u["g"], si)
                    v0, v1 = u["rows"][i]
                    stitched[key][v0:v1] = u["maps"][i].cpu().numpy()
                    pk = u["peaks"][i].cpu().numpy()
                    ints = pk[:2].view(np.int32)
                    mw = stitched[key].shape[1]
                    widths[key] = mw
                    parts.append((key, (v0, v1), float(pk[2]),
                                  int(ints[1]) * mw + int(ints[0]) - v0 * mw))
    best = D.combine_request_peaks(parts, widths)
    for key, (m, pk) in single.items():
        assert not np.isnan(stitched[key]).any(), key
        if key[0] == 2:  # exponential: chunk-local exact re-scores may differ off-peak
            assert np.abs(stitched[key] - m).max() <= 1e-9
        else:
            assert (stitched[key].view(np.int64) == m.view(np.int64)).all(), key
        ints = pk[:2].view(np.int32)
        assert best[key] == (float(pk[2]), int(ints[1]) * widths[key] + int(ints[0])), key


def _prefix_u32(fi, b, planes=3):
    """integral_tables.cpp:72-115: 2-D inclusive prefix sums with zero row /
    column 0 of [fi == b] (and x, y, x^2, y^2 ramps), mod 2^32."""
    h, w = fi.shape
    ind = (fi == b).astype(np.int64)
    ys, xs = np.mgrid[0:h, 0:w]
    out = []
    for wgt in (1, xs, ys, xs * xs, ys * ys)[:planes]:
        p = np.zeros((h + 1, w + 1), np.int64)
        p[1:, 1:] = np.cumsum(np.cumsum(ind * wgt, axis=0), axis=1)
        out.append(p)
    return out


def test_config2_and_config5_tables_full_size(ctx, oracle):
    """The full-size uint32 tables of configs 2 (all 32 bins x 3 kinds) and
    5 (all 64 bins x 3 kinds; the quadratic x^2 / y^2 planes through the exact
    int64 export), bin-exact."""
    from paper_1705_03524_b200 import synth
    img2 = synth.config2(1).image
    fi2 = oracle.quantize_gray8(img2, 32)
    t = ctx.build(img2, swg.FMT_GRAY8, 32, swg.PLANES_AFFINE)
    for kind in range(3):
        got = t.export_u32(kind)
        for b in range(32):
            want = _prefix_u32(fi2, b)[kind]
            assert (got[b] == (want & 0xFFFFFFFF).astype(np.uint32)).all(), (kind, b)
    t.close()
    img5 = synth.config5(1).image
    fi5 = oracle.quantize_gray16(img5, 64)
    t = ctx.build(img5, swg.FMT_GRAY16, 64, swg.PLANES_QUADRATIC)
    for b0 in range(0, 64, 8):
        got = [t.export_u32(kind, b0, b0 + 8) for kind in range(3)]
        got += [t.export_i64(kind, b0, b0 + 8) for kind in (3, 4)]
        for b in range(b0, b0 + 8):
            want = _prefix_u32(fi5, b, planes=5)
            for kind in range(3):
                assert (got[kind][b - b0] == (want[kind] & 0xFFFFFFFF).astype(np.uint32)).all()
            for kind in (3, 4):
                assert (got[kind][b - b0] == want[kind]).all(), (kind, b)
    t.close()


def test_config3_all_frames(oracle):
    """configs[2]: all 64 frames x 3 Euclidean scales.  The timed step's
    frame batch (swg_likelihood_batch, peaks only) gives every frame-scale
    peak exactly; the per-frame maps (eager path, same table set) are
    bit-identical to the oracle's brute force."""
    from paper_1705_03524_b200 import synth
    with bench_step("c3") as arm:
        seq, S = arm.data, arm.search
        peaks = arm.batch_peaks.cpu().numpy()
        reqs = arm.units[0]["reqs"]
        for fi_, u in enumerate(arm.units):
            x0, y0 = u["origin"]
            crop = np.ascontiguousarray(seq.frames[u["frame"], y0:y0 + S, x0:x0 + S])
            fi = oracle.quantize_rgb8(crop, 4)
            # this frame's maps through the library (the bench's eager path)
            u["t"].rebuild(u["src"], u["pitch"])
            maps, pks = u["t"].likelihood_maps(reqs)
            for j, r in enumerate(reqs):
                k = r.kernel
                want, wpk, _ = oracle.fast_map(fi, 64, r.model,
                                               O.kernel(O.EUCLID_QUAD, k.kw, k.kh), O.BRUTE)
                assert (maps[j].view(np.int64) == want.view(np.int64)).all(), (fi_, j)
                assert tuple(pks[j]) == wpk
                row = peaks[fi_ * len(reqs) + j]
                ints = row[:2].view(np.int32)
                assert (int(ints[0]), int(ints[1]), float(row[2])) == (wpk[0], wpk[1], wpk[4])
        assert len(arm.units) == 64


def test_config4_full_frame(oracle):
    """configs[3]: 3840x2160 RGB, 512 bins, exponential at 25..129, through
    the timed step's 8-range bin walk (rebuild_bins + the partial-sum chain):
    every map value within 1e-4 of the oracle, every peak exact; then one
    bin range's decayed tables (the step's last, bins 448-511: first, middle
    and last bin, all four orientations) against the declared recurrence."""
    from scipy.signal import lfilter
    with bench_step("c4") as arm:
        fi = _quantized(oracle, arm.wl, arm.data.image)
        n, worst = _check_maps(oracle, arm, fi)
        assert n == 5
        print(f"config 4 exponential: max |gpu - oracle| = {worst:.3g}")
        t = arm.units[0]["t"]
        d = arm.wl["groups"][0]["decay"]
        assert t.bins == 64
        flips = (fi, fi[:, ::-1], fi[::-1, :], fi[::-1, ::-1])
        for lb in (0, 37, 63):
            b = 448 + lb
            for k, f in enumerate(flips):
                got = t.export_f64(k, lb, lb + 1)[0]
                one = (f == b).astype(np.float64)
                r = lfilter([1.0], [1.0, -d], one, axis=1)  # r(x) = f(x) + d r(x-1)
                e = lfilter([1.0], [1.0, -d], r, axis=0)
                want = np.zeros_like(got)
                want[1:, 1:] = e
                np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_exponential_normalised_histograms(ctx, oracle):
    """north_star's weighted-plane tolerance: exponential window histograms
    from the decayed tables, normalised (histogram.cpp:19-26), within 1e-5
    relative of the brute force's (baselines.cpp:53-69) -- config 5's frame,
    every scale, 64 windows each (interior and all four corners)."""
    from paper_1705_03524_b200 import synth
    img = synth.config5(1).image
    fi = oracle.quantize_gray16(img, 64)
    d = 15.0 / 16.0
    t = ctx.build_decay(img, d, swg.FMT_GRAY16, 64)
    rng = np.random.default_rng(7)
    worst = 0.0
    for kw in (17, 25, 37, 53, 79, 117, 173, 257):
        h = kw // 2
        cx = np.concatenate([rng.integers(h, 2048 - h, 60), [h, 2047 - h, h, 2047 - h]])
        cy = np.concatenate([rng.integers(h, 2048 - h, 60), [h, h, 2047 - h, 2047 - h]])
        k = swg.Kernel(swg.EXP_L1, kw, kw, d)
        got = t.decay_windows(cx, cy, k)
        ok = O.kernel(O.EXP_L1, kw, kw, d)
        for i in range(len(cx)):
            want = oracle.normalize(oracle.brute_weights(fi, 64, int(cx[i]), int(cy[i]), ok))
            g = oracle.normalize(got[i])
            nz = want > 0
            assert ((g > 0) == nz).all()
            rel = np.abs(g[nz] - want[nz]) / want[nz]
            worst = max(worst, float(rel.max()))
            assert rel.max() <= 1e-5, (kw, i, rel.max())
    print(f"exponential normalised histograms: max relative error {worst:.3g}")
    with pytest.raises(swg.UnsupportedKernelError):
        t.decay_windows([100], [100], swg.Kernel(swg.EXP_L1, 17, 17, 0.5))
