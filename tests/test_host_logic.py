"""Host-side logic on CPU: synthetic generators, the bench's
workload / row-band planning, and the exponential kernel's decayed-table
rectangle identity (the algebra k_exp.cu's 16-corner sweep relies on),
checked against the oracle's brute-force weights."""
import numpy as np
import pytest

import bench
from oracle import oracle as O
from paper_1705_03524_b200 import swg, synth


def test_config3_sequence_small():
    seq = synth.config3(3, n_frames=5, h=240, w=400, search=96)
    assert seq.frames.shape == (5, 240, 400, 3) and seq.frames.dtype == np.uint8
    tw, th = seq.size
    for f in range(1, 5):
        dx = seq.track[f][0] - seq.track[f - 1][0]
        dy = seq.track[f][1] - seq.track[f - 1][1]
        assert 0 <= dx <= 4 and 0 <= dy <= 4
    # the target's appearance is pasted unchanged at the ground truth
    patches = [seq.frames[f, cy - th // 2:cy - th // 2 + th, cx - tw // 2:cx - tw // 2 + tw]
               for f, (cx, cy) in enumerate(seq.track)]
    assert all((p == patches[0]).all() for p in patches)
    # open-loop search region: centred on the previous ground truth, clamped
    for f in range(5):
        x0, y0 = synth.search_origin(seq, f)
        assert 0 <= x0 <= 400 - 96 and 0 <= y0 <= 240 - 96
        px, py = seq.track[max(f - 1, 0)]
        assert (x0, y0) == (min(max(px - 48, 0), 304), min(max(py - 48, 0), 144))
    again = synth.config3(3, n_frames=5, h=240, w=400, search=96)
    assert (again.frames == seq.frames).all() and again.track == seq.track


def test_config4_targets_small():
    sc = synth.config4(2, h=270, w=480)
    assert sc.image.shape == (270, 480, 3) and sc.image.dtype == np.uint8
    sizes = [t[2] for t in sc.targets]
    assert len(sizes) == 16 and sizes[0] == 24 and sizes[-1] == 128
    assert sizes == sorted(sizes)


def test_odd_window_mapping():
    # declared even -> odd mapping
    assert [synth.odd_window(s) for s in (32, 64, 96, 48, 24, 128)] == [33, 65, 97, 49, 25, 129]


@pytest.mark.parametrize("H,n_bands", [(2160, 4), (2160, 8), (300, 3), (129, 1)])
def test_band_plan_covers_every_map_row_once(H, n_bands):
    wl = bench.workload("c4")
    scales = wl["groups"][0]["scales"]
    if H < max(k.kh for k, _, _, _ in scales):
        scales = [s for s in scales if s[0].kh <= H]
    BH, plan = bench.band_plan(H, scales, n_bands)
    for si, (k, _, _, _) in enumerate(scales):
        mh = H - k.kh + 1
        covered = []
        for p0, rows in plan:
            v0, v1 = rows[si]
            assert 0 <= p0 and p0 + BH <= H
            if v1 > v0:
                # the band's pixel rows hold every window of its map rows
                assert p0 <= v0 and v1 - 1 + k.kh <= p0 + BH
                covered.extend(range(v0, v1))
        assert covered == list(range(mh))


def test_workloads_and_engines():
    for name in ("c1", "c2", "c3", "c4", "c5", "c5m"):
        wl = bench.workload(name)
        assert wl["kind"] in ("frame", "sequence", "bands")
        for g in wl["groups"]:
            for k, m, rings, _ in g["scales"]:
                assert k.kw % 2 == 1 and k.kh % 2 == 1
                kname, P, e = bench.engine_of(g, k, m)
                assert kname.startswith("k_sweep_") and P in (1, 3, 4, 5) and e in (2, 4, 8)
    c5 = bench.workload("c5")
    kinds = [[k.kind for k, _, _, _ in g["scales"]] for g in c5["groups"]]
    # Manhattan and Euclidean share the quadratic table set ({1, x, y} of {1, x, y, x^2, y^2})
    assert kinds == [[swg.MANHATTAN] * 8 + [swg.EUCLID_QUAD] * 8, [swg.GAUSS_CHEB] * 8,
                     [swg.EXP_L1] * 8]
    quad = c5["groups"][0]
    # Manhattan windows of mass < 2^16 (17, 25, 37) on the narrow 16-bit planes
    assert [bench.engine_of(quad, k, m)[0] for k, m, _, _ in quad["scales"][:8]] == \
        ["k_sweep_affine16"] * 3 + ["k_sweep_affine"] * 5
    assert bench.manhattan_mass(swg.Kernel(swg.MANHATTAN, 49, 49)) < 65536 <= \
        bench.manhattan_mass(swg.Kernel(swg.MANHATTAN, 51, 51))
    assert bench.engine_of(quad, quad["scales"][8][0], swg.SWIH) == ("k_sweep_quad", 5, 4)
    # 257x257 Gaussian: ring 0's box exceeds 16-bit counts, but ring 1's box
    # and ring 0's frame do not -> still the 16-bit sweep (wide ring 0)
    plain = c5["groups"][1]
    assert bench.engine_of(plain, plain["scales"][-1][0], swg.CAKE)[0] == "k_sweep_cake16"
    assert bench.engine_of(plain, swg.Kernel(swg.GAUSS_CHEB, 261, 261, 0.5), swg.CAKE)[0] == \
        "k_sweep_cake"
    assert bench.group_build_bytes(plain, 10, 10, 4) == 11 * 11 * 4 * 2


def _decayed_se(fi, bins, d):
    h, w = fi.shape
    out = np.zeros((bins, h + 1, w + 1))
    for b in range(bins):
        one = (fi == b).astype(np.float64)
        r = np.zeros((h, w + 1))
        for x in range(w):
            r[:, x + 1] = d * r[:, x] + one[:, x]
        for y in range(h):
            out[b, y + 1] = d * out[b, y] + r[y]
    return out


@pytest.mark.parametrize("d,kw,kh", [(0.75, 9, 7), (0.9375, 15, 15), (0.5, 5, 11)])
def test_exponential_rectangle_identity(oracle, d, kw, kh):
    """Quadrant decomposition of w = d^(|dx|+|dy|) over the four flipped
    decayed tables (swg_abi.cu ExpSweep offsets / coefficients) reproduces
    the brute-force weighted histogram (baselines.cpp:53-69) to ~1e-12."""
    h, w = 23, 31
    bins = 5
    img = oracle.random_gray(w, h, 17)
    fi = oracle.quantize_gray8(img, bins)
    flips = [np.ascontiguousarray(f) for f in (fi, fi[:, ::-1], fi[::-1, :], fi[::-1, ::-1])]
    E = [_decayed_se(f, bins, d) for f in flips]
    hx, hy = kw // 2, kh // 2
    ok = O.kernel(O.EXP_L1, kw, kh, d)
    # corner geometry of the four orientations (same tables as the C-ABI fills)
    cx0, cy0 = (1, 0, 1, 0), (1, 1, 0, 0)
    ax, by = (hx + 1, hx, hx + 1, hx), (hy + 1, hy + 1, hy, hy)
    qf = (1.0, d, d, d * d)
    for cy in range(hy, h - hy):
        for cx in range(hx, w - hx):
            acc = np.zeros(bins)
            for o in range(4):
                x = w - 1 - cx if o & 1 else cx
                y = h - 1 - cy if o & 2 else cy
                xs = (cx0[o], cx0[o] - ax[o], cx0[o], cx0[o] - ax[o])
                ys = (cy0[o], cy0[o], cy0[o] - by[o], cy0[o] - by[o])
                cf = (qf[o], -qf[o] * d ** ax[o], -qf[o] * d ** by[o], qf[o] * d ** (ax[o] + by[o]))
                for q in range(4):
                    acc += cf[q] * E[o][:, y + ys[q], x + xs[q]]
            want = oracle.brute_weights(fi, bins, cx, cy, ok)
            np.testing.assert_allclose(acc, want, rtol=0, atol=1e-12)


def test_profiles_traffic_entries_resolve():
    """Every committed ncu traffic entry names a kernel and a scale of its
    config's workload and points at a committed summary holding the DRAM
    bytes it quotes (bench.py's roofline `traffic` comes from these)."""
    import json
    import os
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tr = json.load(open(os.path.join(root, "profiles", "traffic.json")))
    for cfg, entries in tr.items():
        wl = bench.workload(cfg)
        sizes = {f"{k.kw}x{k.kh}" for g in wl["groups"] for k, _, _, _ in g["scales"]}
        for e in entries if isinstance(entries, list) else [entries]:
            assert e["kernel"].startswith(("k_sweep_", "k_stream_")), e
            # one scale, or the scales of one multi-scale cake launch
            scales = re.search(r"\(\s*((?:\d+x\d+/?)+) scales?", e["kernel"]).group(1).split("/")
            assert scales and all(s in sizes for s in scales), (cfg, scales)
            src = os.path.join(root, e["source"])
            assert os.path.exists(src), src
            assert "dram__bytes_read.sum" in open(src).read()
            assert e["dram_bytes"] > 0
