"""The multi-scale cake sweep (k_sweep_cake16_multi): full-ring square
GaussianChebyshev cake maps of one narrow table swept together, each scale
accumulating its own ring coefficients over the box counts shared by all
scales.  Every map and peak must equal the oracle's (the reference's fp64
operation sequence, WeddingCakePlan::histogram_into baselines.cpp:139-148 +
score_weights matching.cpp:78-105) and the one-launch-per-scale path
(SWG_CAKE_GROUP=1) bit for bit, whatever mix of requests the call holds.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1705_03524_b200 import swg

pytestmark = pytest.mark.gpu

K = swg.Kernel


def _models(oracle, fi, bins, sizes, seed):
    rng = np.random.default_rng(seed)
    h, w = fi.shape
    out = []
    for kw in sizes:
        x, y = int(rng.integers(0, w - kw + 1)), int(rng.integers(0, h - kw + 1))
        ok = O.kernel(O.GAUSS_CHEB, kw, kw, 0.5)
        out.append(oracle.target_model(fi[y:y + kw, x:x + kw].copy(), bins, ok, O.CAKE,
                                       kw // 2 + 1))
    return out


def _reqs(sizes, models, sim=swg.BHATTACHARYYA):
    return [swg.MapRequest(K(swg.GAUSS_CHEB, kw, kw, 0.5), m, swg.CAKE, sim, kw // 2 + 1)
            for kw, m in zip(sizes, models)]


def _per_scale(t, reqs, monkeypatch, scores="host"):
    monkeypatch.setenv("SWG_CAKE_GROUP", "1")
    try:
        return t.likelihood_maps(reqs, scores=scores)
    finally:
        monkeypatch.delenv("SWG_CAKE_GROUP")


@pytest.mark.parametrize("bins,seed", [(6, 31), (19, 7), (64, 5)])
def test_cake_multi_vs_oracle(ctx, oracle, monkeypatch, bins, seed):
    """Seven scales (two launches of 4 + 3), the largest with a wide ring 0
    (257^2 > 2^16 pixels), ragged bin octets, centres whose valid scales
    differ inside one warp (the frame is only 300 x 270)."""
    img = oracle.random_gray(300, 270, seed)
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    sizes = [9, 257, 33, 129, 5, 65, 17]  # request order is not scale order
    models = _models(oracle, fi, bins, sizes, seed)
    reqs = _reqs(sizes, models)
    maps, peaks = t.likelihood_maps(reqs)
    ref_maps, ref_peaks = _per_scale(t, reqs, monkeypatch)
    for kw, model, got, pk, rm, rp in zip(sizes, models, maps, peaks, ref_maps, ref_peaks):
        ok = O.kernel(O.GAUSS_CHEB, kw, kw, 0.5)
        want, wpk, _ = oracle.fast_map(fi, bins, model, ok, O.CAKE, O.BHATTACHARYYA,
                                       rings=kw // 2 + 1)
        assert (got == want).all(), kw
        assert pk == oracle.peak(want, kw // 2, kw // 2), kw
        assert (got == rm).all() and pk == rp, kw


def test_cake_multi_mixed_call(ctx, oracle, monkeypatch):
    """Fusable and non-fusable requests in one call (intersection, a row
    range, a partial-ring plan, a Uniform box, a repeated scale with another
    model): every output lands at its own index, equal to the per-scale path."""
    bins = 12
    img = oracle.random_gray(160, 150, 77)
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    sizes = [41, 21, 41, 61, 11]
    models = _models(oracle, fi, bins, sizes, 9)
    reqs = _reqs(sizes, models)
    reqs.append(swg.MapRequest(K(swg.GAUSS_CHEB, 31, 31, 0.5), models[0], swg.CAKE,
                               swg.INTERSECTION, 16))
    reqs.append(swg.MapRequest(K(swg.GAUSS_CHEB, 25, 25, 0.5), models[1], swg.CAKE,
                               swg.BHATTACHARYYA, 13, rows=(10, 70)))
    reqs.append(swg.MapRequest(K(swg.GAUSS_CHEB, 45, 45, 0.5), models[2], swg.CAKE,
                               swg.BHATTACHARYYA, 7))
    reqs.append(swg.MapRequest(K(swg.UNIFORM, 15, 15), models[3], swg.PLAIN))
    order = [7, 0, 5, 1, 8, 2, 6, 3, 4]
    reqs = [reqs[i] for i in order]
    for scores in ("host", "pinned"):
        maps, peaks = t.likelihood_maps(reqs, scores=scores)
        ref_maps, ref_peaks = _per_scale(t, reqs, monkeypatch)
        for i, r in enumerate(reqs):
            assert (np.asarray(maps[i]) == ref_maps[i]).all(), (scores, i)
            assert peaks[i] == ref_peaks[i], (scores, i)
            if r.rows is None and r.method == swg.CAKE:
                ok = O.kernel(O.GAUSS_CHEB, r.kernel.kw, r.kernel.kw, 0.5)
                want, _, _ = oracle.fast_map(fi, bins, r.model, ok, O.CAKE, r.sim,
                                             rings=r.rings)
                assert (np.asarray(maps[i]) == want).all(), i


def test_cake_multi_device_outputs(ctx, oracle, monkeypatch):
    """Device maps and peaks (the bench's path, fanned out over the worker
    streams): equal to the host path and to the per-scale launches."""
    torch = pytest.importorskip("torch")
    bins = 32
    img = oracle.random_gray(257, 200, 3)
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    sizes = [33, 65, 97, 17, 129]
    models = _models(oracle, fi, bins, sizes, 4)
    reqs = _reqs(sizes, models)
    dm = [torch.empty((200 - kw + 1, 257 - kw + 1), dtype=torch.float64, device="cuda")
          for kw in sizes]
    dp = torch.empty((len(sizes), 6), dtype=torch.float64, device="cuda")  # >= swg_peak
    t.likelihood_maps(reqs, scores="none", scores_dev=dm, peaks_dev=dp)
    torch.cuda.synchronize()
    ref_maps, ref_peaks = _per_scale(t, reqs, monkeypatch)
    for i in range(len(sizes)):
        assert (dm[i].cpu().numpy() == ref_maps[i]).all(), sizes[i]


def test_cake_multi_narrow_domain(ctx, oracle, monkeypatch):
    """The smallest scale's centre domain one window wide / tall, the largest
    scale's map a single window."""
    bins = 8
    img = oracle.random_gray(67, 66, 12)
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    sizes = [65, 63, 61, 3]
    models = _models(oracle, fi, bins, sizes, 8)
    reqs = _reqs(sizes, models)
    maps, peaks = t.likelihood_maps(reqs)
    for kw, model, got, pk in zip(sizes, models, maps, peaks):
        ok = O.kernel(O.GAUSS_CHEB, kw, kw, 0.5)
        want = oracle.likelihood_map(fi, bins, model, ok, O.CAKE, O.BHATTACHARYYA,
                                     rings=kw // 2 + 1)
        assert (got == want).all(), kw
        assert pk == oracle.peak(want, kw // 2, kw // 2), kw
