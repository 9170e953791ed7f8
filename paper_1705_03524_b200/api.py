"""Reference-style helpers over the C-ABI (Python harness side).

  normalize        histogram.cpp:19-26 (sequential fp64 sum, then divide)
  target_model     matching.cpp:69-106 (model of a kw x kh template, built
                   the way the chosen method builds its candidates; the
                   template's histogram itself is computed on the GPU)
  MultiScaleMatcher  one table build serving every scale,
                   the batched form of likelihood_map + peak
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from . import swg


def normalize(h: np.ndarray) -> np.ndarray:
    mass = 0.0
    for v in h.tolist():
        mass += v
    if mass == 0.0:
        raise swg.ZeroMassError("normalize: histogram has zero mass")
    return np.asarray(h, np.float64) / mass


def target_model(ctx: swg.Context, templ: np.ndarray, kernel: swg.Kernel, fmt=swg.FMT_GRAY8,
                 bins=16, method=swg.SWIH, rings=4, rule=swg.RING_MEAN) -> np.ndarray:
    """target_model_for_method (matching.cpp:84-106) for a kw x kh template."""
    h, w = templ.shape[:2]
    if (w, h) != (kernel.kw, kernel.kh):
        raise swg.ModelError(f"target model: template {w}x{h} does not match kernel "
                             f"{kernel.kw}x{kernel.kh}")
    if method == swg.CAKE:
        t = ctx.build(templ, fmt, bins, swg.PLANES_PLAIN)
        raw = t.cake_windows([kernel.hx], [kernel.hy], kernel, rings, rule)[0]
    elif method == swg.PLAIN or kernel.kind == swg.UNIFORM:
        t = ctx.build(templ, fmt, bins, swg.PLANES_PLAIN)
        k = swg.Kernel(swg.UNIFORM, kernel.kw, kernel.kh)
        raw = t.query_windows([k.hx], [k.hy], k, swg.PLAIN)[0].astype(np.float64)
    elif kernel.kind == swg.MANHATTAN:
        t = ctx.build(templ, fmt, bins, swg.PLANES_AFFINE)
        raw = t.query_windows([kernel.hx], [kernel.hy], kernel, swg.SWIH)[0].astype(np.float64)
    else:
        # non-affine kernel, brute-force model: one-window brute map on the template
        t = ctx.build(templ, fmt, bins, swg.PLANES_PLAIN)
        return _brute_model(t, kernel)
    return normalize(raw)


def _brute_model(t: swg.Tables, kernel: swg.Kernel) -> np.ndarray:
    """BruteForcePlan on the template's one strict window (matching.cpp:84-106
    with MapMethod::BruteForce; baselines.cpp:24-69): counts for integer
    kernels, fp64 weight sums otherwise, then normalize."""
    fi = t.feature_image()
    raw = t.ctx.brute_windows(fi, t.bins, [kernel.hx], [kernel.hy], kernel)[0]
    return normalize(raw.astype(np.float64))


class MultiScaleMatcher:
    """Builds the integral tables of one frame once and evaluates several
    (kernel, model) scales against them; the B200 form of calling
    likelihood_map (matching.cpp:108-209) + peak (211-223) once per scale."""

    def __init__(self, ctx: swg.Context, width: int, height: int, fmt=swg.FMT_GRAY8, bins=16,
                 planes=swg.PLANES_AFFINE, decay=None):
        self.ctx, self.fmt, self.bins, self.planes = ctx, fmt, bins, planes
        self.width, self.height = width, height
        self.decay = decay  # PLANES_DECAY: the exponential kernel's per-pixel decay
        self.tables = None

    def load(self, pixels):
        if self.tables is None:
            if self.planes == swg.PLANES_DECAY:
                self.tables = self.ctx.build_decay(pixels, self.decay, self.fmt, self.bins)
            else:
                self.tables = self.ctx.build(pixels, self.fmt, self.bins, self.planes)
        else:
            self.tables.rebuild(pixels)
        return self.tables

    def run(self, reqs: Sequence[swg.MapRequest], scores="host", scores_dev=None,
            peaks_dev=None):
        return self.tables.likelihood_maps(reqs, scores, scores_dev, peaks_dev)
