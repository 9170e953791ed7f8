"""GPU parity of the row-streaming chain sweeps (csrc/k_stream.cu).

The planner picks the streaming sweep for Manhattan maps large enough to
fill the GPU with chain segments; SWG_STREAM=1 forces it on any map, so
these tests drive it through small shapes, every chain residue pattern
(hy = 0, 1, 2, ..., window heights above and below a segment), ragged
widths, row ranges, bin-range chains and carried (global-row) tables --
each map and peak bit-identical to the oracle and to the per-window sweep
(SWG_STREAM=0).
"""
import os

import numpy as np
import pytest

import test_gpu_parity as P
from oracle import oracle as O
from paper_1705_03524_b200 import swg

pytestmark = pytest.mark.gpu
K = swg.Kernel


@pytest.fixture
def force_stream(monkeypatch):
    monkeypatch.setenv("SWG_STREAM", "1")


def _with_env(name, val, fn):
    old = os.environ.get(name)
    os.environ[name] = val
    try:
        return fn()
    finally:
        if old is None:
            del os.environ[name]
        else:
            os.environ[name] = old


@pytest.mark.parametrize("kw,kh", [(1, 1), (3, 3), (5, 1), (7, 5), (13, 7), (31, 31), (9, 41),
                                   (65, 33), (21, 75)])
@pytest.mark.parametrize("narrow", [False, True])
def test_stream_manhattan_vs_oracle(ctx, oracle, kw, kh, narrow):
    w, h = 181 + kw, 97 + kh
    img = oracle.random_gray(w, h, kw * 7 + kh)
    img = ((img.astype(np.uint16) + np.roll(img, 1, 1)) // 2).astype(np.uint8)
    bins = 13 if narrow else 24
    fi = oracle.quantize_gray8(img, bins)
    k = K(swg.MANHATTAN, kw, kh)
    ok = O.kernel(O.MANHATTAN, kw, kh)
    mdl = oracle.target_model(fi[5:5 + kh, 9:9 + kw].copy(), bins, ok)
    planes = swg.PLANES_QUADRATIC if narrow else swg.PLANES_AFFINE
    t = ctx.build(img, swg.FMT_GRAY8, bins, planes)
    # the 16-bit sweep needs mass < 2^16 and a map of >= 2^20 windows unless
    # forced; SWG_AFFINE16 is read with the map size, so force it by size:
    # small maps go 32-bit (narrow=True then checks the 5-plane set's planes)
    for sim in (swg.BHATTACHARYYA, swg.INTERSECTION):
        want, wpk, _ = oracle.fast_map(fi, bins, mdl, ok, O.SWIH, sim)
        got, pk = _with_env("SWG_STREAM", "1", lambda: t.likelihood_map(k, mdl, swg.SWIH, sim))
        assert (got == want).all(), (kw, kh, sim)
        assert pk == wpk
        old, opk = _with_env("SWG_STREAM", "0", lambda: t.likelihood_map(k, mdl, swg.SWIH, sim))
        assert (old == got).all() and opk == pk
    # row ranges (chains relative to the range's first row)
    mh = h - kh + 1
    for rows in ((0, 1), (3, min(mh, 3 + kh + 2)), (mh // 3, mh), (1, mh - 1)):
        if rows[0] >= rows[1]:
            continue
        want, _, _ = oracle.fast_map(fi, bins, mdl, ok, O.SWIH, O.BHATTACHARYYA)
        maps, pks = _with_env("SWG_STREAM", "1",
                              lambda: t.likelihood_maps([swg.MapRequest(k, mdl, rows=rows)]))
        assert (maps[0] == want[rows[0]:rows[1]]).all(), rows
        sub = want[rows[0]:rows[1]]
        flat = int(np.argmax(sub))  # first maximum in row-major order
        assert pks[0][:2] == (flat % sub.shape[1], flat // sub.shape[1] + rows[0])
        assert pks[0][4] == sub.max()
    t.close()


@pytest.mark.parametrize("kw,kh", [(3, 3), (17, 17), (37, 37), (25, 9)])
def test_stream_affine16_large_maps(ctx, oracle, kw, kh):
    """Maps of >= 2^20 windows with mass < 2^16: the 16-bit streaming sweep
    (default planner choice) against the oracle and the 32-bit per-window
    sweep."""
    w, h = 1100 + kw, 960 + kh
    img = oracle.random_gray(w, h, 3 + kw)
    img = ((img.astype(np.uint16) + np.roll(img, 1, 0)) // 2).astype(np.uint8)
    bins = 16
    fi = oracle.quantize_gray8(img, bins)
    k = K(swg.MANHATTAN, kw, kh)
    ok = O.kernel(O.MANHATTAN, kw, kh)
    mdl = oracle.target_model(fi[30:30 + kh, 40:40 + kw].copy(), bins, ok)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_AFFINE)
    for sim in (swg.BHATTACHARYYA, swg.INTERSECTION):
        want, wpk, _ = oracle.fast_map(fi, bins, mdl, ok, O.SWIH, sim)
        got, pk = t.likelihood_map(k, mdl, swg.SWIH, sim)
        assert (got == want).all() and pk == wpk
        g32, p32 = _with_env("SWG_AFFINE16", "0", lambda: t.likelihood_map(k, mdl, swg.SWIH, sim))
        assert (g32 == want).all() and p32 == wpk
        gold, pold = _with_env("SWG_STREAM", "0", lambda: t.likelihood_map(k, mdl, swg.SWIH, sim))
        assert (gold == want).all() and pold == wpk
    t.close()


# Existing parity tests rerun with the streaming sweep forced on every
# Manhattan map (the bin-range chain, carried global-row tables, random
# shapes and the narrow-plane cases).
@pytest.mark.parametrize("seed", [1, 2])
def test_stream_forced_random_maps(force_stream, ctx, oracle, seed):
    P.test_maps_vs_oracle_random(ctx, oracle, seed)


@pytest.mark.parametrize("ranges", [[(0, 8), (8, 16), (16, 20)], [(0, 20)]])
def test_stream_forced_bin_range_chain(force_stream, ctx, oracle, ranges):
    P.test_bin_range_chain_bit_exact(ctx, oracle, ranges)


@pytest.mark.parametrize("planes", [swg.PLANES_AFFINE, swg.PLANES_QUADRATIC])
def test_stream_forced_carried_tables(force_stream, ctx, oracle, planes):
    P.test_device_boundary_row_exchange(ctx, oracle, planes)


@pytest.mark.parametrize("seed", [101, 202])
def test_stream_forced_random_configurations(force_stream, ctx, oracle, seed):
    P.test_random_configurations_all_engines(ctx, oracle, seed)


# ---------------------------------------------------------------- quadratic
@pytest.fixture
def force_stream_quad(monkeypatch):
    monkeypatch.setenv("SWG_STREAM_QUAD", "1")


@pytest.mark.parametrize("bins", [8, 16])
def test_stream_quad_forced_maps(force_stream_quad, ctx, oracle, bins):
    P.test_euclid_quadratic_maps_exact(ctx, oracle, bins)


def test_stream_quad_forced_tall_image(force_stream_quad, ctx, oracle):
    P.test_quadratic_tall_image(ctx, oracle)


@pytest.mark.parametrize("ranges", [[(0, 8), (8, 16), (16, 20)], [(0, 20)]])
def test_stream_quad_forced_bin_range_chain(force_stream_quad, ctx, oracle, ranges):
    P.test_bin_range_chain_bit_exact(ctx, oracle, ranges)


def test_stream_quad_forced_carried_tables(force_stream_quad, ctx, oracle):
    P.test_device_boundary_row_exchange(ctx, oracle, swg.PLANES_QUADRATIC)


@pytest.mark.parametrize("seed", [101, 303])
def test_stream_quad_forced_random_configurations(force_stream_quad, ctx, oracle, seed):
    P.test_random_configurations_all_engines(ctx, oracle, seed)


@pytest.mark.parametrize("kw,kh", [(5, 5), (17, 17), (33, 9), (9, 41)])
def test_stream_quad_large_maps(ctx, oracle, kw, kh):
    """Default planner choice on a map large enough for the streaming
    quadratic sweep: identical to the per-window sweep and the oracle's
    brute force on the same rows (a row band, to keep the oracle fast)."""
    w, h = 1500, 700
    img = oracle.random_gray(w, h, kw + kh)
    bins = 24
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_QUADRATIC)
    k = K(swg.EUCLID_QUAD, kw, kh)
    ok = O.kernel(O.EUCLID_QUAD, kw, kh)
    mdl = oracle.target_model(fi[50:50 + kh, 60:60 + kw].copy(), bins, ok, O.BRUTE)
    for sim in (swg.BHATTACHARYYA, swg.INTERSECTION):
        got, pk = t.likelihood_map(k, mdl, swg.SWIH, sim)
        old, opk = _with_env("SWG_STREAM_QUAD", "0", lambda: t.likelihood_map(k, mdl, swg.SWIH, sim))
        assert (got == old).all() and pk == opk
        want, wpk, _ = oracle.fast_map(fi, bins, mdl, ok, O.BRUTE, sim)
        assert (got == want).all() and pk == wpk
    t.close()
