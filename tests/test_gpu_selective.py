"""GPU tests of model-driven (selective) rebuilds, swg_tables_rebuild_for.

A rebuild for a known set of requests writes only the table units those
requests read (bin octets of the 32-bit planes, bin pairs of the decay
planes, holding a nonzero model value).  Every other consumer -- maps with
another model, exports, window queries, the device layout -- first builds
the units it reads, so nothing observable changes: maps, peaks and exports
equal those of a full rebuild, bit for bit.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1705_03524_b200 import swg

pytestmark = pytest.mark.gpu
K = swg.Kernel


def _sparse_model(bins, nz, seed):
    rng = np.random.default_rng(seed)
    m = np.zeros(bins)
    idx = rng.choice(bins, nz, replace=False)
    m[idx] = rng.random(nz) + 0.1
    return m / m.sum()


@pytest.mark.parametrize("planes", [swg.PLANES_AFFINE, swg.PLANES_QUADRATIC])
def test_rebuild_for_integer_tables(ctx, oracle, planes):
    bins = 40  # 5 octets
    img0 = oracle.random_gray(300, 220, 3)
    img1 = oracle.random_gray(300, 220, 4)
    fi1 = oracle.quantize_gray8(img1, bins)
    kind = swg.MANHATTAN if planes == swg.PLANES_AFFINE else swg.EUCLID_QUAD
    k = K(kind, 21, 17)
    ok = O.kernel(kind, 21, 17)
    m_a = np.zeros(bins)
    m_a[[3, 5, 17]] = [0.5, 0.25, 0.25]  # octets 0 and 2
    m_b = _sparse_model(bins, 6, 7)
    om = O.SWIH if kind == swg.MANHATTAN else O.BRUTE
    ts = ctx.build(img0, swg.FMT_GRAY8, bins, planes)
    tf = ctx.build(img0, swg.FMT_GRAY8, bins, planes)
    full = ctx.build(img0, swg.FMT_GRAY8, bins, planes)
    full.rebuild(img1)
    full_bytes = full.built_bytes()
    req_a = swg.MapRequest(k, m_a)
    ts.rebuild_for(img1, [req_a])
    assert 0 < ts.built_bytes() < full_bytes  # 2 of 5 octets
    got, pk = ts.likelihood_map(k, m_a)
    want, wpk, _ = oracle.fast_map(fi1, bins, m_a, ok, om)
    assert (got == want).all() and pk == wpk
    # another model: its stale octets are built on first use
    got_b, pk_b = ts.likelihood_map(k, m_b, sim=swg.INTERSECTION)
    want_b, wpk_b, _ = oracle.fast_map(fi1, bins, m_b, ok, om, O.INTERSECTION)
    assert (got_b == want_b).all() and pk_b == wpk_b
    # exports after a selective rebuild equal a full build's
    tf.rebuild_for(img1, [req_a])
    for kd in range(3):
        assert (tf.export_u32(kd) == full.export_u32(kd)).all(), kd
    assert (tf.export_i64(0) == full.export_i64(0)).all()
    for t in (ts, tf, full):
        t.close()


def test_rebuild_for_decay_tables(ctx, oracle):
    bins, d = 24, 0.875
    img0 = oracle.random_gray(160, 120, 11)
    img1 = oracle.random_gray(160, 120, 12)
    fi1 = oracle.quantize_gray8(img1, bins)
    k = K(swg.EXP_L1, 15, 13, d)
    ok = O.kernel(O.EXP_L1, 15, 13, d)
    m = np.zeros(bins)
    m[[2, 9, 10]] = [0.2, 0.3, 0.5]  # pairs 1, 4, 5
    ts = ctx.build_decay(img0, d, swg.FMT_GRAY8, bins)
    full = ctx.build_decay(img0, d, swg.FMT_GRAY8, bins)
    full.rebuild(img1)
    ts.rebuild_for(img1, [swg.MapRequest(k, m)])
    assert 0 < ts.built_bytes() < full.built_bytes()
    got, pk = ts.likelihood_map(k, m)
    want, wpk = full.likelihood_map(k, m)
    assert (got == want).all() and pk == wpk
    ref, rpk, _ = oracle.fast_map(fi1, bins, m, ok, O.BRUTE)
    assert np.abs(got - ref).max() <= 1e-4 and pk == rpk
    # another model reads other pairs (built on first use); the export too
    m2 = _sparse_model(bins, 5, 3)
    g2, p2 = ts.likelihood_map(k, m2)
    w2, q2 = full.likelihood_map(k, m2)
    assert (g2 == w2).all() and p2 == q2
    assert (ts.export_f64(0) == full.export_f64(0)).all()
    ts.close()
    full.close()


def test_rebuild_for_dense_and_mixed_requests(ctx, oracle):
    """A dense model (every octet), a cake request (16-bit plain planes of a
    plain set) and requests whose union covers every unit build fully."""
    bins = 16
    img = oracle.random_gray(200, 150, 5)
    fi = oracle.quantize_gray8(img, bins)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_AFFINE)
    full = t.built_bytes()
    m1 = np.zeros(bins)
    m1[1] = 1.0
    m2 = np.zeros(bins)
    m2[12] = 1.0
    k = K(swg.MANHATTAN, 11, 11)
    t.rebuild_for(img, [swg.MapRequest(k, m1), swg.MapRequest(k, m2)])
    assert t.built_bytes() == full
    t.rebuild_for(img, [swg.MapRequest(k, m1)])
    assert t.built_bytes() < full
    ok = O.kernel(O.MANHATTAN, 11, 11)
    for m in (m1, m2):
        got, pk = t.likelihood_map(k, m)
        want, wpk, _ = oracle.fast_map(fi, bins, m, ok)
        assert (got == want).all() and pk == wpk
    t.close()
    tp = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
    kc = K(swg.GAUSS_CHEB, 9, 9, 0.5)
    okc = O.kernel(O.GAUSS_CHEB, 9, 9, 0.5)
    mc = oracle.target_model(fi[20:29, 30:39].copy(), bins, okc, O.CAKE, 5)
    tp.rebuild_for(img, [swg.MapRequest(kc, mc, swg.CAKE, rings=5)])
    got, pk = tp.likelihood_map(kc, mc, swg.CAKE, rings=5)
    want, wpk, _ = oracle.fast_map(fi, bins, mc, okc, O.CAKE, rings=5)
    assert (got == want).all() and pk == wpk
    tp.close()


def test_rebuild_for_sparse_env_off(ctx, oracle, monkeypatch):
    """SWG_SPARSE=0: every unit is built and read."""
    monkeypatch.setenv("SWG_SPARSE", "0")
    bins = 24
    img = oracle.random_gray(120, 90, 8)
    t = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_AFFINE)
    full = t.built_bytes()
    m = np.zeros(bins)
    m[0] = 1.0
    t.rebuild_for(img, [swg.MapRequest(K(swg.MANHATTAN, 9, 9), m)])
    assert t.built_bytes() == full
    assert t.request_plan(swg.MapRequest(K(swg.MANHATTAN, 9, 9), m))["bins_read"] == bins
    t.close()


def test_tma_and_thread_stores_build_identical_tables(ctx, oracle, monkeypatch):
    """The TMA tensor stores of the staged rows (default) and the per-thread
    stores (SWG_NO_TMA=1, read when a table set first builds) write the same
    planes: 16- / 32-bit integral sets at widths that do and do not fill the
    last warp segment, and the decayed set."""
    for w, h in ((2048, 37), (1000, 23), (257, 64)):
        img = oracle.random_gray(w, h, w + h)
        bins = 24
        tm = {}
        for env in ("0", "1"):
            if env == "1":
                monkeypatch.setenv("SWG_NO_TMA", "1")
            else:
                monkeypatch.delenv("SWG_NO_TMA", raising=False)
            tq = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_QUADRATIC)
            tp = ctx.build(img, swg.FMT_GRAY8, bins, swg.PLANES_PLAIN)
            td = ctx.build_decay(img, 0.9375, swg.FMT_GRAY8, bins)
            tm[env] = ([tq.export_u32(k) for k in range(3)], tp.export_u32(0),
                       [td.export_f64(k) for k in range(4)])
            for t in (tq, tp, td):
                t.close()
        a, b = tm["0"], tm["1"]
        assert all((x == y).all() for x, y in zip(a[0], b[0]))
        assert (a[1] == b[1]).all()
        assert all((x == y).all() for x, y in zip(a[2], b[2]))
        fi = oracle.quantize_gray8(img, bins)
        p, _, _ = oracle.build_tables(fi, bins)
        assert (a[1] == p.astype(np.uint32)).all()


def test_likelihood_maps_async_rotating_scratch(ctx, oracle):
    """swg_likelihood_maps_async over several table sets back to back (map
    copies, zero-copy maps and the exponential re-score on rotating scratch
    slots), host outputs read after swg_ctx_synchronize: identical to the
    synchronous calls, over two frames (slot reuse)."""
    import ctypes as C
    from paper_1705_03524_b200.swg import Peak, _check, lib
    bins, d = 16, 0.875
    frames = [oracle.random_gray(260, 200, s) for s in (31, 32)]
    fi0 = oracle.quantize_gray8(frames[0], bins)
    sets = [ctx.build(frames[0], swg.FMT_GRAY8, bins, swg.PLANES_AFFINE),
            ctx.build(frames[0], swg.FMT_GRAY8, bins, swg.PLANES_PLAIN),
            ctx.build_decay(frames[0], d, swg.FMT_GRAY8, bins)]
    reqs = []
    for kw in (9, 15, 21, 27, 33):  # five requests: the copy path
        reqs.append((0, swg.MapRequest(K(swg.MANHATTAN, kw, kw),
                                       oracle.target_model(fi0[5:5 + kw, 7:7 + kw].copy(), bins,
                                                           O.kernel(O.MANHATTAN, kw, kw)))))
    for kw in (11, 25):  # two requests: zero-copy maps
        okc = O.kernel(O.GAUSS_CHEB, kw, kw, 0.5)
        reqs.append((1, swg.MapRequest(K(swg.GAUSS_CHEB, kw, kw, 0.5),
                                       oracle.target_model(fi0[3:3 + kw, 9:9 + kw].copy(), bins,
                                                           okc, O.CAKE, kw // 2 + 1),
                                       swg.CAKE, rings=kw // 2 + 1)))
    for kw in (13, 19):
        oke = O.kernel(O.EXP_L1, kw, kw, d)
        reqs.append((2, swg.MapRequest(K(swg.EXP_L1, kw, kw, d),
                                       oracle.target_model(fi0[8:8 + kw, 4:4 + kw].copy(), bins,
                                                           oke, O.BRUTE))))
    for img in frames:
        want = {}
        for si, t in enumerate(sets):
            rs = [r for s, r in reqs if s == si]
            t.rebuild(img)
            want[si] = t.likelihood_maps(rs)
        keep = []
        outs = {}
        for si, t in enumerate(sets):
            rs = [r for s, r in reqs if s == si]
            t.rebuild_for(img, rs)
            maps = [swg.PinnedBuffer(t.map_shape(r.kernel), np.float64) for r in rs]
            pkb = swg.PinnedBuffer((C.sizeof(Peak) * len(rs),), np.uint8)
            pk = (Peak * len(rs)).from_address(pkb.array.ctypes.data)
            hp = (C.c_void_p * len(rs))(*[m.array.ctypes.data for m in maps])
            creqs, k2 = swg.Tables._creqs(rs, t.total_bins)
            keep += [maps, pkb, pk, hp, creqs, k2]
            _check(lib().swg_likelihood_maps_async(t._h, len(rs), C.addressof(creqs),
                                                   C.addressof(hp), None, C.addressof(pk), None))
            outs[si] = (maps, pk)
        ctx.synchronize()
        for si in outs:
            maps, pk = outs[si]
            wmaps, wpks = want[si]
            for m, w in zip(maps, wmaps):
                assert (m.array == w).all(), si
            assert [p.astuple() for p in pk] == wpks, si
    for t in sets:
        t.close()
