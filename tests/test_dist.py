"""Multi-GPU host logic on CPU with gloo, world_size 2:
row-band maps == full map, boundary prefix-row exchange rebuilds the global
integral tables exactly, and the peak gather applies the reference tie rule.
The oracle stands in for each rank's GPU work here; on the box the same
functions run with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_03524_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        orc = O.Oracle()
        img = orc.random_gray(57, 83, 4)
        bins = 8
        fi = orc.quantize_gray8(img, bins)
        # --- banded IH build + boundary prefix-row exchange
        y0, y1 = D.table_bands(83, world)[rank]
        local = orc.build_tables(np.ascontiguousarray(fi[y0:y1]), bins)
        rows = D.exchange_last_rows(D.last_rows(local, y0))
        glob = D.globalize_band_tables(local, y0, D.band_carry(rows, rank))
        full = orc.build_tables(fi, bins)
        ok_tables = all((g == f[:, y0:y1 + 1, :]).all() for g, f in zip(glob, full))
        # --- row-band map + global peak
        k = O.kernel(O.MANHATTAN, 9, 7)
        model = orc.target_model(np.ascontiguousarray(fi[20:27, 30:39]), bins, k)
        band = D.row_bands(83, 7, world)[rank]
        (v0, v1), (p0, p1) = band.map_rows, band.pixel_rows
        part = orc.likelihood_map(np.ascontiguousarray(fi[p0:p1]), bins, model, k)
        mw = part.shape[1]
        u, v, _, _, s = orc.peak(part, 4, 3)
        pk = D.gather_peak(s, (v + v0) * mw + u, mw, 4, 3)
        fullmap = orc.likelihood_map(fi, bins, model, k)
        q.put((rank, ok_tables, bool((part == fullmap[v0:v1]).all()),
               pk == orc.peak(fullmap, 4, 3)))
    finally:
        dist.destroy_process_group()


def test_two_rank_bands_exchange_and_peak():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_t, ok_map, ok_peak in res:
        assert ok_t and ok_map and ok_peak, (rank, ok_t, ok_map, ok_peak)


def test_tie_rule_across_ranks():
    assert D.reduce_peaks([(0.5, 10), (0.9, 40), (0.9, 12), (0.1, 0)]) == (0.9, 12)
    assert D.reduce_peaks([(0.7, 3)]) == (0.7, 3)


def test_band_geometry_covers_the_map():
    for h, kh, world in ((83, 7, 2), (1024, 97, 8), (40, 39, 4)):
        bands = D.row_bands(h, kh, world)
        assert bands[0].map_rows[0] == 0 and bands[-1].map_rows[1] == h - kh + 1
        for a, b in zip(bands, bands[1:]):
            assert a.map_rows[1] == b.map_rows[0]
        for bd in bands:
            assert bd.pixel_rows[1] - bd.pixel_rows[0] == (bd.map_rows[1] - bd.map_rows[0]) + \
                (kh - 1 if bd.map_rows[1] > bd.map_rows[0] else 0)
    assert D.frame_shards(64, 8, 3) == list(range(3, 64, 8))


def _chain_worker(rank, world, port, q):
    """Bin-range chain (config 4 on N GPUs): rank g owns bins [b_g, b_g+1),
    continues each window's running Bhattacharyya sum and mass in bin order
    and passes them on; the oracle's window histograms stand in for the
    rank's table sweep.  The last rank's map must equal the single-table
    map bit for bit."""
    import math
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        orc = O.Oracle()
        img = orc.random_gray(40, 31, 6)
        bins = 20
        fi = orc.quantize_gray8(img, bins)
        k = O.kernel(O.MANHATTAN, 7, 5)
        model = orc.target_model(np.ascontiguousarray(fi[10:15, 12:19]), bins, k)
        mw, mh = 40 - 7 + 1, 31 - 5 + 1
        raw = np.array([[orc.brute_counts(fi, bins, u + 3, v + 2, k) for u in range(mw)]
                        for v in range(mh)])
        b0, b1 = D.bin_ranges(bins, world)[rank]

        def compute(chunk, pin):
            r0, r1 = chunk
            out = torch.zeros(r1 - r0, mw, 2, dtype=torch.float64)
            for v in range(r0, r1):
                for u in range(mw):
                    s, mass = (0.0, 0.0) if pin is None else (float(pin[v - r0, u, 0]),
                                                              float(pin[v - r0, u, 1]))
                    for b in range(b0, b1):  # score_counts order (matching.cpp:20-35)
                        mass += float(raw[v, u, b])
                        s += math.sqrt(model[b] * float(raw[v, u, b]))
                    out[v - r0, u, 0], out[v - r0, u, 1] = s, mass
            if rank < world - 1:
                return out
            sc = out[..., 0] / torch.sqrt(out[..., 1])
            return sc.clamp(0.0, 1.0)

        chunks = D.row_chunks(mh, 4)
        res = D.run_bin_chain(rank, world, chunks, compute,
                              lambda c: torch.zeros(c[1] - c[0], mw, 2, dtype=torch.float64))
        ok = True
        if rank == world - 1:
            got = torch.cat(res).numpy()
            want = orc.likelihood_map(fi, bins, model, k)
            ok = bool((got == want).all())
        q.put((rank, (b0, b1), ok))
    finally:
        dist.destroy_process_group()


def test_bin_range_chain_three_ranks():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chain_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert [r[1] for r in res] == [(0, 8), (8, 16), (16, 20)]
    assert all(r[2] for r in res)


def test_bin_range_geometry():
    assert D.bin_ranges(512, 8) == [(64 * g, 64 * g + 64) for g in range(8)]
    assert D.bin_ranges(20, 2) == [(0, 16), (16, 20)]
    assert D.bin_ranges(8, 3) == [(0, 8), (8, 8), (8, 8)]
    assert D.row_chunks(10, 3) == [(0, 4), (4, 8), (8, 10)]


def _plan_worker(rank, world, port, q):
    """One frame's (kernel, scale) requests over ranks (config 2 / 5 on N
    GPUs, dist.plan_frame): each rank sweeps only its Work items -- row
    chunks of the maps, on the table sets it builds -- and the ranks gather
    the chunk peaks.  The oracle stands in for the rank's GPU sweeps; the
    stitched maps and combined peaks must equal the single-rank result."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        orc = O.Oracle()
        img = orc.random_gray(70, 64, 9)
        bins = 8
        fi = orc.quantize_gray8(img, bins)
        h, w = fi.shape
        kernels = [(0, O.kernel(O.MANHATTAN, 9, 9), O.SWIH, 1),
                   (0, O.kernel(O.MANHATTAN, 21, 15), O.SWIH, 1),
                   (1, O.kernel(O.GAUSS_CHEB, 13, 13), O.CAKE, 7),
                   (1, O.kernel(O.GAUSS_CHEB, 31, 31), O.CAKE, 16)]
        models = [orc.target_model(np.ascontiguousarray(fi[5:5 + k.kh, 7:7 + k.kw]), bins, k,
                                   m, r) for _, k, m, r in kernels]
        reqs = [((g, i), g, h - k.kh + 1, float((h - k.kh + 1) * r * (1 + g)))
                for i, (g, k, m, r) in enumerate(kernels)]
        plan = D.plan_frame(reqs, [3.0, 1.0], world, min_rows=4)
        parts, maps = [], {}
        for wk in plan[rank]:
            g, k, m, r = kernels[wk.key[1]]
            v0, v1 = wk.rows
            # the window rows [v0, v1) from the pixel rows they touch
            part = orc.likelihood_map(np.ascontiguousarray(fi[v0:v1 + k.kh - 1]), bins,
                                      models[wk.key[1]], k, m, rings=r)
            u, v, _, _, s = orc.peak(part, k.kw // 2, k.kh // 2)
            parts.append((wk.key, (v0, v1), s, v * part.shape[1] + u))
            maps[(wk.key, wk.rows)] = part
        every = [None] * world
        dist.all_gather_object(every, (parts, maps))
        allparts = [p for e, _ in every for p in e]
        widths = {(g, i): w - k.kw + 1 for i, (g, k, _, _) in enumerate(kernels)}
        best = D.combine_request_peaks(allparts, widths)
        ok = True
        for i, (g, k, m, r) in enumerate(kernels):
            full = orc.likelihood_map(fi, bins, models[i], k, m, rings=r)
            st = np.full_like(full, np.nan)
            for _, mp_ in every:
                for (key, (v0, v1)), part in mp_.items():
                    if key == (g, i):
                        st[v0:v1] = part
            pk = orc.peak(full, k.kw // 2, k.kh // 2)
            ok &= bool((st == full).all())
            ok &= best[(g, i)] == (pk[4], pk[1] * full.shape[1] + pk[0])
        covered = sorted((wk.key, wk.rows) for p in plan for wk in p)
        q.put((rank, ok, len(plan[rank]), covered))
    finally:
        dist.destroy_process_group()


def test_one_frame_plan_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert all(r[1] for r in res), res
    assert all(r[2] >= 1 for r in res)  # both ranks have work


def test_plan_frame_geometry():
    """Every (request, map row) on exactly one rank; LPT balance; ranks pay
    only the builds of the table sets they sweep; deterministic."""
    reqs = [((g, s), g, 2048 - 16 * s, 1.0 + 0.4 * s + 0.5 * g) for g in range(4)
            for s in range(8)]
    build = [1.0, 0.3, 1.6, 2.5]
    for world in (1, 2, 3, 4, 8):
        plan = D.plan_frame(reqs, build, world)
        assert plan == D.plan_frame(reqs, build, world)
        rows = {}
        for p in plan:
            for wk in p:
                rows.setdefault(wk.key, []).append(wk.rows)
        for key, g, mh, _ in reqs:
            rs = sorted(rows[key])
            assert rs[0][0] == 0 and rs[-1][1] == mh
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        loads = [sum(wk.cost for wk in p) + sum(build[g] for g in {wk.group for wk in p})
                 for p in plan]
        total = sum(c for *_, c in reqs)
        assert max(loads) <= (total + sum(build)) / world * 1.35 + 0.6
    one = D.plan_frame([((0, 0), 0, 100, 5.0)], [0.1], 4, min_rows=8)
    assert sum(len(p) for p in one) == 4  # a single request splits by rows


def _records(tables, bins):
    """Oracle int64 tables (3, bins, h+1, w+1) -> the device record layout of
    the last row (octets, planes, w+1, 8) as int32 words mod 2^32."""
    import torch
    p = np.stack([t[:, -1, :] for t in tables])  # (3, bins, w+1)
    g = -(-bins // 8)
    out = np.zeros((g, 3, p.shape[2], 8), np.int64)
    for b in range(bins):
        out[b // 8, :, :, b % 8] = p[:, b, :]
    return D._wrap32(torch.from_numpy(out))


def test_device_carry_equals_host_exchange():
    """dist.device_carry (the device boundary-row exchange's arithmetic, on
    int32 record rows mod 2^32) == the exact host exchange (band_carry)."""
    import torch
    from oracle import oracle as O
    orc = O.Oracle()
    img = orc.random_gray(40, 90, 12)
    bins = 11
    fi = orc.quantize_gray8(img, bins)
    bands = D.table_bands(90, 4)
    local = [orc.build_tables(np.ascontiguousarray(fi[y0:y1]), bins) for y0, y1 in bands]
    lasts = [_records(t, bins) for t in local]
    rows = [D.last_rows(t, y0) for t, (y0, _) in zip(local, bands)]
    for r in range(4):
        host = D.band_carry(rows, r)  # (3, bins, w+1) exact
        dev = D.device_carry(lasts, [y0 for y0, _ in bands], r)
        want = _records([host[k][:, None, :] for k in range(3)], bins)
        assert torch.equal(dev, want), r


class _FakeBand:
    """CPU stand-in for a device table set (last_row / add_carry)."""

    def __init__(self, last):
        self.last, self.carry = last, None

    def last_row(self):
        return self.last

    def add_carry(self, y0, carry):
        self.carry = (y0, carry)


def _xchg_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from oracle import oracle as O
        orc = O.Oracle()
        img = orc.random_gray(33, 61, 3)
        bins = 9
        fi = orc.quantize_gray8(img, bins)
        bands = D.table_bands(61, world)
        y0, y1 = bands[rank]
        local = orc.build_tables(np.ascontiguousarray(fi[y0:y1]), bins)
        band = _FakeBand(_records(local, bins))
        carry = D.exchange_last_rows_device(band, y0)
        rows = [D.last_rows(orc.build_tables(np.ascontiguousarray(fi[a:b]), bins), a)
                for a, b in bands]
        want = _records([D.band_carry(rows, rank)[k][:, None, :] for k in range(3)], bins)
        q.put((rank, bool(torch.equal(carry, want)) and band.carry[0] == y0))
    finally:
        dist.destroy_process_group()


def test_device_row_exchange_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xchg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok in res), res
