"""Multi-GPU partitioning of the SWIH hot path.

One process per GPU; torch.distributed (NCCL on the box, gloo in the CPU
tests) carries the few small exchanges.  The path partitions without a
data-path collective:

* frames       — `frame_shards`: frames of a batch round-robin over ranks.
* row bands    — `row_bands`: rank r owns map rows [v0, v1) and receives
                 pixel rows [v0, v1 + kh - 1) (an input halo).  Window
                 histograms do not depend on the crop, so its local tables
                 give bit-identical map rows with no table exchange.
* global IH    — `band_carry` / `globalize_band_tables`: to export the GLOBAL
                 integral tables from row bands, every rank all-gathers its
                 band's last prefix row ((W+1)*b*3 values) and adds the sum of
                 the earlier bands' rows — the boundary prefix-row exchange.
                 y-ramps also shift by y0 * plain (local y = global y - y0).
* peak         — `gather_peak`: all-gather of each rank's (score, global
                 row-major index) and the reference tie rule
                 (matching.cpp:211-223): max score, then smallest index.
* bin ranges   — `bin_ranges` / `run_bin_chain`: rank g holds the tables of
                 bins [b_g, b_g+1) only (1/G of the planes: config 4's 512
                 bins) and continues each window's running Bhattacharyya sum
                 and mass in bin order: partial sums flow g -> g+1 with
                 point-to-point send/recv, pipelined by row chunks, and the
                 last rank finishes scores, map and peak.  Same fp64
                 operation sequence as one GPU -> bit-identical (an
                 all-reduce would reorder the sum: SURVEY §8e).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np


@dataclass(frozen=True)
class Band:
    rank: int
    map_rows: Tuple[int, int]    # [v0, v1) of the strict map
    pixel_rows: Tuple[int, int]  # [y0, y1) of the image this rank needs


def frame_shards(n_frames: int, world: int, rank: int) -> List[int]:
    return list(range(rank, n_frames, world))


def row_bands(height: int, kh: int, world: int) -> List[Band]:
    """Split the strict map of an image of `height` rows (kernel height kh)
    into `world` contiguous, near-equal row bands."""
    mh = height - kh + 1
    if mh < 1:
        raise ValueError("kernel taller than the image")
    out = []
    for r in range(world):
        v0 = r * mh // world
        v1 = (r + 1) * mh // world
        out.append(Band(r, (v0, v1), (v0, v1 + kh - 1 if v1 > v0 else v0)))
    return out


def table_bands(height: int, world: int) -> List[Tuple[int, int]]:
    """Pixel-row bands [y0, y1) covering the image, for a banded IH build."""
    return [(r * height // world, (r + 1) * height // world) for r in range(world)]


def band_carry(last_rows: Sequence[np.ndarray], rank: int) -> np.ndarray:
    """Exclusive sum of the earlier bands' last prefix rows."""
    carry = np.zeros_like(last_rows[0])
    for r in range(rank):
        carry = carry + last_rows[r]
    return carry


def globalize_band_tables(local: Tuple[np.ndarray, np.ndarray, np.ndarray], y0: int,
                          carry: np.ndarray) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Local int64 tables of pixel rows [y0, y0+h) (bins, h+1, W+1), zero at
    their own row 0 -> global tables rows y0 .. y0+h.  carry: (3, bins, W+1),
    the global prefix row at y0 of (plain, xramp, yramp)."""
    p, x, y = local
    gp = p + carry[0][:, None, :]
    gx = x + carry[1][:, None, :]
    gy = y + np.int64(y0) * p + carry[2][:, None, :]
    return gp, gx, gy


def last_rows(local: Tuple[np.ndarray, np.ndarray, np.ndarray], y0: int) -> np.ndarray:
    """This band's contribution to the prefix row below it: (3, bins, W+1)."""
    p, x, y = local
    return np.stack([p[:, -1, :], x[:, -1, :], y[:, -1, :] + np.int64(y0) * p[:, -1, :]])


def exchange_last_rows(mine: np.ndarray, group=None) -> List[np.ndarray]:
    """all_gather of every band's last prefix row (the boundary exchange)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(mine))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return [q.cpu().numpy() for q in parts]


def better(a: Tuple[float, int], b: Tuple[float, int]) -> bool:
    """Reference tie rule: higher score, then smaller row-major index."""
    return a[0] > b[0] or (a[0] == b[0] and a[1] < b[1])


def reduce_peaks(cands: Sequence[Tuple[float, int]]) -> Tuple[float, int]:
    best = (-2.0, 1 << 62)
    for c in cands:
        if better(c, best):
            best = c
    return best


def gather_peak(score: float, index: int, map_width: int, hx: int, hy: int,
                group=None) -> Optional[tuple]:
    """Global peak over ranks: (map_x, map_y, center_x, center_y, score)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    # the score travels as its IEEE bits so the comparison stays exact
    bits = np.array([score], np.float64).view(np.int64)[0]
    mine = torch.tensor([int(bits), int(index)], dtype=torch.int64, device=dev)
    parts = [torch.empty_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, mine, group=group)
    cands = []
    for p in parts:
        b, i = p.cpu().tolist()
        cands.append((float(np.array([b], np.int64).view(np.float64)[0]), int(i)))
    s, i = reduce_peaks(cands)
    u, v = i % map_width, i // map_width
    return (u, v, u + hx, v + hy, s)


def bin_ranges(bins: int, world: int, align: int = 8) -> List[Tuple[int, int]]:
    """Contiguous bin ranges, one per rank, split on `align`-bin boundaries
    (whole table records) as evenly as the octet count allows."""
    units = -(-bins // align)
    out, start = [], 0
    for g in range(world):
        n = units // world + (1 if g < units % world else 0)
        b0, b1 = min(start * align, bins), min((start + n) * align, bins)
        out.append((b0, b1))
        start += n
    return out


def row_chunks(rows: int, n_chunks: int) -> List[Tuple[int, int]]:
    step = -(-rows // max(n_chunks, 1))
    return [(r, min(r + step, rows)) for r in range(0, rows, step)]


def run_bin_chain(rank: int, world: int, chunks: Sequence[Tuple[int, int]], compute,
                  make_buffer, group=None):
    """Pipelined chain over ranks.  For each row chunk c: receive the running
    sums from rank-1 (unless first), compute(c, partial_in) -> partial_out
    (None on the last rank, which finishes the chunk), send to rank+1.
    `make_buffer(c)` allocates a receive buffer for chunk c.  Returns the
    last rank's per-chunk results."""
    import torch.distributed as dist
    results = []
    for c in chunks:
        pin = None
        if rank > 0:
            pin = make_buffer(c)
            dist.recv(pin, src=rank - 1, group=group)
        out = compute(c, pin)
        if rank < world - 1:
            dist.send(out, dst=rank + 1, group=group)
        else:
            results.append(out)
    return results


# ---------------------------------------------------------------- one frame
@dataclass(frozen=True)
class Work:
    """One sweep request of a frame, or a row chunk of it: (kernel, scale)
    index `key` on table set `group`, map rows [v0, v1), estimated cost."""
    key: Tuple[int, int]
    group: int
    rows: Tuple[int, int]
    cost: float


def _lpt(items: Sequence[Work], build: Sequence[float], world: int):
    """Longest-processing-time assignment; a rank pays a table set's build
    the first time it takes a request on it (the build is replicated on
    every rank that sweeps it: a local rebuild at HBM speed beats shipping
    the tables over NVLink)."""
    load = [0.0] * world
    sets: List[set] = [set() for _ in range(world)]
    out: List[List[Work]] = [[] for _ in range(world)]
    for it in sorted(items, key=lambda w: (-w.cost, w.key, w.rows)):
        best, best_load = 0, None
        for r in range(world):
            l = load[r] + it.cost + (0.0 if it.group in sets[r] else build[it.group])
            if best_load is None or l < best_load - 1e-12:
                best, best_load = r, l
        load[best] = best_load
        sets[best].add(it.group)
        out[best].append(it)
    return out, load


def _objective(load):
    """Makespan, then how many ranks share it (a split that only removes one
    of several equally busiest ranks is progress)."""
    top = max(load)
    return (round(top, 9), sum(1 for l in load if l >= top - 1e-9))


def plan_frame(requests: Sequence[Tuple[Tuple[int, int], int, int, float]],
               build: Sequence[float], world: int, min_rows: int = 64,
               max_splits: int = 256) -> List[List[Work]]:
    """Partition ONE frame's (kernel, scale) requests over `world` ranks
    (SURVEY §8e "Scales / kernels"): requests = (key, group, map rows, cost).
    LPT over whole requests first; while the busiest rank's largest item can
    be halved by map rows (>= 2 * min_rows) and halving shortens the
    makespan (or leaves fewer ranks at it), split it.  Deterministic, so every rank derives the same plan
    with no communication; every (request, map row) lands on exactly one
    rank.  Returns per-rank Work lists (requests in their original order)."""
    items = [Work(k, g, (0, rows), c) for k, g, rows, c in requests if rows > 0]
    plan, load = _lpt(items, build, world)
    for _ in range(max_splits if world > 1 else 0):
        top = max(range(world), key=lambda r: (load[r], -r))
        big = max(plan[top], key=lambda w: (w.cost, w.rows[1] - w.rows[0]), default=None)
        if big is None or big.rows[1] - big.rows[0] < 2 * min_rows:
            break
        mid = (big.rows[0] + big.rows[1]) // 2
        trial = [w for w in items if w != big] + [
            Work(big.key, big.group, (big.rows[0], mid), big.cost / 2),
            Work(big.key, big.group, (mid, big.rows[1]), big.cost / 2)]
        p2, l2 = _lpt(trial, build, world)
        if _objective(l2) >= _objective(load):
            break
        items, plan, load = trial, p2, l2
    order = {k: i for i, (k, _, _, _) in enumerate(requests)}
    return [sorted(p, key=lambda w: (order[w.key], w.rows)) for p in plan]


def combine_request_peaks(parts: Sequence[Tuple[Tuple[int, int], Tuple[int, int], float, int]],
                          map_widths) -> dict:
    """Per request key: the global peak (score, row-major index) over the row
    chunks the ranks swept.  parts: (key, rows, score, index within the
    chunk's rows); map_widths[key] = map width.  Reference tie rule."""
    best = {}
    for key, (v0, _), s, i in parts:
        gi = i + v0 * map_widths[key]
        if key not in best or better((s, gi), best[key]):
            best[key] = (s, gi)
    return best


# ---------------------------------------------------------------- device rows
def _wrap32(x):
    """int64 tensor -> the same values modulo 2^32 as int32 (two's complement)."""
    import torch
    x = x & 0xFFFFFFFF
    return torch.where(x >= 2 ** 31, x - 2 ** 32, x).to(torch.int32)


def band_contribution(last, y0: int):
    """A band's contribution to the global prefix row below it, from its
    LOCAL last record row (device int32 tensor (octets, planes, w+1, 8) of
    swg_tables_last_row): rows shift by y0, so the y-ramp gains y0 * count
    (and the y^2 ramp 2 y0 y + y0^2 count).  Modulo 2^32 like the tables."""
    c = last.to("cpu" if not last.is_cuda else last.device).long() & 0xFFFFFFFF
    out = c.clone()
    if c.shape[1] > 2:
        out[:, 2] = c[:, 2] + y0 * c[:, 0]
    if c.shape[1] > 4:
        out[:, 4] = c[:, 4] + 2 * y0 * c[:, 2] + y0 * y0 * c[:, 0]
    return out


def device_carry(lasts, y0s, rank: int):
    """Exclusive sum of the earlier bands' contributions (the carry rank
    `rank` adds to its local tables), as int32 words."""
    import torch
    acc = torch.zeros_like(lasts[0], dtype=torch.int64)
    for r in range(rank):
        acc = acc + band_contribution(lasts[r], y0s[r])
    return _wrap32(acc)


def exchange_last_rows_device(tables, y0: int, group=None):
    """The boundary prefix-row exchange on the device: all-gather every
    band's last record row (NCCL over NVLink on the box; gloo stages through
    the host in the CPU tests) and each band's origin, then turn this band's
    local 32-bit tables into the global rows y0.. (swg_tables_add_carry).
    Returns the carry."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    last = tables.last_row()
    nccl = dist.get_backend(group) == "nccl"
    send = last if nccl else last.cpu()
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    origins = [None] * world
    dist.all_gather_object(origins, int(y0), group=group)
    carry = device_carry([p.to(last.device) for p in parts], origins, rank).to(last.device)
    tables.add_carry(y0, carry.contiguous())
    return carry
