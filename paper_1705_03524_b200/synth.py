"""Seeded synthetic inputs standing in for the paper's VOT2016 / WAMI imagery
(BASELINE.json configs; declared in DESIGN.md "Synthetic inputs").

All generators are integer-exact and deterministic for a given seed (numpy
PCG64), so the oracle and the GPU path are fed identical bytes.

  blurred_noise    uniform noise -> separable Gaussian blur (integer taps,
                   round-half-up) -> uint8/uint16/RGB
  plant            add a textured patch with a mean offset (clamped)
  config1..config5 the five BASELINE.json workloads
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def odd_window(s: int) -> int:
    """Declared even->odd scale mapping: kw = 2*round(s/2)+1."""
    return 2 * int(round(s / 2.0)) + 1


def gaussian_taps(sigma: float, scale: int = 1 << 12) -> np.ndarray:
    r = int(np.ceil(3 * sigma))
    x = np.arange(-r, r + 1, dtype=np.float64)
    return np.round(np.exp(-x * x / (2 * sigma * sigma)) * scale).astype(np.int64)


def _blur_axis(img: np.ndarray, taps: np.ndarray, axis: int) -> np.ndarray:
    r = len(taps) // 2
    pad = [(0, 0)] * img.ndim
    pad[axis] = (r, r)
    p = np.pad(img, pad, mode="reflect")
    acc = np.zeros(img.shape, np.int64)
    n = img.shape[axis]
    for i, t in enumerate(taps):
        sl = [slice(None)] * img.ndim
        sl[axis] = slice(i, i + n)
        acc += t * p[tuple(sl)]
    s = int(taps.sum())
    return (acc + s // 2) // s


def blurred_noise(h: int, w: int, seed: int, sigma: float = 3.0, channels: int = 0,
                  maxval: int = 255) -> np.ndarray:
    rng = np.random.default_rng(seed)
    shape = (h, w) if channels == 0 else (h, w, channels)
    img = rng.integers(0, maxval + 1, size=shape, dtype=np.int64)
    taps = gaussian_taps(sigma)
    img = _blur_axis(_blur_axis(img, taps, 0), taps, 1)
    # stretch the blurred field back over the full range (keeps bins populated)
    lo, hi = np.percentile(img, 0.5), np.percentile(img, 99.5)
    img = np.clip((img - lo) * maxval // max(hi - lo, 1), 0, maxval)
    return img


def plant(img: np.ndarray, cy: int, cx: int, ph: int, pw: int, offset: int, seed: int,
          maxval: int = 255) -> None:
    """Adds a textured patch (its own blurred noise, mean-shifted) in place."""
    rng = np.random.default_rng(seed)
    y0, x0 = cy - ph // 2, cx - pw // 2
    shape = (ph, pw) + img.shape[2:]
    tex = rng.integers(-24, 25, size=shape, dtype=np.int64)
    tex = _blur_axis(_blur_axis(tex, gaussian_taps(1.0), 0), gaussian_taps(1.0), 1)
    region = img[y0:y0 + ph, x0:x0 + pw]
    img[y0:y0 + ph, x0:x0 + pw] = np.clip(region // 2 + (maxval + 1) // 4 + offset + tex, 0, maxval)


def crop(img: np.ndarray, cx: int, cy: int, kw: int, kh: int) -> np.ndarray:
    hx, hy = (kw - 1) // 2, (kh - 1) // 2
    return np.ascontiguousarray(img[cy - hy:cy + hy + 1, cx - hx:cx + hx + 1])


@dataclass
class Scene:
    image: np.ndarray                  # uint8 HxW, uint16 HxW or uint8 HxWx3
    targets: list = field(default_factory=list)  # (cx, cy, w, h)


def gray_scene(h: int, w: int, seed: int, targets, offset: int = 48, maxval: int = 255) -> Scene:
    img = blurred_noise(h, w, seed, maxval=maxval)
    rng = np.random.default_rng(seed + 1)
    placed = []
    for i, (tw, th) in enumerate(targets):
        cx = int(rng.integers(tw, w - tw))
        cy = int(rng.integers(th, h - th))
        off = offset if i % 2 == 0 else -offset
        plant(img, cy, cx, th, tw, off * (maxval // 255), seed + 100 + i, maxval)
        placed.append((cx, cy, tw, th))
    dtype = np.uint8 if maxval == 255 else np.uint16
    return Scene(img.astype(dtype), placed)


def config1(seed: int = 1) -> Scene:
    """256x256 u8, one planted 32x32 target (BASELINE config 1)."""
    return gray_scene(256, 256, seed, [(32, 32)])


def config2(seed: int = 1) -> Scene:
    """1024x1024 u8, four planted targets (BASELINE config 2)."""
    return gray_scene(1024, 1024, seed, [(32, 32), (64, 64), (96, 96), (64, 64)])


def config5(seed: int = 1) -> Scene:
    """2048x2048 u16 gamma field (BASELINE config 5)."""
    rng = np.random.default_rng(seed)
    g = rng.gamma(2.0, 1.0, size=(2048, 2048))
    taps = gaussian_taps(3.0)
    g = (g * 4096).astype(np.int64)
    g = _blur_axis(_blur_axis(g, taps, 0), taps, 1)
    g = np.clip(g * 65535 // max(int(np.percentile(g, 99.9)), 1), 0, 65535)
    return Scene(g.astype(np.uint16), [])


def _texture(ph: int, pw: int, channels: int, seed: int, base: int, maxval: int = 255):
    """A target's own appearance: blurred texture around a base level."""
    rng = np.random.default_rng(seed)
    shape = (ph, pw) + ((channels,) if channels else ())
    tex = rng.integers(-40, 41, size=shape, dtype=np.int64)
    tex = _blur_axis(_blur_axis(tex, gaussian_taps(1.0), 0), gaussian_taps(1.0), 1)
    return np.clip(base + tex, 0, maxval)


@dataclass
class Sequence:
    frames: np.ndarray                 # (F, H, W, 3) uint8
    track: list                        # ground-truth (cx, cy) per frame
    size: tuple                        # target (w, h)
    search: int                        # search-region side


def config3(seed: int = 1, n_frames: int = 64, h: int = 1080, w: int = 1920,
            target=(48, 64), search: int = 256) -> Sequence:
    """64 RGB frames 1920x1080: static blurred colour noise, one 48x64 (w x h)
    target translating 0-4 px/frame per axis (BASELINE config 3).  The
    target's appearance is fixed (pasted), so the tracker's model from
    frame 0 applies to every frame."""
    bg = blurred_noise(h, w, seed, channels=3).astype(np.uint8)
    tw, th = target
    rng = np.random.default_rng(seed + 7)
    base = rng.integers(40, 216, size=3)
    tex = _texture(th, tw, 3, seed + 11, 0) + base
    tex = np.clip(tex, 0, 255).astype(np.uint8)
    cx, cy = w // 3, h // 3
    frames = np.empty((n_frames, h, w, 3), np.uint8)
    track = []
    for f in range(n_frames):
        if f:
            cx += int(rng.integers(0, 5))
            cy += int(rng.integers(0, 5))
        frames[f] = bg
        frames[f, cy - th // 2:cy - th // 2 + th, cx - tw // 2:cx - tw // 2 + tw] = tex
        track.append((cx, cy))
    return Sequence(frames, track, (tw, th), search)


def search_origin(seq: Sequence, f: int):
    """Open-loop search region of frame f: centred on frame f-1's ground
    truth (frame 0: its own), clamped to the frame."""
    cx, cy = seq.track[max(f - 1, 0)]
    h, w = seq.frames.shape[1:3]
    s = seq.search
    return (int(np.clip(cx - s // 2, 0, w - s)), int(np.clip(cy - s // 2, 0, h - s)))


def config4(seed: int = 1, h: int = 2160, w: int = 3840, n_targets: int = 16) -> Scene:
    """3840x2160 RGB blurred colour noise with 16 planted targets of sizes
    24..128 (BASELINE config 4)."""
    img = blurred_noise(h, w, seed, channels=3)
    rng = np.random.default_rng(seed + 1)
    sizes = np.round(np.geomspace(24, 128, n_targets)).astype(int)
    placed = []
    for i, s in enumerate(sizes):
        s = int(s)
        cx = int(rng.integers(s, w - s))
        cy = int(rng.integers(s, h - s))
        base = rng.integers(30, 226, size=3)
        tex = _texture(s, s, 3, seed + 200 + i, 0) + base
        img[cy - s // 2:cy - s // 2 + s, cx - s // 2:cx - s // 2 + s] = np.clip(tex, 0, 255)
        placed.append((cx, cy, s, s))
    return Scene(img.astype(np.uint8), placed)
