"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no filter taps, no butterflies, no
subband layout). It only draws the input signals d(n) / images with the shapes, value
distributions and structure of BASELINE.json's configs; the recipes are stated in
DESIGN.md §"Input recipe" and SURVEY.md §8(d):

* c1  1 x 1024, uniform[-1, 1], seed 42                      (BASELINE configs[0])
* c2  4096 x 65536, 3 sinusoids + N(0, 0.1), seed [1002, i]  (BASELINE configs[1])
* c3  512 x 512 uint8 image G(), seed 2184                     (BASELINE configs[2])
* c4  256 x 2048 x 2048 images G()/255, seed [3003, i]         (BASELINE configs[3])
* c5  32768 x 32768 image G()/255: rectangles seed 4004,
      noise per 256-row band seed [4004, band]                 (BASELINE configs[4])

They stand in for the paper's laser-Doppler recording (§V) and the Lena
image (§V, Fig. 12), neither of which is available.  Every generator is
seeded per unit (signal, image, row band) so any rank or test regenerates any shard.
"""
from __future__ import annotations

import numpy as np

SEEDS = {"c1": 42, "c2": 1002, "c3": 2184, "c4": 3003, "c5": 4004}

# Canonical shapes of BASELINE.json's five configs.
CONFIGS = {
    "c1": dict(kind="1d", n=1024, batch=1, levels=1),
    "c2": dict(kind="1d", n=65536, batch=4096, levels=10),
    "c3": dict(kind="2d", h=512, w=512, batch=1, levels=3),
    "c4": dict(kind="2d", h=2048, w=2048, batch=256, levels=5),
    "c5": dict(kind="2d", h=32768, w=32768, batch=1, levels=8),
}

C5_BAND_ROWS = 256
N_RECTS = 20


def c1_signal(n: int = 1024, seed: int = SEEDS["c1"]) -> np.ndarray:
    """BASELINE configs[0]: one signal of n samples ~ uniform[-1, 1] (fp32)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n).astype(np.float32)


def c2_signal(i: int, n: int = 65536, seed: int = SEEDS["c2"]) -> np.ndarray:
    """BASELINE configs[1], signal i: sum of 3 unit-amplitude sinusoids with frequencies
    log-uniform in [2^-12, 2^-2] cycles/sample and phases U[0, 2pi), plus N(0, sigma=0.1)."""
    rng = np.random.default_rng([seed, i])
    f = np.exp2(rng.uniform(-12.0, -2.0, 3))
    phi = rng.uniform(0.0, 2.0 * np.pi, 3)
    t = np.arange(n, dtype=np.float64)
    s = np.zeros(n, dtype=np.float64)
    for k in range(3):
        s += np.sin(2.0 * np.pi * f[k] * t + phi[k])
    s += rng.normal(0.0, 0.1, n)
    return s.astype(np.float32)


def c2_batch(first: int, count: int, n: int = 65536, seed: int = SEEDS["c2"]) -> np.ndarray:
    return np.stack([c2_signal(first + i, n, seed) for i in range(count)])


def _draw_rects(h: int, w: int, rng: np.random.Generator, count: int = N_RECTS):
    """Rectangle parameters, drawn in order (height, width, top, left, value) per rect."""
    rects = []
    for _ in range(count):
        rh = int(rng.integers(max(1, h // 16), max(1, h // 4) + 1))
        rw = int(rng.integers(max(1, w // 16), max(1, w // 4) + 1))
        top = int(rng.integers(0, h - rh + 1))
        left = int(rng.integers(0, w - rw + 1))
        val = int(rng.integers(0, 256))
        rects.append((top, left, rh, rw, val))
    return rects


def _paint(h: int, w: int, rows: slice, rects) -> np.ndarray:
    """Radial gradient 255*(1 - r/r_max) for the given row range, rectangles painted over it."""
    r0, r1 = rows.start, rows.stop
    cy, cx = (h - 1) / 2.0, (w - 1) / 2.0
    rmax = np.hypot(cy, cx) if (h > 1 or w > 1) else 1.0
    y = np.arange(r0, r1, dtype=np.float64)[:, None] - cy
    x = np.arange(w, dtype=np.float64)[None, :] - cx
    img = 255.0 * (1.0 - np.hypot(y, x) / rmax)
    for top, left, rh, rw, val in rects:
        a, b = max(top, r0), min(top + rh, r1)
        if a < b:
            img[a - r0:b - r0, left:left + rw] = val
    return img


def _finish(img: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    img = img + rng.normal(0.0, 8.0, img.shape)
    return np.rint(np.clip(img, 0.0, 255.0)).astype(np.uint8)


def image_u8(h: int, w: int, rng: np.random.Generator) -> np.ndarray:
    """Image generator G(H, W, rng): gradient + 20 rectangles + N(0, 8) noise, clipped,
    rounded half-to-even and cast to uint8 (BASELINE configs[2])."""
    rects = _draw_rects(h, w, rng)
    return _finish(_paint(h, w, slice(0, h), rects), rng)


def c3_image(size: int = 512, seed: int = SEEDS["c3"]) -> np.ndarray:
    """BASELINE configs[2]: uint8 image converted to fp32 exactly."""
    return image_u8(size, size, np.random.default_rng(seed)).astype(np.float32)


def c4_image(i: int, size: int = 2048, seed: int = SEEDS["c4"]) -> np.ndarray:
    """BASELINE configs[3], image i: G(size, size) as fp32(u8) / fp32(255)."""
    u8 = image_u8(size, size, np.random.default_rng([seed, i]))
    return u8.astype(np.float32) / np.float32(255.0)


def c4_image_u8(i: int, size: int = 2048, seed: int = SEEDS["c4"]) -> np.ndarray:
    """The 8-bit image behind c4_image(i) (for the uint8 lowpass path, §8(f) f1)."""
    return image_u8(size, size, np.random.default_rng([seed, i]))


def c4_batch(first: int, count: int, size: int = 2048, seed: int = SEEDS["c4"]) -> np.ndarray:
    return np.stack([c4_image(first + i, size, seed) for i in range(count)])


def c5_rows(r0: int, r1: int, size: int = 32768, seed: int = SEEDS["c5"],
            band_rows: int = C5_BAND_ROWS) -> np.ndarray:
    """BASELINE configs[4], rows [r0, r1) of the size x size image (r0, r1 multiples of
    band_rows): rectangles from default_rng(seed), noise per band from default_rng([seed, band])."""
    assert r0 % band_rows == 0 and r1 % band_rows == 0 and 0 <= r0 < r1 <= size
    rects = _draw_rects(size, size, np.random.default_rng(seed))
    out = np.empty((r1 - r0, size), dtype=np.float32)
    for b in range(r0 // band_rows, r1 // band_rows):
        a = b * band_rows
        img = _paint(size, size, slice(a, a + band_rows), rects)
        u8 = _finish(img, np.random.default_rng([seed, b]))
        out[a - r0:a - r0 + band_rows] = u8.astype(np.float32) / np.float32(255.0)
    return out


def uniform(shape, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Generic seeded fp32 uniform input for ragged / edge-case parity tests."""
    return np.random.default_rng(seed).uniform(lo, hi, shape).astype(np.float32)


# --------------------------------------------------------------------------- parallel fill
def _fill_worker(args):
    from multiprocessing import shared_memory
    name, shape, dtype, kind, lo, hi, kw = args
    shm = shared_memory.SharedMemory(name=name)
    try:
        arr = np.ndarray(shape, dtype=dtype, buffer=shm.buf)
        if kind == "c2":
            for i in range(lo, hi):
                arr[i] = c2_signal(kw["first"] + i, n=shape[-1])
        elif kind == "c4":
            for i in range(lo, hi):
                arr[i] = c4_image(kw["first"] + i, size=shape[-1])
        elif kind == "c4u8":
            for i in range(lo, hi):
                arr[i] = c4_image_u8(kw["first"] + i, size=shape[-1])
        elif kind == "c5":
            br = kw["band_rows"]
            arr[lo * br:hi * br] = c5_rows(kw["r0"] + lo * br, kw["r0"] + hi * br, size=kw["size"], band_rows=br)
        else:
            raise ValueError(kind)
    finally:
        shm.close()
    return hi - lo


def generate(kind: str, *, first: int = 0, count: int | None = None, size: int | None = None,
             r0: int = 0, r1: int | None = None, workers: int | None = None, out: np.ndarray | None = None):
    """Fill a (possibly pinned, caller-provided) fp32 array with config `kind` units in parallel
    across host cores.  c2: signals [first, first+count); c4: images [first, first+count);
    c5: rows [r0, r1) of the size x size image.  Bit-identical to the per-unit generators."""
    import os
    from concurrent.futures import ProcessPoolExecutor
    from multiprocessing import shared_memory
    cfg = CONFIGS["c4" if kind == "c4u8" else kind]
    dtype = np.uint8 if kind == "c4u8" else np.float32
    if kind == "c2":
        n = size or cfg["n"]
        count = cfg["batch"] if count is None else count
        shape, units, kw = (count, n), count, {"first": first}
    elif kind in ("c4", "c4u8"):
        s = size or cfg["h"]
        count = cfg["batch"] if count is None else count
        shape, units, kw = (count, s, s), count, {"first": first}
    elif kind == "c5":
        s = size or cfg["h"]
        r1 = s if r1 is None else r1
        shape, units = (r1 - r0, s), (r1 - r0) // C5_BAND_ROWS
        kw = {"r0": r0, "size": s, "band_rows": C5_BAND_ROWS}
    else:
        raise ValueError(kind)
    workers = workers or min(32, len(os.sched_getaffinity(0)))
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    shm = shared_memory.SharedMemory(create=True, size=max(nbytes, 1))
    try:
        step = max(1, -(-units // (workers * 4)))
        tasks = [(shm.name, shape, dtype, kind, lo, min(units, lo + step), kw) for lo in range(0, units, step)]
        if workers <= 1 or len(tasks) <= 1:
            for t in tasks:
                _fill_worker(t)
        else:
            import multiprocessing as mp
            # forkserver: the caller may already hold CUDA / threads, where fork() is unsafe
            with ProcessPoolExecutor(workers, mp_context=mp.get_context("forkserver")) as ex:
                list(ex.map(_fill_worker, tasks))
        src = np.ndarray(shape, dtype=dtype, buffer=shm.buf)
        if out is None:
            out = np.empty(shape, dtype=dtype)
        np.copyto(out.reshape(shape), src)
        del src
    finally:
        shm.close()
        shm.unlink()
    return out
