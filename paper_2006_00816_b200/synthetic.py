"""Seeded synthetic inputs for the hot path: eyeblink-camera-like ring
frames, the face68 mean shape and random-init ERT cascades.  numpy only; used by bench.py,
__graft_entry__ and the tests.  The same arrays are fed to the GPU path and to the CPU
checkers, so nothing here needs to match the reference's own RNG streams."""

import numpy as np


def random_ert(L=68, T=15, K=500, F=4, seed=0, mean_xy=None, thr_range=64.0, off_range=0.15, leaf_range=0.02,
               shrinkage=0.1):
    """Random-init ERT cascade: anchors uniform, offsets U(-0.15,0.15), thresholds
    U(-64,64), leaves U(-0.02,0.02), shrinkage 0.1.  numpy-seeded; the same arrays are fed to the
    GPU path and to both CPU checkers."""
    rng = np.random.default_rng(seed)
    S, NL = (1 << F) - 1, 1 << F
    if mean_xy is None:
        mean_xy = face68_mean_shape_np() if L == 68 else rng.uniform(0.2, 0.8, (L, 2))
    return {
        "L": L, "T": T, "K": K, "F": F, "shrinkage": shrinkage,
        "mean_xy": np.ascontiguousarray(mean_xy, dtype=np.float64),
        "anchors": rng.integers(0, L, (T * K * S, 2), dtype=np.int32),
        "split_params": np.concatenate([rng.uniform(-off_range, off_range, (T * K * S, 4)),
                                        rng.uniform(-thr_range, thr_range, (T * K * S, 1))], axis=1),
        "leaves": rng.uniform(-leaf_range, leaf_range, (T * K * NL, L, 2)),
    }


def face68_mean_shape_np():
    """numpy restatement of tests/helpers.cpp:156-179 (face68_mean_shape)."""
    pts = np.zeros((68, 2))
    pi = np.pi
    for i in range(17):
        a = pi * float(i) / 16.0
        pts[i] = (0.5 - 0.38 * np.cos(a), 0.52 + 0.40 * np.sin(a))
    for i in range(17, 22):
        pts[i] = (0.22 + 0.06 * (i - 17), 0.30)
    for i in range(22, 27):
        pts[i] = (0.54 + 0.06 * (i - 22), 0.30)
    for i in range(27, 31):
        pts[i] = (0.5, 0.36 + 0.05 * (i - 27))
    for i in range(31, 36):
        pts[i] = (0.42 + 0.04 * (i - 31), 0.56)

    def hexa(base, cx, cy, rx, ry):
        pts[base:base + 6] = [(cx - rx, cy), (cx - rx / 2, cy - ry), (cx + rx / 2, cy - ry), (cx + rx, cy),
                              (cx + rx / 2, cy + ry), (cx - rx / 2, cy + ry)]
    hexa(36, 0.35, 0.42, 0.08, 0.045)
    hexa(42, 0.65, 0.42, 0.08, 0.045)
    for i in range(48, 60):
        a = 2.0 * pi * float(i - 48) / 12.0
        pts[i] = (0.5 + 0.14 * np.cos(a), 0.72 + 0.06 * np.sin(a))
    for i in range(60, 68):
        a = 2.0 * pi * float(i - 60) / 8.0
        pts[i] = (0.5 + 0.08 * np.cos(a), 0.72 + 0.03 * np.sin(a))
    return pts


def ring_frames_np(n, w, h, seed=0, size_frac=0.5, jitter=0.1):
    """Synthetic eyeblink-camera frames: flat 20 + U(-1.5,1.5) noise + a
    concentric-ring target (dark core 30 / bright ring 225 / dark outer 60, radii
    0.18/0.34/0.47 of the box side, as tests/helpers.cpp:33-52 draws it), centre jittered per
    frame, rounded to u8 exactly like the PGM round trip.  Vectorised numpy; returns (n,h,w) u8."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    out = np.empty((n, h, w), np.uint8)
    size = size_frac * min(w, h)
    for i in range(n):
        img = 20.0 + rng.uniform(-1.5, 1.5, (h, w))
        img = np.clip(img, 0.0, 255.0)
        cx = w / 2 + rng.uniform(-jitter, jitter) * w
        cy = h / 2 + rng.uniform(-jitter, jitter) * h
        r = np.hypot(xx - cx, yy - cy)
        img = np.where(r <= 0.47 * size, 60.0, img)
        img = np.where(r <= 0.34 * size, 225.0, img)
        img = np.where(r <= 0.18 * size, 30.0, img)
        out[i] = np.floor(np.clip(img, 0, 255) + 0.5).astype(np.uint8)
    return out


def ring_frame_global(i, w, h, seed=1000, size_frac=0.5, jitter=0.1):
    """Frame `i` of a global synthetic sequence (the ring frames of ring_frames_np), generated
    from (seed, i) alone, so any shard [begin, end) of a global batch can be built by the
    rank that owns it and the shards concatenate to the same sequence for any world size."""
    return ring_frames_np(1, w, h, seed=(seed, i), size_frac=size_frac, jitter=jitter)[0]


def ring_frames_range(begin, end, w, h, seed=1000):
    """Frames [begin, end) of the global sequence of ring_frame_global, (end-begin, h, w) u8."""
    out = np.empty((max(0, end - begin), h, w), np.uint8)
    for j, i in enumerate(range(begin, end)):
        out[j] = ring_frame_global(i, w, h, seed)
    return out
