"""The BASELINE.json configurations as parity cases (the bench line is C1's 640x480 workload).

Each config runs at its full batch on the device; the CPU oracle checks a seeded subset of
frames / boxes exactly (it needs seconds per 1080p frame and ~5-10 ms per 15x500x4 face),
and size-independent properties cover the rest: a frame's result does not depend on the batch
it rides in (batch invariance), a box's landmarks do not depend on the other boxes (order
invariance), and repeated runs are bit-identical (determinism).

  C2  320x240 eyeblink stream, batch 16
  C3  1280x720, batch 64, full pyramid
  C4  landmark-only: 10k face boxes, 15-cascade x 500-tree depth-4 random-init ERT
  C5  1920x1080, batch 256 per GPU: the full batch, three frames checked against the
      oracle, batch invariance against one-frame batches (and a 32-frame determinism case)"""

import numpy as np
import pytest

from pyoracle import random_ert, ring_frames_np

pytestmark = pytest.mark.gpu


def _check_frames(ctx, oracle, model, ert, frames, idx):
    dets, lms = ctx.detect_landmarks(frames)
    faces = 0
    for i in idx:
        img = frames[i].astype(np.float64)
        want = oracle.detect_faces(img, model)
        assert np.array_equal(dets[i], want), i
        for j, d in enumerate(want[:3]):
            xy, _, _ = oracle.predict_landmarks(img, (d["x"], d["y"], d["w"], d["h"]), ert)
            assert np.max(np.abs(lms[i][j] - xy)) <= 1e-9
            faces += 1
    return dets, lms, faces


def test_c2_qvga_stream_batch16(ctx, oracle, pattern_model):
    frames = ring_frames_np(16, 320, 240, seed=202)
    ert = random_ert(T=4, K=100, F=4, seed=21)
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(ert)
    _, _, faces = _check_frames(ctx, oracle, pattern_model, ert, frames, range(16))
    assert faces >= 12


def test_c3_720p_batch64(ctx, oracle, pattern_model):
    frames = ring_frames_np(64, 1280, 720, seed=303)
    ert = random_ert(T=3, K=60, F=4, seed=31)
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(ert)
    dets, lms, faces = _check_frames(ctx, oracle, pattern_model, ert, frames, [0, 37, 63])
    assert faces > 0
    # batch invariance: frames 8..11 alone give the same results as inside the 64-frame batch
    d4, l4 = ctx.detect_landmarks(frames[8:12])
    for k in range(4):
        assert np.array_equal(d4[k], dets[8 + k]) and np.array_equal(l4[k], lms[8 + k])


def test_c4_ert_only_10k_boxes(ctx, oracle):
    ert = random_ert(L=68, T=15, K=500, F=4, seed=2020)
    img = np.floor(np.random.default_rng(404).uniform(0, 256, (480, 640)))
    r = np.random.default_rng(405)
    n = 10000
    side = r.integers(120, 280, n)
    boxes = np.stack([r.integers(0, 640 - side + 1), r.integers(0, 480 - side + 1), side, side], 1).astype(np.int32)
    ctx.upload_ert(ert)
    u8 = img.astype(np.uint8)
    xy, leaves = ctx.landmarks(u8, np.zeros(n, np.int32), boxes, want_leaves=True)
    assert xy.shape == (n, 68, 2) and leaves.shape == (n, 15 * 500)
    for i in r.choice(n, 40, replace=False):  # exact leaf indices, landmarks to 1e-9
        wxy, wl, _ = oracle.predict_landmarks(img, tuple(boxes[i]), ert)
        assert np.array_equal(leaves[i], wl), i
        assert np.max(np.abs(xy[i] - wxy)) <= 1e-9
    # every one of the 10k boxes against the unmodified reference library (all host threads):
    # a single flipped leaf decision would move a landmark by >= 1e-3 px, far above 1e-9 (the
    # device sums run in the canonical chunked order)
    import os

    from pyoracle import Reference, reference_available
    if reference_available():
        want = Reference().landmarks_batch_u8(u8[None], np.zeros(n, np.int32), boxes, ert, os.cpu_count() or 1,
                                              want_xy=True)
        assert np.max(np.abs(xy - want)) <= 1e-9
    # order invariance + determinism on all 10k
    perm = r.permutation(n)
    xy2 = ctx.landmarks(u8, np.zeros(n, np.int32), boxes[perm])
    assert np.array_equal(xy2, xy[perm])


def test_c5_1080p_batch(ctx, oracle, pattern_model):
    frames = ring_frames_np(32, 1920, 1080, seed=505)
    ert = random_ert(T=2, K=40, F=4, seed=51)
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(ert)
    dets, lms, faces = _check_frames(ctx, oracle, pattern_model, ert, frames, [5, 30])
    assert faces > 0
    again = ctx.detect_landmarks(frames)
    for k in range(32):
        assert np.array_equal(again[0][k], dets[k]) and np.array_equal(again[1][k], lms[k])


def test_c5_1080p_full_batch256(ctx, oracle, pattern_model):
    """C5 at its stated batch: 256 1920x1080 frames in one call (16 distinct ring frames
    cycled, so generation stays fast), with the bench's 15 x 500 x depth-4 cascade; frames 5,
    130 and 255 against the oracle, and the same frames as one-frame batches."""
    base = ring_frames_np(16, 1920, 1080, seed=515)
    frames = np.ascontiguousarray(base[np.arange(256) % 16])
    ert = random_ert(T=15, K=500, F=4, seed=2020)
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(ert)
    dets, lms, faces = _check_frames(ctx, oracle, pattern_model, ert, frames, [5, 130, 255])
    assert faces > 0 and sum(len(d) for d in dets) >= 256
    for k in (5, 130, 255):
        d1, l1 = ctx.detect_landmarks(frames[k:k + 1])
        assert np.array_equal(d1[0], dets[k]) and np.array_equal(l1[0], lms[k])


def test_bench_workload_vs_oracle(ctx, oracle, pattern_model):
    """bench.py's exact workload: 1024 640x480 ring frames (its default batch) in one call
    with the 15 x 500 x depth-4 cascade (seed 2020) on every kept detection; four frames
    against the oracle."""
    frames = ring_frames_np(1024, 640, 480, seed=1000)
    ert = random_ert(T=15, K=500, F=4, seed=2020)
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(ert)
    dets, lms, faces = _check_frames(ctx, oracle, pattern_model, ert, frames, [0, 257, 700, 1023])
    assert faces > 0 and sum(len(d) for d in dets) > 1024


def test_bench_batch_vs_small_batch_kernels(ctx, pattern_model):
    """The bench's 512-frame batch runs tall (64-row) gradHist segments and the 4-faces-per-CTA
    cascade; a 3-frame batch of the same frames runs 1-row segments and the face-per-CTA
    cascade (k_ert_wide).  Both configurations give bit-identical detections and landmarks."""
    frames = ring_frames_np(512, 640, 480, seed=606)
    ert = random_ert(T=3, K=120, F=4, seed=61)
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(ert)
    dets, lms = ctx.detect_landmarks(frames)
    assert sum(len(d) for d in dets) > 512
    for lo in (0, 200, 509):
        d3, l3 = ctx.detect_landmarks(frames[lo:lo + 3])
        for k in range(3):
            assert np.array_equal(d3[k], dets[lo + k]) and np.array_equal(l3[k], lms[lo + k])


def test_fused_unscored_levels_bit_identical(monkeypatch, pattern_model):
    """1080p: levels 1-5 lie below the smallest eligible face, so the chain runs them as fused
    pairs (k_resample_pair: the unscored level stays in shared memory).  Detections and
    landmarks equal those of the level-by-level chain (BL_PYR_FUSE=0) bit for bit."""
    import paper_2006_00816_b200 as bl
    frames = ring_frames_np(6, 1920, 1080, seed=707)
    ert = random_ert(T=2, K=40, F=4, seed=71)
    out = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("BL_PYR_FUSE", fuse)
        c = bl.Context(0)
        c.upload_detector(pattern_model)
        c.upload_ert(ert)
        out[fuse] = c.detect_landmarks(frames)
        c.close()
    assert sum(len(d) for d in out["1"][0]) > 0
    for k in range(len(frames)):
        assert np.array_equal(out["1"][0][k], out["0"][0][k]) and np.array_equal(out["1"][1][k], out["0"][1][k])


@pytest.mark.parametrize("w,h,n,f64", [(640, 480, 1, False), (320, 240, 16, False), (333, 250, 3, True),
                                       (161, 97, 2, False)])
def test_pyramid_chain_bit_identical(monkeypatch, oracle, pattern_model, w, h, n, f64):
    """Small batches build the pyramid in one cooperative launch (k_pyramid_chain, grid barrier
    between levels); detections and landmarks equal the per-level chain's (BL_PYR_CHAIN=0) bit
    for bit, and the oracle's."""
    import paper_2006_00816_b200 as bl
    frames = ring_frames_np(n, w, h, seed=w + n)
    if f64:
        frames = frames.astype(np.float64) + 0.25
    ert = random_ert(T=2, K=40, F=4, seed=72)
    out = {}
    for chain in ("1", "0"):
        monkeypatch.setenv("BL_PYR_CHAIN", chain)
        c = bl.Context(0)
        c.upload_detector(pattern_model)
        c.upload_ert(ert)
        out[chain] = c.detect_landmarks(frames)
        c.close()
    for k in range(n):
        assert np.array_equal(out["1"][0][k], out["0"][0][k]) and np.array_equal(out["1"][1][k], out["0"][1][k])
    img = frames[0].astype(np.float64)
    assert np.array_equal(out["1"][0][0], oracle.detect_faces(img, pattern_model))
