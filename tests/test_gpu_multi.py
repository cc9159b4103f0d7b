"""Several contexts, threads and devices in one process.

* bl_multi (MultiContext): a batch sharded over device slots (here the same GPU listed twice,
  one device on the lease) gives results bit-identical to one context running it whole.
* Two host threads, each with its own context, run concurrently and agree bit-for-bit.
* Kernel shared-memory opt-ins are per device, set at context creation (no process-wide
  static): a second context works from a fresh thread."""

import threading

import numpy as np
import pytest

import paper_2006_00816_b200 as bl
from pyoracle import random_ert, ring_frames_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def models(pattern_model):
    return pattern_model, random_ert(T=6, K=100, F=4, seed=31)


def _one(frames, models):
    c = bl.Context(0)
    c.upload_detector(models[0])
    c.upload_ert(models[1])
    return c.detect_landmarks(frames, flat=True)


def test_multi_context_matches_single(models):
    frames = ring_frames_np(23, 320, 240, seed=505)
    d0, c0, l0 = _one(frames, models)
    m = bl.MultiContext([0, 0, 0])
    m.set_batch_pixels(4 * 320 * 240)  # several submitted batches per shard
    m.upload_detector(models[0])
    m.upload_ert(models[1])
    d1, c1, l1 = m.detect_landmarks(frames)
    assert np.array_equal(c0, c1)
    assert np.array_equal(d0, d1)
    assert np.array_equal(l0, l1)
    assert len(d0) > 0
    assert m.last_device_ms.shape == (3,)
    # detection only, and an empty batch
    d2, c2 = m.detect_landmarks(frames, landmarks=False)
    assert np.array_equal(d2, d0) and np.array_equal(c2, c0)
    m.close()


def test_two_threads_two_contexts_bit_identical(models):
    frames = ring_frames_np(12, 640, 480, seed=606)
    want = _one(frames, models)
    got = [None, None]
    errs = []

    def work(i):
        try:
            for _ in range(3):
                got[i] = _one(frames, models)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for g in got:
        for a, b in zip(g, want):
            assert np.array_equal(a, b)


def test_upload_refused_while_batches_in_flight(models):
    c = bl.Context(0)
    c.upload_detector(models[0])
    c.upload_ert(models[1])
    frames = ring_frames_np(4, 320, 240, seed=1)
    t = c.submit(frames)
    with pytest.raises(RuntimeError, match="collect the submitted batches"):
        c.upload_ert(models[1])
    c.collect(t)
    c.upload_ert(models[1])  # fine once collected


def test_face_capacity_error_is_not_masked(models):
    """More kept detections than the device face capacity: collect raises the real cause, not
    'unknown ticket'."""
    c = bl.Context(0)
    rng = np.random.default_rng(3)
    det = {"weights": rng.uniform(-1, 1, (5, 3100)), "biases": np.zeros(5), "threshold": 0.0}
    c.upload_detector(det)
    c.upload_ert(models[1])
    c.set_face_capacity(1)
    frames = np.floor(rng.uniform(0, 256, (2, 240, 320))).astype(np.uint8)
    t = c.submit(frames)
    with pytest.raises(RuntimeError, match="device face capacity"):
        c.collect(t)
