"""The frame-sequence runtime: ingest() + run() over a PGM
directory with the detect and landmark stages on the device, against the UNMODIFIED
reference's run() (pipeline.cpp:358-404, blink.cpp:47-93).

CPU: ingest's directory validation and error messages.  GPU: per-frame detections
bit-identical, the face (best detection) identical, its 68 landmarks / EARs / closures and the
EAR baselines within 1e-9 (the ERT similarity transform's libm), and the
sequential (batch 1) and pipelined (batch 16) runs identical to each other -- the reference's
mode-equivalence contract (test_pipeline.cpp:92-123, acceptance C8)."""

import os

import numpy as np
import pytest

import paper_2006_00816_b200 as bl
from pyoracle import Reference, random_ert, ring_frames_np

REF_SO = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libblinkline_ref.so")
needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built")


def write_frames(d, frames):
    os.makedirs(d, exist_ok=True)
    for i, f in enumerate(frames):
        bl.write_pgm(os.path.join(d, f"frame_{i:06d}.pgm"), f)


def _dummy_models():
    det = {"weights": np.zeros((5, 3100)), "biases": np.zeros(5), "threshold": 0.0}
    return det, random_ert(L=68, T=1, K=2, F=1, seed=0)


@needs_ref
@pytest.mark.parametrize("case", ["gap", "dims", "empty", "notdir", "badheader"])
def test_ingest_errors_match_reference(tmp_path, case):
    d = str(tmp_path / "seq")
    frames = ring_frames_np(3, 64, 48, seed=1)
    if case == "gap":
        write_frames(d, frames)
        os.remove(os.path.join(d, "frame_000001.pgm"))
    elif case == "dims":
        write_frames(d, frames)
        bl.write_pgm(os.path.join(d, "frame_000002.pgm"), np.zeros((40, 64)))
    elif case == "empty":
        os.makedirs(d)
        open(os.path.join(d, "notes.txt"), "w").write("x")
    elif case == "notdir":
        d = str(tmp_path / "missing")
    else:
        write_frames(d, frames)
        open(os.path.join(d, "frame_000001.pgm"), "wb").write(b"P7\n")
    det, ert = _dummy_models()
    with pytest.raises(RuntimeError) as ref_err:
        Reference().run(d, det, ert, 30.0)
    with pytest.raises(bl.IoError) as ours:
        bl.ingest(d)
    assert str(ours.value) == str(ref_err.value)


def test_ingest_ok(tmp_path):
    d = str(tmp_path / "seq")
    write_frames(d, ring_frames_np(5, 80, 60, seed=2))
    assert bl.ingest(d) == (5, 80, 60)


@pytest.mark.gpu
@needs_ref
def test_run_matches_reference(tmp_path, ctx, pattern_model):
    d = str(tmp_path / "seq")
    frames = ring_frames_np(20, 320, 240, seed=31)
    frames[7] = 20  # a frame without a face (absent trace markers)
    write_frames(d, frames)
    ert = random_ert(L=68, T=3, K=40, F=3, seed=12)
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(ert)
    ours = ctx.run(d, 30.0, batch_size=1)
    ours16 = ctx.run(d, 30.0, batch_size=16)
    ref = Reference().run(d, pattern_model, ert, 30.0, pipelined=True, batch_size=8)
    fr = ours["frames"]
    assert len(fr) == 20
    # sequential and pipelined device runs are identical (mode equivalence)
    for k in ("n_detections", "face_found", "face", "ear_left", "ear_right", "closure_left", "closure_right"):
        assert np.array_equal(fr[k], ours16["frames"][k]), k
    assert np.array_equal(ours["detections"], ours16["detections"])
    # against the reference run
    assert np.array_equal(fr["n_detections"], ref["n_detections"])
    assert np.array_equal(fr["face_found"], ref["face_found"])
    assert fr["face_found"].sum() >= 15 and fr["face_found"][7] == 0
    assert np.array_equal(ours["detections"], ref["detections"])
    has = fr["face_found"] == 1
    assert np.array_equal(fr["face"][has], ref["faces"][has])
    assert np.nanmax(np.abs(ours["landmarks"][has] - ref["landmarks"][has])) <= 1e-9
    mine = np.stack([fr["ear_left"], fr["ear_right"], fr["closure_left"], fr["closure_right"]], 1)
    assert np.max(np.abs(mine[has] - ref["ears"][has])) <= 1e-9
    assert np.all(np.isnan(ref["ears"][~has]))
    assert np.max(np.abs(ours["baselines"] - ref["baselines"])) <= 1e-9
    assert np.allclose(fr["t"], np.arange(20) / 30.0, rtol=0, atol=0)


@pytest.mark.gpu
def test_run_errors(tmp_path, ctx, pattern_model):
    d = str(tmp_path / "seq")
    write_frames(d, np.full((3, 240, 320), 20, np.uint8))  # no faces anywhere
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(random_ert(L=68, T=1, K=4, F=2, seed=3))
    with pytest.raises(ValueError, match="no frames with a detected face"):
        ctx.run(d, 30.0)
    ctx.upload_ert(random_ert(L=10, T=1, K=4, F=2, seed=3))
    with pytest.raises(ValueError, match="no eye mapping for L=10"):
        ctx.run(d, 30.0)
