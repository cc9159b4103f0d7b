"""Data-format adapters against the UNMODIFIED reference, on CPU:
PGM frames (image.cpp:67-127) and the "hog-v1" / "ert-v1" model files (detector.cpp:291-351,
ert.cpp:358-469).  Files written by either side load bit-identically on the other; malformed
inputs raise the reference's exception class with the reference's message.

Reference tests restated: test_image.cpp:50-119 (PGM parse + error cases), test_detector.cpp:
353-394 and test_ert.cpp:406-443 (model round trips, version / shape errors)."""

import ctypes as C
import os

import numpy as np
import pytest

import paper_2006_00816_b200 as bl
from pyoracle import Reference, random_ert

pytestmark = pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref",
                                                                "libblinkline_ref.so")),
                                reason="reference library not built")


@pytest.fixture(scope="module")
def ref():
    r = Reference()
    L = r.lib
    L.ref_load_pgm.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p, C.c_longlong]
    L.ref_save_pgm.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int]
    L.ref_save_detector_json.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_double]
    L.ref_load_detector_json.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)] + \
        [C.POINTER(C.c_int)] * 4 + [C.POINTER(C.c_double)]
    L.ref_ert_save_json.argtypes = [C.c_void_p, C.c_char_p]
    L.ref_ert_load_json.argtypes = [C.c_char_p, C.c_void_p, C.POINTER(C.c_double), C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p]
    L.ref_last_error.restype = C.c_char_p
    return r


def ref_load_pgm(ref, path):
    w, h = C.c_int(), C.c_int()
    rc = ref.lib.ref_load_pgm(os.fsencode(path), C.byref(w), C.byref(h), None, 0)
    if rc:
        return rc, ref.lib.ref_last_error().decode()
    px = np.empty((h.value, w.value), np.float64)
    ref.lib.ref_load_pgm(os.fsencode(path), C.byref(w), C.byref(h), px.ctypes.data, px.size)
    return 0, px


# ------------------------------------------------------------------------- PGM ----
def test_pgm_roundtrip_both_ways(ref, tmp_path):
    r = np.random.default_rng(5)
    img = r.uniform(-20, 280, (37, 53))  # clamped and rounded on write
    p_ours, p_ref = tmp_path / "ours.pgm", tmp_path / "ref.pgm"
    bl.write_pgm(p_ours, img)
    a = img.ctypes.data
    assert ref.lib.ref_save_pgm(os.fsencode(p_ref), a, 53, 37) == 0
    assert open(p_ours, "rb").read() == open(p_ref, "rb").read()
    rc, px = ref_load_pgm(ref, p_ours)
    assert rc == 0
    assert np.array_equal(bl.read_pgm(p_ref).astype(np.float64), px)


@pytest.mark.parametrize("content", [
    b"P2\n# comment\n3 2\n255\n0 1 2\n# mid\n253 254 255\n",
    b"P5 2 2 200\n\x00\x01\x02\xc8",
    b"P2 1 1 9 9",
])
def test_pgm_valid_files_match(ref, tmp_path, content):
    p = tmp_path / "f.pgm"
    p.write_bytes(content)
    rc, px = ref_load_pgm(ref, p)
    assert rc == 0
    assert np.array_equal(bl.read_pgm(p).astype(np.float64), px)


@pytest.mark.parametrize("content", [
    b"", b"P6\n1 1\n255\n\x00", b"P5\n0 4\n255\n", b"P5\n2 2\n0\n", b"P5\n2 2\n300\n",
    b"P5\n2 2\n255", b"P5\n2 2\n255\n\x00\x01", b"P2\n2 2\n9\n1 2 3", b"P2\n2 1\n5\n1 6",
    b"P5\n2 2\n100\n\x00\x01\x02\xff", b"P5\nx 2\n255\n", b"P5\n99999999999 1\n255\n",
])
def test_pgm_errors_match_reference(ref, tmp_path, content):
    p = tmp_path / "bad.pgm"
    p.write_bytes(content)
    rc, msg = ref_load_pgm(ref, p)
    assert rc == 1  # io_error
    with pytest.raises(bl.IoError) as ei:
        bl.read_pgm(p)
    assert str(ei.value) == msg


def test_pgm_missing_file(ref, tmp_path):
    with pytest.raises(bl.IoError):
        bl.read_pgm(tmp_path / "nope.pgm")


# ---------------------------------------------------------------------- hog-v1 ----
def _det_model(seed):
    r = np.random.default_rng(seed)
    return {"weights": r.normal(0, 1, (5, 3100)), "biases": r.normal(0, 1, 5), "threshold": float(r.normal()),
            "window_cells": 10, "cell_px": 8, "scale_num": 5, "scale_den": 6, "min_face_ratio": 0.2}


def test_detector_json_roundtrip_both_ways(ref, tmp_path):
    m = _det_model(1)
    p_ours, p_ref = tmp_path / "ours.json", tmp_path / "ref.json"
    bl.write_detector_json(p_ours, m)
    w, b = m["weights"], m["biases"]
    assert ref.lib.ref_save_detector_json(os.fsencode(p_ref), w.ctypes.data, b.ctypes.data, m["threshold"], 10, 8,
                                          5, 6, 0.2) == 0
    assert open(p_ours).read() == open(p_ref).read()  # same serializer, same bytes
    got = bl.read_detector_json(p_ref)
    assert np.array_equal(got["weights"], w) and np.array_equal(got["biases"], b)
    assert got["threshold"] == m["threshold"] and got["window_cells"] == 10 and got["min_face_ratio"] == 0.2
    w2, b2 = np.empty_like(w), np.empty(5)
    thr = C.c_double()
    ints = [C.c_int() for _ in range(4)]
    mfr = C.c_double()
    assert ref.lib.ref_load_detector_json(os.fsencode(p_ours), w2.ctypes.data, b2.ctypes.data, C.byref(thr),
                                          *[C.byref(i) for i in ints], C.byref(mfr)) == 0
    assert np.array_equal(w2, w) and np.array_equal(b2, b) and thr.value == m["threshold"]


@pytest.mark.parametrize("text,err", [
    ("{not json", "invalid JSON"),
    ('{"version": "hog-v2"}', "unsupported model version"),
    ('{"version": "hog-v1", "window_cells": 10}', "malformed model file"),
])
def test_detector_json_errors(tmp_path, text, err):
    p = tmp_path / "m.json"
    p.write_text(text)
    with pytest.raises(bl.ModelError, match=err):
        bl.read_detector_json(p)
    with pytest.raises(bl.IoError):
        bl.read_detector_json(tmp_path / "missing.json")


def test_detector_json_wrong_filter_count(tmp_path):
    m = _det_model(2)
    p = tmp_path / "m.json"
    bl.write_detector_json(p, m)
    import json
    j = json.load(open(p))
    j["filters"] = j["filters"][:4]
    json.dump(j, open(p, "w"))
    with pytest.raises(bl.ModelError, match="expected exactly 5 filters"):
        bl.read_detector_json(p)
    j = json.load(open(p))
    bl.write_detector_json(p, m)
    j = json.load(open(p))
    j["filters"][2]["weights"] = j["filters"][2]["weights"][:100]
    json.dump(j, open(p, "w"))
    with pytest.raises(bl.ModelError, match="filter 2 carries 100 weights, expected 3100"):
        bl.read_detector_json(p)


# ---------------------------------------------------------------------- ert-v1 ----
def test_ert_json_roundtrip_both_ways(ref, tmp_path):
    ert = random_ert(L=68, T=2, K=7, F=3, seed=3)
    p_ours, p_ref = tmp_path / "ours.json", tmp_path / "ref.json"
    bl.write_ert_json(p_ours, ert)
    h = ref.ert_handle(ert) if hasattr(ref, "ert_handle") else None
    if h is None:
        h = ref.lib.ref_ert_create(ert["L"], ert["T"], ert["K"], ert["F"], ert["shrinkage"],
                                   ert["mean_xy"].ctypes.data_as(C.POINTER(C.c_double)),
                                   ert["anchors"].ctypes.data_as(C.POINTER(C.c_int32)),
                                   ert["split_params"].ctypes.data_as(C.POINTER(C.c_double)),
                                   ert["leaves"].ctypes.data_as(C.POINTER(C.c_double)))
    try:
        assert ref.lib.ref_ert_save_json(h, os.fsencode(p_ref)) == 0
    finally:
        ref.lib.ref_ert_destroy(h)
    assert open(p_ours).read() == open(p_ref).read()
    got = bl.read_ert_json(p_ref)
    for k in ("L", "T", "K", "F", "shrinkage"):
        assert got[k] == ert[k]
    for k in ("mean_xy", "anchors", "split_params", "leaves"):
        assert np.array_equal(got[k], np.asarray(ert[k]).reshape(got[k].shape)), k
    dims = (C.c_int * 4)()
    sh = C.c_double()
    bufs = {k: np.empty_like(got[k]) for k in ("mean_xy", "anchors", "split_params", "leaves")}
    assert ref.lib.ref_ert_load_json(os.fsencode(p_ours), dims, C.byref(sh), bufs["mean_xy"].ctypes.data,
                                     bufs["anchors"].ctypes.data, bufs["split_params"].ctypes.data,
                                     bufs["leaves"].ctypes.data) == 0
    assert list(dims) == [68, 2, 7, 3] and sh.value == ert["shrinkage"]
    for k, v in bufs.items():
        assert np.array_equal(v, got[k]), k


def test_ert_json_errors(tmp_path):
    ert = random_ert(L=68, T=1, K=2, F=2, seed=4)
    p = tmp_path / "e.json"
    bl.write_ert_json(p, ert)
    import json
    j = json.load(open(p))
    j["version"] = "ert-v0"
    json.dump(j, open(p, "w"))
    with pytest.raises(bl.ModelError, match="unsupported model version"):
        bl.read_ert_json(p)
    bl.write_ert_json(p, ert)
    j = json.load(open(p))
    j["cascade"][0][1]["splits"][0]["a"] = 68
    json.dump(j, open(p, "w"))
    with pytest.raises(bl.ModelError, match="split anchor out of range"):
        bl.read_ert_json(p)
    bl.write_ert_json(p, ert)
    j = json.load(open(p))
    j["cascade"][0][0]["leaves"] = j["cascade"][0][0]["leaves"][:3]
    json.dump(j, open(p, "w"))
    with pytest.raises(bl.ModelError, match="tree split/leaf counts do not match depth F"):
        bl.read_ert_json(p)
    with pytest.raises(bl.IoError):
        bl.read_ert_json(tmp_path / "missing.json")
