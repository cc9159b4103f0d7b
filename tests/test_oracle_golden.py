"""The CPU oracle (oracle/blink_oracle.c) pinned against the reference.

1. Bit-exact against the golden vectors in tests/golden/, produced by the UNMODIFIED reference
   library from the reference's own seeded generators (oracle/make_golden.py).
2. The reference's known-answer unit tests (proj/tests/test_*.cpp) restated against the oracle.
3. When the reference library is available (oracle/_ref, build container), oracle == reference
   on fresh random cases.
"""

import numpy as np
import pytest

from conftest import golden


# ------------------------------------------------------------------ golden vectors ----
def test_pyramid_golden(oracle):
    g = golden("pyramid")
    levels, scales = oracle.build_pyramid(g["image"], 80)
    assert len(levels) == sum(1 for k in g if k.startswith("level"))
    for k, lv in enumerate(levels):
        assert np.array_equal(lv, g[f"level{k}"])
    assert np.array_equal(scales, g["scales"])


@pytest.mark.parametrize("name", ["rand64", "rand16", "rand40x32", "ring", "tie_up", "tie_down", "ramp"])
def test_hog_golden(oracle, name):
    g = golden("hog")
    ori, mag = oracle.compute_gradients(g[f"{name}_img"])
    assert np.array_equal(ori, g[f"{name}_ori"]) and np.array_equal(mag, g[f"{name}_mag"])
    bins = oracle.histogramize(ori, mag)
    assert np.array_equal(bins, g[f"{name}_bins"])
    if bins.size:
        en = oracle.cell_energy(bins)
        assert np.array_equal(en, g[f"{name}_energy"])
        assert np.array_equal(oracle.compute_features(bins, en), g[f"{name}_feat"])
        assert np.array_equal(oracle.extract_features(g[f"{name}_img"]), g[f"{name}_feat"])


def test_tie_asymmetry_pinned(oracle):
    """gx == 0 ties: gy > 0 -> bin 4, gy < 0 -> bin 14 (the glibc table's uy[14] < uy[13];
    SURVEY.md §0.4).  Pinned by the reference-generated tie_up / tie_down fixtures."""
    g = golden("hog")
    assert set(np.unique(g["tie_up_ori"][1:-1, 1:-1])) == {4}
    assert set(np.unique(g["tie_down_ori"][1:-1, 1:-1])) == {14}
    ux, uy = oracle.direction_table()
    assert uy[4] == uy[5] and uy[14] < uy[13]


def test_classifier_golden(oracle):
    g = golden("classifier")
    assert np.array_equal(oracle.score_dense(g["feat"], g["weights"], float(g["bias"])), g["dense"])
    sep = oracle.score_separable(g["feat"], g["weights"], float(g["bias"]))
    assert np.array_equal(sep, g["separable"])
    assert np.array_equal(oracle.threshold_detections(sep, 0.5, 2, 3), g["thr_dets"])


def test_nms_golden(oracle):
    g = golden("nms")
    assert np.array_equal(oracle.nms(g["dets"], 0.5), g["kept"])


@pytest.mark.parametrize("case", ["c1", "planted", "qvga", "blank", "small"])
def test_detect_golden(oracle, pattern_model, case):
    g = golden("detect")
    got = oracle.detect_faces(g[f"{case}_img"].astype(np.float64), pattern_model)
    assert np.array_equal(got, g[f"{case}_dets"])


def test_detect_random_filters_golden(oracle):
    g = golden("detect")
    m = {"weights": g["random_weights"], "biases": g["random_biases"], "threshold": float(g["random_threshold"])}
    assert np.array_equal(oracle.detect_faces(g["qvga_img"].astype(np.float64), m), g["random_dets"])


def test_ert_golden(oracle):
    g = golden("ert")
    ert = {k: g[k] for k in ("anchors", "split_params", "leaves")}
    ert.update(L=int(g["L"]), T=int(g["T"]), K=int(g["K"]), F=int(g["F"]), shrinkage=float(g["shrinkage"]),
               mean_xy=g["mean_xy"])
    img = g["image"].astype(np.float64)
    for i, b in enumerate(g["boxes"]):
        xy, leaf, ev = oracle.predict_landmarks(img, tuple(b), ert)
        assert np.array_equal(xy, g["landmarks"][i])
        assert np.array_equal(leaf, g["leaf_idx"][i])
        assert ev == g["evals"][i] == ert["T"] * ert["K"] * ert["F"]


def test_similarity_golden(oracle):
    g = golden("similarity")
    assert np.array_equal(oracle.similarity_transform(g["frm"], g["to"]), g["tform"])
    from pyoracle import face68_mean_shape_np
    m = face68_mean_shape_np()
    assert np.array_equal(oracle.similarity_transform(m * 1.1 + 0.01, m), g["face_tform"])


# ----------------------------------------------------- reference known-answer tests ----
def test_pyramid_known_answers(oracle):
    levels, scales = oracle.build_pyramid(np.full((480, 640), 10.0), 80)
    assert [lv.shape[0] for lv in levels] == [480, 400, 333, 277, 230, 191, 159, 132, 110, 91]
    import math
    assert list(scales) == [1.0] + [math.pow(5 / 6, k) for k in range(1, 10)]  # glibc pow, image.cpp:169
    assert len(oracle.build_pyramid(np.full((80, 80), 1.0), 80)[0]) == 1
    assert len(oracle.build_pyramid(np.full((60, 60), 1.0), 80)[0]) == 1
    assert np.all(oracle.downscale_bilinear(np.full((12, 12), 100.0)) == 100.0)


def test_hog_known_answers(oracle):
    _, mag = oracle.compute_gradients(np.full((10, 10), 42.0))
    assert np.all(mag == 0)
    ori, mag = oracle.compute_gradients(np.tile(np.arange(8.0), (8, 1)))
    assert np.all(mag[1:7, 1:7] == 2.0) and np.all(ori[1:7, 1:7] == 0)
    ori = np.zeros((32, 32), np.uint8)
    mag = np.zeros((32, 32))
    ori[11, 11], mag[11, 11] = 4, 8.0
    b = oracle.histogramize(ori, mag)
    assert b[1, 1, 4] == 8 * 0.9375 ** 2 and b[0, 0, 4] == 8 * 0.0625 ** 2 and b.sum() == 8.0
    assert oracle.cell_energy(np.ones((1, 1, 18)))[0, 0] == 36.0
    with pytest.raises(ValueError):
        oracle.compute_gradients(np.zeros((5, 2)))


def test_detector_known_answers(oracle):
    feat = np.random.default_rng(31).uniform(-0.2, 0.4, (12, 13, 31))
    w = np.zeros(3100)
    w[5] = 1.0
    assert np.array_equal(oracle.score_dense(feat, w, 0.0), feat[:3, :4, 5])
    sal = np.zeros((4, 5))
    sal[2, 3] = 2.0
    d = oracle.threshold_detections(sal, 1.0, 0, 1)
    assert len(d) == 1 and (d[0]["x"], d[0]["y"], d[0]["w"]) == (24, 16, 80)
    sal = np.zeros((4, 5))
    sal[0, 0] = 2.0
    assert oracle.threshold_detections(sal, 1.0, 2, 0)[0]["w"] == 115
    assert oracle.eligible_scales(640, 480, 10) == list(range(1, 10))
    assert oracle.eligible_scales(640, 480, 4, min_face_ratio=0.0) == [0, 1, 2, 3]
    assert oracle.eligible_scales(100, 100, 2, min_face_ratio=0.9) == [1]
    with pytest.raises(ValueError):
        oracle.score_dense(np.zeros((12, 9, 31)), np.zeros(3100), 0.0)


# ------------------------------------------------------ oracle == reference (live) ----
def _reference():
    from pyoracle import Reference, reference_available
    if not reference_available():
        pytest.skip("reference library not built here")
    return Reference()


def test_oracle_matches_reference_random(oracle, pattern_model):
    ref = _reference()
    r = np.random.default_rng(2024)
    for trial in range(3):
        img = np.floor(r.uniform(0, 256, (int(r.integers(90, 260)), int(r.integers(90, 330)))))
        lv_o, _ = oracle.build_pyramid(img)
        lv_r, _ = ref.build_pyramid(img)
        assert all(np.array_equal(a, b) for a, b in zip(lv_o, lv_r))
        assert np.array_equal(oracle.extract_features(img), ref.extract_features(img))
        assert np.array_equal(oracle.detect_faces(img, pattern_model), ref.detect_faces(img, pattern_model))
    from pyoracle import random_ert
    ert = random_ert(T=2, K=8, F=3, seed=3)
    img = np.floor(r.uniform(0, 256, (120, 160)))
    for box in [(10, 10, 80, 80), (0, 0, 160, 120), (-20, 30, 90, 70)]:
        xo, lo, eo = oracle.predict_landmarks(img, box, ert)
        xr, lr, er = ref.predict_landmarks(img, box, ert)
        assert np.array_equal(xo, xr) and np.array_equal(lo, lr) and eo == er
