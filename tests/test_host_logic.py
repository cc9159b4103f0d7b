"""Host-side logic that needs no GPU: batch geometry (the C-ABI's plan), the C++ drop-in's
scalar API helpers, synthetic-input generators and the bench's roofline accounting."""

import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("w,h,ratio", [(640, 480, 0.2), (320, 240, 0.2), (1280, 720, 0.2), (1920, 1080, 0.2),
                                       (100, 100, 0.9), (640, 480, 0.0), (81, 97, 0.2), (60, 60, 0.2)])
def test_plan_geometry_matches_oracle(oracle, w, h, ratio):
    import paper_2006_00816_b200 as bl
    levels, scored, sc, side = bl.plan_geometry(w, h, min_face_ratio=ratio)
    lv, scales = oracle.build_pyramid(np.zeros((h, w)), 80)
    assert levels == [(x.shape[1], x.shape[0]) for x in lv]
    elig = oracle.eligible_scales(w, h, len(lv), min_face_ratio=ratio)
    want = [k for k in elig if levels[k][0] // 8 >= 10 and levels[k][1] // 8 >= 10]
    assert scored == want
    for i, k in enumerate(scored):
        assert sc[i] == (5.0 / 6.0) ** k or sc[i] == np.power(5.0 / 6.0, k)
        d = oracle.threshold_detections(np.full((1, 1), 1.0), 0.0, k, 0)
        assert side[i] == d[0]["w"]


def test_plan_geometry_survey_configs():
    """SURVEY.md §8a geometry: C1 10 levels / eligible 1-9; C3 12 levels / 4-11; C5 15 / 6-14."""
    import paper_2006_00816_b200 as bl
    lv, sc, _, _ = bl.plan_geometry(640, 480)
    assert len(lv) == 10 and sc == list(range(1, 10))
    lv, sc, _, _ = bl.plan_geometry(320, 240)
    assert len(lv) == 6 and sc == list(range(0, 6))
    lv, sc, _, _ = bl.plan_geometry(1280, 720)
    assert len(lv) == 12 and sc == list(range(4, 12))
    lv, sc, _, _ = bl.plan_geometry(1920, 1080)
    assert len(lv) == 15 and sc == list(range(6, 15))


def test_plan_geometry_errors():
    import paper_2006_00816_b200 as bl
    with pytest.raises(ValueError):
        bl.plan_geometry(640, 480, window_cells=12)
    with pytest.raises(ValueError):
        bl.plan_geometry(0, 480)


def test_cpp_dropin_host_api():
    exe = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", ROOT, "tests/cpp/test_dropin"], check=True)
    r = subprocess.run([exe, "--host"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_synthetic_generators_deterministic():
    from paper_2006_00816_b200.synthetic import face68_mean_shape_np, random_ert, ring_frames_np
    a = ring_frames_np(2, 64, 48, seed=1)
    b = ring_frames_np(2, 64, 48, seed=1)
    assert a.dtype == np.uint8 and a.shape == (2, 48, 64) and np.array_equal(a, b)
    e = random_ert(T=2, K=3, F=2, seed=4)
    assert e["anchors"].shape == (2 * 3 * 3, 2) and e["leaves"].shape == (2 * 3 * 4, 68, 2)
    assert e["anchors"].max() < 68 and np.all(np.abs(e["split_params"][:, :4]) <= 0.15)
    m = face68_mean_shape_np()
    assert m.shape == (68, 2) and np.all((m > 0) & (m < 1))


def test_synthetic_mean_shape_matches_reference():
    from pyoracle import Reference, reference_available
    if not reference_available():
        pytest.skip("reference library not built here")
    from paper_2006_00816_b200.synthetic import face68_mean_shape_np
    assert np.array_equal(Reference().face68_mean_shape(), face68_mean_shape_np())


def test_bench_algorithmic_bytes():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    lw, lh, scored = bench.geometry()
    assert scored == list(range(1, 10))
    a = bench.algorithmic_bytes_per_frame()
    assert a["cells"] == 10164 and a["anchors"] == 5916
    assert abs(a["pyramid"] - 10.90e6) < 0.02e6        # SURVEY.md §8d C1 resample bytes
