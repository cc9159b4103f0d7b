"""Per-stage parity of the CUDA path against the CPU oracle (and the reference's golden
vectors), through the C-ABI.  Bar: bit-exact for every stage the reference defines to the last
bit; ERT landmarks within 1e-9 px (the only non-bit-exact step is the similarity transform's
linear part, taken directly instead of through hypot/atan2/cos/sin), leaf indices exact.

Reference tests restated here: test_image.cpp (bilinear, pyramid dims), test_hog.cpp (ramp,
border ring, atan2 oracle, single-pixel split, mass conservation, all-ones energy, feature
bounds, bin-rotation permutation), test_detector.cpp (zero features, delta filter, box mapping
known answers, NMS oracle, planted pattern), test_ert.cpp (zero-delta mean shape, single tree,
box-translation bitwise, op counts), acceptance C1-C5."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def rng(seed):
    return np.random.default_rng(seed)


# ------------------------------------------------------------------------- image ----
def test_pyramid_golden_bit_exact(ctx):
    g = golden("pyramid")
    levels, scales = ctx.build_pyramid(g["image"], 80)
    assert len(levels) == len([k for k in g if k.startswith("level")])
    for k, lv in enumerate(levels):
        assert np.array_equal(lv, g[f"level{k}"]), k
    assert np.array_equal(scales, g["scales"])


@pytest.mark.parametrize("w,h", [(640, 480), (320, 240), (1280, 720), (1920, 1080), (81, 97), (80, 80), (60, 60)])
def test_pyramid_matches_oracle(ctx, oracle, w, h):
    img = np.floor(rng(w * h).uniform(0, 256, (h, w)))
    lv_o, sc_o = oracle.build_pyramid(img, 80)
    lv_g, sc_g = ctx.build_pyramid(img.astype(np.uint8), 80)
    assert len(lv_o) == len(lv_g)
    for a, b in zip(lv_o, lv_g):
        assert np.array_equal(a, b)
    assert np.array_equal(sc_o, sc_g)


@pytest.mark.parametrize("w,h,win", [(1000, 121, 80), (97, 301, 80), (2000, 130, 80), (333, 1200, 80), (250, 170, 4),
                                     (33, 700, 2), (4096, 200, 80)])
def test_pyramid_odd_shapes(ctx, oracle, w, h, win):
    """Extreme aspect ratios and deep chains down to 2-pixel levels, f64 input (no
    integral-pixel shortcut)."""
    img = rng(w + h).uniform(0, 255, (h, w))
    lv_o, _ = oracle.build_pyramid(img, win)
    lv_g, _ = ctx.build_pyramid(img, win)
    assert len(lv_o) == len(lv_g) > 1
    for a, b in zip(lv_o, lv_g):
        assert np.array_equal(a, b)


def test_pyramid_640x480_dims(ctx):
    levels, _ = ctx.build_pyramid(np.full((480, 640), 10.0), 80)
    assert [lv.shape[0] for lv in levels] == [480, 400, 333, 277, 230, 191, 159, 132, 110, 91]
    assert levels[1].shape == (400, 533)


def test_downscale_constant_and_random(ctx, oracle):
    assert np.all(ctx.downscale_bilinear(np.full((12, 12), 100.0)) == 100.0)
    img = rng(3).uniform(0, 255, (37, 53))
    assert np.array_equal(ctx.downscale_bilinear(img), oracle.downscale_bilinear(img))
    with pytest.raises(ValueError):
        ctx.downscale_bilinear(np.zeros((1, 5)))


# --------------------------------------------------------------------------- hog ----
@pytest.mark.parametrize("name", ["rand64", "rand16", "rand40x32", "ring", "tie_up", "tie_down", "ramp"])
def test_hog_stages_golden(ctx, name):
    g = golden("hog")
    img = g[f"{name}_img"]
    ori, mag = ctx.compute_gradients(img)
    assert np.array_equal(ori, g[f"{name}_ori"])
    assert np.array_equal(mag, g[f"{name}_mag"])
    bins = ctx.histogramize(g[f"{name}_ori"], g[f"{name}_mag"])
    assert np.array_equal(bins, g[f"{name}_bins"])
    if bins.size:
        en = ctx.cell_energy(g[f"{name}_bins"])
        assert np.array_equal(en, g[f"{name}_energy"])
        f = ctx.compute_features(g[f"{name}_bins"], g[f"{name}_energy"])
        assert np.array_equal(f, g[f"{name}_feat"])
        f2, b2, e2 = ctx.extract_features(img, want_cells=True)
        assert np.array_equal(f2, g[f"{name}_feat"])
        assert np.array_equal(b2, g[f"{name}_bins"])
        assert np.array_equal(e2, g[f"{name}_energy"])


def test_orientation_exhaustive_integer_gradients(ctx, oracle):
    """Every integer gradient a u8 frame can produce, plus random and near-tie doubles."""
    gx, gy = np.meshgrid(np.arange(-255, 256, dtype=np.float64), np.arange(-255, 256, dtype=np.float64))
    gx, gy = gx.ravel(), gy.ravel()
    r = rng(9)
    ang = r.uniform(0, 2 * np.pi, 200000)
    ang2 = (np.arange(36) * np.pi / 18)[:, None] + r.uniform(-1e-12, 1e-12, (36, 2000))  # on/near every tie
    # the fast path's threshold margin: angles within 1e-8 .. 1e-4 rad of every bin midpoint
    ang3 = (np.arange(18) * np.pi / 9 + np.pi / 18)[:, None] + \
        np.sign(r.uniform(-1, 1, (18, 4000))) * np.exp(r.uniform(np.log(1e-8), np.log(1e-4), (18, 4000)))
    ang = np.concatenate([ang, ang3.ravel()])
    mags = r.uniform(1e-6, 400, ang.size)
    ex_gx = np.concatenate([gx, mags * np.cos(ang), 10 * np.cos(ang2.ravel()), r.uniform(-1e-13, 1e-13, 1000)])
    ex_gy = np.concatenate([gy, mags * np.sin(ang), 10 * np.sin(ang2.ravel()), r.uniform(-1e-13, 1e-13, 1000)])
    got = ctx.orientation_bins(ex_gx, ex_gy)
    ux, uy = oracle.direction_table()
    dots = ex_gx[:, None] * ux[None, :] + ex_gy[:, None] * uy[None, :]
    want = np.argmax(dots, axis=1)  # numpy argmax: first maximal index == strict-> scan
    assert np.array_equal(got, want.astype(np.uint8))
    # the asymmetric tie the oracle pins: gx == 0 -> bin 4 (gy>0), bin 14 (gy<0)
    assert list(ctx.orientation_bins([0.0, 0.0, 0.0], [10.0, -10.0, 0.0])) == [4, 14, 0]


def test_sqrt_fast_matches_ieee(ctx):
    """The branch-free gradient-magnitude sqrt equals IEEE sqrt on its whole input range."""
    r = rng(13)
    xs = [np.exp(r.uniform(np.log(1e-300), np.log(1e300), 4_000_000)),
          r.uniform(0, 2 * 255.0 ** 2, 4_000_000),                 # the u8 / level-pixel range
          np.arange(1, 2 * 255 ** 2 + 1, dtype=np.float64),          # every integer gradient norm^2
          np.nextafter(np.arange(1, 200001, dtype=np.float64) ** 2, 0),  # just below perfect squares
          np.nextafter(np.arange(1, 200001, dtype=np.float64) ** 2, np.inf)]
    for x in xs:
        fast, ieee = ctx.debug_sqrt(x)
        assert np.array_equal(fast, ieee)
        assert np.array_equal(ieee, np.sqrt(x))


def test_orientation_pathological_magnitudes(ctx, oracle):
    """Gradients far outside fp32 range take the exact slow path inside the batched kernel."""
    img = np.full((48, 48), 1e-310)
    img[::3, ::2] = 0.0
    img[10:20, 10:20] = 3e-200
    img[30:40, 5:15] = 255.0
    f, b, e = ctx.extract_features(img, want_cells=True)
    assert np.array_equal(b, oracle.histogramize(*oracle.compute_gradients(img)))
    assert np.array_equal(f, oracle.extract_features(img))


def test_gradients_basic_cases(ctx):
    ori, mag = ctx.compute_gradients(np.full((10, 10), 42.0))
    assert np.all(mag == 0)
    ramp = np.tile(np.arange(8.0), (8, 1))
    ori, mag = ctx.compute_gradients(ramp)
    assert np.all(mag[1:7, 1:7] == 2.0) and np.all(ori[1:7, 1:7] == 0)
    ori, mag = ctx.compute_gradients(rng(1).uniform(0, 255, (7, 9)))
    assert np.all(mag[0] == 0) and np.all(mag[-1] == 0) and np.all(mag[:, 0] == 0) and np.all(mag[:, -1] == 0)
    with pytest.raises(ValueError):
        ctx.compute_gradients(np.zeros((5, 2)))


def test_histogram_single_pixel_split(ctx):
    ori = np.zeros((32, 32), np.uint8)
    mag = np.zeros((32, 32))
    ori[11, 11], mag[11, 11] = 4, 8.0
    b = ctx.histogramize(ori, mag)
    w1, w0 = 0.9375, 0.0625
    assert b[0, 0, 4] == 8 * w0 * w0 and b[0, 1, 4] == 8 * w1 * w0
    assert b[1, 0, 4] == 8 * w0 * w1 and b[1, 1, 4] == 8 * w1 * w1
    assert b.sum() == 8.0


@pytest.mark.parametrize("seed,w,h,border", [(9, 32, 32, 0), (10, 48, 40, 8), (11, 61, 45, 0), (12, 200, 130, 0)])
def test_histogram_random_fields(ctx, oracle, seed, w, h, border):
    r = rng(seed)
    ori = r.integers(0, 18, (h, w)).astype(np.uint8)
    mag = r.uniform(0, 10, (h, w))
    if border:
        mag[:border] = 0
        mag[-border:] = 0
        mag[:, :border] = 0
        mag[:, -border:] = 0
    assert np.array_equal(ctx.histogramize(ori, mag), oracle.histogramize(ori, mag))


def test_energy_features_known_answers(ctx):
    ones = np.ones((1, 1, 18))
    assert ctx.cell_energy(ones)[0, 0] == 36.0
    z = np.zeros((3, 3, 18))
    assert np.all(ctx.compute_features(z, ctx.cell_energy(z)) == 0)
    cg = rng(21).uniform(0, 4, (4, 5, 18))
    f = ctx.compute_features(cg, ctx.cell_energy(cg))
    assert np.all(f[..., :27] >= 0) and np.all(f[..., :27] <= 0.4 + 1e-12)
    with pytest.raises(ValueError):
        ctx.compute_features(np.zeros((2, 2, 18)), np.zeros((2, 3)))


def test_features_bin_rotation_permutation(ctx):
    cg = rng(23).uniform(0, 4, (5, 5, 18))
    base = ctx.compute_features(cg, ctx.cell_energy(cg))
    for k in (1, 5, 9, 13):
        rot = np.roll(cg, k, axis=2)
        moved = ctx.compute_features(rot, ctx.cell_energy(rot))
        assert np.allclose(np.roll(base[..., :18], k, axis=2), moved[..., :18], rtol=1e-9, atol=0)
        assert np.allclose(np.roll(base[..., 18:27], k % 9, axis=2), moved[..., 18:27], rtol=1e-9, atol=0)
        assert np.allclose(base[..., 27:], moved[..., 27:], rtol=1e-9, atol=0)


@pytest.mark.parametrize("seed,w,h", [(1, 640, 480), (2, 533, 400), (3, 147, 110), (4, 203, 97)])
def test_extract_features_random_frames(ctx, oracle, seed, w, h):
    img = rng(seed).uniform(0, 255, (h, w))
    assert np.array_equal(ctx.extract_features(img), oracle.extract_features(img))


# -------------------------------------------------------------------- classifier ----
def test_score_golden(ctx):
    g = golden("classifier")
    s = ctx.score_separable(g["feat"], g["weights"], float(g["bias"]))
    assert np.array_equal(s, g["separable"])
    assert np.max(np.abs(s - g["dense"])) <= 1e-4  # acceptance C1 contract
    # score_dense in its own (definitional) order: bit-identical to the reference's
    assert np.array_equal(ctx.score_dense(g["feat"], g["weights"], float(g["bias"])), g["dense"])


def test_score_dense_random_vs_oracle(ctx, oracle):
    feat = rng(71).uniform(0, 0.4, (23, 19, 31))
    w = rng(72).uniform(-1, 1, 3100)
    assert np.array_equal(ctx.score_dense(feat, w, 0.3), oracle.score_dense(feat, w, 0.3))
    assert not np.array_equal(ctx.score_dense(feat, w, 0.3), ctx.score_separable(feat, w, 0.3))


def test_score_known_answers(ctx):
    fi = np.zeros((11, 12, 31))
    s = ctx.score_separable(fi, np.zeros(3100), 2.5)
    assert s.shape == (2, 3) and np.all(s == 2.5)
    feat = rng(31).uniform(-0.2, 0.4, (12, 13, 31))
    w = np.zeros(3100)
    w[5] = 1.0
    assert np.array_equal(ctx.score_separable(feat, w, 0.0), feat[:3, :4, 5])
    with pytest.raises(ValueError):
        ctx.score_separable(np.zeros((12, 9, 31)), np.zeros(3100), 0.0)


# ---------------------------------------------------------------------------- nms ----
def test_nms_golden(ctx):
    g = golden("nms")
    assert np.array_equal(ctx.nms(g["dets"], 0.5), g["kept"])


def test_nms_edge_cases(ctx, oracle):
    import paper_2006_00816_b200 as bl
    assert len(ctx.nms(np.zeros(0, bl.DET_DTYPE))) == 0
    d = np.zeros(2, bl.DET_DTYPE)
    d[0] = (10, 10, 50, 50, 1.0, 0, 0)
    d[1] = (10, 10, 50, 50, 2.0, 0, 0)
    k = ctx.nms(d)
    assert len(k) == 1 and k[0]["score"] == 2.0
    # large set (global-memory sort path) against the oracle
    r = rng(7)
    n = 5000
    big = np.zeros(n, bl.DET_DTYPE)
    big["x"], big["y"] = r.integers(0, 600, n), r.integers(0, 400, n)
    big["w"] = big["h"] = r.integers(20, 120, n)
    big["score"] = np.round(r.uniform(0, 1, n), 3)  # many exact score ties -> tie-break order
    big["scale_index"], big["rotation_index"] = r.integers(0, 9, n), r.integers(0, 5, n)
    assert np.array_equal(ctx.nms(big), oracle.nms(big))


@pytest.mark.parametrize("n,xmax,scale_max", [(1500, 600, 9), (2048, 3000, 16), (700, 6000, 9), (300, 500, 20)])
def test_nms_compact_keys_and_fallback(ctx, oracle, n, xmax, scale_max):
    """Up to 2048 detections sort as 16-B keys in shared memory (x, y < 4096, scale < 16,
    rotation < 8 packed into 31 bits); frames outside those limits take the 32-B global-memory
    path.  Both keep the reference's total order under heavy score / position ties."""
    import paper_2006_00816_b200 as bl
    r = rng(n + xmax)
    d = np.zeros(n, bl.DET_DTYPE)
    d["x"], d["y"] = r.integers(0, xmax, n), r.integers(0, 400, n)
    d["x"][: n // 4] = d["x"][n // 4: 2 * (n // 4)]  # equal positions, different scale/rotation
    d["w"] = d["h"] = r.integers(20, 200, n)
    d["score"] = np.round(r.uniform(0, 1, n), 2)
    d["scale_index"], d["rotation_index"] = r.integers(0, scale_max, n), r.integers(0, 5, n)
    assert np.array_equal(ctx.nms(d), oracle.nms(d))


# ---------------------------------------------------------------- detect_faces ----
@pytest.mark.parametrize("case", ["c1", "planted", "qvga", "blank", "small"])
def test_detect_golden(ctx, pattern_model, case):
    g = golden("detect")
    ctx.upload_detector(pattern_model)
    got = ctx.detect(g[f"{case}_img"])[0]
    assert np.array_equal(got, g[f"{case}_dets"]), (got, g[f"{case}_dets"])


def test_detect_random_filters_golden(ctx):
    g = golden("detect")
    ctx.upload_detector({"weights": g["random_weights"], "biases": g["random_biases"],
                         "threshold": float(g["random_threshold"])})
    got = ctx.detect(g["qvga_img"])[0]
    assert len(got) == len(g["random_dets"]) > 10
    assert np.array_equal(got, g["random_dets"])


def test_detect_batch_matches_oracle(ctx, oracle, pattern_model):
    from pyoracle import ring_frames_np
    frames = ring_frames_np(6, 640, 480, seed=5)
    ctx.upload_detector(pattern_model)
    got = ctx.detect(frames)
    for i in range(len(frames)):
        want = oracle.detect_faces(frames[i].astype(np.float64), pattern_model)
        assert np.array_equal(got[i], want), i
    assert sum(len(g) for g in got) > 0


def test_detect_fp64_frames(ctx, oracle, pattern_model):
    img = np.clip(rng(36).uniform(-1.5, 1.5, (240, 320)) + 20, 0, 255)
    yy, xx = np.mgrid[0:240, 0:320]
    r = np.hypot(xx - 150.3, yy - 120.7)
    img = np.where(r < 0.47 * 110, 60.0, img)
    img = np.where(r < 0.34 * 110, 225.0, img)
    img = np.where(r < 0.18 * 110, 30.0, img)
    ctx.upload_detector(pattern_model)
    assert np.array_equal(ctx.detect(img)[0], oracle.detect_faces(img, pattern_model))


def test_detect_random_filters_many_detections(ctx, oracle):
    """Loose threshold: thousands of raw detections per frame exercise the screen cut, the
    exact re-score, and NMS far beyond the pattern detector's handful."""
    r = rng(77)
    model = {"weights": r.uniform(-1, 1, (5, 3100)) * 0.05, "biases": r.uniform(-1, 1, 5), "threshold": 0.3}
    img = np.floor(r.uniform(0, 256, (240, 320)))
    ctx.upload_detector(model)
    got = ctx.detect(img.astype(np.uint8))[0]
    want = oracle.detect_faces(img, model)
    assert len(want) > 20
    assert np.array_equal(got, want)


# --------------------------------------------------------------------------- ert ----
def _golden_ert():
    g = golden("ert")
    ert = {k: g[k] for k in ("anchors", "split_params", "leaves")}
    ert.update(L=int(g["L"]), T=int(g["T"]), K=int(g["K"]), F=int(g["F"]), shrinkage=float(g["shrinkage"]),
               mean_xy=g["mean_xy"])
    return g, ert


def test_ert_golden(ctx):
    g, ert = _golden_ert()
    ctx.upload_ert(ert)
    xy, leaves = ctx.landmarks(g["image"], np.zeros(len(g["boxes"]), np.int32), g["boxes"], want_leaves=True)
    assert np.array_equal(leaves, g["leaf_idx"])
    assert np.max(np.abs(xy - g["landmarks"])) <= 1e-9


def test_ert_random_vs_oracle(ctx, oracle):
    from pyoracle import random_ert
    ert = random_ert(T=4, K=60, F=4, seed=3)
    img = np.floor(rng(5).uniform(0, 256, (200, 260)))
    r = rng(6)
    n = 64
    boxes = np.stack([r.integers(-20, 200, n), r.integers(-20, 150, n), r.integers(30, 160, n),
                      r.integers(30, 160, n)], axis=1).astype(np.int32)
    ctx.upload_ert(ert)
    xy, leaves = ctx.landmarks(img.astype(np.uint8), np.zeros(n, np.int32), boxes, want_leaves=True)
    mism = 0
    for i in range(n):
        wxy, wl, ev = oracle.predict_landmarks(img, tuple(boxes[i]), ert)
        mism += int(not np.array_equal(leaves[i], wl))
        assert np.max(np.abs(xy[i] - wxy)) <= 1e-9
    assert mism == 0


@pytest.mark.parametrize("n", [3, 450])
def test_ert_wide_and_cascade_kernels_agree(monkeypatch, oracle, n):
    """k_ert_wide (face per CTA, small batches) and k_ert_cascade (4 faces per CTA) are the same
    arithmetic: bit-identical landmarks and leaves, both against the oracle."""
    import paper_2006_00816_b200 as bl
    from pyoracle import random_ert
    ert = random_ert(T=3, K=40, F=4, seed=11)
    img = np.floor(rng(12).uniform(0, 256, (240, 320)))
    r = rng(13)
    boxes = np.stack([r.integers(-20, 260, n), r.integers(-20, 180, n), r.integers(30, 160, n),
                      r.integers(30, 160, n)], axis=1).astype(np.int32)
    out = {}
    for mode in ("wide", "cascade"):
        monkeypatch.setenv("BL_ERT", mode)
        c = bl.Context(0)
        c.upload_ert(ert)
        out[mode] = c.landmarks(img.astype(np.uint8), np.zeros(n, np.int32), boxes, want_leaves=True)
        c.close()
    assert np.array_equal(out["wide"][0], out["cascade"][0])
    assert np.array_equal(out["wide"][1], out["cascade"][1])
    for i in range(0, n, max(1, n // 8)):
        wxy, wl, _ = oracle.predict_landmarks(img, tuple(boxes[i]), ert)
        assert np.array_equal(out["wide"][1][i], wl)
        assert np.max(np.abs(out["wide"][0][i] - wxy)) <= 1e-9


@pytest.mark.parametrize("K", [40, 300, 500])
def test_ert_cluster_sizes_agree(monkeypatch, oracle, K):
    """The small-batch cascade as clusters of 2, 4, 8 and 16 (non-portable) CTAs per face (k_ert_wcl: chunks
    spread over the cluster, partials broadcast through DSMEM; 2 = unstaged sums, 4 = two
    chunks per CTA, 8 = one chunk per CTA and ranks without a chunk when K <= 448) is
    bit-identical to the one-CTA kernel and matches the oracle's leaves and landmarks."""
    import paper_2006_00816_b200 as bl
    from pyoracle import random_ert
    ert = random_ert(T=3, K=K, F=4, seed=21)
    img = np.floor(rng(22).uniform(0, 256, (240, 320)))
    r = rng(23)
    n = 5
    boxes = np.stack([r.integers(-20, 260, n), r.integers(-20, 180, n), r.integers(30, 160, n),
                      r.integers(30, 160, n)], axis=1).astype(np.int32)
    out = {}
    for cl in (1, 2, 4, 8, 16):
        monkeypatch.setenv("BL_ERT", "wide")
        monkeypatch.setenv("BL_ERT_CL", str(cl))
        c = bl.Context(0)
        c.upload_ert(ert)
        out[cl] = c.landmarks(img.astype(np.uint8), np.zeros(n, np.int32), boxes, want_leaves=True)
        c.close()
    for cl in (2, 4, 8, 16):
        assert np.array_equal(out[cl][0], out[1][0]), cl
        assert np.array_equal(out[cl][1], out[1][1]), cl
    for i in range(n):
        wxy, wl, _ = oracle.predict_landmarks(img, tuple(boxes[i]), ert)
        assert np.array_equal(out[8][1][i], wl)
        assert np.max(np.abs(out[8][0][i] - wxy)) <= 1e-9


def test_ert_zero_delta_is_mean_shape(ctx):
    from pyoracle import face68_mean_shape_np
    mean = face68_mean_shape_np()
    T, K, F = 3, 4, 2
    S, NL = 3, 4
    ert = {"L": 68, "T": T, "K": K, "F": F, "shrinkage": 0.1, "mean_xy": mean,
           "anchors": np.zeros((T * K * S, 2), np.int32), "split_params": np.zeros((T * K * S, 5)),
           "leaves": np.zeros((T * K * NL, 68, 2))}
    ctx.upload_ert(ert)
    img = np.where(np.arange(64)[None, :] > 32, 200.0, 10.0) * np.ones((64, 1))
    xy = ctx.landmarks(img, [0], [[8, 8, 48, 48]])[0]
    assert np.array_equal(xy[:, 0], 8 + mean[:, 0] * 48) and np.array_equal(xy[:, 1], 8 + mean[:, 1] * 48)


def test_ert_single_tree_known_answer(ctx):
    ert = {"L": 2, "T": 1, "K": 1, "F": 1, "shrinkage": 0.1, "mean_xy": np.array([[0.25, 0.5], [0.75, 0.5]]),
           "anchors": np.array([[1, 0]], np.int32), "split_params": np.array([[0, 0, 0, 0, 50.0]]),
           "leaves": np.array([[[0.1, 0.2], [-0.1, 0.0]], [[9, 9], [9, 9]]], np.float64)}
    ctx.upload_ert(ert)
    img = np.where(np.arange(64)[None, :] > 32, 200.0, 10.0) * np.ones((64, 1))
    xy = ctx.landmarks(img, [0], [[8, 8, 48, 48]])[0]
    assert np.allclose(xy, [[8 + 0.26 * 48, 8 + 0.52 * 48], [8 + 0.74 * 48, 8 + 0.50 * 48]], rtol=1e-12, atol=0)


def test_ert_box_translation_bitwise(ctx):
    from pyoracle import random_ert
    r = rng(43)
    img = r.uniform(0, 255, (96, 96))
    shifted = np.zeros((96, 96))
    shifted[7:, 13:] = img[:-7, :-13]
    ert = random_ert(T=2, K=2, F=2, seed=44, thr_range=20, off_range=0.1)
    ctx.upload_ert(ert)
    a = ctx.landmarks(img, [0], [[20, 24, 40, 40]])[0]
    b = ctx.landmarks(shifted, [0], [[33, 31, 40, 40]])[0]
    assert np.array_equal(b[:, 0], a[:, 0] + 13) and np.array_equal(b[:, 1], a[:, 1] + 7)


def test_ert_degenerate_box_raises(ctx):
    from pyoracle import random_ert
    ctx.upload_ert(random_ert(T=1, K=1, F=1, seed=1))
    with pytest.raises(ValueError):
        ctx.landmarks(np.zeros((32, 32)), [0], [[0, 0, 0, 10]])


# ------------------------------------------------------------------ full pipeline ----
def test_detect_landmarks_pipeline(ctx, oracle, pattern_model):
    from pyoracle import random_ert, ring_frames_np
    frames = ring_frames_np(8, 640, 480, seed=11)
    ert = random_ert(T=3, K=50, F=4, seed=12)
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(ert)
    dets, lms = ctx.detect_landmarks(frames)
    faces = 0
    for i in range(len(frames)):
        img = frames[i].astype(np.float64)
        want = oracle.detect_faces(img, pattern_model)
        assert np.array_equal(dets[i], want)
        for j, d in enumerate(want):
            xy, _, _ = oracle.predict_landmarks(img, (d["x"], d["y"], d["w"], d["h"]), ert)
            assert np.max(np.abs(lms[i][j] - xy)) <= 1e-9
            faces += 1
    assert faces > 0


def test_device_resident_frames_and_launch_count(ctx, pattern_model):
    import torch
    from pyoracle import ring_frames_np
    frames = ring_frames_np(4, 320, 240, seed=2)
    ctx.upload_detector(pattern_model)
    host = ctx.detect(frames)
    before = ctx.launch_count
    dev = ctx.detect(torch.from_numpy(frames).cuda())
    assert ctx.launch_count > before
    for a, b in zip(host, dev):
        assert np.array_equal(a, b)


# --------------------------------------------------------------- pipelined mode ----
def test_submit_collect_matches_sync(ctx, pattern_model):
    from pyoracle import random_ert, ring_frames_np
    ctx.upload_detector(pattern_model)
    ctx.upload_ert(random_ert(T=2, K=20, F=3, seed=9))
    a = ring_frames_np(5, 320, 240, seed=21)
    b = ring_frames_np(5, 320, 240, seed=22)
    sa = ctx.detect_landmarks(a, flat=True)
    sb = ctx.detect_landmarks(b, flat=True)
    import paper_2006_00816_b200 as bl
    assert bl.MAX_IN_FLIGHT >= 3
    ta = ctx.submit(a)
    tb = ctx.submit(b)
    tx = ctx.submit(a)
    extra = [ctx.submit(b if i % 2 else a) for i in range(bl.MAX_IN_FLIGHT - 3)]  # all slots busy
    with pytest.raises(RuntimeError):
        ctx.submit(a)  # one more would reuse a busy slot
    ra = ctx.collect(ta)
    for i, t in enumerate(extra):  # collected in submission order
        got = ctx.collect(t)
        want = sb if i % 2 else sa
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[2], want[2])
    tc = ctx.submit(b)
    rb = ctx.collect(tb)
    rx = ctx.collect(tx)
    rc = ctx.collect(tc)
    for got, want in [(ra, sa), (rb, sb), (rx, sa), (rc, sb)]:
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
        assert np.array_equal(got[2], want[2])
    with pytest.raises(RuntimeError):
        ctx.collect(ta)  # already collected


def test_face_capacity_overflow(ctx):
    """More kept detections than the device face capacity: collect reports it, the synchronous
    call grows the capacity and still returns every detection with landmarks."""
    import paper_2006_00816_b200 as bl
    from pyoracle import random_ert
    r = rng(78)
    model = {"weights": r.uniform(-1, 1, (5, 3100)) * 0.05, "biases": r.uniform(-1, 1, 5), "threshold": 0.3}
    img = np.floor(r.uniform(0, 256, (1, 240, 320))).astype(np.uint8)
    ctx.upload_detector(model)
    ctx.upload_ert(random_ert(T=1, K=4, F=2, seed=1))
    ctx.set_face_capacity(2)
    t = ctx.submit(img)
    with pytest.raises(bl.CapacityError):
        ctx.collect(t)
    dets, counts, lms = ctx.detect_landmarks(img, flat=True)
    assert len(dets) == counts.sum() > 2 and lms.shape[0] == len(dets)
    assert np.array_equal(dets, ctx.detect(img, flat=True)[0])
    ctx.set_face_capacity(64)
