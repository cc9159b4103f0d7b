"""The two classifier screens (tcgen05 implicit GEMM, CUDA-core fp32) against the oracle.

The screen only nominates candidates; the exact fp64 re-score decides.  So the contract is:
(1) every raw screen sum lies within the rigorous bound delta of the exact separable score
(detector.cpp:66-100) -- nothing the reference keeps can be screened out; (2) detections are
bit-identical to the oracle whichever screen runs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _features(r, ch, cw):
    # inside the feature range the cut assumes (compute_features output is in [0, 0.8486])
    f = r.uniform(0.0, 0.4, (ch, cw, 31))
    f[..., 27:] = r.uniform(0.0, 0.8486, (ch, cw, 4))
    f[r.uniform(size=(ch, cw)) < 0.1] = 0.0
    return f


@pytest.mark.parametrize("cw,ch,seed", [(66, 50, 1), (10, 10, 2), (15, 11, 3), (57, 41, 4), (161, 121, 5),
                                        (238, 133, 6)])
def test_tc_screen_within_bound(ctx, oracle, cw, ch, seed):
    r = np.random.default_rng(seed)
    model = {"weights": r.uniform(-1, 1, (5, 3100)) * r.uniform(0.01, 2.0, (5, 1)),
             "biases": r.uniform(-1, 1, 5), "threshold": 0.0}
    ctx.upload_detector(model)
    feat = _features(r, ch, cw)
    tc, delta = ctx.debug_screen_tc(feat)
    assert tc.shape == (5, ch - 9, cw - 9)
    for k in range(5):
        exact = oracle.score_separable(feat, model["weights"][k], 0.0)
        err = np.abs(tc[k].astype(np.float64) - exact)
        assert np.all(np.isfinite(tc[k]))
        assert err.max() <= delta[k], (k, err.max(), delta[k])
        # the bound is not vacuous: the fp16 operand error is well inside it
        assert err.max() < 0.5 * delta[k]


def test_tc_screen_wide_weight_range(ctx, oracle):
    """Weights spanning 1e-9 .. 1 in one filter and a filter of tiny weights: after the
    per-filter power-of-two scaling the smallest land in the fp16 subnormal range, which the
    bound covers with its absolute term."""
    r = np.random.default_rng(31)
    w = np.sign(r.uniform(-1, 1, (5, 3100))) * np.exp(r.uniform(np.log(1e-9), 0.0, (5, 3100)))
    w[3] *= 1e-7
    w[4] *= 3e4
    model = {"weights": w, "biases": r.uniform(-1, 1, 5), "threshold": 0.0}
    ctx.upload_detector(model)
    feat = _features(r, 30, 40)
    feat[..., 7] = r.uniform(0, 1e-6, (30, 40))  # features in the fp16 subnormal range too
    tc, delta = ctx.debug_screen_tc(feat)
    for k in range(5):
        exact = oracle.score_separable(feat, w[k], 0.0)
        err = np.abs(tc[k].astype(np.float64) - exact)
        assert err.max() <= delta[k], (k, err.max(), delta[k])


def test_tc_screen_zero_and_single_weight(ctx, oracle):
    feat = _features(np.random.default_rng(9), 20, 30)
    w = np.zeros((5, 3100))
    w[1, 5] = 1.0      # picks feature 5 of cell (0, 0) of the window
    w[2, 3099] = -2.0  # last weight: cell (9, 9), feature 30
    ctx.upload_detector({"weights": w, "biases": np.zeros(5), "threshold": 0.0})
    tc, delta = ctx.debug_screen_tc(feat)
    assert np.all(tc[0] == 0) and np.all(tc[3] == 0) and np.all(tc[4] == 0)
    assert np.max(np.abs(tc[1] - feat[:11, :21, 5])) <= delta[1]
    assert np.max(np.abs(tc[2] + 2.0 * feat[9:20, 9:30, 30])) <= delta[2]


def _detect_both(ctx, frames, model):
    ctx.upload_detector(model)
    out = {}
    for mode in ("tc", "fp32"):
        ctx.set_screen(mode)
        out[mode] = ctx.detect(frames)
    ctx.set_screen("tc")
    return out


def test_screens_agree_with_oracle_random_filters(ctx, oracle):
    r = np.random.default_rng(78)
    model = {"weights": r.uniform(-1, 1, (5, 3100)) * 0.05, "biases": r.uniform(-1, 1, 5), "threshold": 0.3}
    frames = np.floor(r.uniform(0, 256, (3, 240, 320))).astype(np.uint8)
    got = _detect_both(ctx, frames, model)
    for i in range(len(frames)):
        want = oracle.detect_faces(frames[i].astype(np.float64), model)
        assert len(want) > 20
        assert np.array_equal(got["tc"][i], want)
        assert np.array_equal(got["fp32"][i], want)


def test_screens_agree_with_oracle_pattern(ctx, oracle, pattern_model):
    from pyoracle import ring_frames_np
    frames = ring_frames_np(4, 640, 480, seed=11)
    got = _detect_both(ctx, frames, pattern_model)
    n = 0
    for i in range(len(frames)):
        want = oracle.detect_faces(frames[i].astype(np.float64), pattern_model)
        n += len(want)
        assert np.array_equal(got["tc"][i], want)
        assert np.array_equal(got["fp32"][i], want)
    assert n > 0


def test_screen_mode_validation(ctx):
    with pytest.raises(Exception):
        ctx.set_screen("bf16")


def test_screens_non_finite_weights(ctx, oracle, pattern_model):
    """A NaN or infinite weight makes that filter's scores NaN / +-inf in the reference; the
    screen then cannot bound its error (delta = inf, every anchor nominated) and the exact
    re-score decides exactly as the reference does."""
    from pyoracle import ring_frames_np
    m = {k: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v) for k, v in pattern_model.items()}
    m["weights"] = np.array(m["weights"], dtype=np.float64, copy=True)
    m["weights"][2, 17] = np.nan
    m["weights"][3, 1000] = np.inf
    frames = ring_frames_np(2, 320, 240, seed=12)
    got = _detect_both(ctx, frames, m)
    for i in range(len(frames)):
        want = oracle.detect_faces(frames[i].astype(np.float64), m)
        assert np.array_equal(got["tc"][i], want)
        assert np.array_equal(got["fp32"][i], want)
