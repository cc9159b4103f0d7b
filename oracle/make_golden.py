"""TEST INFRASTRUCTURE ONLY -- writes tests/golden/*.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference or a built oracle/_ref):

    python oracle/make_golden.py

Every fixture is produced by calling the reference library (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile) on inputs made by the reference's own seeded
generators (tests/helpers.cpp: random_image, add_noise, draw_pattern, pattern_detector,
face68_mean_shape).  The committed .npz files then pin the C oracle
(tests/test_oracle_golden.py) and travel to the GPU box, where /root/reference does not
exist.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from pyoracle import DET_DTYPE, Reference, random_ert  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")



def main():
    os.makedirs(OUT, exist_ok=True)
    r = Reference()

    # --- pattern detector (helpers.cpp:116-191): 5 identical filters, threshold 0.
    pd = r.pattern_detector()
    np.savez_compressed(os.path.join(OUT, "pattern_detector.npz"), weights=pd["weights"][0], bias=pd["biases"][0],
                        threshold=pd["threshold"])

    # --- pyramid: ring frame 200x150 (noise seed 1000) and 640x480 dims only.
    f = r.ring_frame(200, 150, 1000, 100.0, 75.0, 80.0)
    levels, scales = r.build_pyramid(f, 80)
    np.savez_compressed(os.path.join(OUT, "pyramid.npz"), image=f, scales=scales,
                        **{f"level{k}": lv for k, lv in enumerate(levels)})

    # --- gradient/histogram/energy/features on the reference test images.
    hog = {}
    for name, img in [
        ("rand64", r.random_image(64, 64, 102)),        # acceptance C2 generator
        ("rand16", r.random_image(16, 16, 77)),         # test_hog.cpp:110-123
        ("rand40x32", r.random_image(40, 32, 24)),      # test_hog.cpp:334-340
        ("ring", r.ring_frame(96, 80, 7, 48.0, 40.0, 60.0)),
        ("tie_up", np.tile((10.0 * np.arange(24))[:, None], (1, 24))),         # I=10y: gx=0, gy>0
        ("tie_down", np.tile((240.0 - 10.0 * np.arange(24))[:, None], (1, 24))),  # gx=0, gy<0
        ("ramp", np.tile(np.arange(8.0)[None, :], (8, 1))),                     # test_hog.cpp:81-92
    ]:
        ori, mag = r.compute_gradients(img)
        bins = r.histogramize(ori, mag)
        en = r.cell_energy(bins) if bins.size else np.zeros(bins.shape[:2])
        feat = r.compute_features(bins, en) if bins.size else np.zeros(bins.shape[:2] + (31,))
        hog.update({f"{name}_img": img, f"{name}_ori": ori, f"{name}_mag": mag, f"{name}_bins": bins,
                    f"{name}_energy": en, f"{name}_feat": feat})
    np.savez_compressed(os.path.join(OUT, "hog.npz"), **hog)

    # --- classifier: random features/filter (detector test generators use urand(-0.2,0.4),
    #     urand(-1,1)); here numpy-seeded, evaluated by the reference scorers.
    rng = np.random.default_rng(31)
    feat = rng.uniform(-0.2, 0.4, (12, 16, 31))
    wts = rng.uniform(-1, 1, 3100)
    bias = float(rng.uniform(-1, 1))
    dense = r.score_dense(feat, wts, bias)
    sep = r.score_separable(feat, wts, bias)
    thr_dets = r.threshold_detections(sep, 0.5, 2, 3)
    np.savez_compressed(os.path.join(OUT, "classifier.npz"), feat=feat, weights=wts, bias=bias, dense=dense,
                        separable=sep, thr_dets=thr_dets)

    # --- NMS on a random set (test_detector.cpp:189-208 shape).
    rng = np.random.default_rng(33)
    dets = np.zeros(200, DET_DTYPE)
    dets["x"] = rng.integers(0, 100, 200)
    dets["y"] = rng.integers(0, 100, 200)
    dets["w"] = rng.integers(20, 60, 200)
    dets["h"] = dets["w"]
    dets["score"] = rng.uniform(0, 1, 200)
    dets["scale_index"] = rng.integers(0, 4, 200)
    dets["rotation_index"] = rng.integers(0, 5, 200)
    np.savez_compressed(os.path.join(OUT, "nms.npz"), dets=dets, kept=r.nms(dets, 0.5))

    # --- end-to-end detection with the pattern detector.
    det = {}
    cases = [
        ("c1", r.ring_frame(640, 480, 1000, 300.0, 250.0, 160.0), True),     # acceptance C5-like, u8
        ("planted", r.ring_frame(640, 480, 36, 300.0, 250.0, 160.0, round_u8=False), False),  # test_detector.cpp:265-277
        ("qvga", r.ring_frame(320, 240, 1001, 150.0, 130.0, 110.0), True),   # C2 geometry, all levels eligible
        ("blank", np.full((240, 320), 20.0), True),
        ("small", np.full((60, 60), 20.0), True),
    ]
    for name, img, integral in cases:
        d = r.detect_faces(img, pd)
        det[f"{name}_img"] = img.astype(np.uint8) if integral else img
        det[f"{name}_dets"] = d
    # random-init filters: many raw detections, stresses threshold + NMS
    rng = np.random.default_rng(5)
    rnd = {"weights": rng.uniform(-1, 1, (5, 3100)) * 0.05, "biases": rng.uniform(-1, 1, 5), "threshold": 0.7}
    img = det["qvga_img"].astype(np.float64)
    det["random_weights"] = rnd["weights"]
    det["random_biases"] = rnd["biases"]
    det["random_threshold"] = rnd["threshold"]
    det["random_dets"] = r.detect_faces(img, rnd)
    np.savez_compressed(os.path.join(OUT, "detect.npz"), **det)

    # --- ERT: small random cascade over the face68 mean shape, random-texture frame.
    mean = r.face68_mean_shape()
    ert = random_ert(L=68, T=3, K=10, F=4, seed=11, mean_xy=mean)
    img = np.floor(r.random_image(160, 120, 43) + 0.5)
    boxes = np.array([[20, 10, 80, 80], [0, 0, 160, 120], [90, 50, 60, 60], [-10, -5, 50, 50]], np.int32)
    xs, leaves, evals = [], [], []
    for b in boxes:
        xy, lf, ev = r.predict_landmarks(img, tuple(b), ert)
        xs.append(xy)
        leaves.append(lf)
        evals.append(ev)
    np.savez_compressed(os.path.join(OUT, "ert.npz"), image=img.astype(np.uint8), boxes=boxes, mean_xy=mean,
                        anchors=ert["anchors"], split_params=ert["split_params"], leaves=ert["leaves"],
                        T=ert["T"], K=ert["K"], F=ert["F"], L=ert["L"], shrinkage=ert["shrinkage"],
                        landmarks=np.array(xs), leaf_idx=np.array(leaves), evals=np.array(evals))

    # --- similarity transform known answers + sampling.
    rng = np.random.default_rng(41)
    frm = rng.uniform(0, 1, (7, 2))
    c = frm.mean(axis=0)
    to = np.stack([c[0] - (frm[:, 1] - c[1]), c[1] + (frm[:, 0] - c[0])], axis=1)
    np.savez_compressed(os.path.join(OUT, "similarity.npz"), frm=frm, to=to, tform=r.similarity_transform(frm, to),
                        face_tform=r.similarity_transform(mean * 1.1 + 0.01, mean))
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
