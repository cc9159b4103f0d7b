"""TEST INFRASTRUCTURE ONLY -- ctypes faces over the two CPU checkers.

* ``Oracle()``     -> oracle/liboracle.so, the plain-C restatement (blink_oracle.c)
* ``Reference()``  -> oracle/_ref/libblinkline_ref.so, the UNMODIFIED reference
                      library (/root/reference/proj/src) behind oracle/ref_capi.cpp

Both expose the same numpy-level methods, so a test can run the same case
through either one.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module; the product package
never does.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

DET_DTYPE = np.dtype(
    [("x", "<i4"), ("y", "<i4"), ("w", "<i4"), ("h", "<i4"), ("score", "<f8"),
     ("scale_index", "<i4"), ("rotation_index", "<i4")], align=True)
assert DET_DTYPE.itemsize == 32

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


def ensure_built(ref: bool = False) -> None:
    """Build the oracle library (and optionally the reference) if missing."""
    target = os.path.join(HERE, "_ref", "libblinkline_ref.so") if ref else os.path.join(HERE, "liboracle.so")
    if os.path.exists(target):
        return
    if ref and not os.path.isdir("/root/reference/proj"):
        raise FileNotFoundError("oracle/_ref/libblinkline_ref.so missing and /root/reference absent")
    subprocess.run(["make", "-s", "-C", HERE] + (["ref"] if ref else []), check=True)


def reference_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libblinkline_ref.so")) or os.path.isdir("/root/reference/proj")


class _Base:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        L = self.lib
        p = self.prefix
        self._f = lambda name: getattr(L, p + name)
        sigs = {
            "build_pyramid": (C.c_int, [_dp, C.c_int, C.c_int, C.c_int, _dp, C.c_size_t, _ip, _dp, C.c_int]),
            "downscale_bilinear": (C.c_int, [_dp, C.c_int, C.c_int, _dp]),
            "compute_gradients": (C.c_int, [_dp, C.c_int, C.c_int, _u8p, _dp]),
            "histogramize": (C.c_int, [_u8p, _dp, C.c_int, C.c_int, _dp]),
            "cell_energy": (C.c_int, [_dp, C.c_int, C.c_int, _dp]),
            "compute_features": (C.c_int, [_dp, _dp, C.c_int, C.c_int, _dp]),
            "extract_features": (C.c_int, [_dp, C.c_int, C.c_int, _dp]),
            "score_dense": (C.c_int, [_dp, C.c_int, C.c_int, _dp, C.c_double, _dp]),
            "score_separable": (C.c_int, [_dp, C.c_int, C.c_int, _dp, C.c_double, _dp]),
            "threshold_detections": (C.c_int, [_dp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                               C.c_int, C.c_int, C.c_int, _vp, C.c_int]),
            "nms": (C.c_int, [_vp, C.c_int, C.c_double, _vp]),
            "iou": (C.c_double, [C.c_int] * 8),
            "eligible_scales": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                          C.c_int, _ip]),
            "similarity_transform": (C.c_int, [_dp, _dp, C.c_int, _dp]),
            "last_error": (C.c_char_p, []),
        }
        for name, (res, args) in sigs.items():
            fn = self._f(name)
            fn.restype = res
            fn.argtypes = args

    def _check(self, rc):
        if rc < 0:
            raise ValueError(self._f("last_error")().decode())
        return rc

    # ---------------------------------------------------------------- image
    def build_pyramid(self, img, window=80):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        dims = np.zeros(128, np.int32)
        scales = np.zeros(64, np.float64)
        n = self._check(self._f("build_pyramid")(_ptr(img), w, h, window, None, 0, _ptr(dims, _ip), _ptr(scales), 64))
        total = int(sum(int(dims[2 * k]) * int(dims[2 * k + 1]) for k in range(n)))
        out = np.zeros(total, np.float64)
        self._check(self._f("build_pyramid")(_ptr(img), w, h, window, _ptr(out), total, _ptr(dims, _ip), _ptr(scales), 64))
        levels, off = [], 0
        for k in range(n):
            lw, lh = int(dims[2 * k]), int(dims[2 * k + 1])
            levels.append(out[off:off + lw * lh].reshape(lh, lw))
            off += lw * lh
        return levels, scales[:n].copy()

    def downscale_bilinear(self, img):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        out = np.zeros((h * 5 // 6, w * 5 // 6), np.float64)
        self._check(self._f("downscale_bilinear")(_ptr(img), w, h, _ptr(out)))
        return out

    # ------------------------------------------------------------------ hog
    def compute_gradients(self, img):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        ori = np.zeros((h, w), np.uint8)
        mag = np.zeros((h, w), np.float64)
        self._check(self._f("compute_gradients")(_ptr(img), w, h, _ptr(ori, _u8p), _ptr(mag)))
        return ori, mag

    def histogramize(self, ori, mag):
        ori = np.ascontiguousarray(ori, dtype=np.uint8)
        mag = np.ascontiguousarray(mag, dtype=np.float64)
        h, w = mag.shape
        bins = np.zeros((h // 8, w // 8, 18), np.float64)
        self._check(self._f("histogramize")(_ptr(ori, _u8p), _ptr(mag), w, h, _ptr(bins)))
        return bins

    def cell_energy(self, bins):
        bins = np.ascontiguousarray(bins, dtype=np.float64)
        ch, cw = bins.shape[:2]
        e = np.zeros((ch, cw), np.float64)
        self._check(self._f("cell_energy")(_ptr(bins), cw, ch, _ptr(e)))
        return e

    def compute_features(self, bins, energy):
        bins = np.ascontiguousarray(bins, dtype=np.float64)
        energy = np.ascontiguousarray(energy, dtype=np.float64)
        ch, cw = bins.shape[:2]
        f = np.zeros((ch, cw, 31), np.float64)
        self._check(self._f("compute_features")(_ptr(bins), _ptr(energy), cw, ch, _ptr(f)))
        return f

    def extract_features(self, img):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        f = np.zeros((h // 8, w // 8, 31), np.float64)
        self._check(self._f("extract_features")(_ptr(img), w, h, _ptr(f)))
        return f

    # ------------------------------------------------------------- detector
    def _score(self, name, feat, weights, bias):
        feat = np.ascontiguousarray(feat, dtype=np.float64)
        weights = np.ascontiguousarray(weights, dtype=np.float64).reshape(3100)
        ch, cw = feat.shape[:2]
        out = np.zeros((max(ch - 9, 0), max(cw - 9, 0)), np.float64)
        self._check(self._f(name)(_ptr(feat), cw, ch, _ptr(weights), float(bias), _ptr(out)))
        return out

    def score_dense(self, feat, weights, bias):
        return self._score("score_dense", feat, weights, bias)

    def score_separable(self, feat, weights, bias):
        return self._score("score_separable", feat, weights, bias)

    def threshold_detections(self, scores, thr, scale_index, rotation_index, window_cells=10, cell_px=8,
                             scale_num=5, scale_den=6):
        scores = np.ascontiguousarray(scores, dtype=np.float64)
        sh, sw = scores.shape
        out = np.zeros(sw * sh + 1, DET_DTYPE)
        n = self._check(self._f("threshold_detections")(_ptr(scores), sw, sh, float(thr), window_cells, cell_px,
                                                        scale_num, scale_den, scale_index, rotation_index,
                                                        out.ctypes.data, len(out)))
        return out[:n].copy()

    def nms(self, dets, iou_thr=0.5):
        dets = np.ascontiguousarray(dets, dtype=DET_DTYPE)
        out = np.zeros(len(dets) + 1, DET_DTYPE)
        n = self._check(self._f("nms")(dets.ctypes.data, len(dets), float(iou_thr), out.ctypes.data))
        return out[:n].copy()

    def iou(self, a, b):
        return self._f("iou")(*[int(v) for v in a], *[int(v) for v in b])

    def eligible_scales(self, w, h, n_levels, window_cells=10, cell_px=8, scale_num=5, scale_den=6,
                        min_face_ratio=0.2):
        out = np.zeros(max(n_levels, 1), np.int32)
        n = self._check(self._f("eligible_scales")(w, h, window_cells, cell_px, scale_num, scale_den,
                                                   float(min_face_ratio), n_levels, _ptr(out, _ip)))
        return [int(v) for v in out[:n]]

    # ------------------------------------------------------------------ ert
    def similarity_transform(self, frm, to):
        frm = np.ascontiguousarray(frm, dtype=np.float64)
        to = np.ascontiguousarray(to, dtype=np.float64)
        out = np.zeros(4, np.float64)
        self._check(self._f("similarity_transform")(_ptr(frm), _ptr(to), len(frm), _ptr(out)))
        return out


class Oracle(_Base):
    """The plain-C restatement (oracle/blink_oracle.c)."""

    prefix = "orc_"

    class _Det(C.Structure):
        _fields_ = [("weights", _dp), ("biases", _dp), ("threshold", C.c_double), ("window_cells", C.c_int),
                    ("cell_px", C.c_int), ("scale_num", C.c_int), ("scale_den", C.c_int),
                    ("min_face_ratio", C.c_double)]

    class _Ert(C.Structure):
        _fields_ = [("L", C.c_int), ("T", C.c_int), ("K", C.c_int), ("F", C.c_int), ("shrinkage", C.c_double),
                    ("mean_xy", _dp), ("anchors", _ip), ("split_params", _dp), ("leaves", _dp)]

    def __init__(self):
        ensure_built(False)
        super().__init__(os.path.join(HERE, "liboracle.so"))
        L = self.lib
        L.orc_detect_faces.restype = C.c_int
        L.orc_detect_faces.argtypes = [_dp, C.c_int, C.c_int, C.POINTER(self._Det), _vp, C.c_int]
        L.orc_predict_landmarks.restype = C.c_int
        L.orc_predict_landmarks.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.POINTER(self._Ert), _dp, _u8p, C.POINTER(C.c_uint64)]
        L.orc_sample_intensity.restype = C.c_double
        L.orc_sample_intensity.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp,
                                           C.c_int, C.c_double, C.c_double]
        L.orc_direction_table.restype = None
        L.orc_direction_table.argtypes = [_dp, _dp]

    def direction_table(self):
        ux = np.zeros(18)
        uy = np.zeros(18)
        self.lib.orc_direction_table(_ptr(ux), _ptr(uy))
        return ux, uy

    def detect_faces(self, img, model):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        wts = np.ascontiguousarray(model["weights"], dtype=np.float64).reshape(5 * 3100)
        bs = np.ascontiguousarray(model["biases"], dtype=np.float64)
        d = self._Det(_ptr(wts), _ptr(bs), float(model["threshold"]), model.get("window_cells", 10),
                      model.get("cell_px", 8), model.get("scale_num", 5), model.get("scale_den", 6),
                      float(model.get("min_face_ratio", 0.2)))
        cap = 1 << 16
        out = np.zeros(cap, DET_DTYPE)
        n = self._check(self.lib.orc_detect_faces(_ptr(img), w, h, C.byref(d), out.ctypes.data, cap))
        return out[:min(n, cap)].copy()

    def predict_landmarks(self, img, box, ert):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        keep = [np.ascontiguousarray(ert["mean_xy"], dtype=np.float64),
                np.ascontiguousarray(ert["anchors"], dtype=np.int32),
                np.ascontiguousarray(ert["split_params"], dtype=np.float64),
                np.ascontiguousarray(ert["leaves"], dtype=np.float64)]
        m = self._Ert(ert["L"], ert["T"], ert["K"], ert["F"], float(ert["shrinkage"]), _ptr(keep[0]),
                      _ptr(keep[1], _ip), _ptr(keep[2]), _ptr(keep[3]))
        xy = np.zeros((ert["L"], 2), np.float64)
        leaf = np.zeros(ert["T"] * ert["K"], np.uint8)
        ev = C.c_uint64(0)
        self._check(self.lib.orc_predict_landmarks(_ptr(img), w, h, *[int(v) for v in box], C.byref(m), _ptr(xy),
                                                   _ptr(leaf, _u8p), C.byref(ev)))
        return xy, leaf, int(ev.value)

    def sample_intensity(self, img, box, shape_xy, tform4, anchor, ox, oy):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        s = np.ascontiguousarray(shape_xy, dtype=np.float64)
        t = np.ascontiguousarray(tform4, dtype=np.float64)
        return self.lib.orc_sample_intensity(_ptr(img), w, h, *[int(v) for v in box], _ptr(s), _ptr(t), anchor,
                                             float(ox), float(oy))


class Reference(_Base):
    """The unmodified reference library (oracle/_ref/libblinkline_ref.so)."""

    def run(self, frames_dir, det, ert, fps, pipelined=False, batch_size=16, det_cap=100000):
        """The reference's run() (pipeline.cpp:396-404) -> the same dict as Context.run, or
        raises RuntimeError with the reference's message (first ingest/run error)."""
        L = self.lib
        L.ref_run.restype = C.c_int
        L.ref_run.argtypes = [C.c_char_p, _dp, _dp, C.c_double, _vp, C.c_double, C.c_int, C.c_int, _ip, _ip, _ip,
                              _vp, _dp, _dp, _vp, C.c_int, _ip, _dp]
        w = np.ascontiguousarray(det["weights"], np.float64).reshape(5, 3100)
        b = np.ascontiguousarray(det["biases"], np.float64)
        h = self.ert_handle(ert)
        try:
            nmax = 4096  # frames per test directory
            n = np.zeros(1, np.int32)
            nd = np.zeros(nmax, np.int32)
            ff = np.zeros(nmax, np.int32)
            faces = np.zeros(nmax, DET_DTYPE)
            lm_buf = np.full((nmax, int(ert["L"]), 2), np.nan)
            ears = np.zeros((nmax, 4))
            dets = np.zeros(det_cap, DET_DTYPE)
            tot = np.zeros(1, np.int32)
            base = np.zeros(2)
            rc = L.ref_run(os.fsencode(frames_dir), _ptr(w), _ptr(b), float(det["threshold"]), h, float(fps),
                           int(pipelined), int(batch_size), _ptr(n, _ip), _ptr(nd, _ip), _ptr(ff, _ip),
                           faces.ctypes.data, _ptr(lm_buf), _ptr(ears), dets.ctypes.data, det_cap, _ptr(tot, _ip),
                           _ptr(base))
            if rc:
                raise RuntimeError(self.lib.ref_last_error().decode())
            k = int(n[0])
            return {"n_detections": nd[:k], "face_found": ff[:k], "faces": faces[:k], "landmarks": lm_buf[:k],
                    "ears": ears[:k], "detections": dets[:int(tot[0])], "baselines": base}
        finally:
            pass  # h is owned by the ert_handle cache (destroying it here left a dangling entry)

    prefix = "ref_"

    def __init__(self):
        ensure_built(True)
        super().__init__(os.path.join(HERE, "_ref", "libblinkline_ref.so"))
        L = self.lib
        L.ref_detect_faces.restype = C.c_int
        L.ref_detect_faces.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_double, _vp, C.c_int]
        L.ref_ert_create.restype = _vp
        L.ref_ert_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _dp, _ip, _dp, _dp]
        L.ref_ert_destroy.restype = None
        L.ref_ert_destroy.argtypes = [_vp]
        L.ref_predict_landmarks.restype = C.c_int
        L.ref_predict_landmarks.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _dp,
                                            C.POINTER(C.c_uint64)]
        L.ref_ert_leaf_indices.restype = C.c_int
        L.ref_ert_leaf_indices.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _u8p,
                                           _dp]
        L.ref_sample_intensity.restype = C.c_double
        L.ref_sample_intensity.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_int,
                                           _dp, C.c_int, C.c_double, C.c_double]
        L.ref_pattern_detector.restype = C.c_int
        L.ref_pattern_detector.argtypes = [_dp, _dp, _dp]
        L.ref_face68_mean_shape.restype = None
        L.ref_face68_mean_shape.argtypes = [_dp]
        L.ref_random_image.restype = None
        L.ref_random_image.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, _dp]
        L.ref_ring_frame.restype = None
        L.ref_ring_frame.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_int,
                                     _dp]
        L.ref_run_batch_u8.restype = C.c_longlong
        L.ref_run_batch_u8.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double, _vp, C.c_int, _ip,
                                       _dp]
        L.ref_landmarks_batch_u8.restype = C.c_int
        L.ref_landmarks_batch_u8.argtypes = [_u8p, C.c_int, C.c_int, _ip, _ip, C.c_int, _vp, C.c_int, _dp]
        self._erts = {}

    def detect_faces(self, img, model):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        wts = np.ascontiguousarray(model["weights"], dtype=np.float64).reshape(5 * 3100)
        bs = np.ascontiguousarray(model["biases"], dtype=np.float64)
        cap = 1 << 16
        out = np.zeros(cap, DET_DTYPE)
        n = self._check(self.lib.ref_detect_faces(_ptr(img), w, h, _ptr(wts), _ptr(bs), float(model["threshold"]),
                                                  model.get("window_cells", 10), model.get("cell_px", 8),
                                                  model.get("scale_num", 5), model.get("scale_den", 6),
                                                  float(model.get("min_face_ratio", 0.2)), out.ctypes.data, cap))
        return out[:min(n, cap)].copy()

    def ert_handle(self, ert):
        key = id(ert)
        if key not in self._erts:
            keep = [np.ascontiguousarray(ert["mean_xy"], dtype=np.float64),
                    np.ascontiguousarray(ert["anchors"], dtype=np.int32),
                    np.ascontiguousarray(ert["split_params"], dtype=np.float64),
                    np.ascontiguousarray(ert["leaves"], dtype=np.float64)]
            h = self.lib.ref_ert_create(ert["L"], ert["T"], ert["K"], ert["F"], float(ert["shrinkage"]),
                                        _ptr(keep[0]), _ptr(keep[1], _ip), _ptr(keep[2]), _ptr(keep[3]))
            if not h:
                raise ValueError(self.lib.ref_last_error().decode())
            self._erts[key] = (h, ert)
        return self._erts[key][0]

    def predict_landmarks(self, img, box, ert):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        hd = self.ert_handle(ert)
        xy = np.zeros((ert["L"], 2), np.float64)
        ev = C.c_uint64(0)
        self._check(self.lib.ref_predict_landmarks(_ptr(img), w, h, *[int(v) for v in box], hd, _ptr(xy),
                                                   C.byref(ev)))
        leaf = np.zeros(ert["T"] * ert["K"], np.uint8)
        xy2 = np.zeros((ert["L"], 2), np.float64)
        self._check(self.lib.ref_ert_leaf_indices(_ptr(img), w, h, *[int(v) for v in box], hd, _ptr(leaf, _u8p),
                                                  _ptr(xy2)))
        if not np.array_equal(xy, xy2):
            raise AssertionError("leaf-index restatement diverged from predict_landmarks")
        return xy, leaf, int(ev.value)

    def sample_intensity(self, img, box, shape_xy, tform4, anchor, ox, oy):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        s = np.ascontiguousarray(shape_xy, dtype=np.float64)
        t = np.ascontiguousarray(tform4, dtype=np.float64)
        return self.lib.ref_sample_intensity(_ptr(img), w, h, *[int(v) for v in box], _ptr(s), len(s), _ptr(t),
                                             anchor, float(ox), float(oy))

    # fixtures from the reference's own generators (tests/helpers.cpp)
    def pattern_detector(self):
        w = np.zeros(3100)
        b = C.c_double(0)
        t = C.c_double(0)
        self._check(self.lib.ref_pattern_detector(_ptr(w), C.byref(b), C.byref(t)))
        return {"weights": np.tile(w, (5, 1)), "biases": np.full(5, b.value), "threshold": t.value}

    def face68_mean_shape(self):
        xy = np.zeros((68, 2))
        self.lib.ref_face68_mean_shape(_ptr(xy))
        return xy

    def random_image(self, w, h, seed, lo=0.0, hi=255.0):
        out = np.zeros((h, w))
        self.lib.ref_random_image(w, h, seed, lo, hi, _ptr(out))
        return out

    def ring_frame(self, w, h, seed, cx, cy, size, round_u8=True):
        out = np.zeros((h, w))
        self.lib.ref_ring_frame(w, h, seed, cx, cy, size, int(round_u8), _ptr(out))
        return out

    def run_batch_u8(self, frames, model, ert, threads):
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        n, h, w = frames.shape
        wts = np.ascontiguousarray(model["weights"], dtype=np.float64).reshape(5 * 3100)
        bs = np.ascontiguousarray(model["biases"], dtype=np.float64)
        counts = np.zeros(n, np.int32)
        cs = C.c_double(0)
        hd = self.ert_handle(ert) if ert is not None else None
        faces = self.lib.ref_run_batch_u8(_ptr(frames, _u8p), n, w, h, _ptr(wts), _ptr(bs), float(model["threshold"]),
                                          hd, threads, _ptr(counts, _ip), C.byref(cs))
        if faces < 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return int(faces), counts, cs.value

    def landmarks_batch_u8(self, frames, frame_of_box, boxes, ert, threads, want_xy=False):
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        n, h, w = frames.shape
        fob = np.ascontiguousarray(frame_of_box, dtype=np.int32)
        bx = np.ascontiguousarray(boxes, dtype=np.int32)
        out = np.zeros((len(bx), ert["L"], 2)) if want_xy else None
        self._check(self.lib.ref_landmarks_batch_u8(_ptr(frames, _u8p), w, h, _ptr(fob, _ip), _ptr(bx, _ip), len(bx),
                                                    self.ert_handle(ert), threads, _ptr(out) if want_xy else None))
        return out


# Synthetic-input generators live with the product (bench.py uses them without importing
# oracle/); re-exported here for the tests.  Loaded by file path: importing the package would
# map the GPU library into a CPU-checker process (the --impl reference arm must not).
def _load_synthetic():
    import importlib.util
    path = os.path.join(os.path.dirname(HERE), "paper_2006_00816_b200", "synthetic.py")
    spec = importlib.util.spec_from_file_location("_bl_synthetic", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


_syn = _load_synthetic()
face68_mean_shape_np, random_ert, ring_frames_np = _syn.face68_mean_shape_np, _syn.random_ert, _syn.ring_frames_np
