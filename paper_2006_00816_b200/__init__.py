"""paper_2006_00816_b200 -- B200-native face detection + 68-landmark hot path.

Python face of the C-ABI in include/blinkline_b200.h (ctypes; the shared library is built
in-tree by ``make`` / ``__graft_entry__.build()``).  There is no CPU fallback: importing the
package loads ``libblinkline_b200.so`` and fails loudly if it is missing; every call runs on
the GPU.

The functions mirror the reference library's hot-path API (proj/include/blinkline) with the
same names and argument meaning -- ``build_pyramid``, ``compute_gradients``,
``histogramize``, ``cell_energy``, ``compute_features``, ``extract_features``,
``score_separable``, ``nms``, ``detect_faces``, ``predict_landmarks`` -- plus the batched
entry points the device path is built for (``Context.detect``, ``Context.landmarks``,
``Context.detect_landmarks``).  Precondition failures raise ``ValueError`` (the reference's
std::invalid_argument), model problems ``ModelError``, device failures ``RuntimeError``.

Models are plain dicts:
  detector: {"weights": (5, 3100) float64, "biases": (5,), "threshold": float,
             optional "window_cells", "cell_px", "scale_num", "scale_den", "min_face_ratio"}
  ert:      {"L", "T", "K", "F", "shrinkage", "mean_xy": (L, 2), "anchors": (T*K*S, 2) int32,
             "split_params": (T*K*S, 5), "leaves": (T*K*2^F, L, 2)}
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

__all__ = [
    "Context", "MultiContext", "ModelError", "DET_DTYPE", "library_path", "lib",
    "build_pyramid", "downscale_bilinear", "compute_gradients", "histogramize", "cell_energy",
    "compute_features", "extract_features", "score_separable", "score_dense", "nms",
    "orientation_bins", "detect_faces", "predict_landmarks", "default_context",
    "read_pgm", "write_pgm", "read_detector_json", "write_detector_json", "read_ert_json", "write_ert_json",
    "IoError", "ingest", "FRAME_DTYPE",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# BL_LIBRARY selects an alternative build of the same library (kernel-variant experiments,
# tools/build_variant.sh); there is no CPU fallback either way.
library_path = os.environ.get("BL_LIBRARY") or os.path.join(_HERE, "libblinkline_b200.so")

if not os.path.exists(library_path):
    raise ImportError(
        f"{library_path} is missing: build the CUDA extension first (make, or __graft_entry__.build()). "
        "There is no CPU fallback.")

lib = C.CDLL(library_path, mode=C.RTLD_GLOBAL)

DET_DTYPE = np.dtype([("x", "<i4"), ("y", "<i4"), ("w", "<i4"), ("h", "<i4"), ("score", "<f8"),
                      ("scale_index", "<i4"), ("rotation_index", "<i4")], align=True)
assert DET_DTYPE.itemsize == 32

BL_OK, BL_ERR_INVALID, BL_ERR_MODEL, BL_ERR_CUDA, BL_ERR_CAPACITY, BL_ERR_STATE, BL_ERR_IO = range(7)
BL_PIX_U8, BL_PIX_F64 = 0, 1
SCREEN_TCGEN05, SCREEN_FP32 = 0, 1
MAX_IN_FLIGHT = 4  # BL_MAX_IN_FLIGHT
STAGES = ["h2d", "pyramid", "gradhist", "features", "screen", "rescore", "nms", "ert", "d2h"]


FRAME_DTYPE = np.dtype([("frame_index", "<i4"), ("n_detections", "<i4"), ("face_found", "<i4"), ("pad", "<i4"),
                        ("face", DET_DTYPE), ("ear_left", "<f8"), ("ear_right", "<f8"), ("closure_left", "<f8"),
                        ("closure_right", "<f8"), ("t", "<f8"), ("decode_ms", "<f8"), ("detect_ms", "<f8"),
                        ("landmark_ms", "<f8")], align=True)


class ModelError(RuntimeError):
    """The reference's blinkline::model_error."""


class IoError(OSError):
    """The reference's blinkline::io_error (unreadable file, malformed PGM)."""


class CapacityError(RuntimeError):
    def __init__(self, msg, total=None):
        super().__init__(msg)
        self.total = total


_vp, _i32, _i64, _u64, _dbl, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
_P = C.POINTER
_SIGS = {
    "bl_abi_version": (C.c_int, []),
    "bl_plan_geometry": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dbl, _vp, _vp, _vp, _vp,
                                   C.c_int, _P(C.c_int), _P(C.c_int)]),
    "bl_last_error": (C.c_char_p, []),
    "bl_device_count": (C.c_int, [_P(C.c_int)]),
    "bl_ctx_create": (C.c_int, [C.c_int, _P(_vp)]),
    "bl_ctx_destroy": (None, [_vp]),
    "bl_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "bl_ctx_synchronize": (C.c_int, [_vp]),
    "bl_ctx_launch_count": (C.c_int, [_vp, _P(_u64)]),
    "bl_ctx_enable_stage_timing": (C.c_int, [_vp, C.c_int]),
    "bl_ctx_stage_times": (C.c_int, [_vp, _P(C.c_float), _P(C.c_int)]),
    "bl_ctx_enable_graphs": (C.c_int, [_vp, C.c_int]),
    "bl_ctx_set_screen": (C.c_int, [_vp, C.c_int]),
    "bl_detector_upload": (C.c_int, [_vp, _vp, _vp, _dbl, C.c_int, C.c_int, C.c_int, C.c_int, _dbl]),
    "bl_ert_upload": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _dbl, _vp, _vp, _vp, _vp]),
    "bl_detect": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _sz, _sz, _vp, _i64, _vp, _P(_i64)]),
    "bl_submit": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _sz, _sz, C.c_int, _P(_u64)]),
    "bl_collect": (C.c_int, [_vp, _u64, _vp, _i64, _vp, _P(_i64), _vp]),
    "bl_ctx_set_face_capacity": (C.c_int, [_vp, C.c_int]),
    "bl_ctx_get_face_capacity": (C.c_int, [_vp, _P(C.c_int)]),
    "bl_host_alloc": (C.c_int, [_sz, _P(_vp)]),
    "bl_host_free": (None, [_vp]),
    "bl_multi_create": (C.c_int, [_vp, C.c_int, _P(_vp)]),
    "bl_multi_destroy": (None, [_vp]),
    "bl_multi_size": (C.c_int, [_vp, _P(C.c_int)]),
    "bl_multi_context": (C.c_int, [_vp, C.c_int, _P(_vp)]),
    "bl_multi_set_batch_pixels": (C.c_int, [_vp, _i64]),
    "bl_multi_detector_upload": (C.c_int, [_vp, _vp, _vp, _dbl, C.c_int, C.c_int, C.c_int, C.c_int, _dbl]),
    "bl_multi_ert_upload": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _dbl, _vp, _vp, _vp, _vp]),
    "bl_multi_detect_landmarks": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _sz, _sz, _vp, _i64,
                                            _vp, _P(_i64), _vp, _vp]),
    "bl_landmarks": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _sz, _sz, _vp, _vp, _i64, _vp, _vp]),
    "bl_detect_landmarks": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _sz, _sz, _vp, _i64, _vp,
                                      _P(_i64), _vp]),
    "bl_build_pyramid": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _sz, _vp, _vp, C.c_int,
                                   _P(C.c_int)]),
    "bl_downscale_bilinear": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "bl_compute_gradients": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp]),
    "bl_histogramize": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, _vp]),
    "bl_cell_energy": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "bl_compute_features": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, _vp]),
    "bl_extract_features": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp]),
    "bl_score_window": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _dbl, _vp]),
    "bl_score_window_dense": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _dbl, _vp]),
    "bl_ctx_share_models": (C.c_int, [_vp, _vp, C.c_int]),
    "bl_nms": (C.c_int, [_vp, _vp, _i64, _dbl, _vp, _P(_i64)]),
    "bl_orientation_bins": (C.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "bl_debug_sqrt": (C.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "bl_debug_screen_tc": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp]),
    "bl_read_pgm": (C.c_int, [C.c_char_p, _P(C.c_int), _P(C.c_int), _vp, _sz]),
    "bl_ctx_model_info": (C.c_int, [_vp, _P(C.c_int)]),
    "bl_ingest": (C.c_int, [C.c_char_p, _P(C.c_int), _P(C.c_int), _P(C.c_int)]),
    "bl_run": (C.c_int, [_vp, C.c_char_p, C.c_double, C.c_int, _vp, _i64, _vp, _i64, _P(_i64), _vp, _vp]),
    "bl_write_pgm": (C.c_int, [C.c_char_p, _vp, C.c_int, C.c_int]),
    "bl_read_detector_json": (C.c_int, [C.c_char_p, _vp, _vp, _P(C.c_double), _P(C.c_int), _P(C.c_int),
                                        _P(C.c_int), _P(C.c_int), _P(C.c_double)]),
    "bl_write_detector_json": (C.c_int, [C.c_char_p, _vp, _vp, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_double]),
    "bl_ert_file_open": (C.c_int, [C.c_char_p, _P(_vp), _P(C.c_int), _P(C.c_int), _P(C.c_int), _P(C.c_int),
                                   _P(C.c_double)]),
    "bl_ert_file_copy": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "bl_ert_file_upload": (C.c_int, [_vp, _vp]),
    "bl_ert_file_close": (None, [_vp]),
    "bl_write_ert_json": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _vp, _vp, _vp,
                                    _vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = sorted(_SIGS)


def _err(rc, total=None):
    if rc == BL_OK:
        return
    msg = lib.bl_last_error().decode()
    if rc == BL_ERR_INVALID:
        raise ValueError(msg)
    if rc == BL_ERR_MODEL:
        raise ModelError(msg)
    if rc == BL_ERR_IO:
        raise IoError(msg)
    if rc == BL_ERR_CAPACITY:
        raise CapacityError(msg, total)
    raise RuntimeError(f"blinkline_b200: {msg}")


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _addr(a):
    """Data pointer of a numpy array or a torch tensor (device or host)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _frames(frames):
    """Normalise a frame batch: numpy/torch (n,h,w) or (h,w), u8 or f64 -> (obj, pix, n, h, w)."""
    if hasattr(frames, "data_ptr"):  # torch tensor, possibly on the GPU
        import torch
        t = frames if frames.dim() == 3 else frames.unsqueeze(0)
        t = t.contiguous()
        if t.dtype == torch.uint8:
            pix = BL_PIX_U8
        elif t.dtype == torch.float64:
            pix = BL_PIX_F64
        else:
            raise ValueError("frames must be uint8 or float64")
        return t, pix, t.shape[0], t.shape[1], t.shape[2]
    a = np.asarray(frames)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ValueError("frames must be (n, h, w) or (h, w)")
    if a.dtype == np.uint8:
        a, pix = np.ascontiguousarray(a), BL_PIX_U8
    else:
        a, pix = np.ascontiguousarray(a, dtype=np.float64), BL_PIX_F64
    return a, pix, a.shape[0], a.shape[1], a.shape[2]


class Context:
    """One device context (stream, models, pre-sized batch arenas) on one GPU."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _err(lib.bl_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self._lock = threading.Lock()
        self._inflight = {}
        self.ert_L = None

    def close(self):
        if getattr(self, "_h", None):
            lib.bl_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- plumbing
    def set_stream(self, stream_ptr):
        _err(lib.bl_ctx_set_stream(self._h, stream_ptr))

    def synchronize(self):
        _err(lib.bl_ctx_synchronize(self._h))

    @property
    def launch_count(self) -> int:
        v = C.c_uint64()
        _err(lib.bl_ctx_launch_count(self._h, C.byref(v)))
        return int(v.value)

    def enable_graphs(self, on=True):
        """CUDA-graph replay of the pipelined path (default on; results identical either way)."""
        _err(lib.bl_ctx_enable_graphs(self._h, int(on)))

    def enable_stage_timing(self, on=True):
        _err(lib.bl_ctx_enable_stage_timing(self._h, int(on)))

    def stage_times(self):
        ms = (C.c_float * len(STAGES))()
        _err(lib.bl_ctx_stage_times(self._h, ms, None))
        return dict(zip(STAGES, [float(v) for v in ms]))

    # ---------------------------------------------------------------- models
    def upload_detector(self, model):
        w = _np(model["weights"], np.float64).reshape(5, 3100)
        b = _np(model["biases"], np.float64).reshape(5)
        _err(lib.bl_detector_upload(self._h, w.ctypes.data, b.ctypes.data, float(model["threshold"]),
                                    int(model.get("window_cells", 10)), int(model.get("cell_px", 8)),
                                    int(model.get("scale_num", 5)), int(model.get("scale_den", 6)),
                                    float(model.get("min_face_ratio", 0.2))))

    def run(self, frames_dir, fps, batch_size=16, det_cap=None):
        """run() (pipeline.hpp:59-60) over a frame_%06d.pgm directory with the uploaded models:
        {"frames": FRAME_DTYPE[n], "detections": DET_DTYPE[...] in frame order,
         "landmarks": (n, L, 2) (NaN rows where no face), "baselines": (left, right)}."""
        n, w, h = ingest(frames_dir)
        L = C.c_int()
        _err(lib.bl_ctx_model_info(self._h, C.byref(L)))
        frames = np.zeros(n, FRAME_DTYPE)
        cap = det_cap if det_cap is not None else n * 64
        dets = np.zeros(cap, DET_DTYPE)
        lms = np.full((n, L.value, 2), np.nan)
        base = np.zeros(2)
        tot = _i64()
        _err(lib.bl_run(self._h, os.fsencode(frames_dir), float(fps), int(batch_size), frames.ctypes.data, n,
                        dets.ctypes.data, cap, C.byref(tot), lms.ctypes.data, base.ctypes.data))
        return {"frames": frames, "detections": dets[:tot.value], "landmarks": lms, "baselines": base}

    def load_detector(self, path):
        """Parse a "hog-v1" model file (load_detector_model) and upload it."""
        self.upload_detector(read_detector_json(path))

    def load_ert(self, path):
        """Parse an "ert-v1" model file (load_ert_model) and upload it without a host copy
        through Python."""
        h = _vp()
        dims = [C.c_int() for _ in range(4)]
        sh = C.c_double()
        _err(lib.bl_ert_file_open(os.fsencode(path), C.byref(h), *[C.byref(d) for d in dims], C.byref(sh)))
        try:
            _err(lib.bl_ert_file_upload(h, self._h))
        finally:
            lib.bl_ert_file_close(h)
        self.ert_L = dims[0].value
        self.ert_TK = dims[1].value * dims[2].value

    def upload_ert(self, ert):
        m = _np(ert["mean_xy"], np.float64)
        a = _np(ert["anchors"], np.int32)
        s = _np(ert["split_params"], np.float64)
        lv = _np(ert["leaves"], np.float64)
        _err(lib.bl_ert_upload(self._h, int(ert["L"]), int(ert["T"]), int(ert["K"]), int(ert["F"]),
                               float(ert["shrinkage"]), m.ctypes.data, a.ctypes.data, s.ctypes.data,
                               lv.ctypes.data))
        self.ert_L = int(ert["L"])
        self.ert_TK = int(ert["T"]) * int(ert["K"])

    # -------------------------------------------------------------- hot path
    def _split(self, out, counts, lm, flat):
        if flat:
            return (out, counts, lm) if lm is not None else (out, counts)
        offs = np.concatenate([[0], np.cumsum(counts)])
        n = len(counts)
        dets = [out[offs[i]:offs[i + 1]] for i in range(n)]
        if lm is None:
            return dets
        return dets, [lm[offs[i]:offs[i + 1]] for i in range(n)]

    def _sync_call(self, frames, landmarks, cap, flat):
        a, pix, n, h, w = _frames(frames)
        cap = cap or max(1024, 64 * n)
        while True:
            out = np.empty(cap, DET_DTYPE)
            lm = np.empty((cap, self.ert_L or 1, 2)) if landmarks else None
            counts = np.zeros(n, np.int32)
            total = C.c_int64(0)
            if landmarks:
                rc = lib.bl_detect_landmarks(self._h, _addr(a), pix, n, w, h, w, w * h, out.ctypes.data, cap,
                                             counts.ctypes.data, C.byref(total), lm.ctypes.data)
            else:
                rc = lib.bl_detect(self._h, _addr(a), pix, n, w, h, w, w * h, out.ctypes.data, cap,
                                   counts.ctypes.data, C.byref(total))
            if rc == BL_ERR_CAPACITY and total.value > cap:
                cap = int(total.value)
                continue
            _err(rc, total.value)
            break
        t = int(total.value)
        return self._split(out[:t], counts, lm[:t] if lm is not None else None, flat)

    def detect(self, frames, cap=None, flat=False):
        """detect_faces over a batch -> list of DET_DTYPE arrays (one per frame), or with
        flat=True (detections of all frames back to back, per-frame counts)."""
        return self._sync_call(frames, False, cap, flat)

    def detect_landmarks(self, frames, cap=None, flat=False):
        """Detect, then landmark every kept detection -> (dets per frame, landmarks per frame),
        or with flat=True (dets, counts, landmarks) back to back."""
        return self._sync_call(frames, True, cap, flat)

    # pipelined mode: up to MAX_IN_FLIGHT batches in flight (H2D, landmark cascade and result
    # copies overlap detection)
    def submit(self, frames, landmarks=True):
        a, pix, n, h, w = _frames(frames)
        t = C.c_uint64(0)
        _err(lib.bl_submit(self._h, _addr(a), pix, n, w, h, w, w * h, int(landmarks), C.byref(t)))
        # keep the frames alive until collected; the batch's device face capacity is fixed at submit
        self._inflight[t.value] = (a, n, landmarks, n * self.face_capacity())
        return t.value

    def collect(self, ticket, flat=True, cap=None):
        if ticket not in self._inflight:
            raise RuntimeError("blinkline_b200: unknown or collected ticket")
        a, n, landmarks, dev_cap = self._inflight[ticket]
        cap = cap or max(1024, 64 * n)
        while True:
            out = np.empty(cap, DET_DTYPE)
            lm = np.empty((cap, self.ert_L or 1, 2)) if landmarks else None
            counts = np.zeros(n, np.int32)
            total = C.c_int64(0)
            rc = lib.bl_collect(self._h, ticket, out.ctypes.data, cap, counts.ctypes.data, C.byref(total),
                                lm.ctypes.data if lm is not None else None)
            if rc == BL_ERR_CAPACITY and cap < total.value <= dev_cap:
                # only the OUTPUT buffer was short: the results stay on the device, collect again
                # (beyond the device face capacity the batch is gone: raise the real cause)
                cap = int(total.value)
                continue
            del self._inflight[ticket]
            _err(rc, total.value)
            break
        t = int(total.value)
        return self._split(out[:t], counts, lm[:t] if lm is not None else None, flat)

    def set_face_capacity(self, faces_per_frame):
        _err(lib.bl_ctx_set_face_capacity(self._h, int(faces_per_frame)))

    def face_capacity(self):
        v = C.c_int(0)
        _err(lib.bl_ctx_get_face_capacity(self._h, C.byref(v)))
        return v.value

    def landmarks(self, frames, frame_of_box, boxes, want_leaves=False):
        """predict_landmarks for (frame, box) pairs -> (n_boxes, L, 2) [, leaf idx (n_boxes, T*K)]."""
        a, pix, n, h, w = _frames(frames)
        if hasattr(boxes, "data_ptr"):  # torch tensors (e.g. boxes already on the device)
            import torch
            fob = frame_of_box.to(torch.int32).contiguous()
            bx = boxes.to(torch.int32).contiguous().reshape(-1, 4)
            nb = int(bx.shape[0])
        else:
            fob = _np(frame_of_box, np.int32)
            bx = _np(boxes, np.int32).reshape(-1, 4)
            nb = len(bx)
        xy = np.zeros((nb, self.ert_L, 2))
        leaves = np.zeros((nb, self.ert_TK), np.uint8) if want_leaves else None
        _err(lib.bl_landmarks(self._h, _addr(a), pix, n, w, h, w, w * h, _addr(fob), _addr(bx), nb,
                              xy.ctypes.data, leaves.ctypes.data if want_leaves else None))
        return (xy, leaves) if want_leaves else xy

    # -------------------------------------------------------- stage functions
    def build_pyramid(self, img, window=80):
        a, pix, n, h, w = _frames(img)
        dims = np.zeros(128, np.int32)
        scales = np.zeros(64)
        nl = C.c_int(0)
        _err(lib.bl_build_pyramid(self._h, _addr(a), pix, w, h, window, None, 0, dims.ctypes.data,
                                  scales.ctypes.data, 64, C.byref(nl)))
        nl = nl.value
        total = int(sum(int(dims[2 * k]) * int(dims[2 * k + 1]) for k in range(nl)))
        out = np.zeros(total)
        _err(lib.bl_build_pyramid(self._h, _addr(a), pix, w, h, window, out.ctypes.data, total, dims.ctypes.data,
                                  scales.ctypes.data, 64, C.byref(C.c_int(0))))
        levels, off = [], 0
        for k in range(nl):
            lw, lh = int(dims[2 * k]), int(dims[2 * k + 1])
            levels.append(out[off:off + lw * lh].reshape(lh, lw))
            off += lw * lh
        return levels, scales[:nl].copy()

    def downscale_bilinear(self, img):
        img = _np(img, np.float64)
        h, w = img.shape
        out = np.zeros((h * 5 // 6, w * 5 // 6))
        _err(lib.bl_downscale_bilinear(self._h, img.ctypes.data, w, h, out.ctypes.data))
        return out

    def compute_gradients(self, img):
        img = _np(img, np.float64)
        h, w = img.shape
        ori = np.zeros((h, w), np.uint8)
        mag = np.zeros((h, w))
        _err(lib.bl_compute_gradients(self._h, img.ctypes.data, w, h, ori.ctypes.data, mag.ctypes.data))
        return ori, mag

    def histogramize(self, ori, mag):
        ori = _np(ori, np.uint8)
        mag = _np(mag, np.float64)
        h, w = mag.shape
        bins = np.zeros((h // 8, w // 8, 18))
        _err(lib.bl_histogramize(self._h, ori.ctypes.data, mag.ctypes.data, w, h, bins.ctypes.data))
        return bins

    def cell_energy(self, bins):
        bins = _np(bins, np.float64)
        ch, cw = bins.shape[:2]
        e = np.zeros((ch, cw))
        _err(lib.bl_cell_energy(self._h, bins.ctypes.data, cw, ch, e.ctypes.data))
        return e

    def compute_features(self, bins, energy):
        bins = _np(bins, np.float64)
        energy = _np(energy, np.float64)
        ch, cw = bins.shape[:2]
        if energy.shape != (ch, cw):
            raise ValueError("compute_features: cell and energy grids must share dimensions")
        f = np.zeros((ch, cw, 31))
        _err(lib.bl_compute_features(self._h, bins.ctypes.data, energy.ctypes.data, cw, ch, f.ctypes.data))
        return f

    def extract_features(self, img, want_cells=False):
        img = _np(img, np.float64)
        h, w = img.shape
        f = np.zeros((h // 8, w // 8, 31))
        bins = np.zeros((h // 8, w // 8, 18))
        en = np.zeros((h // 8, w // 8))
        _err(lib.bl_extract_features(self._h, img.ctypes.data, w, h, f.ctypes.data, bins.ctypes.data,
                                     en.ctypes.data))
        return (f, bins, en) if want_cells else f

    def score_separable(self, feat, weights, bias):
        feat = _np(feat, np.float64)
        wts = _np(weights, np.float64).reshape(3100)
        ch, cw = feat.shape[:2]
        out = np.zeros((max(ch - 9, 0), max(cw - 9, 0)))
        _err(lib.bl_score_window(self._h, feat.ctypes.data, cw, ch, wts.ctypes.data, float(bias), out.ctypes.data))
        return out

    def score_dense(self, feat, weights, bias):
        """score_dense (detector.cpp:45-64): the definitional single-accumulator order."""
        feat = _np(feat, np.float64)
        wts = _np(weights, np.float64).reshape(3100)
        ch, cw = feat.shape[:2]
        out = np.zeros((max(ch - 9, 0), max(cw - 9, 0)))
        _err(lib.bl_score_window_dense(self._h, feat.ctypes.data, cw, ch, wts.ctypes.data, float(bias),
                                       out.ctypes.data))
        return out

    def share_models(self, other):
        """Use `other`'s uploaded models (same device; one device copy for both)."""
        _err(lib.bl_ctx_share_models(self._h, other._h, 3))
        self.ert_L, self.ert_TK = other.ert_L, getattr(other, "ert_TK", None)

    def nms(self, dets, iou_threshold=0.5):
        dets = _np(dets, DET_DTYPE)
        out = np.zeros(max(len(dets), 1), DET_DTYPE)
        kept = C.c_int64(0)
        _err(lib.bl_nms(self._h, dets.ctypes.data if len(dets) else None, len(dets), float(iou_threshold),
                        out.ctypes.data, C.byref(kept)))
        return out[:kept.value].copy()

    def set_screen(self, mode):
        """'tc' (tcgen05 implicit GEMM, default) or 'fp32' (CUDA-core FMA) classifier screen."""
        _err(lib.bl_ctx_set_screen(self._h, {"tc": SCREEN_TCGEN05, "fp32": SCREEN_FP32}[mode]))

    def debug_screen_tc(self, features):
        """Raw tcgen05 screen sums of every anchor of one feature image (ch, cw, 31) against the
        uploaded detector: (scores[5][sh][sw] float32, delta[5] rigorous error bounds)."""
        f = _np(features, np.float64)
        ch, cw = f.shape[0], f.shape[1]
        sc = np.zeros((5, ch - 9, cw - 9), np.float32)
        dl = np.zeros(5, np.float64)
        _err(lib.bl_debug_screen_tc(self._h, f.ctypes.data, cw, ch, sc.ctypes.data, dl.ctypes.data))
        return sc, dl

    def debug_sqrt(self, x):
        x = _np(x, np.float64).ravel()
        fast, ieee = np.zeros_like(x), np.zeros_like(x)
        _err(lib.bl_debug_sqrt(self._h, x.ctypes.data, len(x), fast.ctypes.data, ieee.ctypes.data))
        return fast, ieee

    def orientation_bins(self, gx, gy):
        gx = _np(gx, np.float64).ravel()
        gy = _np(gy, np.float64).ravel()
        out = np.zeros(len(gx), np.uint8)
        _err(lib.bl_orientation_bins(self._h, gx.ctypes.data, gy.ctypes.data, len(gx), out.ctypes.data))
        return out


def plan_geometry(w, h, window_cells=10, cell_px=8, scale_num=5, scale_den=6, min_face_ratio=0.2):
    """Host-only batch geometry: (level dims [(w,h)...], scored levels, scale per scored level,
    box side per scored level).  No GPU needed."""
    dims = np.zeros(128, np.int32)
    scored = np.zeros(64, np.int32)
    sc = np.zeros(64)
    side = np.zeros(64, np.int32)
    nl, ns = C.c_int(0), C.c_int(0)
    _err(lib.bl_plan_geometry(w, h, window_cells, cell_px, scale_num, scale_den, float(min_face_ratio),
                              dims.ctypes.data, scored.ctypes.data, sc.ctypes.data, side.ctypes.data, 64,
                              C.byref(nl), C.byref(ns)))
    levels = [(int(dims[2 * k]), int(dims[2 * k + 1])) for k in range(nl.value)]
    return levels, [int(v) for v in scored[:ns.value]], sc[:ns.value].copy(), [int(v) for v in side[:ns.value]]


# ------------------------------------------------ reference-named module functions
_tls = threading.local()



class MultiContext:
    """Frame sharding over several GPUs in one process (bl_multi_*): one
    context and one host worker thread per listed device, contiguous frame shards, results
    gathered in frame order on the host.  ``devices`` may repeat a device."""

    def __init__(self, devices):
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        _err(lib.bl_multi_create(devs, len(devices), C.byref(h)))
        self._h = h
        self.devices = list(devices)
        self.ert_L = None
        self.last_device_ms = None

    def close(self):
        if getattr(self, "_h", None):
            lib.bl_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_batch_pixels(self, pixels):
        _err(lib.bl_multi_set_batch_pixels(self._h, int(pixels)))

    def upload_detector(self, model):
        w = _np(model["weights"], np.float64).reshape(5, 3100)
        b = _np(model["biases"], np.float64).reshape(5)
        _err(lib.bl_multi_detector_upload(self._h, w.ctypes.data, b.ctypes.data, float(model["threshold"]),
                                          int(model.get("window_cells", 10)), int(model.get("cell_px", 8)),
                                          int(model.get("scale_num", 5)), int(model.get("scale_den", 6)),
                                          float(model.get("min_face_ratio", 0.2))))

    def upload_ert(self, ert):
        m = _np(ert["mean_xy"], np.float64)
        a = _np(ert["anchors"], np.int32)
        sp = _np(ert["split_params"], np.float64)
        lv = _np(ert["leaves"], np.float64)
        _err(lib.bl_multi_ert_upload(self._h, int(ert["L"]), int(ert["T"]), int(ert["K"]), int(ert["F"]),
                                     float(ert["shrinkage"]), m.ctypes.data, a.ctypes.data, sp.ctypes.data,
                                     lv.ctypes.data))
        self.ert_L = int(ert["L"])

    def detect_landmarks(self, frames, landmarks=True, flat=True):
        """Host frames (n, h, w) u8/f64 -> (dets, counts, landmarks) back to back in frame order
        (landmarks=False: (dets, counts))."""
        a, pix, n, h, w = _frames(frames)
        if hasattr(a, "is_cuda") and a.is_cuda:
            raise ValueError("MultiContext takes host frames (each device uploads its own shard)")
        cap = max(1, n * 64)
        out = np.empty(cap, DET_DTYPE)
        lm = np.empty((cap, self.ert_L or 1, 2)) if landmarks else None
        counts = np.zeros(n, np.int32)
        total = _i64()
        ms = np.zeros(len(self.devices))
        _err(lib.bl_multi_detect_landmarks(self._h, _addr(a), pix, n, w, h, w, w * h, out.ctypes.data, cap,
                                           counts.ctypes.data, C.byref(total),
                                           lm.ctypes.data if lm is not None else None, ms.ctypes.data))
        self.last_device_ms = ms
        t = int(total.value)
        if flat:
            return (out[:t], counts, lm[:t]) if landmarks else (out[:t], counts)
        offs = np.concatenate([[0], np.cumsum(counts)])
        dets = [out[offs[i]:offs[i + 1]] for i in range(n)]
        if not landmarks:
            return dets
        return dets, [lm[:t][offs[i]:offs[i + 1]] for i in range(n)]


def default_context(device: int | None = None) -> Context:
    dev = int(os.environ.get("BLINKLINE_DEVICE", "0")) if device is None else device
    ctx = getattr(_tls, "ctx", None)
    if ctx is None or ctx.device != dev:
        ctx = Context(dev)
        _tls.ctx = ctx
        _tls.det_key = None
        _tls.ert_key = None
    return ctx


def _with_detector(model):
    ctx = default_context()
    key = (id(model), float(model["threshold"]), hash(_np(model["weights"], np.float64).tobytes()),
           hash(_np(model["biases"], np.float64).tobytes()))
    if _tls.det_key != key:
        ctx.upload_detector(model)
        _tls.det_key = key
    return ctx


def _with_ert(ert):
    ctx = default_context()
    key = (id(ert), int(ert["T"]), int(ert["K"]), int(ert["F"]), int(ert["L"]))
    if _tls.ert_key != key:
        ctx.upload_ert(ert)
        _tls.ert_key = key
    return ctx


def build_pyramid(img, window=80):
    return default_context().build_pyramid(img, window)


def downscale_bilinear(img):
    return default_context().downscale_bilinear(img)


def compute_gradients(img):
    return default_context().compute_gradients(img)


def histogramize(ori, mag):
    return default_context().histogramize(ori, mag)


def cell_energy(bins):
    return default_context().cell_energy(bins)


def compute_features(bins, energy):
    return default_context().compute_features(bins, energy)


def extract_features(img):
    return default_context().extract_features(img)


def score_separable(feat, weights, bias):
    return default_context().score_separable(feat, weights, bias)


def score_dense(feat, weights, bias):
    return default_context().score_dense(feat, weights, bias)


def nms(dets, iou_threshold=0.5):
    return default_context().nms(dets, iou_threshold)


def orientation_bins(gx, gy):
    return default_context().orientation_bins(gx, gy)


def detect_faces(img, model):
    """detect_faces(img, model) -> DET_DTYPE array (detector.hpp:87)."""
    return _with_detector(model).detect(img)[0]


def predict_landmarks(img, box, ert, want_leaves=False):
    """predict_landmarks(img, box, model) -> (L, 2) image-pixel landmarks (ert.hpp:86)."""
    ctx = _with_ert(ert)
    r = ctx.landmarks(img, [0], [list(box)], want_leaves=want_leaves)
    return (r[0][0], r[1][0]) if want_leaves else r[0]


# ------------------------------------------------------------------ data formats
def read_pgm(path):
    """load_pgm (image.hpp:25) as an (h, w) uint8 array (PGM samples are integers <= 255)."""
    w, h = C.c_int(), C.c_int()
    p = os.fsencode(path)
    _err(lib.bl_read_pgm(p, C.byref(w), C.byref(h), None, 0))
    out = np.empty((h.value, w.value), np.uint8)
    _err(lib.bl_read_pgm(p, C.byref(w), C.byref(h), out.ctypes.data, out.size))
    return out


def write_pgm(path, img):
    """save_pgm (image.hpp:28): binary P5, values clamped to [0, 255] and rounded."""
    a = _np(img, np.float64)
    _err(lib.bl_write_pgm(os.fsencode(path), a.ctypes.data, a.shape[1], a.shape[0]))


def read_detector_json(path):
    """load_detector_model (detector.hpp:100) -> the dict Context.upload_detector takes."""
    p = os.fsencode(path)
    thr, mfr = C.c_double(), C.c_double()
    wc, cp, sn, sd = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    _err(lib.bl_read_detector_json(p, None, None, C.byref(thr), C.byref(wc), C.byref(cp), C.byref(sn), C.byref(sd),
                                   C.byref(mfr)))
    w = np.empty((5, wc.value * wc.value * 31), np.float64)
    b = np.empty(5, np.float64)
    _err(lib.bl_read_detector_json(p, w.ctypes.data, b.ctypes.data, C.byref(thr), C.byref(wc), C.byref(cp),
                                   C.byref(sn), C.byref(sd), C.byref(mfr)))
    return {"weights": w, "biases": b, "threshold": thr.value, "window_cells": wc.value, "cell_px": cp.value,
            "scale_num": sn.value, "scale_den": sd.value, "min_face_ratio": mfr.value}


def write_detector_json(path, model):
    """save_model(DetectorModel) (detector.hpp:99)."""
    w = _np(model["weights"], np.float64).reshape(5, -1)
    b = _np(model["biases"], np.float64).reshape(5)
    _err(lib.bl_write_detector_json(os.fsencode(path), w.ctypes.data, b.ctypes.data, float(model["threshold"]),
                                    int(model.get("window_cells", 10)), int(model.get("cell_px", 8)),
                                    int(model.get("scale_num", 5)), int(model.get("scale_den", 6)),
                                    float(model.get("min_face_ratio", 0.2))))


def read_ert_json(path):
    """load_ert_model (ert.hpp:129) -> the dict Context.upload_ert takes."""
    h = _vp()
    L, T, K, F = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    sh = C.c_double()
    _err(lib.bl_ert_file_open(os.fsencode(path), C.byref(h), C.byref(L), C.byref(T), C.byref(K), C.byref(F),
                              C.byref(sh)))
    try:
        S, NL = (1 << F.value) - 1, 1 << F.value
        n = T.value * K.value
        out = {"L": L.value, "T": T.value, "K": K.value, "F": F.value, "shrinkage": sh.value,
               "mean_xy": np.empty((L.value, 2), np.float64),
               "anchors": np.empty((n * S, 2), np.int32), "split_params": np.empty((n * S, 5), np.float64),
               "leaves": np.empty((n * NL, L.value, 2), np.float64)}
        _err(lib.bl_ert_file_copy(h, out["mean_xy"].ctypes.data, out["anchors"].ctypes.data,
                                  out["split_params"].ctypes.data, out["leaves"].ctypes.data))
        return out
    finally:
        lib.bl_ert_file_close(h)


def write_ert_json(path, ert):
    """save_model(ErtModel) (ert.hpp:128)."""
    m = _np(ert["mean_xy"], np.float64)
    a = _np(ert["anchors"], np.int32)
    s = _np(ert["split_params"], np.float64)
    lv = _np(ert["leaves"], np.float64)
    _err(lib.bl_write_ert_json(os.fsencode(path), int(ert["L"]), int(ert["T"]), int(ert["K"]), int(ert["F"]),
                               float(ert["shrinkage"]), m.ctypes.data, a.ctypes.data, s.ctypes.data, lv.ctypes.data))


def ingest(frames_dir):
    """ingest (pipeline.hpp:33): validates a frame_%06d.pgm directory -> (n_frames, w, h)."""
    n, w, h = C.c_int(), C.c_int(), C.c_int()
    _err(lib.bl_ingest(os.fsencode(frames_dir), C.byref(n), C.byref(w), C.byref(h)))
    return n.value, w.value, h.value
