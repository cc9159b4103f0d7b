"""The drop-in boundary without a GPU: the C-ABI library loads, exports every entry point
include/*.h declares, the Python and C++ layers bind exactly that surface, and there is no
silent CPU fallback (creating a device context fails loudly when no GPU is present)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "blinkline_b200.h")
LIB = os.path.join(ROOT, "paper_2006_00816_b200", "libblinkline_b200.so")
CPPLIB = os.path.join(ROOT, "paper_2006_00816_b200", "libblinkline_gpu.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+\**(bl_\w+)\s*\(", src, flags=re.M)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.split()}


def test_header_declares_the_hot_path():
    d = declared()
    for name in ["bl_ctx_create", "bl_detector_upload", "bl_ert_upload", "bl_detect", "bl_landmarks",
                 "bl_detect_landmarks", "bl_build_pyramid", "bl_compute_gradients", "bl_histogramize",
                 "bl_cell_energy", "bl_compute_features", "bl_extract_features", "bl_score_window", "bl_nms",
                 "bl_plan_geometry"]:
        assert name in d


def test_library_exports_every_declared_symbol():
    ex = exported(LIB)
    missing = [s for s in declared() if s not in ex]
    assert not missing, missing


def test_library_loads_and_binds_every_symbol():
    lib = ctypes.CDLL(LIB)
    for s in declared():
        assert getattr(lib, s) is not None
    assert lib.bl_abi_version() == 1


def test_python_binding_covers_header():
    import paper_2006_00816_b200 as bl
    assert sorted(bl.EXPORTED) == declared()


def test_cpp_dropin_exports_reference_api():
    syms = subprocess.run(["nm", "-DC", "--defined-only", CPPLIB], capture_output=True, text=True,
                          check=True).stdout
    for fn in ["blinkline::detect_faces(", "blinkline::predict_landmarks(", "blinkline::build_pyramid(",
               "blinkline::extract_features(", "blinkline::compute_gradients(", "blinkline::histogramize(",
               "blinkline::nms(", "blinkline::score_separable(", "blinkline::gpu::detect_faces_batch("]:
        assert fn in syms, fn


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2006_00816_b200 as bl
    with pytest.raises(RuntimeError):
        bl.Context(0)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2006_00816_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in text and "blink_oracle" not in text and "liboracle" not in text, f
    ldd = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "blinkline_ref" not in ldd
