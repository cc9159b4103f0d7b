"""The C++ drop-in API on the GPU (tests/cpp/test_dropin.cpp --gpu): the reference's unit-test
cases called exactly as a reference user calls blinkline::detect_faces / predict_landmarks."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_on_gpu():
    exe = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", ROOT, "tests/cpp/test_dropin"], check=True)
    r = subprocess.run([exe, "--gpu", os.path.join(ROOT, "tests", "golden", "pattern_detector.bin")],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
