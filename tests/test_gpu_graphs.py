"""CUDA-graph replay of the pipelined path (bl_ctx_enable_graphs): bit-identical to eager
launches across batch shapes, slots, lanes, input buffers, host/device inputs and model swaps."""

import numpy as np
import pytest

import paper_2006_00816_b200 as bl
from pyoracle import random_ert, ring_frames_np

pytestmark = pytest.mark.gpu


def _ctx(det, ert, graphs):
    c = bl.Context(0)
    c.enable_graphs(graphs)
    c.upload_detector(det)
    c.upload_ert(ert)
    return c


def _stream(c, batches):
    out = []
    pend = []
    for b in batches:
        pend.append(c.submit(b))
        if len(pend) == bl.MAX_IN_FLIGHT:
            out.append(c.collect(pend.pop(0)))
    while pend:
        out.append(c.collect(pend.pop(0)))
    return out


def _same(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        for u, v in zip(x, y):
            assert np.array_equal(u, v)


def test_graphs_match_eager(pattern_model):
    import torch
    ert = random_ert(T=5, K=64, F=4, seed=77)
    small = ring_frames_np(16, 320, 240, seed=1)
    big = ring_frames_np(8, 640, 480, seed=2)
    dev = torch.from_numpy(small).cuda()
    dev2 = torch.from_numpy(small[::-1].copy()).cuda()
    batches = [small, small, big, dev, dev2, dev, small[:5], big, dev2, small, small, big] * 2
    eager = _stream(_ctx(pattern_model, ert, False), batches)
    g = _ctx(pattern_model, ert, True)
    got = _stream(g, batches)
    _same(eager, got)
    # model swap: captured graphs are invalidated
    ert2 = random_ert(T=3, K=32, F=3, seed=78)
    g.upload_ert(ert2)
    e2 = _ctx(pattern_model, ert2, False)
    _same(_stream(e2, batches[:6]), _stream(g, batches[:6]))
    # synchronous calls go through the same slots
    a = g.detect_landmarks(big)
    b = e2.detect_landmarks(big)
    for u, v in zip(a, b):
        for x, y in zip(u, v):
            assert np.array_equal(x, y)


def test_graph_launch_count_matches_eager(pattern_model):
    ert = random_ert(T=3, K=32, F=4, seed=5)
    frames = ring_frames_np(4, 320, 240, seed=9)
    counts = []
    for graphs in (False, True):
        c = _ctx(pattern_model, ert, graphs)
        _stream(c, [frames] * 4)  # warm-up / capture
        l0 = c.launch_count
        _stream(c, [frames] * 8)
        counts.append(c.launch_count - l0)
    assert counts[0] == counts[1] > 0
