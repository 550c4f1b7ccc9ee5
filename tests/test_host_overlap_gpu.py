"""Overlapped host-buffer path of primkit_conv_run (pinned buffers, forward /
backward data): the batch runs in image chunks so host->device copies,
compute and device->host copies of neighbouring chunks overlap. Results must
be bit-identical to the single-shot path and the op counters must advance
once for the whole problem (reference semantics, tensor.hpp:21-27)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from paper_1910_00078_b200 import abi
from paper_1910_00078_b200.primkit import operand_shapes, problem

from conftest import rel_l2

pytestmark = pytest.mark.gpu

CASES = [
    (dict(n=6, c=64, h=14, w=14, k=128, y=3, x=3, pad=1), abi.FORWARD, "ImplicitGemm", abi.BF16),
    (dict(n=5, c=64, h=12, w=12, k=64, y=1, x=1), abi.FORWARD, "Direct", abi.F32),
    (dict(n=7, c=128, h=14, w=14, k=64, y=3, x=3, pad=1, stride=2), abi.BACKWARD_DATA,
     "Im2colGemm", abi.BF16),
]


def _pinned(torch, arr):
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).pin_memory()
    return t, C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_float))


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_chunked_host_path_matches(lib, ci):
    torch = pytest.importorskip("torch")
    shp, d, solver, et = CASES[ci]
    p = problem(**shp, direction=d, etype=et)
    sa, sb, so = operand_shapes(lib, p)
    rng = np.random.default_rng(11 + ci)
    a = rng.uniform(-1, 1, sa).astype(np.float32)
    b = rng.uniform(-1, 1, sb).astype(np.float32)
    if et == abi.BF16:
        a, b = oracle.round_bf16(a), oracle.round_bf16(b)
    h = lib.handle()
    ws = h.workspace_bytes(solver, p)

    def run(chunk_kb):
        ta, pa = _pinned(torch, a)
        tb, pb = _pinned(torch, b)
        to, po = _pinned(torch, np.zeros(so, np.float32))
        os.environ["PK_HOST_CHUNK_KB"] = str(chunk_kb)
        try:
            h.reset_counters()
            lib.check(lib.lib.primkit_conv_run(h.ptr, C.byref(p), solver.encode(), pa, pb, po,
                                               C.c_size_t(ws)))
        finally:
            os.environ.pop("PK_HOST_CHUNK_KB", None)
        return to.numpy().copy(), h.counters()

    single, c_single = run(0)          # chunking disabled
    per_img = 4 * max(np.prod(sa[1:]), np.prod(so[1:]))
    chunked, c_chunked = run(per_img * 2 / 1024)  # two images per chunk
    assert np.array_equal(single, chunked)
    assert c_single == c_chunked
    want = (oracle.conv_forward(p, a, b) if d == abi.FORWARD else oracle.conv_backward_data(p, a, b))
    assert rel_l2(chunked, want) <= (1e-2 if et == abi.BF16 else 1e-4)
