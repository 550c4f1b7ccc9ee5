import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def lib():
    from paper_1910_00078_b200.primkit import library
    return library()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.reference()
    if r is None:
        pytest.skip("reference oracle library (oracle/_ref) not built")
    return r


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def rel_l2(got, want) -> float:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))


def max_rel(got, want) -> float:
    """The reference's own metric: max |g - w| / max(1, |w|) (test_util.hpp:24-33)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want)))) if got.size else 0.0


def nchw_to_dev(a, pitch=None):
    """Packed NCHW f32 -> the device layout (NHWC, channel pitch roundup(C, 8))."""
    n, c, h, w = a.shape
    pitch = pitch or (c + 7) // 8 * 8
    out = np.zeros((n, h, w, pitch), np.float32)
    out[..., :c] = a.transpose(0, 2, 3, 1)
    return out


def oracle_sampled(p, a, b, got, ns=4096, seed=0):
    """(got, want) on ns sampled coordinates of a host-ABI conv result `got`
    (packed NCHW / filter layout) for operands a, b in the reference operand
    order, with the oracle's f64 direct formula (groups 1, convolution mode)."""
    import oracle
    from paper_1910_00078_b200 import abi
    rng = np.random.default_rng(seed)
    A, B = nchw_to_dev(np.asarray(a, np.float32)), nchw_to_dev(np.asarray(b, np.float32))
    dims = got.shape
    if p.direction == abi.BACKWARD_WEIGHTS:
        k, c, r, s = dims
        ks = rng.choice(k, min(64, k), replace=False)
        taps = np.stack([rng.integers(0, r, 64), rng.integers(0, s, 64), rng.integers(0, c, 64)], 1)
        want = oracle.sample_backward_weights(p, A, B, ks, taps, bf16=False).ravel()
        return got[ks[:, None], taps[None, :, 2], taps[None, :, 0], taps[None, :, 1]].ravel(), want
    idx = np.stack([rng.integers(0, m, ns) for m in dims], 1)
    fn = oracle.sample_forward if p.direction == abi.FORWARD else oracle.sample_backward_data
    want = fn(p, A, B, idx, bf16=False)
    return got[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]], want
