import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the C-ABI kernels")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def lib():
    from paper_1212_1639_b200 import _lib

    return _lib.load()


@pytest.fixture(scope="session")
def gpu(lib):
    """The loaded C-ABI library on a machine with a visible CUDA device."""
    n = lib.pf_device_count()
    if n < 1:
        pytest.fail("gpu-marked test run without a visible CUDA device")
    return lib


def fixture_run_kwargs(d):
    """Model / prior keyword arguments recorded in a run_* golden fixture."""
    from paper_1212_1639_b200 import InverseGammaPrior, Priors, TrendNoiseModel

    if "prior" in d:
        p = d["prior"]
        s2 = InverseGammaPrior(p[2], p[3]) if p[2] > 0 else float(p[3])
        t2 = InverseGammaPrior(p[4], p[5]) if p[4] > 0 else float(p[5])
        return "learn", Priors(x0_mean=p[0], x0_var=p[1], sigma2=s2, tau2=t2)
    m = d["model"]
    return "filter", TrendNoiseModel(sigma2=float(m[0]), tau2=float(m[1]),
                                     x0_mean=float(m[2]), x0_var=float(m[3]))


def random_cdf(rng, n, zero_fraction=0.0, dtype=np.float64):
    """Valid CDF from exponential weights with optional exact zeros (the
    reference suite's helper, tests/conftest.py:16-25), built by the oracle."""
    from oracle import restate as R

    w = rng.exponential(size=n).astype(dtype)
    if zero_fraction:
        mask = rng.random(n) < zero_fraction
        if mask.all():
            mask[rng.integers(n)] = False
        w[mask] = 0.0
    prefix = np.cumsum(w)
    return R.finalize_cdf(prefix, prefix[-1])
