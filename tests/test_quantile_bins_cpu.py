"""The resolve's sub-bin map (csrc/quantile.cuh sub_bin) is evaluated in fp64:
floor((key - lo) nb / (hi - lo + 1)) as a correctly rounded double division,
truncated.  Check that it equals the integer floor division at every bin edge
(and around it) for random intervals, for both histogram widths -- the select
kernels invert it with the integer formula."""
import numpy as np
import pytest


@pytest.mark.parametrize("nb", [2048, 4096])
def test_fp64_sub_bin_is_exact_integer_division(nb):
    rng = np.random.default_rng(nb)
    for _ in range(60):
        lo = int(rng.integers(0, 2**32 - 1))
        hi = int(rng.integers(lo, 2**32))
        span = hi - lo + 1
        edges = {lo + (x * span + nb - 1) // nb for x in range(nb + 1)}
        ks = {k for e in edges for k in (e - 1, e, e + 1) if lo <= k <= hi}
        ks |= set(int(k) for k in rng.integers(lo, hi + 1, 5000, dtype=np.uint64)) | {lo, hi}
        ks = np.array(sorted(ks), dtype=np.uint64)
        ref = np.array([(int(k) - lo) * nb // span for k in ks], dtype=np.uint64)
        got = ((ks - np.uint64(lo)).astype(np.float64) * nb / float(span)).astype(np.uint64)
        assert np.array_equal(ref, got), (lo, hi)
