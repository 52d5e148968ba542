"""Resampling CDF by the two-pass adder tree, on the device.

Semantics and results follow the reference bit for bit (prefix_sum.py):
``forward_adder`` pairs neighbours level by level, ``backward_adder`` walks
back down (right child = parent, left child = parent - right sibling's
forward sum), and ``parallel_cdf`` divides by the root, applies the running
max, clips to [0, 1] and pins the last entry to 1.  The device evaluates the
same tree as per-tile subtrees plus a top tree (csrc/cdf.cuh), which is why
the results do not depend on the launch geometry -- the analogue of the
reference's lane-count invariance.

``sequential_cumsum`` / ``sequential_cdf`` are the reference's left-to-right
oracles used by its sequential-baseline resamplers; a strictly sequential
floating-point recurrence has no exact parallel form, so they are host
utilities here and are not on the cut-point path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import check_weights, is_power_of_two
from .errors import AllWeightsZeroError, NotPowerOfTwoError


@dataclass
class AdderTree:
    """Pairwise partial sums: levels[0] is the input, the top level its total."""

    levels: list

    @property
    def n(self):
        return len(self.levels[0])

    @property
    def total(self):
        return self.levels[-1][0]


def _float_array(w):
    w = np.asarray(w)
    if w.dtype not in (np.float32, np.float64):
        w = w.astype(np.float64)
    return np.ascontiguousarray(w)


def sequential_cumsum(weights):
    """Left-to-right inclusive prefix sums (prefix_sum.py:41-43)."""
    return np.cumsum(np.asarray(weights))


def _device_tree(w):
    n = len(w)
    levels_flat = np.empty(2 * n - 1, dtype=w.dtype)
    prefix = np.empty(n, dtype=w.dtype)
    lib = _lib.require_device()
    _lib.check(lib.pf_adder_tree(_lib.vptr(w), n, _lib.dtype_code(w.dtype),
                                 _lib.vptr(levels_flat), _lib.vptr(prefix)), lib)
    levels, off, m = [], 0, n
    while True:
        levels.append(levels_flat[off:off + m].copy())
        off += m
        if m == 1:
            break
        m //= 2
    return levels, prefix


def forward_adder(weights, backend=None):
    """All tree levels (prefix_sum.py:46-69); NotPowerOfTwoError unless 2^k."""
    w = _float_array(weights)
    n = w.shape[0]
    if not is_power_of_two(n):
        raise NotPowerOfTwoError(f"forward adder needs a power-of-two input, got {n}")
    levels, _ = _device_tree(w)
    levels[0] = np.asarray(weights) if np.asarray(weights).dtype == w.dtype else w
    return AdderTree(levels)


def backward_adder(tree, backend=None):
    """Inclusive prefix sums from an adder tree (prefix_sum.py:72-91)."""
    w = _float_array(tree.levels[0])
    _, prefix = _device_tree(w)
    return prefix


def _finalize_check(total):
    if not np.isfinite(total):
        raise AllWeightsZeroError("weight total is not finite")
    if total <= 0:
        raise AllWeightsZeroError()


def parallel_cdf(weights, backend=None, pad=False):
    """q(i) = s(i)/s(N) from the two adder passes (prefix_sum.py:109-127).
    ``pad=True`` zero-extends a non-power-of-two input.  A CUDA tensor stays
    on the device (device_ops.parallel_cdf) and a device tensor comes back."""
    if _lib.is_cuda_tensor(weights):
        from . import device_ops

        return device_ops.parallel_cdf(weights, pad=pad)
    w = check_weights(weights)
    w = _float_array(w)
    n = w.shape[0]
    if not is_power_of_two(n):
        if not pad:
            raise NotPowerOfTwoError(
                f"parallel CDF needs a power-of-two particle count, got {n} "
                "(set pad=True to zero-pad)")
        m = 1 << (n - 1).bit_length()
        w = np.concatenate([w, np.zeros(m - n, dtype=w.dtype)])
    q = np.empty_like(w)
    total = _lib.C.c_double(0.0)
    lib = _lib.require_device()
    _lib.check(lib.pf_tree_cdf(_lib.vptr(w), len(w), _lib.dtype_code(w.dtype), _lib.vptr(q),
                               _lib.C.byref(total)), lib)
    return q


def _finalize_cdf(prefix, total):
    """prefix_sum.py:94-106 on host arrays (divide, running max, clip, pin)."""
    _finalize_check(total)
    q = prefix / total
    np.maximum.accumulate(q, out=q)
    np.clip(q, q.dtype.type(0), q.dtype.type(1), out=q)
    q[-1] = 1
    return q


def sequential_cdf(weights):
    """CDF from a plain left-to-right cumulative sum (prefix_sum.py:130-134)."""
    w = check_weights(weights)
    prefix = np.cumsum(w)
    return _finalize_cdf(prefix, prefix[-1])
