"""Exact multinomial resampling by the cut-point method, on the device.

``cut_points_parallel`` (resampling.py:110-134): slot j owns cut-table
entries (L_{j-1}, L_j] with L_j = ceil(N q_j); ``cutpoint_indices``
(resampling.py:146-158): start at I_ceil(N u) and advance while u > q(k),
i.e. the smallest 1-based k with u <= q(k).  Inside the filter loop the same
lookup runs fused into the step kernel (csrc/step.cuh); these wrappers expose
it at kernel level with the reference's signatures and 1-based indices.

The reference's sequential baselines (naive / sorted / stratified /
systematic, resampling.py:29-87) search the same CDF with searchsorted
'right' semantics; their device versions here (and in the filter loop, on
the reference's sequential-cumsum CDF) give the reference's indices.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .rng import uniforms_at


def _cdf_array(cdf):
    q = np.asarray(cdf)
    if q.dtype not in (np.float32, np.float64):
        q = q.astype(np.float64)
    return np.ascontiguousarray(q)


def cut_points_bruteforce(cdf):
    """O(N^2) oracle: idx[j] = min{ i : q(i) > (j-1)/N } (resampling.py:93-107)."""
    q = np.asarray(cdf)
    n = len(q)
    thresholds = np.arange(n, dtype=q.dtype) / q.dtype.type(n)
    out = np.empty(n, dtype=np.int64)
    block = max(1, (1 << 24) // n)
    for lo in range(0, n, block):
        hi = min(lo + block, n)
        out[lo:hi] = np.argmax(q[None, :] > thresholds[lo:hi, None], axis=1) + 1
    return out


def cut_points_parallel(cdf, backend=None):
    """1-based cut-point table (resampling.py:110-134)."""
    if _lib.is_cuda_tensor(cdf):
        from . import device_ops

        return device_ops.cut_points_parallel(cdf)
    q = _cdf_array(cdf)
    out = np.empty(len(q), dtype=np.int64)
    lib = _lib.require_device()
    _lib.check(lib.pf_cut_table(_lib.vptr(q), len(q), _lib.dtype_code(q.dtype),
                                _lib.ptr(out, _lib.C.c_int64)), lib)
    return out


def cutpoint_indices(cdf, cuts, u):
    """Cut-point lookup for an array of uniforms (resampling.py:146-158)."""
    if _lib.is_cuda_tensor(cdf):
        from . import device_ops

        return device_ops.cutpoint_indices(cdf, _on_device(cuts, cdf), _on_device(u, cdf))
    q = _cdf_array(cdf)
    cuts = np.ascontiguousarray(np.asarray(cuts, dtype=np.int64))
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    shape = u.shape
    u = u.reshape(-1)
    out = np.empty(len(u), dtype=np.int64)
    lib = _lib.require_device()
    _lib.check(lib.pf_cutpoint_lookup(_lib.vptr(q), _lib.ptr(cuts, _lib.C.c_int64), len(q),
                                      _lib.dtype_code(q.dtype), _lib.ptr(u), len(u),
                                      _lib.ptr(out, _lib.C.c_int64)), lib)
    return out.reshape(shape)


def cut_point_draw(cdf, cuts, u):
    """One cut-point lookup (resampling.py:137-143)."""
    return int(cutpoint_indices(cdf, cuts, np.array([float(u)]))[0])


def resample_cutpoint(cdf, streams, backend=None):
    """Exact multinomial resampling (resampling.py:161-177): one uniform per
    stream, cut table, lookup; 1-based indices.  A CUDA-tensor CDF stays on
    the device and device indices come back."""
    if _lib.is_cuda_tensor(cdf):
        return _resample_cutpoint_device(cdf, streams)
    q = _cdf_array(cdf)
    n = len(q)
    c = streams.lockstep_counter() if hasattr(streams, "lockstep_counter") else None
    lib = _lib.require_device()
    if c is not None and len(streams) == n and np.array_equal(
            streams.stream_ids, np.arange(n, dtype=np.uint64)):
        out = np.empty(n, dtype=np.int64)
        _lib.check(lib.pf_resample_cutpoint(_lib.vptr(q), n, _lib.dtype_code(q.dtype),
                                            np.uint64(streams.seed), np.uint64(c),
                                            _lib.ptr(out, _lib.C.c_int64)), lib)
        streams.skip(1)
        return out
    u = streams.uniforms()
    return cutpoint_indices(q, cut_points_parallel(q), u)


def _on_device(x, like):
    import torch

    return torch.as_tensor(x, device=like.device)


def _resample_cutpoint_device(cdf, streams):
    from . import device_ops

    n = cdf.shape[0]
    c = streams.lockstep_counter() if hasattr(streams, "lockstep_counter") else None
    if c is not None and len(streams) == n and np.array_equal(
            streams.stream_ids, np.arange(n, dtype=np.uint64)):
        out = device_ops.resample_cutpoint(cdf, streams.seed, c)
        streams.skip(1)
        return out
    u = _on_device(streams.uniforms(), cdf)
    return device_ops.cutpoint_indices(cdf, device_ops.cut_points_parallel(cdf), u)


def merge_indices(cdf, u, sort_first=False):
    """Smallest 1-based i with u < q(i) (resampling.py:29-36), on the device;
    ``sort_first`` sorts u ascending first (resample_sorted)."""
    q = _cdf_array(cdf)
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    shape = u.shape
    u = u.reshape(-1)
    out = np.empty(len(u), dtype=np.int64)
    lib = _lib.require_device()
    _lib.check(lib.pf_merge_indices(_lib.vptr(q), len(q), _lib.dtype_code(q.dtype), _lib.ptr(u), len(u),
                                    int(bool(sort_first)), _lib.ptr(out, _lib.C.c_int64)), lib)
    return out.reshape(shape)


def resample_naive(cdf, streams):
    """Exact multinomial by a head-to-tail scan per draw (resampling.py:51-54):
    the same answer as searchsorted 'right' on the slot's own uniform."""
    return merge_indices(cdf, streams.uniforms())


def resample_sorted(cdf, streams):
    """Exact multinomial with pre-sorted uniforms (resampling.py:57-67).
    Returns ``(indices, sort_ns)``; the sort runs on the device inside the
    merge call, so its time is reported as 0 here (the filter loop times it
    with CUDA events, PhaseTimings.resample_sort_only)."""
    return merge_indices(cdf, streams.uniforms(), sort_first=True), 0


def resample_stratified(cdf, streams):
    """One uniform per stratum (resampling.py:70-75): u_j = (j + v_j) / N."""
    n = len(cdf)
    v = streams.uniforms()
    return merge_indices(cdf, (np.arange(n) + v) / n)


def resample_systematic(cdf, stream):
    """One shared offset (resampling.py:78-87): u_j = (j + v) / N."""
    n = len(cdf)
    v = stream.uniform()
    return merge_indices(cdf, (np.arange(n) + v) / n)


__all__ = [
    "cut_point_draw", "cut_points_bruteforce", "cut_points_parallel", "cutpoint_indices",
    "merge_indices", "resample_cutpoint", "resample_naive", "resample_sorted",
    "resample_stratified", "resample_systematic", "uniforms_at",
]
