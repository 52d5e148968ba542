"""Kernel-level operations on device-resident torch tensors.

The host-array wrappers (rng.uniforms_at, prefix_sum.parallel_cdf,
resampling.cut_points_parallel / cutpoint_indices / resample_cutpoint,
filtering.weighted_quantiles) dispatch here when they are handed a CUDA
tensor.  Each call enqueues the same kernels as the host form on torch's
current stream of the tensor's device through the C ABI's ``*_d`` entries
(include/parsmc_b200.h) -- no host copies, no host synchronisation -- and
returns a tensor on that device.  Results are bit-identical to the host
forms on the same inputs.

The reference raises on an all-zero or non-finite weight total
(prefix_sum.py:94-106).  ``parallel_cdf`` keeps that behaviour by reading
back the 8-byte total (``check=True``, the default); ``check=False`` leaves
the call fully asynchronous and the caller checks the returned total.
"""

from __future__ import annotations

from . import _lib
from .errors import AllWeightsZeroError, NotPowerOfTwoError


def _torch():
    import torch

    return torch


def _flat(t, dtype=None):
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.reshape(-1).contiguous()


def _float_tensor(t):
    torch = _torch()
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    return t.contiguous()


def _as_words(x, device):
    """64-bit words as int64 (torch's uint64 support is partial; the kernels
    read the same bits as uint64)."""
    torch = _torch()
    t = torch.as_tensor(x, device=device)
    if t.dtype == torch.uint64:
        return t.contiguous().view(torch.int64)
    return t.to(torch.int64)


def uniforms_at(seed, stream_ids, counters):
    """rng.py:122-140 for device stream ids / counters (broadcast)."""
    torch = _torch()
    ids = _as_words(stream_ids, stream_ids.device)
    ctr = _as_words(counters, stream_ids.device)
    ids, ctr = torch.broadcast_tensors(ids, ctr)
    shape = ids.shape
    ids, ctr = _flat(ids), _flat(ctr)
    out = torch.empty(ids.numel(), dtype=torch.float64, device=ids.device)
    lib = _lib.require_device()
    with torch.cuda.device(ids.device):
        _lib.check(lib.pf_uniforms_at_d(int(seed) & (2**64 - 1), _lib.dptr(ids), _lib.dptr(ctr), ids.numel(),
                                        _lib.dptr(out), _lib.current_stream(ids)), lib)
    return out.reshape(shape)


def parallel_cdf(weights, pad=False, check=True, return_total=False):
    """prefix_sum.py:109-127 on a device weight vector (float32 / float64)."""
    torch = _torch()
    w = _float_tensor(weights)
    if w.dim() != 1:
        raise ValueError("weights must be a 1-d tensor")
    n = w.shape[0]
    if n == 0:
        raise ValueError("weights must be non-empty")
    if n & (n - 1):
        if not pad:
            raise NotPowerOfTwoError(
                f"parallel CDF needs a power-of-two particle count, got {n} (set pad=True to zero-pad)")
        m = 1 << (n - 1).bit_length()
        w = torch.cat([w, w.new_zeros(m - n)])
    q = torch.empty_like(w)
    total = torch.empty(1, dtype=torch.float64, device=w.device)
    lib = _lib.require_device()
    with torch.cuda.device(w.device):
        _lib.check(lib.pf_tree_cdf_d(_lib.dptr(w), w.shape[0], _lib.device_dtype_code(w), _lib.dptr(q),
                                     _lib.dptr(total), _lib.current_stream(w)), lib)
    if check:
        tot = float(total.item())
        if tot != tot or tot in (float("inf"), float("-inf")):
            raise AllWeightsZeroError("weight total is not finite")
        if tot <= 0:
            raise AllWeightsZeroError()
    return (q, total) if return_total else q


def cut_points_parallel(cdf):
    """resampling.py:110-134: 1-based int64 cut table of a device CDF."""
    torch = _torch()
    q = _float_tensor(cdf)
    n = q.shape[0]
    out = torch.empty(n, dtype=torch.int64, device=q.device)
    lib = _lib.require_device()
    with torch.cuda.device(q.device):
        _lib.check(lib.pf_cut_table_d(_lib.dptr(q), n, _lib.device_dtype_code(q), _lib.dptr(out),
                                      _lib.current_stream(q)), lib)
    return out


def cutpoint_indices(cdf, cuts, u):
    """resampling.py:146-158 over device uniforms (any shape); 1-based."""
    torch = _torch()
    q = _float_tensor(cdf)
    cuts = _flat(cuts, torch.int64)
    shape = u.shape
    uf = _flat(u, torch.float64)
    out = torch.empty(uf.numel(), dtype=torch.int64, device=q.device)
    lib = _lib.require_device()
    with torch.cuda.device(q.device):
        _lib.check(lib.pf_cutpoint_lookup_d(_lib.dptr(q), _lib.dptr(cuts), q.shape[0], _lib.device_dtype_code(q),
                                            _lib.dptr(uf), uf.numel(), _lib.dptr(out), _lib.current_stream(q)), lib)
    return out.reshape(shape)


def resample_cutpoint(cdf, seed, counter):
    """resampling.py:161-177 for streams 0..n-1 at one lockstep counter."""
    torch = _torch()
    q = _float_tensor(cdf)
    n = q.shape[0]
    out = torch.empty(n, dtype=torch.int64, device=q.device)
    lib = _lib.require_device()
    with torch.cuda.device(q.device):
        _lib.check(lib.pf_resample_cutpoint_d(_lib.dptr(q), n, _lib.device_dtype_code(q), int(seed) & (2**64 - 1),
                                              int(counter), _lib.dptr(out), _lib.current_stream(q)), lib)
    return out


def weighted_quantiles(values, weights, probs):
    """filtering.py:135-140 on device values / weights; probs may be host."""
    torch = _torch()
    v = _flat(values, torch.float64)
    w = _float_tensor(weights).reshape(-1)
    if w.numel() != v.numel():
        raise ValueError("values and weights differ in length")
    p = torch.as_tensor(probs, dtype=torch.float64).reshape(-1).to(v.device).contiguous()
    out = torch.empty(p.numel(), dtype=torch.float64, device=v.device)
    lib = _lib.require_device()
    with torch.cuda.device(v.device):
        _lib.check(lib.pf_weighted_quantiles_d(_lib.dptr(v), _lib.dptr(w), _lib.device_dtype_code(w), v.numel(),
                                               _lib.dptr(p), p.numel(), _lib.dptr(out), _lib.current_stream(v)), lib)
    return out
