"""Counter-based Philox4x64-10 streams, evaluated on the device.

Same contract as the reference (rng.py:1-13): every uniform is a pure
function of (seed, stream_id, counter); draw k of a stream is word k & 3 of
the Philox block with counter (k >> 2, 0, 0, 0) and key (seed, stream_id),
mapped to ((w >> 12) + 1/2) 2^-52.  The words are bit-identical to the
reference's and to ``numpy.random.Philox`` (tests/test_gpu_kernels.py).
Inside the filter loop the engine evaluates Philox in registers of the fused
step kernel; the classes here serve the kernel-level API.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib

AUX_STREAM_BASE = 1 << 62  # rng.py:34


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def philox4x64_block(c0, c1, c2, c3, k0, k1):
    """Philox4x64-10 on arbitrary (broadcastable) counters and keys
    (rng.py:49-63); returns four uint64 word arrays."""
    arrs = np.broadcast_arrays(*(np.asarray(v, dtype=np.uint64) for v in (c0, c1, c2, c3, k0, k1)))
    shape = arrs[0].shape
    n = int(np.prod(shape)) if shape else 1
    ctr = np.ascontiguousarray(np.stack([a.reshape(-1) for a in arrs[:4]]))
    key = np.ascontiguousarray(np.stack([a.reshape(-1) for a in arrs[4:]]))
    out = np.empty((4, n), dtype=np.uint64)
    lib = _lib.require_device()
    _lib.check(lib.pf_philox4x64(_lib.ptr(ctr, _lib.C.c_uint64), _lib.ptr(key, _lib.C.c_uint64), n,
                                 _lib.ptr(out, _lib.C.c_uint64)), lib)
    return tuple(out[i].reshape(shape) for i in range(4))


def philox_block_lanes(block, seed, stream_ids):
    """Four words per stream id at one shared block counter (rng.py:103-110)."""
    ids = _u64(stream_ids)
    out = np.empty((4, len(ids)), dtype=np.uint64)
    lib = _lib.require_device()
    _lib.check(lib.pf_philox_block(np.uint64(seed), _lib.ptr(ids, _lib.C.c_uint64), len(ids),
                                   np.uint64(block), _lib.ptr(out, _lib.C.c_uint64)), lib)
    return out


def uniforms_at(seed, stream_ids, counters):
    """Uniform(0,1) draw for each (stream_id, counter) pair (rng.py:122-140).
    CUDA-tensor stream ids run on the device stream (device_ops)."""
    if _lib.is_cuda_tensor(stream_ids):
        from . import device_ops

        return device_ops.uniforms_at(seed, stream_ids, counters)
    ids, ctr = np.broadcast_arrays(np.asarray(stream_ids, dtype=np.uint64),
                                   np.asarray(counters, dtype=np.uint64))
    shape = ids.shape
    ids, ctr = _u64(ids.reshape(-1)), _u64(ctr.reshape(-1))
    out = np.empty(len(ids))
    lib = _lib.require_device()
    _lib.check(lib.pf_uniforms_at(np.uint64(seed), _lib.ptr(ids, _lib.C.c_uint64),
                                  _lib.ptr(ctr, _lib.C.c_uint64), len(ids), _lib.ptr(out)), lib)
    return out.reshape(shape)


def ndtri(u, method="exact"):
    """Standard-normal quantile on the device (scipy.special.ndtri as the
    reference calls it, rng.py:223-224).  ``method="exact"`` is the Cephes
    restatement, ``"table"`` the piecewise table the hot path evaluates."""
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    out = np.empty_like(u)
    lib = _lib.require_device()
    fn = lib.pf_ndtri if method == "exact" else lib.pf_ndtri_table
    _lib.check(fn(_lib.ptr(u.reshape(-1)), u.size, _lib.ptr(out.reshape(-1))), lib)
    return out


def gammaincinv(a, u, method="table"):
    """Gamma(a, 1) quantile on the device (scipy.special.gammaincinv as used
    at rng.py:226-229).  ``method="table"`` is the hot-path per-shape table,
    ``"accurate"`` the Halley solver the table is fitted to."""
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    a_arr = np.asarray(a, dtype=np.float64)
    a_b, u_b = np.broadcast_arrays(a_arr, u)
    out = np.empty(u_b.shape)
    lib = _lib.require_device()
    code = 0 if method == "table" else 1
    flat_a = a_b.reshape(-1)
    flat_u = np.ascontiguousarray(u_b.reshape(-1))
    flat_o = out.reshape(-1)
    for shape in np.unique(flat_a):
        sel = flat_a == shape
        uu = np.ascontiguousarray(flat_u[sel])
        gg = np.empty_like(uu)
        _lib.check(lib.pf_gammaincinv(float(shape), _lib.ptr(uu), len(uu), code, _lib.ptr(gg)), lib)
        flat_o[sel] = gg
    return out


def _to_unit_open(word):
    """(w >> 12 + 1/2) 2^-52 (rng.py:113-119); host helper for tests."""
    return ((np.asarray(word, dtype=np.uint64) >> np.uint64(12)).astype(np.float64) + 0.5) * 2.0**-52


@dataclass
class RngStream:
    """A single counter-based stream (rng.py:143-172)."""

    seed: int
    stream_id: int = 0
    counter: int = 0

    def uniform(self):
        u = uniforms_at(self.seed, [self.stream_id], [self.counter])
        self.counter += 1
        return float(u[0])

    def uniforms(self, n):
        ctr = np.uint64(self.counter) + np.arange(n, dtype=np.uint64)
        self.counter += int(n)
        return uniforms_at(self.seed, np.uint64(self.stream_id), ctr)

    def normal(self):
        return float(ndtri(np.array([self.uniform()]))[0])

    def normals(self, n):
        return ndtri(self.uniforms(n))

    def advance(self, n):
        self.counter += int(n)
        return self


@dataclass
class StreamArray:
    """One stream per particle lane, advancing in lockstep (rng.py:175-233)."""

    seed: int
    stream_ids: np.ndarray
    counters: np.ndarray
    _unused: int = field(default=0, repr=False)

    @classmethod
    def for_lanes(cls, seed, n, counter=0):
        return cls(seed=int(seed), stream_ids=np.arange(n, dtype=np.uint64),
                   counters=np.full(n, counter, dtype=np.uint64))

    def __len__(self):
        return len(self.stream_ids)

    def uniforms(self):
        u = uniforms_at(self.seed, self.stream_ids, self.counters)
        self.counters = self.counters + np.uint64(1)
        return u

    def normals(self):
        return ndtri(self.uniforms())

    def inverse_gammas(self, shape, scale):
        """scale / Gamma^-1(shape, u): inverse-gamma draws (rng.py:226-229)."""
        return scale / gammaincinv(shape, self.uniforms())

    def skip(self, n):
        self.counters = self.counters + np.uint64(n)
        return self

    def lockstep_counter(self):
        c = int(self.counters[0]) if len(self.counters) else 0
        if len(self.counters) and int(self.counters[-1]) != c:
            return None
        if len(self.counters) and not (self.counters == self.counters[0]).all():
            return None
        return c
