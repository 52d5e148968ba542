"""ctypes binding of libparsmc_b200.so (the C ABI in include/parsmc_b200.h).

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``).
There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import (
    AllWeightsZeroError,
    DeviceError,
    NonFiniteWeightError,
    NotPowerOfTwoError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libparsmc_b200.so")
# PARSMC_B200_LIB: load a variant build instead (A/B experiments; scripts/)
LIB_PATH = os.environ.get("PARSMC_B200_LIB", LIB_PATH)

PF_OK = 0
PF_ERR_ALL_WEIGHTS_ZERO = 1
PF_ERR_NON_FINITE_WEIGHT = 2
PF_ERR_NOT_POWER_OF_TWO = 3
PF_ERR_VALUE = 4
PF_ERR_CUDA = 5
PF_ERR_OUT_OF_MEMORY = 6
PF_ERR_NOT_IMPLEMENTED = 7
PF_DTYPE_F64 = 0
PF_DTYPE_F32 = 1
RESAMPLER_CODES = {"cutpoint": 0, "naive": 1, "sorted": 2, "stratified": 3, "systematic": 4, "spacings": 5}

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p


class PfConfig(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("seed", C.c_uint64),
        ("learn", C.c_int32), ("learn_sigma2", C.c_int32), ("learn_tau2", C.c_int32),
        ("precision", C.c_int32),
        ("x0_mean", C.c_double), ("x0_var", C.c_double), ("sqrt_x0_var", C.c_double),
        ("sigma2_shape", C.c_double), ("sigma2_scale", C.c_double),
        ("tau2_shape", C.c_double), ("tau2_scale", C.c_double),
        ("sigma2_fixed", C.c_double), ("tau2_fixed", C.c_double),
        ("sqrt_tau2_fixed", C.c_double), ("log_term_fixed", C.c_double),
        ("track_quantiles", C.c_int32), ("keep_indices", C.c_int32),
        ("keep_final", C.c_int32), ("store_particles", C.c_int32),
        ("phase_timing", C.c_int32), ("gamma_method", C.c_int32),
        ("device", C.c_int32), ("resampler", C.c_int32),
    ]


class PfFeed(C.Structure):
    _fields_ = [("z", _dp), ("g_sigma", _dp), ("g_tau", _dp), ("w", _dp)]


class PfOutputs(C.Structure):
    _fields_ = [
        ("filtered_mean", _dp), ("filtered_quantiles", _dp),
        ("sigma2_mean", _dp), ("sigma2_sd", _dp), ("sigma2_quantiles", _dp),
        ("tau2_mean", _dp), ("tau2_sd", _dp), ("tau2_quantiles", _dp),
        ("indices", _i64p),
        ("final_states", _dp), ("final_sigma2", _dp), ("final_tau2", _dp),
        ("final_a_sigma", _dp), ("final_b_sigma", _dp), ("final_a_tau", _dp),
        ("final_b_tau", _dp),
        ("hist_states", _dp), ("hist_sigma2", _dp), ("hist_tau2", _dp),
        ("hist_a_sigma", _dp), ("hist_b_sigma", _dp), ("hist_a_tau", _dp),
        ("hist_b_tau", _dp),
        ("phase_ns", C.c_int64 * 7), ("failed_step", C.c_int64),
        ("ess", _dp),
    ]


# name -> (restype, argtypes); the exported symbol set of include/parsmc_b200.h
SIGNATURES = {
    "pf_version": (C.c_char_p, []),
    "pf_last_error_message": (C.c_char_p, []),
    "pf_abi_sizes": (C.c_int, [_i64p]),
    "pf_last_error_step": (C.c_int64, []),
    "pf_device_count": (C.c_int, []),
    "pf_launch_count": (C.c_int64, []),
    "pf_engine_create": (C.c_int, [C.POINTER(PfConfig), C.POINTER(C.c_void_p)]),
    "pf_engine_reconfigure": (C.c_int, [C.c_void_p, C.POINTER(PfConfig)]),
    "pf_engine_run": (C.c_int, [C.c_void_p, _dp, C.c_int64, C.POINTER(PfFeed), C.POINTER(PfOutputs)]),
    "pf_engine_run_resident": (C.c_int, [C.c_void_p, C.c_int64]),
    "pf_engine_run_batch": (C.c_int, [C.c_void_p, _u64p, C.c_int32, _dp, C.c_int64, C.POINTER(PfOutputs)]),
    "pf_engine_last_timing": (C.c_int, [C.c_void_p, _dp, _dp, _i64p, _i64p]),
    "pf_engine_quantile_stats": (C.c_int, [C.c_void_p, _i64p]),
    "pf_engine_last_path": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "pf_engine_destroy": (C.c_int, [C.c_void_p]),
    "pf_group_create": (C.c_int, [C.POINTER(PfConfig), C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p)]),
    "pf_group_reconfigure": (C.c_int, [C.c_void_p, C.POINTER(PfConfig)]),
    "pf_group_run": (C.c_int, [C.c_void_p, _dp, C.c_int64, C.POINTER(PfOutputs)]),
    "pf_group_last_timing": (C.c_int, [C.c_void_p, _dp]),
    "pf_group_destroy": (C.c_int, [C.c_void_p]),
    "pf_shard_create": (C.c_int, [C.POINTER(PfConfig), C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "pf_shard_reconfigure": (C.c_int, [C.c_void_p, C.POINTER(PfConfig)]),
    "pf_shard_ipc_handle_bytes": (C.c_int32, []),
    "pf_shard_ipc_handles": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pf_shard_open_peers": (C.c_int, [C.c_void_p, C.c_void_p]),
    "pf_shard_exchange": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), _i64p]),
    "pf_shard_exchange_host": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "pf_shard_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "pf_shard_synchronize": (C.c_int, [C.c_void_p]),
    "pf_shard_begin": (C.c_int, [C.c_void_p, _dp, C.c_int64, C.POINTER(PfOutputs)]),
    "pf_shard_phase": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    "pf_shard_finish": (C.c_int, [C.c_void_p]),
    "pf_shard_last_timing": (C.c_int, [C.c_void_p, _dp]),
    "pf_shard_close_peers": (C.c_int, [C.c_void_p]),
    "pf_shard_destroy": (C.c_int, [C.c_void_p]),
    "pf_philox_block": (C.c_int, [C.c_uint64, _u64p, C.c_int64, C.c_uint64, _u64p]),
    "pf_philox4x64": (C.c_int, [_u64p, _u64p, C.c_int64, _u64p]),
    "pf_uniforms_at": (C.c_int, [C.c_uint64, _u64p, _u64p, C.c_int64, _dp]),
    "pf_ndtri": (C.c_int, [_dp, C.c_int64, _dp]),
    "pf_ndtri_table": (C.c_int, [_dp, C.c_int64, _dp]),
    "pf_gammaincinv": (C.c_int, [C.c_double, _dp, C.c_int64, C.c_int32, _dp]),
    "pf_tree_cdf": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, _dp]),
    "pf_adder_tree": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    "pf_cut_table": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, _i64p]),
    "pf_cutpoint_lookup": (C.c_int, [C.c_void_p, _i64p, C.c_int64, C.c_int32, _dp, C.c_int64, _i64p]),
    "pf_merge_indices": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, _dp, C.c_int64, C.c_int32, _i64p]),
    "pf_resample_cutpoint": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_uint64, _i64p]),
    "pf_weighted_quantiles": (C.c_int, [_dp, C.c_void_p, C.c_int32, C.c_int64, _dp, C.c_int32, _dp]),
    # device-pointer forms: every pointer is device memory, last arg the stream
    "pf_uniforms_at_d": (C.c_int, [C.c_uint64, _vp, _vp, C.c_int64, _vp, _vp]),
    "pf_tree_cdf_d": (C.c_int, [_vp, C.c_int64, C.c_int32, _vp, _vp, _vp]),
    "pf_cut_table_d": (C.c_int, [_vp, C.c_int64, C.c_int32, _vp, _vp]),
    "pf_cutpoint_lookup_d": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp, C.c_int64, _vp, _vp]),
    "pf_resample_cutpoint_d": (C.c_int, [_vp, C.c_int64, C.c_int32, C.c_uint64, C.c_uint64, _vp, _vp]),
    "pf_weighted_quantiles_d": (C.c_int, [_vp, _vp, C.c_int32, C.c_int64, _vp, C.c_int32, _vp, _vp]),
}

_lib = None


def load():
    """Load the C-ABI library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: build it with `make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def device_count():
    return int(load().pf_device_count())


def require_device():
    lib = load()
    if lib.pf_device_count() < 1:
        raise DeviceError("no CUDA device visible: the parsmc-b200 engine runs only on the GPU")
    return lib


def check(rc, lib=None):
    """Map a C status code onto the reference's exception classes."""
    if rc == PF_OK:
        return
    lib = lib or load()
    msg = (lib.pf_last_error_message() or b"").decode()
    step = int(lib.pf_last_error_step())
    if rc == PF_ERR_ALL_WEIGHTS_ZERO:
        if step > 0:
            raise AllWeightsZeroError(step=step)
        if "not finite" in msg:
            raise AllWeightsZeroError("weight total is not finite")
        raise AllWeightsZeroError()
    if rc == PF_ERR_NON_FINITE_WEIGHT:
        raise NonFiniteWeightError(msg)
    if rc == PF_ERR_NOT_POWER_OF_TWO:
        raise NotPowerOfTwoError(msg)
    if rc == PF_ERR_VALUE:
        raise ValueError(msg)
    if rc == PF_ERR_NOT_IMPLEMENTED:
        raise NotImplementedError(msg)
    if rc == PF_ERR_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise DeviceError(f"CUDA error: {msg}")


def ptr(a, ctype=C.c_double):
    """Data pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def vptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def dtype_code(dt):
    dt = np.dtype(dt)
    if dt == np.float64:
        return PF_DTYPE_F64
    if dt == np.float32:
        return PF_DTYPE_F32
    raise TypeError(f"unsupported dtype {dt}")


def is_cuda_tensor(x):
    """True for a torch tensor on a CUDA device (checked without importing
    torch when the caller never did)."""
    return type(x).__module__.startswith("torch") and bool(getattr(x, "is_cuda", False))


def dptr(t):
    """Device pointer of a contiguous torch CUDA tensor (or None)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def current_stream(t):
    """The torch current stream of t's device, as the void* the *_d entries take."""
    import torch

    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def device_dtype_code(t):
    import torch

    if t.dtype == torch.float64:
        return PF_DTYPE_F64
    if t.dtype == torch.float32:
        return PF_DTYPE_F32
    raise TypeError(f"expected a float32 or float64 tensor, got {t.dtype}")
