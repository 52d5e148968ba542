"""Python handle on the device engine (pf_engine_* in include/parsmc_b200.h)."""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .models import LOG_TWO_PI


def make_config(n, seed, *, learn, learn_sigma2, learn_tau2, precision, x0_mean, x0_var,
                sigma2_shape=0.0, sigma2_scale=0.0, tau2_shape=0.0, tau2_scale=0.0,
                sigma2_fixed=1.0, tau2_fixed=1.0, track_quantiles=False, keep_indices=False,
                keep_final=False, store_particles=False, phase_timing=True, gamma_method=0,
                device=0, resampler="cutpoint"):
    """Fill a pf_config; scalar terms the reference computes with numpy on the
    host (np.sqrt(tau2), np.log(sigma2)) are computed here the same way so the
    device sees identical bits."""
    c = _lib.PfConfig()
    c.n = int(n)
    c.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    c.learn = int(bool(learn))
    c.learn_sigma2 = int(bool(learn_sigma2))
    c.learn_tau2 = int(bool(learn_tau2))
    c.precision = _lib.PF_DTYPE_F32 if precision == "single" else _lib.PF_DTYPE_F64
    c.x0_mean = float(x0_mean)
    c.x0_var = float(x0_var)
    c.sqrt_x0_var = math.sqrt(x0_var)                                    # filtering.py:235
    c.sigma2_shape, c.sigma2_scale = float(sigma2_shape), float(sigma2_scale)
    c.tau2_shape, c.tau2_scale = float(tau2_shape), float(tau2_scale)
    c.sigma2_fixed = float(sigma2_fixed)
    c.tau2_fixed = float(tau2_fixed)
    c.sqrt_tau2_fixed = float(np.sqrt(float(tau2_fixed)))                # filtering.py:274
    c.log_term_fixed = float(-0.5 * (LOG_TWO_PI + np.log(float(sigma2_fixed))))  # filtering.py:293
    c.track_quantiles = int(bool(track_quantiles))
    c.keep_indices = int(bool(keep_indices))
    c.keep_final = int(bool(keep_final))
    c.store_particles = int(bool(store_particles))
    c.phase_timing = int(bool(phase_timing))
    c.gamma_method = int(gamma_method)
    c.device = int(device)
    c.resampler = _lib.RESAMPLER_CODES[resampler]
    return c


class Engine:
    """One device-resident particle system of ``n`` slots."""

    def __init__(self, cfg):
        self.lib = _lib.require_device()
        self.h = C.c_void_p()
        _lib.check(self.lib.pf_engine_create(C.byref(cfg), C.byref(self.h)), self.lib)
        self.cfg = cfg

    def reconfigure(self, cfg):
        _lib.check(self.lib.pf_engine_reconfigure(self.h, C.byref(cfg)), self.lib)
        self.cfg = cfg

    def run(self, y, outputs, feed=None):
        y = np.ascontiguousarray(y, dtype=np.float64)
        fd = None
        if feed is not None:
            fd = _lib.PfFeed()
            for k in ("z", "g_sigma", "g_tau", "w"):
                a = feed.get(k)
                setattr(fd, k, None if a is None else _lib.ptr(a))
        rc = self.lib.pf_engine_run(self.h, _lib.ptr(y), len(y),
                                    None if fd is None else C.byref(fd), C.byref(outputs))
        _lib.check(rc, self.lib)

    def run_batch(self, seeds, y, outputs):
        """``len(seeds)`` independent replications in one launch sequence
        (pf_engine_run_batch); outputs hold [R][T] rows."""
        y = np.ascontiguousarray(y, dtype=np.float64)
        sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        rc = self.lib.pf_engine_run_batch(self.h, _lib.ptr(sd, C.c_uint64), len(sd), _lib.ptr(y), len(y),
                                          C.byref(outputs))
        _lib.check(rc, self.lib)

    def run_resident(self, t_len):
        _lib.check(self.lib.pf_engine_run_resident(self.h, int(t_len)), self.lib)

    def last_timing(self):
        tot, step = C.c_double(), C.c_double()
        nsteps, nk = C.c_int64(), C.c_int64()
        _lib.check(self.lib.pf_engine_last_timing(self.h, C.byref(tot), C.byref(step),
                                                  C.byref(nsteps), C.byref(nk)), self.lib)
        return {"total_ms": tot.value, "step_kernel_ms": step.value,
                "step_kernel_launches": nsteps.value, "kernels": nk.value}

    def quantile_stats(self):
        s = (C.c_int64 * 4)()
        _lib.check(self.lib.pf_engine_quantile_stats(self.h, s), self.lib)
        return {"unresolved": s[0], "fallbacks": s[1], "max_candidates": s[2], "resolves": s[3]}

    PATH_FLAGS = {"fused_draws": 1, "rank_tables": 2, "fused_top": 4}

    def last_path(self):
        """Kernel path of the last run (pf_engine_last_path): which of the
        benchmarked variants actually executed."""
        f = C.c_int32()
        _lib.check(self.lib.pf_engine_last_path(self.h, C.byref(f)), self.lib)
        return {k: bool(f.value & b) for k, b in self.PATH_FLAGS.items()}

    def close(self):
        if self.h:
            self.lib.pf_engine_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Group:
    """One filter sharded over several devices (pf_group_* in the C ABI)."""

    def __init__(self, cfg, devices):
        self.lib = _lib.require_device()
        self.h = C.c_void_p()
        devs = (C.c_int32 * len(devices))(*devices)
        _lib.check(self.lib.pf_group_create(C.byref(cfg), len(devices), devs, C.byref(self.h)), self.lib)
        self.cfg = cfg
        self.devices = list(devices)

    def reconfigure(self, cfg):
        _lib.check(self.lib.pf_group_reconfigure(self.h, C.byref(cfg)), self.lib)
        self.cfg = cfg

    def run(self, y, outputs, feed=None):
        if feed is not None:
            raise NotImplementedError("oracle feeds are not supported by sharded runs")
        y = np.ascontiguousarray(y, dtype=np.float64)
        _lib.check(self.lib.pf_group_run(self.h, _lib.ptr(y), len(y), C.byref(outputs)), self.lib)

    def last_timing(self):
        tot = C.c_double()
        _lib.check(self.lib.pf_group_last_timing(self.h, C.byref(tot)), self.lib)
        return {"total_ms": tot.value}

    def close(self):
        if self.h:
            self.lib.pf_group_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
