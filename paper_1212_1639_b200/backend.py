"""Execution backend: the seam through which callers select the device.

The reference's ``Backend(mode, lanes, min_chunk)`` (backend.py:15-82) owns a
thread pool of CPU worker lanes.  Here the same object owns the *device
engines*: one resident particle system per (model, n, seed, flags)
configuration, reused across calls until ``close()``.  Every mode runs on the
GPU -- ``"sequential"`` / ``"parallel"`` are accepted so existing callers are
drop-in, and because the reference's results never depend on the lane count
(backend.py:1-8) mapping them onto the device preserves its semantics.
``lanes`` and ``min_chunk`` keep their meaning for ``split``.
"""

from __future__ import annotations

from . import _lib

MODES = ("cuda", "sequential", "parallel")


class Backend:
    """Device engine owner.

    Parameters
    ----------
    mode : {"cuda", "sequential", "parallel"}
        All modes execute on the CUDA device.
    lanes : int
        Kept for API compatibility (``split``); has no effect on results.
    min_chunk : int
        Kept for API compatibility (``split``).
    device : int
        CUDA device ordinal.
    shards : int
        Split one filter's particles into this many shards (1, 2, 4, 8) of
        consecutive slots -- the multi-GPU run of SURVEY §8e.  Results are
        bit-identical to one shard in ancestors and particles.
    devices : sequence of int, optional
        Device of each shard (default: all on ``device``); distinct devices
        must have peer access (NVLink / NVSwitch).
    process_group : torch.distributed group or True, optional
        One process per GPU: every rank of the group calls the same function
        with the same arguments (SPMD) and owns ``n / world`` consecutive
        particle slots on ``device``; all ranks return the full outputs
        (``distributed.py``).  ``True`` means the default group.
    """

    def __init__(self, mode="cuda", lanes=1, min_chunk=4096, device=0, shards=1, devices=None,
                 process_group=None):
        if mode not in MODES:
            raise ValueError(f"unknown backend mode: {mode!r}")
        if lanes < 1:
            raise ValueError("lanes must be >= 1")
        shards = int(shards)
        if shards not in (1, 2, 4, 8):
            raise ValueError("shards must be 1, 2, 4 or 8")
        if devices is not None:
            devices = [int(d) for d in devices]
            if len(devices) != shards:
                raise ValueError("devices must list one device per shard")
        self.mode = mode
        self.lanes = lanes if mode == "parallel" else 1
        self.min_chunk = min_chunk
        self.device = int(device)
        self.shards = shards
        self.devices = devices if devices is not None else [self.device] * shards
        self.process_group = None
        if process_group is not None and process_group is not False:
            if shards != 1 or devices is not None:
                raise ValueError("process_group and shards/devices are exclusive")
            import torch.distributed as dist

            if not dist.is_initialized():
                raise ValueError("process_group needs an initialised torch.distributed process group")
            self.process_group = None if process_group is True else process_group
            self.world = dist.get_world_size(self.process_group)
            self.rank = dist.get_rank(self.process_group)
        self.distributed = process_group is not None and process_group is not False
        self._engines = {}
        self._pool = None

    def split(self, n):
        """Contiguous lane ranges covering [0, n) (backend.py:39-50)."""
        k = min(self.lanes, max(1, n // self.min_chunk))
        base, extra = divmod(n, k)
        out, lo = [], 0
        for i in range(k):
            hi = lo + base + (1 if i < extra else 0)
            if hi > lo:
                out.append((lo, hi))
            lo = hi
        return out

    def run(self, n, fn):
        """Invoke ``fn(lo, hi)`` over disjoint ranges covering [0, n)
        (backend.py:52-70): the host-side seam reference callers drive
        directly.  Returns only once every lane has finished (the phase
        barrier), and re-raises a lane's exception.  ``fn`` is the caller's
        own host code; the device engines never go through it."""
        if n <= 0:
            return
        ranges = self.split(n)
        if self.mode != "parallel" or len(ranges) == 1:
            for lo, hi in ranges:
                fn(lo, hi)
            return
        if self._pool is None:
            from concurrent.futures import ThreadPoolExecutor

            self._pool = ThreadPoolExecutor(max_workers=self.lanes)
        futures = [self._pool.submit(fn, lo, hi) for lo, hi in ranges]
        for f in futures:
            f.result()  # waits for every lane; re-raises lane exceptions in order

    def engine(self, key, factory):
        """The cached engine for ``key`` (created by ``factory()`` once)."""
        eng = self._engines.get(key)
        if eng is None:
            eng = factory()
            self._engines[key] = eng
        return eng

    def close(self):
        for eng in self._engines.values():
            eng.close()
        self._engines.clear()
        if self._pool is not None:
            self._pool.shutdown(wait=True)
            self._pool = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        # garbage collection runs at different times on different ranks: no
        # collective teardown here (ShardRank.release is rank-local)
        try:
            for eng in self._engines.values():
                (getattr(eng, "release", None) or eng.close)()
            self._engines.clear()
            if self._pool is not None:
                self._pool.shutdown(wait=False)
        except Exception:
            pass

    def __repr__(self):
        tail = f", rank={self.rank}/{self.world}" if self.distributed else ""
        return (f"Backend(mode={self.mode!r}, lanes={self.lanes}, device={self.device}, "
                f"shards={self.shards}{tail})")


def device_available():
    """True when the C-ABI library loads and sees a CUDA device."""
    try:
        return _lib.device_count() > 0
    except Exception:
        return False
