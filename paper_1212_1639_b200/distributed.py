"""One process per GPU: a particle-sharded filter driven over torch.distributed.

The reference's only parallelism is ``Backend`` lanes (backend.py:39-70) --
threads over contiguous lane ranges whose results do not depend on the lane
count (backend.py:1-8).  Its B200 counterpart at scale is one process per GPU:
rank r owns the N/world consecutive particle slots ``[r N/world, (r+1)
N/world)``, and every rank calls the same public function (SPMD)::

    dist.init_process_group("nccl")            # torchrun, one rank per GPU
    backend = parsmc.Backend("cuda", device=local_rank, process_group=dist.group.WORLD)
    out = parsmc.run_particle_learning(parsmc.Priors(), y, 1 << 27, seed=0, backend=backend)

Every rank returns the same outputs, bit-identical to one device (ancestors
and particles; moments within fp64 rounding of the single-device order).

Per time step the ranks exchange (pf_shard_* in include/parsmc_b200.h):

* an all-gather of one partial record per rank (global max log-weight and
  moment sums -- the reference's per-step reductions, filtering.py:288-300);
* an all-gather of one adder-tree subtree total per rank (the top of the
  reference's tree, prefix_sum.py:46-91);
* one barrier, after which rank 0 resolves the weighted quantiles.

The data-dependent reads of resampling (a slot's cut-point lookup and its
ancestor's 32-byte record, resampling.py:146-177) are direct loads from the
owning rank's memory through CUDA IPC mappings -- NVLink P2P between GPUs.
Under NCCL the collectives are enqueued on the engine's own CUDA stream, so
the host never waits inside the time loop; under gloo (CPU tests, or two
ranks sharing one GPU) each exchange round-trips through host memory.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from . import errors as _errors

PF_XCHG_PARTIAL = 0
PF_XCHG_TOTAL = 1


class _DevicePtr:
    """Zero-copy ``__cuda_array_interface__`` view of library-owned memory."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None, "stream": None}


def shard_slots(n, rank, world):
    """The slot range ``[lo, hi)`` rank ``rank`` owns of an ``n``-particle filter."""
    if world < 1 or world & (world - 1) or world > 8:
        raise ValueError("world size must be 1, 2, 4 or 8")
    ns = n // world
    return rank * ns, (rank + 1) * ns


class ShardRank:
    """This process's shard of one filter sharded over a process group.

    Same interface as :class:`~paper_1212_1639_b200.engine.Engine` for the
    driver in ``filtering.py``; :meth:`run_arrays` takes the full-size output
    arrays, fills the summaries on every rank and gathers the per-particle
    outputs (indices, final particles) from all ranks.
    """

    def __init__(self, cfg, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.device = int(cfg.device)
        self.h = C.c_void_p()
        self.cfg = cfg
        # creation is collective: a rank that fails still meets the others,
        # and every rank raises (none is left waiting in the peer exchange)
        err = None
        try:
            self.lib = _lib.require_device()
            _lib.check(self.lib.pf_shard_create(C.byref(cfg), self.rank, self.world, C.byref(self.h)), self.lib)
        except Exception as exc:  # noqa: BLE001 -- agreed on below
            err = exc
        self._raise_agreed(err, release=True)
        self._open_peers()
        try:
            self._bind_exchange()
        except Exception as exc:  # noqa: BLE001
            err = exc
        self._raise_agreed(err, release=True)

    # ---------------------------------------------------- rank agreement
    @staticmethod
    def _status_of(exc):
        if exc is None:
            return None
        return (type(exc), exc.args, getattr(exc, "step", None))

    @staticmethod
    def _rebuild(status):
        typ, args, step = status
        if step is not None and issubclass(typ, _errors.AllWeightsZeroError):
            return typ(step=step)
        try:
            return typ(*args)
        except Exception:  # noqa: BLE001 -- an exception type with another signature
            return _errors.DeviceError(f"{typ.__name__}: {args}")

    def _agreed_status(self, exc):
        """Every rank's status (None or its exception), exchanged before any
        data collective: the first failing rank's, or None when all ran."""
        allst = [None] * self.world
        self.dist.all_gather_object(allst, self._status_of(exc), group=self.group)
        return next((st for st in allst if st is not None), None)

    def _raise_agreed(self, exc, release=False):
        st = self._agreed_status(exc)
        if st is None:
            return
        if release:
            self._release_local()
        raise exc if exc is not None else self._rebuild(st)

    # ------------------------------------------------------------ set-up
    def _open_peers(self):
        err, mine = None, b""
        try:
            hb = int(self.lib.pf_shard_ipc_handle_bytes())
            h = np.zeros(hb, dtype=np.uint8)
            _lib.check(self.lib.pf_shard_ipc_handles(self.h, h.ctypes.data_as(C.c_void_p)), self.lib)
            mine = h.tobytes()
        except Exception as exc:  # noqa: BLE001
            err = exc
        allh = [None] * self.world
        self.dist.all_gather_object(allh, (mine, self._status_of(err)), group=self.group)
        bad = next((st for _, st in allh if st is not None), None)
        if bad is not None:
            self._release_local()
            raise err if err is not None else self._rebuild(bad)
        try:
            buf = np.frombuffer(b"".join(m for m, _ in allh), dtype=np.uint8).copy()
            _lib.check(self.lib.pf_shard_open_peers(self.h, buf.ctypes.data_as(C.c_void_p)), self.lib)
        except Exception as exc:  # noqa: BLE001
            err = exc
        # doubles as the barrier: every rank has mapped its peers before any
        # rank starts a run
        self._raise_agreed(err, release=True)

    def _bind_exchange(self):
        self.slot = {}
        self.dptr = {}
        for which in (PF_XCHG_PARTIAL, PF_XCHG_TOTAL):
            p = C.c_void_p()
            sb = C.c_int64()
            _lib.check(self.lib.pf_shard_exchange(self.h, which, C.byref(p), C.byref(sb)), self.lib)
            self.slot[which] = sb.value
            self.dptr[which] = p.value
        if self.nccl:
            import torch

            s = C.c_void_p()
            _lib.check(self.lib.pf_shard_stream(self.h, C.byref(s)), self.lib)
            dev = torch.device("cuda", self.device)
            self.stream = torch.cuda.ExternalStream(s.value, device=dev)
            self.xbuf = {w: torch.as_tensor(_DevicePtr(self.dptr[w], self.slot[w] * self.world), device=dev)
                         for w in self.dptr}
            self.token = torch.zeros(1, dtype=torch.int32, device=dev)
        else:
            import torch

            self.xhost = {w: torch.zeros(self.slot[w] * self.world, dtype=torch.uint8) for w in self.slot}

    def reconfigure(self, cfg):
        _lib.check(self.lib.pf_shard_reconfigure(self.h, C.byref(cfg)), self.lib)
        self.cfg = cfg

    # ---------------------------------------------------------- exchange
    def _all_gather(self, which):
        sb = self.slot[which]
        lo = self.rank * sb
        if self.nccl:
            buf = self.xbuf[which]
            self.dist.all_gather_into_tensor(buf, buf[lo:lo + sb], group=self.group)
        else:
            buf = self.xhost[which]
            mine = buf[lo:lo + sb]
            _lib.check(self.lib.pf_shard_exchange_host(self.h, which, 1, C.c_void_p(mine.data_ptr())), self.lib)
            parts = list(buf.split(sb))
            self.dist.all_gather(parts, mine.clone(), group=self.group)
            _lib.check(self.lib.pf_shard_exchange_host(self.h, which, 0, C.c_void_p(buf.data_ptr())), self.lib)

    def _barrier(self):
        if self.nccl:
            self.dist.all_reduce(self.token, group=self.group)
        else:
            _lib.check(self.lib.pf_shard_synchronize(self.h), self.lib)
            self.dist.barrier(group=self.group)

    def _phase(self, k, t):
        _lib.check(self.lib.pf_shard_phase(self.h, k, t), self.lib)

    def _loop(self, y, out):
        t_len = len(y)
        rc = self.lib.pf_shard_begin(self.h, _lib.ptr(y), t_len, C.byref(out))
        if rc:
            # keep the ranks in step: a bad input fails on every rank alike
            _lib.check(rc, self.lib)
        for t in range(1, t_len + 1):
            self._phase(1, t)
            self._all_gather(PF_XCHG_PARTIAL)
            self._phase(2, t)
            self._all_gather(PF_XCHG_TOTAL)
            self._phase(3, t)
            self._barrier()
            self._phase(4, t)
        # rank 0's resolve of step T reads every rank's last particles
        self._barrier()
        return self.lib.pf_shard_finish(self.h)

    # --------------------------------------------------------------- run
    def run(self, y, outputs, feed=None):
        """Run with a caller-built ``PfOutputs`` holding THIS rank's slots."""
        if feed is not None:
            raise NotImplementedError("oracle feeds are not supported by sharded runs")
        y = np.ascontiguousarray(y, dtype=np.float64)
        if self.nccl:
            import torch

            with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                rc = self._loop(y, outputs)
        else:
            rc = self._loop(y, outputs)
        _lib.check(rc, self.lib)

    def run_arrays(self, y, arrays, n):
        """Run, then give every rank the full outputs in ``arrays`` (the
        full-size dict ``filtering._alloc_outputs`` builds)."""
        t_len = len(y)
        lo, hi = shard_slots(n, self.rank, self.world)
        ns = hi - lo
        out = _lib.PfOutputs()
        local = {}
        for k, v in arrays.items():
            if k == "indices":
                local[k] = np.empty((t_len, ns), dtype=np.int64)
            elif k.startswith("final_"):
                local[k] = np.empty(ns)
            elif self.rank == 0:
                local[k] = v
        for k, v in local.items():
            setattr(out, k, _lib.ptr(v, C.c_int64 if v.dtype == np.int64 else C.c_double))
        status = None
        try:
            self.run(y, out)
        except Exception as exc:  # noqa: BLE001 -- re-raised on every rank below
            status = exc
        # every rank enters the agreement whatever happened locally; if any
        # rank failed, every rank raises (rank 0's resolve / finish included)
        self._raise_agreed(status)
        self._publish(arrays, local, t_len, ns)

    def _publish(self, arrays, local, t_len, ns):
        import torch

        dev = torch.device("cuda", self.device) if self.nccl else torch.device("cpu")
        summaries = sorted(k for k in arrays if k != "indices" and not k.startswith("final_"))
        if summaries:
            flat = np.concatenate([arrays[k].ravel() for k in summaries]) if self.rank == 0 else \
                np.empty(sum(arrays[k].size for k in summaries))
            tb = torch.from_numpy(flat).to(dev)
            self.dist.broadcast(tb, src=0, group=self.group)
            flat = tb.cpu().numpy()
            off = 0
            for k in summaries:
                sz = arrays[k].size
                arrays[k][...] = flat[off:off + sz].reshape(arrays[k].shape)
                off += sz
        for k, v in local.items():
            if k != "indices" and not k.startswith("final_"):
                continue
            src = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
            parts = [torch.empty_like(src) for _ in range(self.world)]
            self.dist.all_gather(parts, src, group=self.group)
            for r, p in enumerate(parts):
                if k == "indices":
                    arrays[k][:, r * ns:(r + 1) * ns] = p.cpu().numpy()
                else:
                    arrays[k][r * ns:(r + 1) * ns] = p.cpu().numpy()

    def last_timing(self):
        tot = C.c_double()
        _lib.check(self.lib.pf_shard_last_timing(self.h, C.byref(tot)), self.lib)
        return {"total_ms": tot.value}

    def close(self):
        """Collective teardown (explicit ``close`` / ``Backend.close`` /
        ``with``, called by every rank): unmap the peers, meet the other
        ranks, then free -- no rank frees memory a peer still maps."""
        if self.h:
            self.lib.pf_shard_close_peers(self.h)
            if self.dist.is_initialized():
                self.dist.barrier(group=self.group)
            self.lib.pf_shard_destroy(self.h)
            self.h = C.c_void_p()

    def release(self):
        """Non-collective teardown (garbage collection): a barrier here could
        pair with an unrelated collective on a peer, so only this rank's
        mappings of its peers are dropped and its own memory is left to the
        process exit (a peer may still map it)."""
        self._release_local()

    def _release_local(self):
        if getattr(self, "h", None):
            try:
                self.lib.pf_shard_close_peers(self.h)
            finally:
                self.h = C.c_void_p()

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass
