"""Benchmark: particle-steps/s (N*T/s) of the full particle-learning cycle.

Workload (BASELINE.json configs[2]): the paper's trend+noise model, particle
learning of sigma2 and tau2 with Priors() (IG(5,4), IG(5,0.4), x0~N(0,10)),
N = 2^24 particles, T = 1000 synthetic observations simulated from aux
stream 2^62+1 (bench.py:36 of the reference), seed 0, cut-point resampler,
fp64, track_quantiles=False -- exactly the reference bench's par_cutpoint
cell (bench.py:28-34,130-143), so parameter mean/sd/5 quantiles are computed
every step.  One bench "step" = one complete filter run (init + T time
steps).  State arrays (2 x 512 MiB records + 128 MiB log-weights ...) are
far larger than the 126 MB L2, so no explicit flush is needed.

  value  = N*T*K / (device time of K resident runs, CUDA events), max over ranks
  e2e    = same metric through the public API run_particle_learning() with a
           host y and host outputs (host->device and device->host inside)
  --impl reference  times the reference's CPU algorithm (oracle port, numpy +
           scipy, all host threads as Backend lanes) on a bounded sample.

Multi-GPU (--gpus N under torchrun, N > 1): ONE filter of --n-shard particles
(default N x 2^24, so 2^24 per GPU as at N = 1; N = 8 is BASELINE configs[3],
2^27) sharded over the N GPUs, one process per GPU (distributed.py /
pf_shard_*): per step an NCCL all-gather of one partial record and one
subtree total per rank plus one barrier, all enqueued on the engine's stream,
and cross-rank resampling reads through CUDA IPC (NVLink P2P).  value =
N_particles*T*K / max over ranks of the device time.  Work per GPU is fixed
as N grows: scaling "weak" (pass --n-shard for a fixed total, "strong").
--multi replicas instead runs an independent filter per rank.  --shards G
runs G shards on one GPU from one process (pf_group_*, the same kernels).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALG_BYTES_STEP_KERNEL = 84  # lookup 12 + gather 32 + write 32 + log-weight 8
ALG_BYTES_CYCLE = 112       # whole PL cycle per particle-step


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > i + 2 and r[i + 2].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(force=False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or force:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch.distributed as dist

    if world > 1 or dist.is_initialized():
        import torch.distributed as dist

        dist.barrier()


def cpu_reference_run(n, t_len, lanes):
    """The reference's par_cutpoint cell restated (oracle port), timed."""
    from oracle import restate as R

    _, y = R.simulate(1.0, 0.1, 0.0, t_len, 0)
    pool = R.Lanes(lanes)
    try:
        R.run_loop(y[:1], min(n, 1024), 0, track_quantiles=False, lanes=pool)  # warm-up
        t0 = time.perf_counter()
        R.run_loop(y, n, 0, track_quantiles=False, lanes=pool)
        dt = time.perf_counter() - t0
    finally:
        pool.close()
    return n * t_len / dt, dt


def _aggregate_worker(args):
    n, t_len, barrier_ = args
    from oracle import restate as R

    _, y = R.simulate(1.0, 0.1, 0.0, t_len, 0)
    R.run_loop(y[:1], min(n, 1024), 0, track_quantiles=False)  # warm-up (imports, scipy)
    barrier_.wait()
    t0 = time.time()
    R.run_loop(y, n, 0, track_quantiles=False)
    return t0, time.time()


def cpu_aggregate_run(n, t_len, procs):
    """BASELINE.md §3 all-cores aggregate: ``procs`` concurrent single-lane
    processes, one replication each (the reference's gammaincinv / argsort
    are single-threaded, so lanes barely help one run).  Returns
    particle-steps/s over the wall span of all timed runs."""
    from multiprocessing import get_context

    ctx = get_context("spawn")
    with ctx.Manager() as mgr:
        b = mgr.Barrier(procs)
        with ctx.Pool(procs) as pool:
            spans = pool.map(_aggregate_worker, [(n, t_len, b)] * procs)
    wall = max(e for _, e in spans) - min(s for s, _ in spans)
    return procs * n * t_len / wall, wall


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_block(n, t_len, aggregate=True):
    """The cpu_baseline object: the reference's par_cutpoint cell (oracle port,
    all host threads as Backend lanes) on a bounded sample at N = n, plus the
    all-cores aggregate and the host model."""
    lanes = os.cpu_count() or 1
    v, dt = cpu_reference_run(n, t_len, lanes)
    out = {"value": v, "unit": "particle-steps/s", "cores": lanes, "kind": "port",
           "sample": f"oracle/restate.py run_loop N={n} T={t_len} ({dt:.1f} s, {lanes} lanes, one run)",
           "cpu_model": cpu_model(),
           "survey_measured_reference": "SURVEY.md §6.3: the unmodified reference measured in the "
                                        "build container (8 vCPU), same cell"}
    if aggregate:
        agg, wall = cpu_aggregate_run(n, t_len, lanes)
        out["aggregate_all_cores"] = {"value": agg, "unit": "particle-steps/s", "procs": lanes,
                                      "sample": f"{lanes} concurrent 1-lane runs of N={n} T={t_len} "
                                                f"({wall:.1f} s wall)"}
    return out


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    lanes = os.cpu_count() or 1
    n, t_len = args.ref_n, args.ref_t
    vals = []
    for _ in range(args.warmup):
        cpu_reference_run(min(n, 1 << 16), 2, lanes)
    for _ in range(args.steps):
        v, _ = cpu_reference_run(n, t_len, lanes)
        vals.append(v)
    vals.sort()
    value = vals[len(vals) // 2]
    line = {
        "impl": "reference",
        "metric": "particle-steps/sec (N*T/s), full particle-learning cycle",
        "value": value, "unit": "particle-steps/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": n * t_len / value * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"PL trend+noise, Priors(), cutpoint, N={args.n}, T={args.t} "
                               f"(CPU sample N={n}, T={t_len})", "N": args.n, "T": args.t},
        "cpu_baseline": {"value": value, "unit": "particle-steps/s", "cores": lanes,
                         "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"oracle/restate.py run_loop N={n} T={t_len}, {lanes} lanes, "
                                   f"median of {args.steps}"},
        "e2e": {"value": value, "unit": "particle-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_traffic():
    """ncu dram bytes per step-kernel launch, from the committed profile summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "step_kernel_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--t", type=int, default=1000)
    ap.add_argument("--ref-n", type=int, default=1 << 20, help="CPU sample particles (BASELINE.md §3: N >= 2^20)")
    ap.add_argument("--ref-t", type=int, default=10, help="CPU sample steps (cost is linear in T)")
    ap.add_argument("--no-cpu-aggregate", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--multi", default="shard", choices=["shard", "replicas"])
    ap.add_argument("--n-shard", type=int, default=None,
                    help="particles of the sharded filter (default: world x --n, weak scaling)")
    ap.add_argument("--shards", type=int, default=1)
    ap.add_argument("--resampler", default="cutpoint", choices=["cutpoint", "spacings"],
                    help="cutpoint: the reference's exact parallel resampler (parity path); spacings: "
                         "the K7 ordered-uniform perf mode (exact multinomial, streaming gathers)")
    ap.add_argument("--process-group", action="store_true",
                    help="run the one-process-per-GPU sharded path even with one rank")
    args = ap.parse_args()
    world, rank, local = dist_setup(force=args.process_group)
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return

    import numpy as np

    import paper_1212_1639_b200 as P
    from paper_1212_1639_b200 import _lib

    if (world > 1 and args.multi == "shard") or args.shards > 1 or args.process_group:
        return run_sharded(args, world, rank, local)
    lib = _lib.require_device()
    n, t_len = args.n, args.t
    _, y = P.simulate(P.TrendNoiseModel(), t_len, P.RngStream(0, P.rng.AUX_STREAM_BASE + 1))
    backend = P.Backend("cuda", device=local)
    # first call: engine creation + gamma tables (excluded, like the
    # reference bench's numba warm-up, bench.py:153-161)
    P.run_particle_learning(P.Priors(), y, n, seed=0, backend=backend, track_quantiles=False,
                            resampler=args.resampler)
    eng = next(iter(backend._engines.values()))
    cfg = eng.cfg
    for _ in range(args.warmup):
        eng.run_resident(t_len)
    # ---- value: K resident runs, device events
    barrier(world)
    k0 = lib.pf_launch_count()
    step_ms = []
    with ClockSampler(local) as clk:
        tot_ms = 0.0
        for _ in range(args.steps):
            eng.run_resident(t_len)
            tm = eng.last_timing()
            tot_ms += tm["total_ms"]
            step_ms.append(tm["step_kernel_ms"])
    launches = lib.pf_launch_count() - k0
    barrier(world)
    tot_ms = max_over_ranks(tot_ms, world)
    value = world * n * t_len * args.steps / (tot_ms / 1e3)
    # ---- e2e: public API, host y in / host summaries out
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = P.run_particle_learning(P.Priors(), y, n, seed=0, backend=backend,
                                      track_quantiles=False, resampler=args.resampler)
        _ = out.param_posterior["sigma2"].mean[-1]
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    e2e = world * n * t_len * args.steps / e2e_s
    d2h = 8 * t_len * (1 + 2 * 7)  # filtered mean + 2 params x (mean, sd, 5 quantiles)
    h2d = 8 * t_len + _lib.C.sizeof(_lib.PfConfig)
    backend.close()
    del cfg

    peak, peak_kind = _peaks()
    kern_ms = float(np.mean(step_ms))
    achieved = ALG_BYTES_STEP_KERNEL * n / (kern_ms / 1e3) / 1e9
    traffic = load_traffic()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_block(args.ref_n, args.ref_t, aggregate=not args.no_cpu_aggregate)
    if rank == 0:
        line = {
            "metric": "particle-steps/sec (N*T/s), full particle-learning cycle",
            "value": value, "unit": "particle-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"PL trend+noise, Priors(), {args.resampler}, N=2^{n.bit_length() - 1}, "
                                   f"T={t_len}, seed 0, track_quantiles=False",
                       "N": n, "T": t_len, "parallelism": f"replicas x{world}",
                       "l2": "working set >> L2 (no flush needed)"},
            "e2e": {"value": e2e, "unit": "particle-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": {"bound": "hbm", "kernel": "step_kernel", "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": None if traffic is None else traffic.get("bytes_per_launch"),
                         "alg_bytes_per_particle": ALG_BYTES_STEP_KERNEL,
                         "step_kernel_ms": kern_ms,
                         "cycle_frac": ALG_BYTES_CYCLE * n * t_len / (tot_ms / args.steps / 1e3) / 1e9 / peak},
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_sharded(args, world, rank, local):
    """One filter sharded over G shards: G = world GPUs, one process each
    (torchrun; Backend(process_group=...)), or --shards G on one GPU from
    one process (pf_group_*)."""
    import paper_1212_1639_b200 as P
    from paper_1212_1639_b200 import _lib

    G = world if world > 1 else args.shards
    fixed_total = args.n_shard is not None
    n = (args.n_shard if fixed_total else world * args.n) if world > 1 else args.n
    t_len = args.t
    spmd = world > 1 or args.process_group
    _, y = P.simulate(P.TrendNoiseModel(), t_len, P.RngStream(0, P.rng.AUX_STREAM_BASE + 1))
    lib = _lib.require_device()
    if spmd:
        backend = P.Backend("cuda", device=local, process_group=True)
        where = f"one process per GPU, {G} ranks (NCCL exchange, CUDA IPC peer reads)"
    else:
        backend = P.Backend("cuda", shards=G, devices=[local] * G)
        where = f"{G} shards on GPU {local} (one process)"

    def once():
        return P.run_particle_learning(P.Priors(), y, n, seed=0, backend=backend, track_quantiles=False,
                                       resampler=args.resampler)

    once()
    eng = next(iter(backend._engines.values()))
    for _ in range(args.warmup):
        once()
    barrier(world)
    tot_ms = 0.0
    k0 = lib.pf_launch_count()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            out = once()
            tot_ms += eng.last_timing()["total_ms"]
            _ = out.param_posterior["sigma2"].mean[-1]
        e2e_s = time.perf_counter() - t0
    launches = lib.pf_launch_count() - k0
    clk_summary = clk.summary()
    backend.close()
    barrier(world)
    tot_ms = max_over_ranks(tot_ms, world)
    e2e_s = max_over_ranks(e2e_s, world)
    launches = int(max_over_ranks(float(launches), world))
    if rank == 0:
        peak, peak_kind = _peaks()
        per_gpu = ALG_BYTES_CYCLE * n * t_len / (tot_ms / args.steps / 1e3) / 1e9 / G
        line = {
            "metric": "particle-steps/sec (N*T/s), full particle-learning cycle",
            "value": n * t_len * args.steps / (tot_ms / 1e3), "unit": "particle-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if (world > 1 and fixed_total) else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"PL trend+noise, Priors(), {args.resampler}, N=2^{n.bit_length() - 1} sharded "
                                   f"over {G} shards, T={t_len}, seed 0, track_quantiles=False",
                       "N": n, "T": t_len, "parallelism": where,
                       "l2": "working set >> L2 (no flush needed)"},
            "e2e": {"value": n * t_len * args.steps / e2e_s, "unit": "particle-steps/s",
                    "h2d_bytes_per_step": 8 * t_len, "d2h_bytes_per_step": 8 * t_len * 15},
            "roofline": {"bound": "hbm", "kernel": "whole cycle", "achieved": per_gpu, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s per GPU", "frac": per_gpu / peak,
                         "traffic": None, "alg_bytes_per_particle": ALG_BYTES_CYCLE},
            "cpu_baseline": None,
            "gpu_launches": launches,
            "clocks": clk_summary,
        }
        print(json.dumps(line), flush=True)
    if spmd:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
