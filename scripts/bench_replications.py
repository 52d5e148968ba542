"""BASELINE configs[4]: R Monte Carlo replications of particle learning at
N = 2^20 particles, T = 100 steps (the paper's T), replication r
seeded with r, spread round robin over the GPUs of one node (torchrun: one
rank per GPU; replicas only, no collective on the data path).

Prints one JSON line: particle-steps/s = R * N * T / (max over ranks of the
device time of the rank's runs), plus the wall time.

  python scripts/bench_replications.py [--reps R] [--n N] [--t T]
  torchrun --nproc-per-node 8 scripts/bench_replications.py --reps 1000
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (dist helpers)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=64)
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--t", type=int, default=100)
    ap.add_argument("--concurrency", type=int, default=1)
    ap.add_argument("--batch", type=int, default=32,
                    help="replications per launch sequence (pf_engine_run_batch); 1 = one at a time")
    args = ap.parse_args()
    world, rank, local = bench.dist_setup()
    import paper_1212_1639_b200 as P
    from paper_1212_1639_b200.replications import rank_seeds

    _, y = P.simulate(P.TrendNoiseModel(), args.t, P.RngStream(0, P.rng.AUX_STREAM_BASE + 1))
    seeds = rank_seeds(range(args.reps), rank, world)
    backend = P.Backend("cuda", device=local)
    P.run_particle_learning(P.Priors(), y, args.n, seed=10 ** 6, backend=backend, track_quantiles=False)
    eng = next(iter(backend._engines.values()))
    bench.barrier(world)
    dev_ms = 0.0
    t0 = time.perf_counter()
    if args.batch > 1:
        from paper_1212_1639_b200.filtering import run_batch

        run_batch(P.Priors(), y, args.n, list(range(10 ** 6, 10 ** 6 + min(args.batch, len(seeds)))),
                  backend=backend, track_quantiles=False)  # warm-up: buffers and the captured loop
        bench.barrier(world)
        t0 = time.perf_counter()
        for lo in range(0, len(seeds), args.batch):
            outs = run_batch(P.Priors(), y, args.n, seeds[lo:lo + args.batch], backend=backend,
                             track_quantiles=False)
            dev_ms += eng.last_timing()["total_ms"]
            _ = [o.param_posterior["sigma2"].mean[-1] for o in outs]
    elif args.concurrency > 1:
        from paper_1212_1639_b200.replications import run_replications

        outs = run_replications(P.Priors(), y, args.n, seeds, backend=backend, concurrency=args.concurrency,
                                track_quantiles=False)
        _ = [o.param_posterior["sigma2"].mean[-1] for o in outs]
    else:
        for s in seeds:
            out = P.run_particle_learning(P.Priors(), y, args.n, seed=s, backend=backend, track_quantiles=False)
            dev_ms += eng.last_timing()["total_ms"]
            _ = out.param_posterior["sigma2"].mean[-1]
    wall = time.perf_counter() - t0
    if args.concurrency > 1:
        dev_ms = wall * 1e3  # concurrent engines: device time is the wall time of the batch
    bench.barrier(world)
    dev_ms = bench.max_over_ranks(dev_ms, world)
    wall = bench.max_over_ranks(wall, world)
    backend.close()
    if rank == 0:
        tot = args.reps * args.n * args.t
        print(json.dumps({"metric": "particle-steps/sec, Monte Carlo replications (configs[4])",
                          "value": tot / (dev_ms / 1e3), "unit": "particle-steps/s",
                          "wall_value": tot / wall, "n_gpus": world, "replications": args.reps,
                          "N": args.n, "T": args.t, "ms_per_replication": dev_ms / max(1, len(seeds)),
                          "scaling": "weak", "parallelism": f"replicas x{world}",
                          "concurrency_per_gpu": args.concurrency, "batch": args.batch}), flush=True)


if __name__ == "__main__":
    main()
