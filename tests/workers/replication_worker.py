"""torchrun worker for tests/test_gpu_batch.py: BASELINE configs[4]'s
replicas-only layout -- each rank runs its round-robin share of the seeds
(replications.rank_seeds) as batched replications on its device, and rank 0
gathers every replication's summaries (no collective on the data path; one
final gather).  Ranks may share one GPU (gloo)."""
import argparse
import os

import numpy as np
import torch
import torch.distributed as dist

import paper_1212_1639_b200 as P
from paper_1212_1639_b200.replications import rank_seeds, run_replications


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--particles", type=int, default=1 << 12)
    ap.add_argument("--series-len", type=int, default=10)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--batch", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    _, y = P.simulate(P.TrendNoiseModel(), a.series_len, P.RngStream(1, P.rng.AUX_STREAM_BASE + 1))
    mine = rank_seeds(range(a.reps), rank, world)
    outs = run_replications(P.Priors(), y, a.particles, mine, batch=a.batch)
    local = {s: (o.filtered_mean, o.param_posterior["sigma2"].mean, o.param_posterior["tau2"].quantiles)
             for s, o in zip(mine, outs)}
    allr = [None] * world
    dist.all_gather_object(allr, local)
    if rank == 0:
        merged = {}
        for d in allr:
            merged.update(d)
        np.savez(a.out, seeds=np.array(sorted(merged)),
                 fmean=np.stack([merged[s][0] for s in sorted(merged)]),
                 smean=np.stack([merged[s][1] for s in sorted(merged)]),
                 tq=np.stack([merged[s][2] for s in sorted(merged)]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
