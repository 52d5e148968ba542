"""torchrun worker for tests/test_gpu_dist.py: every rank runs the same
sharded filter through the public API with Backend(process_group=...) and
rank 0 saves the outputs.  Ranks may share one GPU (gloo) or own one each
(nccl)."""
import argparse
import os

import numpy as np
import torch
import torch.distributed as dist

import paper_1212_1639_b200 as P


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--particles", type=int, default=1 << 14)
    ap.add_argument("--series-len", type=int, default=16)
    ap.add_argument("--kind", default="learning", choices=["learning", "filter", "single", "degenerate"])
    ap.add_argument("--same-gpu", action="store_true")
    ap.add_argument("--runs", type=int, default=1)
    ap.add_argument("--resampler", default="cutpoint")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = 0 if a.same_gpu else local
    torch.cuda.set_device(dev)
    dist.init_process_group(a.backend)
    rank = dist.get_rank()
    _, y = P.simulate(P.TrendNoiseModel(), a.series_len, P.RngStream(1, P.rng.AUX_STREAM_BASE + 1))
    res = {}
    if a.kind == "degenerate":
        # every rank must raise the reference's AllWeightsZeroError(step=2)
        with P.Backend("cuda", device=dev, process_group=True) as b:
            try:
                P.run_particle_filter(P.TrendNoiseModel(sigma2=1e-300, tau2=0.1), [0.0, 1e200], a.particles,
                                      seed=1, backend=b)
                step = -1
            except P.AllWeightsZeroError as e:
                step = e.step
        steps = [None] * dist.get_world_size()
        dist.all_gather_object(steps, step)
        if rank == 0:
            np.savez(a.out, steps=np.array(steps))
        dist.barrier()
        dist.destroy_process_group()
        return
    with P.Backend("cuda", device=dev, process_group=True) as b:
        for r in range(a.runs):
            seed = 5 + r
            if a.kind == "filter":
                o = P.run_particle_filter(P.TrendNoiseModel(), y, a.particles, seed=seed, backend=b,
                                          keep_indices=True, keep_final=True, track_quantiles=True)
            else:
                prec = "single" if a.kind == "single" else "double"
                o = P.run_particle_learning(P.Priors(), y, a.particles, seed=seed, backend=b, keep_indices=True,
                                            keep_final=True, track_quantiles=True, precision=prec,
                                            resampler=a.resampler)
            res[f"indices{r}"] = o.resampled_indices
            res[f"states{r}"] = o.final_particles.states
            res[f"fmean{r}"] = o.filtered_mean
            res[f"fq{r}"] = o.filtered_quantiles
            if a.kind != "filter":
                for nm in ("sigma2", "tau2"):
                    res[f"{nm}{r}"] = getattr(o.final_particles.params, nm)
                    res[f"{nm}_mean{r}"] = o.param_posterior[nm].mean
                    res[f"{nm}_sd{r}"] = o.param_posterior[nm].sd
                    res[f"{nm}_q{r}"] = o.param_posterior[nm].quantiles
    # every rank holds the full outputs: check they agree with rank 0's
    digest = float(np.sum(res["indices0"] % 9973)) + float(np.nansum(res["fmean0"]))
    allv = [None] * dist.get_world_size()
    dist.all_gather_object(allv, digest)
    assert all(v == allv[0] for v in allv), allv
    if rank == 0:
        np.savez(a.out, **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
