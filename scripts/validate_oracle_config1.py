"""BASELINE configs[1]: oracle-mode equivalence at full size -- N = 2^20
particles, T = 1000, particle learning with Priors(), seed 0, cut-point.

The reference's own draws are regenerated exactly as the reference makes them
(Philox block t of stream j -> scipy ndtri / gammaincinv at a_t = a0 + t/2,
rng.py:223-229, filtering.py:277-288) with a process pool, fed to both the
CPU oracle (oracle/restate.py run_loop, pinned to the reference's golden runs)
and the device engine (noise=...).  Checks: ancestor indices of all T steps
bit-identical, final particles bit-identical, filtered mean / parameter
mean / sd within 1e-10 relative, parameter quantiles equal.  Prints one JSON
line.  Run on the GPU box:  python scripts/validate_oracle_config1.py [log2n] [T]
"""
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import restate as R  # noqa: E402

LOG2N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
N = 1 << LOG2N
SEED = 0


def draws(t):
    from scipy.special import gammaincinv, ndtri

    ids = np.arange(N, dtype=np.uint64)
    w = R.block_words(SEED, ids, t)
    a = 5.0
    for _ in range(t):
        a = a + 0.5
    z = ndtri(R.unit_open(w[0]))
    gs = gammaincinv(a, R.unit_open(w[1]))
    gt = gammaincinv(a, R.unit_open(w[2]))
    return t, z, gs, gt


def main():
    t0 = time.time()
    _, y = R.simulate(1.0, 0.1, 0.0, T, 0)
    feed = {k: np.empty((T + 1, N)) for k in ("z", "g_sigma", "g_tau")}
    with Pool(os.cpu_count()) as pool:
        for t, z, gs, gt in pool.imap_unordered(draws, range(T + 1), chunksize=4):
            feed["z"][t], feed["g_sigma"][t], feed["g_tau"][t] = z, gs, gt
    t_feed = time.time() - t0
    ref = R.run_loop(y, N, SEED, track_quantiles=False, keep_indices=True, keep_final=True, feed=feed)
    t_oracle = time.time() - t0 - t_feed
    import paper_1212_1639_b200 as P

    out = P.run_particle_learning(P.Priors(), y, N, seed=SEED, track_quantiles=False, keep_indices=True,
                                  keep_final=True, noise=feed)
    steps_equal = int(sum(np.array_equal(out.resampled_indices[t], ref["indices"][t]) for t in range(T)))
    first_diff = next((t + 1 for t in range(T) if not np.array_equal(out.resampled_indices[t], ref["indices"][t])), None)

    def rel(a, b):
        return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(np.abs(b), 1e-300)))

    res = {
        "config": f"configs[1] oracle mode: N=2^{LOG2N}, T={T}, PL Priors(), seed {SEED}, cutpoint",
        "steps_with_identical_ancestors": steps_equal, "T": T, "first_differing_step": first_diff,
        "final_states_identical": bool(np.array_equal(out.final_particles.states, ref["final"]["states"])),
        "final_sigma2_identical": bool(np.array_equal(out.final_particles.params.sigma2, ref["final"]["sigma2"])),
        "filtered_mean_max_rel": rel(out.filtered_mean, ref["filtered_mean"]),
        "sigma2_mean_max_rel": rel(out.param_posterior["sigma2"].mean, ref["sigma2"]["mean"]),
        "tau2_mean_max_rel": rel(out.param_posterior["tau2"].mean, ref["tau2"]["mean"]),
        "sigma2_sd_max_rel": rel(out.param_posterior["sigma2"].sd, ref["sigma2"]["sd"]),
        "param_quantiles_equal_steps": int(sum(
            np.array_equal(out.param_posterior[nm].quantiles[t], ref[nm]["quantiles"][t])
            for nm in ("sigma2", "tau2") for t in range(T))),
        "param_quantile_rows": 2 * T,
        "seconds": {"feed": round(t_feed, 1), "oracle": round(t_oracle, 1)},
    }
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
