"""store_particles / keep_indices cost (the paper's Store phase):
wall time of the public API with and without the per-step snapshots.

Usage: python scripts/bench_store.py [log2n] [T]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1212_1639_b200 as P  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 20
T = int(sys.argv[2]) if len(sys.argv) > 2 else 30
n = 1 << k
_, y = P.simulate(P.TrendNoiseModel(), T, P.RngStream(0, P.rng.AUX_STREAM_BASE + 1))
res = {}
with P.Backend() as b:
    for name, kw in (("plain", {}), ("keep_indices", {"keep_indices": True}),
                     ("store", {"store_particles": True}), ("store+indices", {"store_particles": True, "keep_indices": True})):
        P.run_particle_learning(P.Priors(), y, n, seed=1, backend=b, **kw)  # warm-up (engine, tables, graphs)
        walls = []
        for rep in range(3):  # fresh output arrays every run (as a user gets them): best of 3
            t0 = time.perf_counter()
            out = P.run_particle_learning(P.Priors(), y, n, seed=2 + rep, backend=b, **kw)
            walls.append(time.perf_counter() - t0)
            del out
        wall = min(walls)
        out = P.run_particle_learning(P.Priors(), y, n, seed=2, backend=b, **kw)
        res[name] = {"wall_s": round(wall, 4), "ms_per_step": round(wall / T * 1e3, 3),
                     "store_ns": out.timings.store, "bytes_per_step_d2h": (56 if "store" in name else 0) * n +
                     (8 * n if "indices" in name else 0)}
print(json.dumps({"N": n, "T": T, **res}))
