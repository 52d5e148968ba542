"""Short device run for ncu / diagnostics: PL at N=2^k, T steps.

Usage: python scripts/prof_run.py [log2n] [T] [track_quantiles]

One API run of T steps (engine, gamma tables), then one resident run.  With
PF_PROFILE_FROM_STEP=t set, the resident run brackets steps t..T with
cudaProfilerStart/Stop (ncu --profile-from-start off: steady-state steps).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1212_1639_b200 as P  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 24
T = int(sys.argv[2]) if len(sys.argv) > 2 else 5
tq = len(sys.argv) > 3 and sys.argv[3] == "1"
_, y = P.simulate(P.TrendNoiseModel(), T, P.RngStream(0, P.rng.AUX_STREAM_BASE + 1))
b = P.Backend()
P.run_particle_learning(P.Priors(), y, 1 << k, seed=0, backend=b, track_quantiles=tq)
eng = next(iter(b._engines.values()))
print("api run", eng.last_timing(), eng.quantile_stats())
eng.run_resident(T)
print("resident", eng.last_timing(), eng.quantile_stats())
b.close()
