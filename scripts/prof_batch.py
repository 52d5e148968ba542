"""Batched replications under ncu / diagnostics: R x N=2^k particles, T steps.

Usage: python scripts/prof_batch.py [log2n] [T] [R]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1212_1639_b200 as P  # noqa: E402
from paper_1212_1639_b200.filtering import run_batch  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 20
T = int(sys.argv[2]) if len(sys.argv) > 2 else 30
R = int(sys.argv[3]) if len(sys.argv) > 3 else 16
_, y = P.simulate(P.TrendNoiseModel(), T, P.RngStream(0, P.rng.AUX_STREAM_BASE + 1))
with P.Backend() as b:
    run_batch(P.Priors(), y, 1 << k, list(range(R)), backend=b, track_quantiles=False)
    eng = next(iter(b._engines.values()))
    for _ in range(2):
        run_batch(P.Priors(), y, 1 << k, list(range(R, 2 * R)), backend=b, track_quantiles=False)
        print("batch", R, "x 2^%d" % k, eng.last_timing(), eng.quantile_stats(), flush=True)
