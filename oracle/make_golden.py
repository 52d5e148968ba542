"""Generate golden fixtures by running the REAL reference -- test infrastructure.

Run in the build container only (the GPU box has no /root/reference):

    python oracle/make_golden.py

The reference package is copied to a temp dir first so numba's on-disk
cache (``@njit(cache=True)``, rng.py:66 / resampling.py:39) never writes into
the read-only reference tree.  Outputs go to ``tests/golden/*.npz``; they are
small, committed, and are what both the CPU oracle tests and the GPU parity
tests compare against.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
REF = "/root/reference/pkg"


def import_reference():
    tmp = tempfile.mkdtemp(prefix="parsmc_ref_")
    shutil.copytree(REF, os.path.join(tmp, "pkg"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba"))
    sys.path.insert(0, os.path.join(tmp, "pkg", "src"))
    import parsmc  # noqa: F401

    return tmp


def philox_fixture(P):
    from parsmc.rng import philox4x64_block, philox_block_lanes, uniforms_at

    rng = np.random.default_rng(2024)
    ids = np.concatenate([np.arange(64, dtype=np.uint64),
                          rng.integers(0, 2**64, size=192, dtype=np.uint64),
                          np.array([2**62, 2**62 + 1, 2**64 - 1], dtype=np.uint64)])
    seeds = np.array([0, 1, 17, 2**63 + 5, 2**64 - 1], dtype=np.uint64)
    blocks = np.array([0, 1, 2, 1000, 123456, 2**63 + 17, 2**62 - 1], dtype=np.uint64)
    words = np.empty((len(seeds), len(blocks), 4, len(ids)), dtype=np.uint64)
    for i, s in enumerate(seeds):
        for j, b in enumerate(blocks):
            words[i, j] = philox_block_lanes(int(b), int(s), ids)
    # spot-check the vectorised path agrees (the reference's own invariant)
    z = np.zeros_like(ids)
    v = philox4x64_block(np.full_like(ids, blocks[3]), z, z, z, seeds[2], ids)
    assert all(np.array_equal(v[w], words[2, 3, w]) for w in range(4))
    # uniforms at scattered (stream, counter) pairs
    us = rng.integers(0, 2**64, size=500, dtype=np.uint64)
    uc = rng.integers(0, 2**64, size=500, dtype=np.uint64)
    uu = uniforms_at(7, us, uc)
    np.savez_compressed(os.path.join(OUT, "philox.npz"), ids=ids, seeds=seeds,
                        blocks=blocks, words=words, u_streams=us, u_counters=uc,
                        u_seed=np.uint64(7), u_values=uu)


def cdf_fixture():
    from parsmc.prefix_sum import parallel_cdf
    from parsmc.resampling import cut_points_parallel, cutpoint_indices
    from parsmc.rng import StreamArray

    rng = np.random.default_rng(77)
    cases = {}
    k = 0

    def add(w, tag):
        nonlocal k
        w = np.asarray(w)
        q = parallel_cdf(w)
        cuts = cut_points_parallel(q)
        sa = StreamArray.for_lanes(11 + k, len(w))
        u = sa.uniforms()
        idx = cutpoint_indices(q, cuts, u)
        cases[f"c{k}_w"] = w
        cases[f"c{k}_q"] = q
        cases[f"c{k}_cuts"] = cuts
        cases[f"c{k}_u"] = u
        cases[f"c{k}_idx"] = idx
        cases[f"c{k}_tag"] = np.array(tag)
        k += 1

    add(np.array([2.0, 4.0, 3.0, 1.0]), "table1")
    add(np.ones(4), "uniform4")
    add(np.array([5.0]), "single")
    for n in (2, 8, 64, 1024, 1 << 14):
        add(rng.exponential(size=n), f"exp{n}")
    for n in (16, 512, 4096):
        w = rng.exponential(size=n)
        w[rng.random(n) < 0.5] = 0.0
        w[0] = 0.0
        if w.sum() == 0:
            w[-1] = 1.0
        add(w, f"zeros{n}")
    w = np.zeros(256)
    w[97] = 3.0
    add(w, "pointmass")
    add(rng.integers(0, 1024, size=2048).astype(np.float64), "ints")
    add(np.exp(-0.5 * rng.normal(scale=4.0, size=1 << 16) ** 2), "peaky")
    add(rng.exponential(size=1024).astype(np.float32), "fp32_1024")
    add(np.array([2, 4, 3, 1], dtype=np.float32), "fp32_table1")
    cases["count"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "cdf.npz"), **cases)


def special_fixture():
    from scipy.special import gammaincinv, ndtri

    rng = np.random.default_rng(5)
    kk = rng.integers(0, 2**52, size=20000, dtype=np.uint64)
    u = (kk.astype(np.float64) + 0.5) * 2.0**-52
    ext = np.array([2.0**-53, 1 - 2.0**-53, 0.5, 0.13533528323661269189,
                    1 - 0.13533528323661269189, 1e-10, 1 - 1e-10, 0.25, 0.75,
                    3 * 2.0**-53, 1 - 3 * 2.0**-53])
    u = np.concatenate([ext, u])
    shapes = np.array([0.5, 1.0, 2.3, 5.0, 5.5, 12.0, 55.0, 55.5, 255.0, 505.0, 1005.0])
    g = np.stack([gammaincinv(a, u[:4000]) for a in shapes])
    np.savez_compressed(os.path.join(OUT, "special.npz"), u=u, ndtri=ndtri(u),
                        shapes=shapes, gammaincinv=g, u_g=u[:4000])


class Recorder:
    """Hooks the reference's module-level names to capture per-step draws."""

    def __init__(self):
        import parsmc.filtering as F
        import parsmc.rng as R

        self.F, self.R = F, R
        self.orig = (F.gammaincinv, R.gammaincinv, R.StreamArray.normals,
                     F.parallel_cdf, F.resample_cutpoint)
        self.calls = {"z": [], "g": [], "g0": [], "w": [], "q": [], "idx": []}
        calls = self.calls
        g_f, g_r, normals, pcdf, rcut = self.orig

        def F_g(a, u):
            out = g_f(a, u)
            calls["g"].append(np.array(out))
            return out

        def R_g(a, u):
            out = g_r(a, u)
            calls["g0"].append(np.array(out))
            return out

        def nrm(self_):
            out = normals(self_)
            calls["z"].append(np.array(out))
            return out

        def cdf(w, backend=None, pad=False):
            q = pcdf(w, backend, pad)
            calls["w"].append(np.array(w))
            calls["q"].append(np.array(q))
            return q

        def rc(cdf_, streams, backend=None):
            idx = rcut(cdf_, streams, backend)
            calls["idx"].append(np.array(idx))
            return idx

        F.gammaincinv, R.gammaincinv, R.StreamArray.normals = F_g, R_g, nrm
        F.parallel_cdf, F.resample_cutpoint = cdf, rc

    def restore(self):
        F, R = self.F, self.R
        (F.gammaincinv, R.gammaincinv, R.StreamArray.normals,
         F.parallel_cdf, F.resample_cutpoint) = self.orig


def run_fixture(name, kind, n, t_len, seed, data_seed, priors=None, model=None,
                precision="double", resampler="cutpoint"):
    from parsmc import (InverseGammaPrior, Priors, RngStream, TrendNoiseModel,
                        run_particle_filter, run_particle_learning, simulate)

    model_sim = TrendNoiseModel()
    _, y = simulate(model_sim, t_len, RngStream(data_seed, 2**62 + 1))
    rec = Recorder()
    try:
        kw = dict(seed=seed, keep_indices=True, keep_final=True, track_quantiles=True,
                  precision=precision, resampler=resampler)
        if kind == "learn":
            pri = priors if priors is not None else Priors()
            out = run_particle_learning(pri, y, n, **kw)
        else:
            out = run_particle_filter(model if model is not None else TrendNoiseModel(),
                                      y, n, **kw)
    finally:
        rec.restore()
    c = rec.calls
    d = {"y": y, "n": np.array(n), "seed": np.array(seed), "precision": np.array(precision),
         "resampler": np.array(resampler),
         "filtered_mean": out.filtered_mean, "filtered_quantiles": out.filtered_quantiles,
         "indices": out.resampled_indices,
         "final_states": out.final_particles.states, "z": np.stack(c["z"])}
    for k in ("w", "q", "idx"):  # only the cut-point path goes through these hooks
        if c[k]:
            d[k] = np.stack(c[k])
    if kind == "learn":
        pri = priors if priors is not None else Priors()
        d["prior"] = np.array([pri.x0_mean, pri.x0_var,
                               *(([pri.sigma2.shape, pri.sigma2.scale]) if pri.learns_sigma2 else [-1.0, pri.sigma2]),
                               *(([pri.tau2.shape, pri.tau2.scale]) if pri.learns_tau2 else [-1.0, pri.tau2])])
        g = c["g"]
        per = int(pri.learns_sigma2) + int(pri.learns_tau2)
        g0 = c["g0"]
        if pri.learns_sigma2:
            d["g_sigma"] = np.stack([g0[0]] + [g[per * t] for t in range(t_len)])
        if pri.learns_tau2:
            off = int(pri.learns_sigma2)
            d["g_tau"] = np.stack([g0[off]] + [g[per * t + off] for t in range(t_len)])
        for nm, s in (out.param_posterior or {}).items():
            d[f"{nm}_mean"] = s.mean
            d[f"{nm}_sd"] = s.sd
            d[f"{nm}_quantiles"] = s.quantiles
        fp = out.final_particles
        d["final_sigma2"] = fp.params.sigma2
        d["final_tau2"] = fp.params.tau2
        d["final_b_sigma"] = fp.suffstats.b_sigma
        d["final_b_tau"] = fp.suffstats.b_tau
        d["final_a_sigma"] = fp.suffstats.a_sigma
        d["final_a_tau"] = fp.suffstats.a_tau
    else:
        m = model if model is not None else TrendNoiseModel()
        d["model"] = np.array([m.sigma2, m.tau2, m.x0_mean, m.x0_var])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)


def resampler_fixtures():
    """The reference's sequential baseline resamplers (resampling.py:29-87) in
    the loop (filtering.py:305-316), including a non-power-of-two N."""
    from parsmc import TrendNoiseModel

    run_fixture("run_pl_sorted", "learn", 1000, 10, seed=21, data_seed=2, resampler="sorted")
    run_fixture("run_pl_systematic", "learn", 1024, 10, seed=22, data_seed=3, resampler="systematic")
    run_fixture("run_pl_stratified", "learn", 768, 10, seed=23, data_seed=4, resampler="stratified")
    run_fixture("run_pl_naive", "learn", 300, 8, seed=24, data_seed=5, resampler="naive")
    run_fixture("run_pf_sorted", "filter", 999, 10, seed=25, data_seed=6, resampler="sorted",
                model=TrendNoiseModel())
    run_fixture("run_pl_sorted_single", "learn", 1000, 8, seed=26, data_seed=7, resampler="sorted",
                precision="single")


def main():
    os.makedirs(OUT, exist_ok=True)
    tmp = import_reference()
    if len(sys.argv) > 1 and sys.argv[1] == "resamplers":
        try:
            resampler_fixtures()
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
        print("resampler fixtures written to", OUT)
        return
    try:
        from parsmc import InverseGammaPrior, Priors, TrendNoiseModel

        philox_fixture(None)
        cdf_fixture()
        special_fixture()
        run_fixture("run_pl", "learn", 1024, 20, seed=13, data_seed=0)
        run_fixture("run_pl_fixed_tau", "learn", 512, 16, seed=4, data_seed=31,
                    priors=Priors(sigma2=InverseGammaPrior(5, 4), tau2=0.1))
        run_fixture("run_pl_priors", "learn", 256, 12, seed=8, data_seed=1,
                    priors=Priors(x0_mean=0.5, x0_var=3.0,
                                  sigma2=InverseGammaPrior(3.0, 2.5),
                                  tau2=InverseGammaPrior(7.5, 0.9)))
        run_fixture("run_pf", "filter", 512, 20, seed=5, data_seed=123)
        run_fixture("run_pf_model", "filter", 64, 10, seed=17, data_seed=9,
                    model=TrendNoiseModel(sigma2=1.3, tau2=0.2, x0_mean=0.5, x0_var=2.0))
        run_fixture("run_pl_single", "learn", 512, 12, seed=3, data_seed=12,
                    precision="single")
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
