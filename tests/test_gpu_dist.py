"""One process per GPU (distributed.py, pf_shard_* in the C ABI): a filter
sharded over a torch.distributed process group must be bit-identical to the
single-device engine in ancestors and final particles, with the same moments
(to rounding) and weighted quantiles -- the reference's results do not depend
on how the particles are split (backend.py:1-8).  The ranks here share one
B200 over gloo; the peer reads take the same CUDA IPC path as across GPUs."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_1212_1639_b200 as P

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(tmp_path, world, *args):
    out = str(tmp_path / "dist.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "workers", "dist_shard_worker.py"), "--out", out, "--same-gpu", *args]
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return dict(np.load(out, allow_pickle=True))


def _series(t_len, seed=1):
    _, y = P.simulate(P.TrendNoiseModel(), t_len, P.RngStream(seed, P.rng.AUX_STREAM_BASE + 1))
    return y


def _single(kind, n, t_len, seed):
    y = _series(t_len)
    with P.Backend("cuda") as b:
        if kind == "filter":
            return P.run_particle_filter(P.TrendNoiseModel(), y, n, seed=seed, backend=b, keep_indices=True,
                                         keep_final=True, track_quantiles=True)
        prec = "single" if kind == "single" else "double"
        return P.run_particle_learning(P.Priors(), y, n, seed=seed, backend=b, keep_indices=True,
                                       keep_final=True, track_quantiles=True, precision=prec)


def _check(one, d, r, learn=True):
    assert np.array_equal(one.resampled_indices, d[f"indices{r}"])
    assert np.array_equal(one.final_particles.states, d[f"states{r}"])
    np.testing.assert_allclose(one.filtered_mean, d[f"fmean{r}"], rtol=1e-12, atol=1e-13)
    assert np.array_equal(one.filtered_quantiles, d[f"fq{r}"])
    if learn:
        for nm in ("sigma2", "tau2"):
            assert np.array_equal(getattr(one.final_particles.params, nm), d[f"{nm}{r}"])
            np.testing.assert_allclose(one.param_posterior[nm].mean, d[f"{nm}_mean{r}"], rtol=1e-12)
            np.testing.assert_allclose(one.param_posterior[nm].sd, d[f"{nm}_sd{r}"], rtol=1e-9)
            assert np.array_equal(one.param_posterior[nm].quantiles, d[f"{nm}_q{r}"])


@pytest.mark.parametrize("world", [2, 4])
def test_process_group_learning_matches_single_device(gpu, tmp_path, world):
    n, t_len = 1 << 15, 16
    d = _launch(tmp_path, world, "--particles", str(n), "--series-len", str(t_len), "--runs", "2")
    for r in range(2):
        _check(_single("learning", n, t_len, 5 + r), d, r)


def test_process_group_filter_matches_single_device(gpu, tmp_path):
    n, t_len = 1 << 14, 12
    d = _launch(tmp_path, 2, "--particles", str(n), "--series-len", str(t_len), "--kind", "filter")
    _check(_single("filter", n, t_len, 5), d, 0, learn=False)


def test_process_group_single_precision(gpu, tmp_path):
    n, t_len = 1 << 14, 10
    d = _launch(tmp_path, 2, "--particles", str(n), "--series-len", str(t_len), "--kind", "single")
    _check(_single("single", n, t_len, 5), d, 0)


def test_process_group_nccl_path(gpu, tmp_path):
    # NCCL refuses two ranks on one GPU; a one-rank NCCL group still runs the
    # stream-ordered path (in-place all-gathers on the engine's stream, the
    # IPC-free own-rank tables, the device-side barrier).
    n, t_len = 1 << 14, 12
    d = _launch(tmp_path, 1, "--particles", str(n), "--series-len", str(t_len), "--backend", "nccl", "--runs", "2")
    for r in range(2):
        _check(_single("learning", n, t_len, 5 + r), d, r)


def test_process_group_rank_tables(gpu, tmp_path):
    # N >= 2^21: the ranks' lookups use the per-shard rank tables (owner
    # shard's grp / fq / f32 through the IPC mappings), boundary groups the
    # cut / q walk -- still bit-identical to one device.
    n, t_len = 1 << 21, 6
    d = _launch(tmp_path, 2, "--particles", str(n), "--series-len", str(t_len))
    _check(_single("learning", n, t_len, 5), d, 0)


def test_process_group_degeneracy_raises_on_every_rank(gpu, tmp_path):
    # the reference's AllWeightsZeroError(step=t) (filtering.py:294-296),
    # raised identically by every rank (all see the same partial records)
    d = _launch(tmp_path, 2, "--particles", str(1 << 13), "--kind", "degenerate")
    assert list(d["steps"]) == [2, 2]
