"""Kernel-level C entries in their device-pointer + stream form (the
``pf_*_d`` entries, include/parsmc_b200.h).

Each takes device buffers and a cudaStream_t, enqueues the same kernels as
the host-pointer form and returns without synchronising.  Checked here:
bit-identical results to the host form (which the other kernel tests pin
to the oracle and the reference's fixtures), work ordered on a side stream,
and the reference's error behaviour where the entry can still raise it.
"""

import numpy as np
import pytest

import paper_1212_1639_b200 as P
from paper_1212_1639_b200 import device_ops
from oracle import restate as R

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", [1, 1024, 1 << 16, 1 << 20])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_tree_cdf_device_equals_host(gpu, n, dtype):
    rng = np.random.default_rng(n)
    w = rng.exponential(size=n).astype(dtype)
    w[rng.random(n) < 0.05] = 0
    host = P.parallel_cdf(w)
    dev = P.parallel_cdf(_dev(w))
    assert dev.is_cuda and dev.dtype == torch.from_numpy(w).dtype
    np.testing.assert_array_equal(dev.cpu().numpy(), host)
    if dtype == np.float64 and n <= 1 << 16:
        np.testing.assert_array_equal(host, R.tree_cdf(w))


def test_tree_cdf_device_pad_and_errors(gpu):
    w = np.arange(1, 7, dtype=np.float64)
    np.testing.assert_array_equal(P.parallel_cdf(_dev(w), pad=True).cpu().numpy(), P.parallel_cdf(w, pad=True))
    with pytest.raises(P.NotPowerOfTwoError):
        P.parallel_cdf(_dev(w))
    with pytest.raises(P.AllWeightsZeroError):
        P.parallel_cdf(_dev(np.zeros(8)))
    with pytest.raises(P.AllWeightsZeroError):
        P.parallel_cdf(_dev(np.array([1.0, np.inf, 0.0, 2.0])))


@pytest.mark.parametrize("n", [1, 7, 4096, 1 << 20])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cut_table_and_lookup_device_equal_host(gpu, n, dtype):
    rng = np.random.default_rng(n + 1)
    w = rng.exponential(size=n)
    w[rng.random(n) < 0.1] = 0
    w[0] = 1.0
    q = R.sequential_cdf(w).astype(dtype) if n & (n - 1) else P.parallel_cdf(w.astype(dtype))
    q[-1] = 1
    cuts_h = P.cut_points_parallel(q)
    cuts_d = P.cut_points_parallel(_dev(q))
    assert cuts_d.dtype == torch.int64
    np.testing.assert_array_equal(cuts_d.cpu().numpy(), cuts_h)
    u = rng.random((3, max(1, n // 2)))
    idx_h = P.cutpoint_indices(q, cuts_h, u)
    idx_d = P.cutpoint_indices(_dev(q), cuts_d, _dev(u))
    assert idx_d.shape == u.shape
    np.testing.assert_array_equal(idx_d.cpu().numpy(), idx_h)


def test_resample_cutpoint_device_equals_host(gpu):
    n = 1 << 18
    q = P.parallel_cdf(np.random.default_rng(5).exponential(size=n))
    s_h = P.StreamArray.for_lanes(42, n)
    s_d = P.StreamArray.for_lanes(42, n)
    for _ in range(3):
        a = P.resample_cutpoint(q, s_h)
        b = P.resample_cutpoint(_dev(q), s_d)
        np.testing.assert_array_equal(b.cpu().numpy(), a)


def test_uniforms_at_device_equals_host(gpu):
    rng = np.random.default_rng(9)
    ids = rng.integers(0, 2**63, size=5000, dtype=np.uint64) * 2 + 1
    ctr = rng.integers(0, 1 << 40, size=5000, dtype=np.uint64)
    host = P.rng.uniforms_at(77, ids, ctr)
    dev = P.rng.uniforms_at(77, _dev(ids.view(np.int64)), _dev(ctr.view(np.int64)))
    np.testing.assert_array_equal(dev.cpu().numpy(), host)
    np.testing.assert_array_equal(host, R.uniforms_at(77, ids, ctr))


@pytest.mark.parametrize("wdtype", [np.float64, np.float32])
def test_weighted_quantiles_device_equals_host(gpu, wdtype):
    rng = np.random.default_rng(3)
    n = 1 << 17
    v = rng.normal(size=n)
    v[:100] = v[100:200]                      # ties
    w = rng.exponential(size=n).astype(wdtype)
    w[rng.random(n) < 0.2] = 0
    probs = np.array([0.0, 0.025, 0.5, 0.975, 1.0])
    host = P.weighted_quantiles(v, w, probs)
    dev = P.weighted_quantiles(_dev(v), _dev(w), probs)
    np.testing.assert_array_equal(dev.cpu().numpy(), host)


def test_device_entries_order_on_a_side_stream(gpu):
    """Everything runs on torch's current stream: a chain of device calls on
    a side stream, behind a long-running producer on that stream, sees the
    producer's output without any host synchronisation in between."""
    n = 1 << 22
    w = torch.rand(n, dtype=torch.float64, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        torch.cuda._sleep(50_000_000)          # keep the stream busy ~tens of ms
        w2 = w * 2.0                           # producer on the same stream
        q = device_ops.parallel_cdf(w2, check=False)
        cuts = P.cut_points_parallel(q)
        u = torch.rand(n, dtype=torch.float64, device="cuda")
        idx = P.cutpoint_indices(q, cuts, u)
    side.synchronize()
    wh = w.cpu().numpy() * 2.0
    qh = P.parallel_cdf(wh)
    np.testing.assert_array_equal(q.cpu().numpy(), qh)
    np.testing.assert_array_equal(idx.cpu().numpy(), P.cutpoint_indices(qh, P.cut_points_parallel(qh), u.cpu().numpy()))
