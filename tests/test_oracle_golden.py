"""The CPU oracle (oracle/restate.py) pinned against the reference.

Golden vectors in tests/golden/ were produced by running the reference
package itself (oracle/make_golden.py); the known-answer values are the
reference test suite's own (tests/test_prefix_sum.py, test_resampling.py).
No GPU needed.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import restate as R


def test_philox_words_match_reference():
    d = golden("philox")
    for i, s in enumerate(d["seeds"]):
        for j, b in enumerate(d["blocks"]):
            got = R.block_words(int(s), d["ids"], int(b))
            assert np.array_equal(got, d["words"][i, j])


def test_uniforms_at_match_reference():
    d = golden("philox")
    got = R.uniforms_at(int(d["u_seed"]), d["u_streams"], d["u_counters"])
    assert np.array_equal(got, d["u_values"])


def test_philox_matches_numpy_bit_generator():
    # numpy's Philox pre-increments its counter (tests/test_rng.py:14-37)
    rng = np.random.default_rng(11)
    for _ in range(10):
        ctr = rng.integers(0, 2**63, size=4, dtype=np.uint64)
        key = rng.integers(0, 2**64, size=2, dtype=np.uint64)
        want = np.random.Philox(counter=ctr, key=key).random_raw(4)
        c = [int(x) for x in ctr]
        c[0] += 1
        got = R.philox4x64_10(*(np.uint64(x) for x in c), key[0], key[1])
        assert [int(g) for g in got] == [int(w) for w in want]


def test_table1_known_answers():
    levels = R.forward_adder(np.array([2.0, 4.0, 3.0, 1.0]))
    assert [list(lv) for lv in levels] == [[2, 4, 3, 1], [6, 4], [10]]
    assert np.array_equal(R.backward_adder(levels), [2, 6, 9, 10])
    q = R.tree_cdf(np.array([2.0, 4.0, 3.0, 1.0]))
    assert np.allclose(q, [0.2, 0.6, 0.9, 1.0]) and q[-1] == 1.0
    assert np.array_equal(R.tree_cdf(np.ones(4)), [0.25, 0.5, 0.75, 1.0])


def test_cutpoint_known_answers():
    q4 = np.array([0.2, 0.6, 0.9, 1.0])
    assert np.array_equal(R.cut_points(q4), [1, 2, 2, 3])
    assert np.array_equal(R.cut_points_bruteforce(q4), [1, 2, 2, 3])
    got = R.cutpoint_indices(q4, R.cut_points(q4), np.array([0.55, 0.95, 0.05, 0.70]))
    assert np.array_equal(got, [2, 4, 1, 3])


def test_cdf_cut_lookup_match_reference_fixtures():
    d = golden("cdf")
    for k in range(int(d["count"])):
        w = d[f"c{k}_w"]
        q = R.tree_cdf(w)
        assert q.dtype == w.dtype
        assert np.array_equal(q, d[f"c{k}_q"]), str(d[f"c{k}_tag"])
        cuts = R.cut_points(q)
        assert np.array_equal(cuts, d[f"c{k}_cuts"])
        idx = R.cutpoint_indices(q, cuts, d[f"c{k}_u"])
        assert np.array_equal(idx, d[f"c{k}_idx"])


@pytest.mark.parametrize("chunk", [1, 2, 8, 64, 2048])
def test_chunked_tree_is_bit_identical(chunk):
    # the device's tile/top decomposition of the adder tree
    d = golden("cdf")
    for k in range(int(d["count"])):
        w = d[f"c{k}_w"]
        assert np.array_equal(R.tree_cdf_chunked(w, chunk), d[f"c{k}_q"])


def test_cut_points_equal_bruteforce_random():
    rng = np.random.default_rng(10)
    for n in (2, 8, 64, 256):
        for _ in range(10):
            w = rng.exponential(size=n) * (rng.random(n) > 0.3)
            w[rng.integers(n)] += 1.0
            q = R.tree_cdf(w)
            assert np.array_equal(R.cut_points(q), R.cut_points_bruteforce(q))


def test_lookup_equals_searchsorted_left():
    rng = np.random.default_rng(3)
    w = rng.exponential(size=1024)
    q = R.tree_cdf(w)
    u = rng.random(5000)
    assert np.array_equal(R.cutpoint_indices(q, R.cut_points(q), u),
                          np.searchsorted(q, u, side="left") + 1)


RUNS = ["run_pl", "run_pl_fixed_tau", "run_pl_priors", "run_pf", "run_pf_model", "run_pl_single"]
# the reference's sequential baseline resamplers (resampling.py:29-87), some at non-power-of-two N
RESAMPLER_RUNS = ["run_pl_sorted", "run_pl_systematic", "run_pl_stratified", "run_pl_naive",
                  "run_pf_sorted", "run_pl_sorted_single"]


def _oracle_kwargs(d):
    kw = {"resampler": str(d["resampler"])} if "resampler" in d else {}
    if "prior" in d:
        p = d["prior"]
        s2 = (p[2], p[3]) if p[2] > 0 else float(p[3])
        t2 = (p[4], p[5]) if p[4] > 0 else float(p[5])
        return dict(x0_mean=p[0], x0_var=p[1], sigma2=s2, tau2=t2, **kw)
    m = d["model"]
    return dict(x0_mean=m[2], x0_var=m[3], sigma2=float(m[0]), tau2=float(m[1]), **kw)


@pytest.mark.parametrize("name", RUNS + RESAMPLER_RUNS)
def test_full_loop_restatement_matches_reference(name):
    d = golden(name)
    rec = {}
    out = R.run_loop(d["y"], int(d["n"]), int(d["seed"]), precision=str(d["precision"]),
                     keep_indices=True, keep_final=True, record=rec, **_oracle_kwargs(d))
    assert np.array_equal(out["filtered_mean"], d["filtered_mean"])
    assert np.array_equal(out["filtered_quantiles"], d["filtered_quantiles"])
    assert np.array_equal(out["indices"], d["indices"])
    assert np.array_equal(out["final"]["states"], d["final_states"])
    for nm in ("sigma2", "tau2"):
        if f"{nm}_mean" in d:
            assert np.array_equal(out[nm]["mean"], d[f"{nm}_mean"])
            assert np.array_equal(out[nm]["sd"], d[f"{nm}_sd"])
            assert np.array_equal(out[nm]["quantiles"], d[f"{nm}_quantiles"])
    # recorded draws agree with the reference's hooked calls
    z = np.stack([rec["z"][t] for t in sorted(rec["z"])])
    assert np.array_equal(z, d["z"])


def test_feed_reproduces_reference():
    # oracle mode on the oracle itself: feeding the recorded draws is exact
    d = golden("run_pl")
    feed = {"z": d["z"], "g_sigma": d["g_sigma"], "g_tau": d["g_tau"]}
    out = R.run_loop(d["y"], int(d["n"]), int(d["seed"]), keep_indices=True, feed=feed,
                     **_oracle_kwargs(d))
    assert np.array_equal(out["indices"], d["indices"])


def test_kalman_hand_case():
    m, v = R.kalman_filter([2.0], 1.0, 0.0, 0.0, 10.0)
    assert m[0] == pytest.approx(20 / 11, rel=1e-14) and v[0] == pytest.approx(10 / 11, rel=1e-14)


@pytest.mark.filterwarnings("ignore:overflow encountered:RuntimeWarning")  # the degenerate weights themselves
def test_degenerate_step_raises():
    with pytest.raises(R.Degenerate) as ei:
        R.run_loop(np.array([1e200]), 16, 0, sigma2=1e-300, tau2=0.1)
    assert ei.value.step == 1
