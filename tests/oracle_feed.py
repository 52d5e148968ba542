"""Oracle-mode inputs at large N, built in parallel on the host.

The reference's noise draws for oracle mode -- z = ndtri(u0), g_sigma =
gammaincinv(a_t, u1), g_tau = gammaincinv(a_t, u2) from Philox block t of
every particle stream (rng.py:221-229, filtering.py:225-252,272-290) -- are
regenerated with the oracle's Philox (oracle/restate.py block_words) and
scipy, the reference's own pinned dependency.  scipy's gammaincinv is
single-threaded and ~0.6 us per value, so at N = 2^22..2^24 the rows are
computed over a process pool.  Test infrastructure only.
"""

from __future__ import annotations

import os
from multiprocessing import get_context

import numpy as np

from oracle import restate as R

_CHUNK = 1 << 20


def _rows(args):
    seed, lo, hi, block, a_s, a_t = args
    from scipy.special import gammaincinv, ndtri

    ids = np.arange(lo, hi, dtype=np.uint64)
    w = R.block_words(seed, ids, block)
    z = ndtri(R.unit_open(w[0]))
    gs = gammaincinv(a_s, R.unit_open(w[1])) if a_s else None
    gt = gammaincinv(a_t, R.unit_open(w[2])) if a_t else None
    return lo, z, gs, gt


def shapes(a0, t_len):
    """a_t for t = 0..T as the reference accumulates it (a = a + 0.5 per
    step, filtering.py:279,285)."""
    a = [float(a0)]
    for _ in range(t_len):
        a.append(a[-1] + 0.5)
    return a


def make_feed(n, t_len, seed, sigma2_shape=5.0, tau2_shape=5.0, procs=None):
    """{"z", "g_sigma", "g_tau"} of shape [T+1, n] (row 0 = init); a shape of
    0 / None means that variance is known (no gamma row)."""
    procs = procs or min(32, os.cpu_count() or 1)
    feed = {"z": np.empty((t_len + 1, n))}
    sa = shapes(sigma2_shape, t_len) if sigma2_shape else None
    ta = shapes(tau2_shape, t_len) if tau2_shape else None
    if sa:
        feed["g_sigma"] = np.empty((t_len + 1, n))
    if ta:
        feed["g_tau"] = np.empty((t_len + 1, n))
    jobs = [(seed, lo, min(n, lo + _CHUNK), t, sa[t] if sa else None, ta[t] if ta else None)
            for t in range(t_len + 1) for lo in range(0, n, _CHUNK)]
    with get_context("spawn").Pool(procs) as pool:
        for (lo, z, gs, gt), job in zip(pool.imap(_rows, jobs), jobs):
            t, hi = job[3], job[2]
            feed["z"][t, lo:hi] = z
            if gs is not None:
                feed["g_sigma"][t, lo:hi] = gs
            if gt is not None:
                feed["g_tau"][t, lo:hi] = gt
    return feed
