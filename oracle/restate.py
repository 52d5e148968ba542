"""CPU restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *oracle*: a plain-numpy restatement of the reference
package ``parsmc`` (arXiv 1212.1639 particle filtering / particle learning),
used only by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` arm as the checker.  Nothing in the
product package (``paper_1212_1639_b200``) imports it; the product path runs
on the GPU through the C-ABI library and fails loudly when that is missing.

Every function cites the reference file:line it restates (paths relative to
the reference's ``pkg/src/parsmc/``).  Third-party arithmetic on the path is
called, not re-derived, because it is the reference's own dependency and is
installed in this image:

* ``scipy.special.ndtri`` / ``scipy.special.gammaincinv`` -- scipy>=1.10
  (pinned at ``pyproject.toml:10-15``; 1.18.1 installed).  Used at
  ``rng.py:223-229`` and ``filtering.py:280,286``.
* numpy ``exp``/``log``/``sum``/``dot``/``argsort``/``cumsum`` -- numpy>=1.24
  (2.3.5 installed).

Parity is *pinned*: ``tests/test_oracle_golden.py`` checks this restatement
against golden vectors produced by importing the reference itself
(``oracle/make_golden.py``) and against the reference test-suite's own
known-answer values (Table 1, Q4 traces, ...).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.special import gammaincinv, ndtri

# ---------------------------------------------------------------- Philox ---
# rng.py:24-27 -- Random123 Philox4x64 multipliers and Weyl key increments.
PHILOX_M0 = np.uint64(0xD2E7470EE14C6C93)
PHILOX_M1 = np.uint64(0xCA5A826395121157)
PHILOX_W0 = np.uint64(0x9E3779B97F4A7C15)
PHILOX_W1 = np.uint64(0xBB67AE8584CAA73B)
AUX_STREAM_BASE = 1 << 62  # rng.py:34
DATA_STREAM_ID = AUX_STREAM_BASE + 1  # bench.py:36

_LO32 = np.uint64(0xFFFFFFFF)
_SH32 = np.uint64(32)


def _mul_128(a, b):
    """(high, low) 64-bit halves of the 128-bit product a*b (rng.py:37-46)."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    with np.errstate(over="ignore"):
        low = a * b
        al, ah = a & _LO32, a >> _SH32
        bl, bh = b & _LO32, b >> _SH32
        mid = al * bh + ((al * bl) >> _SH32)
        high = ah * bh + (mid >> _SH32) + (((mid & _LO32) + ah * bl) >> _SH32)
    return high, low


def philox4x64_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox4x64 rounds (rng.py:49-63): returns the 4 output words."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) for c in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64)
    k1 = np.asarray(k1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for _ in range(10):
            h0, l0 = _mul_128(PHILOX_M0, c0)
            h1, l1 = _mul_128(PHILOX_M1, c2)
            c0, c1, c2, c3 = h1 ^ c1 ^ k0, l1, h0 ^ c3 ^ k1, l0
            k0 = k0 + PHILOX_W0
            k1 = k1 + PHILOX_W1
    return c0, c1, c2, c3


def unit_open(words):
    """uint64 -> (k + 1/2) 2^-52 with k = w >> 12, strictly inside (0,1)
    (rng.py:113-119)."""
    k = np.asarray(words, dtype=np.uint64) >> np.uint64(12)
    return (k.astype(np.float64) + 0.5) * 2.0**-52


def block_words(seed, stream_ids, block):
    """All 4 words of Philox block ``block`` for each stream id: key =
    (seed, stream_id), counter = (block, 0, 0, 0) (rng.py:66-110)."""
    ids = np.asarray(stream_ids, dtype=np.uint64)
    z = np.zeros_like(ids)
    b = np.full_like(ids, np.uint64(block))
    return np.stack(philox4x64_10(b, z, z, z, np.uint64(seed), ids))


def uniforms_at(seed, stream_ids, counters):
    """Uniform for each (stream, counter): word counter&3 of block counter>>2
    (rng.py:122-140)."""
    ids = np.asarray(stream_ids, dtype=np.uint64)
    ctr = np.asarray(counters, dtype=np.uint64)
    ids, ctr = np.broadcast_arrays(ids, ctr)
    z = np.zeros(ids.shape, dtype=np.uint64)
    w = np.stack(philox4x64_10(ctr >> np.uint64(2), z, z, z, np.uint64(seed), ids))
    sel = (ctr & np.uint64(3)).astype(np.int64)
    out = np.take_along_axis(w.reshape(4, -1), sel.reshape(1, -1), axis=0).reshape(ids.shape)
    return unit_open(out)


def stream_normals(seed, stream_id, counter, count):
    """``RngStream(seed, stream_id, counter).normals(count)`` (rng.py:148-157)."""
    ctr = np.uint64(counter) + np.arange(count, dtype=np.uint64)
    return ndtri(uniforms_at(seed, np.uint64(stream_id), ctr))


# ------------------------------------------------------------ model spec ---
LOG_TWO_PI = math.log(2.0 * math.pi)  # models.py:20


def simulate(sigma2, tau2, x0_mean, t_len, seed, stream_id=DATA_STREAM_ID):
    """models.py:91-102: 2T normals from one stream; states = x0 + cumsum."""
    z = stream_normals(seed, stream_id, 0, 2 * t_len)
    eps = math.sqrt(tau2) * z[:t_len]
    nu = math.sqrt(sigma2) * z[t_len:]
    states = x0_mean + np.cumsum(eps)
    return states, states + nu


def kalman_filter(y, sigma2, tau2, m0=0.0, c0=10.0):
    """models.py:128-147: exact local-level recursion."""
    means = np.empty(len(y))
    variances = np.empty(len(y))
    m, c = float(m0), float(c0)
    for t, yt in enumerate(np.asarray(y, dtype=np.float64)):
        r = c + tau2
        k = r / (r + sigma2)
        m = m + k * (yt - m)
        c = (1.0 - k) * r
        means[t] = m
        variances[t] = c
    return means, variances


# ------------------------------------------------------------- tree CDF ---
class Lanes:
    """Contiguous-range lane runner with a barrier per call -- the
    reference's ``Backend`` (backend.py:15-70).  Results never depend on the
    lane count; only wall time does."""

    def __init__(self, lanes=1, min_chunk=4096):
        self.lanes = max(1, int(lanes))
        self.min_chunk = min_chunk
        self._pool = ThreadPoolExecutor(self.lanes) if self.lanes > 1 else None

    def split(self, n):  # backend.py:39-50
        k = min(self.lanes, max(1, n // self.min_chunk))
        base, extra = divmod(n, k)
        out, lo = [], 0
        for i in range(k):
            hi = lo + base + (1 if i < extra else 0)
            if hi > lo:
                out.append((lo, hi))
            lo = hi
        return out

    def run(self, n, fn):  # backend.py:52-70
        if n <= 0:
            return
        ranges = self.split(n)
        if self._pool is None or len(ranges) == 1:
            for lo, hi in ranges:
                fn(lo, hi)
            return
        for f in [self._pool.submit(fn, lo, hi) for lo, hi in ranges]:
            f.result()

    def close(self):
        if self._pool is not None:
            self._pool.shutdown()
            self._pool = None


_SERIAL = Lanes(1)


def forward_adder(w, lanes=_SERIAL):
    """prefix_sum.py:46-69: levels[d][i] = levels[d-1][2i] + levels[d-1][2i+1]."""
    w = np.asarray(w)
    n = len(w)
    if n < 1 or n & (n - 1):
        raise ValueError(f"power-of-two length required, got {n}")
    levels = [w]
    prev = w
    while len(prev) > 1:
        out = np.empty(len(prev) // 2, dtype=prev.dtype)

        def comb(lo, hi, prev=prev, out=out):
            out[lo:hi] = prev[2 * lo:2 * hi:2] + prev[2 * lo + 1:2 * hi:2]

        lanes.run(len(out), comb)
        levels.append(out)
        prev = out
    return levels


def backward_adder(levels, lanes=_SERIAL):
    """prefix_sum.py:72-91: right child = parent; left child = parent minus
    the forward sum of its right sibling.  Returns inclusive prefix sums."""
    s = levels[-1].copy()
    for d in range(len(levels) - 2, -1, -1):
        w = levels[d]
        child = np.empty(len(w), dtype=s.dtype)

        def branch(lo, hi, parent=s, w=w, child=child):
            child[2 * lo + 1:2 * hi:2] = parent[lo:hi]
            child[2 * lo:2 * hi:2] = parent[lo:hi] - w[2 * lo + 1:2 * hi:2]

        lanes.run(len(s), branch)
        s = child
    return s


def finalize_cdf(prefix, total):
    """prefix_sum.py:94-106: divide, running max, clip [0,1], pin last = 1.
    Returns None where the reference raises AllWeightsZeroError."""
    if not np.isfinite(total) or total <= 0:
        return None
    q = prefix / total
    np.maximum.accumulate(q, out=q)
    np.clip(q, q.dtype.type(0), q.dtype.type(1), out=q)
    q[-1] = 1
    return q


def tree_cdf(w, lanes=_SERIAL):
    """parallel_cdf (prefix_sum.py:109-127) without the pad option."""
    levels = forward_adder(np.asarray(w), lanes)
    return finalize_cdf(backward_adder(levels, lanes), levels[-1][0])


def tree_cdf_chunked(w, chunk):
    """Two-level restatement of the same tree: per-chunk subtrees, a top tree
    over chunk totals, and a per-chunk backward pass seeded from the chunk's
    node value -- the decomposition the device kernels use.  Bit-identical to
    :func:`tree_cdf` (asserted in tests)."""
    w = np.asarray(w)
    n = len(w)
    chunk = min(chunk, n)
    g = n // chunk
    sub = w.reshape(g, chunk)
    # forward inside chunks (same pairing as forward_adder restricted to a subtree)
    lv = [sub]
    while lv[-1].shape[1] > 1:
        p = lv[-1]
        lv.append(p[:, 0::2] + p[:, 1::2])
    totals = lv[-1][:, 0]
    top = forward_adder(totals)
    node = backward_adder(top)  # inclusive prefix at every chunk end
    s = node.reshape(g, 1)
    for d in range(len(lv) - 2, -1, -1):
        wd = lv[d]
        child = np.empty_like(wd)
        child[:, 1::2] = s
        child[:, 0::2] = s - wd[:, 1::2]
        s = child
    return finalize_cdf(s.reshape(n), top[-1][0])


def shard_exchange(totals, n_total):
    """Host restatement of the sharded CDF exchange (the device's
    cdf_top_shard_kernel): from the G shard subtree totals (each a node of
    the adder tree, prefix_sum.py:64), rebuild the top levels -> the root,
    run the backward adder (prefix_sum.py:86-87) down to every shard node,
    and derive each shard's carry (running max of the shard nodes before it;
    a node never exceeds its parent) and stratum bound L_end = ceil(N q_end)
    (resampling.py:124).  Returns (root, nodes, carries, lend)."""
    totals = np.asarray(totals)
    top = forward_adder(totals)
    nodes = backward_adder(top)
    root = top[-1][0]
    carries = np.empty_like(nodes)
    lend = np.empty(len(nodes), dtype=np.int64)
    m = totals.dtype.type(-np.inf)
    for g in range(len(nodes)):
        carries[g] = m
        m = max(m, nodes[g])
        qe = totals.dtype.type(1) if g == len(nodes) - 1 else min(max(m / root, 0), 1)
        lend[g] = int(np.ceil(totals.dtype.type(qe) * totals.dtype.type(n_total)))
    return root, nodes, carries, lend


def tree_cdf_shard(w_shard, shard, node, carry, root, n_total):
    """The CDF values of one shard's particles given its node value and
    carry from :func:`shard_exchange`: backward adder inside the shard's
    subtree, divide by the root, running max seeded with the carry, clip,
    pin the global last element (prefix_sum.py:72-106)."""
    w_shard = np.asarray(w_shard)
    ns = len(w_shard)
    lv = forward_adder(w_shard)
    lv[-1] = np.array([node], dtype=w_shard.dtype)
    s = backward_adder(lv)
    q = s / root
    q = np.maximum.accumulate(np.concatenate([[carry / root], q]))[1:]
    np.clip(q, q.dtype.type(0), q.dtype.type(1), out=q)
    if (shard + 1) * ns == n_total:
        q[-1] = 1
    return q


# ------------------------------------------------------------ cut points ---
def cut_points(q):
    """resampling.py:110-134: L_j = ceil(N q_j); slots (L_{j-1}, L_j] get j
    (1-based)."""
    q = np.asarray(q)
    n = len(q)
    bounds = np.ceil(q * q.dtype.type(n)).astype(np.int64)
    counts = np.diff(bounds, prepend=0)
    out = np.empty(n, dtype=np.int64)
    out[: bounds[-1]] = np.repeat(np.arange(1, n + 1, dtype=np.int64), counts)
    return out


def cut_points_bruteforce(q):
    """resampling.py:93-107: idx[j] = min{ i : q(i) > (j-1)/N } (1-based)."""
    q = np.asarray(q)
    n = len(q)
    thr = np.arange(n, dtype=q.dtype) / q.dtype.type(n)
    return np.argmax(q[None, :] > thr[:, None], axis=1).astype(np.int64) + 1


def cutpoint_indices(q, cuts, u):
    """resampling.py:146-158: k = I[ceil(N u)]; advance while u > q(k)."""
    q = np.asarray(q)
    n = len(q)
    k = cuts[np.ceil(u * n).astype(np.int64) - 1].copy()
    active = u > q[k - 1]
    while active.any():
        k[active] += 1
        (where,) = np.nonzero(active)
        active[where] = u[where] > q[k[where] - 1]
    return k


# --------------------------------- K7 ordered uniforms (perf mode, B200) ---
SPACINGS_STREAM = AUX_STREAM_BASE + 2


def spacings_uniforms(words, seed, t):
    """The ordered uniforms of the B200 `spacings` resampler (csrc/cdf.cuh K7;
    not a reference algorithm -- a restatement of ours, checked statistically
    against the reference's exact `sorted` scheme, resampling.py:57-67):
    E_j = -log(unit_open(w3_j)), S = cumsum(E), E_aux from stream 2^62+2
    block t word 0, U_k = S_k / (S_N + E_aux), snapped to the odd 53-bit grid
    of unit_open (K = floor(U 2^53) | 1)."""
    e = -np.log(unit_open(np.asarray(words, dtype=np.uint64)))
    s = np.cumsum(e)
    aux = -math.log(float(unit_open(block_words(seed, np.array([SPACINGS_STREAM], dtype=np.uint64), t)[0])[0]))
    u = s * (1.0 / (s[-1] + aux))
    k = np.floor(u * 2.0 ** 53).astype(np.uint64) | np.uint64(1)
    k = np.minimum(k, np.uint64(2 ** 53 - 1))
    return k.astype(np.float64) * 2.0 ** -53


def spacings_uniforms_shard(words_local, totals, shard, seed, t):
    """Sharded K7 (csrc/cdf.cuh spacings_words_kernel): shard `shard` scans its
    own exponentials; `totals` are every shard's sums (exchanged), giving its
    offset and the grand total S_(N+1) = sum(totals) + E_aux."""
    e = -np.log(unit_open(np.asarray(words_local, dtype=np.uint64)))
    s = np.cumsum(e)
    off = float(sum(totals[:shard]))
    tot = float(sum(totals))
    aux = -math.log(float(unit_open(block_words(seed, np.array([SPACINGS_STREAM], dtype=np.uint64), t)[0])[0]))
    u = (off + s) * (1.0 / (tot + aux))
    k = np.floor(u * 2.0 ** 53).astype(np.uint64) | np.uint64(1)
    k = np.minimum(k, np.uint64(2 ** 53 - 1))
    return k.astype(np.float64) * 2.0 ** -53


def spacings_indices(q, cuts, words, seed, t):
    """1-based ancestors of the spacings resampler: the cut-point lookup of the
    ordered uniforms (nondecreasing in the slot)."""
    return cutpoint_indices(q, cuts, spacings_uniforms(words, seed, t))


# ------------------------------------------- sequential baselines (CPU) ---
def sequential_cdf(w):
    """prefix_sum.py:130-134: plain left-to-right cumsum (in the weights'
    dtype), finalised against its own last element."""
    w = np.asarray(w)
    prefix = np.cumsum(w)
    return finalize_cdf(prefix, prefix[-1])


def merge_indices(q, u):
    """resampling.py:29-36: smallest 1-based i with u < q(i)."""
    return np.searchsorted(q, u, side="right") + 1


def resample_uniforms(scheme, u_slot, n, v_aux=None):
    """The uniforms each baseline resampler searches for (resampling.py:
    51-87): naive -> the slot's own uniform; sorted -> all of them sorted;
    stratified -> (j + v_j)/n; systematic -> (j + v)/n with one aux draw."""
    if scheme == "naive":
        return u_slot
    if scheme == "sorted":
        return np.sort(u_slot)
    if scheme == "stratified":
        return (np.arange(n) + u_slot) / n
    if scheme == "systematic":
        return (np.arange(n) + v_aux) / n
    raise ValueError(scheme)


# -------------------------------------------------------------- summaries --
PARAM_PROBS = (0.005, 0.05, 0.5, 0.95, 0.995)  # filtering.py:40
STATE_PROBS = (0.05, 0.5, 0.95)  # filtering.py:41


def weighted_quantiles(values, weights, probs):
    """filtering.py:135-140: smallest value (stable order) with cum-weight >= pW."""
    order = np.argsort(values, kind="stable")
    cw = np.cumsum(weights[order], dtype=np.float64)
    pos = np.searchsorted(cw, np.asarray(probs) * cw[-1], side="left")
    return np.asarray(values, dtype=np.float64)[order[np.minimum(pos, len(order) - 1)]]


def param_summary_row(draws, weights, w_sum):
    """filtering.py:151-155."""
    mean = float(np.dot(weights, draws) / w_sum)
    var = float(np.dot(weights, (draws - mean) ** 2) / w_sum)
    return mean, math.sqrt(max(var, 0.0)), weighted_quantiles(draws, weights, PARAM_PROBS)


# ------------------------------------------------------------ driver loop --
class Degenerate(Exception):
    """Where the reference raises AllWeightsZeroError(step=t)."""

    def __init__(self, step):
        super().__init__(f"all particle weights are zero (at time step {step})")
        self.step = step


def run_loop(y, n, seed=0, *, x0_mean=0.0, x0_var=10.0,
             sigma2=(5.0, 4.0), tau2=(5.0, 0.4), precision="double",
             track_quantiles=True, keep_indices=False, keep_final=False,
             lanes=_SERIAL, feed=None, record=None, resampler="cutpoint"):
    """Restatement of ``filtering._run_loop`` (filtering.py:200-374) for the
    cut-point resampler.

    ``sigma2``/``tau2`` are ``(shape, scale)`` inverse-gamma priors (the
    parameter is learned) or plain floats (known, as in run_particle_filter
    and in ``Priors`` with a fixed value, models.py:57-88).  ``feed`` may hold
    per-step arrays ``z``, ``g_sigma``, ``g_tau`` of shape [T+1, n] (row 0 =
    init) replacing the ndtri/gammaincinv outputs -- the oracle-mode noise
    injection.  ``record`` (a dict) receives per-step z, g, lw, w, u, idx.
    """
    y = np.asarray(y, dtype=np.float64)
    n = int(n)
    dtype = np.float64 if precision == "double" else np.float32
    learn_s = isinstance(sigma2, tuple)
    learn_t = isinstance(tau2, tuple)
    ids = np.arange(n, dtype=np.uint64)
    t_len = len(y)

    def words(block):
        return block_words(seed, ids, block)

    def rec(key, t, val):
        if record is not None:
            record.setdefault(key, {})[t] = np.array(val, copy=True)

    def normal(w, t):
        z = feed["z"][t] if feed is not None else ndtri(unit_open(w))
        rec("z", t, z)
        return z

    def gamma(w, a, key, t):
        if feed is not None:
            g = feed[key][t]
        else:
            g = gammaincinv(a, unit_open(w))
        rec(key, t, g)
        return g

    # init (filtering.py:220-252): block 0, slots 0..2, slot 3 unused
    w0 = words(0)
    states = (x0_mean + math.sqrt(x0_var) * normal(w0[0], 0)).astype(dtype)
    a_s = b_s = a_t = b_t = None
    if learn_s:
        a_s = np.full(n, float(sigma2[0]))
        b_s = np.full(n, float(sigma2[1]))
        s2 = b_s / gamma(w0[1], a_s, "g_sigma", 0)
    else:
        s2 = float(sigma2)
    if learn_t:
        a_t = np.full(n, float(tau2[0]))
        b_t = np.full(n, float(tau2[1]))
        t2 = b_t / gamma(w0[2], a_t, "g_tau", 0)
    else:
        t2 = float(tau2)

    out = {
        "filtered_mean": np.empty(t_len),
        "filtered_quantiles": np.empty((t_len, 3)) if track_quantiles else None,
        "indices": np.empty((t_len, n), dtype=np.int64) if keep_indices else None,
    }
    for name, on in (("sigma2", learn_s), ("tau2", learn_t)):
        if on:
            out[name] = {"mean": np.empty(t_len), "sd": np.empty(t_len),
                         "quantiles": np.empty((t_len, 5))}

    for t in range(1, t_len + 1):
        yt = float(y[t - 1])
        wt = words(t)
        # propagate (filtering.py:272-290)
        z = normal(wt[0], t)
        step = np.sqrt(t2) * z
        new_states = (states + step).astype(dtype, copy=False)
        resid = yt - new_states.astype(np.float64, copy=False)
        if learn_s:
            b_s = b_s + 0.5 * resid * resid
            a_s = a_s + 0.5
            s2 = b_s / gamma(wt[1], a_s, "g_sigma", t)
        if learn_t:
            b_t = b_t + 0.5 * step * step
            a_t = a_t + 0.5
            t2 = b_t / gamma(wt[2], a_t, "g_tau", t)
        states = new_states
        # weights + CDF (filtering.py:292-303)
        lw = -0.5 * (LOG_TWO_PI + np.log(s2)) - 0.5 * resid * resid / s2
        rec("lw", t, lw)
        shift = float(np.max(lw))
        if not math.isfinite(shift):
            raise Degenerate(t)
        wts = np.exp(lw - shift).astype(dtype, copy=False)
        if feed is not None and "w" in feed:
            wts = feed["w"][t].astype(dtype)
        rec("w", t, wts)
        w_sum = float(wts.sum(dtype=np.float64))
        # cutpoint: the adder tree; the baselines: a sequential cumsum
        # (filtering.py:299-302)
        q = tree_cdf(wts, lanes) if resampler in ("cutpoint", "spacings") else sequential_cdf(wts)
        if q is None:
            raise Degenerate(t)
        # resample (filtering.py:305-317) with u = slot 3 of block t
        u = unit_open(wt[3])
        if resampler == "spacings":  # B200 perf mode (K7)
            idx = spacings_indices(q, cut_points(q), wt[3], seed, t)
        elif resampler == "cutpoint":  # resampling.py:161-177
            cuts = cut_points(q)
            idx = np.empty(n, dtype=np.int64)

            def lane(lo, hi):
                idx[lo:hi] = cutpoint_indices(q, cuts, u[lo:hi])

            lanes.run(n, lane)
        else:
            # systematic draws one uniform from the aux stream 2^62 (counter t-1)
            v_aux = (uniforms_at(seed, np.array([AUX_STREAM_BASE], dtype=np.uint64),
                                 np.array([t - 1], dtype=np.uint64))[0]
                     if resampler == "systematic" else None)
            idx = merge_indices(q, resample_uniforms(resampler, u, n, v_aux))
        rec("u", t, u)
        rec("idx", t, idx)
        take = idx - 1
        pre_x, pre_s2, pre_t2 = states, s2, t2
        states = states[take]
        if learn_s:
            s2, a_s, b_s = s2[take], a_s[take], b_s[take]
        if learn_t:
            t2, a_t, b_t = t2[take], a_t[take], b_t[take]
        # summaries from the weighted pre-resample set (filtering.py:344-357)
        out["filtered_mean"][t - 1] = np.dot(wts, pre_x) / w_sum
        if track_quantiles:
            out["filtered_quantiles"][t - 1] = weighted_quantiles(pre_x, wts, STATE_PROBS)
        for name, draws, on in (("sigma2", pre_s2, learn_s), ("tau2", pre_t2, learn_t)):
            if on:
                m, sd, qq = param_summary_row(draws, wts, w_sum)
                out[name]["mean"][t - 1] = m
                out[name]["sd"][t - 1] = sd
                out[name]["quantiles"][t - 1] = qq
        if keep_indices:
            out["indices"][t - 1] = idx
    if keep_final:
        def arr(v):
            return v if isinstance(v, np.ndarray) else np.full(n, v)
        out["final"] = {"states": states.copy(), "sigma2": arr(s2), "tau2": arr(t2),
                        "a_sigma": arr(a_s if a_s is not None else 0.0),
                        "b_sigma": arr(b_s if b_s is not None else 0.0),
                        "a_tau": arr(a_t if a_t is not None else 0.0),
                        "b_tau": arr(b_t if b_t is not None else 0.0)}
    return out
