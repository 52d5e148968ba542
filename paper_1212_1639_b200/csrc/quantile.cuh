// Exact weighted quantiles of the per-step particle summaries
// (filtering.py:135-155: smallest value, in stable value order, whose
// cumulative weight reaches p * W), without sorting N values per step.
//
//  1. The step kernel writes a 32-bit monotone key per particle and quantity
//     (float32 rounded down, order-preserving bit image) and the step's
//     weighted mean / sd of each quantity.
//  2. The CDF reduce pass (which already forms the exact weight w) predicts a
//     narrow key window per target -- mean_t + sd_t * (standardized quantile
//     of step t-1) +- h -- and, per particle, adds w to "weight below the
//     window" or appends (key, index, w) to the target's candidate list.
//  3. On a side stream, per target: a fixed-point (exact, order-independent)
//     sub-bin histogram of the candidates locates the sub-bin holding the
//     crossing; the candidates of that sub-bin and its neighbours are ordered
//     by their exact value (recomputed from the particle record) and index
//     (argsort(kind="stable")), and summed in that order from the exact
//     weight below them.  The window half-width h adapts to the observed
//     prediction error.
//  4. If the crossing is not inside the window (or the window overflowed),
//     conditional fallback kernels histogram the missed interval over all
//     particles, re-window to one bin and resolve again.  They exit at once
//     when nothing missed.
// The weight sums differ from numpy's sequential cumsum only in rounding, so
// a quantile can move by one order statistic only at an exact near-tie.
#pragma once
#include "step.cuh"

namespace pf {

constexpr int Q_MAXQ = 3;        // quantities: 0 = x, 1 = sigma2, 2 = tau2
constexpr int Q_MAXT = 13;       // targets: 3 state + 5 + 5 parameter probs
constexpr int Q_SUB = 2048;      // sub-bins per window
constexpr int Q_FB = 4096;       // fallback bins per missed interval
constexpr int Q_LIST = 4096;     // exact-resolve list capacity (per target)
constexpr int Q_RESOLVE_SMEM = Q_LIST * (8 + 8 + 4);
// Window half-widths: the first step's (standardized units), then sized in
// probability mass from the observed prediction error.  Narrow windows keep
// the candidate lists short; a miss costs the fallback passes (two sweeps),
// which is cheaper than classifying a few percent of all particles as
// candidates every step.
constexpr double Q_H0 = 0.05;
#ifndef PF_Q_MASS_MIN
#define PF_Q_MASS_MIN 1.25e-4
#endif
#ifndef PF_Q_MASS_MAX
#define PF_Q_MASS_MAX 0.012
#endif
#ifndef PF_Q_MASS_K
#define PF_Q_MASS_K 6.0
#endif
constexpr double Q_MASS_MIN = PF_Q_MASS_MIN;
constexpr double Q_MASS_MAX = PF_Q_MASS_MAX;
constexpr double Q_MASS_K = PF_Q_MASS_K;  // half-width in units of the recent prediction error

enum : uint32_t { QS_OK = 0, QS_MISS_LO = 1, QS_MISS_HI = 2, QS_OVERFLOW = 3, QS_CROWD = 4,
                  QS_REFILL = 5, QS_FB = 6, QS_RETRY = 7, QS_LOCATED = 8 };

PF_HD uint32_t key_of_float(float f) {
  union { float f; uint32_t u; } c;
  c.f = f;
  return (c.u & 0x80000000u) ? ~c.u : (c.u | 0x80000000u);
}
PF_D uint32_t key_rd(double v) { return key_of_float(__double2float_rd(v)); }
PF_D uint32_t key_ru(double v) { return key_of_float(__double2float_ru(v)); }

struct QCand {
  uint32_t key;
  uint32_t idx;
  double w;
};

// Persistent (across steps) per-target state + per-step scratch.
struct QTarget {
  double p;          // probability
  int q;             // quantity
  int col;           // output column
  double zprev;      // standardized quantile of the previous step
  double h;          // window half-width (standardized units)
  double ema;        // running prediction error
  // per step
  uint32_t klo, khi; // key window (inclusive)
  double wbelow;     // weight with key < klo
  uint32_t count;    // candidates appended
  uint32_t status;
  uint32_t ilo, ihi; // fallback interval
  double ibelow;     // weight below the fallback interval
  uint32_t missed;   // the predicted window missed this step
  double wmass;      // candidate weight inside the window
  int side;          // fallback retry side (-1 below, +1 above)
  int bstar;         // crossing sub-bin
  double cum0;       // weight below sub-bin bstar-1
  uint32_t nlist;    // candidates kept for the exact resolve
};

PF_HD double normal_pdf(double z) { return 0.3989422804014327 * exp(-0.5 * z * z); }

struct QShared {
  double W;                    // total weight of the step (fp64 sum of w)
  double mean[Q_MAXQ], sd[Q_MAXQ];
  unsigned int counter;        // last-CTA ticket of the reduce pass
  unsigned int fb_counter;
  int any_miss;
  int fb_active[2];
  int ntarget;
};

struct QArgs {
  int ntarget;                 // 0 = quantiles off
  QTarget* tg;
  QShared* sh;
  const uint32_t* keys[Q_MAXQ];  // this step's keys (null if quantity absent)
  QCand* cand;                 // [ntarget][cap]
  uint32_t cap;
  double* part;                // reduce-pass partials [grid][Q_MAXT+1]
  unsigned long long* hist;    // [ntarget][Q_SUB] fixed-point weights
  unsigned long long* fhist;   // [ntarget][Q_FB]
  double fx_scale;             // fixed-point units per unit weight
  unsigned int* stats;         // [0] unresolved, [1] fallbacks, [2] max candidates, [3] resolves
  uint32_t* lidx;              // [ntarget][Q_LIST] exact-resolve lists
  double* lw;
  // sharded runs: every shard's passes feed shard 0's state; partial slots
  // pbase + block of ptotal (0: this launch alone), particle index offset
  int pbase, ptotal;
  uint32_t gbase;
  // batched replications (gridDim.z = R, step.cuh RepStride): per-replication
  // strides of the slot arrays, the partial slots and the [T] output rows
  int64_t rslots, rpart, rT;
};

// Replication blockIdx.z's quantile state: targets [R][Q_MAXT], shared pair
// [R][2] (by parity), candidates [R][ntarget cap], partials, histograms and
// lists [R][...]; the stats counters are shared (atomic).
PF_D void q_rep(QArgs& qa) {
  const int64_t r = blockIdx.z;
  if (r == 0) return;
  qa.tg += r * Q_MAXT;
  qa.sh += 2 * r;
#pragma unroll
  for (int q = 0; q < Q_MAXQ; ++q)
    if (qa.keys[q]) qa.keys[q] += r * qa.rslots;
  qa.cand += r * (int64_t)qa.ntarget * qa.cap;
  qa.part += r * qa.rpart;
  qa.hist += r * (int64_t)Q_MAXT * Q_SUB;
  qa.fhist += r * (int64_t)Q_MAXT * Q_FB;
  qa.lidx += r * (int64_t)Q_MAXT * Q_LIST;
  qa.lw += r * (int64_t)Q_MAXT * Q_LIST;
}

PF_D int q_pslot(const QArgs& qa) { return qa.pbase + (int)blockIdx.x; }
PF_D unsigned q_ptotal(const QArgs& qa) { return qa.ptotal ? (unsigned)qa.ptotal : gridDim.x; }

// Window of target k for this step from mean/sd of its quantity.
PF_D void window_of(const QTarget& t, double mean, double sd, uint32_t* lo, uint32_t* hi) {
  if (!(sd > 0.0) || !isfinite(sd) || !isfinite(mean)) {
    *lo = 0u;
    *hi = 0xFFFFFFFFu;
    return;
  }
  const double c = mean + sd * t.zprev;
  *lo = key_rd(c - t.h * sd);
  *hi = key_ru(c + t.h * sd);
}

// floor((key - lo) nb / (hi - lo + 1)) for lo <= key <= hi, nb <= 4096, in
// fp64: the numerator (< 2^44) and denominator (<= 2^32) are exact, and a
// non-integer quotient (< 2^12) lies at least 2^-32 from an integer -- far
// beyond the division's 2^-41 absolute rounding -- so the truncation is the
// exact integer quotient (a 64-bit integer division costs ~4x the issue).
PF_D uint32_t sub_bin(uint32_t key, uint32_t lo, uint32_t hi, int nb) {
  const double num = (double)(key - lo) * (double)nb;
  const double den = (double)((uint64_t)(hi - lo) + 1);
  return (uint32_t)(num / den);
}

// Exact value of quantity q for particle idx at step t (resolve side).
struct QValueSrc {
  const Rec* rec;        // records written by step t (single run)
  const Rec* recs[PF_MAX_SHARDS];  // sharded run: per-shard records, nsh > 0
  int nsh, lg;
  uint64_t seed;
  const uint64_t* seedp; // non-null: read the seed from device memory (graph replays)
  int64_t t;
  GammaSrc gs;           // step t's sigma2 table
  const double* feed_gs; // oracle feed row t
  double sigma2_fixed, tau2_fixed;
  int learn_s, learn_t;
};

PF_D double quantity_value(const QValueSrc& s, int q, uint32_t idx) {
  const Rec r = s.nsh ? s.recs[idx >> s.lg][idx & ((1u << s.lg) - 1u)] : s.rec[idx];
  if (q == 0) return r.x;
  if (q == 2) return s.learn_t ? r.tau2 : s.tau2_fixed;
  if (!s.learn_s) return s.sigma2_fixed;
  double g;
  if (s.feed_gs) {
    g = s.feed_gs[idx];
  } else {
    const Philox4 P = philox_block(s.seedp ? *s.seedp : s.seed, (uint64_t)idx, (uint64_t)s.t);
    g = gamma_draw(s.gs, unit_open(P.w[1]));
  }
  return r.bs / g;
}

// --------------------------------------------- classify (in CDF reduce) ---
// Called by cdf_reduce for every element; accumulates below-window weight
// into acc[k] and appends window candidates (warp-aggregated).
// Windows of a step per quantity q; classification slot s = q * Q_PER + k
// holds target base[q] + k.  Static slot indices keep the bounds and the
// below-window sums in registers.
constexpr int Q_PER = 5;                  // max targets per quantity
constexpr int Q_SLOTS = Q_MAXQ * Q_PER;   // 15
struct QWin {
  uint32_t lo[Q_SLOTS], hi[Q_SLOTS];
  int nq[Q_MAXQ];    // targets of quantity q
  int base[Q_MAXQ];  // index of its first target in qa.tg
};

// CTA-level candidate staging (shared memory).
constexpr int Q_AGG = 512;
struct QAgg {
  QCand c[Q_AGG];
  uint32_t pos[Q_AGG];
  uint8_t tk[Q_AGG];
  uint32_t cnt[Q_MAXT];
  uint32_t base[Q_MAXT];
  int fill;
};

PF_D void q_agg_init(QAgg& agg) {
  if (threadIdx.x == 0) agg.fill = 0;
  if (threadIdx.x < Q_MAXT) agg.cnt[threadIdx.x] = 0;
}

PF_D void q_classify(const QArgs& qa, const QWin& win, QAgg& agg, uint32_t i, double w,
                     double (&acc)[Q_SLOTS], bool valid) {
  const int lane = threadIdx.x & 31;
  uint32_t key[Q_MAXQ];
  uint32_t inwin = 0;
#pragma unroll
  for (int q = 0; q < Q_MAXQ; ++q) {
    key[q] = (valid && win.nq[q]) ? qa.keys[q][i] : 0u;
#pragma unroll
    for (int k = 0; k < Q_PER; ++k) {
      const int s = q * Q_PER + k;
      if (k < win.nq[q] && valid) {
        if (key[q] < win.lo[s]) acc[s] += w;
        else if (key[q] <= win.hi[s]) inwin |= 1u << s;
      }
    }
  }
  uint32_t any = __reduce_or_sync(0xffffffffu, inwin);
  while (any) {
    const int s = __ffs(any) - 1;
    any &= any - 1;
    const int q = s / Q_PER;
    const int qb = q == 0 ? win.base[0] : (q == 1 ? win.base[1] : win.base[2]);  // static indices
    const int t = qb + (s - q * Q_PER);
    const unsigned m = __ballot_sync(0xffffffffu, (inwin >> s) & 1u);
    const int leader = __ffs(m) - 1;
    // stage in the CTA buffer (shared atomics); spill straight to the global
    // list (one global atomic per warp) only if the buffer is full
    int slot = 0;
    uint32_t kpos = 0;
    if (lane == leader) {
      slot = atomicAdd(&agg.fill, __popc(m));
      if (slot + __popc(m) <= Q_AGG) kpos = atomicAdd(&agg.cnt[t], (uint32_t)__popc(m));
      else kpos = 0x80000000u | atomicAdd(&qa.tg[t].count, (uint32_t)__popc(m));
    }
    slot = __shfl_sync(0xffffffffu, slot, leader);
    kpos = __shfl_sync(0xffffffffu, kpos, leader);
    if ((inwin >> s) & 1u) {
      const uint32_t rank = __popc(m & ((1u << lane) - 1u));
      QCand c;
      c.key = q == 0 ? key[0] : (q == 1 ? key[1] : key[2]);
      c.idx = i;
      c.w = w;
      if (kpos & 0x80000000u) {
        const uint32_t pos = (kpos & 0x7FFFFFFFu) + rank;
        if (pos < qa.cap) qa.cand[(size_t)t * qa.cap + pos] = c;
        if (slot + (int)rank < Q_AGG) agg.tk[slot + rank] = 0xFF;  // reserved, unused
      } else {
        agg.c[slot + rank] = c;
        agg.tk[slot + rank] = (uint8_t)t;
        agg.pos[slot + rank] = kpos + rank;
      }
    }
  }
}

// Flush the CTA's staged candidates: one global atomic per target reserves
// space, then the whole CTA copies.  Called by all threads.
PF_D void q_flush(const QArgs& qa, QAgg& agg) {
  __syncthreads();
  if (threadIdx.x < Q_MAXT) {
    const uint32_t c = agg.cnt[threadIdx.x];
    agg.base[threadIdx.x] = c ? atomicAdd(&qa.tg[threadIdx.x].count, c) : 0u;
  }
  __syncthreads();
  const int nfill = min(agg.fill, Q_AGG);
  for (int s = threadIdx.x; s < nfill; s += blockDim.x) {
    const int k = agg.tk[s];
    if (k == 0xFF) continue;
    const uint32_t pos = agg.base[k] + agg.pos[s];
    if (pos < qa.cap) qa.cand[(size_t)k * qa.cap + pos] = agg.c[s];
  }
  __syncthreads();
  if (threadIdx.x == 0) agg.fill = 0;
  if (threadIdx.x < Q_MAXT) agg.cnt[threadIdx.x] = 0;
  __syncthreads();
}

// Block-reduce the below-window sums and W, combine CTAs in fixed order.
// Last-CTA sum of P partial rows of NS slots (row stride `stride`), by the
// whole CTA: thread t sums slot t % NS over rows t / NS, t / NS + G, ...
// (G groups, independent L2 loads in flight), then threads
// < NS add the G group sums in group order.  Deterministic (fixed order for
// a given P and blockDim); the serial form kept ~600 dependent L2 loads on
// one thread per slot, tens of microseconds per step.  Returns the slot sum
// in threads < NS.
template <int NS, int G>
PF_D double q_sum_rows(const double* part, unsigned P, int stride, double (*grp)[NS]) {
  // grp: G x NS shared scratch (the caller's warp-sum array, free again here)
  const int s = (int)threadIdx.x % NS, g = (int)threadIdx.x / NS;
  double v = 0.0;
  __syncthreads();
  if (g < G) {
#pragma unroll 4
    for (unsigned b = g; b < P; b += G) v += __ldcg(&part[(size_t)b * stride + s]);
    grp[g][s] = v;
  }
  __syncthreads();
  double tot = 0.0;
  if ((int)threadIdx.x < NS)
    for (int k = 0; k < G; ++k) tot += grp[k][threadIdx.x];
  return tot;
}

PF_D void q_reduce_partials(const QArgs& qa, const QWin& win, double (&acc)[Q_SLOTS], double wsum) {
  __shared__ double red[8][Q_SLOTS + 1];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s <= Q_SLOTS; ++s) {
    double v = s < Q_SLOTS ? acc[s < Q_SLOTS ? s : 0] : wsum;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][s] = v;
  }
  __syncthreads();
  if (threadIdx.x <= Q_SLOTS) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    qa.part[(size_t)q_pslot(qa) * (Q_SLOTS + 1) + threadIdx.x] = s;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&qa.sh->counter, 1u) == q_ptotal(qa) - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double s = q_sum_rows<Q_SLOTS + 1, 8>(qa.part, q_ptotal(qa), Q_SLOTS + 1, red);
  if (threadIdx.x <= Q_SLOTS) {
    if (threadIdx.x == Q_SLOTS) {
      qa.sh->W = s;
    } else {
      const int q = threadIdx.x / Q_PER, k = threadIdx.x - q * Q_PER;
      if (k < win.nq[q]) {
        QTarget& t = qa.tg[win.base[q] + k];
        t.wbelow = s;
        t.klo = win.lo[threadIdx.x];
        t.khi = win.hi[threadIdx.x];
      }
    }
  }
  if (threadIdx.x == 0) qa.sh->counter = 0;
}

// Windows of this step (identical in every CTA: same inputs, same code).
// Targets are grouped by quantity in qa.tg (x, sigma2, tau2 order).
PF_D void q_make_windows(const QArgs& qa, QWin& win) {
  if (threadIdx.x == 0) {
    for (int q = 0; q < Q_MAXQ; ++q) {
      win.nq[q] = 0;
      win.base[q] = 0;
    }
    for (int s = 0; s < Q_SLOTS; ++s) {
      win.lo[s] = 0xFFFFFFFFu;
      win.hi[s] = 0u;
    }
    for (int t = qa.ntarget - 1; t >= 0; --t) {
      const int q = qa.tg[t].q;
      win.base[q] = t;
      ++win.nq[q];
    }
    for (int t = 0; t < qa.ntarget; ++t) {
      const QTarget& tg = qa.tg[t];
      const int s = tg.q * Q_PER + (t - win.base[tg.q]);
      window_of(tg, qa.sh->mean[tg.q], qa.sh->sd[tg.q], &win.lo[s], &win.hi[s]);
    }
  }
  __syncthreads();
}


// K2 with the quantile window pass fused in: the tile's exact subtree sum
// (as cdf_reduce_kernel) plus, for every element, the below-window weight /
// candidate classification against this step's windows.
template <typename T>
__global__ void __launch_bounds__(CDF_THREADS)
cdf_reduce_q_kernel(WSrc src, int R, T* __restrict__ tile_tot, T* __restrict__ chunk_tot,
                    const int64_t* __restrict__ fail, QArgs qa) {
  if (fail && *fail) return;
  __shared__ T wt[CDF_THREADS / 32];
  __shared__ T tt[64];
  __shared__ QWin win;
  __shared__ QAgg agg;
  q_agg_init(agg);
  q_make_windows(qa, win);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double M = src.mode == 0 ? *src.M : 0.0;
  const int64_t chunk = blockIdx.x;
  const QWin wr = win;  // register copy
  double acc[Q_SLOTS];
#pragma unroll
  for (int k = 0; k < Q_SLOTS; ++k) acc[k] = 0.0;
  double wsum = 0.0;
  for (int r = 0; r < R; ++r) {
    const int64_t tile = chunk * R + r;
    const int64_t base = tile * CDF_TILE + threadIdx.x * CDF_V;
    T v[CDF_V], l1[4], l2[2], g;
    load_tile_weights<T>(src, base, M, v);
#pragma unroll
    for (int e = 0; e < CDF_V; ++e) {
      const double w = (double)v[e];
      wsum += w;
      q_classify(qa, wr, agg, (uint32_t)(base + e), w, acc, true);
    }
    thread_tree8<T>(v, l1, l2, g);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) g = g + __shfl_xor_sync(0xffffffffu, g, o);
    if (lane == 0) wt[warp] = g;
    __syncthreads();
    if (threadIdx.x == 0) {
      T a0 = wt[0] + wt[1], a1 = wt[2] + wt[3], a2 = wt[4] + wt[5], a3 = wt[6] + wt[7];
      T tot = (a0 + a1) + (a2 + a3);
      tt[r] = tot;
      tile_tot[tile] = tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int len = R; len > 1; len >>= 1)
      for (int i = 0; i < len / 2; ++i) tt[i] = tt[2 * i] + tt[2 * i + 1];
    chunk_tot[chunk] = tt[0];
  }
  q_flush(qa, agg);
  q_reduce_partials(qa, win, acc, wsum);  // shared copy: dynamic indices there
}

// K2 with the quantile windows, region form (the hot path).  The K window
// bounds of a quantity (lo_k and hi_k + 1) cut the key line into 2K+1
// regions; an element's region r = #{bounds <= key} costs 2K compares, its
// weight goes to a per-thread region sum in shared memory, and
//   key < lo_k          <=>  r <= idx_k     (idx_k = #{bounds < lo_k})
//   lo_k <= key <= hi_k <=>  idx_k < r <= jdx_k (jdx_k = #{bounds < hi_k+1})
// so the below-window weights are prefix sums of the region sums and the
// in-window test is one table lookup.  Same outputs as cdf_reduce_q_kernel
// (wbelow per target, candidate lists), at a fraction of the instructions.
// QM: bit q set when quantity q (x, sigma2, tau2) has targets.
struct QRegions {
  uint32_t b[Q_MAXQ][2 * Q_PER];   // sorted bounds (64-bit-safe: hi+1 clamped)
  uint8_t idx[Q_MAXQ][Q_PER];      // #{bounds < lo_k}
  uint16_t inmask[Q_MAXQ][2 * Q_PER + 1];  // window slots (bit s) containing region r
};

PF_D void q_make_regions(const QWin& win, QRegions& rg) {
  if (threadIdx.x < Q_MAXQ) {
    const int q = threadIdx.x;
    const int K = win.nq[q];
    uint32_t b[2 * Q_PER];
    uint32_t hp1[Q_PER];
    for (int k = 0; k < K; ++k) {
      const int s = q * Q_PER + k;
      hp1[k] = win.hi[s] == 0xFFFFFFFFu ? 0xFFFFFFFFu : win.hi[s] + 1u;
      b[2 * k] = win.lo[s];
      b[2 * k + 1] = hp1[k];
    }
    // insertion sort (<= 10 values)
    for (int i = 1; i < 2 * K; ++i) {
      const uint32_t v = b[i];
      int j = i - 1;
      while (j >= 0 && b[j] > v) {
        b[j + 1] = b[j];
        --j;
      }
      b[j + 1] = v;
    }
    for (int i = 0; i < 2 * Q_PER; ++i) rg.b[q][i] = i < 2 * K ? b[i] : 0xFFFFFFFFu;
    for (int r = 0; r <= 2 * Q_PER; ++r) rg.inmask[q][r] = 0;
    for (int k = 0; k < K; ++k) {
      const int s = q * Q_PER + k;
      int il = 0, ih = 0;
      for (int i = 0; i < 2 * K; ++i) {
        il += b[i] < win.lo[s];
        ih += b[i] < hp1[k];
      }
      // a window reaching the top key also holds 0xFFFFFFFF (hi + 1 clamped)
      if (win.hi[s] == 0xFFFFFFFFu) ih = 2 * Q_PER;
      rg.idx[q][k] = (uint8_t)il;
      for (int r = il + 1; r <= ih && r <= 2 * Q_PER; ++r) rg.inmask[q][r] |= (uint16_t)(1u << s % 16);
    }
  }
  __syncthreads();
}

// TREE = false: the classification alone (side stream), persistent over
// tiles (R = number of tiles); TREE = true: fused into K2 (one chunk of R
// tiles per CTA, with the exact subtree sums).
// Flush of a CTA buffer filled by warp-compacted appends: per-target
// positions by shared atomics, one global atomic per target, then the copy.
// Called by all threads.
PF_D void q_flush_compact(const QArgs& qa, QAgg& agg) {
  __syncthreads();
  const int nfill = min(agg.fill, Q_AGG);
  for (int s = threadIdx.x; s < nfill; s += blockDim.x) agg.pos[s] = atomicAdd(&agg.cnt[agg.tk[s]], 1u);
  __syncthreads();
  if (threadIdx.x < Q_MAXT) {
    const uint32_t c = agg.cnt[threadIdx.x];
    agg.base[threadIdx.x] = c ? atomicAdd(&qa.tg[threadIdx.x].count, c) : 0u;
  }
  __syncthreads();
  for (int s = threadIdx.x; s < nfill; s += blockDim.x) {
    const int k = agg.tk[s];
    const uint32_t pos = agg.base[k] + agg.pos[s];
    if (pos < qa.cap) qa.cand[(size_t)k * qa.cap + pos] = agg.c[s];
  }
  __syncthreads();
  if (threadIdx.x == 0) agg.fill = 0;
  if (threadIdx.x < Q_MAXT) agg.cnt[threadIdx.x] = 0;
  __syncthreads();
}

// THR threads per CTA; a "tile" here is THR * CDF_V consecutive particles
// (TREE requires THR == CDF_THREADS: the tile is K2's).  The classification-
// only launch uses THR = 128 with <= 64 registers and ~35 KB of shared
// memory, so a CTA fits beside a resident step-kernel CTA and the side
// stream's classification overlaps the step kernel instead of the CDF chain.
template <typename T, int QM, bool TREE, int THR = CDF_THREADS>
__global__ void __launch_bounds__(THR, 65536 / (64 * THR))
cdf_reduce_qr_kernel(WSrc src, int R, T* __restrict__ tile_tot, T* __restrict__ chunk_tot,
                     const int64_t* __restrict__ fail, QArgs qa) {
  static_assert(!TREE || THR == CDF_THREADS, "the fused tree pass uses K2's tiles");
  if (gridDim.z > 1) {
    q_rep(qa);
    src = wsrc_rep(src, qa.rslots);
    if (fail) fail += blockIdx.z;
  }
  if (fail && *fail) return;
  constexpr int NR = 2 * Q_PER + 1;
  __shared__ T wt[CDF_THREADS / 32];
  __shared__ T tt[64];
  __shared__ QWin win;
  __shared__ QAgg agg;
  __shared__ QRegions rg;
  // per-thread region sums (dynamic shared memory, present quantities only)
  double* rsum = pf_gtab;
  auto RS = [&](int q, int r) -> double& {
    const int qi = __popc((unsigned)QM & ((1u << q) - 1u));
    return rsum[(qi * NR + r) * THR + threadIdx.x];
  };
  __shared__ uint32_t sb[Q_MAXQ][16];  // sorted bounds padded to 15 (+1) for the binary search
  q_agg_init(agg);
  q_make_windows(qa, win);
  q_make_regions(win, rg);
  if (threadIdx.x < Q_MAXQ * 16) {
    const int q = threadIdx.x >> 4, i = threadIdx.x & 15;
    sb[q][i] = i < 2 * Q_PER ? rg.b[q][i] : 0xFFFFFFFFu;
  }
#pragma unroll
  for (int q = 0; q < Q_MAXQ; ++q)
    if (QM & (1 << q))
#pragma unroll
      for (int r = 0; r < NR; ++r) RS(q, r) = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double M = src.mode == 0 ? *src.M : 0.0;
  const int64_t chunk = blockIdx.x;
  double wsum = 0.0;
  const int nloop = TREE ? R : (int)((R - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x);
  for (int r = 0; r < nloop; ++r) {
    const int64_t tile = TREE ? chunk * R + r : (int64_t)blockIdx.x + (int64_t)r * gridDim.x;
    const int64_t base = tile * (THR * CDF_V) + threadIdx.x * CDF_V;
    T v[CDF_V], l1[4], l2[2], g;
    load_tile_weights<T>(src, base, M, v);
    uint32_t key[Q_MAXQ][CDF_V];
#pragma unroll
    for (int q = 0; q < Q_MAXQ; ++q) {
      if (!(QM & (1 << q))) continue;
      const uint4* kp = reinterpret_cast<const uint4*>(qa.keys[q] + base);
      const uint4 k0 = __ldcs(kp), k1 = __ldcs(kp + 1);
      key[q][0] = k0.x; key[q][1] = k0.y; key[q][2] = k0.z; key[q][3] = k0.w;
      key[q][4] = k1.x; key[q][5] = k1.y; key[q][6] = k1.z; key[q][7] = k1.w;
    }
    uint32_t anyin = 0;
    uint32_t inw[CDF_V];
#pragma unroll
    for (int e = 0; e < CDF_V; ++e) {
      const double w = (double)v[e];
      wsum += w;
      inw[e] = 0;
#pragma unroll
      for (int q = 0; q < Q_MAXQ; ++q) {
        if (!(QM & (1 << q))) continue;
        // #{bounds <= key}: branch-free binary search over 15 sorted bounds
        const uint32_t kk = key[q][e];
        int rr = kk >= sb[q][7] ? 8 : 0;
        rr += kk >= sb[q][rr + 3] ? 4 : 0;
        rr += kk >= sb[q][rr + 1] ? 2 : 0;
        rr += kk >= sb[q][rr] ? 1 : 0;
        rr = rr < 2 * Q_PER ? rr : 2 * Q_PER;
        RS(q, rr) += w;
        inw[e] |= (uint32_t)rg.inmask[q][rr];
      }
      anyin |= inw[e];
    }
    // candidates: one warp-wide scan and one shared atomic per warp per tile
    // reserve the buffer; per-target positions are assigned at the flush
    {
      int mine = 0;
#pragma unroll
      for (int e = 0; e < CDF_V; ++e) mine += __popc(inw[e]);
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tq = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += tq;
      }
      const int wtot = __shfl_sync(0xffffffffu, incl, 31);
      if (wtot) {
        int wb = 0;
        if (lane == 31) wb = atomicAdd(&agg.fill, wtot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        int pos = wb + incl - mine;
#pragma unroll
        for (int e = 0; e < CDF_V; ++e) {
          uint32_t mk = inw[e];
          while (mk) {
            const int sl = __ffs(mk) - 1;
            mk &= mk - 1;
            const int q = sl / Q_PER;
            const int tq = win.base[q] + (sl - q * Q_PER);
            QCand c;
            c.key = q == 0 ? key[0][e] : (q == 1 ? key[1][e] : key[2][e]);
            c.idx = qa.gbase + (uint32_t)(base + e);
            c.w = (double)v[e];
            if (pos < Q_AGG) {
              agg.c[pos] = c;
              agg.tk[pos] = (uint8_t)tq;
            } else {  // buffer full: straight to the global list
              const uint32_t gp = atomicAdd(&qa.tg[tq].count, 1u);
              if (gp < qa.cap) qa.cand[(size_t)tq * qa.cap + gp] = c;
            }
            ++pos;
          }
        }
      }
    }
    if (!TREE) {
      __syncthreads();
      if (agg.fill > Q_AGG / 2) q_flush_compact(qa, agg);
    }
    if (TREE) {
      thread_tree8<T>(v, l1, l2, g);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) g = g + __shfl_xor_sync(0xffffffffu, g, o);
      if (lane == 0) wt[warp] = g;
      __syncthreads();
      if (threadIdx.x == 0) {
        T a0 = wt[0] + wt[1], a1 = wt[2] + wt[3], a2 = wt[4] + wt[5], a3 = wt[6] + wt[7];
        T tot = (a0 + a1) + (a2 + a3);
        tt[r] = tot;
        tile_tot[tile] = tot;
      }
      __syncthreads();
    }
  }
  if (TREE && threadIdx.x == 0) {
    for (int len = R; len > 1; len >>= 1)
      for (int i = 0; i < len / 2; ++i) tt[i] = tt[2 * i] + tt[2 * i + 1];
    chunk_tot[chunk] = tt[0];
  }
  // per-thread below-window sums from the region sums
  double acc[Q_SLOTS];
#pragma unroll
  for (int sl = 0; sl < Q_SLOTS; ++sl) acc[sl] = 0.0;
#pragma unroll
  for (int q = 0; q < Q_MAXQ; ++q) {
    if (!(QM & (1 << q))) continue;
    double pre[NR];
    double run = 0.0;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      run += RS(q, r);
      pre[r] = run;
    }
#pragma unroll
    for (int k = 0; k < Q_PER; ++k) {
      const int il = rg.idx[q][k];
      double a = 0.0;
#pragma unroll
      for (int r = 0; r < NR; ++r) a = (r == il) ? pre[r] : a;
      acc[q * Q_PER + k] = a;
    }
  }
  q_flush_compact(qa, agg);
  q_reduce_partials(qa, win, acc, wsum);
}

// Window pass on its own (n below one CDF tile, where K2 is not used).
template <typename T>
__global__ void __launch_bounds__(256)
q_window_kernel(WSrc src, int64_t n, const int64_t* __restrict__ fail, QArgs qa) {
  if (fail && *fail) return;
  __shared__ QWin win;
  __shared__ QAgg agg;
  q_agg_init(agg);
  q_make_windows(qa, win);
  const double M = src.mode == 0 ? *src.M : 0.0;
  const QWin wr = win;  // register copy
  double acc[Q_SLOTS];
#pragma unroll
  for (int k = 0; k < Q_SLOTS; ++k) acc[k] = 0.0;
  double wsum = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t iters = (n + stride - 1) / stride;
  for (int64_t it = 0; it < iters; ++it) {  // uniform trip count: warp-collective classify
    const int64_t i = it * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = i < n;
    const double w = valid ? (double)weight_of<T>(src.src[i], M, src.mode) : 0.0;
    wsum += w;
    q_classify(qa, wr, agg, (uint32_t)(valid ? i : 0), w, acc, valid);
  }
  q_flush(qa, agg);
  q_reduce_partials(qa, win, acc, wsum);  // shared copy: dynamic indices there
}

// ------------------------------------------------------- resolve (side) ---
// Exclusive scan, in place, of n (a multiple of blockDim.x) values in shared
// memory; returns the total.  Integer addition: exact in any order.
PF_D unsigned long long block_exclusive_scan(unsigned long long* a, int n) {
  __shared__ unsigned long long ws[32];
  __shared__ unsigned long long total;
  const int per = n / blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned long long loc = 0;
  for (int i = 0; i < per; ++i) loc += a[threadIdx.x * per + i];
  unsigned long long inc = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < nw; ++w) {
      const unsigned long long t = ws[w];
      ws[w] = s;
      s += t;
    }
    total = s;
  }
  __syncthreads();
  unsigned long long run = ws[warp] + inc - loc;
  for (int i = 0; i < per; ++i) {
    const unsigned long long t = a[threadIdx.x * per + i];
    a[threadIdx.x * per + i] = run;
    run += t;
  }
  __syncthreads();
  return total;
}

// R1: fixed-point sub-bin histogram of target k's candidates (threads i0,
// i0 + stride, ... of the caller's launch).
PF_D void q_hist_dev(const QArgs& qa, int k, int fallback_round, uint32_t i0, uint32_t stride) {
  QTarget& t = qa.tg[k];
  if (fallback_round && t.status != QS_REFILL) return;
  const uint32_t n = min(t.count, qa.cap);
  const uint32_t lo = t.klo, hi = t.khi;
  for (uint32_t i = i0; i < n; i += stride) {
    const QCand c = qa.cand[(size_t)k * qa.cap + i];
    const uint32_t b = sub_bin(c.key, lo, hi, Q_SUB);
    atomicAdd(&qa.hist[(size_t)k * Q_SUB + b], (unsigned long long)llrint(c.w * qa.fx_scale));
  }
}

__global__ void __launch_bounds__(256) q_hist_kernel(QArgs qa, const int64_t* fail, int fallback_round) {
  if (*fail) return;
  const int k = blockIdx.y;
  if (k >= qa.ntarget) return;
  q_hist_dev(qa, k, fallback_round, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// Bitonic sort of (value, idx, w) triples in shared memory, ascending by
// (value, idx) -- the order of np.argsort(values, kind="stable").
PF_D void bitonic_sort(double* v, uint32_t* id, double* w, int n2) {
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const bool gt = (v[i] > v[l]) || (v[i] == v[l] && id[i] > id[l]);
          if (gt == up) {
            double tv = v[i]; v[i] = v[l]; v[l] = tv;
            uint32_t ti = id[i]; id[i] = id[l]; id[l] = ti;
            double tw = w[i]; w[i] = w[l]; w[l] = tw;
          }
        }
      }
      __syncthreads();
    }
}

// R2a: one CTA per target.  Prefix the sub-bin histogram, classify the
// window (hit / miss low / miss high / overflow), locate the crossing
// sub-bin b* and the exact-enough weight below its left neighbour.
PF_D void q_locate_dev(const QArgs& qa, int k, int fallback_round) {
  QTarget& tg = qa.tg[k];
  if (fallback_round && tg.status != QS_REFILL) return;
  __shared__ unsigned long long pre[Q_SUB + 1];
  __shared__ int bstar;
  __shared__ uint32_t status;
  const double T = tg.p * qa.sh->W;
  const double wb = tg.wbelow;
  const unsigned long long* H = qa.hist + (size_t)k * Q_SUB;
  for (int b = threadIdx.x; b < Q_SUB; b += blockDim.x) pre[b] = __ldcg(H + b);
  __syncthreads();
  const unsigned long long tot = block_exclusive_scan(pre, Q_SUB);
  if (threadIdx.x == 0) {
    atomicMax(&qa.stats[2], tg.count);
    atomicAdd(&qa.stats[3], 1u);
    pre[Q_SUB] = tot;
    status = QS_OK;
    if (tg.count > qa.cap) status = QS_OVERFLOW;
    else if (!(T > wb)) status = QS_MISS_LO;
    else if (T > wb + (double)tot / qa.fx_scale) status = QS_MISS_HI;
    bstar = Q_SUB - 1;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < Q_SUB; j += blockDim.x)
    if (wb + (double)pre[j + 1] / qa.fx_scale >= T && !(wb + (double)pre[j] / qa.fx_scale >= T))
      atomicMin(&bstar, j);
  __syncthreads();
  if (threadIdx.x == 0) {
    tg.wmass = (double)tot / qa.fx_scale;
    tg.nlist = 0;
    if (status != QS_OK) {
      tg.status = status;
      qa.sh->any_miss = 1;
    } else {
      tg.status = QS_LOCATED;
      tg.bstar = bstar;
      tg.cum0 = wb + (double)pre[max(bstar - 1, 0)] / qa.fx_scale;
    }
  }
}

__global__ void __launch_bounds__(1024)
q_locate_kernel(QArgs qa, const int64_t* fail, int fallback_round) {
  if (*fail) return;
  q_locate_dev(qa, blockIdx.x, fallback_round);
}

// R2b: grid pass over the candidate lists: keep the candidates of sub-bins
// b*-1 .. b*+1 (a few hundred) for the exact resolve.
PF_D void q_filter_dev(const QArgs& qa, int k, uint32_t i0, uint32_t stride) {
  QTarget& t = qa.tg[k];
  if (t.status != QS_LOCATED) return;
  const uint32_t n = min(t.count, qa.cap);
  const int b0 = max(t.bstar - 1, 0), b1 = min(t.bstar + 1, Q_SUB - 1);
  const uint32_t lo = t.klo, hi = t.khi;
  for (uint32_t i = i0; i < n; i += stride) {
    const QCand c = qa.cand[(size_t)k * qa.cap + i];
    const int b = (int)sub_bin(c.key, lo, hi, Q_SUB);
    if (b >= b0 && b <= b1) {
      const uint32_t pos = atomicAdd(&t.nlist, 1u);
      if (pos < Q_LIST) {
        qa.lidx[(size_t)k * Q_LIST + pos] = c.idx;
        qa.lw[(size_t)k * Q_LIST + pos] = c.w;
      }
    }
  }
}

__global__ void __launch_bounds__(256) q_filter_kernel(QArgs qa, const int64_t* fail) {
  if (*fail) return;
  const int k = blockIdx.y;
  if (k >= qa.ntarget) return;
  q_filter_dev(qa, k, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// R2c: one CTA per target: exact values of the kept candidates, stable
// (value, index) order, cumulative weight from cum0 -> the quantile; then
// the window predictor update.
extern __shared__ unsigned long long qsm[];  // q_finish / q_round dynamic shared memory

PF_D void q_finish_dev(const QArgs& qa, const QValueSrc& vs, double* out_x, double* out_s, double* out_t,
                       int64_t t_step, int k) {
  QTarget& tg = qa.tg[k];
  if (tg.status != QS_LOCATED) return;
  // dynamic smem: sv[Q_LIST] f64 | sw[Q_LIST] f64 | sid[Q_LIST] u32
  double* sv = reinterpret_cast<double*>(qsm);
  double* sw = sv + Q_LIST;
  uint32_t* sid = reinterpret_cast<uint32_t*>(sw + Q_LIST);
  const int m = (int)__ldcg(&tg.nlist);
  if (m > Q_LIST) {
    if (threadIdx.x == 0) {
      tg.status = QS_CROWD;
      qa.sh->any_miss = 1;
    }
    return;
  }
  int n2 = 1;
  while (n2 < m) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    if (i < m) {
      sid[i] = qa.lidx[(size_t)k * Q_LIST + i];
      sw[i] = qa.lw[(size_t)k * Q_LIST + i];
      sv[i] = quantity_value(vs, tg.q, sid[i]);
    } else {
      sv[i] = INFINITY;
      sid[i] = 0xFFFFFFFFu;
      sw[i] = 0.0;
    }
  }
  __syncthreads();
  bitonic_sort(sv, sid, sw, n2);
  if (threadIdx.x == 0) {
    const double T = tg.p * qa.sh->W;
    double cum = tg.cum0;
    double val = m > 0 ? sv[m - 1] : NAN;
    for (int i = 0; i < m; ++i) {
      cum += sw[i];
      if (cum >= T) { val = sv[i]; break; }
    }
    double* o = tg.q == 0 ? out_x : (tg.q == 1 ? out_s : out_t);
    const int ncol = tg.q == 0 ? 3 : 5;
    o[(t_step - 1) * ncol + tg.col] = val;
    // predictor update: standardized position; the half-width is sized in
    // probability mass (the step-to-step drift of a quantile is ~0.1-0.4%
    // of mass whether it sits in the bulk or a tail), converted to
    // standardized units through a normal-density proxy.
    const double mean = qa.sh->mean[tg.q], sd = qa.sh->sd[tg.q];
    if (sd > 0.0 && isfinite(val)) {
      const double z = (val - mean) / sd;
      const double phi = fmax(normal_pdf(z), 1e-4);
      const double em = fabs(z - tg.zprev) * phi;
      tg.ema = 0.7 * tg.ema + 0.3 * em;
      const double mass = fmin(Q_MASS_MAX, fmax(Q_MASS_MIN, Q_MASS_K * fmax(em, tg.ema)));
      tg.h = fmin(2.0, mass / phi);
      tg.zprev = z;
    }
    tg.status = QS_OK;
  }
}

__global__ void __launch_bounds__(1024)
q_finish_kernel(QArgs qa, QValueSrc vs, double* out_x, double* out_s, double* out_t, int64_t t_step,
                const int64_t* fail) {
  if (*fail) return;
  q_finish_dev(qa, vs, out_x, out_s, out_t, t_step, blockIdx.x);
}


// F0: interval for each target that missed.  Attempt 0 uses a secant
// estimate from the missing mass, bounded so the histogram pass touches few
// particles; attempt 1 (only if attempt 0's interval did not hold the
// crossing either) takes everything on the missing side.
PF_D void q_prep_target(const QArgs& qa, int attempt, int k) {
  QTarget& t = qa.tg[k];
  const uint32_t st = t.status;
  const double W = qa.sh->W, T = t.p * W;
  const double mean = qa.sh->mean[t.q], sd = qa.sh->sd[t.q];
  uint32_t lo, hi;
  if (attempt == 0 && (st == QS_MISS_LO || st == QS_MISS_HI || st == QS_OVERFLOW || st == QS_CROWD)) {
    const bool ok_sd = sd > 0.0 && isfinite(sd) && isfinite(mean);
    if (st == QS_MISS_LO) {
      lo = 0;
      hi = t.klo ? t.klo - 1 : 0;
      if (ok_sd) {
        const double zc = t.zprev - t.h;
        const double dm = fmax(t.wbelow - T, 0.0) / W;
        const double dz = 3.0 * dm / fmax(normal_pdf(zc), 1e-3) + 0.05;
        const uint32_t l = key_rd(mean + sd * (zc - dz));
        if (l <= hi) lo = l;
      }
    } else if (st == QS_MISS_HI) {
      lo = t.khi == 0xFFFFFFFFu ? t.khi : t.khi + 1;
      hi = 0xFFFFFFFFu;
      if (ok_sd) {
        const double zc = t.zprev + t.h;
        const double dm = fmax(T - t.wbelow - t.wmass, 0.0) / W;
        const double dz = 3.0 * dm / fmax(normal_pdf(zc), 1e-3) + 0.05;
        const uint32_t h2 = key_ru(mean + sd * (zc + dz));
        if (h2 >= lo) hi = h2;
      }
    } else {
      lo = t.klo;
      hi = t.khi;
    }
  } else if (attempt == 1 && st == QS_RETRY) {
    if (t.side < 0) { lo = 0; hi = t.ilo ? t.ilo - 1 : 0; }
    else { lo = t.ihi == 0xFFFFFFFFu ? t.ihi : t.ihi + 1; hi = 0xFFFFFFFFu; }
  } else {
    return;
  }
  t.ilo = lo;
  t.ihi = hi;
  t.status = QS_FB;
  t.missed = 1;
  qa.sh->fb_active[attempt] = 1;
}

__global__ void q_fallback_prep_kernel(QArgs qa, int attempt, const int64_t* fail) {
  if (*fail || !qa.sh->any_miss) return;
  const int k = threadIdx.x;
  if (k >= qa.ntarget) return;
  q_prep_target(qa, attempt, k);
}

// F1: full pass over the particles for targets in fallback: fixed-point
// histogram of the interval + fp64 weight below it.  The first QFB_SMEM_T
// targets in fallback accumulate in a per-CTA shared-memory histogram
// (flushed once per CTA): a whole-side interval holds millions of particles,
// and global atomics on 4096 bins would serialise on them.  A bin is two
// 32-bit words with an explicit carry (64-bit shared atomics are CAS loops
// on this architecture; 32-bit adds are native): the low word's adder that
// wraps it adds the carry to the high word, so the pair holds the exact
// 64-bit sum.  Integer sums: the same bins in any order.
constexpr int QFB_SMEM_T = 2;
constexpr int QFB_SMEM_BYTES = QFB_SMEM_T * Q_FB * 8;
// BATCH: launched with gridDim.z = R replications (the offsets modify the
// parameters, which costs the single-run instantiation a local copy).
template <int BATCH = 0>
__global__ void __launch_bounds__(256)
q_fallback_hist_kernel(QArgs qa, const double* __restrict__ lw, int wmode, const double* Mp, int64_t n,
                       int single, int attempt, const int64_t* fail) {
  if (BATCH) {
    q_rep(qa);
    lw += blockIdx.z * n;
    Mp += 2 * blockIdx.z;
    fail += blockIdx.z;
  }
  if (*fail || !qa.sh->fb_active[attempt]) return;
  __shared__ uint32_t ilo[Q_MAXT], ihi[Q_MAXT];
  __shared__ int act[Q_MAXT], tq[Q_MAXT], slot[Q_MAXT];
  __shared__ bool last;
  extern __shared__ uint32_t shist[];  // [QFB_SMEM_T][Q_FB][lo, hi]
  if (threadIdx.x == 0) {
    int ns = 0;
    for (int k = 0; k < Q_MAXT; ++k) {
      const bool on = k < qa.ntarget && qa.tg[k].status == QS_FB;
      act[k] = on;
      tq[k] = on ? qa.tg[k].q : 0;
      ilo[k] = on ? qa.tg[k].ilo : 0u;
      ihi[k] = on ? qa.tg[k].ihi : 0u;
      slot[k] = (on && ns < QFB_SMEM_T) ? ns++ : -1;
    }
  }
  for (int i = threadIdx.x; i < 2 * QFB_SMEM_T * Q_FB; i += blockDim.x) shist[i] = 0u;
  __syncthreads();
  const double M = wmode == 0 ? *Mp : 0.0;
  double acc[Q_MAXT];
#pragma unroll
  for (int k = 0; k < Q_MAXT; ++k) acc[k] = 0.0;
  // FU particles per thread per iteration with all their loads issued up
  // front (memory-level parallelism); each thread still visits its particles
  // in the order i, i + stride, i + 2 stride, ... so the fp64 below-interval
  // sums are the same as a one-at-a-time loop's.
  constexpr int FU = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += FU * stride) {
    double w[FU];
    bool ok[FU];
#pragma unroll
    for (int u = 0; u < FU; ++u) {
      const int64_t i = i0 + u * stride;
      ok[u] = i < n;
      w[u] = ok[u] ? lw[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < FU; ++u) {
      double x = wmode == 0 ? exp(w[u] - M) : w[u];
      if (single) x = (double)(float)x;
      w[u] = ok[u] ? x : 0.0;
    }
#pragma unroll
    for (int k = 0; k < Q_MAXT; ++k) {
      if (!act[k]) continue;
      const uint32_t* kq = qa.keys[tq[k]];
      uint32_t key[FU];
#pragma unroll
      for (int u = 0; u < FU; ++u) key[u] = ok[u] ? kq[i0 + u * stride] : 0xFFFFFFFFu;
#pragma unroll
      for (int u = 0; u < FU; ++u) {
        if (!ok[u] || key[u] > ihi[k]) continue;
        if (key[u] < ilo[k]) {
          acc[k] += w[u];
        } else {
          const unsigned long long v = (unsigned long long)llrint(w[u] * qa.fx_scale);
          const uint32_t b = sub_bin(key[u], ilo[k], ihi[k], Q_FB);
          if (slot[k] >= 0) {
            uint32_t* cell = shist + 2 * (slot[k] * Q_FB + b);
            const uint32_t vlo = (uint32_t)v;
            const uint32_t old = atomicAdd(cell, vlo);
            const uint32_t vhi = (uint32_t)(v >> 32) + (old + vlo < old ? 1u : 0u);
            if (vhi) atomicAdd(cell + 1, vhi);
          } else {
            atomicAdd(&qa.fhist[(size_t)k * Q_FB + b], v);
          }
        }
      }
    }
  }
  __syncthreads();
  for (int k = 0; k < Q_MAXT; ++k) {
    if (slot[k] < 0) continue;
    for (int b = threadIdx.x; b < Q_FB; b += blockDim.x) {
      const uint32_t* cell = shist + 2 * (slot[k] * Q_FB + b);
      const unsigned long long v = ((unsigned long long)cell[1] << 32) | cell[0];
      if (v) atomicAdd(&qa.fhist[(size_t)k * Q_FB + b], v);
    }
  }
  // deterministic combine of the below-interval sums
  __shared__ double red[8][Q_MAXT + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < Q_MAXT; ++k) {
    double v = acc[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < Q_MAXT) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    qa.part[(size_t)q_pslot(qa) * (Q_MAXT + 1) + threadIdx.x] = s;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&qa.sh->fb_counter, 1u) == q_ptotal(qa) - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double s = q_sum_rows<Q_MAXT + 1, 8>(qa.part, q_ptotal(qa), Q_MAXT + 1, red);
  if (threadIdx.x < qa.ntarget && act[threadIdx.x]) qa.tg[threadIdx.x].ibelow = s;
  if (threadIdx.x == 0) qa.sh->fb_counter = 0;
}

// F2: pick the fallback bin holding the crossing; it becomes the new window
// (one CTA per target).  If the interval does not hold it (attempt 0's
// bounded guess fell short) the target is marked for attempt 1.
template <int BATCH = 0>
__global__ void __launch_bounds__(1024) q_fallback_select_kernel(QArgs qa, int attempt, const int64_t* fail,
                                                                  int fuse_prep = 0) {
  if (BATCH) {
    q_rep(qa);
    fail += blockIdx.z;
  }
  if (*fail || !qa.sh->fb_active[attempt]) return;
  const int k = blockIdx.x;
  QTarget& t = qa.tg[k];
  if (t.status != QS_FB) return;
  __shared__ unsigned long long pre[Q_FB + 1];
  __shared__ int bsel;
  const double T = t.p * qa.sh->W;
  unsigned long long* F = qa.fhist + (size_t)k * Q_FB;
  for (int j = threadIdx.x; j < Q_FB; j += blockDim.x) {
    pre[j] = F[j];
    F[j] = 0ull;  // leave the row clean for the next attempt / step
  }
  if (threadIdx.x == 0) bsel = Q_FB;
  __syncthreads();
  const unsigned long long tot = block_exclusive_scan(pre, Q_FB);
  if (threadIdx.x == 0) pre[Q_FB] = tot;
  __syncthreads();
  for (int j = threadIdx.x; j < Q_FB; j += blockDim.x)
    if (t.ibelow + (double)pre[j + 1] / qa.fx_scale >= T && !(t.ibelow + (double)pre[j] / qa.fx_scale >= T))
      atomicMin(&bsel, j);
  __syncthreads();
  // clear this target's sub-bin histogram for the resolve round that follows
  for (int j = threadIdx.x; j < Q_SUB; j += blockDim.x) qa.hist[(size_t)k * Q_SUB + j] = 0ull;
  if (threadIdx.x != 0) return;
  atomicAdd(&qa.stats[1], 1u);
  const bool below = !(T > t.ibelow);
  const bool above = T > t.ibelow + (double)tot / qa.fx_scale;
  if ((below || above) && attempt == 0 && !(t.ilo == 0 && below) && !(t.ihi == 0xFFFFFFFFu && above)) {
    t.side = below ? -1 : 1;
    t.status = QS_RETRY;
    if (fuse_prep) q_prep_target(qa, 1, k);  // attempt 1's interval (F0), without its own launch
    return;
  }
  const int b = bsel < Q_FB ? bsel : (below ? 0 : Q_FB - 1);
  const unsigned long long s = pre[b];
  // key range of fallback bin b: smallest keys mapping to b and b+1
  const uint64_t span = (uint64_t)(t.ihi - t.ilo) + 1;
  const uint64_t lo_off = ((uint64_t)b * span + Q_FB - 1) / Q_FB;
  const uint64_t hi_off = ((uint64_t)(b + 1) * span + Q_FB - 1) / Q_FB;  // exclusive
  t.klo = (uint32_t)(t.ilo + lo_off);
  t.khi = (uint32_t)(t.ilo + (hi_off > lo_off ? hi_off - 1 : lo_off));
  t.wbelow = t.ibelow + (double)s / qa.fx_scale;
  t.count = 0;
  t.status = QS_REFILL;
}

// F3: append the candidates of the re-windowed targets.
template <int BATCH = 0>
__global__ void __launch_bounds__(256) q_fallback_fill_kernel(QArgs qa, const double* __restrict__ lw, int wmode,
                                                              const double* Mp, int64_t n, int single,
                                                              const int64_t* fail) {
  if (BATCH) {
    q_rep(qa);
    lw += blockIdx.z * n;
    Mp += 2 * blockIdx.z;
    fail += blockIdx.z;
  }
  if (*fail || !qa.sh->fb_active[0]) return;
  __shared__ int act[Q_MAXT], tq[Q_MAXT];
  __shared__ uint32_t klo[Q_MAXT], khi[Q_MAXT];
  if (threadIdx.x < Q_MAXT) {
    const int k = threadIdx.x;
    const bool on = k < qa.ntarget && qa.tg[k].status == QS_REFILL;
    act[k] = on;
    tq[k] = on ? qa.tg[k].q : 0;
    klo[k] = on ? qa.tg[k].klo : 1u;
    khi[k] = on ? qa.tg[k].khi : 0u;
  }
  __syncthreads();
  const double M = wmode == 0 ? *Mp : 0.0;
  constexpr int FU = 4;  // particles per thread per iteration, loads up front
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += FU * stride) {
#pragma unroll
    for (int k = 0; k < Q_MAXT; ++k) {
      if (!act[k]) continue;
      const uint32_t* kq = qa.keys[tq[k]];
      uint32_t key[FU];
#pragma unroll
      for (int u = 0; u < FU; ++u) key[u] = i0 + u * stride < n ? kq[i0 + u * stride] : 0u;
#pragma unroll
      for (int u = 0; u < FU; ++u) {
        const int64_t i = i0 + u * stride;
        if (i >= n || key[u] < klo[k] || key[u] > khi[k]) continue;
        double w = wmode == 0 ? exp(lw[i] - M) : lw[i];
        if (single) w = (double)(float)w;
        const uint32_t pos = atomicAdd(&qa.tg[k].count, 1u);
        if (pos < qa.cap) {
          QCand c;
          c.key = key[u];
          c.idx = qa.gbase + (uint32_t)i;
          c.w = w;
          qa.cand[(size_t)k * qa.cap + pos] = c;
        }
      }
    }
  }
}

// Every particle of the step, per source (one per shard; a single run has
// one): the overflow path of q_select_kernel walks these instead of the
// truncated candidate list.
struct QAll {
  int nsrc;                                    // 0: not available (count the target unresolved)
  int64_t ns;                                  // particles per source
  const uint32_t* keys[PF_MAX_SHARDS][Q_MAXQ];
  const double* lw[PF_MAX_SHARDS];             // log-weights (or fed weights, wmode 1)
  const double* M[PF_MAX_SHARDS];              // the step's max log-weight
  int wmode, single;
};

// S: last resort for a target whose re-windowed candidates still crowd the
// exact list (heavy ties): weighted radix select over the exact 64-bit value
// images of all candidates (one CTA per target).  Smallest value v with
// wbelow + sum_{value <= v} w >= p W -- the same answer as the stable-order
// cumulative search.  A window that held more candidates than the list
// (tg.count > cap: e.g. tau2 = 0, where resampling leaves long runs of
// identical states) is selected exactly over every particle whose key lies
// in the window, read from `all`; the weights are formed as the candidate
// passes form them, so the answer is the one the full list would give.
PF_D void q_select_dev(const QArgs& qa, const QValueSrc& vs, double* __restrict__ scratch, double* out_x,
                       double* out_s, double* out_t, int64_t t_step, unsigned int* unresolved, const QAll& all,
                       int k) {
  QTarget& tg = qa.tg[k];
  if (tg.status == QS_OK) return;
  __shared__ unsigned long long hist[256];
  __shared__ uint64_t prefix;
  __shared__ double base;
  const bool over = tg.count > qa.cap;
  const bool exact_all = over && all.nsrc > 0;
  const uint32_t m = min(tg.count, qa.cap);
  double* val = scratch + (size_t)k * qa.cap;
  const QCand* cand = qa.cand + (size_t)k * qa.cap;
  if (!exact_all)
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) val[i] = quantity_value(vs, tg.q, cand[i].idx);
  const double T = tg.p * qa.sh->W;
  const uint32_t klo = tg.klo, khi = tg.khi;
  if (threadIdx.x == 0) {
    prefix = 0;
    base = tg.wbelow;
  }
  __syncthreads();
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint64_t pfx = prefix;
    if (exact_all) {
      for (int h = 0; h < all.nsrc; ++h) {
        const uint32_t* kq = all.keys[h][tg.q];
        const double M = all.wmode == 0 ? *all.M[h] : 0.0;
        for (int64_t i = threadIdx.x; i < all.ns; i += blockDim.x) {
          const uint32_t key = kq[i];
          if (key < klo || key > khi) continue;
          const uint64_t b = ordered_bits(quantity_value(vs, tg.q, (uint32_t)(h * all.ns + i)));
          if (shift == 56 || (b >> (shift + 8)) == pfx) {
            double w = all.wmode == 0 ? exp(all.lw[h][i] - M) : all.lw[h][i];
            if (all.single) w = (double)(float)w;
            atomicAdd(&hist[(b >> shift) & 255], (unsigned long long)llrint(w * qa.fx_scale));
          }
        }
      }
    } else {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint64_t b = ordered_bits(val[i]);
        if (shift == 56 || (b >> (shift + 8)) == pfx)
          atomicAdd(&hist[(b >> shift) & 255], (unsigned long long)llrint(cand[i].w * qa.fx_scale));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      int d = -1, lastnz = 0;
      for (int j = 0; j < 256; ++j) {
        if (hist[j]) lastnz = j;
        if (d < 0 && hist[j] && base + (double)(s + hist[j]) / qa.fx_scale >= T) d = j;
        if (d < 0) s += hist[j];
      }
      if (d < 0) { d = lastnz; s -= hist[lastnz]; }
      base += (double)s / qa.fx_scale;
      prefix = (pfx << 8) | (uint64_t)d;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint64_t b = prefix;
    union { uint64_t u; double d; } c;
    c.u = (b >> 63) ? (b & 0x7FFFFFFFFFFFFFFFull) : ~b;
    const double v = m ? c.d : NAN;
    double* o = tg.q == 0 ? out_x : (tg.q == 1 ? out_s : out_t);
    const int ncol = tg.q == 0 ? 3 : 5;
    o[(t_step - 1) * ncol + tg.col] = v;
    if (over && !exact_all) atomicAdd(unresolved, 1u);  // the host raises on this
    tg.status = QS_OK;
  }
}

__global__ void __launch_bounds__(1024)
q_select_kernel(QArgs qa, QValueSrc vs, double* __restrict__ scratch, double* out_x, double* out_s,
                double* out_t, int64_t t_step, const int64_t* fail, unsigned int* unresolved, QAll all) {
  if (*fail || !qa.sh->any_miss) return;
  q_select_dev(qa, vs, scratch, out_x, out_s, out_t, t_step, unresolved, all, blockIdx.x);
}

// One step's exact resolve for the single-device engine in two launches
// instead of eight: one CTA per target runs, in order, the candidate
// histogram (R1), the crossing location (R2a), the filter (R2b) and the
// exact stable-order finish (R2c) -- the same device code as the separate
// kernels, which the sharded runs still launch.  Round 0 then prepares the
// target's fallback interval if its window missed (F0, attempt 0); round 1
// (re-windowed targets only) ends with the weighted radix select (S) for a
// target that is still unresolved.  A target is owned by one CTA from start
// to end, so the CTA barrier is the only ordering needed.
template <int BATCH = 0>
__global__ void __launch_bounds__(1024)
q_round_kernel(QArgs qa, QValueSrc vs, double* __restrict__ scratch, double* out_x, double* out_s, double* out_t,
               int64_t t_step, const int64_t* fail, int round, unsigned int* unresolved, QAll all) {
  if (BATCH) {
    const int64_t r = blockIdx.z;
    q_rep(qa);
    vs.rec += r * qa.rslots;
    if (vs.seedp) vs.seedp += r;
    scratch += r * (int64_t)qa.ntarget * qa.cap;
    if (out_x) out_x += r * qa.rT * 3;
    if (out_s) out_s += r * qa.rT * 5;
    if (out_t) out_t += r * qa.rT * 5;
    fail += r;
    for (int q = 0; q < Q_MAXQ; ++q)
      if (all.keys[0][q]) all.keys[0][q] += r * qa.rslots;
    all.lw[0] += r * qa.rslots;
    if (all.M[0]) all.M[0] += 2 * r;
  }
  if (*fail) return;
  const int k = blockIdx.x;
  // round 1 ends the step for its target (q_step_end_kernel's reset, one
  // launch fewer on the side chain): target state, its histogram slice, and
  // (CTA 0) the shared miss / fallback flags -- nothing later in the step
  // reads them
  auto end_step = [&]() {
    __syncthreads();
    for (int i = threadIdx.x; i < Q_SUB; i += blockDim.x) qa.hist[(size_t)k * Q_SUB + i] = 0ull;
    if (threadIdx.x == 0) {
      QTarget& tg = qa.tg[k];
      tg.missed = 0;
      tg.count = 0;
      tg.status = QS_OK;
      if (k == 0) {
        qa.sh->any_miss = 0;
        qa.sh->fb_active[0] = qa.sh->fb_active[1] = 0;
      }
    }
  };
  if (round && qa.tg[k].status == QS_OK) {  // resolved in round 0 (uniform over the CTA)
    end_step();
    return;
  }
  q_hist_dev(qa, k, round, threadIdx.x, blockDim.x);
  __syncthreads();
  q_locate_dev(qa, k, round);
  __syncthreads();
  q_filter_dev(qa, k, threadIdx.x, blockDim.x);
  __syncthreads();
  q_finish_dev(qa, vs, out_x, out_s, out_t, t_step, k);
  __syncthreads();
  if (round == 0) {
    if (threadIdx.x == 0 && qa.tg[k].status != QS_OK) q_prep_target(qa, 0, k);
  } else {
    q_select_dev(qa, vs, scratch, out_x, out_s, out_t, t_step, unresolved, all, k);
    end_step();
  }
}

// End of step: widen windows that missed, clear the per-step histograms
// and counters for the next step.
template <int BATCH = 0>
__global__ void __launch_bounds__(1024) q_step_end_kernel(QArgs qa, int had_miss_possible) {
  if (BATCH) q_rep(qa);
  for (int i = threadIdx.x; i < qa.ntarget * Q_SUB; i += blockDim.x) qa.hist[i] = 0ull;
  __syncthreads();
  const int k = threadIdx.x;
  if (k < qa.ntarget) {
    QTarget& t = qa.tg[k];
    t.missed = 0;
    t.count = 0;
    t.status = QS_OK;
  }
  if (k == 0) {
    qa.sh->any_miss = 0;
    qa.sh->fb_active[0] = qa.sh->fb_active[1] = 0;
  }
  (void)had_miss_possible;
}

}  // namespace pf
