// Resampling CDF by the paper's two-pass adder tree, bit-identical to the
// reference (prefix_sum.py:46-106), plus the cut-point table and lookup
// (resampling.py:110-158).
//
// The reference builds the tree level by level over all N weights:
//   forward   levels[d][i] = levels[d-1][2i] + levels[d-1][2i+1]   (:64)
//   backward  right child = parent, left child = parent - w[right]  (:86-87)
//   finalize  q = s/total, running max, clip [0,1], q[N-1] = 1      (:94-106)
// Any power-of-two aligned tile is a subtree of that tree, so the device
// splits it into
//   K2 cdf_reduce  : per 2048-element tile, the exact subtree sum (thread
//                    pairwise tree -> warp xor-butterfly -> 8-warp tree),
//                    and per chunk of R tiles the subtree over tile sums;
//   K3 cdf_top     : one CTA, the tree over chunk sums -> root, then the
//                    top-down backward pass to every chunk node, and the
//                    exclusive running max of chunk node values (a leaf
//                    never exceeds its subtree node, so a chunk's max q is
//                    its node value / total);
//   K4 cdf_expand  : per tile, rebuild the subtree, run the backward pass
//                    from the tile node, divide, running max, clip, pin,
//                    and scatter the cut-point table L_j = ceil(N q_j).
// Addition is commutative in IEEE arithmetic, so the butterfly computes
// node(2i)+node(2i+1) exactly as the reference does.
#pragma once
#include <math.h>

#include "common.cuh"
#include "philox.cuh"

namespace pf {

constexpr int CDF_THREADS = 256;
constexpr int CDF_V = 8;                         // consecutive elements per thread
constexpr int CDF_TILE = CDF_THREADS * CDF_V;    // 2048
constexpr int CDF_MAX_CHUNKS = 4096;             // top tree lives in one CTA
constexpr int CDF_SMALL_MAX = 1024;              // n <= this: single-CTA path

// Weight source: mode 0 -> w = exp(src - M) (the reference's
// np.exp(log_w - shift), filtering.py:297); mode 1 -> w = src.
struct WSrc {
  const double* src;
  const double* M;  // device scalar (mode 0)
  int mode;
};

// Batched replications (gridDim.z = R, step.cuh RepStride): the weight
// source of replication blockIdx.z -- its n_r log-weights and its max, held
// per replication by step parity ([R][2]).
PF_D WSrc wsrc_rep(WSrc s, int64_t n_r) {
  const int64_t r = blockIdx.z;
  s.src += r * n_r;
  if (s.M) s.M += 2 * r;
  return s;
}

template <typename T>
PF_D T weight_of(double v, double M, int mode) {
  return mode == 0 ? (T)exp(v - M) : (T)v;
}

template <typename T>
PF_D void load_tile_weights(const WSrc& s, int64_t base, double M, T (&v)[CDF_V]) {
  const double2* p = reinterpret_cast<const double2*>(s.src + base);
#pragma unroll
  for (int k = 0; k < CDF_V / 2; ++k) {
    double2 d = p[k];
    v[2 * k] = weight_of<T>(d.x, M, s.mode);
    v[2 * k + 1] = weight_of<T>(d.y, M, s.mode);
  }
}

// Tile plan for n >= CDF_TILE: G0 tiles of 2048, chunks of R tiles.
struct CdfPlan {
  int64_t n;
  int64_t tiles;
  int64_t chunks;
  int R;
  bool small;
};

inline CdfPlan cdf_plan(int64_t n) {
  CdfPlan p;
  p.n = n;
  p.small = n < CDF_TILE;
  if (p.small) {
    p.tiles = p.chunks = 1;
    p.R = 1;
    return p;
  }
  p.tiles = n / CDF_TILE;
  p.R = 1;
  while (p.tiles / p.R > CDF_MAX_CHUNKS) p.R *= 2;
  p.chunks = p.tiles / p.R;
  return p;
}

// Exact tree over 8 values held by thread: returns the three levels.
template <typename T>
PF_D void thread_tree8(const T (&v)[8], T (&l1)[4], T (&l2)[2], T& l3) {
#pragma unroll
  for (int i = 0; i < 4; ++i) l1[i] = v[2 * i] + v[2 * i + 1];
  l2[0] = l1[0] + l1[1];
  l2[1] = l1[2] + l1[3];
  l3 = l2[0] + l2[1];
}

// ------------------------------------------------------------------ K3 ---
// The top of the adder tree over the G chunk totals (prefix_sum.py:46-91):
// forward levels, backward pass down to the G chunk node values, and the
// exclusive running max of the nodes (the carry into each chunk).  One CTA;
// its scratch (fw: 2G, b0/b1: G each) is shared memory (cdf_top_kernel) or
// global memory reached through L2 (K2's last CTA, below).
struct SmemIO {
  template <typename T>
  PF_D static T ld(const T* p) { return *p; }
  template <typename T>
  PF_D static void st(T* p, T v) { *p = v; }
};
struct GlobalIO {  // L1-bypassing: the scratch is rewritten every step
  template <typename T>
  PF_D static T ld(const T* p) { return __ldcg(p); }
  template <typename T>
  PF_D static void st(T* p, T v) { __stcg(p, v); }
};

template <typename T, typename IO>
PF_D void top_tree_body(const T* __restrict__ chunk_tot, int64_t G, T* fw, T* b0, T* b1, T* __restrict__ node,
                        T* __restrict__ carry, T* __restrict__ total_out, int64_t* fail, int64_t step) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t i = tid; i < G; i += nt) IO::st(fw + i, __ldcg(chunk_tot + i));
  __syncthreads();
  int64_t off = 0, len = G;
  while (len > 1) {
    for (int64_t i = tid; i < len / 2; i += nt) IO::st(fw + off + len + i, (T)(IO::ld(fw + off + 2 * i) + IO::ld(fw + off + 2 * i + 1)));
    __syncthreads();
    off += len;
    len >>= 1;
  }
  const T total = IO::ld(fw + off);
  // backward: level offsets from the top down
  T* par = b0;
  T* chi = b1;
  if (tid == 0) IO::st(par, total);
  __syncthreads();
  int64_t plen = 1;
  int64_t loff = off;  // offset of the parent level in fw
  while (plen < G) {
    const int64_t clen = plen * 2;
    const int64_t coff = loff - clen;
    for (int64_t i = tid; i < clen; i += nt) {
      const T p = IO::ld(par + (i >> 1));
      IO::st(chi + i, (i & 1) ? p : (T)(p - IO::ld(fw + coff + i + 1)));
    }
    __syncthreads();
    T* tmp = par;
    par = chi;
    chi = tmp;
    plen = clen;
    loff = coff;
  }
  // par[0..G) = chunk node values.  Exclusive running max -> carry
  // (max is exact, so any scan order gives the reference's
  // np.maximum.accumulate bits).
  for (int64_t i = tid; i < G; i += nt) node[i] = IO::ld(par + i);
  {
    __shared__ T wm[32];
    const int64_t per = (G + nt - 1) / nt;
    const int64_t lo = tid * per;
    const int64_t hi = lo + per < G ? lo + per : G;
    T loc = (T)(-INFINITY);
    for (int64_t i = lo; i < hi; ++i) loc = fmax(loc, IO::ld(par + i));
    const int lane = tid & 31, warp = tid >> 5;
    T incl = loc;
    for (int o = 1; o < 32; o <<= 1) {
      const T other = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = fmax(incl, other);
    }
    if (lane == 31) wm[warp] = incl;
    __syncthreads();
    T pre = (T)(-INFINITY);
    for (int w = 0; w < warp; ++w) pre = fmax(pre, wm[w]);
    T ex = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane > 0) pre = fmax(pre, ex);
    for (int64_t i = lo; i < hi; ++i) {
      carry[i] = pre;
      pre = fmax(pre, IO::ld(par + i));
    }
  }
  if (tid == 0) {
    *total_out = total;
    if (!(total > (T)0) || !isfinite((double)total)) {
      if (fail) atomicCAS((unsigned long long*)fail, 0ull, (unsigned long long)(-step));
    }
  }
}

// K2 + K3 fused: when top.ctr is set, the last CTA to finish its chunk runs
// the top tree (no separate single-CTA launch, which a concurrent
// side-stream kernel holding every SM's resources could delay).
template <typename T>
struct TopFuse {
  unsigned int* ctr = nullptr;  // zero between launches; the last CTA resets it
  T* scratch = nullptr;         // 4G
  T* node = nullptr;
  T* carry = nullptr;
  T* total = nullptr;
  int64_t* fail = nullptr;
  int64_t step = 0;
};

// ------------------------------------------------------------------ K2 ---
template <typename T>
__global__ void __launch_bounds__(CDF_THREADS)
cdf_reduce_kernel(WSrc src, int R, T* __restrict__ tile_tot, T* __restrict__ chunk_tot,
                  const int64_t* __restrict__ fail, TopFuse<T> top = TopFuse<T>(),
                  double* __restrict__ wout = nullptr) {
  // wout (optional): the step's weights w = exp(lw - M) as computed here, for
  // K4 and the quantile classification to read (WSrc mode 1) instead of
  // recomputing the exp -- the same values, so the same bits
  if (gridDim.z > 1) {  // batched replications: replication blockIdx.z's tree
    const int64_t r = blockIdx.z, G = gridDim.x;
    if (wout) wout += r * G * R * CDF_TILE;
    src = wsrc_rep(src, G * R * CDF_TILE);
    tile_tot += r * G * R;
    chunk_tot += r * G;
    if (fail) fail += r;
    if (top.ctr) {
      top.ctr += r;
      top.scratch += r * 4 * G;
      top.node += r * G;
      top.carry += r * G;
      top.total += 2 * r;
      top.fail += r;
    }
  }
  pdl_wait();
  pdl_launch_dependents();
  if (fail && *fail) return;
  __shared__ T wt[CDF_THREADS / 32];
  __shared__ T tt[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double M = src.mode == 0 ? *src.M : 0.0;
  const int64_t chunk = blockIdx.x;
  for (int r = 0; r < R; ++r) {
    const int64_t tile = chunk * R + r;
    T v[CDF_V], l1[4], l2[2], g;
    load_tile_weights<T>(src, tile * CDF_TILE + threadIdx.x * CDF_V, M, v);
    if (wout) {
      double2* wp = reinterpret_cast<double2*>(wout + tile * CDF_TILE + threadIdx.x * CDF_V);
#pragma unroll
      for (int k = 0; k < CDF_V / 2; ++k) __stcg(wp + k, make_double2((double)v[2 * k], (double)v[2 * k + 1]));
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
  if (top.ctr) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(top.ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int64_t G = gridDim.x;
    top_tree_body<T, GlobalIO>(chunk_tot, G, top.scratch, top.scratch + 2 * G, top.scratch + 3 * G, top.node,
                               top.carry, top.total, top.fail, top.step);
    if (threadIdx.x == 0) *top.ctr = 0u;
  }
}

// One CTA of 1024 threads; dynamic smem = (2G + 2G) * sizeof(T).
template <typename T>
__global__ void __launch_bounds__(1024)
cdf_top_kernel(const T* __restrict__ chunk_tot, int64_t G, T* __restrict__ node,
               T* __restrict__ carry, T* __restrict__ total_out, int64_t* fail, int64_t step) {
  pdl_wait();
  pdl_launch_dependents();
  if (fail && *fail) return;
  extern __shared__ unsigned char smem_raw[];
  T* fw = reinterpret_cast<T*>(smem_raw);  // forward levels, 2G-1 nodes
  top_tree_body<T, SmemIO>(chunk_tot, G, fw, fw + 2 * G, fw + 3 * G, node, carry, total_out, fail, step);
}

// ------------------------------------------------ stratum lookup tables ---
// For N = 2^n with n >= 21 the cut-point lookup runs on integers against a
// compact, L2-resident rank structure instead of q / the cut table.
//
// A uniform u = K 2^-53 (K odd, 53 bits: unit_open) falls in stratum
// s = ceil(N u) = (K >> B) + 1, B = 53 - n, at offset r = K & (2^B - 1).  The
// particles whose CDF value lies in stratum s (L_k = ceil(N q_k) = s) are
// the consecutive run [I_s, I_{s+1}), I_s = first k with L_k >= s (the
// reference's cut point, resampling.py:124-131).  For such k,
//   u > q_k  <=>  r > F_k,   F_k = floor(q_k 2^53) - (s-1) 2^B  (exact),
// and F is nondecreasing along the run, so cutpoint_indices (resampling.py:
// 146-158: start at I_s, advance while u > q(k)) returns
//   I_s + #{ k in [I_s, I_{s+1}) : r > F_k }.
// Tables (rebuilt every step by K4 + group_build_kernel):
//   cut  int32 [N+1]   I_s (0-based), cut[N] = N       (fallback, group build)
//   grp  16 B per 8 strata: base = I of the group's first stratum and the 8
//        cumulative run ends (bytes, relative to base), so I_s and c_s are two
//        byte extracts (overflow bit 31 of base when the group's 8 runs hold
//        more than 255 particles: lookups then read cut[] directly)
//   fq   uint8 [N]     F_k >> (B-8) clamped to 255 (monotone quantisation)
//   f32  uint32 [N]    F_k clamped to 2^32-1 (exact, read only when fq ties)
// grp + fq are 3 B per particle (48 MB at 2^24) and are read with an L2
// evict_last policy, so a lookup is L2 hits; the ancestor's record gather is
// the one random DRAM access per slot (a random read moves a 128 B DRAM atom
// on B200, measured: scripts/micro/gather.cu).  Same answer as the
// reference, bit for bit.
struct alignas(16) Grp {
  uint32_t base;  // bit 31: overflow
  uint32_t pad;
  uint64_t cum;   // byte i: I_{first stratum + i + 1} - base
};
constexpr int STRATA_MIN_LOG2N = 21;
constexpr int GRP_STRATA = 8;
constexpr uint32_t GRP_OVERFLOW = 0x80000000u;

struct RankOut {  // K4 outputs on the strata path
  int32_t* cut;
  uint8_t* fq;
  uint32_t* f32;
  int B;
};

template <typename T>
PF_D uint32_t strata_f(T q, int64_t L, double unitB /* 2^B */) {
  if (L <= 0) return 0u;
  const double x = (double)q * 9007199254740992.0;          // q 2^53, exact
  const double sub = (double)(L - 1) * unitB;               // exact
  const double d = floor(x - sub);                          // exact (Sterbenz)
  return d >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)d;
}

// One thread per group of 8 strata: cumulative run ends from the cut table.
__global__ void __launch_bounds__(256)
group_build_kernel(const int32_t* __restrict__ cut, int64_t ngroups, Grp* __restrict__ grp,
                   const int64_t* __restrict__ fail) {
  pdl_wait();
  pdl_launch_dependents();
  if (fail && *fail) return;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* c = cut + g * GRP_STRATA;
    const uint32_t base = (uint32_t)c[0];
    uint64_t cum = 0;
    bool over = false;
#pragma unroll
    for (int i = 0; i < GRP_STRATA; ++i) {
      const uint32_t e = (uint32_t)(c[i + 1] - (int32_t)base);
      over |= e > 255u;
      cum |= (uint64_t)(e & 255u) << (8 * i);
    }
    Grp r;
    r.base = base | (over ? GRP_OVERFLOW : 0u);
    r.pad = 0;
    r.cum = cum;
    grp[g] = r;
  }
}

// ------------------------------------------------------------------ K4 ---
template <typename T>
PF_D T clip01(T x) { return fmin(fmax(x, (T)0), (T)1); }

template <typename T, bool STRATA = false>
__global__ void __launch_bounds__(CDF_THREADS)
cdf_expand_kernel(WSrc src, int64_t n, int R, const T* __restrict__ tile_tot,
                  const T* __restrict__ node, const T* __restrict__ carry,
                  const T* __restrict__ total_p, T* __restrict__ q_out,
                  int32_t* __restrict__ cut_out, const int64_t* __restrict__ fail,
                  RankOut ro = RankOut(), int64_t gbase = 0) {
  if (gridDim.z > 1) {  // batched replications (non-strata tables only)
    const int64_t r = blockIdx.z, G = gridDim.x;
    src = wsrc_rep(src, n);
    tile_tot += r * G * R;
    node += r * G;
    carry += r * G;
    total_p += 2 * r;
    q_out += r * n;
    cut_out += r * n;
    if (fail) fail += r;
  }
  pdl_wait();
  pdl_launch_dependents();
  if (fail && *fail) return;
  __shared__ T wt[CDF_THREADS / 32];
  __shared__ T wmax[CDF_THREADS / 32];
  __shared__ T tnode[64], tcarry[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double M = src.mode == 0 ? *src.M : 0.0;
  const T total = *total_p;
  const T nf = (T)n;
  const int64_t chunk = blockIdx.x;
  if (threadIdx.x == 0) {
    // subtree over this chunk's R tile sums: forward, then backward from the
    // chunk node; per-tile carries of the running max.
    T fwl[128];  // R <= 32 (n <= 2^28)
    for (int r = 0; r < R; ++r) fwl[r] = tile_tot[chunk * R + r];
    int offs[8], k = 0, off = 0, len = R;
    offs[k++] = 0;
    while (len > 1) {
      for (int i = 0; i < len / 2; ++i) fwl[off + len + i] = fwl[off + 2 * i] + fwl[off + 2 * i + 1];
      off += len;
      len >>= 1;
      offs[k++] = off;
    }
    T bw[64], nb[64];
    bw[0] = node[chunk];
    int plen = 1;
    for (int lvl = k - 2; lvl >= 0; --lvl) {
      const int co = offs[lvl];
      for (int i = 0; i < plen * 2; ++i) nb[i] = (i & 1) ? bw[i >> 1] : (T)(bw[i >> 1] - fwl[co + i + 1]);
      plen *= 2;
      for (int i = 0; i < plen; ++i) bw[i] = nb[i];
    }
    // carries are node values (prefix-sum units); the running max of q over
    // the preceding elements is (max node) / total since division by a
    // positive total is monotone.
    T m = carry[chunk];
    for (int r = 0; r < R; ++r) {
      tnode[r] = bw[r];
      tcarry[r] = m / total;
      m = fmax(m, bw[r]);
    }
  }
  __syncthreads();
  for (int r = 0; r < R; ++r) {
    const int64_t tile = chunk * R + r;
    const int64_t base = tile * CDF_TILE + threadIdx.x * CDF_V;
    T v[CDF_V], l1[4], l2[2], l3;
    load_tile_weights<T>(src, base, M, v);
    thread_tree8<T>(v, l1, l2, l3);
    T p[5];
    T g = l3;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      p[k] = __shfl_xor_sync(0xffffffffu, g, 1 << k);
      g = g + p[k];
    }
    if (lane == 0) wt[warp] = g;
    __syncthreads();
    // backward: tile node -> warp node (3 levels over 8 warp sums)
    T val = tnode[r];
    {
      const T a0 = wt[0] + wt[1], a1 = wt[2] + wt[3], a2 = wt[4] + wt[5], a3 = wt[6] + wt[7];
      const T b0 = a0 + a1, b1 = a2 + a3;
      const T A[4] = {a0, a1, a2, a3};
      if (!((warp >> 2) & 1)) val = val - b1;
      const int h = warp >> 1;  // pair index 0..3
      if (!(h & 1)) val = val - A[h + 1];
      if (!(warp & 1)) val = val - wt[warp + 1];
      (void)b0;
    }
    // warp node -> lane node
#pragma unroll
    for (int k = 4; k >= 0; --k)
      if (!((lane >> k) & 1)) val = val - p[k];
    // lane node -> 8 leaves
    T s[CDF_V];
    {
      const T n2l = val - l2[1], n2r = val;
      const T n1[4] = {n2l - l1[1], n2l, n2r - l1[3], n2r};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        s[2 * i] = n1[i] - v[2 * i + 1];
        s[2 * i + 1] = n1[i];
      }
    }
    // q = s / total, thread-local running max
    T run[CDF_V];
    T m = (T)(-INFINITY);
#pragma unroll
    for (int i = 0; i < CDF_V; ++i) {
      const T qi = s[i] / total;
      m = fmax(m, qi);
      run[i] = m;
    }
    // exclusive prefix max across lanes and warps, seeded by the tile carry
    T incl = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T other = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = fmax(incl, other);
    }
    T excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = (T)(-INFINITY);
    __syncthreads();  // wt reads done before wmax reuse ordering
    if (lane == 31) wmax[warp] = incl;
    __syncthreads();
    T pre = tcarry[r];
    for (int w = 0; w < warp; ++w) pre = fmax(pre, wmax[w]);
    pre = fmax(pre, excl);
    // finalize and scatter the cut table
    const double unitB = STRATA ? ldexp(1.0, ro.B) : 0.0;
    T qv[CDF_V];
    int64_t Lprev = (int64_t)ceil(clip01(pre) * nf);
    uint64_t fqw = 0;
    uint32_t fx[CDF_V];
#pragma unroll
    for (int i = 0; i < CDF_V; ++i) {
      T qi = clip01(fmax(pre, run[i]));
      if (gbase + base + i == n - 1) qi = (T)1;
      qv[i] = qi;
      const int64_t L = (int64_t)ceil(qi * nf);
      int32_t* ct = STRATA ? ro.cut : cut_out;
      // strata [Lprev, L) start at this particle: usually 0, 1 or 2 of them,
      // so the first two stores are predicated and only longer runs loop
      const int32_t v = (int32_t)(gbase + base + i);
      if (L > Lprev) {
        ct[Lprev] = v;
        if (L > Lprev + 1) {
          ct[Lprev + 1] = v;
          for (int64_t kk = Lprev + 2; kk < L; ++kk) ct[kk] = v;
        }
      }
      if (STRATA) {
        const uint32_t f = strata_f<T>(qi, L, unitB);
        fx[i] = f;
        const uint32_t h = f >> (ro.B - 8);
        fqw |= (uint64_t)(h > 255u ? 255u : h) << (8 * i);
      }
      Lprev = L > Lprev ? L : Lprev;
    }
    if (STRATA) {
      *reinterpret_cast<uint64_t*>(ro.fq + base) = fqw;
      uint4* fp = reinterpret_cast<uint4*>(ro.f32 + base);
      fp[0] = make_uint4(fx[0], fx[1], fx[2], fx[3]);
      fp[1] = make_uint4(fx[4], fx[5], fx[6], fx[7]);
      if (q_out) {  // sharded runs keep q for the boundary lookups
#pragma unroll
        for (int i = 0; i < CDF_V; ++i) q_out[base + i] = qv[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < CDF_V; ++i) q_out[base + i] = qv[i];
    }
    __syncthreads();
  }
}

// ------------------------------------------------ sharded (multi-GPU) ---
// G shards of N/G consecutive particles: each shard is a subtree of the
// reference's adder tree, so the run is bit-identical to one device.
//   K3a cdf_shard_total: the shard's subtree total (forward tree over its
//       chunk totals) -> the exchange array (one value per shard);
//   K3b cdf_top_shard: every shard rebuilds the G-level top tree from the
//       exchanged totals (root = the reference's total), runs the backward
//       adder down to all shard nodes, then down its own chunks; the carry
//       into a shard is the running max of the shard nodes before it (a
//       node never exceeds its parent, so a shard's largest prefix is its
//       node); and the stratum boundaries L_end of every shard for the
//       cross-shard cut-point lookup.
constexpr int PF_MAX_SHARDS = 8;

template <typename T>
__global__ void __launch_bounds__(1024)
cdf_shard_total_kernel(const T* __restrict__ chunk_tot, int64_t C, T* __restrict__ xtot, int shard,
                       const int64_t* fail) {
  if (fail && *fail) return;
  extern __shared__ unsigned char smem_raw[];
  T* fw = reinterpret_cast<T*>(smem_raw);  // 2C
  for (int64_t i = threadIdx.x; i < C; i += blockDim.x) fw[i] = chunk_tot[i];
  __syncthreads();
  int64_t off = 0, len = C;
  while (len > 1) {
    for (int64_t i = threadIdx.x; i < len / 2; i += blockDim.x) fw[off + len + i] = fw[off + 2 * i] + fw[off + 2 * i + 1];
    __syncthreads();
    off += len;
    len >>= 1;
  }
  if (threadIdx.x == 0) {
    xtot[shard] = fw[off];
    __threadfence_system();
  }
}

template <typename T>
__global__ void __launch_bounds__(1024)
cdf_top_shard_kernel(const T* __restrict__ chunk_tot, int64_t C, const T* __restrict__ xtot, int G, int shard,
                     int64_t n_total, T* __restrict__ node, T* __restrict__ carry, T* __restrict__ total_out,
                     int64_t* __restrict__ lend, int64_t* fail, int64_t step) {
  if (fail && *fail) return;
  extern __shared__ unsigned char smem_raw[];
  T* fw = reinterpret_cast<T*>(smem_raw);  // forward levels of the chunk tree, 2C
  T* b0 = fw + 2 * C;
  T* b1 = b0 + C;
  __shared__ T snode[PF_MAX_SHARDS];
  __shared__ T sroot, scarry;
  // top tree over the G shard totals, backward to the shard nodes (thread 0)
  if (threadIdx.x == 0) {
    T lv[2 * PF_MAX_SHARDS];
    for (int g = 0; g < G; ++g) lv[g] = __ldcg(&xtot[g]);
    int offs[4], k = 0, off = 0, len = G;
    offs[k++] = 0;
    while (len > 1) {
      for (int i = 0; i < len / 2; ++i) lv[off + len + i] = lv[off + 2 * i] + lv[off + 2 * i + 1];
      off += len;
      len >>= 1;
      offs[k++] = off;
    }
    const T root = lv[off];
    T bw[PF_MAX_SHARDS], nb[PF_MAX_SHARDS];
    bw[0] = root;
    int plen = 1;
    for (int lvl = k - 2; lvl >= 0; --lvl) {
      const int co = offs[lvl];
      for (int i = 0; i < plen * 2; ++i) nb[i] = (i & 1) ? bw[i >> 1] : (T)(bw[i >> 1] - lv[co + i + 1]);
      plen *= 2;
      for (int i = 0; i < plen; ++i) bw[i] = nb[i];
    }
    // carries (exclusive running max of shard nodes) and stratum bounds
    T m = (T)(-INFINITY);
    const T nf = (T)n_total;
    for (int g = 0; g < G; ++g) {
      snode[g] = bw[g];
      if (g == shard) scarry = m;
      m = fmax(m, bw[g]);
      const T qe = (g == G - 1) ? (T)1 : clip01(m / root);
      lend[g] = (int64_t)ceil(qe * nf);
    }
    sroot = root;
    *total_out = root;
    if (!(root > (T)0) || !isfinite((double)root)) {
      if (fail) atomicCAS((unsigned long long*)fail, 0ull, (unsigned long long)(-step));
    }
  }
  // forward tree over this shard's chunk totals
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t i = tid; i < C; i += nt) fw[i] = chunk_tot[i];
  __syncthreads();
  int64_t off = 0, len = C;
  while (len > 1) {
    for (int64_t i = tid; i < len / 2; i += nt) fw[off + len + i] = fw[off + 2 * i] + fw[off + 2 * i + 1];
    __syncthreads();
    off += len;
    len >>= 1;
  }
  // backward from the shard node
  T* par = b0;
  T* chi = b1;
  if (tid == 0) par[0] = snode[shard];
  __syncthreads();
  int64_t plen = 1, loff = off;
  while (plen < C) {
    const int64_t clen = plen * 2, coff = loff - clen;
    for (int64_t i = tid; i < clen; i += nt) {
      const T pv = par[i >> 1];
      chi[i] = (i & 1) ? pv : (T)(pv - fw[coff + i + 1]);
    }
    __syncthreads();
    T* tmp = par;
    par = chi;
    chi = tmp;
    plen = clen;
    loff = coff;
  }
  for (int64_t i = tid; i < C; i += nt) node[i] = par[i];
  // chunk carries: running max seeded with the shard carry (serial over the
  // shard's chunks: C <= 4096)
  __syncthreads();
  if (tid == 0) {
    T m = scarry;
    for (int64_t i = 0; i < C; ++i) {
      carry[i] = m;
      m = fmax(m, par[i]);
    }
  }
  (void)sroot;
}

// Cross-shard cut-point lookup (resampling.py:146-158): the stratum's owner
// shard from the L_end bounds, I_s from its cut table, then the advance
// over q(k) wherever particle k lives.
template <typename TQ>
struct ShardLookup {
  const int32_t* cut[PF_MAX_SHARDS];  // full-size (N) per shard, own strata written
  const TQ* q[PF_MAX_SHARDS];         // per shard, local particles
  const int64_t* lend;                // [G], this shard's copy
  int G;
  int lg;                             // log2(N / G)
  int64_t n;                          // N total
};

template <typename TQ>
PF_D int64_t sharded_lookup(const ShardLookup<TQ>& L, uint64_t w3) {
  const double u = unit_open(w3);
  const int64_t s0 = (int64_t)ceil(u * (double)L.n) - 1;
  int g = 0;
  while (g < L.G - 1 && __ldcg(&L.lend[g]) <= s0) ++g;
  int64_t k = __ldcg(&L.cut[g][s0]);
  const int64_t mask = ((int64_t)1 << L.lg) - 1;
  while (u > (double)__ldcg(&L.q[k >> L.lg][k & mask])) ++k;
  return k;
}

// ---------------------------------------- sequential baseline resamplers ---
// The reference's CPU comparators (resampling.py:29-87) run on a plain
// left-to-right cumsum (sequential_cdf, prefix_sum.py:130-134).  Its rounding
// chain is inherently sequential, so one thread walks it -- bit-identical to
// numpy's cumsum (in the weights' dtype), then _finalize_cdf against the last
// prefix.  Fine for the baselines' role (and for N = 10^4, BASELINE
// configs[0]); O(N) latency-bound at large N.
template <typename T>
__global__ void seq_cdf_kernel(WSrc src, int64_t n, T* __restrict__ q, int64_t* fail, int64_t step) {
  if (*fail || threadIdx.x != 0 || blockIdx.x != 0) return;
  const double M = src.mode == 0 ? *src.M : 0.0;
  T s = (T)0;
  for (int64_t i = 0; i < n; ++i) {
    s = s + weight_of<T>(src.src[i], M, src.mode);
    q[i] = s;
  }
  const T total = s;
  if (!(total > (T)0) || !isfinite((double)total)) {
    atomicCAS((unsigned long long*)fail, 0ull, (unsigned long long)(-step));
    return;
  }
  T m = (T)(-INFINITY);
  for (int64_t i = 0; i < n; ++i) {
    m = fmax(m, q[i] / total);
    q[i] = clip01(m);
  }
  q[n - 1] = (T)1;
}

// The uniform each slot searches for: naive -> its own; stratified ->
// (j + v_j)/n; systematic -> (j + v)/n with the step's single aux draw;
// sorted -> written as sortable keys (positive doubles order as uint64).
enum { RS_CUT = 0, RS_NAIVE = 1, RS_SORTED = 2, RS_STRAT = 3, RS_SYST = 4 };

__global__ void resample_uniforms_kernel(int scheme, const uint64_t* __restrict__ u3, int64_t n, uint64_t seed,
                                         int64_t t, double* __restrict__ u_out, const int64_t* fail) {
  if (*fail) return;
  __shared__ double vaux;
  if (scheme == RS_SYST) {
    // aux stream 2^62 (rng.py:34), one draw per step: counter t-1
    if (threadIdx.x == 0) {
      const uint64_t c = (uint64_t)(t - 1);
      const Philox4 P = philox_block(seed, 1ull << 62, c >> 2);
      vaux = unit_open(P.w[c & 3]);
    }
    __syncthreads();
  }
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double v = unit_open(u3[j]);
    double u;
    if (scheme == RS_STRAT) u = ((double)j + v) / (double)n;
    else if (scheme == RS_SYST) u = ((double)j + vaux) / (double)n;
    else u = v;
    u_out[j] = u;
  }
}

// --------------------------------------- K7: ordered uniforms (spacings) ---
// Perf-mode exact multinomial resampling (PF_RESAMPLE_SPACINGS).  The
// reference's `sorted` scheme (resampling.py:57-67) sorts N uniforms and
// merges them against the CDF (merge_indices, :29-36).  Here the sorted
// uniforms are produced in order without a sort: with E_1..E_(N+1) i.i.d.
// standard exponentials and S_k = E_1 + ... + E_k, (S_1, ..., S_N) / S_(N+1)
// are distributed as the order statistics of N uniforms.  E_j comes from slot
// j's resampling word (Philox word 3 of block t, the word cutpoint uses) and
// E_(N+1) from the aux stream SPACINGS_STREAM; the scan is one pass over the
// words (device prefix sum).  The ordered uniform of slot k is handed to the
// next step as a resampling word (u = K 2^-53, K odd: the cut-point lookup's
// input), so the lookup machinery is shared with cutpoint -- and because the
// uniforms are nondecreasing in k, so are the ancestors: the step kernel's
// record gathers stream instead of landing on random 128 B atoms, and in a
// sharded run a shard's ancestors lie in the shard except at its ends.
constexpr uint64_t SPACINGS_STREAM = (1ull << 62) + 2;  // aux stream (rng.py:34 numbering)

struct ExpOfWord {  // E_j = -log(unit_open(w3_j)), a standard exponential
  const uint64_t* w3;
  __host__ __device__ double operator()(int64_t j) const { return -log(unit_open(w3[j])); }
};

PF_HD double spacings_aux_exp(uint64_t seed, int64_t t) {
  const Philox4 P = philox_block(seed, SPACINGS_STREAM, (uint64_t)t);
  return -log(unit_open(P.w[0]));
}

// Resampling word of the ordered uniform U = S / S_tot: K = floor(U 2^53) | 1
// (odd, < 2^53), stored so that unit_open(word) = K 2^-53.
PF_D uint64_t spacings_word(double S, double inv_tot) {
  uint64_t K = (uint64_t)(S * inv_tot * 9007199254740992.0);
  K |= 1ull;
  if (K > 9007199254740991ull) K = 9007199254740991ull;
  return (K >> 1) << 12;
}

// words[j] for a shard's slots: S_local (inclusive prefix sums over the
// shard), the shard's offset (sum of the earlier shards' E totals) and the
// grand total S_(N+1) (all shards' totals + the aux exponential).  One device
// / one shard: offset 0, totals = {S_local[n-1]}.
__global__ void spacings_words_kernel(const double* __restrict__ S, int64_t n, const double* __restrict__ totals,
                                      int nshards, int shard, uint64_t seed, int64_t t, uint64_t* __restrict__ words,
                                      const int64_t* __restrict__ fail) {
  if (fail && *fail) return;
  double off = 0.0, tot = 0.0;
  for (int h = 0; h < nshards; ++h) {  // fixed order: identical on every shard
    const double th = totals ? __ldcg(totals + h) : S[n - 1];
    if (h < shard) off += th;
    tot += th;
  }
  tot += spacings_aux_exp(seed, t);
  const double inv = 1.0 / tot;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    words[j] = spacings_word(off + S[j], inv);
}

// Sharded K7: the shard's exponential total goes into its exchange record
// (after its scan; the record itself was written by its step kernel).
template <typename XRec>
__global__ void spacings_shard_total_kernel(const double* __restrict__ S, int64_t ns, XRec* xrec, int shard) {
  xrec[shard].se = S[ns - 1];
  __threadfence_system();
}

// merge_indices (resampling.py:29-36): searchsorted(q, u, 'right'), 0-based.
template <typename T>
__global__ void merge_kernel(const T* __restrict__ q, int64_t n, const double* __restrict__ u, int64_t m,
                             int32_t* __restrict__ anc, const int64_t* fail) {
  if (*fail) return;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    const double uj = u[j];
    int64_t lo = 0, hi = n;  // first i with q[i] > u
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((double)q[mid] <= uj) lo = mid + 1; else hi = mid;
    }
    anc[j] = (int32_t)(lo < n ? lo : n - 1);
  }
}

// ------------------------------------------------------- small n path ---
// n <= CDF_SMALL_MAX: one CTA, levels in shared memory (the reference's
// level loops verbatim), finalize and cut table by one thread.
template <typename T>
__global__ void __launch_bounds__(256)
cdf_small_kernel(WSrc src, int64_t n, T* __restrict__ q_out, int32_t* __restrict__ cut_out,
                 T* __restrict__ total_out, int64_t* fail, int64_t step) {
  if (fail && *fail) return;
  __shared__ T fw[2 * CDF_SMALL_MAX];
  __shared__ T bw[2 * CDF_SMALL_MAX];
  const double M = src.mode == 0 ? *src.M : 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) fw[i] = weight_of<T>(src.src[i], M, src.mode);
  __syncthreads();
  int64_t off = 0, len = n;
  while (len > 1) {
    for (int64_t i = threadIdx.x; i < len / 2; i += blockDim.x)
      fw[off + len + i] = fw[off + 2 * i] + fw[off + 2 * i + 1];
    __syncthreads();
    off += len;
    len >>= 1;
  }
  const T total = fw[off];
  // backward level by level into bw (same offsets as fw)
  if (threadIdx.x == 0) bw[off] = total;
  __syncthreads();
  int64_t plen = 1, poff = off;
  while (plen < n) {
    const int64_t clen = plen * 2, coff = poff - clen;
    for (int64_t i = threadIdx.x; i < clen; i += blockDim.x) {
      const T p = bw[poff + (i >> 1)];
      bw[coff + i] = (i & 1) ? p : (T)(p - fw[coff + i + 1]);
    }
    __syncthreads();
    plen = clen;
    poff = coff;
  }
  if (threadIdx.x == 0) {
    *total_out = total;
    if (!(total > (T)0) || !isfinite((double)total)) {
      if (fail) atomicCAS((unsigned long long*)fail, 0ull, (unsigned long long)(-step));
      return;
    }
    T m = (T)(-INFINITY);
    int64_t Lprev = 0;
    const T nf = (T)n;
    for (int64_t i = 0; i < n; ++i) {
      m = fmax(m, bw[i] / total);
      T qi = clip01(m);
      if (i == n - 1) qi = (T)1;
      q_out[i] = qi;
      const int64_t L = (int64_t)ceil(qi * nf);
      for (int64_t k = Lprev; k < L; ++k) cut_out[k] = (int32_t)i;
      Lprev = L > Lprev ? L : Lprev;
    }
  }
}

// -------------------------------------------------------------- lookup ---
// cutpoint_indices (resampling.py:146-158): k = I[ceil(N u) - 1], then
// advance while u > q(k).  Returns the 0-based ancestor.  Equals
// searchsorted(q, u, 'left').
template <typename T>
PF_D int64_t cutpoint_lookup(const T* __restrict__ q, const int32_t* __restrict__ cut, int64_t n,
                             double u) {
  const int64_t s = (int64_t)ceil(u * (double)n);
  int64_t k = cut[s - 1];
  while (u > (double)q[k]) ++k;
  return k;
}

// The resampling table of one step: (q, cut) for small n, the rank
// structure for n >= 2^21 (see Grp).  ancestor_of() takes the raw Philox
// word whose unit_open() is the resampling uniform.
template <typename TQ>
struct Lookup {
  const int32_t* anc;   // non-null: ancestors precomputed (baseline resamplers)
  const TQ* q;
  const int32_t* cut;
  const Grp* grp;       // non-null: strata path
  const uint8_t* fq;
  const uint32_t* f32;
  int B;
  int64_t n;
};

// L2 eviction-priority hints: the rank tables are re-read by every slot of
// the step (keep them), the ancestor records are touched ~once (stream them).
PF_D uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
PF_D Grp ld_grp(const Grp* p, uint64_t pol) {
  uint32_t a, b, c, d;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p), "l"(pol));
  Grp g;
  g.base = a;
  g.pad = b;
  g.cum = (uint64_t)c | ((uint64_t)d << 32);
  return g;
}
PF_D uint64_t ld_fq8(const uint8_t* p, uint64_t pol) {  // 8-byte aligned
  uint64_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
PF_D uint32_t ld_fq(const uint8_t* p, uint64_t pol) {
  uint16_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return (uint32_t)v;
}

// Run start I_s and length c_s of stratum s0 (0-based).
template <typename TQ>
PF_D void stratum_run(const Lookup<TQ>& L, const Grp& g, uint64_t s0, int64_t& first, int& cnt) {
  if (g.base & GRP_OVERFLOW) {
    first = L.cut[s0];
    cnt = (int)(L.cut[s0 + 1] - first);
    return;
  }
  const int sh = 8 * (int)(s0 & (GRP_STRATA - 1));
  const uint32_t end = (uint32_t)(g.cum >> sh) & 255u;
  const uint32_t beg = sh ? (uint32_t)(g.cum >> (sh - 8)) & 255u : 0u;
  first = (int64_t)g.base + beg;
  cnt = (int)(end - beg);
}

// #{k in [first, first+cnt) : r > F_k}, F nondecreasing along the run.
template <typename TQ>
PF_D int64_t run_count(const Lookup<TQ>& L, int64_t first, int cnt, uint32_t r, uint64_t pol) {
  const uint32_t rh = r >> (L.B - 8);
  int64_t k = first;
  for (int m = 0; m < cnt; ++m, ++k) {
    const uint32_t h = ld_fq(L.fq + k, pol);
    if (rh < h) break;
    if (rh == h && r <= __ldg(L.f32 + k)) break;
  }
  return k;
}

// Same count from the two aligned 8-byte words of fq covering bytes
// first .. first+7 (fq is padded by 16 bytes): the bytes below r's are a
// prefix of the run (fq is nondecreasing along it), counted with one SIMD
// byte compare; an equal byte, or a run longer than 8, takes run_count.
template <typename TQ>
PF_D int64_t run_count_win(const Lookup<TQ>& L, int64_t first, int cnt, uint32_t r, uint64_t w0, uint64_t w1,
                           uint64_t pol) {
  if (cnt == 0) return first;
  const uint32_t rh = r >> (L.B - 8);
  const int sh = (int)(first & 7) * 8;
  const uint64_t win = sh ? ((w0 >> sh) | (w1 << (64 - sh))) : w0;
  const int m = cnt < 8 ? cnt : 8;
  const uint32_t rb = rh * 0x01010101u;
  const uint64_t cm = (uint64_t)__vcmpltu4((uint32_t)win, rb) |
                      ((uint64_t)__vcmpltu4((uint32_t)(win >> 32), rb) << 32);
  const uint64_t mask = m == 8 ? ~0ull : ((1ull << (8 * m)) - 1ull);
  const int k = __popcll(cm & mask) >> 3;
  if (k < m) {
    if (((win >> (8 * k)) & 0xFFu) != rh) return first + k;
  } else if (cnt <= 8) {
    return first + cnt;
  }
  return run_count(L, first + k, cnt - k, r, pol);
}

template <typename TQ>
PF_D int64_t ancestor_of(const Lookup<TQ>& L, uint64_t w3) {
  if (L.grp) {
    const uint64_t pol = l2_policy_last();
    const uint64_t K = ((w3 >> 12) << 1) | 1ull;  // u = K 2^-53
    const uint64_t s0 = K >> L.B;                 // stratum - 1
    const uint32_t r = (uint32_t)(K & ((1ull << L.B) - 1ull));
    const Grp g = ld_grp(L.grp + (s0 / GRP_STRATA), pol);
    int64_t first;
    int cnt;
    stratum_run(L, g, s0, first, cnt);
    return run_count(L, first, cnt, r, pol);
  }
  return cutpoint_lookup<TQ>(L.q, L.cut, L.n, unit_open(w3));
}

// SB lookups at once: two rounds of independent L2 loads (all groups, then
// all fq windows), then the rare exact / long-run walks.
template <typename TQ, int SB>
PF_D void ancestors_of(const Lookup<TQ>& L, const uint64_t (&w3)[SB], const bool (&ok)[SB],
                       int64_t (&anc)[SB]) {
  if (L.grp) {
    const uint64_t pol = l2_policy_last();
    uint32_t r[SB];
    uint64_t s0[SB];
    Grp G[SB];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const uint64_t K = ((w3[b] >> 12) << 1) | 1ull;
      s0[b] = ok[b] ? (K >> L.B) : 0;
      r[b] = (uint32_t)(K & ((1ull << L.B) - 1ull));
    }
#pragma unroll
    for (int b = 0; b < SB; ++b) G[b] = ld_grp(L.grp + (s0[b] / GRP_STRATA), pol);
    int64_t first[SB];
    int cnt[SB];
#pragma unroll
    for (int b = 0; b < SB; ++b) stratum_run(L, G[b], s0[b], first[b], cnt[b]);
    uint64_t w0[SB], w1[SB];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const uint8_t* p = L.fq + (first[b] & ~7ll);
      w0[b] = ld_fq8(p, pol);
      w1[b] = ld_fq8(p + 8, pol);
    }
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const int64_t k = run_count_win(L, first[b], cnt[b], r[b], w0[b], w1[b], pol);
      if (ok[b]) anc[b] = k;
    }
    return;
  }
#pragma unroll
  for (int b = 0; b < SB; ++b)
    if (ok[b]) anc[b] = cutpoint_lookup<TQ>(L.q, L.cut, L.n, unit_open(w3[b]));
}

// ------------------------------------------- sharded rank-table lookup ---
// The rank tables of a sharded run, per shard g: grp over the GLOBAL stratum
// groups (entries valid only for groups whose 8 strata and closing cut lie
// in g's stratum range [L_end[g-1], L_end[g]); boundary groups carry pad = 1
// and take the cut/q walk), fq / f32 over g's own particles.  A lookup reads
// the owner shard's tables (peer memory when it is another GPU) and counts
// in the owner's run exactly as ancestor_of does on one device.
constexpr uint32_t GRP_BOUNDARY = 1u;

struct ShardRank {
  const Grp* grp[PF_MAX_SHARDS];      // [N / 8] per shard (global groups)
  const uint8_t* fq[PF_MAX_SHARDS];   // [N / G (+16)] per shard
  const uint32_t* f32[PF_MAX_SHARDS];
  int B;                              // 53 - log2(N)
  int on;
};

// One thread per global group that intersects this shard's stratum range.
__global__ void __launch_bounds__(256)
group_build_shard_kernel(const int32_t* __restrict__ cut, const int64_t* __restrict__ lend, int shard, int G,
                         int64_t n, Grp* __restrict__ grp, const int64_t* __restrict__ fail) {
  pdl_wait();
  if (fail && *fail) return;
  const int64_t lo = shard ? __ldcg(&lend[shard - 1]) : 0, hi = __ldcg(&lend[shard]);
  const int64_t g0 = lo / GRP_STRATA, g1 = (hi + GRP_STRATA - 1) / GRP_STRATA;
  for (int64_t gi = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < g1;
       gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = gi * GRP_STRATA;
    const bool full = s >= lo && (s + GRP_STRATA < hi || (shard == G - 1 && s + GRP_STRATA <= n));
    Grp r;
    r.pad = full ? 0u : GRP_BOUNDARY;
    r.base = GRP_OVERFLOW;
    r.cum = 0;
    if (full) {
      const int32_t* c = cut + s;
      const uint32_t base = (uint32_t)c[0];
      uint64_t cum = 0;
      bool over = false;
#pragma unroll
      for (int i = 0; i < GRP_STRATA; ++i) {
        const uint32_t e = (uint32_t)(c[i + 1] - (int32_t)base);
        over |= e > 255u;
        cum |= (uint64_t)(e & 255u) << (8 * i);
      }
      r.base = base | (over ? GRP_OVERFLOW : 0u);
      r.cum = cum;
    }
    grp[gi] = r;
  }
}

template <typename TQ>
PF_D int64_t sharded_lookup_rank(const ShardLookup<TQ>& SL, const ShardRank& R, uint64_t w3) {
  const uint64_t K = ((w3 >> 12) << 1) | 1ull;  // u = K 2^-53
  const uint64_t s0 = K >> R.B;
  int g = 0;
  while (g < SL.G - 1 && __ldcg(&SL.lend[g]) <= (int64_t)s0) ++g;
  const uint64_t pol = l2_policy_last();
  const Grp gr = ld_grp(R.grp[g] + s0 / GRP_STRATA, pol);
  if (gr.pad & GRP_BOUNDARY) return sharded_lookup<TQ>(SL, w3);
  // the owner's tables, addressed by global particle index
  const int64_t gb = (int64_t)g << SL.lg;
  Lookup<TQ> L;
  L.anc = nullptr;
  L.q = nullptr;
  L.cut = SL.cut[g];
  L.grp = R.grp[g];
  L.fq = R.fq[g] - gb;
  L.f32 = R.f32[g] - gb;
  L.B = R.B;
  L.n = SL.n;
  const uint32_t r = (uint32_t)(K & ((1ull << R.B) - 1ull));
  int64_t first;
  int cnt;
  stratum_run(L, gr, s0, first, cnt);
  return run_count(L, first, cnt, r, pol);
}

}  // namespace pf
