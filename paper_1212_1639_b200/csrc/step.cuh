// Particle kernels of the full PF / PL cycle (filtering.py:220-358).
//
//  K0  init_kernel        x0, sigma2_0, tau2_0 per slot (filtering.py:225-252)
//  K1  step_kernel        for slot j at step t:
//                           resample of step t-1: cut-point lookup of
//                           u(j, 4(t-1)+3) against q_{t-1} and a joint gather
//                           of the ancestor's record (filtering.py:305-330)
//                           -- fused here so the gathered tuple never makes an
//                           extra trip through HBM;
//                           propagate + sufficient statistics + parameter
//                           draws from Philox block t (filtering.py:272-290);
//                           log-weight (filtering.py:293);
//                           block max and online-rescaled moment partials
//                           for the summaries (filtering.py:344-355); the
//                           last CTA reduces them (max is NaN-propagating,
//                           AllWeightsZeroError(step) if not finite).
//  K6  materialize_kernel post-resample particle system (store / keep_final).
#pragma once
#include "cdf.cuh"
#include "philox.cuh"
#include "special.cuh"

namespace pf {

constexpr double LOG_TWO_PI = 1.8378770664093453;  // math.log(2*math.pi), models.py:20
#ifndef PF_STEP_SB
#define PF_STEP_SB 2
#endif
#ifndef PF_FD_THREADS
#define PF_FD_THREADS 768
#endif
#ifndef PF_FD_SB
#define PF_FD_SB 1
#endif
constexpr int STEP_SB = PF_STEP_SB;  // slots per thread per pipeline stage (double buffered)
// STEP_SB = 1 is supported again.  The round-1 SB = 1 build failed memcheck
// ("out-of-range shared or local address" at the STS of the staged tau2
// draw): its SASS formed that store's address from R1, the stack-pointer
// register (profiles/r02_memcheck_summary.txt), i.e. the generic-pointer
// store of a draw into its shared stage slot was mis-addressed.  Draws now
// stay in registers (no generic stores into the stage at all); memcheck and
// racecheck are clean for SB = 1 and SB = 2.  SB = 2 stays the default
// (measured faster).
constexpr int FD_THREADS = PF_FD_THREADS;  // CTA width of the fused-draws step kernel
// The fused-draws kernel runs 768 threads with one slot per thread per stage
// (80 registers, 24 warps per SM) -- measured faster than 512 x 2 (122
// registers, 16 warps), 640 x 1, 896 x 1 and 1024 x 1 (the last two spill);
// the 256-thread kernel (draws kernel beside it) keeps two slots.
constexpr int FD_SB = PF_FD_SB;
template <bool FD>
constexpr int step_sb() { return FD ? FD_SB : STEP_SB; }

// Order-preserving 32-bit image of a double (float32 rounded down, sign
// folded): the quantile keys of quantile.cuh.
PF_D uint32_t key_rd_(double v) {
  const uint32_t b = __float_as_uint(__double2float_rd(v));
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Carried per-slot state.  sigma2 is not carried: it is redrawn before it
// is used (filtering.py:280) and recomputed from the record when a
// post-resample system is materialised.  a_sigma / a_tau are per-step
// scalars (every particle adds 1/2 per step, filtering.py:279,285).
struct alignas(32) Rec {
  double x, tau2, bs, bt;
};

enum : int { M_LS = 1, M_LT = 2, M_SINGLE = 4 };

struct GammaSrc {
  const double* table;  // GT_TABLE_DOUBLES for this step's shape (method 0)
  double shape;         // method 1
  int method;
};

PF_D double gamma_draw(const GammaSrc& g, double u) {
  if (g.method == 0) return gt_eval(g.table, u);
  return gamma_quantile_accurate(g.shape, u);
}

// Per-step tables staged in shared memory by the step kernel; indexing the
// extern symbol directly keeps the loads LDS (not generic LD).
extern __shared__ double pf_gtab[];

// Staged tables are coefficient-major ([k][seg]): the lanes of a warp read
// coefficient k of their own (random) segments, which then spread over all
// 16 double-wide bank pairs instead of the 4 a 12-double segment stride
// leaves (4x fewer shared-memory wavefronts).  Same coefficients and Horner
// order as gt_eval on the global [seg][k] table, so the values are identical.
PF_D double gamma_table_slot(int slot, double u) {
  double t;
  const int seg = gt_segment_bf(u, &t);
  const double* c = pf_gtab + slot * GT_TABLE_DOUBLES + seg;
  double r = c[GT_DEG * GT_NSEG];
#pragma unroll
  for (int k = GT_DEG - 1; k >= 0; --k) r = fma(r, t, c[k * GT_NSEG]);
  return r;
}

PF_D double gamma_draw_slot(const GammaSrc& g, int slot, double u) {
  if (slot < 0) return gamma_draw(g, u);
  double t;
  const int seg = gt_segment_bf(u, &t);
  const double* c = pf_gtab + slot * GT_TABLE_DOUBLES + seg;
  double r = c[GT_DEG * GT_NSEG];
#pragma unroll
  for (int k = GT_DEG - 1; k >= 0; --k) r = fma(r, t, c[k * GT_NSEG]);
  return r;
}

// -------------------------------------------------------- table build ---
__global__ void __launch_bounds__(32)
gamma_table_build_kernel(const double* __restrict__ shapes, double* __restrict__ tables) {
  const int seg = blockIdx.x;
  const double a = shapes[blockIdx.y];
  double* out = tables + (size_t)blockIdx.y * GT_TABLE_DOUBLES + seg * GT_NC;
  __shared__ double f[GT_NC];
  const int j = threadIdx.x;
  const double PI = 3.14159265358979323846;
  if (j < GT_NC) {
    const double tj = cos(PI * (j + 0.5) / GT_NC);
    double u, v;
    bool up;
    gt_point(seg, tj, &u, &v, &up);
    f[j] = gamma_quantile_pv(a, u, v, !up);
  }
  __syncthreads();
  if (j == 0) cheb_to_mono(f, out);
}

// --------------------------------------------------------------- init ---
struct InitArgs {
  int64_t n;
  uint64_t seed;
  double x0_mean, sqrt_x0_var;
  double bs0, bt0;          // prior scales
  double sigma2_fixed, tau2_fixed;
  GammaSrc gs, gt;
  const double* feed_z;     // row 0 of the oracle feed (or null)
  const double* feed_gs;
  const double* feed_gt;
  Rec* rec;
  double* s2_init;          // optional: sigma2 draws (T == 0 keep_final)
  int64_t gbase;            // global index of this shard's first slot
  const uint64_t* seedp;    // batched replications: seedp[r] is replication r's seed
};

template <int MODE>
__global__ void __launch_bounds__(256) init_kernel(InitArgs a) {
  constexpr bool LS = MODE & M_LS, LT = MODE & M_LT, SINGLE = MODE & M_SINGLE;
  // batched replications (gridDim.z = R): replication blockIdx.z's slots
  const int64_t rz = blockIdx.z;
  Rec* rec = a.rec + rz * a.n;
  const uint64_t seed = a.seedp ? a.seedp[rz] : a.seed;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const Philox4 P = philox_block(seed, (uint64_t)(a.gbase + j), 0);
    const double z = a.feed_z ? a.feed_z[j] : ndtri(unit_open(P.w[0]));
    double x0 = a.x0_mean + a.sqrt_x0_var * z;
    if (SINGLE) x0 = (double)(float)x0;
    double s2 = a.sigma2_fixed, t2 = a.tau2_fixed;
    if (LS) s2 = a.bs0 / (a.feed_gs ? a.feed_gs[j] : gamma_draw(a.gs, unit_open(P.w[1])));
    if (LT) t2 = a.bt0 / (a.feed_gt ? a.feed_gt[j] : gamma_draw(a.gt, unit_open(P.w[2])));
    Rec r;
    r.x = x0;
    r.tau2 = t2;
    r.bs = a.bs0;
    r.bt = a.bt0;
    rec[j] = r;
    if (a.s2_init) a.s2_init[j] = s2;
  }
}

// ---------------------------------------------------------------- step ---
struct Partial {
  double m, s0, sx, s2x, s1s, s2s, s1t, s2t, s2w, bad;  // s2w: sum of squared weights (ESS)
  double se;  // K7 (spacings): the shard's sum of slot exponentials (set after its scan)
};

struct Scalars {
  double M;        // max log-weight of the current step
  double W;        // total weight (moment normalizer)
  double cs, ct;   // moment shifts (previous step means)
  double cx;
  unsigned int counter;
  unsigned int pad;
};

struct StepOut {   // device arrays indexed by t-1
  double* fmean;
  double* s_mean;
  double* s_sd;
  double* t_mean;
  double* t_sd;
  double* ess;     // optional: (sum w)^2 / sum w^2 (extension; the reference has no ESS)
};

struct DrawArgs {
  int64_t n;
  int64_t t;
  uint64_t seed;
  GammaSrc gs, gt;
  const double* ntab;    // normal-quantile table (null: Cephes ndtri)
  double* z;
  double* g_s;
  double* g_t;
  uint64_t* u3;
  const int64_t* fail;
  int64_t gbase;         // global index of this shard's first slot (stream id offset)
  const uint64_t* seedp; // non-null: the seed is read from device memory (graph replays)
};

PF_D uint64_t seed_of(uint64_t seed, const uint64_t* seedp) { return seedp ? *seedp : seed; }

// Batched replications: one launch runs R independent filters of n slots
// (gridDim.z = R, replication r = blockIdx.z).  Replication r owns slots
// [r n, (r+1) n) of every per-slot array, row r of the [R][T] outputs and
// entry r of the per-replication state (seed, scalars, status, max by
// parity [R][2], moment partials [R][grid.x]).  Offsets are applied once at
// kernel entry; gridDim.z = 1 is the single run, unchanged.
struct RepStride {
  int64_t out;       // output row length (T)
  int64_t qsh_bytes; // bytes between replications' QShared pairs
};

template <typename TQ>
struct StepArgs {
  int64_t n;
  int64_t t;             // 1-based step
  uint64_t seed;
  double y;
  double sigma2_fixed, tau2_fixed, sqrt_tau2_fixed, log_term_fixed;
  const Rec* rec_in;
  Rec* rec_out;
  double* lw;            // log-weights (or fed weights when feed_w)
  double* Mout;          // max log-weight of this step (per-parity slot)
  const uint64_t* u3;    // resampling words of step t-1 (draws_kernel)
  Lookup<TQ> lk;         // resampling table of step t-1 (t > 1)
  int64_t* idx_out;      // optional 1-based ancestors of step t-1
  const double* z;       // step t normals / gamma draws: draws_kernel output,
  const double* g_s;     // or the oracle feed rows
  const double* g_t;
  const double* feed_w;
  uint32_t* kx;          // optional order-preserving 32-bit keys for the
  uint32_t* ks;          // weighted quantiles (quantile.cuh)
  uint32_t* kt;
  double* qmom;          // optional: mean[3], sd[3] of x, sigma2, tau2
  Partial* partials;
  Scalars* sc;
  StepOut out;
  int64_t* fail;
  Partial* xrec;         // sharded run: shard partials [G] (null: single run)
  int shard;
  DrawArgs dr;           // FD: this step's draws are computed here (tables, seed, u3 out)
  ShardLookup<TQ> slk;   // sharded run (slk.G > 0): cross-shard lookup
  ShardRank srk;         // sharded run: per-shard rank tables (srk.on)
  const double* spS;     // K7 (spacings): prefix sums of step t-1's slot exponentials -- the
                         // resampling words are formed from them here instead of read from u3
  const double* sp_tot;  // sharded K7: every shard's exponential total of step t-1 (slk.G of them)
  const double* yp;      // non-null: the observation is yp[t-1] (device memory; graph replays)
  int dbg_identity;      // diagnostics only (PF_DEBUG_IDENTITY_ANC): skip the lookup, ancestor = slot
  double ref_slack;      // moment-reference slack (64; 0 = rescale at every new max)
  const Rec* recs[PF_MAX_SHARDS];  // sharded run: every shard's records of step t-1
  RepStride rp;          // batched replications (gridDim.z > 1)
};

PF_D double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
PF_D double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// exp(x) for the moment weights (x = lw - m <= ref_slack): k = rint(64 x /
// ln 2) via the 1.5 2^52 shifter, r = x - k ln2/64 (two-part constant),
// e^r by a degree-5 Taylor polynomial (|r| <= ln2/128: truncation 4e-17),
// times 2^(k/64) from a 64-entry shared table and 2^floor(k/64) by exponent
// add.  Relative error < 3e-16; x < -700 gives 0 (e^-700 of the step's
// largest weight is far below the moments' 1e-10 tolerance).
// ~16 instructions against ~45 for exp(); the CDF's weights keep exp()
// (they must round like the reference's).
constexpr int EXP_TAB = 64;
PF_D double exp_moment(double x, const double* tab) {
  const double SH = 6755399441055744.0;                  // 1.5 * 2^52
  const double INV = 92.33248261689366;               // 64 / ln 2
  const double C_HI = 0.010830424696249145;             // ln2/64 rounded
  const double C_LO = 3.623510646634843e-19;            // ln2/64 - C_HI
  const double kd = fma(x, INV, SH);
  const int k = (int)__double2loint(kd);
  const double kf = kd - SH;
  double r = fma(-kf, C_HI, x);
  r = fma(-kf, C_LO, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  double v = p * tab[k & (EXP_TAB - 1)];
  const int hi = __double2hiint(v) + (int)((unsigned)(k >> 6) << 20);
  v = __hiloint2double(hi, __double2loint(v));
  return x < -700.0 ? 0.0 : v;
}

// Combine `count` partials (each rescaled to its own max) in a fixed order:
// M = max (NaN when any partial saw a NaN / +inf log-weight), S = sums
// rescaled to M.  Called by all threads of one CTA; results in thread 0.
PF_D void reduce_partials(const Partial* p, int count, double (*red)[10], double& M_out, double& bad_out,
                          double (&S)[8]) {
  __shared__ double mfin;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double M = -INFINITY, badsum = 0.0;
  for (int b = threadIdx.x; b < count; b += blockDim.x) {
    M = fmax(M, __ldcg(&p[b].m));
    badsum += __ldcg(&p[b].bad);
  }
  M = warp_max(M);
  badsum = warp_sum(badsum);
  __syncthreads();
  if (lane == 0) { red[warp][0] = M; red[warp][1] = badsum; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = red[0][0], bb = red[0][1];
    for (int w = 1; w < nw; ++w) { mm = fmax(mm, red[w][0]); bb += red[w][1]; }
    mfin = (bb > 0.0) ? NAN : mm;
    bad_out = bb;
  }
  __syncthreads();
  M = mfin;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = threadIdx.x; b < count; b += blockDim.x) {
    const double mb2 = __ldcg(&p[b].m);
    const double f = (mb2 == -INFINITY) ? 0.0 : exp(mb2 - M);
    acc[0] += f * __ldcg(&p[b].s0);
    acc[1] += f * __ldcg(&p[b].sx);
    acc[2] += f * __ldcg(&p[b].s2x);
    acc[3] += f * __ldcg(&p[b].s1s);
    acc[4] += f * __ldcg(&p[b].s2s);
    acc[5] += f * __ldcg(&p[b].s1t);
    acc[6] += f * __ldcg(&p[b].s2t);
    acc[7] += (f * f) * __ldcg(&p[b].s2w);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double sv = warp_sum(acc[k]);
    if (lane == 0) red[warp][k] = sv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 8; ++k) S[k] = 0.0;
    for (int w = 0; w < nw; ++w)
      for (int k = 0; k < 8; ++k) S[k] += red[w][k];
    M_out = M;
  }
}

// Step t's summaries from the combined sums (filtering.py:344-355), the
// moment shifts of the next step, the max log-weight and the degeneracy
// check (filtering.py:294-296).  One thread.
template <bool LS, bool LT>
PF_D void finalize_step(int64_t t, double M, double bsum, const double (&S)[8], bool feedw, double cs,
                        double ct, double cx, const StepOut& out, double* qmom, Scalars* sc, double* Mout,
                        int64_t* fail) {
  (void)bsum;
  const int64_t i = t - 1;
  const double W = S[0];
  const double fm = S[1] / W;
  out.fmean[i] = fm;
  if (out.ess) out.ess[i] = (W * W) / S[7];
  {
    const double d = fm - cx;
    const double var = S[2] / W - d * d;
    if (qmom) { qmom[0] = fm; qmom[3] = sqrt(fmax(var, 0.0)); }
    sc->cx = fm;
  }
  if (LS) {
    const double d = S[3] / W;
    const double var = S[4] / W - d * d;
    out.s_mean[i] = cs + d;
    out.s_sd[i] = sqrt(fmax(var, 0.0));
    sc->cs = cs + d;
    if (qmom) { qmom[1] = cs + d; qmom[4] = out.s_sd[i]; }
  }
  if (LT) {
    const double d = S[5] / W;
    const double var = S[6] / W - d * d;
    out.t_mean[i] = ct + d;
    out.t_sd[i] = sqrt(fmax(var, 0.0));
    sc->ct = ct + d;
    if (qmom) { qmom[2] = ct + d; qmom[5] = out.t_sd[i]; }
  }
  sc->M = feedw ? 0.0 : M;
  *Mout = feedw ? 0.0 : M;
  sc->W = W;
  sc->counter = 0;
  if (!feedw && !(M > -INFINITY && M < INFINITY))
    atomicCAS((unsigned long long*)fail, 0ull, (unsigned long long)t);
}

// ---------------------------------------------------------------- draws ---
// K1a: the record-independent half of step t -- Philox block t of every
// stream, the normal draw and the two inverse-gamma draws (filtering.py:
// 273,280,286; counter layout rng.py:221-224) -- compute-bound work that
// runs on its own stream, concurrently with the memory-bound CDF kernels of
// step t-1.  Writes z, g_sigma, g_tau and the resampling word (slot 3).

PF_D double nt_eval_slot(int off, double u) {
  double t, sc;
  const int seg = nt_segment_bf(u, &t, &sc);
  const double* c = pf_gtab + off + seg;
  double r = c[GT_DEG * NT_NSEG];
#pragma unroll
  for (int k = GT_DEG - 1; k >= 0; --k) r = fma(r, t, c[k * NT_NSEG]);
  return sc * r;
}

// Stage this step's tables in shared memory: gamma table(s) (one copy when
// sigma2 and tau2 share the shape schedule), then the normal table.
template <bool LS, bool LT>
PF_D int stage_tables(const GammaSrc& gs, const GammaSrc& gt, const double* ntab, int& slot_s, int& slot_t,
                      int& noff) {
  slot_s = slot_t = -1;
  const double* srcs[3] = {LS && gs.method == 0 ? gs.table : nullptr,
                           LT && gt.method == 0 && !(LS && gt.table == gs.table) ? gt.table : nullptr, ntab};
  const int len[3] = {GT_TABLE_DOUBLES, GT_TABLE_DOUBLES, NT_TABLE_DOUBLES};
  const int nseg[3] = {GT_NSEG, GT_NSEG, NT_NSEG};
  int off = 0;
  for (int k = 0; k < 3; ++k) {
    if (!srcs[k]) continue;
    // global [seg][coef] -> shared [coef][seg]
    for (int i = threadIdx.x; i < len[k]; i += blockDim.x) {
      const int sg = i / GT_NC, cf = i - sg * GT_NC;
      pf_gtab[off + cf * nseg[k] + sg] = __ldg(srcs[k] + i);
    }
    if (k == 0) slot_s = off / GT_TABLE_DOUBLES;
    else if (k == 1) slot_t = off / GT_TABLE_DOUBLES;
    else noff = off;
    off += len[k];
  }
  if (LS && LT && gs.method == 0 && gt.table == gs.table) slot_t = slot_s;
  __syncthreads();
  return off;
}

template <int MODE>
__global__ void __launch_bounds__(256) draws_kernel(DrawArgs a) {
  constexpr bool LS = MODE & M_LS, LT = MODE & M_LT;
  {
    const int64_t r = blockIdx.z, o = r * a.n;
    a.z += o; a.g_s += o; a.g_t += o; a.u3 += o;
    a.fail += r;
    if (a.seedp) a.seedp += r;
  }
  if (*a.fail) return;
  int slot_s, slot_t, noff = -1;
  stage_tables<LS, LT>(a.gs, a.gt, a.ntab, slot_s, slot_t, noff);
  const uint64_t seed = seed_of(a.seed, a.seedp);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const Philox4 P = philox_block(seed, (uint64_t)(a.gbase + j), (uint64_t)a.t);
    a.u3[j] = P.w[3];
    const double u0 = unit_open(P.w[0]);
    a.z[j] = noff >= 0 ? nt_eval_slot(noff, u0) : ndtri(u0);
    if (LS) a.g_s[j] = gamma_draw_slot(a.gs, slot_s, unit_open(P.w[1]));
    if (LT) a.g_t[j] = gamma_draw_slot(a.gt, slot_t, unit_open(P.w[2]));
  }
}

// ---------------------------------------------------------------- K1b ---
PF_D void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
PF_D void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src));
}

// FD: compute the step's draws (Philox block t, ndtri and gamma tables
// staged in shared memory) for each batch while its record gathers are in
// flight -- the issue slots the latency-bound gather pipeline leaves idle --
// instead of a separate compute-bound draws kernel and a round trip of the
// draws through HBM.
template <int MODE, typename TQ, bool FD = false, bool BATCH = false>
__global__ void __launch_bounds__(FD ? FD_THREADS : 256, 1) step_kernel(StepArgs<TQ> a) {
  constexpr bool LS = MODE & M_LS, LT = MODE & M_LT, SINGLE = MODE & M_SINGLE;
  constexpr int SB = step_sb<FD>();  // slots per thread per pipeline stage
  // batched replications (gridDim.z = R): replication blockIdx.z's slice of
  // every array (locals: the kernel parameters themselves stay read-only)
  // (BATCH = false: the single-run instantiation, rz = ro = 0 at compile time)
  const int64_t rz = BATCH ? (int64_t)blockIdx.z : 0, ro = rz * a.n;
  // (per-slot arrays are indexed at ro + j below; ro = 0 for a single run)
  Lookup<TQ> lk_b = a.lk;
  if (BATCH) {
    lk_b.q += ro;
    lk_b.cut += ro;
  }
  const Lookup<TQ>& lk_ = BATCH ? lk_b : a.lk;  // single run: the parameter itself
  Partial* const partials_ = a.partials + rz * gridDim.x;
  Scalars* const sc_ = a.sc + rz;
  int64_t* const fail_ = a.fail + rz;
  const uint64_t* const dseedp_ = (BATCH && a.dr.seedp) ? a.dr.seedp + rz : a.dr.seedp;
  // the step's tables are constant over the run: stage them while the
  // previous kernel (group build / K4) drains, then wait for its outputs
  int slot_s = -1, slot_t = -1, noff = -1, tab_doubles = 0;
  __shared__ double s_exp[EXP_TAB];  // 2^(i/64) for exp_moment
  if (threadIdx.x < EXP_TAB) s_exp[threadIdx.x] = exp2((double)threadIdx.x / EXP_TAB);
  if (FD) tab_doubles = stage_tables<LS, LT>(a.dr.gs, a.dr.gt, a.dr.ntab, slot_s, slot_t, noff);
  else __syncthreads();
  pdl_wait();
  if (*fail_) return;
  const bool feedw = a.feed_w != nullptr;
  const double cs = sc_->cs, ct = sc_->ct, cx = sc_->cx;
  const double yobs = a.yp ? a.yp[a.t - 1] : a.y;
  const uint64_t dseed = seed_of(a.dr.seed, dseedp_);
  // m: reference of this thread's moment sums (moved, with a rescale, only
  // when a log-weight exceeds it by more than ref_slack = 64 -- e <= e^64
  // keeps the fp64 sums far from overflow); mx: the true running max, the
  // step's M.
  double m = feedw ? 0.0 : -INFINITY;
  double mx = m;
  double s0 = 0, sx = 0, s2x = 0, s1s = 0, s2s = 0, s1t = 0, s2t = 0, s2w = 0;
  bool bad = false;

  // Software pipeline over batches of SB x blockDim slots (batches are
  // dealt to CTAs round robin).  Iteration i: resolve the ancestors of batch
  // i+1 (cut-point lookups against L2-resident tables) and start, with
  // cp.async into the other half of a double buffer, their 32-byte record
  // gathers (the one random DRAM access per slot) and the coalesced loads
  // of their draws; then wait for batch i (issued one iteration earlier) and
  // run its arithmetic while batch i+1's reads are in flight.  Each thread
  // reads back only what it staged itself.
  const int nth = blockDim.x;
  const int64_t batch = (int64_t)SB * nth;
  const int64_t nbatches = (a.n + batch - 1) / batch;
  char* smem = reinterpret_cast<char*>(pf_gtab + ((tab_doubles + 3) & ~3));
  const size_t buf_bytes = (size_t)SB * nth * (sizeof(Rec) + 3 * sizeof(double));
  auto rec_at = [&](int buf, int b) {
    return reinterpret_cast<Rec*>(smem + buf * buf_bytes) + b * nth + threadIdx.x;
  };
  auto val_at = [&](int buf, int k, int b) {
    return reinterpret_cast<double*>(smem + buf * buf_bytes + (size_t)SB * nth * sizeof(Rec)) +
           (k * SB + b) * nth + threadIdx.x;
  };
  // K7: the ordered uniform of slot j is S_j / S_(N+1) (spacings_words_kernel
  // forms the same words for the store / final resample)
  double sp_inv = 0.0, sp_off = 0.0;
  if (a.spS && a.t > 1) {
    double tot = 0.0;
    if (a.sp_tot) {  // sharded: the shard's offset and the grand total, in shard order
      for (int h = 0; h < a.slk.G; ++h) {
        const double th = __ldcg(a.sp_tot + h);
        if (h < a.shard) sp_off += th;
        tot += th;
      }
    } else {
      tot += __ldcg(a.spS + a.n - 1);
    }
    sp_inv = 1.0 / (tot + spacings_aux_exp(seed_of(a.seed, dseedp_), a.t - 1));
  }
  // resampling words are loaded one pipeline stage ahead of their lookups
  auto load_w3 = [&](int64_t bi, uint64_t (&w3)[SB]) {
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const int64_t j = bi * batch + b * (int64_t)nth + threadIdx.x;
      const bool live = a.t > 1 && bi < nbatches && j < a.n;
      w3[b] = !live ? 0ull : a.spS ? spacings_word(sp_off + __ldcs(a.spS + j), sp_inv) : __ldcs(a.u3 + (ro + j));
    }
  };
  auto issue = [&](int64_t bi, int buf, const uint64_t (&w3)[SB]) {
    int64_t jj[SB], anc[SB];
    bool ok[SB];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      jj[b] = bi * batch + b * (int64_t)nth + threadIdx.x;
      ok[b] = jj[b] < a.n;
      anc[b] = jj[b];
    }
    if (a.t > 1 && !a.dbg_identity) {
      if (a.slk.G > 0) {
#pragma unroll
        for (int b = 0; b < SB; ++b)
          if (ok[b]) anc[b] = a.srk.on ? sharded_lookup_rank<TQ>(a.slk, a.srk, w3[b]) : sharded_lookup<TQ>(a.slk, w3[b]);
      } else if (lk_.anc) {  // baseline resamplers: ancestors precomputed
#pragma unroll
        for (int b = 0; b < SB; ++b)
          if (ok[b]) anc[b] = lk_.anc[jj[b]];
      } else {
        ancestors_of<TQ, SB>(lk_, w3, ok, anc);
      }
      if (a.idx_out) {
#pragma unroll
        for (int b = 0; b < SB; ++b)
          if (ok[b]) a.idx_out[jj[b]] = anc[b] + 1;
      }
    }
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      if (!ok[b]) continue;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(rec_at(buf, b));
      // ancestors are global indices in a sharded run (identity, local, at t = 1)
      const Rec* rp = (a.slk.G > 0 && a.t > 1)
          ? a.recs[anc[b] >> a.slk.lg] + (anc[b] & (((int64_t)1 << a.slk.lg) - 1))
          : a.rec_in + (ro + anc[b]);
      const char* src = reinterpret_cast<const char*>(rp);
      cp_async16(dst, src);
      cp_async16(dst + 16, src + 16);
      // precomputed draws (draws kernel) or the oracle feed
      if (a.z) cp_async8((uint32_t)__cvta_generic_to_shared(val_at(buf, 0, b)), a.z + (ro + jj[b]));
      if (LS && a.g_s) cp_async8((uint32_t)__cvta_generic_to_shared(val_at(buf, 1, b)), a.g_s + (ro + jj[b]));
      if (LT && a.g_t) cp_async8((uint32_t)__cvta_generic_to_shared(val_at(buf, 2, b)), a.g_t + (ro + jj[b]));
    }
    asm volatile("cp.async.commit_group;");
  };
  // One slot's arithmetic (filtering.py:272-298,345): propagate, sufficient
  // statistics, log-weight, quantile keys, moment partials.
  auto slot_math = [&](int64_t j, const Rec& r, double z, double gsd, double gtd) {
    const double sq = LT ? sqrt(r.tau2) : a.sqrt_tau2_fixed;
    const double step = sq * z;
    double xn = r.x + step;
    if (SINGLE) xn = (double)(float)xn;
    const double resid = yobs - xn;
    const double h = (0.5 * resid) * resid;
    Rec o;
    o.x = xn;
    o.bs = r.bs;
    o.bt = r.bt;
    double s2 = a.sigma2_fixed, t2 = a.tau2_fixed;
    if (LS) {
      o.bs = r.bs + h;
      s2 = o.bs / gsd;
    }
    if (LT) {
      o.bt = r.bt + (0.5 * step) * step;
      t2 = o.bt / gtd;
    }
    o.tau2 = t2;
    a.rec_out[ro + j] = o;
    // ---- log-weight (filtering.py:293)
    double lw;
    if (LS)
      lw = (-0.5) * (LOG_TWO_PI + log(s2)) - h / s2;
    else
      lw = a.log_term_fixed - h / s2;
    double e;
    if (feedw) {
      e = a.feed_w[j];
      a.lw[ro + j] = e;
    } else {
      a.lw[ro + j] = lw;
      if (!(lw == lw) || lw == INFINITY) bad = true;
      if (lw > mx) mx = lw;
      if (lw > m + a.ref_slack) {
        const double sc = exp(m - lw);
        s0 *= sc; sx *= sc; s2x *= sc; s1s *= sc; s2s *= sc; s1t *= sc; s2t *= sc; s2w *= sc * sc;
        m = lw;
        e = 1.0;
      } else {
        e = lw > -INFINITY ? exp_moment(lw - m, s_exp) : 0.0;
      }
    }
    if (a.kx) a.kx[ro + j] = key_rd_(xn);
    if (a.ks) a.ks[ro + j] = key_rd_(s2);
    if (a.kt) a.kt[ro + j] = key_rd_(t2);
    s0 += e;
    s2w = fma(e, e, s2w);
    sx = fma(e, xn, sx);
    const double dxx = xn - cx;
    s2x = fma(e * dxx, dxx, s2x);
    const double ds = s2 - cs, dt = t2 - ct;
    const double eds = e * ds, edt = e * dt;
    s1s += eds;
    s2s = fma(eds, ds, s2s);
    s1t += edt;
    s2t = fma(edt, dt, s2t);
  };
  int cur = 0;
  int64_t bi = blockIdx.x;
  uint64_t w3n[SB];
  load_w3(bi, w3n);
  if (bi < nbatches) issue(bi, 0, w3n);
  load_w3(bi + gridDim.x, w3n);
  for (; bi < nbatches; bi += gridDim.x) {
    if (bi + gridDim.x < nbatches) {
      issue(bi + gridDim.x, cur ^ 1, w3n);
      load_w3(bi + 2 * (int64_t)gridDim.x, w3n);
    } else {
      asm volatile("cp.async.commit_group;");
    }
    // FD: this batch's draws (Philox block t, filtering.py:273,280,286) in
    // registers, computed while its record gathers (issued one iteration
    // earlier) are still in flight; the slots' Philox networks and the three
    // table polynomials are independent chains the scheduler interleaves.
    // The resampling word goes to memory for the next step's lookups.
    double dz[SB], dgs[SB], dgt[SB];
    if (FD) {
#pragma unroll
      for (int b = 0; b < SB; ++b) {
        const int64_t j = bi * batch + b * (int64_t)nth + threadIdx.x;
        const Philox4 P = philox_block(dseed, (uint64_t)(a.dr.gbase + j), (uint64_t)a.t);
        if (j < a.n) a.dr.u3[ro + j] = P.w[3];
        // tables only (FD runs with gamma_method 0): no call into the
        // accurate solvers, which would cost the kernel a stack frame
        dz[b] = nt_eval_slot(noff, unit_open(P.w[0]));
        dgs[b] = LS ? gamma_table_slot(slot_s, unit_open(P.w[1])) : 1.0;
        dgt[b] = LT ? gamma_table_slot(slot_t, unit_open(P.w[2])) : 1.0;
      }
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const int64_t j = bi * batch + b * (int64_t)nth + threadIdx.x;
      if (j >= a.n) continue;
      // drawn here (FD) unless an oracle feed was staged; precomputed draws
      // (draws kernel) are staged too
      const double z = (FD && !a.z) ? dz[b] : *val_at(cur, 0, b);
      const double gsd = !LS ? 1.0 : (FD && !a.g_s) ? dgs[b] : *val_at(cur, 1, b);
      const double gtd = !LT ? 1.0 : (FD && !a.g_t) ? dgt[b] : *val_at(cur, 2, b);
      slot_math(j, *rec_at(cur, b), z, gsd, gtd);
    }
    cur ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  pdl_launch_dependents();  // only the CTA reductions remain

  // ---- CTA reduction with rescaling to the CTA max
  __shared__ double red[32][10];
  __shared__ double mblk;
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double wm = warp_max(mx);
  if (lane == 0) red[warp][0] = wm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = red[0][0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mm = fmax(mm, red[w][0]);
    mblk = mm;
  }
  __syncthreads();
  const double mb = mblk;
  const double scl = (m == -INFINITY) ? 0.0 : exp(m - mb);
  double v[9] = {s0 * scl, sx * scl, s2x * scl, s1s * scl, s2s * scl, s1t * scl, s2t * scl,
                 s2w * (scl * scl), bad ? 1.0 : 0.0};
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) red[warp][k] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      for (int k = 0; k < 9; ++k) acc[k] += red[w][k];
    Partial p;
    p.m = mb;
    p.s0 = acc[0]; p.sx = acc[1]; p.s2x = acc[2]; p.s1s = acc[3]; p.s2s = acc[4]; p.s1t = acc[5];
    p.s2t = acc[6];
    p.s2w = acc[7];
    p.bad = acc[8];
    partials_[blockIdx.x] = p;
    __threadfence();
    const unsigned int ticket = atomicAdd(&sc_->counter, 1u);
    last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;

  // ---- last CTA: combine the partials (fixed order -> deterministic)
  __threadfence();
  double M, bsum, S[8];
  reduce_partials(partials_, (int)gridDim.x, red, M, bsum, S);
  if (threadIdx.x != 0) return;
  if (a.xrec) {
    // sharded run: this shard's partial goes to the exchange array; the
    // combine kernel finalises the step from all shards' partials
    Partial p;
    p.m = M;
    p.s0 = S[0]; p.sx = S[1]; p.s2x = S[2]; p.s1s = S[3]; p.s2s = S[4]; p.s1t = S[5]; p.s2t = S[6];
    p.s2w = S[7];
    p.bad = bsum;
    p.se = 0.0;
    a.xrec[a.shard] = p;
    __threadfence_system();
    sc_->counter = 0;
    return;
  }
  StepOut o = a.out;
  double* qmom = a.qmom;
  if (rz) {
    const int64_t ro_ = rz * a.rp.out;
    o.fmean += ro_;
    if (o.s_mean) { o.s_mean += ro_; o.s_sd += ro_; }
    if (o.t_mean) { o.t_mean += ro_; o.t_sd += ro_; }
    if (o.ess) o.ess += ro_;
    if (qmom) qmom = reinterpret_cast<double*>(reinterpret_cast<char*>(qmom) + rz * a.rp.qsh_bytes);
  }
  finalize_step<LS, LT>(a.t, M, bsum, S, feedw, cs, ct, cx, o, qmom, sc_, a.Mout + 2 * rz, fail_);
}

// Sharded run: every shard finalises step t from the G shard partials (the
// same fixed-order combination, so all shards hold identical M / shifts).
template <int MODE>
__global__ void __launch_bounds__(256) combine_kernel(const Partial* __restrict__ xrec, int G, int64_t t,
                                                      int feedw, StepOut out, double* qmom, Scalars* sc,
                                                      double* Mout, int64_t* fail, double* sp_tot = nullptr) {
  constexpr bool LS = MODE & M_LS, LT = MODE & M_LT;
  if (*fail) return;
  // K7: keep every shard's exponential total of step t for step t+1's words
  if (sp_tot && (int)threadIdx.x < G) sp_tot[threadIdx.x] = __ldcg(&xrec[threadIdx.x].se);
  __shared__ double red[8][10];
  const double cs = sc->cs, ct = sc->ct, cx = sc->cx;
  double M, bsum, S[8];
  reduce_partials(xrec, G, red, M, bsum, S);
  if (threadIdx.x != 0) return;
  finalize_step<LS, LT>(t, M, bsum, S, feedw != 0, cs, ct, cx, out, qmom, sc, Mout, fail);
}

// -------------------------------------------------------- materialize ---
template <typename TQ>
struct MatArgs {
  int64_t n;
  int64_t t;               // block index of the draws (0 = init system)
  uint64_t seed;
  int resample;            // 1: ancestors by lookup of u3 against q/cut
  const Rec* rec;
  const uint64_t* u3;
  Lookup<TQ> lk;
  const double* s2_direct; // sigma2 per slot when no resample (init)
  GammaSrc gs;
  const double* feed_gs;   // oracle feed row t (indexed by ancestor)
  int learn_s, learn_t;
  double sigma2_fixed, tau2_fixed, a_s, a_t;
  int64_t* idx;            // outputs (each optional)
  double* x;
  double* s2;
  double* t2;
  double* as;
  double* bs;
  double* at;
  double* bt;
  const int64_t* fail;
};

template <typename TQ>
__global__ void __launch_bounds__(256) materialize_kernel(MatArgs<TQ> a) {
  if (*a.fail) return;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.n;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t anc = j;
    if (a.resample) anc = a.lk.anc ? (int64_t)a.lk.anc[j] : ancestor_of<TQ>(a.lk, a.u3[j]);
    if (a.idx) a.idx[j] = anc + 1;
    const Rec r = a.rec[anc];
    if (a.x) a.x[j] = r.x;
    if (a.s2) {
      double s2 = a.sigma2_fixed;
      if (a.learn_s) {
        if (a.s2_direct) {
          s2 = a.s2_direct[anc];
        } else {
          const Philox4 P = philox_block(a.seed, (uint64_t)anc, (uint64_t)a.t);
          const double g = a.feed_gs ? a.feed_gs[anc] : gamma_draw(a.gs, unit_open(P.w[1]));
          s2 = r.bs / g;
        }
      }
      a.s2[j] = s2;
    }
    if (a.t2) a.t2[j] = a.learn_t ? r.tau2 : a.tau2_fixed;
    if (a.as) a.as[j] = a.learn_s ? a.a_s : 0.0;
    if (a.bs) a.bs[j] = a.learn_s ? r.bs : 0.0;
    if (a.at) a.at[j] = a.learn_t ? a.a_t : 0.0;
    if (a.bt) a.bt[j] = a.learn_t ? r.bt : 0.0;
  }
}

// Sharded run: post-resample system of the last step (keep_final /
// keep_indices row T) with the cross-shard lookup and remote records.
template <typename TQ>
struct GroupMatArgs {
  int64_t ns, gbase, t;
  uint64_t seed;
  const uint64_t* u3;
  ShardLookup<TQ> slk;
  const Rec* recs[PF_MAX_SHARDS];
  GammaSrc gs;
  int learn_s, learn_t;
  double sigma2_fixed, tau2_fixed, a_s, a_t;
  int64_t* idx;
  double *x, *s2, *t2, *as, *bs, *at, *bt;
  const int64_t* fail;
};

template <typename TQ>
__global__ void __launch_bounds__(256) group_materialize_kernel(GroupMatArgs<TQ> a) {
  if (*a.fail) return;
  const int64_t mask = ((int64_t)1 << a.slk.lg) - 1;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.ns;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t anc = sharded_lookup<TQ>(a.slk, a.u3[j]);
    if (a.idx) a.idx[j] = anc + 1;
    const Rec r = a.recs[anc >> a.slk.lg][anc & mask];
    if (a.x) a.x[j] = r.x;
    if (a.s2) {
      double s2 = a.sigma2_fixed;
      if (a.learn_s) {
        const Philox4 P = philox_block(a.seed, (uint64_t)anc, (uint64_t)a.t);
        s2 = r.bs / gamma_draw(a.gs, unit_open(P.w[1]));
      }
      a.s2[j] = s2;
    }
    if (a.t2) a.t2[j] = a.learn_t ? r.tau2 : a.tau2_fixed;
    if (a.as) a.as[j] = a.learn_s ? a.a_s : 0.0;
    if (a.bs) a.bs[j] = a.learn_s ? r.bs : 0.0;
    if (a.at) a.at[j] = a.learn_t ? a.a_t : 0.0;
    if (a.bt) a.bt[j] = a.learn_t ? r.bt : 0.0;
  }
}

}  // namespace pf
