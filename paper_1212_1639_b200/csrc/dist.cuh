// One process per GPU: the particle-sharded run (group.cuh) split into the
// per-step phases a rank executes between its collectives.
//
// Included by engine.cu inside its anonymous namespace.  The Python driver
// (paper_1212_1639_b200/distributed.py) owns the process group and runs per
// step:
//     phase 1  ancestor lookups + step kernel -> this rank's partial record
//     all-gather of the G partial records                 (72 B per rank)
//     phase 2  combine (global max, moments) + K2 -> this rank's subtree total
//     all-gather of the G subtree totals                  (8 B per rank)
//     phase 3  top tree + K4 (cut table, q) + quantile classification
//     barrier
//     phase 4  (rank 0) exact quantile resolve
// The collectives are the only cross-rank ordering: under NCCL they run on
// the engine's stream (no host sync); under gloo the phases synchronise and
// copy the records through host memory.  Data-dependent reads of other
// ranks' memory -- cut tables, q, 32-byte records for resampling, rank 0's
// quantile state for the classification, every rank's records / keys /
// log-weights for rank 0's resolve -- go through CUDA IPC mappings (NVLink
// P2P between GPUs).  Bit-identical to the single-device engine.
#pragma once

struct pf_shard {
  pf_config cfg;  // n = N (all ranks)
  int rank = 0, world = 1;
  int64_t ns = 0;
  int lg = 0;
  pf_engine* e = nullptr;
  // exchange arrays (this rank's device copies, filled by the collectives)
  Partial* xrec = nullptr;  // [world]
  void* xtot = nullptr;     // [world] subtree totals (TQ)
  int32_t* gcut = nullptr;  // full-size cut table, this rank's strata written
  void* gq = nullptr;       // q of this rank's particles
  int64_t* lend = nullptr;  // [PF_MAX_SHARDS]
  // rank tables (N >= 2^21): grp over the global stratum groups, fq / f32
  // over this rank's particles
  bool rank_on = false;
  bool resolve_pending = false;  // rank 0: a resolve on the side stream not yet joined
  Grp* sgrp = nullptr;
  uint8_t* sfq = nullptr;
  uint32_t* sf32 = nullptr;
  std::vector<const Grp*> p_grp;
  std::vector<const uint8_t*> p_fq;
  std::vector<const uint32_t*> p_f32;
  // peers' buffers (IPC-mapped; own entries point at local memory)
  std::vector<const int32_t*> p_cut;
  std::vector<const void*> p_q;
  std::vector<const Rec*> p_rec[2];
  std::vector<const uint32_t*> p_keys;
  std::vector<const double*> p_lw;
  std::vector<const double*> p_mbuf;
  // rank 0's quantile state (mapped on every rank)
  QTarget* q_tg = nullptr;
  QShared* q_sh = nullptr;
  QCand* q_cand = nullptr;
  double* q_part = nullptr;
  unsigned long long* q_hist = nullptr;
  unsigned long long* q_fhist = nullptr;
  unsigned int* q_unres = nullptr;
  std::vector<void*> opened;  // IPC mappings to close
  // run state
  std::vector<double> y_host;
  int64_t T = 0;
  int cur = 0;
  int ntg = 0;
  bool want_fq = false;
  uint32_t qcap = 0;
  int cls_grid = 0;
  int qm = 0;
  bool fused = false;  // draws computed inside the step kernel (FD)
  pf_outputs* out = nullptr;
};

namespace {

// Exported buffers, in handle order.
enum { XH_REC0, XH_REC1, XH_CUT, XH_Q, XH_KEYS, XH_LW, XH_MBUF, XH_GRP, XH_FQ, XH_F32, XH_QTG, XH_QSH, XH_QCAND,
       XH_QPART, XH_QHIST, XH_QFHIST, XH_QUNRES, XH_COUNT };

template <int MODE, typename TQ>
struct ShardOps {
  static constexpr bool LS = MODE & M_LS, LT = MODE & M_LT;
  static constexpr int SINGLE = (MODE & M_SINGLE) ? 1 : 0;

  static int begin(pf_shard* s, const double* y, int64_t T, pf_outputs* out) {
    pf_engine* e = s->e;
    const pf_config& c = s->cfg;
    const int64_t ns = s->ns, N = c.n;
    int rc;
    s->y_host.assign(y, y + T);
    s->T = T;
    s->resolve_pending = false;
    s->cur = 0;
    s->out = out;
    const size_t TT = (size_t)(T > 0 ? T : 1);
    if ((rc = build_tables(e, T)) != PF_OK) return rc;
    CK(e->o_fm.ensure(TT));
    CK(e->o_ess.ensure(TT));
    if (LS) { CK(e->o_sm.ensure(TT)); CK(e->o_ssd.ensure(TT)); CK(e->o_sq.ensure(TT * 5)); }
    if (LT) { CK(e->o_tm.ensure(TT)); CK(e->o_tsd.ensure(TT)); CK(e->o_tq.ensure(TT * 5)); }
    // the quantile state was sized (and exported) at create from the config
    s->want_fq = c.track_quantiles != 0;
    if (s->want_fq) CK(e->o_fq.ensure(TT * 3));
    if (out && out->indices) CK(e->idx.ensure(ns));
    CK(e->dz.ensure(2 * ns));
    CK(e->dgs.ensure(2 * ns));
    CK(e->dgt.ensure(2 * ns));
    Scalars s0h;
    memset(&s0h, 0, sizeof(s0h));
    s0h.cs = (LS && c.sigma2_shape > 1.0) ? c.sigma2_scale / (c.sigma2_shape - 1.0) : 0.0;
    s0h.ct = (LT && c.tau2_shape > 1.0) ? c.tau2_scale / (c.tau2_shape - 1.0) : 0.0;
    CK(cudaMemcpyAsync(e->sc.p, &s0h, sizeof(Scalars), cudaMemcpyHostToDevice, e->st));
    CK(cudaMemsetAsync(e->fail.p, 0, sizeof(int64_t), e->st));
    // quantile targets: rank 0 initialises the shared state
    std::vector<QTarget> tgs;
    {
      const double sp[3] = {0.05, 0.5, 0.95};
      const double pp[5] = {0.005, 0.05, 0.5, 0.95, 0.995};
      auto add = [&](int q, const double* ps, int np) {
        for (int i = 0; i < np; ++i) {
          QTarget t;
          memset(&t, 0, sizeof(t));
          t.p = ps[i];
          t.q = q;
          t.col = i;
          t.zprev = ndtri(ps[i]);
          t.h = Q_H0;
          tgs.push_back(t);
        }
      };
      if (s->want_fq) add(0, sp, 3);
      if (LS) add(1, pp, 5);
      if (LT) add(2, pp, 5);
    }
    s->ntg = (int)tgs.size();
    s->qm = (s->want_fq ? 1 : 0) | (LS ? 2 : 0) | (LT ? 4 : 0);
    const CdfPlan plan = cdf_plan(ns);
    s->cls_grid = (int)std::min<int64_t>(plan.tiles, (int64_t)sm_count() * 2);
    s->qcap = (uint32_t)std::max<int64_t>(4096, N / 4);
    if (s->rank == 0 && s->ntg) {
      CK(cudaMemcpyAsync(s->q_tg, tgs.data(), s->ntg * sizeof(QTarget), cudaMemcpyHostToDevice, e->st));
      CK(cudaMemsetAsync(s->q_sh, 0, 2 * sizeof(QShared), e->st));
      CK(cudaMemsetAsync(s->q_hist, 0, (size_t)Q_MAXT * Q_SUB * 8, e->st));
      CK(cudaMemsetAsync(s->q_fhist, 0, (size_t)Q_MAXT * Q_FB * 8, e->st));
      CK(cudaMemsetAsync(s->q_unres, 0, 4 * sizeof(unsigned int), e->st));
    }
    // init + draws of step 1
    InitArgs a;
    memset(&a, 0, sizeof(a));
    a.n = ns;
    a.seed = c.seed;
    a.x0_mean = c.x0_mean;
    a.sqrt_x0_var = c.sqrt_x0_var;
    a.bs0 = c.sigma2_scale;
    a.bt0 = c.tau2_scale;
    a.sigma2_fixed = c.sigma2_fixed;
    a.tau2_fixed = c.tau2_fixed;
    a.gs = gamma_src(e, true, 0);
    a.gt = gamma_src(e, false, 0);
    a.rec = e->rec[0].p;
    a.gbase = (int64_t)s->rank * ns;
    CK(cudaEventRecord(e->ev0, e->st));
    init_kernel<MODE><<<grid_for(ns, 256), 256, 0, e->st>>>(a);
    LAUNCHED();
    // Fused draws (as the engine's large-N path): the step kernel evaluates
    // its own normal / gamma draws from the per-step tables in shared memory.
    static const int fused_env = [] {
      const char* v = getenv("PF_FUSED_DRAWS");
      return v ? atoi(v) : -1;
    }();
    s->fused = c.gamma_method == 0 && e->ntab && fused_env != 0;
    if (T >= 1 && !s->fused) return draws(s, 1);
    return PF_OK;
  }

  static int draws(pf_shard* s, int64_t t) {
    pf_engine* e = s->e;
    const bool share_tab = LS && LT && e->tab_s == e->tab_t && s->cfg.gamma_method == 0;
    const int ngt = s->cfg.gamma_method == 0 ? (LS ? 1 : 0) + (LT && !share_tab ? 1 : 0) : 0;
    const size_t draw_smem = ((size_t)ngt * GT_TABLE_DOUBLES + (e->ntab ? NT_TABLE_DOUBLES : 0)) * sizeof(double);
    CK(cudaFuncSetAttribute(draws_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)((2 * GT_TABLE_DOUBLES + NT_TABLE_DOUBLES) * sizeof(double))));
    DrawArgs d;
    memset(&d, 0, sizeof(d));
    d.n = s->ns;
    d.t = t;
    d.seed = s->cfg.seed;
    d.gs = gamma_src(e, true, t);
    d.gt = gamma_src(e, false, t);
    d.ntab = e->ntab;
    const size_t off = (size_t)(t & 1) * s->ns;
    d.z = e->dz.p + off;
    d.g_s = e->dgs.p + off;
    d.g_t = e->dgt.p + off;
    d.u3 = e->du3.p + off;
    d.fail = e->fail.p;
    d.gbase = (int64_t)s->rank * s->ns;
    draws_kernel<MODE><<<grid_for(s->ns, 256, sm_count() * 2), 256, draw_smem, e->st>>>(d);
    LAUNCHED();
    return PF_OK;
  }

  // Phase 1: ancestors (step t-1's resample) + step kernel -> xrec[rank].
  // Rank 0: the main stream waits for the last resolve (before the partial
  // all-gather that follows phase 1, or the outputs).
  static int join_resolve(pf_shard* s, int64_t t_resolved) {
    if (!s->resolve_pending) return PF_OK;
    CK(cudaStreamWaitEvent(s->e->st, s->e->ev_q[t_resolved & 1], 0));
    s->resolve_pending = false;
    return PF_OK;
  }

  static int phase1(pf_shard* s, int64_t t) {
    pf_engine* e = s->e;
    const pf_config& c = s->cfg;
    const int64_t ns = s->ns;
    const int par = (int)(t & 1);
    const bool FDm = s->fused;
    const int threads = FDm ? FD_THREADS : 256;
    const int sbx = FDm ? FD_SB : STEP_SB;
    const bool share_tab = LS && LT && e->tab_s == e->tab_t && c.gamma_method == 0;
    const int ngt = c.gamma_method == 0 ? (LS ? 1 : 0) + (LT && !share_tab ? 1 : 0) : 0;
    const size_t draw_smem = ((size_t)ngt * GT_TABLE_DOUBLES + (e->ntab ? NT_TABLE_DOUBLES : 0)) * sizeof(double);
    const size_t step_smem = (FDm ? (size_t)(((draw_smem / 8) + 3) & ~size_t(3)) * 8 : 0) +
                             (size_t)2 * sbx * threads * (sizeof(Rec) + 3 * sizeof(double));
    static DevOnce attr;
    if (attr.pending()) {
      CK(cudaFuncSetAttribute(step_kernel<MODE, TQ, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)((2 * GT_TABLE_DOUBLES + NT_TABLE_DOUBLES + 4) * sizeof(double) +
                                    2 * FD_SB * FD_THREADS * (sizeof(Rec) + 3 * sizeof(double)))));
      CK(cudaFuncSetAttribute(step_kernel<MODE, TQ, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(2 * STEP_SB * 256 * (sizeof(Rec) + 3 * sizeof(double)))));
      attr.mark();
    }
    int occ = 0;
    if (FDm)
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, step_kernel<MODE, TQ, true>, threads, step_smem));
    else
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, step_kernel<MODE, TQ, false>, threads, step_smem));
    const int64_t nb = (ns + sbx * threads - 1) / (sbx * threads);
    const int grid = (int)std::min<int64_t>(nb, (int64_t)sm_count() * std::max(occ, 1));
    StepArgs<TQ> a;
    memset(&a, 0, sizeof(a));
    a.n = ns;
    a.t = t;
    a.seed = c.seed;
    a.y = s->y_host[(size_t)(t - 1)];
    a.sigma2_fixed = c.sigma2_fixed;
    a.tau2_fixed = c.tau2_fixed;
    a.sqrt_tau2_fixed = c.sqrt_tau2_fixed;
    a.log_term_fixed = c.log_term_fixed;
    a.rec_in = e->rec[s->cur].p;
    a.rec_out = e->rec[s->cur ^ 1].p;
    a.lw = e->lw.p + (size_t)par * ns;
    a.Mout = e->mbuf.p + par;
    a.u3 = e->du3.p + (size_t)((t - 1) & 1) * ns;
    a.idx_out = (s->out && s->out->indices && t > 1) ? e->idx.p : nullptr;
    const size_t off = (size_t)par * ns;
    a.z = e->dz.p + off;
    a.g_s = e->dgs.p + off;
    a.g_t = e->dgt.p + off;
    uint32_t* kb = s->ntg ? e->keys.p + (size_t)par * 3 * ns : nullptr;
    a.kx = (s->ntg && s->want_fq) ? kb : nullptr;
    a.ks = (s->ntg && LS) ? kb + ns : nullptr;
    a.kt = (s->ntg && LT) ? kb + 2 * (size_t)ns : nullptr;
    a.partials = e->partials.p;
    a.sc = e->sc.p;
    a.out.fmean = e->o_fm.p;
    a.out.s_mean = e->o_sm.p;
    a.out.s_sd = e->o_ssd.p;
    a.out.t_mean = e->o_tm.p;
    a.out.t_sd = e->o_tsd.p;
    a.out.ess = nullptr;  // sharded: the combine kernel writes it
    a.fail = e->fail.p;
    a.xrec = s->xrec;
    a.ref_slack = 64.0;
    a.shard = s->rank;
    a.slk.G = s->world;
    a.slk.lg = s->lg;
    a.slk.n = c.n;
    a.slk.lend = s->lend;
    for (int h = 0; h < s->world; ++h) {
      a.slk.cut[h] = s->p_cut[h];
      a.slk.q[h] = (const TQ*)s->p_q[h];
      a.recs[h] = s->p_rec[s->cur][h];
      if (s->rank_on) {
        a.srk.grp[h] = s->p_grp[h];
        a.srk.fq[h] = s->p_fq[h];
        a.srk.f32[h] = s->p_f32[h];
      }
    }
    a.srk.B = 53 - ilog2(c.n);
    a.srk.on = s->rank_on && t > 1;
    const bool spacings = c.resampler == PF_RESAMPLE_SPACINGS;  // K7: ordered uniforms
    if (spacings && t > 1) {  // words of step t-1 from its scan and every rank's total
      a.spS = e->spS.p;
      a.sp_tot = e->sptot.p + (size_t)((t - 1) & 1) * PF_MAX_SHARDS;
    }
    if (FDm) {
      a.dr.n = ns;
      a.dr.t = t;
      a.dr.seed = c.seed;
      a.dr.gs = gamma_src(e, true, t);
      a.dr.gt = gamma_src(e, false, t);
      a.dr.ntab = e->ntab;
      a.dr.u3 = e->du3.p + (size_t)par * ns;  // resampling words of step t
      a.dr.fail = e->fail.p;
      a.dr.gbase = (int64_t)s->rank * ns;
      a.z = a.g_s = a.g_t = nullptr;
      step_kernel<MODE, TQ, true><<<grid, threads, step_smem, e->st>>>(a);
      LAUNCHED();
    } else {
      step_kernel<MODE, TQ, false><<<grid, threads, step_smem, e->st>>>(a);
      LAUNCHED();
      if (t < s->T) {
        int rc = draws(s, t + 1);
        if (rc != PF_OK) return rc;
      }
    }
    if (spacings) {
      // K7: this rank's prefix sums of its step-t exponentials; the total
      // rides in its exchange record (all-gathered after phase 1)
      auto it = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                                ExpOfWord{e->du3.p + (size_t)par * ns});
      size_t tb = e->sptmp_bytes;
      CK(cub::DeviceScan::InclusiveSum(e->sptmp.p, tb, it, e->spS.p, (int)ns, e->st));
      spacings_shard_total_kernel<<<1, 1, 0, e->st>>>(e->spS.p, ns, s->xrec, s->rank);
      g_launches.fetch_add(2);
    }
    if (s->out && s->out->indices && t > 1)
      CK(cudaMemcpyAsync(s->out->indices + (size_t)(t - 2) * ns, e->idx.p, ns * sizeof(int64_t),
                         cudaMemcpyDeviceToHost, e->st));
    s->cur ^= 1;
    return join_resolve(s, t - 1);
  }

  // Phase 2: combine the G partials (every rank identically) + K2 -> xtot[rank].
  static int phase2(pf_shard* s, int64_t t) {
    pf_engine* e = s->e;
    const int64_t ns = s->ns;
    const int par = (int)(t & 1);
    StepOut so;
    so.fmean = e->o_fm.p;
    so.s_mean = e->o_sm.p;
    so.s_sd = e->o_ssd.p;
    so.t_mean = e->o_tm.p;
    so.t_sd = e->o_tsd.p;
    so.ess = e->o_ess.p;
    double* qmom = (s->rank == 0 && s->ntg) ? &(s->q_sh + par)->mean[0] : nullptr;
    combine_kernel<MODE><<<1, 256, 0, e->st>>>(s->xrec, s->world, t, 0, so, qmom, e->sc.p, e->mbuf.p + par,
                                               e->fail.p,
                                               s->cfg.resampler == PF_RESAMPLE_SPACINGS
                                                   ? e->sptot.p + (size_t)(t & 1) * PF_MAX_SHARDS : nullptr);
    LAUNCHED();
    const CdfPlan plan = cdf_plan(ns);
    WSrc w;
    w.src = e->lw.p + (size_t)par * ns;
    w.M = e->mbuf.p + par;
    w.mode = 0;
    CdfBufs& b = e->cdf;
    cdf_reduce_kernel<TQ><<<(int)plan.chunks, CDF_THREADS, 0, e->st>>>(w, plan.R, (TQ*)b.tile_tot.p,
                                                                       (TQ*)b.chunk_tot.p, e->fail.p);
    LAUNCHED();
    const size_t top_smem = 4 * (size_t)plan.chunks * sizeof(TQ);
    CK(cudaFuncSetAttribute(cdf_shard_total_kernel<TQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            4 * CDF_MAX_CHUNKS * (int)sizeof(TQ)));
    cdf_shard_total_kernel<TQ><<<1, 1024, top_smem, e->st>>>((TQ*)b.chunk_tot.p, plan.chunks, (TQ*)s->xtot,
                                                             s->rank, e->fail.p);
    LAUNCHED();
    return PF_OK;
  }

  static QArgs qargs(pf_shard* s, int par) {
    QArgs qa;
    memset(&qa, 0, sizeof(qa));
    qa.ntarget = s->ntg;
    qa.tg = s->q_tg;
    qa.sh = s->q_sh + par;
    qa.cand = s->q_cand;
    qa.cap = s->qcap;
    qa.part = s->q_part;
    qa.hist = s->q_hist;
    qa.fhist = s->q_fhist;
    qa.stats = s->q_unres;
    qa.fx_scale = std::ldexp(1.0, 62 - ilog2(s->cfg.n));
    return qa;
  }

  // Phase 3: top tree from the G totals + K4 (q, cut table) + classification.
  static int phase3(pf_shard* s, int64_t t) {
    pf_engine* e = s->e;
    const int64_t ns = s->ns, N = s->cfg.n;
    const int par = (int)(t & 1);
    if (s->ntg) {  // the side stream's classification starts from here (M and keys of step t)
      CK(cudaEventRecord(e->ev_b, e->st));
      CK(cudaStreamWaitEvent(e->side, e->ev_b, 0));
    }
    const CdfPlan plan = cdf_plan(ns);
    const size_t top_smem = 4 * (size_t)plan.chunks * sizeof(TQ);
    CK(cudaFuncSetAttribute(cdf_top_shard_kernel<TQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            4 * CDF_MAX_CHUNKS * (int)sizeof(TQ)));
    CdfBufs& b = e->cdf;
    cdf_top_shard_kernel<TQ><<<1, 1024, top_smem, e->st>>>((TQ*)b.chunk_tot.p, plan.chunks, (TQ*)s->xtot,
                                                           s->world, s->rank, N, (TQ*)b.node.p, (TQ*)b.carry.p,
                                                           (TQ*)b.total.p, s->lend, e->fail.p, t);
    LAUNCHED();
    WSrc w;
    w.src = e->lw.p + (size_t)par * ns;
    w.M = e->mbuf.p + par;
    w.mode = 0;
    if (s->rank_on) {
      RankOut ro{s->gcut, s->sfq, s->sf32, 53 - ilog2(N)};
      cdf_expand_kernel<TQ, true><<<(int)plan.chunks, CDF_THREADS, 0, e->st>>>(
          w, N, plan.R, (TQ*)b.tile_tot.p, (TQ*)b.node.p, (TQ*)b.carry.p, (TQ*)b.total.p, (TQ*)s->gq, s->gcut,
          e->fail.p, ro, (int64_t)s->rank * ns);
      LAUNCHED();
      group_build_shard_kernel<<<grid_for(ns / GRP_STRATA, 256, sm_count() * 8), 256, 0, e->st>>>(
          s->gcut, s->lend, s->rank, s->world, N, s->sgrp, e->fail.p);
    } else {
      cdf_expand_kernel<TQ, false><<<(int)plan.chunks, CDF_THREADS, 0, e->st>>>(
          w, N, plan.R, (TQ*)b.tile_tot.p, (TQ*)b.node.p, (TQ*)b.carry.p, (TQ*)b.total.p, (TQ*)s->gq, s->gcut,
          e->fail.p, RankOut(), (int64_t)s->rank * ns);
    }
    LAUNCHED();
    if (s->ntg) {
      // the window classification on the side stream, beside K3 / K4: it
      // needs only this step's M and keys (phase 2); the barrier after this
      // phase orders it before rank 0's resolve
      QArgs q2 = qargs(s, par);
      uint32_t* kb = e->keys.p + (size_t)par * 3 * ns;
      q2.keys[0] = s->want_fq ? kb : nullptr;
      q2.keys[1] = LS ? kb + ns : nullptr;
      q2.keys[2] = LT ? kb + 2 * (size_t)ns : nullptr;
      q2.pbase = s->rank * s->cls_grid;
      q2.ptotal = s->world * s->cls_grid;
      q2.gbase = (uint32_t)((int64_t)s->rank * ns);
      int rc = launch_classify<TQ>(s->qm, s->cls_grid, w, (int)plan.tiles, e->fail.p, q2, e->side);
      if (rc != PF_OK) return rc;
      CK(cudaEventRecord(e->ev_e, e->side));
      CK(cudaStreamWaitEvent(e->st, e->ev_e, 0));
    }
    return PF_OK;
  }

  // Phase 4 (rank 0): the exact quantile resolve over every rank's candidates.
  static int phase4(pf_shard* s, int64_t t) {
    if (s->rank != 0 || !s->ntg) return PF_OK;
    pf_engine* e = s->e;
    const pf_config& c = s->cfg;
    const int64_t ns = s->ns, N = c.n;
    const int par = (int)(t & 1);
    const int ntg = s->ntg;
    // rank 0's resolve of step t runs on its side stream, overlapping step
    // t+1's step kernel; phase 1 of step t+1 holds rank 0's main stream (and
    // with it every rank, through the partial all-gather) until it is done
    cudaStream_t ss = e->side;
    CK(cudaEventRecord(e->ev_b, e->st));
    CK(cudaStreamWaitEvent(ss, e->ev_b, 0));
    QArgs qa = qargs(s, par);
    qa.lidx = e->qlidx.p;
    qa.lw = e->qlw.p;
    QValueSrc vs;
    memset(&vs, 0, sizeof(vs));
    vs.nsh = s->world;
    vs.lg = s->lg;
    for (int h = 0; h < s->world; ++h) vs.recs[h] = s->p_rec[s->cur][h];
    vs.seed = c.seed;
    vs.t = t;
    vs.gs = gamma_src(e, true, t);
    vs.sigma2_fixed = c.sigma2_fixed;
    vs.tau2_fixed = c.tau2_fixed;
    vs.learn_s = LS;
    vs.learn_t = LT;
    double *ox = e->o_fq.p, *os = e->o_sq.p, *ot = e->o_tq.p;
    const int hgrid = std::max(1, std::min(64, (int)((N / 64 + 255) / 256)));
    CK(cudaFuncSetAttribute(q_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Q_RESOLVE_SMEM));
    const int fb_grid = grid_for(ns, 256, sm_count() * 2);
    for (int round = 0; round < 2; ++round) {
      q_hist_kernel<<<dim3(hgrid, ntg), 256, 0, ss>>>(qa, e->fail.p, round);
      q_locate_kernel<<<ntg, 1024, 0, ss>>>(qa, e->fail.p, round);
      q_filter_kernel<<<dim3(hgrid, ntg), 256, 0, ss>>>(qa, e->fail.p);
      q_finish_kernel<<<ntg, 1024, Q_RESOLVE_SMEM, ss>>>(qa, vs, ox, os, ot, t, e->fail.p);
      g_launches.fetch_add(4);
      if (round == 0) {
        for (int attempt = 0; attempt < 2; ++attempt) {
          if (int r_ = fb_hist_smem()) return r_;
          q_fallback_prep_kernel<<<1, 32, 0, ss>>>(qa, attempt, e->fail.p);
          for (int h = 0; h < s->world; ++h) {  // every rank's particles (IPC reads)
            QArgs q2 = qa;
            const uint32_t* kb = s->p_keys[h] + (size_t)par * 3 * ns;
            q2.keys[0] = s->want_fq ? kb : nullptr;
            q2.keys[1] = LS ? kb + ns : nullptr;
            q2.keys[2] = LT ? kb + 2 * (size_t)ns : nullptr;
            q2.pbase = h * fb_grid;
            q2.ptotal = s->world * fb_grid;
            q2.gbase = (uint32_t)((int64_t)h * ns);
            q_fallback_hist_kernel<<<fb_grid, 256, QFB_SMEM_BYTES, ss>>>(q2, s->p_lw[h] + (size_t)par * ns, 0,
                                                            s->p_mbuf[h] + par, ns, SINGLE, attempt, e->fail.p);
          }
          q_fallback_select_kernel<<<ntg, 1024, 0, ss>>>(qa, attempt, e->fail.p);
          g_launches.fetch_add(2 + s->world);
        }
        for (int h = 0; h < s->world; ++h) {
          QArgs q2 = qa;
          const uint32_t* kb = s->p_keys[h] + (size_t)par * 3 * ns;
          q2.keys[0] = s->want_fq ? kb : nullptr;
          q2.keys[1] = LS ? kb + ns : nullptr;
          q2.keys[2] = LT ? kb + 2 * (size_t)ns : nullptr;
          q2.gbase = (uint32_t)((int64_t)h * ns);
          q_fallback_fill_kernel<<<fb_grid, 256, 0, ss>>>(q2, s->p_lw[h] + (size_t)par * ns, 0, s->p_mbuf[h] + par,
                                                          ns, SINGLE, e->fail.p);
        }
        g_launches.fetch_add(s->world);
      }
    }
    QAll all;
    memset(&all, 0, sizeof(all));
    all.nsrc = s->world;
    all.ns = ns;
    for (int h = 0; h < s->world; ++h) {  // every rank's particles (IPC reads)
      const uint32_t* kb = s->p_keys[h] + (size_t)par * 3 * ns;
      all.keys[h][0] = s->want_fq ? kb : nullptr;
      all.keys[h][1] = LS ? kb + ns : nullptr;
      all.keys[h][2] = LT ? kb + 2 * (size_t)ns : nullptr;
      all.lw[h] = s->p_lw[h] + (size_t)par * ns;
      all.M[h] = s->p_mbuf[h] + par;
    }
    all.single = SINGLE;
    q_select_kernel<<<ntg, 1024, 0, ss>>>(qa, vs, e->qscratch.p, ox, os, ot, t, e->fail.p, s->q_unres, all);
    q_step_end_kernel<<<1, 1024, 0, ss>>>(qa, 1);
    g_launches.fetch_add(2);
    CK(cudaEventRecord(e->ev_q[t & 1], ss));
    s->resolve_pending = true;
    return PF_OK;
  }

  // Final resample of step T (this rank's slots) and the outputs.
  static int finish(pf_shard* s) {
    pf_engine* e = s->e;
    const pf_config& c = s->cfg;
    const int64_t ns = s->ns, T = s->T;
    if (int rc = join_resolve(s, T)) return rc;
    pf_outputs* out = s->out;
    const bool keep_idx = out && out->indices;
    const bool keep_final = out && (out->final_states || out->final_sigma2);
    if (T >= 1 && (keep_idx || keep_final)) {
      GroupMatArgs<TQ> m;
      memset(&m, 0, sizeof(m));
      m.ns = ns;
      m.gbase = (int64_t)s->rank * ns;
      m.t = T;
      m.seed = c.seed;
      m.u3 = e->du3.p + (size_t)(T & 1) * ns;
      if (c.resampler == PF_RESAMPLE_SPACINGS) {
        spacings_words_kernel<<<grid_for(ns, 256), 256, 0, e->st>>>(
            e->spS.p, ns, e->sptot.p + (size_t)(T & 1) * PF_MAX_SHARDS, s->world, s->rank, c.seed, T, e->spw.p,
            e->fail.p);
        LAUNCHED();
        m.u3 = e->spw.p;
      }
      m.slk.G = s->world;
      m.slk.lg = s->lg;
      m.slk.n = c.n;
      m.slk.lend = s->lend;
      for (int h = 0; h < s->world; ++h) {
        m.slk.cut[h] = s->p_cut[h];
        m.slk.q[h] = (const TQ*)s->p_q[h];
        m.recs[h] = s->p_rec[s->cur][h];
      }
      m.gs = gamma_src(e, true, T);
      m.learn_s = LS;
      m.learn_t = LT;
      m.sigma2_fixed = c.sigma2_fixed;
      m.tau2_fixed = c.tau2_fixed;
      m.a_s = shape_at(e, true, T);
      m.a_t = shape_at(e, false, T);
      m.idx = keep_idx ? e->idx.p : nullptr;
      double* dst[7] = {out->final_states, out->final_sigma2, out->final_tau2, out->final_a_sigma,
                        out->final_b_sigma, out->final_a_tau, out->final_b_tau};
      DevBuf<double>* bufs[7] = {&e->m_x, &e->m_s2, &e->m_t2, &e->m_as, &e->m_bs, &e->m_at, &e->m_bt};
      double** slots[7] = {&m.x, &m.s2, &m.t2, &m.as, &m.bs, &m.at, &m.bt};
      for (int k = 0; k < 7; ++k) {
        *slots[k] = nullptr;
        if (keep_final && dst[k]) {
          CK(bufs[k]->ensure(ns));
          *slots[k] = bufs[k]->p;
        }
      }
      m.fail = e->fail.p;
      group_materialize_kernel<TQ><<<grid_for(ns, 256), 256, 0, e->st>>>(m);
      LAUNCHED();
      if (keep_idx)
        CK(cudaMemcpyAsync(out->indices + (size_t)(T - 1) * ns, e->idx.p, ns * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, e->st));
      for (int k = 0; k < 7; ++k)
        if (*slots[k]) CK(cudaMemcpyAsync(dst[k], *slots[k], ns * sizeof(double), cudaMemcpyDeviceToHost, e->st));
    }
    if (out && T > 0) {
      auto cp = [&](double* h, DevBuf<double>& d, size_t cnt) -> int {
        if (h) CK(cudaMemcpyAsync(h, d.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, e->st));
        return PF_OK;
      };
      int rc;
      if ((rc = cp(out->filtered_mean, e->o_fm, T)) != PF_OK) return rc;
    if (out->ess && (rc = cp(out->ess, e->o_ess, T)) != PF_OK) return rc;
      if (s->want_fq && (rc = cp(out->filtered_quantiles, e->o_fq, T * 3)) != PF_OK) return rc;
      if (LS && ((rc = cp(out->sigma2_mean, e->o_sm, T)) || (rc = cp(out->sigma2_sd, e->o_ssd, T)) ||
                 (rc = cp(out->sigma2_quantiles, e->o_sq, T * 5))))
        return rc;
      if (LT && ((rc = cp(out->tau2_mean, e->o_tm, T)) || (rc = cp(out->tau2_sd, e->o_tsd, T)) ||
                 (rc = cp(out->tau2_quantiles, e->o_tq, T * 5))))
        return rc;
    }
    CK(cudaEventRecord(e->ev1, e->st));
    int64_t f = 0;
    CK(cudaMemcpyAsync(&f, e->fail.p, sizeof(int64_t), cudaMemcpyDeviceToHost, e->st));
    CK(cudaStreamSynchronize(e->st));
    CK(cudaGetLastError());
    float ms = 0;
    cudaEventElapsedTime(&ms, e->ev0, e->ev1);
    e->last_total_ms = ms;
    if (out) {
      for (int k = 0; k < 7; ++k) out->phase_ns[k] = 0;
      out->phase_ns[6] = (int64_t)llround(ms * 1e6);
      out->failed_step = f;
    }
    if (f > 0)
      return set_err(PF_ERR_ALL_WEIGHTS_ZERO, "all particle weights are zero (at time step " + std::to_string(f) + ")",
                     f);
    if (f < 0) return set_err(PF_ERR_ALL_WEIGHTS_ZERO, "all particle weights are zero", 0);
    if (s->rank == 0 && s->ntg) return check_quantile_unresolved(s->q_unres);
    return PF_OK;
  }
};

struct ShardFns {
  int (*begin)(pf_shard*, const double*, int64_t, pf_outputs*);
  int (*phase[4])(pf_shard*, int64_t);
  int (*finish)(pf_shard*);
};

template <int MODE, typename TQ>
ShardFns shard_fns() {
  using O = ShardOps<MODE, TQ>;
  return ShardFns{O::begin, {O::phase1, O::phase2, O::phase3, O::phase4}, O::finish};
}

ShardFns pick_shard_fns(int mode) {
  switch (mode) {
    case 0: return shard_fns<0, double>();
    case 1: return shard_fns<1, double>();
    case 2: return shard_fns<2, double>();
    case 3: return shard_fns<3, double>();
    case 4: return shard_fns<4, float>();
    case 5: return shard_fns<5, float>();
    case 6: return shard_fns<6, float>();
    default: return shard_fns<7, float>();
  }
}

int shard_mode(const pf_config& c) {
  return (c.learn && c.learn_sigma2 ? M_LS : 0) | (c.learn && c.learn_tau2 ? M_LT : 0) |
         (c.precision == PF_DTYPE_F32 ? M_SINGLE : 0);
}

}  // namespace
