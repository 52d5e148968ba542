// Particle-sharded run of ONE filter over G shards (multi-GPU).
//
// Included by engine.cu inside its anonymous namespace (uses pf_engine and
// the kernels).  Shard g owns the N/G consecutive slots [g N/G, (g+1) N/G)
// and lives on devices[g] (shards may share a device: the tests run G
// shards on one B200).  Every shard is a subtree of the reference's adder
// tree, so the run is bit-identical to one device in ancestors and
// particles.  Per step t the shards exchange, through peer memory on shard
// 0's device (NVLink P2P when the devices differ), only:
//   * one Partial record each (max log-weight, NaN flag, moment sums): every
//     shard then finalises the step identically (global max M, moments);
//   * one subtree total each: every shard rebuilds the top tree -> root,
//     its shard node and carry, and all shards' stratum bounds L_end;
// plus the data-dependent reads of resampling: a slot's cut-point lookup
// reads the owner shard's cut table and q, and the ancestor's 32-byte
// record is gathered from whichever shard holds it.  Weighted quantiles:
// every shard classifies its own particles into shard 0's window state;
// shard 0 resolves.  Phases are ordered across shard streams by events.
#pragma once

struct pf_group {
  pf_config cfg;  // n = N (all shards)
  int G = 0;
  int64_t ns = 0;  // slots per shard
  int lg = 0;      // log2(ns)
  std::vector<int> dev;
  std::vector<pf_engine*> sh;
  // exchange (on shard 0's device)
  Partial* xrec = nullptr;
  void* xtot = nullptr;
  // per shard: full-size cut table (global strata), q of its slots, L_end copy
  std::vector<int32_t*> gcut;
  std::vector<void*> gq;
  std::vector<int64_t*> lend;
  // per shard rank tables (N >= 2^21): grp over the global stratum groups,
  // fq / f32 over the shard's particles
  bool rank_on = false;
  std::vector<Grp*> sgrp;
  std::vector<uint8_t*> sfq;
  std::vector<uint32_t*> sf32;
  std::vector<cudaEvent_t> evA, evB, evC, evK, evD;
  cudaEvent_t evM = nullptr;  // shard 0's combine (quantile windows) done
  double last_ms = 0;
};

namespace {

int set_device(int d) {
  CK(cudaSetDevice(d));
  return PF_OK;
}

template <int MODE, typename TQ>
int run_group(pf_group* g, const double* y, int64_t T, pf_outputs* out) {
  constexpr bool LS = MODE & M_LS, LT = MODE & M_LT;
  constexpr int SINGLE = (MODE & M_SINGLE) ? 1 : 0;
  const pf_config& c = g->cfg;
  const int G = g->G;
  const int64_t ns = g->ns, N = c.n;
  pf_engine* e0 = g->sh[0];
  int rc;
  const bool spacings = c.resampler == PF_RESAMPLE_SPACINGS;  // K7: ordered uniforms
  const bool want_fq = out ? out->filtered_quantiles != nullptr : c.track_quantiles != 0;
  const bool keep_idx = out && out->indices;
  const bool keep_final = out && (out->final_states || out->final_sigma2);
  const size_t TT = (size_t)(T > 0 ? T : 1);
  const CdfPlan plan = cdf_plan(ns);
  if (plan.small) return set_err(PF_ERR_VALUE, "sharded runs need at least 4096 particles per shard");
  const int sms = sm_count();

  // ---- per-shard setup
  for (int s = 0; s < G; ++s) {
    pf_engine* e = g->sh[s];
    if ((rc = set_device(g->dev[s])) != PF_OK) return rc;
    if ((rc = build_tables(e, T)) != PF_OK) return rc;
    CK(e->o_fm.ensure(TT));
    CK(e->o_ess.ensure(TT));
    if (LS) { CK(e->o_sm.ensure(TT)); CK(e->o_ssd.ensure(TT)); CK(e->o_sq.ensure(TT * 5)); }
    if (LT) { CK(e->o_tm.ensure(TT)); CK(e->o_tsd.ensure(TT)); CK(e->o_tq.ensure(TT * 5)); }
    if (want_fq) CK(e->o_fq.ensure(TT * 3));
    if (keep_idx) CK(e->idx.ensure(ns));
    if (want_fq || LS || LT) CK(e->keys.ensure((size_t)6 * ns));  // quantile keys [2][3][ns]
    // sharded runs precompute the draws (draws_kernel, by step parity)
    CK(e->dz.ensure(2 * ns));
    CK(e->dgs.ensure(2 * ns));
    CK(e->dgt.ensure(2 * ns));
    Scalars s0h;
    memset(&s0h, 0, sizeof(s0h));
    s0h.cs = (LS && c.sigma2_shape > 1.0) ? c.sigma2_scale / (c.sigma2_shape - 1.0) : 0.0;
    s0h.ct = (LT && c.tau2_shape > 1.0) ? c.tau2_scale / (c.tau2_shape - 1.0) : 0.0;
    CK(cudaMemcpyAsync(e->sc.p, &s0h, sizeof(Scalars), cudaMemcpyHostToDevice, e->st));
    CK(cudaMemsetAsync(e->fail.p, 0, sizeof(int64_t), e->st));
  }

  // ---- weighted-quantile targets (shard 0's state, fed by every shard)
  const bool want_sq = LS, want_tq = LT;
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
    if (want_fq) add(0, sp, 3);
    if (want_sq) add(1, pp, 5);
    if (want_tq) add(2, pp, 5);
  }
  const int ntg = (int)tgs.size();
  const int qm = (want_fq ? 1 : 0) | (want_sq ? 2 : 0) | (want_tq ? 4 : 0);
  int cls_grid = 0;
  QArgs qa;
  memset(&qa, 0, sizeof(qa));
  if ((rc = set_device(g->dev[0])) != PF_OK) return rc;
  if (ntg) {
    // the classify grid must be the same on every shard (partial slots)
    cls_grid = (int)std::min<int64_t>(plan.tiles, (int64_t)sms * 2);
    const uint32_t qcap = (uint32_t)std::max<int64_t>(4096, N / 4);
    CK(e0->qtg.ensure(Q_MAXT));
    CK(e0->qsh.ensure(2));
    CK(e0->qcand.ensure((size_t)ntg * qcap));
    CK(e0->qscratch.ensure((size_t)ntg * qcap));
    CK(e0->qpart.ensure((size_t)std::max<int64_t>((int64_t)G * cls_grid, sms * 8) * (Q_SLOTS + 1)));
    CK(e0->qhist.ensure((size_t)Q_MAXT * Q_SUB));
    CK(e0->qfhist.ensure((size_t)Q_MAXT * Q_FB));
    CK(e0->qunres.ensure(4));
    CK(e0->qlidx.ensure((size_t)Q_MAXT * Q_LIST));
    CK(e0->qlw.ensure((size_t)Q_MAXT * Q_LIST));
    cudaStream_t s0 = e0->st;
    CK(cudaMemcpyAsync(e0->qtg.p, tgs.data(), ntg * sizeof(QTarget), cudaMemcpyHostToDevice, s0));
    CK(cudaMemsetAsync(e0->qsh.p, 0, 2 * sizeof(QShared), s0));
    CK(cudaMemsetAsync(e0->qhist.p, 0, (size_t)Q_MAXT * Q_SUB * 8, s0));
    CK(cudaMemsetAsync(e0->qfhist.p, 0, (size_t)Q_MAXT * Q_FB * 8, s0));
    CK(cudaMemsetAsync(e0->qunres.p, 0, 4 * sizeof(unsigned int), s0));
    qa.ntarget = ntg;
    qa.tg = e0->qtg.p;
    qa.cand = e0->qcand.p;
    qa.cap = qcap;
    qa.part = e0->qpart.p;
    qa.hist = e0->qhist.p;
    qa.fhist = e0->qfhist.p;
    qa.stats = e0->qunres.p;
    qa.lidx = e0->qlidx.p;
    qa.lw = e0->qlw.p;
    qa.fx_scale = std::ldexp(1.0, 62 - ilog2(N));
    CK(cudaStreamSynchronize(s0));
  }

  // ---- kernel attributes and grids (all shards: same shapes)
  const bool share_tab = LS && LT && e0->tab_s == e0->tab_t && c.gamma_method == 0;
  const int ngt = c.gamma_method == 0 ? (LS ? 1 : 0) + (LT && !share_tab ? 1 : 0) : 0;
  const size_t draw_smem = ((size_t)ngt * GT_TABLE_DOUBLES + (e0->ntab ? NT_TABLE_DOUBLES : 0)) * sizeof(double);
  const size_t step_smem = (size_t)2 * STEP_SB * 256 * (sizeof(Rec) + 3 * sizeof(double));
  const size_t top_smem = 4 * (size_t)plan.chunks * sizeof(TQ);
  for (int s = 0; s < G; ++s) {
    if ((rc = set_device(g->dev[s])) != PF_OK) return rc;
    CK(cudaFuncSetAttribute(draws_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)((2 * GT_TABLE_DOUBLES + NT_TABLE_DOUBLES) * sizeof(double))));
    CK(cudaFuncSetAttribute(step_kernel<MODE, TQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_smem));
    CK(cudaFuncSetAttribute(cdf_shard_total_kernel<TQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            4 * CDF_MAX_CHUNKS * (int)sizeof(TQ)));
    CK(cudaFuncSetAttribute(cdf_top_shard_kernel<TQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            4 * CDF_MAX_CHUNKS * (int)sizeof(TQ)));
  }
  int occ = 0, docc = 0;
  if ((rc = set_device(g->dev[0])) != PF_OK) return rc;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, step_kernel<MODE, TQ>, 256, step_smem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&docc, draws_kernel<MODE>, 256, draw_smem));
  occ = std::max(occ, 1);
  docc = std::max(docc, 1);
  const int64_t nbatches = (ns + STEP_SB * 256 - 1) / (STEP_SB * 256);
  const int step_grid = (int)std::min<int64_t>(nbatches, (int64_t)sms * occ);
  const int draw_grid = (int)std::min<int64_t>((ns + 255) / 256, (int64_t)sms * docc);

  auto shard_gamma = [&](pf_engine* e, bool sigma, int64_t t) { return gamma_src(e, sigma, t); };
  auto launch_draws = [&](int s, int64_t t, cudaStream_t strm) {
    pf_engine* e = g->sh[s];
    DrawArgs d;
    memset(&d, 0, sizeof(d));
    d.n = ns;
    d.t = t;
    d.seed = c.seed;
    d.gs = shard_gamma(e, true, t);
    d.gt = shard_gamma(e, false, t);
    d.ntab = e->ntab;
    const size_t off = (size_t)(t & 1) * ns;
    d.z = e->dz.p + off;
    d.g_s = e->dgs.p + off;
    d.g_t = e->dgt.p + off;
    d.u3 = e->du3.p + off;
    d.fail = e->fail.p;
    d.gbase = (int64_t)s * ns;
    draws_kernel<MODE><<<draw_grid, 256, draw_smem, strm>>>(d);
    LAUNCHED();
  };
  auto wait_all = [&](cudaStream_t strm, std::vector<cudaEvent_t>& evs) -> int {
    for (int s = 0; s < G; ++s) CK(cudaStreamWaitEvent(strm, evs[s], 0));
    return PF_OK;
  };

  CK(cudaEventRecord(e0->ev0, e0->st));
  // ---- init + first draws
  for (int s = 0; s < G; ++s) {
    pf_engine* e = g->sh[s];
    if ((rc = set_device(g->dev[s])) != PF_OK) return rc;
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
    a.gs = shard_gamma(e, true, 0);
    a.gt = shard_gamma(e, false, 0);
    a.rec = e->rec[0].p;
    a.gbase = (int64_t)s * ns;
    CK(cudaStreamWaitEvent(e->st, e0->ev0, 0));
    init_kernel<MODE><<<grid_for(ns, 256), 256, 0, e->st>>>(a);
    LAUNCHED();
    if (T >= 1) launch_draws(s, 1, e->st);
  }

  int cur = 0;
  for (int64_t t = 1; t <= T; ++t) {
    const int par = (int)(t & 1);
    // ---- K1b on every shard (after every shard's tables of step t-1)
    for (int s = 0; s < G; ++s) {
      pf_engine* e = g->sh[s];
      if ((rc = set_device(g->dev[s])) != PF_OK) return rc;
      cudaStream_t st = e->st;
      if (t > 1) {
        if ((rc = wait_all(st, g->evC)) != PF_OK) return rc;
        CK(cudaStreamWaitEvent(st, e->ev_draw, 0));
        if (ntg && t > 2) CK(cudaStreamWaitEvent(st, e0->ev_q[t & 1], 0));
      }
      StepArgs<TQ> a;
      memset(&a, 0, sizeof(a));
      a.n = ns;
      a.t = t;
      a.seed = c.seed;
      a.y = y[t - 1];
      a.sigma2_fixed = c.sigma2_fixed;
      a.tau2_fixed = c.tau2_fixed;
      a.sqrt_tau2_fixed = c.sqrt_tau2_fixed;
      a.log_term_fixed = c.log_term_fixed;
      a.rec_in = e->rec[cur].p;
      a.rec_out = e->rec[cur ^ 1].p;
      a.lw = e->lw.p + (size_t)par * ns;
      a.Mout = e->mbuf.p + par;
      a.u3 = e->du3.p + (size_t)((t - 1) & 1) * ns;
      a.idx_out = (keep_idx && t > 1) ? e->idx.p : nullptr;
      const size_t off = (size_t)par * ns;
      a.z = e->dz.p + off;
      a.g_s = e->dgs.p + off;
      a.g_t = e->dgt.p + off;
      uint32_t* kb = ntg ? e->keys.p + (size_t)par * 3 * ns : nullptr;
      a.kx = (ntg && want_fq) ? kb : nullptr;
      a.ks = (ntg && want_sq) ? kb + ns : nullptr;
      a.kt = (ntg && want_tq) ? kb + 2 * (size_t)ns : nullptr;
      a.partials = e->partials.p;
      a.sc = e->sc.p;
      a.out.fmean = e->o_fm.p;
      a.out.s_mean = e->o_sm.p;
      a.out.s_sd = e->o_ssd.p;
      a.out.t_mean = e->o_tm.p;
      a.out.t_sd = e->o_tsd.p;
      a.out.ess = nullptr;  // sharded: the combine kernel writes it
      a.fail = e->fail.p;
      a.xrec = g->xrec;
      a.ref_slack = 64.0;
      a.shard = s;
      a.slk.G = G;
      a.slk.lg = g->lg;
      a.slk.n = N;
      a.slk.lend = g->lend[s];
      for (int h = 0; h < G; ++h) {
        a.slk.cut[h] = g->gcut[h];
        a.slk.q[h] = (const TQ*)g->gq[h];
        a.recs[h] = g->sh[h]->rec[cur].p;
        if (g->rank_on) {
          a.srk.grp[h] = g->sgrp[h];
          a.srk.fq[h] = g->sfq[h];
          a.srk.f32[h] = g->sf32[h];
        }
      }
      a.srk.B = 53 - ilog2(N);
      a.srk.on = g->rank_on && t > 1;
      if (spacings && t > 1) {  // words of step t-1 from its scan and every shard's total
        a.spS = e->spS.p;
        a.sp_tot = e->sptot.p + (size_t)((t - 1) & 1) * PF_MAX_SHARDS;
      }
      step_kernel<MODE, TQ><<<step_grid, 256, step_smem, st>>>(a);
      LAUNCHED();
      if (spacings) {
        // K7: this shard's prefix sums of its step-t exponentials; its total
        // joins the exchange record the combine kernels read
        auto it = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                                  ExpOfWord{e->du3.p + (size_t)(t & 1) * ns});
        size_t tb = e->sptmp_bytes;
        CK(cub::DeviceScan::InclusiveSum(e->sptmp.p, tb, it, e->spS.p, (int)ns, st));
        spacings_shard_total_kernel<<<1, 1, 0, st>>>(e->spS.p, ns, g->xrec, s);
        g_launches.fetch_add(2);
      }
      CK(cudaEventRecord(g->evA[s], st));
      if (t < T) {
        CK(cudaStreamWaitEvent(e->dstream, g->evA[s], 0));
        launch_draws(s, t + 1, e->dstream);
        CK(cudaEventRecord(e->ev_draw, e->dstream));
      }
      if (keep_idx && t > 1)
        CK(cudaMemcpyAsync(out->indices + (size_t)(t - 2) * N + (size_t)s * ns, e->idx.p, ns * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, st));
    }
    cur ^= 1;
    // ---- combine (every shard: global M, shifts; shard 0: outputs, windows)
    for (int s = 0; s < G; ++s) {
      pf_engine* e = g->sh[s];
      if ((rc = set_device(g->dev[s])) != PF_OK) return rc;
      if ((rc = wait_all(e->st, g->evA)) != PF_OK) return rc;
      StepOut so;
      so.fmean = e->o_fm.p;
      so.s_mean = e->o_sm.p;
      so.s_sd = e->o_ssd.p;
      so.t_mean = e->o_tm.p;
      so.t_sd = e->o_tsd.p;
      so.ess = e->o_ess.p;
      double* qmom = (s == 0 && ntg) ? &(e0->qsh.p + par)->mean[0] : nullptr;
      combine_kernel<MODE><<<1, 256, 0, e->st>>>(g->xrec, G, t, 0, so, qmom, e->sc.p, e->mbuf.p + par,
                                                 e->fail.p,
                                                 spacings ? e->sptot.p + (size_t)(t & 1) * PF_MAX_SHARDS : nullptr);
      LAUNCHED();
      if (s == 0) CK(cudaEventRecord(g->evM, e->st));
      // ---- K2 (local) and this shard's subtree total
      WSrc w;
      w.src = e->lw.p + (size_t)par * ns;
      w.M = e->mbuf.p + par;
      w.mode = 0;
      CdfBufs& b = e->cdf;
      cdf_reduce_kernel<TQ><<<(int)plan.chunks, CDF_THREADS, 0, e->st>>>(w, plan.R, (TQ*)b.tile_tot.p,
                                                                         (TQ*)b.chunk_tot.p, e->fail.p);
      LAUNCHED();
      cdf_shard_total_kernel<TQ><<<1, 1024, top_smem, e->st>>>((TQ*)b.chunk_tot.p, plan.chunks, (TQ*)g->xtot, s,
                                                               e->fail.p);
      LAUNCHED();
      CK(cudaEventRecord(g->evB[s], e->st));
    }
    // ---- K3b + K4 on every shard; classification of the quantile windows
    for (int s = 0; s < G; ++s) {
      pf_engine* e = g->sh[s];
      if ((rc = set_device(g->dev[s])) != PF_OK) return rc;
      if ((rc = wait_all(e->st, g->evB)) != PF_OK) return rc;
      CdfBufs& b = e->cdf;
      cdf_top_shard_kernel<TQ><<<1, 1024, top_smem, e->st>>>((TQ*)b.chunk_tot.p, plan.chunks, (TQ*)g->xtot, G, s, N,
                                                             (TQ*)b.node.p, (TQ*)b.carry.p, (TQ*)b.total.p,
                                                             g->lend[s], e->fail.p, t);
      LAUNCHED();
      WSrc w;
      w.src = e->lw.p + (size_t)par * ns;
      w.M = e->mbuf.p + par;
      w.mode = 0;
      if (g->rank_on) {
        RankOut ro{g->gcut[s], g->sfq[s], g->sf32[s], 53 - ilog2(N)};
        cdf_expand_kernel<TQ, true><<<(int)plan.chunks, CDF_THREADS, 0, e->st>>>(
            w, N, plan.R, (TQ*)b.tile_tot.p, (TQ*)b.node.p, (TQ*)b.carry.p, (TQ*)b.total.p, (TQ*)g->gq[s],
            g->gcut[s], e->fail.p, ro, (int64_t)s * ns);
        LAUNCHED();
        group_build_shard_kernel<<<grid_for(ns / GRP_STRATA, 256, sms * 8), 256, 0, e->st>>>(
            g->gcut[s], g->lend[s], s, G, N, g->sgrp[s], e->fail.p);
      } else {
        cdf_expand_kernel<TQ, false><<<(int)plan.chunks, CDF_THREADS, 0, e->st>>>(
            w, N, plan.R, (TQ*)b.tile_tot.p, (TQ*)b.node.p, (TQ*)b.carry.p, (TQ*)b.total.p, (TQ*)g->gq[s],
            g->gcut[s], e->fail.p, RankOut(), (int64_t)s * ns);
      }
      LAUNCHED();
      CK(cudaEventRecord(g->evC[s], e->st));
      if (ntg) {
        // windows of step t need shard 0's combine and the predictor of t-1
        CK(cudaStreamWaitEvent(e->side, g->evC[s], 0));
        CK(cudaStreamWaitEvent(e->side, g->evM, 0));
        if (t > 1) CK(cudaStreamWaitEvent(e->side, e0->ev_q[(t - 1) & 1], 0));
        QArgs q2 = qa;
        q2.sh = e0->qsh.p + par;
        uint32_t* kb = e->keys.p + (size_t)par * 3 * ns;
        q2.keys[0] = want_fq ? kb : nullptr;
        q2.keys[1] = want_sq ? kb + ns : nullptr;
        q2.keys[2] = want_tq ? kb + 2 * (size_t)ns : nullptr;
        q2.pbase = s * cls_grid;
        q2.ptotal = G * cls_grid;
        q2.gbase = (uint32_t)((int64_t)s * ns);
        if ((rc = launch_classify<TQ>(qm, cls_grid, w, (int)plan.tiles, e->fail.p, q2, e->side)) != PF_OK)
          return rc;
        CK(cudaEventRecord(g->evK[s], e->side));
      }
    }
    // ---- exact resolve on shard 0's side stream
    if (ntg) {
      if ((rc = set_device(g->dev[0])) != PF_OK) return rc;
      cudaStream_t ss = e0->side;
      if ((rc = wait_all(ss, g->evK)) != PF_OK) return rc;
      qa.sh = e0->qsh.p + par;
      QValueSrc vs;
      memset(&vs, 0, sizeof(vs));
      vs.nsh = G;
      vs.lg = g->lg;
      for (int h = 0; h < G; ++h) vs.recs[h] = g->sh[h]->rec[cur].p;
      vs.seed = c.seed;
      vs.t = t;
      vs.gs = shard_gamma(e0, true, t);
      vs.feed_gs = nullptr;
      vs.sigma2_fixed = c.sigma2_fixed;
      vs.tau2_fixed = c.tau2_fixed;
      vs.learn_s = LS;
      vs.learn_t = LT;
      double *ox = e0->o_fq.p, *os = e0->o_sq.p, *ot = e0->o_tq.p;
      const int hgrid = std::max(1, std::min(64, (int)((N / 64 + 255) / 256)));
      static DevOnce resolve_attr;
      if (resolve_attr.pending()) {
        CK(cudaFuncSetAttribute(q_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Q_RESOLVE_SMEM));
        resolve_attr.mark();
      }
      const int fb_grid = grid_for(ns, 256, sms * 2);
      for (int round = 0; round < 2; ++round) {
        q_hist_kernel<<<dim3(hgrid, ntg), 256, 0, ss>>>(qa, e0->fail.p, round);
        q_locate_kernel<<<ntg, 1024, 0, ss>>>(qa, e0->fail.p, round);
        q_filter_kernel<<<dim3(hgrid, ntg), 256, 0, ss>>>(qa, e0->fail.p);
        q_finish_kernel<<<ntg, 1024, Q_RESOLVE_SMEM, ss>>>(qa, vs, ox, os, ot, t, e0->fail.p);
        g_launches.fetch_add(4);
        if (round == 0) {
          for (int attempt = 0; attempt < 2; ++attempt) {
            if ((rc = fb_hist_smem()) != PF_OK) return rc;
          q_fallback_prep_kernel<<<1, 32, 0, ss>>>(qa, attempt, e0->fail.p);
            for (int s = 0; s < G; ++s) {  // every shard's particles (peer reads)
              pf_engine* e = g->sh[s];
              QArgs q2 = qa;
              uint32_t* kb = e->keys.p + (size_t)par * 3 * ns;
              q2.keys[0] = want_fq ? kb : nullptr;
              q2.keys[1] = want_sq ? kb + ns : nullptr;
              q2.keys[2] = want_tq ? kb + 2 * (size_t)ns : nullptr;
              q2.pbase = s * fb_grid;
              q2.ptotal = G * fb_grid;
              q2.gbase = (uint32_t)((int64_t)s * ns);
              q_fallback_hist_kernel<<<fb_grid, 256, QFB_SMEM_BYTES, ss>>>(q2, e->lw.p + (size_t)par * ns, 0, e->mbuf.p + par, ns,
                                                              SINGLE, attempt, e0->fail.p);
            }
            q_fallback_select_kernel<<<ntg, 1024, 0, ss>>>(qa, attempt, e0->fail.p);
            g_launches.fetch_add(2 + G);
          }
          for (int s = 0; s < G; ++s) {
            pf_engine* e = g->sh[s];
            QArgs q2 = qa;
            uint32_t* kb = e->keys.p + (size_t)par * 3 * ns;
            q2.keys[0] = want_fq ? kb : nullptr;
            q2.keys[1] = want_sq ? kb + ns : nullptr;
            q2.keys[2] = want_tq ? kb + 2 * (size_t)ns : nullptr;
            q2.gbase = (uint32_t)((int64_t)s * ns);
            q_fallback_fill_kernel<<<fb_grid, 256, 0, ss>>>(q2, e->lw.p + (size_t)par * ns, 0, e->mbuf.p + par, ns,
                                                            SINGLE, e0->fail.p);
          }
          g_launches.fetch_add(G);
        }
      }
      QAll all;
      memset(&all, 0, sizeof(all));
      all.nsrc = G;
      all.ns = ns;
      for (int s = 0; s < G; ++s) {
        pf_engine* e = g->sh[s];
        uint32_t* kb = e->keys.p + (size_t)par * 3 * ns;
        all.keys[s][0] = want_fq ? kb : nullptr;
        all.keys[s][1] = want_sq ? kb + ns : nullptr;
        all.keys[s][2] = want_tq ? kb + 2 * (size_t)ns : nullptr;
        all.lw[s] = e->lw.p + (size_t)par * ns;
        all.M[s] = e->mbuf.p + par;
      }
      all.single = SINGLE;
      q_select_kernel<<<ntg, 1024, 0, ss>>>(qa, vs, e0->qscratch.p, ox, os, ot, t, e0->fail.p, e0->qunres.p, all);
      q_step_end_kernel<<<1, 1024, 0, ss>>>(qa, 1);
      g_launches.fetch_add(2);
      CK(cudaEventRecord(e0->ev_q[t & 1], ss));
    }
  }

  // ---- final resample (keep_indices row T, keep_final) per shard
  for (int s = 0; s < G; ++s) {
    pf_engine* e = g->sh[s];
    if ((rc = set_device(g->dev[s])) != PF_OK) return rc;
    cudaStream_t st = e->st;
    if (T >= 1 && (keep_idx || keep_final)) {
      if ((rc = wait_all(st, g->evC)) != PF_OK) return rc;
      // ancestors of the last resample through the cross-shard lookup: a
      // one-step StepArgs-free path (materialize with the sharded lookup)
      GroupMatArgs<TQ> m;
      memset(&m, 0, sizeof(m));
      m.ns = ns;
      m.gbase = (int64_t)s * ns;
      m.t = T;
      m.seed = c.seed;
      m.u3 = e->du3.p + (size_t)(T & 1) * ns;
      if (spacings) {
        spacings_words_kernel<<<grid_for(ns, 256), 256, 0, st>>>(e->spS.p, ns, e->sptot.p + (size_t)(T & 1) * PF_MAX_SHARDS,
                                                                 G, s, c.seed, T, e->spw.p, e->fail.p);
        LAUNCHED();
        m.u3 = e->spw.p;
      }
      m.slk.G = G;
      m.slk.lg = g->lg;
      m.slk.n = N;
      m.slk.lend = g->lend[s];
      for (int h = 0; h < G; ++h) {
        m.slk.cut[h] = g->gcut[h];
        m.slk.q[h] = (const TQ*)g->gq[h];
        m.recs[h] = g->sh[h]->rec[cur].p;
      }
      m.gs = shard_gamma(e, true, T);
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
      group_materialize_kernel<TQ><<<grid_for(ns, 256), 256, 0, st>>>(m);
      LAUNCHED();
      if (keep_idx)
        CK(cudaMemcpyAsync(out->indices + (size_t)(T - 1) * N + (size_t)s * ns, e->idx.p, ns * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, st));
      for (int k = 0; k < 7; ++k)
        if (*slots[k])
          CK(cudaMemcpyAsync(dst[k] + (size_t)s * ns, *slots[k], ns * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
  }

  // ---- outputs (shard 0) and status of every shard
  if ((rc = set_device(g->dev[0])) != PF_OK) return rc;
  cudaStream_t s0 = e0->st;
  if (ntg) {
    CK(cudaStreamWaitEvent(s0, e0->ev_q[0], 0));
    CK(cudaStreamWaitEvent(s0, e0->ev_q[1], 0));
  }
  for (int s = 1; s < G; ++s) {
    CK(cudaEventRecord(g->evD[s], g->sh[s]->st));
    CK(cudaStreamWaitEvent(s0, g->evD[s], 0));
  }
  if (out && T > 0) {
    auto cp = [&](double* h, DevBuf<double>& d, size_t cnt) -> int {
      if (h) CK(cudaMemcpyAsync(h, d.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, s0));
      return PF_OK;
    };
    if ((rc = cp(out->filtered_mean, e0->o_fm, T)) != PF_OK) return rc;
    if (out->ess && (rc = cp(out->ess, e0->o_ess, T)) != PF_OK) return rc;
    if (want_fq && (rc = cp(out->filtered_quantiles, e0->o_fq, T * 3)) != PF_OK) return rc;
    if (LS && ((rc = cp(out->sigma2_mean, e0->o_sm, T)) || (rc = cp(out->sigma2_sd, e0->o_ssd, T)) ||
               (rc = cp(out->sigma2_quantiles, e0->o_sq, T * 5))))
      return rc;
    if (LT && ((rc = cp(out->tau2_mean, e0->o_tm, T)) || (rc = cp(out->tau2_sd, e0->o_tsd, T)) ||
               (rc = cp(out->tau2_quantiles, e0->o_tq, T * 5))))
      return rc;
  }
  CK(cudaEventRecord(e0->ev1, s0));
  int64_t fail_h = 0;
  for (int s = 0; s < G; ++s) {
    if ((rc = set_device(g->dev[s])) != PF_OK) return rc;
    int64_t f = 0;
    CK(cudaMemcpyAsync(&f, g->sh[s]->fail.p, sizeof(int64_t), cudaMemcpyDeviceToHost, g->sh[s]->st));
    CK(cudaStreamSynchronize(g->sh[s]->st));
    CK(cudaStreamSynchronize(g->sh[s]->side));
    CK(cudaStreamSynchronize(g->sh[s]->dstream));
    if (f && !fail_h) fail_h = f;
  }
  CK(cudaGetLastError());
  float ms = 0;
  cudaSetDevice(g->dev[0]);
  cudaEventElapsedTime(&ms, e0->ev0, e0->ev1);
  g->last_ms = ms;
  if (out) {
    for (int k = 0; k < 7; ++k) out->phase_ns[k] = 0;
    out->phase_ns[6] = (int64_t)llround(ms * 1e6);
    out->failed_step = fail_h;
  }
  if (fail_h > 0)
    return set_err(PF_ERR_ALL_WEIGHTS_ZERO,
                   "all particle weights are zero (at time step " + std::to_string(fail_h) + ")", fail_h);
  if (fail_h < 0) return set_err(PF_ERR_ALL_WEIGHTS_ZERO, "all particle weights are zero", 0);
  if (ntg) {
    if ((rc = set_device(g->dev[0])) != PF_OK) return rc;
    if ((rc = check_quantile_unresolved(e0->qunres.p)) != PF_OK) return rc;
  }
  return PF_OK;
}

using GroupRunFn = int (*)(pf_group*, const double*, int64_t, pf_outputs*);

GroupRunFn pick_group_run(int mode) {
  switch (mode) {
    case 0: return run_group<0, double>;
    case 1: return run_group<1, double>;
    case 2: return run_group<2, double>;
    case 3: return run_group<3, double>;
    case 4: return run_group<4, float>;
    case 5: return run_group<5, float>;
    case 6: return run_group<6, float>;
    case 7: return run_group<7, float>;
  }
  return nullptr;
}

}  // namespace
