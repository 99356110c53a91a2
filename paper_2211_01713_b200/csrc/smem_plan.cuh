// smem_plan.cuh -- one plan per CTA with the scenario's search state in shared
// memory (single plans of up to about 1,900 workloads: BASELINE C1/C2).
//
// A single plan is a chain of m dependent steps (planner.py:290-319); the
// per-step latency is what a user waits for.  k_place<.., 8> keeps the state in
// global memory and lets each lane run one candidate's Alg. 2 serially, so a
// step costs several L2 round trips plus the slowest candidate's chain of
// Neumaier folds.  Here:
//   * the open GPUs' check terms live in shared memory, keyed by placement
//     index k (every workload is a resident of exactly one GPU): CRec / CNext
//     of fast.cuh, the committed units, a per-GPU header with the power and
//     cache sums, the pool's resident lists (pool index -> k) and the slack
//     order (sj / spos / sdesc / sE) that commit_step maintains;
//   * one WARP evaluates one candidate: lane i holds resident i (lane n the
//     newcomer), an evaluation is O(1) per lane (fast.cuh's certified-margin
//     test), and the pass order of Alg. 2 (planner.py:152-161: the first
//     violating resident from the current position is bumped, then the device
//     is re-evaluated) is a ballot and a find-first-set;
//   * a decision inside the margin, a GPU with 32 or more residents, or a
//     power sum the frequency screen rejects runs exact_candidate (fast.cuh)
//     on lane 0 -- the exact evaluation sequence;
//   * the commit is commit_step (place.cuh) on the shared-memory slack order
//     and the global full records (which the exact fallback and the
//     _build_plan predictions read), then the committed GPU's compact terms
//     are rebuilt from those records.
// The plan and the predictions are written by k_place (Hand hand-off, as for
// the cooperative kernel).  Scenarios that need the exact sequence (PlanStats,
// an input that can raise, a prologue error) or fail a screen are declined.
#pragma once

namespace igp {

#ifndef IGP_SMEM_WARPS
#define IGP_SMEM_WARPS 16
#endif
constexpr int SMEM_WARPS = IGP_SMEM_WARPS;

struct SmemLayout {
  size_t cr, cn, hd, gst, sdesc, sj, spos, su, spool, sE, total;
};

__host__ __device__ inline size_t sm_align(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline SmemLayout smem_layout(int m, long long pool_recs, int cap) {
  SmemLayout L;
  const size_t mm = (size_t)(m > 0 ? m : 1);
  size_t o = 0;
  L.cr = o; o = sm_align(o + mm * sizeof(CRec));
  L.cn = o; o = sm_align(o + mm * sizeof(CNext));
  L.hd = o; o = sm_align(o + mm * sizeof(CHead));
  L.gst = o; o = sm_align(o + mm * 8);
  L.sdesc = o; o = sm_align(o + mm * 8);
  L.sj = o; o = sm_align(o + mm * 4);
  L.spos = o; o = sm_align(o + mm * 4);
  L.su = o; o = sm_align(o + mm * 2);
  L.spool = o; o = sm_align(o + (size_t)pool_recs * 2);
  L.sE = o; o = sm_align(o + (size_t)(cap + 2) * 4);
  L.total = o;
  return L;
}

struct __align__(16) SmemNew {  // one step's newcomer: its check record, constants, solo row
  double nw[R_NF];
  double cold[C_NF];
  double ntab[TB * 4];
};

struct SmemCtl {
  SmemNew nb[2];  // double-buffered: step k+1's newcomer arrives during step k
  unsigned best[2];  // step k's argmin key in best[k & 1]
  unsigned wbest[SMEM_WARPS];  // each warp's best key (its row holds the unit vector)
  int pool_top, abort_code;
};

// Step k's newcomer into buffer b: 42 LDGSTS of 16 bytes (threads 0..41).
__device__ __forceinline__ void smem_fetch_newcomer(SmemNew &b, const double *nwt, const double *cold,
                                                    const double *tbl, int k, int t) {
  constexpr int C1 = R_NF * 8 / 16, C2 = C1 + C_NF * 8 / 16, C3 = C2 + TB * 4 * 8 / 16;
  if (t < C1) cp_async16(b.nw + 2 * t, nwt + (size_t)k * R_NF + 2 * t);
  else if (t < C2) cp_async16(b.cold + 2 * (t - C1), cold + (size_t)k * C_NF + 2 * (t - C1));
  else if (t < C3) cp_async16(b.ntab + 2 * (t - C2), tbl + (size_t)k * TB * 4 + 2 * (t - C2));
  cp_async_commit();
}

// fmax / f to ~1e-15 relative: the fast path only needs the value, not the
// IEEE quotient (two Newton steps on the fp32 reciprocal)
__device__ __forceinline__ double approx_inv(double fmax, double f) {
  double r = (double)__frcp_rn((float)f);
  r = r * (2.0 - f * r);
  r = r * (2.0 - f * r);
  return fmax * r;
}

// The compact terms of the residents of GPU j (after commit_step), keyed by
// placement index, from the full records in global memory.
__device__ __forceinline__ void smem_compact(const ScenState &Z, CRec *cr, CNext *cn, CHead *hd,
                                             uint16_t *su, const uint16_t *spool,
                                             const unsigned long long *gst, int j, int lane) {
  const unsigned long long g = gst[j];
  const int n = (int)((g >> 16) & 0xffffu), off = (int)(g >> 32);
  if (lane == 0) {
    const double *gf = Z.gfold + (size_t)j * 4;
    CHead h;
    h.P = __ldcg(gf) + __ldcg(gf + 1);
    h.C = __ldcg(gf + 2) + __ldcg(gf + 3);
    hd[j] = h;
  }
  for (int r = lane; r < n; r += 32) {
    const int kk = spool[off + r];
    const double *rr = Z.rec + (size_t)(off + r) * R_NF;
    const double ka = __ldcg(rr + R_KA), ca = __ldcg(rr + R_CA), tsn = __ldcg(rr + R_TSN);
    const double ac = __ldcg(rr + R_ACACHE), pw = __ldcg(rr + R_PW);
    CRec c;
    c.A = tsn + ka;
    c.B = ka * ac;
    c.ca = ca;
    c.beta = fast_beta(__ldcg(rr + R_THALF), __ldcg(rr + R_TLOAD), __ldcg(rr + R_TFB));
    cr[kk] = c;
    const double *nx = Z.nxt + (size_t)(off + r) * 4;
    const double ka1 = __ldcg(nx), pw1 = __ldcg(nx + 1), ca1 = __ldcg(nx + 2);
    CNext q;
    q.A1 = tsn + ka1;
    q.B1 = ka1 * ac;
    q.dca = ca1 - ca;
    q.dpw = pw1 - pw;
    cn[kk] = q;
    const unsigned long long mv = __ldcg(reinterpret_cast<const unsigned long long *>(Z.meta + off + r));
    su[kk] = reinterpret_cast<const Meta *>(&mv)->u;
  }
}

template <int MAXN>
__global__ void __launch_bounds__(SMEM_WARPS * 32, 1) k_plan_smem(PlanParams P) {
  constexpr unsigned NO_KEY = 0xffffffffu;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ SmemCtl ctl;
  const int t = threadIdx.x, lane = t & 31, wi = t >> 5;
  const int s = blockIdx.x;
  Hand *const hdp = P.hand + s;
  const Hw &hw = P.hw;
  const int m = P.m, cap = hw.cap;
  if (P.perr[s] != INT_MAX || P.sflags[s] != 0 || !hw.margin_ok) {
    if (t == 0) hdp->k_done = P.k0;  // declined: k_place plans it
    return;
  }
  const SmemLayout SL = smem_layout(m, P.pool_recs, P.cap_ld);
  CRec *const cr = reinterpret_cast<CRec *>(dsm + SL.cr);
  CNext *const cn = reinterpret_cast<CNext *>(dsm + SL.cn);
  CHead *const hd = reinterpret_cast<CHead *>(dsm + SL.hd);
  unsigned long long *const gst = reinterpret_cast<unsigned long long *>(dsm + SL.gst);
  unsigned long long *const sdesc = reinterpret_cast<unsigned long long *>(dsm + SL.sdesc);
  int32_t *const sj = reinterpret_cast<int32_t *>(dsm + SL.sj);
  int32_t *const spos = reinterpret_cast<int32_t *>(dsm + SL.spos);
  uint16_t *const su = reinterpret_cast<uint16_t *>(dsm + SL.su);
  uint16_t *const spool = reinterpret_cast<uint16_t *>(dsm + SL.spool);
  int32_t *const sE = reinterpret_cast<int32_t *>(dsm + SL.sE);

  const size_t sm = (size_t)s * m;
  const double *cold = P.cold + sm * C_NF;
  const double *nwt = P.nw + sm * R_NF;
  const double *tbl = P.tbl + sm * TB * 4;
  const size_t sp = (size_t)s * (size_t)P.pool_recs;
  const ScenState Z{cold, tbl, gst, sdesc, sj, spos, sE, P.gcap + sm, P.gfold + sm * 4,
                    P.rec + sp * R_NF, P.nxt + sp * 4, P.frec + sp * 2, P.pfx + sp * 4,
                    P.meta + sp, sm};
  uint16_t *const rows = P.lane_units + (size_t)s * P.lanes * P.cap_ld;
  uint16_t *const my_row = rows + (size_t)wi * cap;
  for (int x = t; x < cap + 2; x += blockDim.x) sE[x] = 0;
  if (t == 0) {
    ctl.pool_top = 0;
    ctl.abort_code = 0;
  }
  int G = 0;
  unsigned long long evals = 0, cands = 0, exact = 0;
  const double delta = P.fast_delta;
  smem_fetch_newcomer(ctl.nb[P.k0 & 1], nwt, cold, tbl, P.k0, t);
  if (t == 0) ctl.best[0] = ctl.best[1] = NO_KEY;
  cp_async_wait_all();
  __syncthreads();
  for (int k = P.k0; k < P.k1; ++k) {
#if IGP_TIMING
    const long long tm0 = clock64();
#endif
    // ---- the newcomer (planner.py:291-292): staged during the previous step ----
    if (k + 1 < P.k1) smem_fetch_newcomer(ctl.nb[(k + 1) & 1], nwt, cold, tbl, k + 1, t);
    const SmemNew &NB = ctl.nb[k & 1];
    unsigned *const bestp = &ctl.best[k & 1];
#if IGP_TIMING
    const long long tm1 = clock64();
#endif
    const int need = (int)NB.cold[C_LB];
    const double n_ka = NB.nw[R_KA], n_ca = NB.nw[R_CA], n_pw = NB.nw[R_PW];
    const double n_ac = NB.nw[R_ACACHE];
    const double n_beta = fast_beta(NB.nw[R_THALF], NB.nw[R_TLOAD], NB.nw[R_TFB]);
    const double ksch = NB.cold[C_KSCH], nkern = NB.cold[C_NK];
    const int ncand = sE[need];
    unsigned w_best = NO_KEY;  // this warp's best key (its row holds the unit vector)

    // ---- candidates: one warp each (planner.py:296-311) ----
    for (int c = wi; c < ncand; c += SMEM_WARPS) {
      const int j = sj[c];
      const unsigned long long g = sdesc[c];
      if ((((unsigned)need << 23) | (unsigned)j) > *(volatile unsigned *)bestp) continue;
      cands += lane == 0;
      const int occ = (int)(g & 0xffffu), n = (int)((g >> 16) & 0xffffu), off = (int)(g >> 32);
      int sum = occ + need;
      bool go_exact = n >= 32;
      unsigned key = NO_KEY;
      if (!go_exact) {
        // lane i: resident i (placement index kk), lane n: the newcomer
        const bool act = lane <= n;
        const int kk = lane < n ? (int)spool[off + lane] : -1;
        double A = 0.0, B = 0.0, ca = 0.0, beta = 0.0;
        int u = 0;
        if (lane < n) {
          const CRec r = cr[kk];
          A = r.A;
          B = r.B;
          ca = r.ca;
          beta = r.beta;
          u = su[kk];
        } else if (lane == n) {
          A = (ksch + delta_sch(hw, n + 1)) * nkern + n_ka;
          B = n_ka * n_ac;
          ca = n_ca;
          beta = n_beta;
          u = need;
        }
        double cur_pw = n_pw, cur_ca = n_ca;  // the newcomer's current solo terms
        const CHead h = hd[j];
        double C = h.C + n_ca, Pd = (hw.pidle + h.P) + n_pw;
        int bumps = 0, ci = 0;
        bool flag = false, done = false;
        while (!done) {
          // the device terms (model.py:299-305), O(1) from the sums
          const double f = frequency(hw, Pd);
          const double inv = f == hw.fmax ? 1.0 : approx_inv(hw.fmax, f);
          evals += lane == 0;
          if (!(fabs(hw.af) * fabs(Pd) < 2048.0 * f)) {
            go_exact = true;
            break;
          }
          bool again = true;
          while (again) {  // passes over the same evaluation
            again = false;
            const double d = (A + B * (C - ca)) * inv - beta;
            const bool unc = act && !(fabs(d) > delta * beta);
            const bool vio = act && !unc && d > 0.0;
            const unsigned from = ~((1u << ci) - 1u);
            const unsigned ub = __ballot_sync(FULL, unc) & from, vb = __ballot_sync(FULL, vio) & from;
            const unsigned any = ub | vb;
            if (!any) {  // the rest of the pass is clean
              if (flag) {  // planner.py:147: another pass after a bump
                ci = 0;
                flag = false;
                again = true;
                continue;
              }
              key = ((unsigned)(sum - occ) << 23) | (unsigned)j;  // feasible
              done = true;
              break;
            }
            const int i = __ffs(any) - 1;
            if ((ub >> i) & 1u) {  // inside the margin: the exact sequence decides
              go_exact = true;
              done = true;
              break;
            }
            // t_inf > t_half (planner.py:158): bump resident i
            sum += 1;
            if (sum > cap || ((((unsigned)(sum - occ)) << 23) | (unsigned)j) >
                                 *(volatile unsigned *)bestp) {
              done = true;  // infeasible or pruned
              break;
            }
            double dC = 0.0, dP = 0.0;
            if (lane == i) {
              u += 1;
              if (i == n) {  // the newcomer, from its solo table row
                const int v = u - need;
                Solo so;
                if (v < TB && u <= cap) {
                  so.ka = NB.ntab[v * 4];
                  so.pw = NB.ntab[v * 4 + 1];
                  so.ca = NB.ntab[v * 4 + 2];
                } else {
                  so = solo_from_cold(cold + (size_t)k * C_NF, (double)u * hw.runit);
                }
                A = (ksch + delta_sch(hw, n + 1)) * nkern + so.ka;
                B = so.ka * n_ac;
                dC = so.ca - cur_ca;
                dP = so.pw - cur_pw;
                ca = so.ca;
                cur_ca = so.ca;
                cur_pw = so.pw;
              } else if (bumps == 0) {  // one unit above the committed units
                const CNext q = cn[kk];
                A = q.A1;
                B = q.B1;
                ca += q.dca;
                dC = q.dca;
                dP = q.dpw;
              } else {  // further bumps: the solo table at the new units
#if IGP_TIMING
                if (s == 0 && P.stats) atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 4], 1ull);
#endif
                const Meta mt = Z.meta[off + i];
                const Solo so = solo_lookup(tbl, cold, hw, mt.k, mt.lb, u);
                const Solo s0 = solo_lookup(tbl, cold, hw, mt.k, mt.lb, u - 1);
                const double *rr = Z.rec + (size_t)(off + i) * R_NF;
                A = rr[R_TSN] + so.ka;
                B = so.ka * rr[R_ACACHE];
                ca = so.ca;
                dC = so.ca - s0.ca;
                dP = so.pw - s0.pw;
              }
              bumps += 1;
            }
            C += __shfl_sync(FULL, dC, i);
            Pd += __shfl_sync(FULL, dP, i);
            flag = true;
            ci = i + 1;
            if (ci > n) {  // the pass ended on a bump: another pass
              ci = 0;
              flag = false;
            }
            break;  // re-evaluate (planner.py:161: rows = None)
          }
        }
        if (!go_exact && key != NO_KEY && key < w_best) {
          w_best = key;
          if (act) my_row[lane] = (uint16_t)u;
        }
      }
#if IGP_TIMING
      if (s == 0 && P.stats && lane == 0) {
        atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 5], 1ull);
      }
#endif
      if (go_exact) {  // the exact evaluation sequence, on lane 0
        unsigned long long ev = 0;
        int xs = cap + 1;
        if (lane == 0) {
          exact += 1;
          xs = exact_candidate<MAXN>(hw, Z, NB.nw, ksch, nkern, need, k, j, occ, n, off,
                                     (const volatile unsigned *)bestp, w_best, my_row, ev);
          evals += ev;
        }
        xs = __shfl_sync(FULL, xs, 0);
        key = xs <= cap ? (((unsigned)(xs - occ) << 23) | (unsigned)j) : NO_KEY;
        if (key < w_best) w_best = key;
      }
      if (key != NO_KEY && lane == 0) atomicMin(bestp, key);
      __syncwarp();
    }
    if (lane == 0) ctl.wbest[wi] = w_best;
    __syncthreads();
#if IGP_TIMING
    const long long tm2 = clock64();
#endif
    const unsigned bk = *bestp;
#if IGP_TIMING
    const long long tm3 = clock64();
#endif
    // ---- commit (planner.py:312-319), warp 0 ----
    if (wi == 0) {
      const int jj = bk == NO_KEY ? G : (int)(bk & 0x7fffffu);
      const int nres = bk == NO_KEY ? 0 : (int)((gst[jj] >> 16) & 0xffffu);
      const int off0 = bk == NO_KEY ? 0 : (int)(gst[jj] >> 32);
      const unsigned wb = lane < SMEM_WARPS ? ctl.wbest[lane] : NO_KEY;
      const unsigned hit = __ballot_sync(FULL, bk != NO_KEY && wb == bk);
      const uint16_t *lu_w = bk != NO_KEY ? rows + (size_t)(__ffs(hit) - 1) * cap : nullptr;
      commit_step(P, hw, Z, k, need, bk, lu_w, G, &ctl.pool_top, &ctl.abort_code, NB.nw, ksch,
                  nkern, lane);
      __syncwarp();
      if (!*(volatile int *)&ctl.abort_code) {
        // the resident lists follow the tile (moved when it grew)
        const int off1 = (int)(gst[jj] >> 32);
        if (off1 != off0)
          for (int r = lane; r < nres; r += 32) spool[off1 + r] = spool[off0 + r];
        if (lane == 0) spool[off1 + nres] = (uint16_t)k;
        __syncwarp();
        __threadfence_block();
        smem_compact(Z, cr, cn, hd, su, spool, gst, jj, lane);
      }
    }
    if (bk == NO_KEY) G += 1;
    if (t == 0) ctl.best[(k + 1) & 1] = NO_KEY;  // nobody reads it during step k
    cp_async_wait_all();  // step k+1's newcomer
    __syncthreads();
#if IGP_TIMING
    if (s == 0 && t == 0 && P.stats) {  // phase cycles of scenario 0
      const long long tm4 = clock64();
      atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S], (unsigned long long)(tm1 - tm0));
      atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 1], (unsigned long long)(tm2 - tm1));
      atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 2], (unsigned long long)(tm3 - tm2));
      atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 3], (unsigned long long)(tm4 - tm3));
    }
#endif
    if (ctl.abort_code) break;
  }
  // ---- hand the scenario to k_place, which writes the plan ----
  unsigned long long *gs_out = P.gstate + (size_t)s * P.gstride;
  for (int x = t; x < G; x += blockDim.x) gs_out[x] = gst[x];
  __shared__ unsigned long long tot[3];
  if (t == 0) tot[0] = tot[1] = tot[2] = 0;
  __syncthreads();
  if (lane == 0) {
    atomicAdd(&tot[0], evals);
    atomicAdd(&tot[1], cands);
    atomicAdd(&tot[2], exact);
  }
  __syncthreads();
  if (t == 0) {
    hdp->G = G;
    hdp->pool_top = ctl.pool_top;
    hdp->abort = ctl.abort_code;
    hdp->evals_run = tot[0];
    hdp->cands_run = tot[1];
    hdp->exact_run = tot[2];
    __threadfence();
    hdp->k_done = P.k1;
  }
}

}  // namespace igp
