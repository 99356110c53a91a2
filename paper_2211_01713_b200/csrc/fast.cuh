// fast.cuh -- the certified-margin fast path of the batch placement kernel.
//
// The reference's step (planner.py:290-319) only ever USES the latency model
// through decisions: `t_inf > t_half` (planner.py:158) bumps a unit, and the
// unit sums decide feasibility and the argmin.  A candidate's result -- its
// unit vector, hence its key (inter << 23 | j) -- is therefore determined by
// the sequence of those decisions alone.  This kernel takes every decision
// from a cheap approximation of t_inf together with a rigorous error bound;
// only when a value falls inside the bound (|t - beta| <= delta * beta) does
// the candidate fall back to the exact evaluation (CPython operation order,
// Neumaier sums: exact_candidate below).  Every decision taken on the fast
// side is therefore the exact one and the plan is the reference's bit for
// bit; the _build_plan rows are computed exactly afterwards (k_place's
// predict phase).
//
// Per candidate, Alg. 2 (planner.py:133-162) becomes
//   C  = cache sum of the GPU (header) + newcomer     P = power sum + newcomer
//   f  = frequency(idle + P), inv = fmax / f       (model.py:300-305)
//   resident i:  t = (A_i + B_i * (C - ca_i)) * inv  vs  beta_i
// with A = t_sch + k_act, B = k_act * alpha_cache, beta = t_half - t_load - t_fb
// (model.py:308-313: t_inf > t_half  <=>  t_gpu > beta in real arithmetic).
// A bump moves the resident to its next-unit terms (CNext, precomputed at the
// commit) and adds exact fp64 deltas to C and P: an evaluation is O(1) instead
// of the O(n) Neumaier folds, and a candidate's tile is 32 B per resident
// instead of 64.
//
// Error bound.  A, B, ca, beta and the sums are fp64 values that differ from
// the exact evaluation's only in association and in the Neumaier
// compensation: with every term non-negative (the SF_NO_MARGIN screen) and
// alpha_cache <= 16 (the SF_NO_FAST screen) the approximate t is within about
// 1e-13 relative of the real t_gpu (accumulated sum deltas included), and
// the exact fp64 evaluation is within 1e-15 t_half of real arithmetic.
// beta is used only when beta > t_half / 4096 (else NaN: every test on it is
// "uncertain"), so a test with |t - beta| > 2^-30 beta (>= 2^-42 t_half) has
// the sign of the exact decision.  The frequency's sensitivity to the power
// sum is screened per evaluation (|alpha_f| |P| < 2048 f).
#pragma once

namespace igp {

constexpr double FAST_DELTA = 0x1p-30;    // decision margin, relative to beta
enum { R_EXACT = 4 };

__device__ __forceinline__ double fast_beta(double thalf, double tload, double tfb) {
  const double b = (thalf - tload) - tfb;
  return (b > thalf * 0x1p-12 && b < 1e300) ? b : __longlong_as_double(0x7ff8000000000000ll);
}

// The compact tile of GPU j from its full records (after commit_step).
__device__ __forceinline__ void write_compact(const ScenState &Z, CRec *crec, CNext *cnext, int j,
                                              int lane) {
  const unsigned long long g = Z.gstate[j];
  const int n = (int)((g >> 16) & 0xffffu), off = (int)(g >> 32);
  if (lane == 0) {
    const double *gf = Z.gfold + (size_t)j * 4;
    CHead h;
    h.P = gf[0] + gf[1];
    h.C = gf[2] + gf[3];
    // the 16 bytes just before the first record: one contiguous copy stages both
    *reinterpret_cast<CHead *>(reinterpret_cast<char *>(crec + off) - sizeof(CHead)) = h;
  }
  for (int r = lane; r < n; r += 32) {
    const double *rr = Z.rec + (size_t)(off + r) * R_NF;
    const double ka = rr[R_KA], ca = rr[R_CA], tsn = rr[R_TSN], ac = rr[R_ACACHE];
    CRec c;
    c.A = tsn + ka;
    c.B = ka * ac;
    c.ca = ca;
    c.beta = fast_beta(rr[R_THALF], rr[R_TLOAD], rr[R_TFB]);
    crec[off + r] = c;
    const double *nx = Z.nxt + (size_t)(off + r) * 4;  // k_act, power, cache one unit up
    CNext q;
    q.A1 = tsn + nx[0];
    q.B1 = nx[0] * ac;
    q.dca = nx[2] - ca;
    q.dpw = nx[1] - rr[R_PW];
    cnext[off + r] = q;
  }
}

// Alg. 2 (planner.py:146-162) for GPU j plus the newcomer, in the exact
// evaluation order of k_place (fold from the cached prefix states, the
// division shortcut's margin test): the fallback of an uncertain decision.
// Stops at Sum u > cap or once its key exceeds *thr.  Returns the final Sum u
// (> cap: infeasible or pruned); on a feasible key below *my_best the unit
// vector (residents, then the newcomer) goes to lu.
template <int MAXN>
__device__ __noinline__ int exact_candidate(const Hw &hw, const ScenState &Z, const double *nw,
                                            double ksch, double nkern, int need, int kk, int j,
                                            int occ, int nres, int off, const volatile unsigned *thr,
                                            unsigned my_best, uint16_t *lu,
                                            unsigned long long &evals) {
  const int cap = hw.cap;
  double ka[MAXN + 1], pw[MAXN + 1], ca[MAXN + 1];
  int u[MAXN + 1];
  for (int q = 0; q < nres; ++q) {
    const double *r = Z.rec + (size_t)(off + q) * R_NF;
    ka[q] = r[R_KA];
    ca[q] = r[R_CA];
    pw[q] = r[R_PW];
    u[q] = Z.meta[off + q].u;
  }
  u[nres] = need;
  ka[nres] = nw[R_KA];
  ca[nres] = nw[R_CA];
  pw[nres] = nw[R_PW];
  const double tsn_new = (ksch + delta_sch(hw, nres + 1)) * nkern;
  int sum = occ + need;
  int dirty = nres;  // first resident whose fold terms changed (nres: none)
  while (true) {
    bool bumped = false, need_eval = true, one = true;
    double C = 0.0, f = hw.fmax, inv = 1.0;
    for (int q = 0; q <= nres; ++q) {
      if (need_eval) {  // _eval_entries device terms (model.py:299-305), resident order
        Neumaier fp, fc;
        const double *st =
            dirty == nres ? Z.gfold + (size_t)j * 4 : Z.pfx + (size_t)(off + dirty) * 4;
        fp.s = st[0];
        fp.c = st[1];
        fc.s = st[2];
        fc.c = st[3];
        for (int r = dirty; r < nres; ++r) {
          fp.add(pw[r]);
          fc.add(ca[r]);
        }
        fp.add(pw[nres]);
        fc.add(ca[nres]);
        f = frequency(hw, hw.pidle + fp.result());
        C = fc.result();
        one = f == hw.fmax;
        inv = one ? 1.0 : hw.fmax / f;
        need_eval = false;
        evals += 1;
      }
      double t_sch, acache, t_load, t_fb, t_half;
      if (q == nres) {
        t_sch = tsn_new;
        acache = nw[R_ACACHE];
        t_load = nw[R_TLOAD];
        t_fb = nw[R_TFB];
        t_half = nw[R_THALF];
      } else {
        const double *r = Z.rec + (size_t)(off + q) * R_NF;
        t_sch = r[R_TSN];
        acache = r[R_ACACHE];
        t_load = r[R_TLOAD];
        t_fb = r[R_TFB];
        t_half = r[R_THALF];
      }
      const double x = t_sch + ka[q] * (1.0 + acache * (C - ca[q]));
      double t_gpu = x;  // x / 1.0 == x
      if (!one) {
        t_gpu = x * inv;
        const double tq = (t_load + t_gpu) + t_fb;
        if (!(fabs(tq - t_half) > tq * 0x1p-48 + 0x1p-1000)) t_gpu = x / (f / hw.fmax);
      }
      const double t_inf = (t_load + t_gpu) + t_fb;
      if (t_inf > t_half) {  // planner.py:158: bump, then re-evaluate
        sum += 1;
        if (sum > cap) return sum;
        if ((((unsigned)(sum - occ)) << 23 | (unsigned)j) > *thr) return cap + 1;
        u[q] += 1;
        Solo so;
        if (q == nres) {
          so = solo_lookup(Z.tbl, Z.cold, hw, kk, need, u[q]);
        } else {
          const Meta mt = Z.meta[off + q];
          if (u[q] == (int)mt.u + 1) {  // one unit above the committed units
            const double *nx = Z.nxt + (size_t)(off + q) * 4;
            so.ka = nx[0];
            so.pw = nx[1];
            so.ca = nx[2];
            so.err = (int)nx[3];
          } else {
            so = solo_lookup(Z.tbl, Z.cold, hw, mt.k, mt.lb, u[q]);
          }
        }
        ka[q] = so.ka;
        pw[q] = so.pw;
        ca[q] = so.ca;
        if (q < dirty) dirty = q;
        bumped = true;
        need_eval = true;
      }
    }
    if (!bumped) break;  // a clean pass (planner.py:147)
  }
  const unsigned key = ((unsigned)(sum - occ) << 23) | (unsigned)j;
  if (key < my_best)
    for (int q = 0; q <= nres; ++q) lu[q] = (uint16_t)u[q];
  return sum;
}

#ifndef IGP_FAST_MINB
#define IGP_FAST_MINB 6
#endif
#ifndef IGP_FAST_PF
#define IGP_FAST_PF 1
#endif
#ifndef IGP_FAST_REFILL
#define IGP_FAST_REFILL 28
#endif

struct FastGroup {
  unsigned int best;
  int win_thread, pool_top, abort_code, next;
};

constexpr size_t fast_lane_smem() { return sizeof(FastSlot); }

// One scenario per warp, four per 128-thread CTA, persistent over the batch
// (the scheduling, candidate order, pruning and commit of k_place<.., 1>).
// Scenarios that need the exact sequence (PlanStats, an input that can raise,
// a prologue error) or fail a fast-path screen are declined (Hand.k_done =
// k0) and planned by k_place.
template <int MAXN>
__global__ void __launch_bounds__(128, IGP_FAST_MINB) k_place_fast(PlanParams P) {
  constexpr unsigned NO_KEY = 0xffffffffu;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ FastGroup gsm[4];
  __shared__ __align__(16) double ntb[4][TB * 4];  // the newcomer's solo table row
  __shared__ unsigned long long nbar[4];
  extern __shared__ __align__(16) unsigned char dsm[];
  const int grp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  FastGroup &gs = gsm[grp];
  FastSlot *const sl = reinterpret_cast<FastSlot *>(dsm) + threadIdx.x;
  if (lane == 0) mbar_init(&nbar[grp]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t n_phase = 0;
  const Hw &hw = P.hw;
  const int m = P.m, cap = hw.cap;
  const unsigned lt = (1u << lane) - 1u;
  double *const ntab = ntb[grp];
  const double delta = P.fast_delta;
  for (;;) {
    if (lane == 0) gs.next = atomicAdd(P.sched, 1);
    __syncwarp();
    const int s = gs.next;
    __syncwarp();
    if (s >= P.S) break;
    Hand *const hd = P.hand + s;
    if (P.perr[s] != INT_MAX || P.sflags[s] != 0 || !hw.margin_ok) {
      if (lane == 0) hd->k_done = P.k0;  // declined: k_place plans it
      continue;
    }
    const size_t sm = (size_t)s * m;
    const double *cold = P.cold + sm * C_NF;
    const double *nwt = P.nw + sm * R_NF;
    const double *tbl = P.tbl + sm * TB * 4;
    unsigned long long *gstate = P.gstate + (size_t)s * P.gstride;
    unsigned long long *sdesc = P.sdesc + (size_t)s * P.gstride;
    int32_t *sj = P.sj + sm, *spos = P.spos + sm, *sE = P.sE + (size_t)s * (P.cap_ld + 2);
    const size_t sp = (size_t)s * (size_t)P.pool_recs;
    double *rec = P.rec + sp * R_NF;
    Meta *meta = P.meta + sp;
    CRec *crec = P.crec + sp;
    CNext *cnext = P.cnext + sp;
    uint16_t *const lane_units = P.lane_units + (size_t)s * P.lanes * P.cap_ld;
    uint16_t *const my_row = lane_units + (size_t)lane * cap;
    const ScenState Z{cold, tbl, gstate, sdesc, sj, spos, sE, P.gcap + sm, P.gfold + sm * 4, rec,
                      P.nxt + sp * 4, P.frec + sp * 2, P.pfx + sp * 4, meta, sm};
    for (int x = lane; x < cap + 2; x += 32) sE[x] = 0;
    if (lane == 0) {
      gs.pool_top = 0;
      gs.abort_code = 0;
    }
    int G = 0;
    unsigned long long evals = 0, cands = 0, exact = 0;
    __syncwarp();
    for (int k = P.k0; k < P.k1; ++k) {
      // the newcomer (planner.py:291-292)
      const double *ck = cold + (size_t)k * C_NF;
      const double *nk = nwt + (size_t)k * R_NF;
      const int need = (int)ck[C_LB];
      const double ksch = ck[C_KSCH], nkern = ck[C_NK];
      const double n_ka = nk[R_KA], n_ca = nk[R_CA], n_pw = nk[R_PW], n_ac = nk[R_ACACHE];
      const double n_beta = fast_beta(nk[R_THALF], nk[R_TLOAD], nk[R_TFB]);
      if (lane == 0) {
        gs.best = NO_KEY;
        fence_async_smem();  // last step's reads of ntab before the async overwrite
        mbar_expect_tx(&nbar[grp], TB * 32);
        bulk_g2s(ntab, tbl + (size_t)k * TB * 4, TB * 32, &nbar[grp]);
      }
      bool n_ready = false;
      __syncwarp();
      unsigned my_best = NO_KEY;
      const int ncand = sE[need];
      int qhead = 0;
      int cj = -1, c_n = 0, c_occ = 0, c_off = 0, c_sum = 0, c_i = 0, c_nu = 0;
      bool c_wait = false, c_eval = false, c_flag = false;
      unsigned long long c_cnt = 0;  // bumps per staged resident, 8 bits each
      double c_C = 0.0, c_P = 0.0, c_inv = 1.0, n_cac = 0.0, n_pwc = 0.0;
      double nA = 0.0, nB = 0.0;
      while (true) {
        const unsigned idle = __ballot_sync(FULL, cj < 0);
        // refill idle lanes in batches so the tile copies overlap (k_place)
        if (idle && (__popc(idle) >= IGP_FAST_REFILL || idle == FULL)) {
          if ((idle >> lane) & 1u) {
            const int pos = qhead + __popc(idle & lt);
            if (pos < ncand) {
              const int j = sj[pos];
              const unsigned long long g = sdesc[pos];
              if ((((unsigned)need << 23) | (unsigned)j) <= *(volatile unsigned *)&gs.best) {
                cj = j;
                c_occ = (int)(g & 0xffffu);
                c_n = (int)((g >> 16) & 0xffffu);
                c_off = (int)(g >> 32);
                cands += 1;
                c_sum = c_occ + need;
                c_i = 0;
                c_nu = need;
                c_cnt = 0;
                c_flag = false;
                c_eval = true;
                const double tsn = (ksch + delta_sch(hw, c_n + 1)) * nkern;
                nA = tsn + n_ka;
                nB = n_ka * n_ac;
                n_cac = n_ca;
                n_pwc = n_pw;
                c_wait = c_n <= FSLOT;
                if (c_wait) {  // stage the compact tile: header (16 B) + 32 B per resident
                  const char *src = reinterpret_cast<const char *>(crec + c_off) - sizeof(CHead);
                  char *dst = reinterpret_cast<char *>(sl);
#pragma unroll
                  for (int c = 0; c <= 2 * FSLOT; ++c)
                    if (c <= 2 * c_n) cp_async16(dst + 16 * c, src + 16 * c);
                  cp_async_commit();
#if IGP_FAST_PF
                  // the next-unit terms a bump reads: into L2 with the tile
                  asm volatile("prefetch.global.L2 [%0];" ::"l"(cnext + c_off));
                  if (c_n > 4) asm volatile("prefetch.global.L2 [%0];" ::"l"(cnext + c_off + 4));
#endif
                }
              }
            }
          }
          qhead += __popc(idle);
          __syncwarp();
        }
        const unsigned busy = __ballot_sync(FULL, cj >= 0);
        if (!busy) {
          if (qhead < ncand) continue;
          break;
        }
        if (cj < 0) continue;
        int result = -1;
        if (c_n > FSLOT) {
          result = R_EXACT;
        } else {
          if (c_wait) {
            cp_async_wait_all();
            c_wait = false;
            c_C = sl->h.C + n_ca;
            c_P = (hw.pidle + sl->h.P) + n_pw;
          }
          if (c_eval) {  // the device terms (model.py:299-305), O(1) from the sums
            const double f = frequency(hw, c_P);
            c_inv = f == hw.fmax ? 1.0 : hw.fmax / f;
            c_eval = false;
            evals += 1;
            // the power sum's rounding must not move f past the margin
            if (!(fabs(hw.af) * fabs(c_P) < 2048.0 * f)) result = R_EXACT;
          }
          // the checks this evaluation serves, up to the first violation
          int viol = -1;
          for (int i = c_i; i <= c_n && result < 0; ++i) {
            double A, B, ca, beta;
            if (i == c_n) {
              A = nA;
              B = nB;
              ca = n_cac;
              beta = n_beta;
            } else {
              const CRec r = sl->r[i];
              A = r.A;
              B = r.B;
              ca = r.ca;
              beta = r.beta;
            }
            const double x = A + B * (c_C - ca);
            const double d = x * c_inv - beta;
            if (!(fabs(d) > delta * beta)) {  // inside the margin (or NaN)
              result = R_EXACT;
              break;
            }
            if (d > 0.0) {  // t_inf > t_half (planner.py:158)
              viol = i;
              break;
            }
          }
          if (result < 0) {
            if (viol < 0) {  // the rest of the pass is clean
              if (c_flag) {
                c_i = 0;  // planner.py:147: another pass after a bump
                c_flag = false;
              } else {
                result = R_FEAS;
              }
            } else {
              const int i = viol;
              c_sum += 1;
              if (c_sum > cap) {
                result = R_INFEAS;
              } else if ((((unsigned)(c_sum - c_occ) << 23) | (unsigned)cj) >
                         *(volatile unsigned *)&gs.best) {
                result = R_PRUNED;
              } else {
                if (i == c_n) {  // the newcomer, from its solo table row
                  c_nu += 1;
                  const int v = c_nu - need;
                  Solo so;
                  if (v < TB && c_nu <= cap) {
                    if (!n_ready) {
                      mbar_wait(&nbar[grp], n_phase);
                      n_ready = true;
                    }
                    const double *tv = ntab + v * 4;
                    so.ka = tv[0];
                    so.pw = tv[1];
                    so.ca = tv[2];
                  } else {
                    so = solo_from_cold(ck, (double)c_nu * hw.runit);
                  }
                  const double tsn = (ksch + delta_sch(hw, c_n + 1)) * nkern;
                  nA = tsn + so.ka;
                  nB = so.ka * n_ac;
                  c_C += so.ca - n_cac;
                  c_P += so.pw - n_pwc;
                  n_cac = so.ca;
                  n_pwc = so.pw;
                } else {
                  const unsigned b = (unsigned)(c_cnt >> (8 * i)) & 0xffu;
                  if (b == 0) {  // one unit above the committed units: precomputed
                    const CNext q = cnext[c_off + i];
                    sl->r[i].A = q.A1;
                    sl->r[i].B = q.B1;
                    sl->r[i].ca += q.dca;
                    c_C += q.dca;
                    c_P += q.dpw;
                  } else {  // further bumps: the solo table at the new units
                    const Meta mt = meta[c_off + i];
                    const int u = (int)mt.u + (int)b + 1;
                    const Solo so = solo_lookup(tbl, cold, hw, mt.k, mt.lb, u);
                    const Solo sp0 = solo_lookup(tbl, cold, hw, mt.k, mt.lb, u - 1);
                    const double *rr = rec + (size_t)(c_off + i) * R_NF;
                    sl->r[i].A = rr[R_TSN] + so.ka;
                    sl->r[i].B = so.ka * rr[R_ACACHE];
                    sl->r[i].ca = so.ca;
                    c_C += so.ca - sp0.ca;
                    c_P += so.pw - sp0.pw;
                  }
                  c_cnt += 1ull << (8 * i);
                }
                c_eval = true;
                c_flag = true;
                c_i = i + 1;
                if (c_i > c_n) {  // the pass ended on a bump: another pass
                  c_i = 0;
                  c_flag = false;
                }
              }
            }
          }
        }
        if (result >= 0) {
          unsigned key = NO_KEY;
          if (result == R_EXACT) {
            exact += 1;
            const int sum = exact_candidate<MAXN>(hw, Z, nk, ksch, nkern, need, k, cj, c_occ, c_n,
                                                  c_off, (const volatile unsigned *)&gs.best,
                                                  my_best, my_row, evals);
            if (sum <= cap) key = ((unsigned)(sum - c_occ) << 23) | (unsigned)cj;
          } else if (result == R_FEAS) {
            key = ((unsigned)(c_sum - c_occ) << 23) | (unsigned)cj;
            if (key < my_best) {
              for (int q = 0; q < c_n; ++q)
                my_row[q] = (uint16_t)((int)meta[c_off + q].u + (int)((c_cnt >> (8 * q)) & 0xffu));
              my_row[c_n] = (uint16_t)c_nu;
            }
          }
          if (key != NO_KEY) {
            if (key < my_best) my_best = key;
            atomicMin(&gs.best, key);
          }
          cj = -1;
        }
      }
      __syncwarp();
      if (lane == 0 && !n_ready) mbar_wait(&nbar[grp], n_phase);  // retire this step's row copy
      n_phase ^= 1u;
      const unsigned bk = gs.best;
      if (bk != NO_KEY && my_best == bk) gs.win_thread = lane;
      __syncwarp();
      // ---- commit (planner.py:312-319) ----
      const uint16_t *lu_w = bk != NO_KEY ? lane_units + (size_t)gs.win_thread * cap : nullptr;
      const double nwv[R_NF] = {n_ka, n_ca, 0.0, n_ac, nk[R_TLOAD], nk[R_TFB], nk[R_THALF], n_pw};
      commit_step(P, hw, Z, k, need, bk, lu_w, G, &gs.pool_top, &gs.abort_code, nwv, ksch, nkern,
                  lane);
      __syncwarp();
      if (*(volatile int *)&gs.abort_code) break;
      write_compact(Z, crec, cnext, bk == NO_KEY ? G : (int)(bk & 0x7fffffu), lane);
      if (bk == NO_KEY) G += 1;
      __syncwarp();
    }
    // hand the scenario to k_place, which writes the plan
    unsigned long long ev = evals, cd = cands, ex = exact;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ev += __shfl_xor_sync(FULL, ev, o);
      cd += __shfl_xor_sync(FULL, cd, o);
      ex += __shfl_xor_sync(FULL, ex, o);
    }
    if (lane == 0) {
      hd->G = G;
      hd->pool_top = gs.pool_top;
      hd->abort = gs.abort_code;
      hd->evals_run = ev;
      hd->cands_run = cd;
      hd->exact_run = ex;
      hd->k_done = P.k1;
    }
    __syncwarp();
  }
}

}  // namespace igp
