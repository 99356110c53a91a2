// smem_plan.cuh -- one plan per CTA with the scenario's search state in shared
// memory (single plans of up to about 1,250 workloads: BASELINE C1/C2).
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
  size_t cr, cd, cd2, ska, ska1, ska2, spw, sac, sx, su, slb, hd, gst, gcap, sdesc, sj, spos, spool,
      rows, sE, total;
};

__host__ __device__ inline size_t sm_align(size_t x) { return (x + 15) & ~(size_t)15; }

// Per placement index k (every workload is one GPU's resident once placed):
//   cr    CRec {A = t_sch(n+1) + k_act, B = k_act * alpha_cache, cache, beta}
//   cd / cd2  deltas {cache, power} from u to u+1 / u+1 to u+2
//   ska / ska1 / ska2  k_act at u / u+1 / u+2
//   spw   power at u      sac  alpha_cache     sx  {k_sch, n_kernels}
//   su    committed units slb  lower bound
// Per open GPU: hd (power / cache sums), gst (descriptor), gcap (tile
// capacity), the slack order sdesc / sj / spos / sE; spool maps pool records
// to placement indices; rows holds each warp's best unit vector.
__host__ __device__ inline SmemLayout smem_layout(int m, long long pool_recs, int cap) {
  SmemLayout L;
  const size_t mm = (size_t)(m > 0 ? m : 1);
  size_t o = 0;
  L.cr = o; o = sm_align(o + mm * sizeof(CRec));
  L.cd = o; o = sm_align(o + mm * 16);
  L.cd2 = o; o = sm_align(o + mm * 16);
  L.ska = o; o = sm_align(o + mm * 8);
  L.ska1 = o; o = sm_align(o + mm * 8);
  L.ska2 = o; o = sm_align(o + mm * 8);
  L.spw = o; o = sm_align(o + mm * 8);
  L.sac = o; o = sm_align(o + mm * 8);
  L.sx = o; o = sm_align(o + mm * 16);
  L.su = o; o = sm_align(o + mm * 2);
  L.slb = o; o = sm_align(o + mm * 2);
  L.hd = o; o = sm_align(o + mm * sizeof(CHead));
  L.gst = o; o = sm_align(o + mm * 8);
  L.gcap = o; o = sm_align(o + mm * 4);
  L.sdesc = o; o = sm_align(o + mm * 8);
  L.sj = o; o = sm_align(o + mm * 4);
  L.spos = o; o = sm_align(o + mm * 4);
  L.spool = o; o = sm_align(o + (size_t)pool_recs * 2);
  L.rows = o; o = sm_align(o + (size_t)SMEM_WARPS * (cap + 1) * 2);
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
  int next_cand[2];  // step k's candidate counter in next_cand[k & 1]
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

struct SmemState {  // the shared-memory arrays of one scenario (SmemLayout)
  CRec *cr;
  double2 *cd, *cd2, *sx;
  double *ska, *ska1, *ska2, *spw, *sac;
  uint16_t *su, *slb, *spool, *rows;
  CHead *hd;
  unsigned long long *gst, *sdesc;
  int32_t *gcap, *sj, *spos, *sE;
};

// The commit of step k (planner.py:312-319) by one warp, on the shared-memory
// state: open GPU G at [need] (bk == NO_KEY) or append the newcomer to GPU j
// with the winner's unit vector lu.  Residents whose units changed take their
// solo terms at u and u+1 from the solo table (one L2 round trip, all lanes
// at once); every other input is in shared memory.  The full records in
// global memory -- read by the exact fallback and by k_place's _build_plan --
// are written on the way (records, next-unit terms, meta, prefix fold states,
// the GPU's fold state), with exact fp64 values and Neumaier folds in
// resident order like commit_step.
__device__ __forceinline__ void commit_smem(const PlanParams &P, const Hw &hw, const ScenState &Z,
                                            const SmemState &X, const SmemNew &NB, int k, int need,
                                            unsigned bk, const uint16_t *lu, int G, int *poolp,
                                            int *abortp, int lane) {
  constexpr unsigned NO_KEY = 0xffffffffu;
  constexpr unsigned FULL = 0xffffffffu;
  const int cap = hw.cap;
  const double n_ka = NB.nw[R_KA], n_ca = NB.nw[R_CA], n_pw = NB.nw[R_PW];
  const double ksch = NB.cold[C_KSCH], nkern = NB.cold[C_NK];
#if IGP_TIMING
  const long long c0 = clock64();
#endif
  int j, n_old, occ_old, off;
  if (bk == NO_KEY) {
    j = G;
    n_old = 0;
    occ_old = 0;
    off = 0;
    if (lane == 0) {
      off = *poolp + 1;  // records after the header slot
      if (off + TILE0 > P.pool_recs) *abortp = IGP_E_CAPACITY;
      else *poolp = off + TILE0;
      X.gcap[j] = TILE0;
    }
    off = __shfl_sync(FULL, off, 0);
  } else {
    j = (int)(bk & 0x7fffffu);
    const unsigned long long g = X.gst[j];
    n_old = (int)((g >> 16) & 0xffffu);
    occ_old = (int)(g & 0xffffu);
    off = (int)(g >> 32);
    const int tcap = X.gcap[j];
    if (n_old + 1 > tcap) {  // grow the tile: copy it to a fresh one of twice the size
      int noff = 0;
      if (lane == 0) {
        noff = *poolp + 1;
        if (noff + 2 * tcap > P.pool_recs) *abortp = IGP_E_CAPACITY;
        else *poolp = noff + 2 * tcap;
      }
      noff = __shfl_sync(FULL, noff, 0);
      __syncwarp();
      if (*(volatile int *)abortp == 0) {
        for (int r = lane; r < n_old; r += 32) {
#pragma unroll
          for (int f = 0; f < R_NF; ++f)
            Z.rec[(size_t)(noff + r) * R_NF + f] = Z.rec[(size_t)(off + r) * R_NF + f];
#pragma unroll
          for (int f = 0; f < 4; ++f) Z.nxt[(size_t)(noff + r) * 4 + f] = Z.nxt[(size_t)(off + r) * 4 + f];
          Z.meta[noff + r] = Z.meta[off + r];
          X.spool[noff + r] = X.spool[off + r];
        }
        if (lane == 0) X.gcap[j] = 2 * tcap;
        off = noff;
      }
      __syncwarp();
    }
  }
  if (*(volatile int *)abortp) return;
  const int n = n_old + 1;
  const double dnext = delta_sch(hw, n + 1);  // t_sch for the next candidate size
  int part = 0;
  double f_pw = 0.0, f_ca = 0.0;  // fold inputs of resident `lane`
  for (int r = lane; r < n; r += 32) {
    const bool nwc = r == n_old;
    const int kk = nwc ? k : (int)X.spool[off + r];
    const int nu = lu ? (int)lu[r] : need;
    double *rr = Z.rec + (size_t)(off + r) * R_NF;
    if (nwc) {  // the newcomer's constants (planner.py:291-292)
      X.spool[off + r] = (uint16_t)k;
      X.sx[kk] = make_double2(ksch, nkern);
      X.sac[kk] = NB.nw[R_ACACHE];
      X.slb[kk] = (uint16_t)need;
      rr[R_ACACHE] = NB.nw[R_ACACHE];
      rr[R_TLOAD] = NB.nw[R_TLOAD];
      rr[R_TFB] = NB.nw[R_TFB];
      rr[R_THALF] = NB.nw[R_THALF];
    }
    const bool changed = nwc || nu != (int)X.su[kk];
    double ca_x;
    if (changed) {  // solo terms at nu, nu + 1, nu + 2 (model.py:285-297)
      Solo so, s1, s2;
      if (nwc) {
        const int v = nu - need;
        auto at = [&](int vv, int uu) {
          if (vv == 0) return Solo{n_ka, n_pw, n_ca, 0};
          if (vv < TB && uu <= cap)
            return Solo{NB.ntab[vv * 4], NB.ntab[vv * 4 + 1], NB.ntab[vv * 4 + 2],
                        (int)NB.ntab[vv * 4 + 3]};
          return solo_from_cold(NB.cold, (double)uu * hw.runit);
        };
        so = at(v, nu);
        s1 = at(v + 1, nu + 1);
        s2 = at(v + 2, nu + 2);
      } else {
        const int lb = X.slb[kk];
        Solo sr[3];
        solo_run<3>(Z.tbl, Z.cold, hw, kk, lb, nu, sr);
        so = sr[0];
        s1 = sr[1];
        s2 = sr[2];
      }
      X.ska2[kk] = s2.ka;
      X.cd2[kk] = make_double2(s2.ca - s1.ca, s2.pw - s1.pw);
      X.ska[kk] = so.ka;
      X.spw[kk] = so.pw;
      X.ska1[kk] = s1.ka;
      X.cd[kk] = make_double2(s1.ca - so.ca, s1.pw - so.pw);
      X.su[kk] = (uint16_t)nu;
      rr[R_KA] = so.ka;
      rr[R_CA] = so.ca;
      rr[R_PW] = so.pw;
      double *nx = Z.nxt + (size_t)(off + r) * 4;
      nx[0] = s1.ka;
      nx[1] = s1.pw;
      nx[2] = s1.ca;
      nx[3] = (double)s1.err;
      Z.meta[off + r] = Meta{kk, (uint16_t)nu, X.slb[kk]};
      ca_x = so.ca;
    } else {
      ca_x = X.cr[kk].ca;
    }
    const double2 xs = X.sx[kk];
    const double tsn = (xs.x + dnext) * xs.y;
    rr[R_TSN] = tsn;
    const double ka = X.ska[kk];
    CRec c;
    c.A = tsn + ka;
    c.B = ka * X.sac[kk];
    c.ca = ca_x;
    c.beta = nwc ? fast_beta(NB.nw[R_THALF], NB.nw[R_TLOAD], NB.nw[R_TFB]) : X.cr[kk].beta;
    X.cr[kk] = c;
    if (r < 32) {
      f_pw = X.spw[kk];
      f_ca = ca_x;
    }
    part += nu;
  }
  part = warp_sum(part);
  __syncwarp();
#if IGP_TIMING
  const long long c1 = clock64();
#endif
  // exact prefix fold states of this GPU, in resident order (model.py:299/304)
  Neumaier fp, fc;
  fp.s = fp.c = fc.s = fc.c = 0.0;  // as commit_step (an add from zero is Neumaier.first)
  for (int r = 0; r < n; ++r) {
    double pw, ca;
    if (r < 32) {
      pw = __shfl_sync(FULL, f_pw, r);
      ca = __shfl_sync(FULL, f_ca, r);
    } else {
      const int kk = X.spool[off + r];
      pw = X.spw[kk];
      ca = X.cr[kk].ca;
    }
    if (lane == 0) {
      double *pp = Z.pfx + (size_t)(off + r) * 4;
      pp[0] = fp.s;
      pp[1] = fp.c;
      pp[2] = fc.s;
      pp[3] = fc.c;
    }
    fp.add(pw);
    fc.add(ca);
  }
#if IGP_TIMING
  const long long c2 = clock64();
#endif
  const unsigned long long desc = ((unsigned long long)off << 32) | (unsigned)part | ((unsigned)n << 16);
  if (lane == 0) {
    double *gf = Z.gfold + (size_t)j * 4;
    gf[0] = fp.s;
    gf[1] = fp.c;
    gf[2] = fc.s;
    gf[3] = fc.c;
    CHead h;
    h.P = fp.s + fp.c;
    h.C = fc.s + fc.c;
    X.hd[j] = h;
    X.gst[j] = desc;
  }
  __syncwarp();
  if (bk == NO_KEY)
    slack_insert(X.sj, X.spos, X.sdesc, X.sE, j, desc, cap - need, lane);
  else
    slack_move_down(X.sj, X.spos, X.sdesc, X.sE, j, desc, cap - occ_old, cap - part, lane);
#if IGP_TIMING
  if (lane == 0 && blockIdx.x == 0 && P.stats) {
    const long long c3 = clock64();
    atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 4], (unsigned long long)(c1 - c0));
    atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 5], (unsigned long long)(c2 - c1));
    atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 6], (unsigned long long)(c3 - c2));
  }
#endif
}

template <int MAXN, bool HWS = false>
__global__ void __launch_bounds__(SMEM_WARPS * 32, 1) k_plan_smem(PlanParams P) {
  constexpr unsigned NO_KEY = 0xffffffffu;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ SmemCtl ctl;
  const int t = threadIdx.x, lane = t & 31, wi = t >> 5;
  const int s = blockIdx.x;
  Hand *const hdp = P.hand + s;
  // the profile: the launch's (constant bank), or the scenario's (IGP_F_HWS,
  // staged in shared memory)
  __shared__ Hw shw[HWS ? 1 : 1];
  if constexpr (HWS) {
    if (t == 0) shw[0] = P.hw_s[s];
    __syncthreads();
  }
  const Hw &hw = HWS ? shw[0] : P.hw;
  const int m = P.m, cap = hw.cap;
  if (P.perr[s] != INT_MAX || P.sflags[s] != 0 || !hw.margin_ok) {
    if (t == 0) hdp->k_done = P.k0;  // declined: k_place plans it
    return;
  }
  const SmemLayout SL = smem_layout(m, P.pool_recs, P.cap_ld);
  SmemState X;
  X.cr = reinterpret_cast<CRec *>(dsm + SL.cr);
  X.cd = reinterpret_cast<double2 *>(dsm + SL.cd);
  X.cd2 = reinterpret_cast<double2 *>(dsm + SL.cd2);
  X.ska = reinterpret_cast<double *>(dsm + SL.ska);
  X.ska1 = reinterpret_cast<double *>(dsm + SL.ska1);
  X.ska2 = reinterpret_cast<double *>(dsm + SL.ska2);
  X.spw = reinterpret_cast<double *>(dsm + SL.spw);
  X.sac = reinterpret_cast<double *>(dsm + SL.sac);
  X.sx = reinterpret_cast<double2 *>(dsm + SL.sx);
  X.su = reinterpret_cast<uint16_t *>(dsm + SL.su);
  X.slb = reinterpret_cast<uint16_t *>(dsm + SL.slb);
  X.hd = reinterpret_cast<CHead *>(dsm + SL.hd);
  X.gst = reinterpret_cast<unsigned long long *>(dsm + SL.gst);
  X.gcap = reinterpret_cast<int32_t *>(dsm + SL.gcap);
  X.sdesc = reinterpret_cast<unsigned long long *>(dsm + SL.sdesc);
  X.sj = reinterpret_cast<int32_t *>(dsm + SL.sj);
  X.spos = reinterpret_cast<int32_t *>(dsm + SL.spos);
  X.spool = reinterpret_cast<uint16_t *>(dsm + SL.spool);
  X.rows = reinterpret_cast<uint16_t *>(dsm + SL.rows);
  X.sE = reinterpret_cast<int32_t *>(dsm + SL.sE);
  CRec *const cr = X.cr;
  CHead *const hd = X.hd;
  unsigned long long *const gst = X.gst;
  unsigned long long *const sdesc = X.sdesc;
  int32_t *const sj = X.sj, *const sE = X.sE;
  uint16_t *const su = X.su, *const spool = X.spool;

  const size_t sm = (size_t)s * m;
  const double *cold = P.cold + sm * C_NF;
  const double *nwt = P.nw + sm * R_NF;
  const double *tbl = P.tbl + sm * TB * 4;
  const size_t sp = (size_t)s * (size_t)P.pool_recs;
  const ScenState Z{cold, tbl, gst, sdesc, sj, X.spos, sE, P.gcap + sm, P.gfold + sm * 4,
                    P.rec + sp * R_NF, P.nxt + sp * 4, P.frec + sp * 2, P.pfx + sp * 4,
                    P.meta + sp, sm};
  uint16_t *const my_row = X.rows + (size_t)wi * (cap + 1);
  for (int x = t; x < cap + 2; x += blockDim.x) sE[x] = 0;
  if (t == 0) {
    ctl.pool_top = 0;
    ctl.abort_code = 0;
  }
  int G = 0;
  unsigned long long evals = 0, cands = 0, exact = 0;
  const double delta = P.fast_delta;
  smem_fetch_newcomer(ctl.nb[P.k0 & 1], nwt, cold, tbl, P.k0, t);
  if (t == 0) {
    ctl.best[0] = ctl.best[1] = NO_KEY;
    ctl.next_cand[0] = ctl.next_cand[1] = 0;
  }
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
    // warps take the step's candidates from a shared counter: a long Alg. 2
    // chain does not hold back a candidate statically assigned behind it
    int* const ncp = &ctl.next_cand[k & 1];
    for (;;) {
      int c = 0;
      if (lane == 0) c = atomicAdd(ncp, 1);
      c = __shfl_sync(FULL, c, 0);
      if (c >= ncand) break;
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
                const double2 q = X.cd[kk];
                A += X.ska1[kk] - X.ska[kk];
                B = X.ska1[kk] * X.sac[kk];
                ca += q.x;
                dC = q.x;
                dP = q.y;
              } else if (bumps == 1) {  // two units above: also precomputed
                const double2 q = X.cd2[kk];
                A += X.ska2[kk] - X.ska1[kk];
                B = X.ska2[kk] * X.sac[kk];
                ca += q.x;
                dC = q.x;
                dP = q.y;
              } else {  // further bumps: the solo table at the new units
#if IGP_TIMING
                if (s == 0 && P.stats) atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 4], 1ull);
#endif
                const int lb = X.slb[kk];
                const Solo so = solo_lookup(tbl, cold, hw, kk, lb, u);
                const Solo s0 = solo_lookup(tbl, cold, hw, kk, lb, u - 1);
                A += so.ka - s0.ka;
                B = so.ka * X.sac[kk];
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
      const unsigned wb = lane < SMEM_WARPS ? ctl.wbest[lane] : NO_KEY;
      const unsigned hit = __ballot_sync(FULL, bk != NO_KEY && wb == bk);
      const uint16_t *lu_w = bk != NO_KEY ? X.rows + (size_t)(__ffs(hit) - 1) * (cap + 1) : nullptr;
      commit_smem(P, hw, Z, X, NB, k, need, bk, lu_w, G, &ctl.pool_top, &ctl.abort_code, lane);
    }
    if (bk == NO_KEY) G += 1;
    if (t == 0) {  // step k+1's slots: nobody reads them during step k
      ctl.best[(k + 1) & 1] = NO_KEY;
      ctl.next_cand[(k + 1) & 1] = 0;
    }
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
