// window.cuh -- one plan with speculative lookahead over a window of steps.
//
// Alg. 1 (planner.py:290-319) is a chain of m dependent steps, but step k+1
// depends on step k only through the ONE GPU that step k modifies (or opens):
// every other GPU's state -- and therefore the result of Alg. 2 (planner.py:
// 133-162) for the newcomer of step k+1 on it -- is unchanged.  This kernel
// plans a single scenario in windows of WIN steps with one CTA:
//
//   phase A (all warps): every newcomer i of the window against every
//     candidate GPU of the window-start state (occupied + need_i <= cap,
//     planner.py:297-299), one candidate per thread.  Step i keeps its i+1
//     smallest keys (inter << 23 | j) and the unit vectors behind them; a
//     candidate stops as soon as its key can no longer be among them (units
//     only grow inside Alg. 2).
//   phase B (warp 0, in step order): step i's argmin is the smaller of
//     (a) the first kept key whose GPU no earlier step of the window touched,
//     (b) a fresh Alg. 2 run on every touched GPU that is a candidate now.
//     Earlier steps touched at most i GPUs, so (a) is the exact minimum over
//     the untouched ones and (b) covers the rest.  Then the commit
//     (planner.py:312-319, commit_step, shared with k_place).
//
// The plan is the sequential one bit for bit: an untouched GPU gives the same
// key and unit vector as in step order, keys are unique per j (so the argmin
// does not depend on evaluation order) and ties keep the lowest j exactly as
// `inter < best` does.  What the window buys is latency: a step's candidate
// chains, newcomer loads and CTA barriers are paid once per window, and only
// the touched GPUs are re-run on the critical path.  Used for one scenario in
// the fast mode (IGP_F_WIN); a scenario that needs the exact sequence
// (PlanStats, an input that can raise) is declined and planned by the per-CTA
// kernel, which also writes the plan (the CoopState hand-off of the
// cooperative kernel).
#pragma once

namespace igp {

#ifndef IGP_WIN
#define IGP_WIN 8  // steps per window
#endif
constexpr int WIN = IGP_WIN;
constexpr int WIN_POOL = 24;  // unit vectors kept per step (beyond: recomputed in phase B)
constexpr int WIN_THREADS = 256;
constexpr int WIN_LANE_ROWS = WIN_THREADS + WIN * WIN_POOL;  // lane_units rows it uses

struct WinSmem {
  unsigned int top[WIN][WIN];  // step i: its i+1 smallest keys so far, ascending
  int slot[WIN][WIN];          // pool slot of each kept key (-1: unit vector not kept)
  int lock[WIN];
  int pool_n[WIN];
  int need[WIN], pre[WIN + 1];
  double nwr[WIN][R_NF + 2];   // newcomer record, then k_sch and n_kernels
  int touched[WIN];            // GPUs modified or opened by the window's steps so far
  unsigned int fresh_best;     // phase B: argmin over the re-run touched GPUs
  int pool_top, abort_code, G;
  unsigned long long evals, cands;
};

// Alg. 2 (planner.py:146-162) for GPU j -- nres residents in the pool tile at
// off, occ units -- plus the newcomer of window step i (placement index kk),
// fast mode: it stops at the first Sum u > cap, or once its key exceeds *thr.
// Returns the final Sum u (> cap: infeasible or pruned); the unit vector
// (residents, then the newcomer) is left in lu.  Evaluation, fold order and
// the division shortcut are those of k_place (model.py:273-317).
template <int MAXN>
__device__ int win_candidate(const Hw &hw, const ScenState &Z, const WinSmem &W, int i, int kk,
                             int j, int occ, int nres, int off, const volatile unsigned *thr,
                             bool margin, uint16_t *lu, unsigned long long &evals) {
  const int cap = hw.cap;
  const int need = W.need[i];
  const double *nw = W.nwr[i];
  double ka[MAXN + 1], pw[MAXN + 1], ca[MAXN + 1];
  int u[MAXN + 1];
  for (int q = 0; q < nres; ++q) {
    const double *r = Z.rec + (size_t)(off + q) * R_NF;
    const double2 kc = *reinterpret_cast<const double2 *>(r + R_KA);
    ka[q] = kc.x;
    ca[q] = kc.y;
    pw[q] = r[R_PW];
    u[q] = Z.meta[off + q].u;
  }
  u[nres] = need;
  ka[nres] = nw[R_KA];
  ca[nres] = nw[R_CA];
  pw[nres] = nw[R_PW];
  const double tsn_new = (nw[R_NF] + delta_sch(hw, nres + 1)) * nw[R_NF + 1];
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
        one = f == hw.fmax && hw.margin_ok;
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
        if (margin) {
          const double tq = (t_load + t_gpu) + t_fb;
          if (!(fabs(tq - t_half) > tq * 0x1p-48 + 0x1p-1000)) t_gpu = x / (f / hw.fmax);
        } else {
          t_gpu = x / (f / hw.fmax);
        }
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
#if IGP_SPLIT_NEXT
            const double *nx = Z.nxt + (size_t)(off + q) * 4;
            so.ka = nx[0];
            so.pw = nx[1];
            so.ca = nx[2];
            so.err = (int)nx[3];
#else
            so = solo_lookup(Z.tbl, Z.cold, hw, mt.k, mt.lb, u[q]);
#endif
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
  for (int q = 0; q <= nres; ++q) lu[q] = (uint16_t)u[q];
  return sum;
}

template <int MAXN>
__global__ void __launch_bounds__(WIN_THREADS, 1) k_place_win(PlanParams P) {
  constexpr unsigned NO_KEY = 0xffffffffu;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ WinSmem W;
  const int t = threadIdx.x, lane = t & 31, wi = t >> 5;
  const Hw &hw = P.hw;
  const int m = P.m, cap = hw.cap;
  CoopState *const cs = P.coop;
  const int sflags = P.sflags[0];
  // the exact evaluation sequence (PlanStats, an input that can raise) and a
  // prologue error are the per-CTA kernel's
  if (P.perr[0] != INT_MAX || (sflags & SF_RISKY) || (P.flags & IGP_F_STATS)) {
    if (t == 0) cs->status = P.k0;
    return;
  }
  const bool margin = !(sflags & SF_NO_MARGIN) && hw.margin_ok;
  const ScenState Z{P.cold, P.tbl, P.gstate, P.sdesc, P.sj, P.spos, P.sE, P.gcap, P.gfold,
                    P.rec, P.nxt, P.frec, P.pfx, P.meta, 0};
  uint16_t *const lane_row = P.lane_units + (size_t)t * cap;
  uint16_t *const pool_rows = P.lane_units + (size_t)WIN_THREADS * cap;  // [WIN][WIN_POOL]
  for (int x = t; x < cap + 2; x += WIN_THREADS) P.sE[x] = 0;
  if (t == 0) {
    W.pool_top = 0;
    W.abort_code = 0;
    W.G = 0;
    W.evals = W.cands = 0;
  }
  unsigned long long evals = 0, cands = 0;
  __syncthreads();
  for (int k0 = 0; k0 < m; k0 += WIN) {
    const int d = m - k0 < WIN ? m - k0 : WIN;
    if (t < d) {  // the window's newcomers
      const double *ck = P.cold + (size_t)(k0 + t) * C_NF;
      const double *nk = P.nw + (size_t)(k0 + t) * R_NF;
#pragma unroll
      for (int f = 0; f < R_NF; ++f) W.nwr[t][f] = nk[f];
      W.nwr[t][R_NF] = ck[C_KSCH];
      W.nwr[t][R_NF + 1] = ck[C_NK];
      W.need[t] = (int)ck[C_LB];
      W.lock[t] = 0;
      W.pool_n[t] = 0;
    }
    if (t < WIN * WIN) {
      W.top[t / WIN][t % WIN] = NO_KEY;
      W.slot[t / WIN][t % WIN] = -1;
    }
    __syncthreads();
    if (t == 0) {
      int acc = 0;
      for (int i = 0; i < d; ++i) {
        W.pre[i] = acc;
        acc += P.sE[W.need[i]];  // step i's candidates: the slack-order prefix
      }
      W.pre[d] = acc;
    }
    __syncthreads();
    // ---- phase A: every (step, candidate) pair of the window-start state ----
    const int total = W.pre[d];
    for (int c = t; c < total; c += WIN_THREADS) {
      int i = 0;
      while (c >= W.pre[i + 1]) ++i;
      const int pos = c - W.pre[i];
      const int j = P.sj[pos];
      const unsigned long long g = P.sdesc[pos];
      const volatile unsigned *thr = &W.top[i][i];  // the (i+1)-th smallest key so far
      if ((((unsigned)W.need[i]) << 23 | (unsigned)j) > *thr) continue;
      cands += 1;
      uint16_t lu[MAXN + 1];
      const int occ = (int)(g & 0xffffu), nres = (int)((g >> 16) & 0xffffu);
      const int sum = win_candidate<MAXN>(hw, Z, W, i, k0 + i, j, occ, nres, (int)(g >> 32), thr,
                                          margin, lu, evals);
      if (sum > cap) continue;
      const unsigned key = ((unsigned)(sum - occ) << 23) | (unsigned)j;
      if (key > *thr) continue;
      int slot = atomicAdd(&W.pool_n[i], 1);
      if (slot < WIN_POOL) {
        uint16_t *row = pool_rows + (size_t)(i * WIN_POOL + slot) * cap;
        for (int q = 0; q <= nres; ++q) row[q] = lu[q];
      } else {
        slot = -1;
      }
      __threadfence_block();
      while (atomicCAS(&W.lock[i], 0, 1) != 0) {
      }
      // insert (key, slot) into step i's ascending list of i+1 keys
      volatile unsigned *tp = W.top[i];
      volatile int *sp = W.slot[i];
      if (key < tp[i]) {
        int e = i;
        while (e > 0 && tp[e - 1] > key) {
          tp[e] = tp[e - 1];
          sp[e] = sp[e - 1];
          --e;
        }
        tp[e] = key;
        sp[e] = slot;
      }
      __threadfence_block();
      atomicExch(&W.lock[i], 0);
    }
    __syncthreads();
    // ---- phase B: the window's steps in order, warp 0 ----
    if (wi == 0) {
      int G = W.G, ntouched = 0;
      for (int i = 0; i < d && !W.abort_code; ++i) {
        const int k = k0 + i, need = W.need[i];
        // (a) the smallest kept key on a GPU no earlier step of the window touched
        unsigned spec = NO_KEY;
        int spec_slot = -1;
        for (int e = 0; e <= i; ++e) {
          const unsigned key = W.top[i][e];
          if (key == NO_KEY) break;
          const int j = (int)(key & 0x7fffffu);
          bool hit = false;
          for (int q = 0; q < ntouched; ++q) hit |= W.touched[q] == j;
          if (!hit) {
            spec = key;
            spec_slot = W.slot[i][e];
            break;
          }
        }
        // (b) the touched GPUs that are candidates now, one lane each
        if (lane == 0) W.fresh_best = spec;
        __syncwarp();
        unsigned mine = NO_KEY;
        if (lane < ntouched) {
          const int j = W.touched[lane];
          const unsigned long long g = P.gstate[j];
          const int occ = (int)(g & 0xffffu), nres = (int)((g >> 16) & 0xffffu);
          if (occ + need <= cap && (((unsigned)need << 23) | (unsigned)j) <= W.fresh_best) {
            cands += 1;
            const int sum = win_candidate<MAXN>(hw, Z, W, i, k, j, occ, nres, (int)(g >> 32),
                                                &W.fresh_best, margin, lane_row, evals);
            if (sum <= cap) {
              mine = ((unsigned)(sum - occ) << 23) | (unsigned)j;
              atomicMin(&W.fresh_best, mine);
            }
          }
        }
        __syncwarp();
        unsigned bk = W.fresh_best;
        const uint16_t *lu = nullptr;
        if (bk != NO_KEY) {
          const unsigned who = __ballot_sync(FULL, mine == bk);
          if (who) {
            lu = P.lane_units + (size_t)(__ffs(who) - 1) * cap;
          } else if (spec_slot >= 0) {
            lu = pool_rows + (size_t)(i * WIN_POOL + spec_slot) * cap;
          } else {  // the winner's unit vector was not kept: run it again (lane 0's row)
            const int j = (int)(bk & 0x7fffffu);
            if (lane == 0) {
              const unsigned long long g = P.gstate[j];
              const unsigned none = NO_KEY;
              win_candidate<MAXN>(hw, Z, W, i, k, j, (int)(g & 0xffffu),
                                  (int)((g >> 16) & 0xffffu), (int)(g >> 32), &none, margin,
                                  P.lane_units, evals);
            }
            __syncwarp();
            lu = P.lane_units;
          }
        }
        commit_step(P, hw, Z, k, need, bk, lu, G, &W.pool_top, &W.abort_code, W.nwr[i],
                    W.nwr[i][R_NF], W.nwr[i][R_NF + 1], lane);
        if (lane == 0) W.touched[ntouched] = bk == NO_KEY ? G : (int)(bk & 0x7fffffu);
        if (bk == NO_KEY) G += 1;
        ++ntouched;
        __threadfence();  // the commit's global writes before the next step's reads
        __syncwarp();
      }
      if (lane == 0) W.G = G;
    }
    __syncthreads();
    if (W.abort_code) break;
  }
  // hand the state to the per-CTA kernel, which writes the plan
  atomicAdd(&W.evals, evals);
  atomicAdd(&W.cands, cands);
  __syncthreads();
  if (t == 0) {
    cs->G = W.G;
    cs->pool_top = W.pool_top;
    cs->abort = W.abort_code;
    cs->sflags = sflags;
    cs->evals_run = W.evals;
    cs->cands_run = W.cands;
    cs->status = P.k1;  // an abort is reported by the per-CTA kernel
  }
}

}  // namespace igp
