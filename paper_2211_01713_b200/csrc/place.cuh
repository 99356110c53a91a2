// place.cuh -- the greedy placement (Alg. 1 + Alg. 2) on the device.
//
// Restates planner.py:258-325 (plan), :133-162 (_alloc_units), :218-246
// (_build_plan) and model.py:273-317 (_eval_entries) for S independent
// scenarios.  Included by igniter_kernels.cu (needs prologue_one,
// entry_consts, make_hw from there).
//
// Device layout, per scenario (all in the caller's workspace):
//   per workload, in placement order k (sorted by (-lb, name)):
//     cold[k][12]   constants for unit changes (gamma, k4, k5, batch, alpha/beta
//                   of power and cache, k_sch, n_kernels, lb, input index)
//     nw[k][8]      k's check record at its lower bound (the newcomer's state)
//     tbl[k][16][4] solo (k_act, power, cache, error) at u = lb .. lb+15: a
//                   unit bump is one 32-byte lookup instead of two divisions
//   per open GPU j:
//     gstate[j]     occupied units | residents << 16 (the prefilter scans this)
//     goff/gcap[j]  its tile in the record pool
//     gfold[j][4]   Neumaier (s, c) of the power and cache sums over residents
//   record pool (tiles; a GPU's residents are contiguous, in placement order):
//     rec[r][8]     64-byte check record: k_act, cache, t_sch for the next
//                   candidate size, alpha_cache, t_load, t_feedback, t_half, power
//     frec[r][2]    (power, cache) -- the fold stream
//     pfx[r][4]     Neumaier states of both sums BEFORE this resident
//     meta[r]       workload k, units, lower bound
//   Tiles start with 4 records and double on overflow (copied); the pool holds
//   pool_factor * m records, enough for every realistic plan (E_CAPACITY
//   otherwise, and the host retries with a larger pool).
#pragma once

namespace igp {

constexpr int TB = 16;     // solo-table entries per workload
constexpr int TILE0 = 4;   // initial tile capacity
// pool record of one resident (96 B): its solo terms at the committed units,
// t_sch for the next candidate size, the transfer / budget constants, and the
// solo terms one unit up (a first bump inside a candidate needs no lookup)
#ifndef IGP_SPLIT_NEXT
#define IGP_SPLIT_NEXT 1
#endif
#ifndef IGP_PF_BATCH
#define IGP_PF_BATCH 0  // L2 prefetch of the next refill batch's tiles
#endif
#ifndef IGP_NW_SMEM
#define IGP_NW_SMEM 1  // newcomer record in shared memory (frees registers: +2.5% at 10k with the lean pass)
#endif
#ifndef IGP_PF_DESC
#define IGP_PF_DESC 1  // L1 prefetch of the next refill's slack-order descriptors
#endif
#ifndef IGP_PF_NEXT
#define IGP_PF_NEXT 0  // L2 prefetch of the staged residents' next-unit terms
#endif

#if IGP_SPLIT_NEXT
// 64-byte records; the next-unit solo terms live in a parallel pool array
// (NEXT_AT) that the tile copy does not carry
enum { R_KA = 0, R_CA, R_TSN, R_ACACHE, R_TLOAD, R_TFB, R_THALF, R_PW, R_NF };
#else
enum { R_KA = 0, R_CA, R_TSN, R_ACACHE, R_TLOAD, R_TFB, R_THALF, R_PW, R_KA1, R_PW1, R_CA1,
       R_ERR1, R_NF };
#endif
enum { SF_RISKY = 1, SF_NO_MARGIN = 2, SF_NO_FAST = 4 };
// the certified-margin kernels' error bound assumes alpha_cache <= this (fast.cuh)
constexpr double FAST_MAX_ACACHE = 16.0;
enum { R_FEAS = 0, R_INFEAS = 1, R_PRUNED = 2, R_ERROR = 3 };

struct Meta {
  int32_t k;
  uint16_t u;
  uint16_t lb;
};

// A candidate's resident tile is staged into a per-lane shared-memory slot
// with one TMA bulk copy (records, meta, the GPU's Neumaier fold state);
// residents beyond SLOT are read from the global pool.
#ifndef IGP_SLOT
#define IGP_SLOT 4
#endif
constexpr int SLOT = IGP_SLOT;
static_assert(SLOT >= 1 && SLOT <= 4, "the tile header carries the first four residents' meta");

// A tile in the record pool is one header record followed by the resident
// records; the header mirrors the GPU's Neumaier fold state and the first
// residents' meta, so one bulk copy stages everything a candidate reads.
struct __align__(16) TileHeader {
  double gf[4];  // Neumaier (s, c) of the power and cache sums over residents
  Meta meta[4];  // (workload, units, lower bound) of residents 0..3
#if !IGP_SPLIT_NEXT
  double pad[4];
#endif
};
static_assert(sizeof(TileHeader) == R_NF * 8, "the header occupies one record slot");

struct __align__(16) LaneSlot {
  double gf[4];  // staged header ...
  Meta meta[4];
#if !IGP_SPLIT_NEXT
  double hpad[4];
#endif
  double rec[SLOT][R_NF];  // ... and the first SLOT resident records
};
// the per-lane mbarriers of the slots' bulk copies follow the slot array in
// dynamic shared memory (8 B each, instead of 16 B of padding per slot)
constexpr size_t lane_smem_bytes() { return sizeof(LaneSlot) + sizeof(unsigned long long); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// Per-thread 16-byte async copies (LDGSTS) completing on an mbarrier.  A
// lane's candidate tile is staged this way: cp.async.bulk takes its operands
// from uniform registers, so 32 lanes with 32 different tiles compile to a
// 32-trip ELECT/R2UR/UBLKCP loop (13.5% of k_place's instructions and 10% of
// its stall samples in profiles/r02); LDGSTS issues for all lanes at once.
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
// the barrier's (single) arrival fires when this thread's prior cp.asyncs land
__device__ __forceinline__ void cp_async_arrive(unsigned long long *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// ... or tracked as a per-thread group: cp.async.mbarrier.arrive also takes its
// barrier address from a uniform register (another per-lane ELECT loop, 9.5%
// of the fast kernel's instructions), commit/wait_group do not
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
// candidate tile staging: 0 = cp.async.bulk + mbarrier, 1 = LDGSTS + mbarrier,
// 2 = LDGSTS + commit/wait_group
#ifndef IGP_TILE_LDGSTS
#define IGP_TILE_LDGSTS 2
#endif
// generic-proxy writes -> later async-proxy (TMA) access of the same memory
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Grid-cooperative single plan (IGP_F_COOP): every warp of the GPU works on
// one scenario's step; the last warp to finish the step commits it and
// publishes the step number.  State shared by all warps:
struct CoopState {
  unsigned int best[2];  // argmin key of the q-th processed step in best[q & 1]
  int best_pad[2];
  int done[2];                 // CTAs finished with step q
  int flag;                    // steps committed so far
  int pool_top, abort, G;
  int status;                  // the first step the cooperative kernel did NOT run (k0 when it
                               // declined; k1 when it ran them all); the per-CTA kernel resumes there
  int sflags;                  // risk flags of the steps it ran (stream mode)
  unsigned long long evals_run, cands_run;
};
constexpr int COOP_MAX_LANES = 160 * 512;  // lane_units rows reserved for the cooperative grid

// Compact tiles of the certified-margin fast path (fast.cuh).
#ifndef IGP_FSLOT
#define IGP_FSLOT 7
#endif
// compact resident records staged per lane (a GPU with more residents takes
// the exact evaluation); 7 keeps six 128-thread CTAs per SM within shared memory
constexpr int FSLOT = IGP_FSLOT;
static_assert(FSLOT >= 1 && FSLOT <= 8, "bump counters: 8 bits per staged resident");
struct __align__(16) CRec {  // a resident's check terms at its committed units
  double A, B, ca, beta;
};
struct __align__(16) CNext {  // ... one unit up, as values and exact deltas of the sums
  double A1, B1, dca, dpw;
};
struct __align__(16) CHead {  // a GPU's power and cache sums (compact tile header)
  double P, C;
};
struct __align__(16) FastSlot {
  CHead h;
  CRec r[FSLOT];
};

// Hand-off from k_place_fast to k_place (which writes the plan and the
// _build_plan rows): the step where k_place resumes (k1 = all planned, k0 =
// declined) and the scenario state after the fast steps.
constexpr int HAND_COMPLETE = 0x7fffffff;  // k_done of a scenario the lean pass planned
struct Hand {
  int k_done, G, pool_top, abort;
  unsigned long long evals_run, cands_run, exact_run, pad;
};

struct WsLayout {
  size_t by_rank, order, cold, nw, tbl, gstate, gcap, gfold, rec, frec, pfx, meta,
      lane_units, sflags, perr, sched, coop, win_tid, sdesc, sj, spos, sE, nxt, hws, crec, cnext,
      hand, total;
  int lanes;
  int gstride;          // per-scenario stride of gstate (multiple of 4: 16-byte scan loads)
  long long pool_recs;  // records per scenario
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static int pool_factor(int flags) {
  const int f = (flags >> 8) & 0xff;
  return f ? f : 7;
}

// IGP_F_FAST: the certified-margin kernel (fast.cuh) runs before k_place for
// batches of one-warp scenarios.
static bool fast_path(int flags) {
  return (flags & IGP_F_FAST) && !(flags & (IGP_F_STATS | IGP_F_CTA | IGP_F_GW2 | IGP_F_GW4 |
                                            IGP_F_COOP | IGP_F_WIN | IGP_F_HWS));
}

// The batch path of one-warp scenarios runs the lean pass first (k_place LEAN).
static bool lean_path(int flags) {
#ifdef IGP_NO_LEAN
  return false;
#else
  return !(flags & (IGP_F_FAST | IGP_F_STATS | IGP_F_CTA | IGP_F_GW2 | IGP_F_GW4 | IGP_F_COOP |
                    IGP_F_WIN | IGP_F_HWS | IGP_F_SMEM));
#endif
}

static WsLayout ws_layout(int S, int m, int cap, int flags) {
  WsLayout L;
  size_t off = 0;
  const size_t mm = (size_t)(m > 0 ? m : 1);
  const size_t Sm = (size_t)S * mm;
  const int capx = cap > 0 ? cap : 1;
  L.lanes = (flags & IGP_F_COOP) ? COOP_MAX_LANES : (flags & IGP_F_WIN) ? 512
            : (flags & IGP_F_CTA) ? 256
            : (flags & IGP_F_GW4) ? 128 : (flags & IGP_F_GW2) ? 64 : 32;
  L.pool_recs = (long long)pool_factor(flags) * (long long)mm + 4 * TILE0;
  const size_t Sp = (size_t)S * (size_t)L.pool_recs;
  L.by_rank = off; off = align_up(off + Sm * 4);
  L.order = off; off = align_up(off + Sm * 4);
  L.cold = off; off = align_up(off + Sm * C_NF * 8);
  L.nw = off; off = align_up(off + Sm * R_NF * 8);
  L.tbl = off; off = align_up(off + Sm * TB * 4 * 8);
  L.gstride = (int)((mm + 3) & ~(size_t)3);
  L.gstate = off; off = align_up(off + (size_t)S * L.gstride * 8);
  L.gcap = off; off = align_up(off + Sm * 4);
  L.gfold = off; off = align_up(off + Sm * 4 * 8);
  L.rec = off; off = align_up(off + Sp * R_NF * 8);
  L.frec = off; off = align_up(off + Sp * 2 * 8);
  L.pfx = off; off = align_up(off + Sp * 4 * 8);
  L.meta = off; off = align_up(off + Sp * sizeof(Meta));
  L.lane_units = off; off = align_up(off + (size_t)S * L.lanes * capx * 2);
  L.sflags = off; off = align_up(off + (size_t)S * 4);
  L.perr = off; off = align_up(off + (size_t)S * 4);
  L.sched = off; off = align_up(off + 4);
  L.coop = off; off = align_up(off + sizeof(CoopState));
  L.win_tid = off; off = align_up(off + ((flags & IGP_F_COOP) ? mm * 4 : 4));
  L.sdesc = off; off = align_up(off + (size_t)S * L.gstride * 8);
  L.sj = off; off = align_up(off + Sm * 4);
  L.spos = off; off = align_up(off + Sm * 4);
  L.sE = off; off = align_up(off + (size_t)S * (capx + 2) * 4);
  L.nxt = off; off = align_up(off + (IGP_SPLIT_NEXT ? Sp * 32 : 32));
  L.hws = off; off = align_up(off + ((flags & IGP_F_HWS) ? (size_t)S * sizeof(Hw) : 0));
  const bool fast = fast_path(flags);
  L.crec = off; off = align_up(off + (fast ? Sp * sizeof(CRec) : 0));
  L.cnext = off; off = align_up(off + (fast ? Sp * sizeof(CNext) : 0));
  // the hand-off records (lean pass, certified-margin and shared-memory
  // kernels) are always laid out: S x 48 bytes, so that a workspace sized
  // for one set of flags (e.g. with IGP_F_STATS) serves the others
  L.hand = off; off = align_up(off + (size_t)S * sizeof(Hand));
  L.total = off;
  return L;
}

struct PlanParams {
  Hw hw;
  // IGP_F_HWS: one hardware profile per scenario (select_gpu_type plans every
  // GPU type of a request as one scenario of one launch); nullptr otherwise
  const Hw *hw_s;
  int cap_ld;  // the workspace layout's max_units (largest over the scenarios)
  int S, m, flags;
  // placement steps [k0, k1) of this launch.  Plan mode: [0, m), order from
  // the (-lb, name) sort.  Stream mode (online arrivals, BASELINE config 5):
  // placement order = arrival order, the per-scenario state (open GPUs, pool)
  // persists across launches in sstate, and an arrival whose prologue or
  // candidate evaluation raises is rejected instead of aborting the scenario.
  int k0, k1, stream;
  int32_t *code;    // stream: per arrival error code | risk flags << 8
  int32_t *sstate;  // stream: per scenario {G, pool_top, sticky flags, arrivals}
  // Open GPUs ordered by free units (slack = cap - occupied), descending:
  // sj[p] / sdesc[p] = GPU index / descriptor at position p, spos[j] = the
  // position of GPU j, sE[s] = number of GPUs with slack >= s.  A step's
  // candidates (occupied + need <= cap, planner.py:297-299) are exactly the
  // prefix [0, sE[need]).
  unsigned long long *sdesc;
  int32_t *sj, *spos, *sE;
  CoopState *coop;  // cooperative single plan: shared step state (nullable)
  int32_t *win_tid; // cooperative: thread whose lane_units hold candidate j's units
  const double *wl;     // [S][16][m]
  const int32_t *rank;  // name ranks
  int rank_stride;
  int lanes;
  int gstride;
  long long pool_recs;
  // workspace
  int32_t *by_rank, *order, *sflags, *perr, *gcap;
  int32_t *sched;  // persistent-kernel scenario counter (zeroed before each launch)
  // per open GPU j: occupied units | residents << 16 | tile offset << 32
  unsigned long long *gstate;
  double *cold, *nw, *tbl, *gfold, *rec, *frec, *pfx;
  double *nxt;  // IGP_SPLIT_NEXT: next-unit solo terms per pool record
  Meta *meta;
  uint16_t *lane_units;
  // outputs
  int32_t *gpu_of, *pos, *units, *batch, *lb, *gpu_count;
  double *pred;
  int64_t *stats;
  igp_error *err;
  // certified-margin fast path (fast.cuh); hand == nullptr: not used
  CRec *crec;
  CNext *cnext;
  Hand *hand;
  double fast_delta;  // decision margin relative to beta (FAST_DELTA; IGP_FAST_DELTA overrides)
};

// ---------------------------------------------------------------------------
// prepare stage
// ---------------------------------------------------------------------------
// thread per (scenario, workload): batch, lb, first-error key, risk flags, by_rank
__global__ void k_prologue_plan(PlanParams P) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int span = P.k1 - P.k0;
  if (gid >= (long long)P.S * span) return;
  const int s = (int)(gid / span), i = P.k0 + (int)(gid % span);
  const double *wl = P.wl + (size_t)s * IGP_WL_NF * P.m;
  const Hw &hw = P.hw_s ? P.hw_s[s] : P.hw;
  int b = -1, u = -1;
  double opnd;
  const int rc = prologue_one(wl, P.m, i, hw, nullptr, b, u, opnd);
  const size_t o = (size_t)s * P.m + i;
  P.batch[o] = b;
  P.lb[o] = u;
  if (P.stream) {
    if (rc) {  // the arrival is rejected
      P.code[o] = rc;
      return;
    }
  } else {
    const int32_t *rk = P.rank + (size_t)s * P.rank_stride;
    P.by_rank[(size_t)s * P.m + rk[i]] = i;
    if (rc) {
      atomicMin(&P.perr[s], i);  // first error in INPUT order (planner.py:280-282)
      return;
    }
  }
  // NonPositiveDenominatorError screen: denom(u) = u*r_unit + k4 is
  // non-decreasing in u and k_act(u) = gamma/denom(u) + k5 is monotone in u
  // (direction = sign of gamma) under round-to-nearest, so the two ends of the
  // reachable range [lb, cap] decide whether any evaluation can raise.
  double cold[C_NF], slot[S_NF];
  entry_consts(wl, P.m, i, b, hw, cold, slot);
  const Solo a = solo_from_cold(cold, (double)u * hw.runit);
  const Solo c = solo_from_cold(cold, (double)hw.cap * hw.runit);
  int fl = (a.err || c.err) ? SF_RISKY : 0;
  // The margin test needs every t_inf term non-negative and finite
  // (validated by WorkloadSpec/Coefficients; raw C-ABI callers might not be).
  if (!(slot[S_TLOAD] >= 0.0) || !(slot[S_TFB] >= 0.0) || !(cold[C_KSCH] >= 0.0) ||
      !(cold[C_NK] >= 0.0) || !(slot[S_ACACHE] >= 0.0) || !(slot[S_ACACHE] <= 1e6) ||
      !isfinite(slot[S_TLOAD] + slot[S_TFB] + slot[S_THALF] + cold[C_KSCH] * cold[C_NK]))
    fl |= SF_NO_MARGIN;
  // the certified-margin kernels' error bound assumes alpha_cache <= FAST_MAX_ACACHE
  if (!(slot[S_ACACHE] <= FAST_MAX_ACACHE)) fl |= SF_NO_FAST;
  if (!(u <= 0xffff)) fl |= SF_RISKY;
  if (P.stream) P.code[o] = fl << 8;
  else if (fl) atomicOr(&P.sflags[s], fl);
}

// warp per scenario: stable counting sort by (-lb, name rank) (planner.py:284)
__global__ void k_sort(PlanParams P) {
  __shared__ int hist[4][257];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int s = blockIdx.x * 4 + w;
  if (s >= P.S) return;
  if (P.perr[s] != INT_MAX) return;
  const int cap = P.hw_s ? P.hw_s[s].cap : P.hw.cap, m = P.m;
  const int32_t *lb = P.lb + (size_t)s * m;
  const int32_t *byr = P.by_rank + (size_t)s * m;
  int32_t *order = P.order + (size_t)s * m;
  int *h = hist[w];
  for (int b = lane; b <= cap; b += 32) h[b] = 0;
  __syncwarp();
  for (int i = lane; i < m; i += 32) atomicAdd(&h[cap - lb[i]], 1);
  __syncwarp();
  if (lane == 0) {
    int acc = 0;
    for (int b = 0; b < cap; ++b) {
      const int c = h[b];
      h[b] = acc;
      acc += c;
    }
  }
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < m; base += 32) {
    const int r = base + lane;
    const bool act = r < m;
    const unsigned am = __ballot_sync(0xffffffffu, act);
    if (act) {
      const int i = byr[r];
      const int key = cap - lb[i];
      const unsigned peers = __match_any_sync(am, key);
      const int before = __popc(peers & lt);
      order[h[key] + before] = i;
      __syncwarp(am);
      if (before == 0) h[key] += __popc(peers);
    }
    __syncwarp();
  }
}

// thread per (scenario, placement position k): cold constants + newcomer record
__global__ void k_build(PlanParams P) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int span = P.k1 - P.k0;
  if (gid >= (long long)P.S * span) return;
  const int s = (int)(gid / span), k = P.k0 + (int)(gid % span);
  const size_t sm = (size_t)s * P.m;
  if (P.stream ? (P.code[sm + k] & 0xff) != 0 : P.perr[s] != INT_MAX) return;
  const int i = P.stream ? k : P.order[sm + k];
  const double *wl = P.wl + (size_t)s * IGP_WL_NF * P.m;
  const Hw &hw = P.hw_s ? P.hw_s[s] : P.hw;
  double cold[C_NF], slot[S_NF];
  const int b = P.batch[sm + i], u = P.lb[sm + i];
  entry_consts(wl, P.m, i, b, hw, cold, slot);
  cold[C_LB] = (double)u;
  cold[C_WIN] = (double)i;
  const Solo so = solo_from_cold(cold, (double)u * hw.runit);
  double *cd = P.cold + (sm + k) * C_NF;
#pragma unroll
  for (int f = 0; f < C_NF; ++f) cd[f] = cold[f];
  double *nw = P.nw + (sm + k) * R_NF;
  nw[R_KA] = so.ka;
  nw[R_CA] = so.ca;
  nw[R_TSN] = (double)so.err;  // the newcomer's solo error code at lb
  nw[R_ACACHE] = slot[S_ACACHE];
  nw[R_TLOAD] = slot[S_TLOAD];
  nw[R_TFB] = slot[S_TFB];
  nw[R_THALF] = slot[S_THALF];
  nw[R_PW] = so.pw;
}

// thread per (scenario, k, v): solo table entry at u = lb + v (model.py:285-297)
__global__ void k_table(PlanParams P) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int span = P.k1 - P.k0;
  if (gid >= (long long)P.S * span * TB) return;
  const long long lk = gid / TB;
  const int v = (int)(gid % TB);
  const int s = (int)(lk / span);
  const long long sk = (long long)s * P.m + P.k0 + (lk % span);
  if (P.stream ? (P.code[sk] & 0xff) != 0 : P.perr[s] != INT_MAX) return;
  const double *cd = P.cold + sk * C_NF;
  const Hw &hw = P.hw_s ? P.hw_s[s] : P.hw;
  const int u = (int)cd[C_LB] + v;
  double *t = P.tbl + (sk * TB + v) * 4;
  if (u > hw.cap) {
    t[0] = t[1] = t[2] = t[3] = 0.0;
    return;
  }
  const Solo so = solo_from_cold(cd, (double)u * hw.runit);
  t[0] = so.ka;
  t[1] = so.pw;
  t[2] = so.ca;
  t[3] = (double)so.err;
}

// ---------------------------------------------------------------------------
// place stage
// ---------------------------------------------------------------------------
struct GroupSmem {
  unsigned int best;  // the step's argmin key so far (KEY_INTER_SHIFT packing)
  unsigned long long tot[5];  // model_evals, eval calls, candidates, resident reads, started
  int err_flag;
  int win_thread;
  int err_gpu;
  int pool_top;
  int abort_code;
  int next;  // persistent scheduling: the scenario this group plans next
};

template <int GW>
__device__ __forceinline__ void group_sync() {
  if (GW == 1) __syncwarp();
  else __syncthreads();
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ Solo solo_lookup(const double *tbl, const double *cold, const Hw &hw,
                                            int k, int lb, int u) {
  const int v = u - lb;
  if (v >= 0 && v < TB && u <= hw.cap) {
    const double *t = tbl + ((size_t)k * TB + v) * 4;
    Solo so;
    so.ka = t[0];
    so.pw = t[1];
    so.ca = t[2];
    so.err = (int)t[3];
    return so;
  }
  return solo_from_cold(cold + (size_t)k * C_NF, (double)u * hw.runit);
}

// Solo terms at L consecutive units u, u+1, ... in one round trip: when they
// are all inside the workload's table row, every 16-byte load is issued before
// any is used (a chain of solo_lookup calls compiles to one dependent table
// load after another); otherwise one solo_lookup per unit.
template <int L>
__device__ __forceinline__ void solo_run(const double *tbl, const double *cold, const Hw &hw, int k,
                                         int lb, int u, Solo *out) {
  const int v = u - lb;
  if (v >= 0 && v + L - 1 < TB && u + L - 1 <= hw.cap) {
    const double2 *t = reinterpret_cast<const double2 *>(tbl + ((size_t)k * TB + v) * 4);
    double2 q[2 * L];
#pragma unroll
    for (int i = 0; i < 2 * L; ++i) q[i] = t[i];
#pragma unroll
    for (int i = 0; i < L; ++i) {
      out[i].ka = q[2 * i].x;
      out[i].pw = q[2 * i].y;
      out[i].ca = q[2 * i + 1].x;
      out[i].err = (int)q[2 * i + 1].y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < L; ++i) out[i] = solo_lookup(tbl, cold, hw, k, lb, u + i);
  }
}

struct ErrOut {
  int code, k;
  double a, b, c;
};

__device__ __forceinline__ void err_operands(const Hw &hw, const double *ce, int u, int code,
                                             ErrOut &eo) {
  const double r = (double)u * hw.runit;
  const double denom = r + ce[C_K4];
  eo.code = code;
  if (code == IGP_E_DENOM) {
    eo.a = denom;
    eo.b = r;
    eo.c = ce[C_K4];
  } else {
    eo.a = ce[C_GAMMA] / denom + ce[C_K5];
    eo.b = ce[C_BATCH];
    eo.c = r;
  }
}

// Modified-resident bitmask of a candidate (positions < MAXN).
template <int MAXN>
struct ModMask {
  static constexpr int W = (MAXN + 63) / 64;
  unsigned long long w[W];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int i = 0; i < W; ++i) w[i] = 0ull;
  }
  __device__ __forceinline__ bool test(int i) const {
    unsigned long long x = w[0];
#pragma unroll
    for (int q = 1; q < W; ++q)
      if ((i >> 6) == q) x = w[q];
    return (x >> (i & 63)) & 1ull;
  }
  __device__ __forceinline__ void set(int i) {
#pragma unroll
    for (int q = 0; q < W; ++q)
      if ((i >> 6) == q) w[q] |= 1ull << (i & 63);
  }
};

// One warp moves GPU j (now holding desc, slack b) from slack a > b down the
// slack order: j swaps with the last GPU of each bucket a, a-1, ..., b+1.
// All positions come from the counts before the move, so the swaps run in
// parallel; a bucket that is empty makes its swap a no-op.
__device__ __forceinline__ void slack_move_down(int32_t *sj, int32_t *spos,
                                                unsigned long long *sdesc, int32_t *sE, int j,
                                                unsigned long long desc, int a, int b, int lane) {
  const int steps = a - b;
  const int p0 = spos[j];
  __syncwarp();
  for (int c0 = 0; c0 < steps; c0 += 32) {
    const int i = c0 + lane;
    int q = 0, dst = 0, xj = 0;
    unsigned long long xd = 0;
    if (i < steps) {
      const int sb = a - i;
      q = sE[sb] - 1;
      dst = i == 0 ? p0 : sE[sb + 1] - 1;
      if (q != dst) {  // an empty bucket makes the swap a no-op
        xj = sj[q];
        xd = sdesc[q];
      }
    }
    __syncwarp();
    if (i < steps && q != dst) {
      sj[dst] = xj;
      sdesc[dst] = xd;
      spos[xj] = dst;
    }
    __syncwarp();
  }
  if (lane == 0) {
    const int pf = sE[b + 1] - 1;
    sj[pf] = j;
    sdesc[pf] = desc;
    spos[j] = pf;
  }
  __syncwarp();
  for (int i = lane; i < steps; i += 32) sE[a - i] -= 1;
  __syncwarp();
}

// One warp appends the new GPU j (= G, slack s) and moves it up the order:
// it swaps with the first GPU of each bucket 0, 1, ..., s-1.
__device__ __forceinline__ void slack_insert(int32_t *sj, int32_t *spos,
                                             unsigned long long *sdesc, int32_t *sE, int j,
                                             unsigned long long desc, int s, int lane) {
  for (int c0 = 0; c0 < s; c0 += 32) {
    const int i = c0 + lane;
    int u = 0, dst = 0, xj = 0;
    unsigned long long xd = 0;
    if (i < s) {
      u = sE[i + 1];
      dst = i == 0 ? j : sE[i];
      if (u != dst) {  // an empty bucket makes the swap a no-op
        xj = sj[u];
        xd = sdesc[u];
      }
    }
    __syncwarp();
    if (i < s && u != dst) {
      sj[dst] = xj;
      sdesc[dst] = xd;
      spos[xj] = dst;
    }
    __syncwarp();
  }
  if (lane == 0) {
    const int pf = s > 0 ? sE[s] : j;
    sj[pf] = j;
    sdesc[pf] = desc;
    spos[j] = pf;
    sE[0] = j + 1;
  }
  __syncwarp();
  for (int i = lane; i < s; i += 32) sE[i + 1] += 1;
  __syncwarp();
}

template <bool B>
struct BoolC {
  static constexpr bool value = B;
};
template <int V>
struct IntC {
  static constexpr int value = V;
};

template <int MAXN>
struct LaneArrays {  // values of residents bumped inside the current candidate
  int u[MAXN];
  double ka[MAXN], pw[MAXN], ca[MAXN];
};

// One scenario per group of GW warps (GW == 1: four scenarios per 128-thread
// CTA; GW > 1: one scenario per CTA).
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long *p) {
  return __ldcg(p);
}
__device__ __forceinline__ int ld_cg(const int *p) { return __ldcg(p); }
__device__ __forceinline__ unsigned ld_cg(const unsigned *p) { return __ldcg(p); }

// next-unit solo terms of pool record ri (variables nxt / rec in scope)
#if IGP_SPLIT_NEXT
#define NEXT_AT(ri) (nxt + (size_t)(ri) * 4)
#else
#define NEXT_AT(ri) (rec + (size_t)(ri) * R_NF + R_KA1)
#endif

// Everything the commit of a step touches in one scenario's state.
struct ScenState {
  const double *cold, *tbl;
  unsigned long long *gstate, *sdesc;
  int32_t *sj, *spos, *sE, *gcap;
  double *gfold, *rec, *nxt, *frec, *pfx;
  Meta *meta;
  size_t sm;  // scenario offset of the [S][m] outputs
};

// The commit of step k (planner.py:312-319), run by one warp: open a new GPU
// at [need] when no candidate fits (bk == NO_KEY), else append the newcomer to
// GPU j = bk's low bits with the winner's unit vector lu (residents' units,
// then the newcomer's).  Updates the tile (grown by copying when full), the
// next-unit terms, the fold stream and prefix fold states, the tile header,
// the GPU descriptor and fold state, and the slack order.
__device__ __forceinline__ void commit_step(const PlanParams &P, const Hw &hw, const ScenState &Z,
                                         int k, int need, unsigned bk, const uint16_t *lu,
                                         int G, int *poolp, int *abortp, const double *nwv,
                                         double ksch, double nkern, int lane) {
  constexpr unsigned NO_KEY = 0xffffffffu;
  constexpr unsigned FULL = 0xffffffffu;
  const int cap = hw.cap;
  const double *cold = Z.cold, *tbl = Z.tbl;
  unsigned long long *gstate = Z.gstate, *sdesc = Z.sdesc;
  int32_t *sj = Z.sj, *spos = Z.spos, *sE = Z.sE, *gcap = Z.gcap;
  double *gfold = Z.gfold, *rec = Z.rec, *frec = Z.frec, *pfx = Z.pfx;
  Meta *meta = Z.meta;
  const size_t sm = Z.sm;
  const double nw_ka = nwv[R_KA], nw_ca = nwv[R_CA], nw_pw = nwv[R_PW];
  const double nw_acache = nwv[R_ACACHE], nw_tload = nwv[R_TLOAD];
  const double nw_tfb = nwv[R_TFB], nw_thalf = nwv[R_THALF];
#if IGP_SPLIT_NEXT
  double *nxt = Z.nxt;
#endif
  if (bk == NO_KEY) {
    if (lane == 0) {
      const int off = *poolp + 1;  // records after the header slot
      if (off + TILE0 > P.pool_recs) {
        *abortp = IGP_E_CAPACITY;
      } else {
        *poolp = off + TILE0;
        gcap[G] = TILE0;
        gstate[G] = ((unsigned long long)off << 32) | (unsigned)need | (1u << 16);
        double *r = rec + (size_t)off * R_NF;
        r[R_KA] = nw_ka;
        r[R_CA] = nw_ca;
        r[R_TSN] = (ksch + delta_sch(hw, 2)) * nkern;
        r[R_ACACHE] = nw_acache;
        r[R_TLOAD] = nw_tload;
        r[R_TFB] = nw_tfb;
        r[R_THALF] = nw_thalf;
        r[R_PW] = nw_pw;
        {
          const Solo s1 = solo_lookup(tbl, cold, hw, k, need, need + 1);
          double *nx = NEXT_AT(off);
          nx[0] = s1.ka;
          nx[1] = s1.pw;
          nx[2] = s1.ca;
          nx[3] = (double)s1.err;
        }
        frec[(size_t)off * 2] = nw_pw;
        frec[(size_t)off * 2 + 1] = nw_ca;
        double *pp = pfx + (size_t)off * 4;
        pp[0] = pp[1] = pp[2] = pp[3] = 0.0;
        meta[off] = Meta{k, (uint16_t)need, (uint16_t)need};
        Neumaier fp, fc;
        fp.first(nw_pw);
        fc.first(nw_ca);
        double *gf = gfold + (size_t)G * 4;
        gf[0] = fp.s;
        gf[1] = fp.c;
        gf[2] = fc.s;
        gf[3] = fc.c;
        TileHeader *hd = reinterpret_cast<TileHeader *>(rec + (size_t)(off - 1) * R_NF);
        hd->gf[0] = fp.s;
        hd->gf[1] = fp.c;
        hd->gf[2] = fc.s;
        hd->gf[3] = fc.c;
        hd->meta[0] = meta[off];
        hd->meta[1] = hd->meta[2] = hd->meta[3] = Meta{0, 0, 0};  // staged by tile copies
        if (P.stream) {
          P.gpu_of[sm + k] = G;
          P.pos[sm + k] = 0;
        }
      }
    }
    __syncwarp();
    if (*(volatile int *)abortp == 0)
      slack_insert(sj, spos, sdesc, sE, G, gstate[G], cap - need, lane);
  } else {
    const int j = (int)(bk & 0x7fffffu);
    const int nres = (int)((gstate[j] >> 16) & 0xffffu);
    const int occ_old = (int)(gstate[j] & 0xffffu);
    const int n = nres + 1;
    int off = (int)(gstate[j] >> 32);
    const int tcap = gcap[j];
    if (n > tcap) {  // grow the tile: copy it to a fresh one of twice the size
      int noff = 0;
      if (lane == 0) {
        noff = *poolp + 1;  // records after the header slot
        if (noff + 2 * tcap > P.pool_recs) *abortp = IGP_E_CAPACITY;
        else *poolp = noff + 2 * tcap;
      }
      noff = __shfl_sync(FULL, noff, 0);
      __syncwarp();
      if (*(volatile int *)abortp == 0) {
        for (int r = lane; r < nres; r += 32) {
#pragma unroll
          for (int f = 0; f < R_NF; ++f)
            rec[(size_t)(noff + r) * R_NF + f] = rec[(size_t)(off + r) * R_NF + f];
#if IGP_SPLIT_NEXT
#pragma unroll
          for (int f = 0; f < 4; ++f) NEXT_AT(noff + r)[f] = NEXT_AT(off + r)[f];
#endif
          frec[(size_t)(noff + r) * 2] = frec[(size_t)(off + r) * 2];
          frec[(size_t)(noff + r) * 2 + 1] = frec[(size_t)(off + r) * 2 + 1];
          meta[noff + r] = meta[off + r];
        }
        if (lane == 0) gcap[j] = 2 * tcap;
        off = noff;
      }
      __syncwarp();
    }
    if (*(volatile int *)abortp == 0) {
      const double dnext = delta_sch(hw, n + 1);
      int part = 0;
      // fold inputs and meta of resident `lane`, handed to the prefix fold
      // below by shuffles instead of re-reading them from the pool
      double f_pw = 0.0, f_ca = 0.0;
      unsigned long long f_mt = 0ull;
      for (int r = lane; r < n; r += 32) {
        const int nu = lu[r];
        double *rr = rec + (size_t)(off + r) * R_NF;
        if (r < nres) {
          Meta mt = meta[off + r];
          if (nu == (int)mt.u && r < 32) {
            const double2 fv = *reinterpret_cast<const double2 *>(frec + (size_t)(off + r) * 2);
            f_pw = fv.x;
            f_ca = fv.y;
          }
          if (nu != (int)mt.u) {
            Solo sr[2];
            solo_run<2>(tbl, cold, hw, mt.k, mt.lb, nu, sr);
            const Solo so = sr[0], s1 = sr[1];
            rr[R_KA] = so.ka;
            rr[R_CA] = so.ca;
            rr[R_PW] = so.pw;
            double *nx = NEXT_AT(off + r);
            nx[0] = s1.ka;
            nx[1] = s1.pw;
            nx[2] = s1.ca;
            nx[3] = (double)s1.err;
            frec[(size_t)(off + r) * 2] = so.pw;
            frec[(size_t)(off + r) * 2 + 1] = so.ca;
            mt.u = (uint16_t)nu;
            meta[off + r] = mt;
            if (r < 32) {
              f_pw = so.pw;
              f_ca = so.ca;
            }
          }
          if (r < 32) f_mt = *reinterpret_cast<const unsigned long long *>(&mt);
          const double *ce = cold + (size_t)mt.k * C_NF;
          rr[R_TSN] = (ce[C_KSCH] + dnext) * ce[C_NK];
        } else {
          const Solo so = (nu == need) ? Solo{nw_ka, nw_pw, nw_ca, 0}
                                       : solo_lookup(tbl, cold, hw, k, need, nu);
          const Solo s1 = solo_lookup(tbl, cold, hw, k, need, nu + 1);
          rr[R_KA] = so.ka;
          rr[R_CA] = so.ca;
          rr[R_PW] = so.pw;
          double *nx = NEXT_AT(off + r);
          nx[0] = s1.ka;
          nx[1] = s1.pw;
          nx[2] = s1.ca;
          nx[3] = (double)s1.err;
          rr[R_TSN] = (ksch + dnext) * nkern;
          rr[R_ACACHE] = nw_acache;
          rr[R_TLOAD] = nw_tload;
          rr[R_TFB] = nw_tfb;
          rr[R_THALF] = nw_thalf;
          frec[(size_t)(off + r) * 2] = so.pw;
          frec[(size_t)(off + r) * 2 + 1] = so.ca;
          const Meta mt{k, (uint16_t)nu, (uint16_t)need};
          meta[off + r] = mt;
          if (r < 32) {
            f_pw = so.pw;
            f_ca = so.ca;
            f_mt = *reinterpret_cast<const unsigned long long *>(&mt);
          }
        }
        part += nu;
      }
      part = warp_sum(part);
      __syncwarp();
      // prefix fold states of this GPU, in resident order (every lane folds
      // the shuffled terms identically; lane 0 stores them)
      Neumaier fp, fc;
      fp.s = fp.c = fc.s = fc.c = 0.0;
      for (int r = 0; r < n; ++r) {
        double pw, ca;
        if (r < 32) {
          pw = __shfl_sync(FULL, f_pw, r);
          ca = __shfl_sync(FULL, f_ca, r);
        } else {
          pw = frec[(size_t)(off + r) * 2];
          ca = frec[(size_t)(off + r) * 2 + 1];
        }
        if (lane == 0) {
          double *pp = pfx + (size_t)(off + r) * 4;
          pp[0] = fp.s;
          pp[1] = fp.c;
          pp[2] = fc.s;
          pp[3] = fc.c;
        }
        fp.add(pw);
        fc.add(ca);
      }
      unsigned long long hmeta[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) hmeta[r] = __shfl_sync(FULL, f_mt, r);
      if (lane == 0) {
        gstate[j] = ((unsigned long long)off << 32) | (unsigned)part | ((unsigned)n << 16);
        double *gf = gfold + (size_t)j * 4;
        gf[0] = fp.s;
        gf[1] = fp.c;
        gf[2] = fc.s;
        gf[3] = fc.c;
        TileHeader *hd = reinterpret_cast<TileHeader *>(rec + (size_t)(off - 1) * R_NF);
        hd->gf[0] = fp.s;
        hd->gf[1] = fp.c;
        hd->gf[2] = fc.s;
        hd->gf[3] = fc.c;
        for (int r = 0; r < 4; ++r)  // entries past n are zero (staged by tile copies)
          *reinterpret_cast<unsigned long long *>(&hd->meta[r]) = hmeta[r];
        if (P.stream) {
          P.gpu_of[sm + k] = j;
          P.pos[sm + k] = nres;
        }
      }
      __syncwarp();
      slack_move_down(sj, spos, sdesc, sE, j,
                      ((unsigned long long)off << 32) | (unsigned)part | ((unsigned)n << 16),
                      cap - occ_old, cap - part, lane);
    }
  }
}

// MINB > 0 overrides the resident-CTA target of the one-warp kernel: 5 CTAs
// (20 warps/SM, 102 registers) for large plans, where more resident scenarios
// hide more latency (+6.5% at 10k workloads); the default 4 (128 registers,
// fewer spills) wins on short plans (1k workloads: 81k vs 76k plans/s).
// LEAN: a batch pass compiled without the exact evaluation sequence (PlanStats,
// inputs that can raise): those scenarios are left to a second, full pass
// (Hand.k_done = k0); the rest are planned completely (k_done = HAND_COMPLETE).
// The exact-sequence code no longer shares the hot loop's registers (spills
// 172 instead of 400 bytes at 96 registers).
template <int MAXN, int GW, bool COOP = false, bool HWS = false, int MINB = 0, bool LEAN = false>
__global__ void __launch_bounds__(GW == 1 ? 128 : GW * 32,
                                  MINB ? MINB
                                       : GW == 1 ? IGP_MINB_WARP
                                                 : GW == 2 ? 8 : GW == 4 ? 4 : IGP_MINB_CTA)
k_place(PlanParams P) {
  static_assert(!COOP || GW == 1, "cooperative mode runs one group per warp");
  static_assert(!(COOP && HWS), "a cooperative plan has one hardware profile");
  constexpr int GT = GW * 32;
  constexpr int GPB = (GW == 1) ? 4 : 1;
  // Candidate keys (inter, j) packed into 32 bits, inter << 23 | j: lexicographic
  // order is integer order, so the argmin is a native 32-bit atomicMin
  // (the 64-bit one on shared memory is a CAS loop).  Needs j < 2^23 and
  // inter < 2^9, which igp_plan_* enforce (m < 2^23, max_units <= 256).
  constexpr unsigned NO_KEY = 0xffffffffu;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ GroupSmem gsm[GPB];
  __shared__ __align__(16) double ntb[GPB][TB * 4];  // the newcomer's solo table row
  __shared__ unsigned long long nbar[GPB];          // its bulk copy's mbarrier
  __shared__ Hw shw[HWS ? GPB : 1];                 // IGP_F_HWS: the scenario's profile
#if IGP_NW_SMEM
  __shared__ double nwsm[GPB][R_NF + 2];            // the step's newcomer record, k_sch, n_k
#endif
  extern __shared__ __align__(16) unsigned char dsm[];
  const int grp = threadIdx.x / GT, t = threadIdx.x % GT, wi = t / 32, lane = t % 32;
  GroupSmem &gs = gsm[grp];
  LaneSlot *const sl = reinterpret_cast<LaneSlot *>(dsm) + threadIdx.x;
  unsigned long long *const lbar =
      reinterpret_cast<unsigned long long *>(dsm + blockDim.x * sizeof(LaneSlot)) + threadIdx.x;
  mbar_init(lbar);
  if (t == 0) mbar_init(&nbar[grp]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
#if IGP_TILE_LDGSTS < 2
  uint32_t c_phase = 0;  // parity of this lane's mbarrier
#endif
  uint32_t n_phase = 0;  // parity of the group's newcomer-row mbarrier
  CoopState *const cs = P.coop;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;      // cooperative lane id
  // Persistent groups: each pulls the next scenario when it finishes one, so
  // scenarios of unequal length do not leave SMs idle at the end.
  for (int pass = 0;; ++pass) {
  int s;
  if constexpr (COOP) {
    if (pass) break;
    s = 0;
  } else {
    if (t == 0) gs.next = atomicAdd(P.sched, 1);
    group_sync<GW>();
    s = gs.next;
    group_sync<GW>();
    if (s >= P.S) break;
  }
  double *ntab = ntb[grp];
  if constexpr (HWS) {
    if (t == 0) shw[grp] = P.hw_s[s];
    group_sync<GW>();
  }
  const Hw &hw = *(HWS ? &shw[grp] : &P.hw);
  const int m = P.m, cap = hw.cap;
  const size_t sm = (size_t)s * m;
  igp_error *err = P.err + s;

  if constexpr (!COOP) {
    if (P.hand) {
      if constexpr (LEAN) {  // the exact sequence is the full pass's
        const bool decline =
            P.perr[s] != INT_MAX || (P.sflags[s] & SF_RISKY) || (P.flags & IGP_F_STATS);
        if (t == 0) P.hand[s].k_done = decline ? P.k0 : HAND_COMPLETE;
        if (decline) continue;
      } else if (ld_cg(&P.hand[s].k_done) == HAND_COMPLETE) {
        continue;  // planned by the lean pass
      }
    }
  }

  if (!P.stream && P.perr[s] != INT_MAX) {  // prologue error, input order (planner.py:280-282)
    if (t == 0) {
      const int i = P.perr[s];
      int b, u;
      double opnd = 0.0;
      const double *wl = P.wl + (size_t)s * IGP_WL_NF * m;
      const int rc = prologue_one(wl, m, i, hw, nullptr, b, u, opnd);
      err->code = rc;
      err->workload = i;
      err->gpu = -1;
      err->a = opnd;
      err->b = (double)hw.b_max;
      err->c = 0.0;
      P.gpu_count[s] = 0;
      if (P.stats) {
        const long long z = (P.flags & IGP_F_STATS) ? 0 : -1;
        P.stats[IGP_NSTAT * s] = z;
        P.stats[IGP_NSTAT * s + 1] = z;
        P.stats[IGP_NSTAT * s + 2] = z;
        P.stats[IGP_NSTAT * s + 3] = 0;
        P.stats[IGP_NSTAT * s + 4] = z;
        P.stats[IGP_NSTAT * s + 5] = 0;
      }
    }
    continue;
  }

  const double *cold = P.cold + sm * C_NF;
  const double *nwt = P.nw + sm * R_NF;
  const double *tbl = P.tbl + sm * TB * 4;
  unsigned long long *gstate = P.gstate + (size_t)s * P.gstride;
  unsigned long long *sdesc = P.sdesc + (size_t)s * P.gstride;
  int32_t *sj = P.sj + sm, *spos = P.spos + sm, *sE = P.sE + (size_t)s * (P.cap_ld + 2);
  int32_t *gcap = P.gcap + sm;
  double *gfold = P.gfold + sm * 4;
  const size_t sp = (size_t)s * (size_t)P.pool_recs;
  double *rec = P.rec + sp * R_NF;
#if IGP_SPLIT_NEXT
  double *nxt = P.nxt + sp * 4;
#endif
  double *frec = P.frec + sp * 2;
  double *pfx = P.pfx + sp * 4;
  Meta *meta = P.meta + sp;
  uint16_t *lane_units = P.lane_units + (size_t)s * P.lanes * P.cap_ld;
  int32_t *sst = P.stream ? P.sstate + 4 * (size_t)s : nullptr;
  // stream mode: risk flags of admitted arrivals stick to the scenario
  int sflags = P.stream ? sst[2] : P.sflags[s];
  if constexpr (COOP) {
    // the exact evaluation sequence (PlanStats, a scenario that can raise)
    // runs in the per-CTA kernel; so does a scenario with a prologue error
    if ((!P.stream && P.perr[0] != INT_MAX) || (sflags & SF_RISKY) || (P.flags & IGP_F_STATS)) {
      if (gtid == 0) cs->status = P.k0;
      return;
    }
  }
  // steps the cooperative kernel already ran: resume after them (plan mode:
  // all of them, only the predictions remain; stream mode: up to the first
  // arrival that needs the exact sequence)
  int k_coop = (!COOP && P.coop) ? ld_cg(&P.coop->status) : P.k0;
  const bool coop_done = !COOP && P.coop && k_coop > P.k0;
  if (coop_done) sflags |= P.coop->sflags;
  // steps the certified-margin fast kernel ran (fast.cuh): plan mode, all of
  // them or none; the predictions and outputs below remain
  const Hand *const hdp = (!COOP && P.hand) ? P.hand + s : nullptr;
  const bool fast_done = !LEAN && hdp && !coop_done && hdp->k_done > P.k0;
  if (fast_done) k_coop = hdp->k_done;
  const bool resumed = coop_done || fast_done;
  const unsigned lt = (1u << lane) - 1u;

  LaneArrays<MAXN> L;
  ModMask<MAXN> mod;
  int G = coop_done ? P.coop->G : fast_done ? hdp->G : (P.stream ? sst[0] : 0);
  if (!COOP && G == 0) {  // empty slack order (the cooperative launch zeroes it on the host side)
    for (int x = t; x < cap + 2; x += GT) sE[x] = 0;
  }
  long long tot_evals = 0, tot_calls = 0, tot_cands = 0, tot_rres = 0, tot_run = 0;
  // per-step counters (one lane's share); only exact steps keep the
  // PlanStats-only ones
  int st_evals = 0, st_calls = 0, st_cands = 0, st_rres = 0, st_run = 0;
  int fail_code = 0;
  ErrOut eo_fail;
  eo_fail.code = 0;
  eo_fail.k = -1;
  int *poolp = &gs.pool_top, *abortp = &gs.abort_code;
  if constexpr (COOP) {
    poolp = &cs->pool_top;
    abortp = &cs->abort;
  } else if (t == 0) {
    gs.pool_top = coop_done ? P.coop->pool_top
                  : fast_done ? hdp->pool_top
                              : (P.stream ? sst[1] : 0);
    gs.abort_code = coop_done ? P.coop->abort : fast_done ? hdp->abort : 0;
  }
  group_sync<GW>();
  if (resumed && t == 0) {
    tot_run = (long long)(coop_done ? P.coop->cands_run : hdp->cands_run);
    tot_calls = (long long)(coop_done ? P.coop->evals_run : hdp->evals_run);
  }
  if (!COOP && gs.abort_code) fail_code = 2;  // the cooperative / fast steps ran out of pool
  int q = 0;          // cooperative mode: steps processed by this launch (slot parity)
  int k_stop = P.k1;  // cooperative mode: the first step left to the per-CTA kernel

  for (int k = resumed ? k_coop : P.k0; k < P.k1 && !fail_code; ++k) {
    int aflags = 0;  // this arrival's risk flags (stream mode)
    if (P.stream) {
      const int c = P.code[sm + k];
      if (c & 0xff) {  // rejected by the prologue
        if (t == 0) {
          P.gpu_of[sm + k] = -1;
          P.pos[sm + k] = -1;
          P.units[sm + k] = 0;
        }
        continue;
      }
      aflags = c >> 8;
    }
    if constexpr (COOP) {
      if ((sflags | aflags) & SF_RISKY) {  // the exact sequence: left to the per-CTA kernel
        k_stop = k;
        break;
      }
    }
    const bool exact = !LEAN && ((P.flags & IGP_F_STATS) || ((sflags | aflags) & SF_RISKY));
    const bool margin_rt = !((sflags | aflags) & SF_NO_MARGIN) && hw.margin_ok;
    // the newcomer (planner.py:291-292)
#if IGP_TIMING
    long long tm0 = clock64();
#endif
    const double *ck = cold + (size_t)k * C_NF;
    const double *nk_rec = nwt + (size_t)k * R_NF;
    const int need = (int)ck[C_LB];
#if IGP_NW_SMEM
    // the newcomer's record lives in shared memory for the step (read where
    // used instead of pinning ten doubles in registers across the step loop)
    double *nws = nwsm[grp];
    if (t < R_NF + 2) nws[t] = t < R_NF ? nk_rec[t] : ck[t == R_NF ? C_KSCH : C_NK];
    const double &ksch = nws[R_NF], &nkern = nws[R_NF + 1];
    const double &nw_ka = nws[R_KA], &nw_ca = nws[R_CA], &nw_pw = nws[R_PW];
    const double &nw_acache = nws[R_ACACHE], &nw_tload = nws[R_TLOAD];
    const double &nw_tfb = nws[R_TFB], &nw_thalf = nws[R_THALF];
#else
    const double ksch = ck[C_KSCH], nkern = ck[C_NK];
    const double nw_ka = nk_rec[R_KA], nw_ca = nk_rec[R_CA], nw_pw = nk_rec[R_PW];
    const double nw_acache = nk_rec[R_ACACHE], nw_tload = nk_rec[R_TLOAD];
    const double nw_tfb = nk_rec[R_TFB], nw_thalf = nk_rec[R_THALF];
#endif
    const int nw_err = (int)nk_rec[R_TSN];
    if (t == 0) {
      gs.best = NO_KEY;
      gs.err_flag = 0;
    }
    if (t == 0) {  // the newcomer's solo row: waited for only by a newcomer bump
      fence_async_smem();  // last step's reads of ntab before the async overwrite
      mbar_expect_tx(&nbar[grp], TB * 32);
      bulk_g2s(ntab, tbl + (size_t)k * TB * 4, TB * 32, &nbar[grp]);
    }
    bool n_ready = false;
    group_sync<GW>();
    unsigned my_best = NO_KEY;
    const int ncand = sE[need];  // candidates: the slack-order prefix with slack >= need
#if IGP_TIMING
    long long tm1 = clock64() + ncand * 0;
#endif

    // ---- the step's candidates: per-lane state machine with dynamic refill ----
    // A lane owns at most one candidate GPU.  One loop iteration advances every
    // busy lane by one resident check of Alg. 2 (planner.py:152-161), plus the
    // evaluation it needs first and the unit bump it may cause.  Idle lanes
    // are refilled from a per-warp ring queue fed by a coalesced prefilter
    // scan (planner.py:297-299), in ascending j, so early (low-j, low-inter)
    // keys prune later candidates and lanes never wait for a round's longest
    // candidate.  serial != 0 replays the step in the reference's order on
    // lane 0 of warp 0 only (exact mode, to locate the first raising candidate).
    // serial and exact are compile-time per instantiation, so the common
    // pruned step carries none of the exact-mode bookkeeping
    auto run_step = [&](auto serial_c, auto exact_c, auto margin_c) {
      constexpr bool serial = decltype(serial_c)::value;
      constexpr bool exact = decltype(exact_c)::value;
      // the pruned step also fixes the division shortcut's margin test
      constexpr int MG = decltype(margin_c)::value;  // 0 off, 1 on, 2 runtime
      const bool margin = MG == 2 ? margin_rt : MG == 1;
      int qhead = 0;
      int scan = 0;  // serial replay: next GPU index to test
      // cooperative mode: this lane's next candidate position; consecutive
      // positions go to consecutive CTAs so a step's candidates spread over all SMs
      int c_static = (int)(threadIdx.x * gridDim.x + blockIdx.x);
      const unsigned take_mask = serial ? 1u : FULL;
      int cj = -1, c_nres = 0, c_occ = 0, c_sum = 0, c_i = 0, c_dirty = 0, c_off = 0;
      int c_pend = -1, c_pcode = 0, c_nu = 0;
#if IGP_PF_BATCH
      int pf_pos = INT_MAX;          // a next-refill position whose tile to prefetch
      unsigned long long pf_desc = 0;
#endif
      unsigned c_sb = 0;  // staged residents already bumped inside this candidate
      bool c_flag = false, c_need = false, c_wait = false;
      double c_C = 0.0, c_f = 0.0, c_inv = 1.0, c_tsn = 0.0;
      bool c_one = true;  // f == F: scale = F / F = 1.0 and x / 1.0 == x
      double c_nka = 0.0, c_npw = 0.0, c_nca = 0.0;
      bool stop = false;

      auto finish = [&](int result) {
        if (result == R_ERROR) {
          atomicOr(&gs.err_flag, 1);
          if (serial) {
            int ek, eu;
            if (c_pend == c_nres) {
              ek = k;
              eu = c_nu;
            } else if (c_pend < SLOT) {
              const Meta mt = sl->meta[c_pend];
              ek = mt.k;
              eu = (int)mt.u;
            } else {
              const Meta mt = meta[c_off + c_pend];
              ek = mt.k;
              eu = mod.test(c_pend) ? L.u[c_pend] : (int)mt.u;
            }
            err_operands(hw, cold + (size_t)ek * C_NF, eu, c_pcode, eo_fail);
            eo_fail.k = ek;
            stop = true;
          }
        } else if (result == R_FEAS) {
          const unsigned key = ((unsigned)(c_sum - c_occ) << 23) | (unsigned)cj;
          if (key < my_best) {
            my_best = key;
            if constexpr (COOP) P.win_tid[cj] = gtid;
            uint16_t *lu = lane_units + (size_t)(COOP ? gtid : t) * cap;
            for (int qq = 0; qq < c_nres; ++qq)
              lu[qq] = qq < SLOT ? sl->meta[qq].u
                                 : (mod.test(qq) ? (uint16_t)L.u[qq] : meta[c_off + qq].u);
            lu[c_nres] = (uint16_t)c_nu;
          }
          atomicMin(&gs.best, key);
          if constexpr (COOP) atomicMin(&cs->best[q & 1], key);
        }
        cj = -1;
      };

      while (true) {
        // warp-uniform stop (set by the serial replay's first raising candidate)
        if (serial && __any_sync(FULL, stop)) break;
        const unsigned idle = __ballot_sync(FULL, cj < 0) & take_mask;
#ifndef IGP_REFILL_MIN
#define IGP_REFILL_MIN 28
#endif
        // One-warp scenarios refill idle lanes in batches: the new candidates'
        // tile copies then overlap, instead of each single refill exposing its
        // own latency to the whole warp (+4.6% at 24 of 32 over single
        // refills; 28 a further +0.6%, 20 -0.6%).  A warp with no busy lane
        // always refills.
        constexpr int refill_min = (GW == 1 && !COOP) ? IGP_REFILL_MIN : 1;
        if (idle && (serial || __popc(idle) >= refill_min || idle == (FULL & take_mask))) {
          const int nidle = __popc(idle);
          if constexpr (COOP) {  // the other warps' results prune this warp's candidates
            if (lane == 0) atomicMin(&gs.best, ld_cg(&cs->best[q & 1]));
            __syncwarp();
          }
          // the step's candidates are the slack-order prefix [0, ncand): idle
          // lanes take the next positions
          int cbase = qhead;
          if (!serial) {
            if constexpr (COOP) {
              cbase = 0;
            }
          }
          if ((idle >> lane) & 1u) {
            const int r = __popc(idle & lt);
            // several warps per scenario: positions interleave over the warps,
            // so a step's few candidates spread out instead of filling one warp
            int cpos = GW > 1 ? wi + GW * (cbase + r) : cbase + r;
            if (COOP && !serial) {
              cpos = c_static;
              c_static += (int)(gridDim.x * blockDim.x);
            }
            int j = 0;
            unsigned long long g = 0;
            bool have;
            if (serial) {
              // the serial replay (lane 0 only) follows the reference's candidate
              // order: ascending j through the prefilter (planner.py:296-299)
              while (scan < G && (int)(gstate[scan] & 0xffffu) + need > cap) ++scan;
              have = scan < G;
              if (have) {
                j = scan;
                g = gstate[scan];
                ++scan;
              }
            } else {
              have = cpos < ncand;
              if (have) {
                j = sj[cpos];
                g = sdesc[cpos];
              }
            }
            if (have) {
              if (exact) st_cands += 1;
              const volatile unsigned *bp = &gs.best;
              if (exact || (((unsigned)need << 23) | (unsigned)j) <= *bp) {
                // residents_j + [newcomer] (planner.py:302-304)
                cj = j;
                c_occ = (int)(g & 0xffffu);
                c_nres = (int)((g >> 16) & 0xffffu);
                c_off = (int)(g >> 32);
                if (exact) st_rres += c_nres;
                st_run += 1;
                {  // stage the tile header and the first SLOT records: one bulk copy
                  const int nst = c_nres < SLOT ? c_nres : SLOT;
#if IGP_TILE_LDGSTS
                  {
                    const char *src = reinterpret_cast<const char *>(rec + (size_t)(c_off - 1) * R_NF);
                    char *dst = reinterpret_cast<char *>(sl->gf);
                    constexpr int CPR = R_NF * 8 / 16;  // 16-byte chunks per record
                    const int nch = (1 + nst) * CPR;
#pragma unroll
                    for (int c = 0; c < (1 + SLOT) * CPR; ++c)
                      if (c < nch) cp_async16(dst + 16 * c, src + 16 * c);
#if IGP_TILE_LDGSTS == 2
                    cp_async_commit();
#else
                    cp_async_arrive(lbar);
#endif
                  }
#else
                  const uint32_t bytes = (uint32_t)(1 + nst) * (R_NF * 8);
                  fence_async_smem();
                  mbar_expect_tx(lbar, bytes);
                  bulk_g2s(sl->gf, rec + (size_t)(c_off - 1) * R_NF, bytes, lbar);
#endif
                  c_wait = true;
#if IGP_SPLIT_NEXT && IGP_PF_NEXT
                  // the staged residents' next-unit terms, read on their first
                  // bump: L2 prefetch of their lines.  +1.5% at the headline
                  // for +0.68 TB (+22%) of DRAM reads per launch, most of it
                  // for residents that are never bumped; HBM runs at ~37% of
                  // peak here, so latency, not bandwidth, is the binding cost.
                  // (L1 line prefetch: +1.2%; an exact-size bulk L2 prefetch:
                  // -0.5%; prefetching residents beyond the slot or the next
                  // newcomer: noise.)
                  asm volatile("prefetch.global.L2 [%0];" ::"l"(NEXT_AT(c_off)));
                  asm volatile("prefetch.global.L2 [%0];" ::"l"(NEXT_AT(c_off + nst - 1)));
#endif

                }
                c_sum = c_occ + need;
                c_i = 0;
                c_dirty = c_nres;
                c_flag = false;
                c_need = true;
                c_nu = need;
                c_nka = nw_ka;
                c_npw = nw_pw;
                c_nca = nw_ca;
                c_tsn = (ksch + delta_sch(hw, c_nres + 1)) * nkern;
                mod.clear();
                c_sb = 0;
                c_pend = -1;
                if (exact) {
                  for (int qq = 0; qq < c_nres && c_pend < 0; ++qq) {
                    const Meta mt = meta[c_off + qq];
                    const Solo so = solo_lookup(tbl, cold, hw, mt.k, mt.lb, mt.u);
                    if (so.err) {
                      c_pend = qq;
                      c_pcode = so.err;
                    }
                  }
                  if (c_pend < 0 && nw_err) {
                    c_pend = c_nres;
                    c_pcode = nw_err;
                  }
                }
              }
            }
          }
          qhead += nidle;
#if IGP_PF_DESC
          // the next refill's slack-order descriptors: into L1 now, so the
          // next refill's sj / sdesc loads do not wait on L2 or DRAM
          if constexpr (GW == 1 && !COOP && !serial) {
            const int pp = qhead + lane;
            if (pp < ncand && (lane & 7) == 0) {
              asm volatile("prefetch.global.L1 [%0];" ::"l"(sdesc + pp));
              if ((lane & 15) == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(sj + pp));
            }
          }
#endif
#if IGP_PF_BATCH
          // the next refill's candidates: load their descriptors now (used
          // only after this iteration's tile waits, so the load is not on the
          // critical path) and prefetch their tiles into L2 below
          if constexpr (GW == 1 && !COOP && !serial) {
            pf_pos = qhead + lane;
            if (pf_pos < ncand) pf_desc = sdesc[pf_pos];
          }
#endif
          __syncwarp();
        }
        const unsigned busy = __ballot_sync(FULL, cj >= 0);
        if (!busy) {
          bool more;
          if (serial) more = __shfl_sync(FULL, scan, 0) < G;
          else if (COOP) more = __any_sync(FULL, c_static < ncand);
          else if (GW > 1) more = wi + GW * qhead < ncand;
          else more = qhead < ncand;
          if (!more) break;
          continue;
        }
        if (cj < 0) continue;
        if (c_need) {
          if (c_wait) {
#if IGP_TILE_LDGSTS == 2
            cp_async_wait_all();
#else
            mbar_wait(lbar, c_phase);
            c_phase ^= 1u;
#endif
            c_wait = false;
#if IGP_PF_BATCH
            if constexpr (GW == 1 && !COOP && !serial) {
              if (pf_pos < ncand) {
                const int n2 = (int)((pf_desc >> 16) & 0xffffu);
                const uint32_t b2 = (uint32_t)(1 + (n2 < SLOT ? n2 : SLOT)) * (R_NF * 8);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                 rec + (size_t)((int)(pf_desc >> 32) - 1) * R_NF),
                             "r"(b2)
                             : "memory");
                pf_pos = INT_MAX;
              }
            }
#endif
          }
          if (c_pend >= 0) {
            finish(R_ERROR);
            continue;
          }
          // _eval_entries device terms (model.py:299-305), folded in resident
          // order: from the GPU's cached fold when nothing changed, else from
          // the start over the staged tile (recomputing an unchanged prefix
          // gives the cached prefix state bit for bit), else from the cached
          // prefix state of the first changed resident beyond the slot
          Neumaier fp, fc;
          int q0;
          if (c_dirty == c_nres) {
            fp.s = sl->gf[0];
            fp.c = sl->gf[1];
            fc.s = sl->gf[2];
            fc.c = sl->gf[3];
            q0 = c_nres;
          } else if (c_dirty < SLOT) {
            fp.s = fp.c = fc.s = fc.c = 0.0;
            q0 = 0;
          } else {
            const double *stp = pfx + (size_t)(c_off + c_dirty) * 4;
            fp.s = stp[0];
            fp.c = stp[1];
            fc.s = stp[2];
            fc.c = stp[3];
            q0 = c_dirty;
          }
          for (int qq = q0; qq < c_nres; ++qq) {
            double pw, ca;
            if (qq < SLOT) {
              pw = sl->rec[qq][R_PW];
              ca = sl->rec[qq][R_CA];
            } else if (mod.test(qq)) {
              pw = L.pw[qq];
              ca = L.ca[qq];
            } else {
              const double2 f2 = *reinterpret_cast<const double2 *>(frec + (size_t)(c_off + qq) * 2);
              pw = f2.x;
              ca = f2.y;
            }
            fp.add(pw);
            fc.add(ca);
          }
          fp.add(c_npw);
          fc.add(c_nca);
          const double f = frequency(hw, hw.pidle + fp.result());
          c_C = fc.result();
          // t_gpu = x / scale with scale = f / F (model.py:305-310).  The
          // decision t_inf > t_half uses x * (F / f), within 3 ulps of the
          // quotient, and falls back to the literal x / (f / F) inside the
          // margin; one division per evaluation instead of two.
          c_f = f;
          c_one = f == hw.fmax && hw.margin_ok;
          c_inv = c_one ? 1.0 : hw.fmax / f;
          if (exact) st_evals += c_nres + 1;
          st_calls += 1;
          c_need = false;
        }
        // The checks this evaluation serves (model.py:308-313, planner.py:158):
        // residents c_i, c_i+1, ... see the same device terms until one of
        // them is bumped, so one iteration runs them all and stops at the
        // first violation.
        int viol = -1;
        for (int i = c_i; i <= c_nres; ++i) {
          double ka, ca, t_sch, acache, t_load, t_fb, t_half;
          if (i == c_nres) {
            ka = c_nka;
            ca = c_nca;
            t_sch = c_tsn;
            acache = nw_acache;
            t_load = nw_tload;
            t_fb = nw_tfb;
            t_half = nw_thalf;
          } else if (i < SLOT) {
            const double *r = sl->rec[i];
            ka = r[R_KA];
            ca = r[R_CA];
            t_sch = r[R_TSN];
            acache = r[R_ACACHE];
            t_load = r[R_TLOAD];
            t_fb = r[R_TFB];
            t_half = r[R_THALF];
          } else {
            const double *r = rec + (size_t)(c_off + i) * R_NF;
            const double2 kc = *reinterpret_cast<const double2 *>(r + R_KA);
            const double2 ta = *reinterpret_cast<const double2 *>(r + R_TSN);
            const double2 lf = *reinterpret_cast<const double2 *>(r + R_TLOAD);
            t_half = r[R_THALF];
            t_sch = ta.x;
            acache = ta.y;
            t_load = lf.x;
            t_fb = lf.y;
            if (mod.test(i)) {
              ka = L.ka[i];
              ca = L.ca[i];
            } else {
              ka = kc.x;
              ca = kc.y;
            }
          }
          const double x = t_sch + ka * (1.0 + acache * (c_C - ca));
          double t_gpu = x;  // x / 1.0 == x exactly
          if (!c_one) {
            t_gpu = x * c_inv;
            if (margin) {
              const double tq = (t_load + t_gpu) + t_fb;
              if (!(fabs(tq - t_half) > tq * 0x1p-48 + 0x1p-1000)) t_gpu = x / (c_f / hw.fmax);
            } else {
              t_gpu = x / (c_f / hw.fmax);
            }
          }
          const double t_inf = (t_load + t_gpu) + t_fb;
          if (t_inf > t_half) {
            viol = i;
            break;
          }
        }
        if (viol < 0) {
          c_i = c_nres + 1;  // the rest of the pass is clean
        } else {
          const int i = viol;
          c_sum += 1;
          if (!exact) {
            // units only grow: an overflow or a key that already loses ends
            // the candidate before any further work
            if (c_sum > cap) {
              finish(R_INFEAS);
              continue;
            }
            const volatile unsigned *bp = &gs.best;
            const unsigned key = ((unsigned)(c_sum - c_occ) << 23) | (unsigned)cj;
            if (key > *bp) {
              finish(R_PRUNED);
              continue;
            }
          }
          Solo so;
          if (i == c_nres) {
            c_nu += 1;
            const int v = c_nu - need;
            if (v < TB && c_nu <= cap) {
              if (!n_ready) {
                mbar_wait(&nbar[grp], n_phase);
                n_ready = true;
              }
              const double *tv = ntab + v * 4;
              so.ka = tv[0];
              so.pw = tv[1];
              so.ca = tv[2];
              so.err = (int)tv[3];
            } else {
              so = solo_from_cold(ck, (double)c_nu * hw.runit);
            }
            c_nka = so.ka;
            c_npw = so.pw;
            c_nca = so.ca;
          } else if (i < SLOT) {
            const Meta mt = sl->meta[i];
            const int u = (int)mt.u + 1;
            if (!((c_sb >> i) & 1u)) {  // one unit above the committed units
#if IGP_SPLIT_NEXT
              const double *r = NEXT_AT(c_off + i);
              so.ka = r[0];
              so.pw = r[1];
              so.ca = r[2];
              so.err = (int)r[3];
#else
              const double *r = sl->rec[i];
              so.ka = r[R_KA1];
              so.pw = r[R_PW1];
              so.ca = r[R_CA1];
              so.err = (int)r[R_ERR1];
#endif
              c_sb |= 1u << i;
            } else {
              so = solo_lookup(tbl, cold, hw, mt.k, mt.lb, u);
            }
            sl->meta[i].u = (uint16_t)u;
            sl->rec[i][R_KA] = so.ka;
            sl->rec[i][R_CA] = so.ca;
            sl->rec[i][R_PW] = so.pw;
          } else {
            const Meta mt = meta[c_off + i];
            const int u = (mod.test(i) ? L.u[i] : (int)mt.u) + 1;
            so = solo_lookup(tbl, cold, hw, mt.k, mt.lb, u);
            L.u[i] = u;
            L.ka[i] = so.ka;
            L.pw[i] = so.pw;
            L.ca[i] = so.ca;
            mod.set(i);
          }
          if (i < c_dirty) c_dirty = i;
          if (exact && so.err && c_pend < 0) {
            c_pend = i;
            c_pcode = so.err;
          }
          c_flag = true;
          c_need = true;
          c_i = i + 1;
        }
        if (c_i > c_nres) {
          if (c_flag && c_sum <= cap) {
            c_i = 0;
            c_flag = false;
            // The reference re-evaluates at every pass start (rows = None,
            // planner.py:151); if nothing changed since the last evaluation the
            // values are identical, so only exact PlanStats account for it.
            if (exact && !c_need) {
              st_evals += c_nres + 1;
              st_calls += 1;
            }
          } else {
            finish(c_sum <= cap ? R_FEAS : R_INFEAS);
          }
        }
      }
    };

    if constexpr (!LEAN) {
      if (exact) run_step(BoolC<false>{}, BoolC<true>{}, IntC<2>{});
      else if (margin_rt) run_step(BoolC<false>{}, BoolC<false>{}, IntC<1>{});
      else run_step(BoolC<false>{}, BoolC<false>{}, IntC<0>{});
    } else {
      if (margin_rt) run_step(BoolC<false>{}, BoolC<false>{}, IntC<1>{});
      else run_step(BoolC<false>{}, BoolC<false>{}, IntC<0>{});
    }
#if IGP_TIMING
    long long tm2 = clock64();
#endif
    group_sync<GW>();
    if (t == 0 && !n_ready) mbar_wait(&nbar[grp], n_phase);  // retire this step's row copy
    n_ready = true;
    n_phase ^= 1u;

    if (!LEAN && gs.err_flag) {
      // exact mode only: replay the step in the reference's candidate order to
      // find the first raising candidate and the PlanStats at that point
      st_evals = st_calls = st_cands = st_rres = st_run = 0;
      if constexpr (!LEAN)
        if (wi == 0) run_step(BoolC<true>{}, BoolC<true>{}, IntC<2>{});
      if (t != 0) st_evals = st_calls = st_cands = st_rres = st_run = 0;
      tot_evals += st_evals;
      tot_calls += st_calls;
      tot_cands += st_cands;
      tot_rres += st_rres;
      tot_run += st_run;
      if (P.stream) {  // the arrival is rejected; the state is unchanged
        if (t == 0) {
          P.code[sm + k] = eo_fail.code | (aflags << 8);
          P.gpu_of[sm + k] = -1;
          P.pos[sm + k] = -1;
          P.units[sm + k] = 0;
        }
        st_evals = st_calls = st_cands = st_rres = st_run = 0;
        group_sync<GW>();
        continue;
      }
      fail_code = 1;
      break;
    }
    tot_evals += st_evals;
    tot_calls += st_calls;
    tot_cands += st_cands;
    tot_rres += st_rres;
    tot_run += st_run;
    st_evals = st_calls = st_cands = st_rres = st_run = 0;
    unsigned bk;
    bool committer;
    if constexpr (COOP) {
      // arrive per CTA; warp 0 of the last CTA to finish the step commits
      // it, the other CTAs wait until it is published
      __threadfence();  // this warp's keys, units and win_tid before its arrival
      __syncthreads();
      if (threadIdx.x == 0) gsm[0].next = atomicAdd(&cs->done[q & 1], 1) == (int)gridDim.x - 1;
      __syncthreads();
      const bool last_cta = gsm[0].next != 0;
      committer = last_cta && wi == 0 && grp == 0;
      if (!last_cta) {
        if (threadIdx.x == 0)
          while (ld_cg(&cs->flag) <= q) __nanosleep(32);
        __syncthreads();
      }
      __threadfence();  // acquire: later loads must not hit this SM's stale L1 lines
      bk = ld_cg(&cs->best[q & 1]);
    } else {
      bk = gs.best;
      if (bk != NO_KEY && my_best == bk) gs.win_thread = t;
      group_sync<GW>();
      committer = wi == 0;
    }

#if IGP_TIMING
    long long tm3 = clock64();
#endif
    // ---- commit (planner.py:312-319), one warp of the group ----
    if (committer) {
      const uint16_t *lu_w = nullptr;
      if (bk != NO_KEY) {
        const int wt = COOP ? P.win_tid[(int)(bk & 0x7fffffu)] : gs.win_thread;
        lu_w = lane_units + (size_t)wt * cap;
      }
      const ScenState Z{cold, tbl, gstate, sdesc, sj, spos, sE, gcap, gfold, rec,
#if IGP_SPLIT_NEXT
                        nxt,
#else
                        nullptr,
#endif
                        frec, pfx, meta, sm};
#if IGP_NW_SMEM
      commit_step(P, hw, Z, k, need, bk, lu_w, G, poolp, abortp, nws, ksch, nkern, lane);
#else
      const double nwv[R_NF] = {nw_ka, nw_ca, 0.0, nw_acache, nw_tload, nw_tfb, nw_thalf, nw_pw};
      commit_step(P, hw, Z, k, need, bk, lu_w, G, poolp, abortp, nwv, ksch, nkern, lane);
#endif
    }
#if IGP_TIMING
    if (s == 0 && threadIdx.x == 0 && P.stats) {  // phase cycles of scenario 0, warp 0
      long long tm4 = clock64();
      atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S], (unsigned long long)(tm1 - tm0));
      atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 1], (unsigned long long)(tm2 - tm1));
      atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 2], (unsigned long long)(tm3 - tm2));
      atomicAdd((unsigned long long *)&P.stats[IGP_NSTAT * P.S + 3], (unsigned long long)(tm4 - tm3));
    }
#endif
    if (bk == NO_KEY) G += 1;
    sflags |= aflags;  // an admitted risky arrival can raise in later steps
    if (committer) fence_async_global();  // commit writes -> next step's tile copies
    if constexpr (COOP) {
      if (committer) {  // recycle step k-1's slots for step k+1, then publish step k
        if (lane == 0) {
          cs->done[(q + 1) & 1] = 0;
          cs->best[(q + 1) & 1] = NO_KEY;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(&cs->flag, q + 1);
      }
      ++q;
      if (ld_cg(abortp)) {
        fail_code = 2;
        break;
      }
      __syncthreads();  // the CTA's committer may still use gsm[0].next
      continue;
    }
    __threadfence_block();
    group_sync<GW>();
    if (gs.abort_code) {
      fail_code = 2;
      break;
    }
  }
  if constexpr (COOP) {  // hand the state to the kernel that writes the plan
    unsigned long long ev = (unsigned long long)tot_calls, cd = (unsigned long long)tot_run;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ev += __shfl_xor_sync(FULL, ev, o);
      cd += __shfl_xor_sync(FULL, cd, o);
    }
    if (lane == 0) {
      atomicAdd(&cs->evals_run, ev);
      atomicAdd(&cs->cands_run, cd);
    }
    if (gtid == 0) {
      cs->G = G;
      cs->sflags = sflags;
      cs->status = fail_code ? P.k1 : k_stop;  // an abort is reported by the per-CTA kernel
    }
    return;
  }

  // group totals of the counters
  if (t == 0) gs.tot[0] = gs.tot[1] = gs.tot[2] = gs.tot[3] = gs.tot[4] = 0;
  group_sync<GW>();
  atomicAdd(&gs.tot[0], (unsigned long long)tot_evals);
  atomicAdd(&gs.tot[1], (unsigned long long)tot_calls);
  atomicAdd(&gs.tot[2], (unsigned long long)tot_cands);
  atomicAdd(&gs.tot[3], (unsigned long long)tot_rres);
  atomicAdd(&gs.tot[4], (unsigned long long)tot_run);
  group_sync<GW>();
  if (t == 0 && P.stats) {
    const bool st_ok = (P.flags & IGP_F_STATS) || fail_code == 1;
    P.stats[IGP_NSTAT * s] = st_ok ? (long long)gs.tot[0] : -1;
    P.stats[IGP_NSTAT * s + 1] = st_ok ? (long long)gs.tot[2] : -1;
    P.stats[IGP_NSTAT * s + 2] = st_ok ? (long long)gs.tot[1] : -1;
    P.stats[IGP_NSTAT * s + 3] = (long long)gs.tot[1];
    // resident reads (exact mode); with the fast kernel: the candidates it
    // re-ran with the exact evaluation (decisions inside its margin)
    P.stats[IGP_NSTAT * s + 4] = st_ok ? (long long)gs.tot[3]
                                       : fast_done ? (long long)hdp->exact_run : -1;
    P.stats[IGP_NSTAT * s + 5] = (long long)gs.tot[4];
  }

  if (P.stream && t == 0) {  // persist the scenario state for the next push
    sst[0] = G;
    sst[1] = gs.pool_top;
    sst[2] = sflags;
    sst[3] = P.k1;
  }
  if (P.stream && !P.pred && !fail_code) {
    if (t == 0) {
      err->code = 0;
      err->workload = -1;
      err->gpu = -1;
      err->a = err->b = err->c = 0.0;
      P.gpu_count[s] = G;
    }
    group_sync<GW>();
    continue;
  }

  if (fail_code) {
    if (t == 0) {
      if (fail_code == 1) {
        err->code = eo_fail.code;
        err->workload = (int)cold[(size_t)eo_fail.k * C_NF + C_WIN];
        err->a = eo_fail.a;
        err->b = eo_fail.b;
        err->c = eo_fail.c;
      } else {
        err->code = gs.abort_code;
        err->workload = -1;
        err->a = (double)P.pool_recs;
        err->b = err->c = 0.0;
      }
      err->gpu = -1;
      P.gpu_count[s] = G;
    }
    continue;
  }

  // ---- _build_plan (planner.py:218-246): predict_gpu per device (model.py:320-343) ----
  if (t == 0) gs.err_gpu = INT_MAX;
  group_sync<GW>();
  int my_err_gpu = INT_MAX;
  ErrOut my_eo;
  my_eo.code = 0;
  my_eo.k = -1;
  const bool want_pred = P.pred && !(P.flags & IGP_F_NO_PRED);
  for (int j = t; j < G; j += GT) {
    const int n = (int)((gstate[j] >> 16) & 0xffffu);
    const int off = (int)(gstate[j] >> 32);
    // capacity check: sum(a.r) with a.r = u * r_unit (model.py:331-335)
    Neumaier cs;
    cs.first((double)meta[off].u * hw.runit);
    for (int qq = 1; qq < n; ++qq) cs.add((double)meta[off + qq].u * hw.runit);
    const double total_r = cs.result();
    int ecode = 0;
    if (total_r > hw.rmax + 1e-9) {
      ecode = IGP_E_OVERALLOC;
      if (j < my_err_gpu) {
        my_err_gpu = j;
        my_eo.code = ecode;
        my_eo.k = -1;
        my_eo.a = total_r;
        my_eo.b = hw.rmax;
        my_eo.c = 0.0;
      }
    }
    Neumaier fp, fc;
    for (int qq = 0; qq < n; ++qq) {
      const Meta mt = meta[off + qq];
      const Solo so = solo_from_cold(cold + (size_t)mt.k * C_NF, (double)mt.u * hw.runit);
      if (!ecode && so.err) {
        ecode = so.err;
        if (j < my_err_gpu) {
          my_err_gpu = j;
          err_operands(hw, cold + (size_t)mt.k * C_NF, mt.u, so.err, my_eo);
          my_eo.k = mt.k;
        }
      }
      L.ka[qq] = so.ka;
      L.ca[qq] = so.ca;
      L.pw[qq] = so.pw;
      if (qq == 0) {
        fp.first(so.pw);
        fc.first(so.ca);
      } else {
        fp.add(so.pw);
        fc.add(so.ca);
      }
    }
    const double f = frequency(hw, hw.pidle + fp.result());
    const double C = fc.result();
    const double scale = f / hw.fmax;
    const double dl = delta_sch(hw, n);
    for (int qq = 0; qq < n; ++qq) {
      const Meta mt = meta[off + qq];
      const double *ce = cold + (size_t)mt.k * C_NF;
      const double *rr = rec + (size_t)(off + qq) * R_NF;
      const int w_in = (int)ce[C_WIN];
      P.gpu_of[sm + w_in] = j;
      P.pos[sm + w_in] = qq;
      P.units[sm + w_in] = mt.u;
      if (want_pred) {
        const double t_sch = (ce[C_KSCH] + dl) * ce[C_NK];
        const double t_act = L.ka[qq] * (1.0 + rr[R_ACACHE] * (C - L.ca[qq]));
        const double t_gpu = (t_sch + t_act) / scale;
        const double t_inf = (rr[R_TLOAD] + t_gpu) + rr[R_TFB];
        double *row = P.pred + (sm + w_in) * 10;
        row[0] = rr[R_TLOAD];
        row[1] = t_sch;
        row[2] = t_act;
        row[3] = f;
        row[4] = t_gpu;
        row[5] = rr[R_TFB];
        row[6] = t_inf;
        row[7] = (ce[C_BATCH] / (t_gpu + rr[R_TFB])) * 1000.0;
        row[8] = L.pw[qq];
        row[9] = L.ca[qq];
      }
    }
  }
  if (my_err_gpu != INT_MAX) atomicMin(&gs.err_gpu, my_err_gpu);
  group_sync<GW>();
  const int eg = gs.err_gpu;
  if (eg != INT_MAX && my_err_gpu == eg) {
    err->code = my_eo.code;
    err->workload = my_eo.k >= 0 ? (int)cold[(size_t)my_eo.k * C_NF + C_WIN] : -1;
    err->gpu = eg;
    err->a = my_eo.a;
    err->b = my_eo.b;
    err->c = my_eo.c;
  }
  if (t == 0) {
    if (eg == INT_MAX) {
      err->code = 0;
      err->workload = -1;
      err->gpu = -1;
      err->a = err->b = err->c = 0.0;
    }
    P.gpu_count[s] = G;
  }
  group_sync<GW>();
  }  // persistent scenario loop
}

}  // namespace igp
