/*
 * igniter_b200.h -- C-ABI of the B200-native iGniter provisioning hot path.
 *
 * The reference (gpuplanner, pure Python) has no FFI: its drop-in surface is
 * the Python API re-exported by pkg/src/gpuplanner/__init__.py:3-92.  Each
 * entry point below replaces the computation behind one of those calls; the
 * Python host layer (paper_2211_01713_b200/) keeps the reference signatures
 * and binds these symbols with ctypes (INTEGRATION.md shows the binding).
 *
 *   igp_plan_batch_device / igp_plan_batch_host
 *       replaces plan()            planner.py:258-325  (Alg. 1 + Alg. 2 +
 *                                  _build_plan planner.py:218-246), for one
 *                                  or many independent scenarios
 *   igp_eval_states_device
 *       replaces _eval_entries     model.py:273-317 and predict_gpu
 *                                  model.py:320-343 (batched device states)
 *   igp_alloc_units_device
 *       replaces _alloc_units      planner.py:133-162 behind alloc_gpus
 *                                  planner.py:165-192
 *   igp_stream_*_device
 *       the planner.py:290-319 step applied in arrival order to persistent
 *                                  device state (online re-provisioning; no
 *                                  reference API, see below)
 *   igp_group_search_device
 *       replaces _Search.best_group_alloc oracle.py:77-114 for every subset
 *                                  of a small group (exhaustive_plan's search)
 *   igp_simulate_device
 *       replaces simulate() simulate.py:139-198 (constant-rate arrivals)
 *   igp_solo_grid_device
 *       replaces _Search.best_group_alloc oracle.py:77-114 for one-workload
 *                                  groups over every batch (the solo grid)
 *   igp_components_device, igp_power_demand_device
 *       replace the model's scalar component functions model.py:159-236
 *                                  (transfer_latencies .. gpu_frequency,
 *                                  power_demand), batched
 *   igp_prologue_device
 *       replaces appropriate_batch planner.py:76-92 and _lower_bound_units
 *                                  planner.py:95-120 (lower_bound_resources
 *                                  planner.py:123-130)
 *
 * Conventions
 *   - plain pointers and sizes only; "device" entry points take device
 *     pointers and a cudaStream_t passed as void*; "host" entry points take
 *     host pointers and synchronise before returning.
 *   - workload tables are fp64 structure-of-arrays, field-major:
 *     wl[f * ld + i], fields in IGP_WL_* order (16 fields).  A scenario batch
 *     is S consecutive tables with ld = m (wl[(s * 16 + f) * m + i]).
 *   - hardware profile: 11 doubles in IGP_HW_* order, host memory.
 *   - result rows: 10 doubles in LatencyBreakdown order (model.py:133-146).
 *   - every fp64 operation follows the reference's association and is
 *     rounded separately (built with -fmad=false); builtin-sum sites use the
 *     CPython 3.12 Neumaier fold in resident order.  Results are bit-exact.
 *   - errors: the return value is IGP_E_OK or the first error code; the
 *     igp_error record carries the operands the Python layer needs to raise
 *     the reference's exception with the reference's message.
 *   - the library keeps no pointer after a call returns; scratch lives in a
 *     caller-owned device workspace sized by igp_plan_workspace_bytes().
 */
#ifndef IGNITER_B200_H
#define IGNITER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IGP_ABI_VERSION 1

/* workload fields (WorkloadSpec model.py:19-27, WorkloadCoefficients model.py:40-62) */
enum {
  IGP_WL_SLO = 0, IGP_WL_RATE, IGP_WL_DLOAD, IGP_WL_DFB, IGP_WL_NK, IGP_WL_KSCH,
  IGP_WL_K1, IGP_WL_K2, IGP_WL_K3, IGP_WL_K4, IGP_WL_K5, IGP_WL_ALPHA_P,
  IGP_WL_BETA_P, IGP_WL_ALPHA_CU, IGP_WL_BETA_CU, IGP_WL_ALPHA_CACHE, IGP_WL_NF
};
/* hardware fields (HardwareProfile model.py:73-110) */
enum {
  IGP_HW_PMAX = 0, IGP_HW_FMAX, IGP_HW_PIDLE, IGP_HW_BW, IGP_HW_ALPHA_F,
  IGP_HW_ALPHA_SCH, IGP_HW_BETA_SCH, IGP_HW_RUNIT, IGP_HW_RMAX, IGP_HW_PRICE,
  IGP_HW_FMIN_FRAC, IGP_HW_NF
};

/* error codes -> reference exceptions (errors.py) */
enum {
  IGP_E_OK = 0,
  IGP_E_BATCH_CAP = 1,      /* BatchCapExceededError  planner.py:86-91;  a = b            */
  IGP_E_INFEASIBLE_SLO = 2, /* InfeasibleSloError     planner.py:107-111; a = delta       */
  IGP_E_INFEASIBLE_RES = 3, /* InfeasibleResourceError planner.py:115-119; a = units      */
  IGP_E_DENOM = 4,          /* NonPositiveDenominatorError model.py:286-290; a=denom b=r c=k4 */
  IGP_E_ACTIVE_TIME = 5,    /* NonPositiveDenominatorError model.py:178-183; a=k_act b=batch c=r */
  IGP_E_OVERALLOC = 6,      /* OverAllocatedError     model.py:331-335;  a = total_r b = r_max */
  IGP_E_CAPACITY = 7,       /* a library limit was exceeded (see igp_limits)              */
  IGP_E_CUDA = 8,           /* CUDA runtime error; a = cudaError_t                        */
  IGP_E_ARG = 9             /* invalid argument                                           */
};

typedef struct igp_error {
  int32_t code;
  int32_t workload; /* input-order index of the workload the error names, or -1 */
  int32_t gpu;      /* device index for _build_plan-time errors, or -1 */
  int32_t pad;
  double a, b, c;   /* message operands, see the enum above */
} igp_error;

#define IGP_NSTAT 6 /* int64 counters per scenario in the stats outputs */

/* plan flags */
enum {
  IGP_F_STATS = 1,      /* exact PlanStats (model_evals, candidate_gpus) for every
                           scenario: no overflow early exit, no bound prune */
  IGP_F_NO_PRED = 2,    /* skip the _build_plan breakdown rows */
  IGP_F_SMEM = 8,       /* with IGP_F_CTA: one CTA per scenario keeps the search
                           state in shared memory and evaluates each candidate
                           with one warp (csrc/smem_plan.cuh; up to about 1,250
                           workloads, larger scenarios use the per-CTA kernel);
                           falls back on the device like IGP_F_COOP */
  IGP_F_CTA = 4,        /* one CTA (many warps) per scenario instead of one warp:
                           lower latency for single large plans */
  IGP_F_GW2 = 32,       /* two / four warps per scenario (between the default one */
  IGP_F_GW4 = 64,       /* warp and IGP_F_CTA's eight) */
  IGP_F_COOP = 16,      /* single scenario (n_scen == 1): every warp of the GPU
                           shares each step (grid-cooperative launch); falls back
                           on the device to IGP_F_CTA when the exact sequence is
                           needed (IGP_F_STATS, or a scenario that can raise) */
  IGP_F_WIN = 1 << 28,  /* single scenario (n_scen == 1, max_units <= 128): the
                           windowed speculative kernel plans steps in windows of 8
                           (phase A: every newcomer of the window against the
                           window-start GPUs; phase B: in step order, re-running
                           only the GPUs earlier steps touched); falls back like
                           IGP_F_COOP.  Combine with IGP_F_CTA. */
  IGP_F_FAST = 1 << 29, /* batches of one-warp scenarios: run the certified-margin
                           kernel first (csrc/fast.cuh: every Alg. 2 decision from
                           O(1) compact-tile evaluations with an error bound, the
                           exact evaluation inside the margin; bit-identical plans).
                           Opt-in: measured slower than the exact kernel on the
                           latency-bound batch */
  IGP_F_HWS = 128       /* one hardware profile per scenario: hw points to
                           n_scen x IGP_HW_NF doubles (host) instead of one
                           profile.  select_gpu_type (planner.py:333-364) plans
                           every GPU type of a request as one scenario of ONE
                           launch.  Not combined with IGP_F_COOP or the stream
                           entry points. */
};

int igp_abi_version(void);
/* largest supported max_units(hw) = round(r_max / r_unit) */
int igp_max_cap(void);
/* last CUDA error string of this thread (for IGP_E_CUDA) */
const char *igp_last_error_string(void);

/* Scenarios of m workloads the place kernel runs at once on the current
 * device (resident warps for one-warp scenarios, resident CTAs with
 * IGP_F_CTA): a batch of this many fills the GPU in one wave.  Negative
 * IGP_E_* on a bad profile. */
int igp_plan_batch_slots(int m, const double *hw, int b_max, int flags);

/* Device workspace needed by igp_plan_batch_*() for S scenarios of m workloads
 * (hw: one profile, or n_scen profiles with IGP_F_HWS). */
size_t igp_plan_workspace_bytes(int n_scen, int m, const double *hw, int b_max, int flags);

/*
 * Plan S independent scenarios of m workloads each (Alg. 1, planner.py:258-325).
 *   wl          [S][16][m] fp64
 *   name_rank   [m] (rank_stride = 0, shared by all scenarios) or [S][m]
 *               (rank_stride = m): rank of each name in Python string order,
 *               the tie-break of planner.py:284
 * outputs, all indexed by input order:
 *   gpu_of, pos, units, batch, lb   [S][m] int32  (GPU index, position in that
 *                                   GPU's allocation list, final units, batch,
 *                                   lower-bound units)
 *   pred        [S][m][10] fp64 breakdown rows (NULL or IGP_F_NO_PRED: skipped)
 *   gpu_count   [S]
 *   stats       [S][IGP_NSTAT] int64 {model_evals, candidate_gpus, eval_calls,
 *               evals_run, resident_reads, candidates_run}: the reference's
 *               PlanStats counters (planner.py:64-69), its number of
 *               _eval_entries calls and the residents its candidate trials read
 *               (sum over trials of the GPU's resident count) -- exact with
 *               IGP_F_STATS (or for a scenario that raised), -1 otherwise --
 *               and the device evaluations / candidates this kernel actually ran
 *   err         [S] igp_error
 * returns IGP_E_OK or the first error code over scenarios (per-scenario codes
 * are in err[s].code).
 */
int igp_plan_batch_device(const double *wl, int n_scen, int m, const double *hw, int b_max,
                          const int32_t *name_rank, int rank_stride, int32_t *gpu_of,
                          int32_t *pos, int32_t *units, int32_t *batch, int32_t *lb,
                          double *pred, int32_t *gpu_count, int64_t *stats, igp_error *err,
                          void *workspace, size_t workspace_bytes, int flags, void *stream);

/* The two stages of igp_plan_batch_device, same arguments and workspace:
 * prepare = prologue (batch, lower bound, first input-order error), the
 * (-lb, name) sort and the per-workload entry constants; place = the Alg. 1
 * step loop with Alg. 2 per candidate plus the _build_plan predictions.
 * Exposed so callers can time / overlap the stages separately. */
int igp_plan_prepare_device(const double *wl, int n_scen, int m, const double *hw, int b_max,
                            const int32_t *name_rank, int rank_stride, int32_t *gpu_of,
                            int32_t *pos, int32_t *units, int32_t *batch, int32_t *lb,
                            double *pred, int32_t *gpu_count, int64_t *stats, igp_error *err,
                            void *workspace, size_t workspace_bytes, int flags, void *stream);
int igp_plan_place_device(const double *wl, int n_scen, int m, const double *hw, int b_max,
                          const int32_t *name_rank, int rank_stride, int32_t *gpu_of,
                          int32_t *pos, int32_t *units, int32_t *batch, int32_t *lb,
                          double *pred, int32_t *gpu_count, int64_t *stats, igp_error *err,
                          void *workspace, size_t workspace_bytes, int flags, void *stream);

/* Same contract with HOST buffers: H2D copies, kernels, D2H copies and a
 * stream synchronisation all happen inside the call.  Pinned host memory is
 * recommended.  workspace is device memory of igp_plan_host_workspace_bytes()
 * (the planning scratch plus the device copies of the inputs and outputs),
 * or workspace = NULL with workspace_bytes = 0: the library then allocates
 * and frees it itself, stream-ordered (cudaMallocAsync / cudaFreeAsync).
 * Batches of >= 256 scenarios are pipelined in two scenario chunks on
 * library-owned streams ordered after `stream`: one chunk's kernels overlap
 * the next chunk's H2D and the previous chunk's D2H copies. */
size_t igp_plan_host_workspace_bytes(int n_scen, int m, const double *hw, int b_max, int flags,
                                     int rank_stride, int want_pred);
int igp_plan_batch_host(const double *wl, int n_scen, int m, const double *hw, int b_max,
                        const int32_t *name_rank, int rank_stride, int32_t *gpu_of,
                        int32_t *pos, int32_t *units, int32_t *batch, int32_t *lb,
                        double *pred, int32_t *gpu_count, int64_t *stats, igp_error *err,
                        void *workspace, size_t workspace_bytes, int flags, void *stream);

/*
 * Batched device-state evaluation (_eval_entries model.py:273-317).
 *   wl [16][n_rows] (ld = n_rows), batch [n_rows], r [n_rows], ptr [n_states+1]
 *   rows [n_rows][10]; err [n_states] (first error of each state, in entry order)
 *   check_capacity != 0 adds predict_gpu's Neumaier capacity check
 *   (model.py:331-335) before the evaluation.
 * returns the first error over states (state order).
 */
int igp_eval_states_device(const double *wl, int n_rows, const int32_t *batch,
                           const double *r, const int64_t *ptr, int n_states,
                           const double *hw, int check_capacity, double *rows,
                           igp_error *err, void *stream);

/*
 * Batched Alg. 2 (_alloc_units planner.py:133-162) for alloc_gpus
 * (planner.py:165-192): units start at int(round(r / r_unit)); the result may
 * sum beyond max_units (the reference's infeasibility marker).
 */
int igp_alloc_units_device(const double *wl, int n_rows, const int32_t *batch,
                           const double *r, const int64_t *ptr, int n_states,
                           const double *hw, int32_t *units, igp_error *err, void *stream);

/*
 * appropriate_batch (planner.py:76-92) and _lower_bound_units (:95-120) for m
 * workloads.  batch_in may be NULL (compute the batch) or supply the batch
 * (lower_bound_resources semantics, planner.py:123-130).  code[i] is 0 or the
 * error code of workload i (batch error before lb error).
 */
int igp_prologue_device(const double *wl, int m, const double *hw, int b_max,
                        const int32_t *batch_in, int32_t *batch, int32_t *lb, int32_t *code,
                        igp_error *err, void *stream);

/*
 * Online re-provisioning stream (BASELINE config 5).  The reference has no
 * API for it (plan() always sorts, planner.py:284); each arrival is one step
 * of planner.py:290-319 in ARRIVAL order against persistent device state,
 * with its batch and lower bound from planner.py:76-120.  An arrival whose
 * prologue or candidate evaluation raises is rejected (code = IGP_E_*) and
 * leaves the state unchanged.  n_streams independent streams advance
 * together; each push appends n arrivals to every stream.  All state lives in
 * the caller's device workspace (igp_stream_workspace_bytes); the caller
 * tracks k0 = arrivals pushed so far.
 *   flags:     a single stream (n_streams == 1) may run a push with
 *              IGP_F_COOP: every warp of the GPU shares each arrival's step
 *              (bits 16..27 of flags: the CTA count, 0 = whole GPU); the
 *              per-CTA kernel resumes at the first arrival that needs the
 *              exact sequence.  Pushes with and without it mix freely.
 *   push:      wl_new [S][16][n]; outputs [S][n]: GPU index and position
 *              within that GPU at admission (-1 when rejected), and the code
 *              (IGP_E_* in the low 8 bits); err [S] (device, nullable): a
 *              stream whose record pool overflowed reports IGP_E_CAPACITY
 *              and stops admitting until it is reset with a larger pool
 *   snapshot:  [S][n_arrivals] current GPU, position and units of every
 *              arrival (units 0 when rejected), breakdown rows (nullable),
 *              GPU count and the predict_gpu error record per stream
 */
size_t igp_stream_workspace_bytes(int n_streams, int capacity, const double *hw, int b_max,
                                  int flags);
int igp_stream_reset_device(int n_streams, int capacity, const double *hw, int b_max,
                            void *workspace, size_t workspace_bytes, int flags, void *stream);
int igp_stream_push_device(const double *wl_new, int n_streams, int k0, int n, int capacity,
                           const double *hw, int b_max, int32_t *gpu_of, int32_t *pos,
                           int32_t *code, int64_t *stats, igp_error *err, void *workspace,
                           size_t workspace_bytes, int flags, void *stream);
int igp_stream_snapshot_device(int n_streams, int n_arrivals, int capacity, const double *hw,
                               int b_max, int32_t *gpu_of, int32_t *pos, int32_t *units,
                               double *pred, int32_t *gpu_count, igp_error *err,
                               void *workspace, size_t workspace_bytes, int flags,
                               void *stream);

/*
 * Exhaustive oracle group search (_Search.best_group_alloc, oracle.py:77-114)
 * for every non-empty subset of n <= 6 workloads (in name order, the order
 * of oracle.py:86) at once: best[mask] is the lexicographic minimum of
 * (total units, unit tuple) over the feasible unit vectors drawn from grid
 * (ascending, device) with total <= max_units, packed as
 * total << 9k | u_1 << 9(k-1) | ... | u_k, or ~0 when none is feasible.
 * Feasibility is _Search._feasible (oracle.py:64-75).  err (device int32)
 * receives an IGP_E_DENOM / IGP_E_ACTIVE_TIME code if any enumerated vector
 * raised (the reference raises only for the vectors its pruned recursion
 * evaluates).  The reference's candidate budget (OracleBudget.max_candidates)
 * counts its own pruned evaluations and is not reproduced.
 */
int igp_group_search_device(const double *wl, int n, const int32_t *batch, const double *hw,
                            const int32_t *grid, int n_grid, unsigned long long *best,
                            int32_t *err, void *stream);

/*
 * The latency model's component functions (model.py:159-236), one query per
 * index i, with the reference's operation order (bit-identical results).
 *   wl       [IGP_WL_NF][n] fp64 query fields (field-major; only d_load,
 *            d_feedback and the WorkloadCoefficients fields are read)
 *   batch    [n] int32, r [n] resource fraction, co_cache [n] co-runners'
 *            summed cache utilisation, n_col [n] co-located workloads,
 *            p_dem [n] device power demand (W)
 *   out      [n][10] fp64: t_load, t_feedback (transfer_latencies), r + k4,
 *            solo_active_time, solo_power, solo_cache_util,
 *            sched_delay_increase, sched_delay, active_time_with_interference,
 *            gpu_frequency
 *   code     [n] int32: 0, IGP_E_DENOM (r + k4 <= 0: solo_active_time and
 *            everything built on it raise) or IGP_E_ACTIVE_TIME (k_act <= 0:
 *            solo_power / solo_cache_util raise, model.py:178-183)
 * All pointers are device pointers except hw (host, IGP_HW_* order).
 */
int igp_components_device(int n, const double *wl, const int32_t *batch, const double *r,
                          const double *co_cache, const int32_t *n_col, const double *p_dem,
                          const double *hw, double *out, int32_t *code, void *stream);

/*
 * power_demand (model.py:226-228): hw.power_idle_w + the CPython 3.12 sum
 * (Neumaier-compensated, in order) of n solo powers; *out (device) = the
 * idle draw when n == 0.
 */
int igp_power_demand_device(int n, const double *powers, const double *hw, double *out,
                            void *stream);

/*
 * Request-level replay of a plan (simulate._run_workload simulate.py:98-136
 * and the report of simulate.simulate simulate.py:139-198), constant-rate
 * arrivals (simulate.py:75-84), n workloads with their rate, batch and
 * predicted service time (t_inf).  seg [n+1] (device) holds segment offsets
 * with seg[i+1] - seg[i] >= the workload's arrival count (ceil(duration *
 * rate / 1000) + 2 is enough); lat, starts, sorted are device scratch of
 * seg[n] doubles.  Outputs per workload: measured-latency end offsets,
 * max queue depth, end backlog (UnstableQueueError above 10 x batch,
 * simulate.py:163-166), measured request count, p50 / p99 (NumPy 'linear'
 * percentile of the measured end-to-end latencies) and achieved req/s.
 * Synchronises the stream once (to size the segmented sort).
 */
int igp_simulate_device(int n, const double *rate, const int32_t *batch, const double *service,
                        double duration_ms, double warmup_ms, const int64_t *seg, double *lat,
                        double *starts, double *sorted, int64_t *seg_end, int32_t *max_depth,
                        int32_t *backlog, int32_t *completed, double *p50, double *p99,
                        double *achieved, void *stream);

/*
 * Solo candidate grid (BASELINE config 3): every (workload w, batch b in
 * 1..b_max, units u in 1..max_units) single-entry state of _eval_entries
 * (model.py:273-317) under the feasibility predicate of _Search._feasible
 * (oracle.py:64-75: t_inf <= t_half and throughput >= rate_rps), with the
 * entry built at batch b (_Entry model.py:253-270).  Replaces, per (w, b),
 * _Search.best_group_alloc([w]) (oracle.py:77-114): the scan over u ascends
 * and stops at the first feasible point.
 *   wl          [16][m] fp64
 *   min_units   [m][b_max] int32: smallest feasible u, 0 if none, or -code if
 *               an evaluation raised first (IGP_E_DENOM / IGP_E_ACTIVE_TIME)
 *   best_u/b    [m] int32 (nullable): cheapest feasible point, min u then min b
 *   n_evals     device uint64 (nullable): points evaluated
 */
int igp_solo_grid_device(const double *wl, int m, const double *hw, int b_max,
                         int32_t *min_units, int32_t *best_u, int32_t *best_b,
                         unsigned long long *n_evals, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* IGNITER_B200_H */
