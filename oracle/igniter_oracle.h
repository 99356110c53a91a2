/* igniter_oracle.h -- CPU oracle for the iGniter hot path (TEST INFRASTRUCTURE).
 * See igniter_oracle.c for the reference file:line each function restates. */
#ifndef IGNITER_ORACLE_H
#define IGNITER_ORACLE_H
#include <stdint.h>

/* error codes: identical values to include/igniter_b200.h IGP_E_* */
enum {
  IGO_E_OK = 0, IGO_E_BATCH_CAP = 1, IGO_E_INFEASIBLE_SLO = 2, IGO_E_INFEASIBLE_RES = 3,
  IGO_E_DENOM = 4, IGO_E_ACTIVE_TIME = 5, IGO_E_OVERALLOC = 6
};

typedef struct {
  int32_t code;
  int32_t workload; /* input-order index, -1 if none */
  double a, b, c;   /* message operands (see include/igniter_b200.h igp_error) */
} igo_err;

int igo_max_units(const double *hw);
int igo_prologue(const double *wl, int64_t ld, int m, const double *hw, int b_max,
                 int32_t *batch, int32_t *lb, int32_t *code);
int igo_eval_states(const double *wl, int64_t ld, const int32_t *batch, const double *r,
                    const int64_t *ptr, int n_states, const double *hw, double *rows,
                    igo_err *err);
int igo_alloc_units(const double *wl, int64_t ld, const int32_t *batch, const double *r,
                    const int64_t *ptr, int n_states, const double *hw, int32_t *units_out,
                    igo_err *err);
int igo_plan(const double *wl, int64_t ld, int m, const double *hw, int b_max,
             const int32_t *name_rank, int32_t *gpu_of, int32_t *pos, int32_t *units_out,
             int32_t *batch_out, int32_t *lb_out, double *pred, int32_t *gpu_count,
             int64_t *stats, igo_err *err);
int igo_plan_batch(const double *wl, int n_scen, int m, const double *hw, int b_max,
                   const int32_t *name_rank, int32_t *gpu_of, int32_t *pos, int32_t *units,
                   double *pred, int32_t *gpu_count, int64_t *stats, int n_threads);
int igo_solo_grid(const double *wl, int64_t ld, int m, const double *hw, int b_max,
                  int32_t *min_units, int64_t *n_evals);
int igo_stream(const double *wl, int64_t ld, int n, const double *hw, int b_max,
               int32_t *gpu_of, int32_t *pos, int32_t *code, int32_t *units_final,
               int32_t *gpu_count, int64_t *stats);
int igo_group_search(const double *wl, int64_t ld, int n, const int32_t *batch, const double *hw,
                     const int32_t *grid, int n_grid, uint64_t *best);
#endif
