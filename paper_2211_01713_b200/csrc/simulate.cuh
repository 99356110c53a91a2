// simulate.cuh -- deterministic request-level replay of a plan.
//
// Restates simulate._run_workload (simulate.py:98-136) and the report of
// simulate.simulate (simulate.py:139-198) for constant-rate arrivals
// (simulate.py:75-84), one thread per workload:
//   arrivals t_k = k * (1000 / rate) while t_k < duration; requests queue
//   until a full batch is waiting; the batch starts at max(last member's
//   arrival, server free) and runs for the plan's predicted t_inf.
// The measured end-to-end latencies (arrival >= warmup) of each workload are
// written to its segment of a scratch array, sorted per segment (CUB), and
// reduced to p50 / p99 with NumPy's default 'linear' percentile
// (numpy/lib/_function_base_impl.py: virtual index (n-1) q, _lerp).
#pragma once

namespace igp {

struct SimParams {
  int n;
  double duration, warmup;
  const double *rate;     // [n] req/s
  const int32_t *batch;   // [n]
  const double *service;  // [n] ms
  const long long *seg;   // [n + 1] segment offsets (upper bound on arrivals)
  double *lat;            // measured latencies, per segment
  double *starts;         // batch start times, per segment
  long long *seg_end;     // [n] end of the measured latencies in each segment
  int32_t *max_depth, *backlog, *completed;
};

__global__ void k_sim_replay(SimParams S) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= S.n) return;
  const double spacing = 1000.0 / S.rate[w];  // simulate.py:78
  const int b = S.batch[w];
  const double svc = S.service[w];
  const long long base = S.seg[w];
  double *lat = S.lat + base;
  double *starts = S.starts + base;
  long long nlat = 0, nbatch = 0, pend_lo = 0;  // pending = formed batches [pend_lo, nbatch)
  long long q_head = 0;                          // queue = arrivals [q_head, k]
  double server_free = 0.0;
  long long max_depth = 0;
  long long k = 0;
  for (double t = 0.0; t < S.duration; t = (double)(++k) * spacing) {  // simulate.py:79-84
    const long long qlen = k + 1 - q_head;
    if (qlen >= b) {  // one full batch (the queue holds < b before this arrival)
      const double last = (double)(q_head + b - 1) * spacing;
      const double start = py_max(last, server_free);  // simulate.py:120
      const double done = start + svc;
      for (long long r = q_head; r < q_head + b; ++r) {
        const double arrival = r == 0 ? 0.0 : (double)r * spacing;
        if (arrival >= S.warmup) lat[nlat++] = done - arrival;  // simulate.py:168-172
      }
      starts[nbatch++] = start;
      q_head += b;
      server_free = done;
    }
    while (pend_lo < nbatch && starts[pend_lo] <= t) ++pend_lo;  // simulate.py:126-127
    const long long waiting = (k + 1 - q_head) + (nbatch - pend_lo) * b;
    if (waiting > max_depth) max_depth = waiting;
  }
  long long slipped = 0;  // pending batches whose start lies past the horizon
  for (long long i = pend_lo; i < nbatch; ++i)
    if (starts[i] > S.duration) ++slipped;
  S.backlog[w] = (int32_t)((k - q_head) + slipped * b);  // simulate.py:131-133
  S.max_depth[w] = (int32_t)max_depth;
  S.completed[w] = (int32_t)nlat;
  S.seg_end[w] = base + nlat;
}

// NumPy percentile, method 'linear', on a sorted segment of n > 0 values
__device__ __forceinline__ double np_percentile(const double *v, long long n, double q) {
  const double quant = q / 100.0;
  const double virt = (double)(n - 1) * quant;
  long long prev, next;
  if (virt >= (double)(n - 1)) {
    prev = next = n - 1;
  } else if (virt < 0.0) {
    prev = next = 0;
  } else {
    prev = (long long)floor(virt);
    next = prev + 1;
  }
  const double gamma = virt - (double)prev;
  const double a = v[prev], bnext = v[next];
  const double diff = bnext - a;
  // numpy _lerp: a + diff * t, or b - diff * (1 - t) where t >= 0.5
  return gamma >= 0.5 ? bnext - diff * (1.0 - gamma) : a + diff * gamma;
}

__global__ void k_sim_report(SimParams S, const double *sorted, double *p50, double *p99,
                             double *achieved) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= S.n) return;
  const long long n = S.completed[w];
  const double *v = sorted + S.seg[w];
  p50[w] = n ? np_percentile(v, n, 50.0) : 0.0;
  p99[w] = n ? np_percentile(v, n, 99.0) : 0.0;
  const double window = S.duration - S.warmup;
  achieved[w] = window > 0 ? (double)n / window * 1000.0 : 0.0;  // simulate.py:177
}

}  // namespace igp
