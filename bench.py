#!/usr/bin/env python
"""Benchmark: provisioning plans/s and candidate evals/s at 10k workloads.

Workload (BASELINE.json metric "provisioning plans/sec and candidate evals/sec
at 10k workloads, 1/2/4/8 B200"): a batch of S independent provisioning
scenarios per GPU, each 10,000 synthetic workloads drawn from the reference
generator's distributions (C2 generator scaled to 10k: r_unit 0.025, b<=32,
V100 profile of pkg/tests/support.py:16-33), planned with Alg. 1/Alg. 2 and
the _build_plan predictions.  One step = one full plan of every scenario in
the batch (prepare + place kernels).  Scenarios shard across ranks with no
data-path collective (weak scaling); for N>1 the fixed-size plan records are
gathered over NCCL inside the timed step.

Parity inside the run: after the timed steps, rank 0 plans a spread subset of
the SAME scenarios (first and last included) with the CPU oracle and asserts
that GPU index, position, units and the _build_plan rows are bit-identical.
The reference arm (--impl reference) plans that same subset, rebuilt from the
same per-scenario seeds (synth.scenario_batch), on all host threads.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
  (--gpus N > 1 without torchrun re-launches itself under torch.distributed.run)

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

M_DEFAULT = 10_000
V100 = dict(gpu_type="v100", power_max_w=300.0, freq_max_mhz=1530.0, power_idle_w=53.5,
            pcie_bw_mb_per_ms=10.0, alpha_f=-1.025, alpha_sch_ms=0.00475,
            beta_sch_ms=-0.00902, r_unit=0.025, price_per_hour=3.06)
FLOPS_PER_MODEL_EVAL = 30   # fp64 ops per resident evaluation
FLOPS_PER_EVAL_CALL = 9     # fp64 ops per device evaluation
# a (workload, GPU) trial reads the candidate
# GPU's resident state once -- 8 fp64 terms per resident (k_act, cache, t_sch,
# alpha_cache, t_load, t_feedback, t_half, power) -- plus the GPU descriptor
# and its two Neumaier fold states (8 + 32 B)
BYTES_PER_RESIDENT_READ = 64
BYTES_PER_TRIAL = 40
KERNELS_PER_PLAN_CALL = 7   # k_fill_int, k_prologue_plan, k_sort, k_build, k_table, k_place (lean + full pass)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scenarios", type=int, default=0, help="scenarios per GPU (0 = auto)")
    ap.add_argument("--workloads", type=int, default=M_DEFAULT)
    ap.add_argument("--seed", type=int, default=2211)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--check", type=int, default=16,
                    help="scenarios of the batch checked bit-exact against the CPU oracle "
                         "(at least the host thread count when the CPU baseline runs)")
    ap.add_argument("--flags", type=int, default=0, help="extra IGP_F_* flags")
    ap.add_argument("--ncu-traffic", type=float, default=None,
                    help="dram bytes per k_place launch from an ncu --set full capture of "
                         "this configuration (profiles/), reported as roofline.traffic")
    return ap.parse_args()


def hardware():
    from paper_2211_01713_b200.model import HardwareProfile
    return HardwareProfile(**V100)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


WAVES = 2  # scenarios per resident warp slot per step (see device_batch_size)


def batch_scenarios(sms: int) -> int:
    """Scenarios per GPU per step without a GPU to ask (the reference arm on
    a CPU-only host): WAVES x 20 per SM, the place kernel's resident warp slots."""
    return sms * 20 * WAVES


def check_indices(S: int, n: int) -> np.ndarray:
    """n scenarios spread over the batch, the first and the last included."""
    return np.unique(np.round(np.linspace(0, S - 1, max(2, min(n, S)))).astype(np.int64))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def bench_config(S: int, m: int, world: int) -> dict:
    return {"workload": f"{S} scenarios x {m} workloads per GPU per step "
                        "(C2 generator scaled to 10k, r_unit 0.025, b<=32, V100 profile; "
                        "per-scenario seeds, synth.scenario_batch)",
            "scenarios_per_gpu": S, "workloads_per_scenario": m,
            "l2": "inputs larger than L2 (%.2f GB per GPU)" % (S * 16 * m * 8 / 1e9),
            "parallelism": f"scenario shards x{world}, NCCL all-gather of plan records"}


def spawn_ranks(args) -> None:
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        loaded = [v for v in sm if v > 0.5 * smax] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


def ncu_traffic(S, m):
    """dram__bytes_read.sum + dram__bytes_write.sum of one k_place launch at
    this configuration, from the committed ncu capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(f"k_place S={S} m={m}", {}).get("dram_bytes")
    except (OSError, ValueError):
        return None


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0}


def fp64_peak():
    """Measured FP64 DFMA flop/s of this GPU (tools/fp64_probe.cu)."""
    import torch
    path = os.path.join(REPO, "tools", "libfp64probe.so")
    if not os.path.exists(path):
        return None, "missing tools/libfp64probe.so"
    lib = ctypes.CDLL(path)
    lib.fp64_probe_flops.restype = ctypes.c_double
    lib.fp64_probe_flops.argtypes = [ctypes.c_int, ctypes.c_int]
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return lib.fp64_probe_flops(0, sms), lib.fp64_probe_flops(1, sms)


def cpu_reference(wl, hw_vec, b_max, rank, threads, stats=False):
    """The CPU oracle (restatement of the reference path, _build_plan rows
    included) on host threads; returns (plans/s, seconds, outputs).  Without
    stats the port may stop a candidate early (a faster CPU baseline than the
    reference's full evaluation)."""
    from oracle import oracle
    oracle.build()
    t0 = time.perf_counter()
    r = oracle.plan_batch(wl, hw_vec, b_max, rank, threads, stats=stats, pred=True)
    dt = time.perf_counter() - t0
    assert r["rc"] == 0
    return wl.shape[0] / dt, dt, r


def device_batch_size(m=M_DEFAULT):
    """The GPU arm's batch: two scenarios per resident warp slot of the place
    kernel (igp_plan_batch_slots), so both arms name the same scenarios.  Two
    waves let the host entry overlap the second wave's input copies and the
    first wave's result copies with compute (e2e 2,002 vs 1,939 plans/s with
    one wave; device 2,096 vs 2,074, profiles/r02)."""
    try:
        import torch
        if torch.cuda.is_available():
            from paper_2211_01713_b200 import _device
            from paper_2211_01713_b200.layout import hw_vector
            return WAVES * _device.batch_slots(m, np.array(hw_vector(hardware())), 32, 0)
    except Exception:  # noqa: BLE001 - the CPU arm also runs without a GPU
        pass
    return batch_scenarios(148)


def run_reference(args, rank, world):
    """--impl reference: the CPU path on all host threads (rank 0 only), on
    the checked subset of the GPU arm's own batch (same seeds, same config)."""
    if rank != 0:
        return
    from paper_2211_01713_b200 import synth
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import name_ranks
    hw = hardware()
    threads = args.cpu_threads or os.cpu_count() or 1
    S = args.scenarios or device_batch_size(args.workloads)
    idx = check_indices(S, max(args.check, threads))
    wl, names = synth.scenario_batch(S, args.workloads, hw, seed=args.seed, indices=idx)
    rk = name_ranks(list(names))
    hv = np.array(hw_vector(hw))
    for _ in range(max(args.warmup, 0) and 1):
        cpu_reference(wl[:threads], hv, 32, rk, threads)
    times = []
    for _ in range(args.steps):
        _, dt, _ = cpu_reference(wl, hv, 32, rk, threads)
        times.append(dt)
    total = sum(times)
    n = len(idx)
    value = n * args.steps / total
    sample = (f"{n} of the {S} scenarios of the GPU arm's batch (indices "
              f"{idx[0]}..{idx[-1]}, evenly spread, same per-scenario seeds) x {args.workloads} "
              "workloads per step, plan() with _build_plan rows, one scenario per host thread "
              "at a time (oracle/igniter_oracle.c, pthreads)")
    line = {
        "impl": "reference",
        "metric": "provisioning plans/sec at 10k workloads",
        "value": value, "unit": "plans/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(S, args.workloads, world),
        "cpu_baseline": {"value": value, "unit": "plans/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)  # does not return
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch.distributed as dist
        if args.impl == "reference":
            if rank != 0:
                return
        else:
            dist.init_process_group("nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    from paper_2211_01713_b200 import _device, _native, synth
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import IGP_F_STATS, name_ranks

    lib = _native.lib_for_compute()
    hw = hardware()
    hv = np.array(hw_vector(hw))
    b_max = 32
    m = args.workloads
    S = args.scenarios or WAVES * _device.batch_slots(m, hv, b_max, args.flags, device)
    flags = args.flags
    threads = args.cpu_threads or os.cpu_count() or 1

    # ---- synthetic inputs (different seed per rank: weak scaling) ----
    seed = args.seed + 1000 * rank
    wl_np, names = synth.scenario_batch(S, m, hw, seed=seed)
    rk_np = name_ranks(list(names))
    wl_pin = torch.from_numpy(wl_np).pin_memory()
    rk_pin = torch.from_numpy(rk_np).pin_memory()
    del wl_np
    d_wl = wl_pin.to(device)
    d_rk = rk_pin.to(device)
    i32 = torch.empty((5, S, m), dtype=torch.int32, device=device)
    d_pred = torch.empty((S, m, 10), dtype=torch.float64, device=device)
    d_gc = torch.empty(S, dtype=torch.int32, device=device)
    d_st = torch.empty((S, 6), dtype=torch.int64, device=device)
    d_err = torch.empty((S, ctypes.sizeof(_native.IgpError)), dtype=torch.uint8, device=device)
    ws = torch.empty(max(_device.plan_workspace_bytes(S, m, hv, b_max, fl) for fl in
                         (flags, flags | IGP_F_STATS)), dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device)
    P = _device._ptr
    hp = _device._np_ptr(hv)

    def call(fn, fl):
        rc = fn(P(d_wl), S, m, hp, b_max, P(d_rk), 0, P(i32[0]), P(i32[1]), P(i32[2]), P(i32[3]),
                P(i32[4]), P(d_pred), P(d_gc), P(d_st), P(d_err), P(ws), ws.numel(), fl,
                ctypes.c_void_p(stream.cuda_stream))
        assert rc == 0, rc

    # ---- reference-equivalent work: one exact-stats pass (untimed) ----
    call(lib.igp_plan_batch_device, flags | IGP_F_STATS)
    torch.cuda.synchronize()
    st = d_st.cpu().numpy()
    assert (d_err.cpu().numpy().view(_native.err_dtype())["code"] == 0).all()
    ref_model_evals = int(st[:, 0].sum())
    ref_cands = int(st[:, 1].sum())
    ref_calls = int(st[:, 2].sum())
    ref_res_reads = int(st[:, 4].sum())
    stats_exact = st.copy()
    gpus_exact = d_gc.cpu().numpy().copy()
    units_exact = i32[2].cpu().numpy().copy()

    # N>1: the fixed-size plan records (GPU index + units per workload, GPU
    # count) of every rank's shard are all-gathered over NCCL inside the step
    if world > 1:
        import torch.distributed as dist
        from paper_2211_01713_b200 import shard

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        call(lib.igp_plan_prepare_device, flags)
        if ev is not None:
            ev[1].record(stream)
        call(lib.igp_plan_place_device, flags)
        if ev is not None:
            ev[2].record(stream)
        if world > 1:
            shard.gather_records(shard.pack_records(i32[0], i32[2], d_gc), S * world, world)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # the fast path must reproduce the exact pass bit for bit
    assert np.array_equal(d_gc.cpu().numpy(), gpus_exact)
    assert np.array_equal(i32[2].cpu().numpy(), units_exact)
    performed_calls = int(d_st.cpu().numpy()[:, 3].sum())

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e_start.record(stream)
        for k in range(args.steps):
            step(evs[k])
        e_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    clocks = clk.summary()
    ms_total = e_start.elapsed_time(e_end)
    place_ms = [e[1].elapsed_time(e[2]) for e in evs]
    prep_ms = [e[0].elapsed_time(e[1]) for e in evs]
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    value = S * world * args.steps / (ms_total / 1e3)
    evals_per_s = ref_model_evals * world * args.steps / (ms_total / 1e3)

    # ---- parity of the timed steps' outputs (untimed): the CPU oracle on a
    # spread subset of this batch, plus the CPU baseline timed on the same plans
    dev_out = {"gpu_of": i32[0].cpu().numpy(), "pos": i32[1].cpu().numpy(),
               "units": i32[2].cpu().numpy(), "gpu_count": d_gc.cpu().numpy()}
    cpu = None
    parity = None
    if rank == 0 and args.check > 0:
        idx = check_indices(S, args.check if args.no_cpu_baseline else max(args.check, threads))
        wl_chk = wl_pin.numpy()[idx]
        v, dt, o = cpu_reference(wl_chk, hv, b_max, rk_np, threads)
        pred_chk = d_pred[torch.from_numpy(idx).to(device)].cpu().numpy()
        for key in ("gpu_of", "pos", "units", "gpu_count"):
            assert np.array_equal(dev_out[key][idx], o[key]), f"parity: {key} differs from the oracle"
        assert np.array_equal(pred_chk.view(np.int64), o["pred"].view(np.int64)), \
            "parity: _build_plan rows differ from the oracle"
        # PlanStats: the oracle's exact counters on four of them (untimed)
        sidx = idx[np.unique(np.round(np.linspace(0, len(idx) - 1, 4)).astype(np.int64))]
        _, _, os_ = cpu_reference(wl_pin.numpy()[sidx], hv, b_max, rk_np, threads, stats=True)
        assert np.array_equal(stats_exact[sidx, 0], os_["stats"][:, 0]), "parity: model_evals"
        assert np.array_equal(stats_exact[sidx, 1], os_["stats"][:, 1]), "parity: candidate_gpus"
        parity = {"scenarios_checked": [int(i) for i in idx], "oracle": "oracle/igniter_oracle.c",
                  "fields": "gpu_of, pos, units, gpu_count, _build_plan rows (int64 bit patterns); "
                            "PlanStats model_evals / candidate_gpus of the exact pass on "
                            f"scenarios {[int(i) for i in sidx]}",
                  "result": "bit-exact"}
        if not args.no_cpu_baseline:
            cpu = {"value": v, "unit": "plans/s", "cores": threads, "kind": "port",
                   "cpu_model": cpu_model(),
                   "sample": f"{len(idx)} of this batch's {S} scenarios (indices {idx[0]}..{idx[-1]}, "
                             f"evenly spread) x {m}-workload plans with _build_plan rows, one per "
                             f"host thread at a time, {dt:.1f} s (oracle/igniter_oracle.c "
                             "restatement, pthreads)"}
        del wl_chk, pred_chk, o

    # ---- e2e through the host-buffer C-ABI entry (pinned buffers, copies timed) ----
    e2e = None
    e2e_launches = 0
    if not args.no_e2e:
        wl_host = wl_pin.numpy()
        rk_host = rk_pin.numpy()
        out = {k: torch.empty((S, m), dtype=torch.int32).pin_memory().numpy()
               for k in ("gpu_of", "pos", "units", "batch", "lb")}
        out["pred"] = torch.empty((S, m, 10), dtype=torch.float64).pin_memory().numpy()
        out["gpu_count"] = torch.empty(S, dtype=torch.int32).pin_memory().numpy()
        out["stats"] = torch.empty((S, 6), dtype=torch.int64).pin_memory().numpy()
        out["err"] = torch.zeros(S * _native.err_dtype().itemsize, dtype=torch.uint8).pin_memory().numpy().view(_native.err_dtype())
        del ws
        pred_ref = d_pred.cpu().numpy().view(np.int64) if rank == 0 else None
        del d_pred, d_wl
        torch.cuda.empty_cache()
        _device.plan_host(wl_host, hv, b_max, rk_host, flags=flags, device=device, want_pred=True,
                          out=out)
        torch.cuda.synchronize()
        ea = torch.cuda.Event(enable_timing=True)
        eb = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        ea.record(stream)
        for _ in range(args.steps):
            _device.plan_host(wl_host, hv, b_max, rk_host, flags=flags, device=device,
                              want_pred=True, out=out)
        eb.record(stream)
        torch.cuda.synchronize()
        e2e_ms = ea.elapsed_time(eb)
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        assert np.array_equal(out["units"], units_exact)
        assert np.array_equal(out["gpu_of"], dev_out["gpu_of"])
        if pred_ref is not None:
            assert np.array_equal(out["pred"].view(np.int64), pred_ref)
        h2d = wl_host.nbytes + rk_host.nbytes
        d2h = sum(out[k].nbytes for k in ("gpu_of", "pos", "units", "batch", "lb", "pred",
                                          "gpu_count", "stats", "err"))
        chunks = min(2, max(1, S // 128))
        e2e_launches = KERNELS_PER_PLAN_CALL * chunks * args.steps
        e2e = {"value": S * world * args.steps / (e2e_ms / 1e3), "unit": "plans/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_ms / args.steps,
               "path": f"igp_plan_batch_host (pinned host buffers; {chunks} scenario chunks on "
                       "their own streams: H2D / kernels / D2H overlapped), _build_plan rows "
                       "returned and checked equal to the device leg"}

    # ---- roofline of the dominant kernel (k_place, the place stage) ----
    # Both rooflines count the REFERENCE's work (exact-stats pass), not the
    # smaller amount the pruned fast path performs.
    place_avg = sum(place_ms) / len(place_ms)
    bytes_per_launch = BYTES_PER_RESIDENT_READ * ref_res_reads + BYTES_PER_TRIAL * ref_cands
    achieved_gbs = bytes_per_launch / (place_avg / 1e3) / 1e9
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    roofline = {
        "bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
        "frac": achieved_gbs / hbm_peak if hbm_peak else None,
        "traffic": args.ncu_traffic if args.ncu_traffic is not None else ncu_traffic(S, m),
        "kernel": "k_place (igp_plan_place_device)",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth, burst)"
                       if "hbm_gbs" in peaks else "fallback 6650 GB/s (B200_PROFILING.md)",
        "bytes_definition": f"{BYTES_PER_RESIDENT_READ} B x reference resident reads "
                            f"({ref_res_reads}) + {BYTES_PER_TRIAL} B x reference candidate "
                            f"trials ({ref_cands}) per launch",
        "bytes_per_launch": bytes_per_launch,
        "place_ms_avg": place_avg, "prepare_ms_avg": sum(prep_ms) / len(prep_ms),
        "place_share_of_step": place_avg / (ms_total / args.steps) if world == 1 else None,
    }
    flops_per_launch = FLOPS_PER_MODEL_EVAL * ref_model_evals + FLOPS_PER_EVAL_CALL * ref_calls
    peak_fma, peak_add = fp64_peak()
    achieved_tf = flops_per_launch / (place_avg / 1e3) / 1e12
    roofline_fp64 = {
        "bound": "fp64", "achieved": achieved_tf,
        "peak": (peak_fma / 1e12) if peak_fma else None, "unit": "TFLOP/s",
        "frac": (achieved_tf / (peak_fma / 1e12)) if peak_fma else None,
        "peak_source": "measured DFMA rate on this GPU, tools/fp64_probe.cu "
                       "(MEASURED_PEAKS.json has no FP64 figure)",
        "flops_definition": f"{FLOPS_PER_MODEL_EVAL} x reference model_evals + "
                            f"{FLOPS_PER_EVAL_CALL} x reference _eval_entries calls per launch",
    }

    if rank == 0:
        line = {
            "metric": "provisioning plans/sec at 10k workloads",
            "value": value, "unit": "plans/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": bench_config(S, m, world),
            "candidate_evals_per_s": evals_per_s,
            "candidate_evals_definition": "reference PlanStats.model_evals (planner.py:156-157) "
                                          "of the planned scenarios, from an exact-stats pass",
            "reference_counters_per_gpu_step": {"model_evals": ref_model_evals,
                                                "candidate_gpus": ref_cands,
                                                "eval_calls": ref_calls,
                                                "resident_reads": ref_res_reads,
                                                "eval_calls_run_fast_path": performed_calls},
            "gpu_launches": KERNELS_PER_PLAN_CALL * args.steps + e2e_launches,
            "clocks": clocks,
            "parity": parity,
            "roofline": roofline,
            "roofline_fp64": roofline_fp64,
            "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
