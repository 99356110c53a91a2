"""Multi-scenario entry points on the B200.

* select_gpu_type (planner.py:333-364) as ONE launch with a hardware profile
  per scenario (IGP_F_HWS), against the reference's known answers and against
  the CPU oracle over T >= 4 GPU types with different unit sizes, power caps
  and prices (first type wins ties, infeasible types skipped, error order).
* plan_many(devices=[...]): the batch split into per-device blocks planned by
  concurrent host threads.
* shard.plan_shard at world size 2: two processes, each plans its block of
  scenarios with the CUDA planner on the GPU and the fixed-size plan records
  are all-gathered (gloo over CUDA tensors: both ranks share the one GPU the
  box leases; NCCL refuses two ranks on one device).
"""
import os
import socket

import numpy as np
import pytest

import golden_io as G
from instances import make_v100, random_instance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _simple(name, k3, slo_ms=40.0, rate_rps=100.0):
    import paper_2211_01713_b200 as igp
    return (igp.WorkloadSpec(name, slo_ms, rate_rps, 0.0, 0.0),
            igp.WorkloadCoefficients(n_kernels=1, k_sch_ms=0.0, k1=0.0, k2=0.0, k3=k3, k4=0.0,
                                     k5=0.0, alpha_power_w=0.0, beta_power_w=10.0,
                                     alpha_cacheutil=0.0, beta_cacheutil=0.0, alpha_cache=0.0))


def test_select_gpu_type_known_answer_one_launch():
    # test_planner.py:250-266: the t4 wins with 15 GPUs at $7.89
    import paper_2211_01713_b200 as igp
    v100 = make_v100()
    t4 = igp.HardwareProfile("t4", 70.0, 1590.0, 10.0, 10.0, -1.0, 0.00475, -0.00902,
                             price_per_hour=0.526)
    specs = [_simple(f"w{i:02d}", 9.9)[0] for i in range(15)]
    coefs = {"v100": {s.name: _simple(s.name, 9.9)[1] for s in specs},
             "t4": {s.name: _simple(s.name, 19.8)[1] for s in specs}}
    chosen = igp.select_gpu_type(specs, [v100, t4], coefs)
    assert chosen.gpu_type == "t4" and len(chosen.gpus) == 15
    assert round(chosen.cost_per_hour, 2) == 7.89


def _types():
    return [make_v100(gpu_type="a", price_per_hour=3.06),
            make_v100(gpu_type="b", r_unit=0.01, price_per_hour=2.9),
            make_v100(gpu_type="c", power_max_w=150.0, price_per_hour=2.5),
            make_v100(gpu_type="d", r_unit=0.05, price_per_hour=2.2),
            make_v100(gpu_type="e", pcie_bw_mb_per_ms=0.001, price_per_hour=0.1)]  # infeasible


@pytest.mark.parametrize("m", [60, 700])
def test_select_gpu_type_vs_oracle_per_type(oracle_lib, m):
    import paper_2211_01713_b200 as igp
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import name_ranks, workload_table
    rng = np.random.default_rng(11 + m)
    base = random_instance(rng, m, make_v100())
    specs = [s for s, _ in base]
    types = _types()
    # per-type coefficients: the base ones scaled differently per type
    coefs_by_type = {}
    for t, hw in enumerate(types):
        coefs_by_type[hw.gpu_type] = {
            s.name: igp.WorkloadCoefficients(**{**c.__dict__, "k3": c.k3 * (1.0 + 0.1 * t)})
            for s, c in base}
    chosen = igp.select_gpu_type(specs, types, coefs_by_type)
    # expected: the oracle plans every type; min cost, first on ties, planning errors skipped
    best = None
    for hw in types:
        pairs = [(s, coefs_by_type[hw.gpu_type][s.name]) for s in specs]
        o = oracle_lib.plan(workload_table(pairs), np.array(hw_vector(hw)), 32,
                            name_ranks([s.name for s in specs]))
        if o["rc"] in (1, 2, 3):
            continue
        assert o["rc"] == 0
        cost = o["gpu_count"] * hw.price_per_hour
        if best is None or cost < best[0]:
            best = (cost, hw, o)
    cost, hw, o = best
    assert chosen.gpu_type == hw.gpu_type and chosen.cost_per_hour == cost
    assert chosen.gpu_count == o["gpu_count"]
    idx = {s.name: i for i, s in enumerate(specs)}
    for g in chosen.gpus:
        for k, a in enumerate(g.allocations):
            i = idx[a.workload]
            assert (g.gpu_index, k) == (int(o["gpu_of"][i]), int(o["pos"][i]))
            assert a.r == int(o["units"][i]) * hw.r_unit
            assert np.float64(g.predicted[a.workload].t_inf_ms).view(np.int64) == \
                G.bits(o["pred"][i, 6])


def test_select_gpu_type_error_order():
    import paper_2211_01713_b200 as igp
    from paper_2211_01713_b200.errors import InfeasibleError
    _, coef = _simple("w", 9.9)
    spec = igp.WorkloadSpec("w", 40.0, 400.0, 0.574, 0.004)  # transfers: the slow link bites
    slow = make_v100(gpu_type="slow", pcie_bw_mb_per_ms=0.001)
    fast = make_v100(gpu_type="fast")
    # missing table for the second type: ValueError once it is reached
    with pytest.raises(ValueError, match="missing coefficients for GPU type fast"):
        igp.select_gpu_type([spec], [slow, fast], {"slow": {"w": coef}})
    # every type infeasible
    with pytest.raises(InfeasibleError, match="no GPU type can host all workloads"):
        igp.select_gpu_type([spec], [slow], {"slow": {"w": coef}})


def test_plan_many_device_blocks_vs_oracle(oracle_lib):
    import paper_2211_01713_b200 as igp
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import name_ranks, workload_table
    hw = make_v100()
    rng = np.random.default_rng(5)
    scen = [random_instance(rng, 80, hw, name_fmt=f"s{k}w{{:03d}}") for k in range(7)]
    stats = [igp.PlanStats() for _ in scen]
    plans = igp.plan_many(scen, hw, stats=stats, devices=["cuda:0", "cuda:0", "cuda:0"])
    assert len(plans) == 7
    for sc, p, st in zip(scen, plans, stats):
        o = oracle_lib.plan(workload_table(sc), np.array(hw_vector(hw)), 32,
                            name_ranks([s.name for s, _ in sc]))
        assert p.gpu_count == o["gpu_count"]
        assert st.model_evals == o["model_evals"] and st.candidate_gpus == o["candidate_gpus"]
        idx = {s.name: i for i, (s, _) in enumerate(sc)}
        for g in p.gpus:
            for a in g.allocations:
                assert g.gpu_index == int(o["gpu_of"][idx[a.workload]])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_worker(rank, world, port, n_scen, m, out_path):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from instances import make_v100
    from paper_2211_01713_b200 import shard, synth
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import name_ranks
    hw = make_v100()
    wl, names = synth.scenario_batch(n_scen, m, hw, seed=4096)
    full = shard.plan_shard(wl, hw_vector(hw), 32, name_ranks(list(names)), device="cuda:0")
    assert full.is_cuda
    if rank == 0:
        np.save(out_path, full.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_scen", [6, 5])
def test_two_rank_cuda_planner_record_gather(tmp_path, n_scen):
    import torch.multiprocessing as mp
    from paper_2211_01713_b200 import _device, shard, synth
    from paper_2211_01713_b200.layout import hw_vector
    from paper_2211_01713_b200.planner import name_ranks
    m = 300
    out = str(tmp_path / "full.npy")
    mp.start_processes(_shard_worker, args=(2, _free_port(), n_scen, m, out), nprocs=2,
                       join=True, start_method="spawn")
    gpu_of, units, gc = shard.unpack_records(np.load(out), m)
    hw = make_v100()
    wl, names = synth.scenario_batch(n_scen, m, hw, seed=4096)
    res = _device.plan_device(wl, hw_vector(hw), 32, name_ranks(list(names)))
    np.testing.assert_array_equal(gpu_of, res["gpu_of"])
    np.testing.assert_array_equal(units, res["units"])
    np.testing.assert_array_equal(gc, res["gpu_count"])
