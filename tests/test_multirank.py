"""World-size-2 (and 3) CPU runs of the scenario-sharding path (config 4)
over gloo: each rank plans its contiguous block of scenarios, the fixed-size
plan records are all-gathered, and rank 0 checks the assembled batch against
planning every scenario in one process.  The per-rank planner here is the CPU
oracle (test infrastructure); on GPUs bench.py plugs in the CUDA planner and
NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_01713_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_scen, m, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2211_01713_b200 import synth
    from paper_2211_01713_b200.layout import hw_vector
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from instances import make_v100
    hw = make_v100()
    wl, names = synth.scenarios(n_scen, m, hw, seed=4096)
    rank_arr = oracle.name_ranks(list(names))
    a, b = shard.shard_bounds(n_scen, rank, world)
    r = oracle.plan_batch(wl[a:b], np.array(hw_vector(hw)), 32, rank_arr, 1) if b > a else None
    if r is None:
        local = torch.zeros((0, shard.record_width(m)), dtype=torch.int32)
    else:
        local = torch.from_numpy(shard.pack_records(r["gpu_of"], r["units"], r["gpu_count"]))
    full = shard.gather_records(local, n_scen, world)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_scen", [(2, 6), (2, 5), (3, 7)])
def test_sharded_scenarios_gather_over_gloo(tmp_path, world, n_scen, oracle_lib):
    m = 120
    out = str(tmp_path / "full.npy")
    mp.start_processes(_worker, args=(world, _free_port(), n_scen, m, out), nprocs=world,
                       join=True, start_method="spawn")
    full = np.load(out)
    from paper_2211_01713_b200 import synth
    from paper_2211_01713_b200.layout import hw_vector
    from instances import make_v100
    hw = make_v100()
    wl, names = synth.scenarios(n_scen, m, hw, seed=4096)
    r = oracle_lib.plan_batch(wl, np.array(hw_vector(hw)), 32, oracle_lib.name_ranks(list(names)), 2)
    gpu_of, units, gc = shard.unpack_records(full, m)
    np.testing.assert_array_equal(gpu_of, r["gpu_of"])
    np.testing.assert_array_equal(units, r["units"])
    np.testing.assert_array_equal(gc, r["gpu_count"])


def test_shard_bounds_cover_every_scenario_once():
    for n in (0, 1, 5, 4096):
        for w in (1, 2, 3, 8):
            seen = []
            for r in range(w):
                a, b = shard.shard_bounds(n, r, w)
                seen.extend(range(a, b))
            assert seen == list(range(n))


def _stream_worker(rank, world, port, n_streams, length, out_path):
    """Config 5 sharded as independent streams (SURVEY §8e option B): rank r
    runs its block of streams in arrival order, then the per-arrival records
    are all-gathered exactly like scenario plans."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2211_01713_b200 import synth
    from paper_2211_01713_b200.layout import hw_vector
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from instances import make_v100
    hw = make_v100()
    wl, _ = synth.scenarios(n_streams, length, hw, seed=5)
    hv = np.array(hw_vector(hw))
    a, b = shard.shard_bounds(n_streams, rank, world)
    runs = [oracle.stream(wl[s], hv, 32) for s in range(a, b)]
    if runs:
        local = torch.from_numpy(shard.pack_records(np.stack([r["gpu_of"] for r in runs]),
                                                    np.stack([r["units"] for r in runs]),
                                                    np.array([r["gpu_count"] for r in runs])))
    else:
        local = torch.zeros((0, shard.record_width(length)), dtype=torch.int32)
    full = shard.gather_records(local, n_streams, world)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_streams", [(2, 4), (3, 5)])
def test_sharded_streams_gather_over_gloo(tmp_path, world, n_streams, oracle_lib):
    length = 150
    out = str(tmp_path / "streams.npy")
    mp.start_processes(_stream_worker, args=(world, _free_port(), n_streams, length, out),
                       nprocs=world, join=True, start_method="spawn")
    gpu_of, units, gc = shard.unpack_records(np.load(out), length)
    from paper_2211_01713_b200 import synth
    from paper_2211_01713_b200.layout import hw_vector
    from instances import make_v100
    hw = make_v100()
    wl, _ = synth.scenarios(n_streams, length, hw, seed=5)
    for s in range(n_streams):
        r = oracle_lib.stream(wl[s], np.array(hw_vector(hw)), 32)
        np.testing.assert_array_equal(gpu_of[s], r["gpu_of"])
        np.testing.assert_array_equal(units[s], r["units"])
        assert gc[s] == r["gpu_count"]
