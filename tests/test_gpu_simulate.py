"""Request-level replay (simulate.py:139-198) on the GPU against the
reference's own simulate() fixtures (tests/golden/sim_*.npz)."""
import numpy as np
import pytest

import golden_io as G
from instances import hw_from_golden, workloads_from_golden

import paper_2211_01713_b200 as igp
from paper_2211_01713_b200 import errors
from paper_2211_01713_b200.simulate import SimConfig, replay_arrays, simulate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cfg(d):
    return SimConfig(float(d["duration"]), float(d["warmup"]), str(d["arrival"]))


@pytest.mark.parametrize("case", [c for c in G.names("sim_") if c != "sim_poisson"])
def test_replay_matches_reference(case):
    d = G.load(case)
    r = replay_arrays(d["rate"], d["sim_batch"], d["service"], _cfg(d))
    if str(d["err_class"]) == "UnstableQueueError":
        names = [str(x) for x in d["sim_names"]]
        bad = [i for i in range(len(names)) if r["backlog"][i] > 10 * d["sim_batch"][i]]
        msg = (f"{names[bad[0]]}: queue depth {int(r['backlog'][bad[0]])} exceeds "
               f"{10 * int(d['sim_batch'][bad[0]])} at horizon end")
        assert msg == str(d["err_msg"])
        return
    np.testing.assert_array_equal(r["completed"], d["completed"])
    np.testing.assert_array_equal(r["max_depth"], d["max_depth"])
    np.testing.assert_array_equal(G.bits(r["p50"]), G.bits(d["p50"]))
    np.testing.assert_array_equal(G.bits(r["p99"]), G.bits(d["p99"]))
    np.testing.assert_array_equal(G.bits(r["achieved"]), G.bits(d["achieved"]))


def test_simulate_api_on_device_plan():
    d = G.load("sim_rand60_10s")
    wls = workloads_from_golden(d)
    hw = hw_from_golden(d)
    specs = {s.name: s for s, _ in wls}
    coefs = {s.name: c for s, c in wls}
    rep = simulate(igp.plan(wls, hw), specs, coefs, hw, _cfg(d))
    assert [w.workload for w in rep.workloads] == [str(x) for x in d["sim_names"]]
    np.testing.assert_array_equal(G.bits([w.p99_ms for w in rep.workloads]), G.bits(d["p99"]))
    assert [w.violation for w in rep.workloads] == list(d["violation"])


def test_simulate_errors_like_reference():
    d = G.load("sim_c1_30s")
    wls = workloads_from_golden(d)
    hw = hw_from_golden(d)
    specs = {s.name: s for s, _ in wls}
    coefs = {s.name: c for s, c in wls}
    with pytest.raises(errors.UnstableQueueError) as ei:
        simulate(igp.plan(wls, hw), specs, coefs, hw, _cfg(d))
    assert str(ei.value) == str(d["err_msg"])
    d = G.load("sim_poisson")
    wls = workloads_from_golden(d)
    with pytest.raises(TypeError) as ei:
        simulate(igp.plan(wls, hw), {s.name: s for s, _ in wls}, {s.name: c for s, c in wls}, hw,
                 _cfg(d))
    assert str(ei.value) == str(d["err_msg"])


@pytest.mark.parametrize("case", G.names("simtrace_"))
def test_trace_matches_reference(case, tmp_path):
    from paper_2211_01713_b200.simulate import write_trace_csv
    d = G.load(case)
    wls = workloads_from_golden(d)
    hw = hw_from_golden(d)
    specs = {s.name: s for s, _ in wls}
    coefs = {s.name: c for s, c in wls}
    rep, trace = simulate(igp.plan(wls, hw), specs, coefs, hw, _cfg(d), collect_trace=True)
    names = [str(x) for x in d["sim_names"]]
    assert [r.workload for r in trace] == [names[i] for i in d["trace_w"]]
    for key, attr in (("trace_arrival", "arrival_ms"), ("trace_dispatch", "dispatch_ms"),
                      ("trace_complete", "complete_ms")):
        np.testing.assert_array_equal(G.bits([getattr(r, attr) for r in trace]), G.bits(d[key]))
    np.testing.assert_array_equal(G.bits([w.p99_ms for w in rep.workloads]), G.bits(d["p99"]))
    path = tmp_path / "trace.csv"
    write_trace_csv(path, trace)
    lines = path.read_text().splitlines()
    assert lines[0] == "workload,arrival_ms,dispatch_ms,complete_ms"
    assert len(lines) == len(trace) + 1
    i = len(trace) // 2
    assert lines[1 + i] == (f"{names[d['trace_w'][i]]},{float(d['trace_arrival'][i])!r},"
                            f"{float(d['trace_dispatch'][i])!r},{float(d['trace_complete'][i])!r}")
