"""Host side of the trace rebuild (simulate.py:79-85, :118-124): arrival
counts and per-request records from batch start times, checked against the
reference's own traces (tests/golden/simtrace_*.npz)."""
import numpy as np
import pytest

import golden_io as G

from paper_2211_01713_b200.simulate import SimConfig, _workload_trace, arrival_count


def _loop_count(rate, duration):  # the reference's loop, literally
    spacing = 1000.0 / rate
    t, k, n = 0.0, 0, 0
    while t < duration:
        n += 1
        k += 1
        t = k * spacing
    return n


def test_arrival_count_matches_the_loop():
    rng = np.random.default_rng(3)
    cases = [(100.0, 1000.0), (3.0, 1000.0), (1000.0, 1.0), (7.0, 0.0), (250.0, 4.0)]
    cases += [(float(r), float(d)) for r, d in zip(rng.uniform(1, 6000, 300), rng.uniform(0, 3000, 300))]
    for rate, dur in cases:
        assert arrival_count(rate, dur) == _loop_count(rate, dur), (rate, dur)


@pytest.mark.parametrize("case", G.names("simtrace_"))
def test_trace_rebuild_from_batch_starts(case):
    d = G.load(case)
    cfg = SimConfig(float(d["duration"]), float(d["warmup"]))
    names = [str(x) for x in d["sim_names"]]
    got = []
    for i, name in enumerate(names):
        b = int(d["sim_batch"][i])
        sel = d["trace_w"] == i
        starts = d["trace_dispatch"][sel][::b]  # each batch's first member
        got += _workload_trace(name, float(d["rate"][i]), b, float(d["service"][i]), starts, cfg)
    assert [r.workload for r in got] == [names[i] for i in d["trace_w"]]
    for key, attr in (("trace_arrival", "arrival_ms"), ("trace_dispatch", "dispatch_ms"),
                      ("trace_complete", "complete_ms")):
        np.testing.assert_array_equal(G.bits([getattr(r, attr) for r in got]), G.bits(d[key]))
