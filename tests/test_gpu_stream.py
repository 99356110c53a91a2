"""Online stream (BASELINE config 5) on the GPU vs the reference-internals
driver (golden fixtures, make_golden.py stream_reference) and the CPU oracle."""
import numpy as np
import pytest

import golden_io as G

from paper_2211_01713_b200 import synth
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.stream import StreamPlanner

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _hw(d):
    from instances import hw_from_golden
    return hw_from_golden(d)


def _push_in_chunks(sp, wl, chunks):
    out = {k: [] for k in ("gpu_of", "pos", "code")}
    k = 0
    for c in chunks:
        r = sp.push_arrays(wl[:, :, k:k + c])
        for key in out:
            out[key].append(r[key])
        k += c
    return {key: np.concatenate(v, axis=1) for key, v in out.items()}


@pytest.mark.parametrize("case", G.names("stream_"))
@pytest.mark.parametrize("chunks", ["one", "ragged"])
def test_stream_matches_reference_driver(case, chunks):
    d = G.load(case)
    n = d["wl"].shape[1]
    sizes = [n] if chunks == "one" else [1, 7, 64, 3, n - 75] if n > 80 else [n]
    sp = StreamPlanner(_hw(d), capacity=n, b_max=int(d["b_max"]))
    r = _push_in_chunks(sp, d["wl"][None], sizes)
    np.testing.assert_array_equal(r["gpu_of"][0], d["gpu_of"])
    np.testing.assert_array_equal(r["pos"][0], d["pos"])
    np.testing.assert_array_equal(r["code"][0], d["code"])
    snap = sp.snapshot()
    np.testing.assert_array_equal(snap["units"][0], d["units"])
    np.testing.assert_array_equal(snap["gpu_of"][0], d["gpu_of"])
    assert int(snap["gpu_count"][0]) == int(d["gpu_count"])


def test_many_streams_vs_oracle(oracle_lib):
    from instances import make_v100
    hw = make_v100()
    S, n = 6, 1500
    wl, _ = synth.scenarios(S, n, hw, seed=77)
    sp = StreamPlanner(hw, capacity=n, n_streams=S)
    r = _push_in_chunks(sp, wl, [100] * 15)
    snap = sp.snapshot(with_predictions=True)
    for s in range(S):
        o = oracle_lib.stream(wl[s], np.array(hw_vector(hw)), 32)
        np.testing.assert_array_equal(r["gpu_of"][s], o["gpu_of"])
        np.testing.assert_array_equal(r["pos"][s], o["pos"])
        np.testing.assert_array_equal(r["code"][s], o["code"])
        np.testing.assert_array_equal(snap["units"][s], o["units"])
        assert int(snap["gpu_count"][s]) == o["gpu_count"]
        assert int(snap["err"][s]["code"]) == 0
        assert np.isfinite(snap["pred"][s]).all()


def test_stream_r_unit_001_b128_vs_oracle(oracle_lib):
    from instances import make_v100
    hw = make_v100(r_unit=0.01)
    S, n = 3, 800
    wl, _ = synth.scenarios(S, n, hw, seed=78, slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128)
    sp = StreamPlanner(hw, capacity=n, n_streams=S, b_max=128)
    r = _push_in_chunks(sp, wl, [200, 200, 400])
    snap = sp.snapshot()
    for s in range(S):
        o = oracle_lib.stream(wl[s], np.array(hw_vector(hw)), 128)
        np.testing.assert_array_equal(r["gpu_of"][s], o["gpu_of"])
        np.testing.assert_array_equal(snap["units"][s], o["units"])


def test_stream_pool_overflow_is_reported():
    """A stream whose record pool runs out (pool factor 1 via flags bits 8..15)
    reports it instead of silently dropping arrivals."""
    from instances import make_v100
    from paper_2211_01713_b200.errors import NativeError
    hw = make_v100()
    wl, _ = synth.scenarios(1, 600, hw, seed=79)
    sp = StreamPlanner(hw, capacity=600, flags=1 << 8)
    with pytest.raises(NativeError, match="record pool"):
        sp.push_arrays(wl)


@pytest.mark.parametrize("case", G.names("stream_"))
def test_whole_gpu_stream_matches_reference_driver(case):
    """One stream, every push on the whole GPU (cooperative steps), against
    the reference-internals driver -- including the fixtures' rejected and
    raising arrivals (the per-CTA kernel resumes at the first one that needs
    the exact sequence)."""
    from paper_2211_01713_b200.stream import IGP_F_COOP
    d = G.load(case)
    n = d["wl"].shape[1]
    sp = StreamPlanner(_hw(d), capacity=n, b_max=int(d["b_max"]), whole_gpu=True)
    out = {k: [] for k in ("gpu_of", "pos", "code")}
    k = 0
    for c in ([n] if n < 80 else [5, 60, n - 65]):
        import torch
        dw = torch.from_numpy(np.ascontiguousarray(d["wl"][None, :, k:k + c])).cuda()
        g, p, cd = sp.push_device(dw, flags=sp.flags | IGP_F_COOP | (4 << 16))
        out["gpu_of"].append(g.cpu().numpy())
        out["pos"].append(p.cpu().numpy())
        out["code"].append(cd.cpu().numpy() & 0xFF)
        sp.check_errors()
        k += c
    r = {key: np.concatenate(v, axis=1) for key, v in out.items()}
    np.testing.assert_array_equal(r["gpu_of"][0], d["gpu_of"])
    np.testing.assert_array_equal(r["pos"][0], d["pos"])
    np.testing.assert_array_equal(r["code"][0], d["code"])
    snap = sp.snapshot()
    np.testing.assert_array_equal(snap["units"][0], d["units"])
    assert int(snap["gpu_count"][0]) == int(d["gpu_count"])


def test_whole_gpu_stream_20k_prefix_vs_oracle(oracle_lib):
    """BASELINE config 5 as one stream: the C2 generator's arrivals (seed 5)
    pushed in 2,048-arrival pushes, per-CTA steps first and cooperative
    whole-GPU steps from COOP_FROM_ARRIVALS on (stream.push_flags), bit-exact
    against the oracle's arrival-order driver on a 24,576-arrival prefix."""
    import torch
    from instances import make_v100
    from paper_2211_01713_b200.stream import COOP_FROM_ARRIVALS
    hw = make_v100()
    n = 24_576
    assert n > COOP_FROM_ARRIVALS
    wl, _ = synth.scenarios(1, n, hw, seed=5)
    sp = StreamPlanner(hw, capacity=n, whole_gpu=True)
    d_wl = torch.from_numpy(np.ascontiguousarray(
        wl[0].reshape(16, n // 2048, 2048).transpose(1, 0, 2))).cuda()
    gs, ps, cs = [], [], []
    for c in range(n // 2048):
        g, p, cd = sp.push_device(d_wl[c][None])
        gs.append(g.cpu().numpy()[0])
        ps.append(p.cpu().numpy()[0])
        cs.append(cd.cpu().numpy()[0] & 0xFF)
    sp.check_errors()
    o = oracle_lib.stream(wl[0], np.array(hw_vector(hw)), 32)
    np.testing.assert_array_equal(np.concatenate(gs), o["gpu_of"])
    np.testing.assert_array_equal(np.concatenate(ps), o["pos"])
    np.testing.assert_array_equal(np.concatenate(cs), o["code"])
    snap = sp.snapshot(with_predictions=True)
    np.testing.assert_array_equal(snap["units"][0], o["units"])
    assert int(snap["gpu_count"][0]) == o["gpu_count"]
