"""Small runs of every kernel family for compute-sanitizer (tools/gpu_sanitize.sh)."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
import numpy as np
import paper_2211_01713_b200 as igp
from paper_2211_01713_b200 import _device, synth
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.planner import IGP_F_COOP, IGP_F_CTA, IGP_F_STATS, name_ranks
from paper_2211_01713_b200.stream import StreamPlanner
from paper_2211_01713_b200.simulate import SimConfig, simulate
from instances import make_v100, twelve_workload_instance, random_instance
hw = make_v100()
hv = hw_vector(hw)
wl, names = synth.scenarios(6, 300, hw, seed=3)
rk = name_ranks(list(names))
for fl in (0, IGP_F_STATS, IGP_F_CTA, 32, 64):
    _device.plan_device(wl, hv, 32, rk, flags=fl)
w1, n1 = synth.scenarios(1, 800, hw, seed=4)
_device.plan_device(w1, hv, 32, name_ranks(list(n1)), flags=IGP_F_COOP | IGP_F_CTA)
sp = StreamPlanner(hw, capacity=300, n_streams=3)
sp.push_arrays(wl[:3, :, :150]); sp.push_arrays(wl[:3, :, 150:]); sp.snapshot(with_predictions=True)
inst = twelve_workload_instance()
p = igp.plan(inst, hw)
igp.predict_gpu(p.gpus[0].allocations, {s.name: s for s, _ in inst}, {s.name: c for s, c in inst}, hw)
igp.exhaustive_plan(inst[:3], hw)
simulate(igp.plan(inst[:6], hw), {s.name: s for s, _ in inst}, {s.name: c for s, c in inst}, hw,
         SimConfig(2000.0, 100.0))
_device.solo_grid(wl[0][:, :50], hv, 32)
rng = np.random.default_rng(1)
ri = random_instance(rng, 4, hw)
igp.alloc_gpus({s.name: s for s, _ in ri}, {s.name: c for s, c in ri}, hw, [], ri[0][0].name,
               igp.appropriate_batch(ri[0][0], hw), 0.05)
simulate(igp.plan(inst[:4], hw), {s.name: s for s, _ in inst}, {s.name: c for s, c in inst}, hw,
         SimConfig(300.0, 50.0), collect_trace=True)
_device.components(wl[0][:, :64], np.arange(1, 65), np.full(64, 0.1), np.full(64, 0.5),
                   np.arange(64) % 9, np.linspace(100.0, 500.0, 64), hv)
igp.power_demand(hw, [50.0, 60.5, 70.25]); igp.power_demand(hw, [])
# round 2: the shared-memory plan kernel (one CTA per scenario; a declined
# scenario and the wide-margin exact path), the certified-margin batch kernel,
# select_gpu_type in one launch
IGP_F_SMEM, IGP_F_FAST = 8, 1 << 29
w2, n2 = synth.scenarios(3, 400, hw, seed=5)
r2 = name_ranks(list(n2))
_device.plan_device(w2[:1], hv, 32, r2, flags=IGP_F_SMEM | IGP_F_CTA)
w2b = w2.copy(); w2b[1, 0, 10] = 1e-3  # a prologue error: declined
_device.plan_device(w2b, hv, 32, r2, flags=IGP_F_SMEM | IGP_F_CTA)
os.environ["IGP_FAST_DELTA"] = "0.5"
_device.plan_device(w2[:1], hv, 32, r2, flags=IGP_F_SMEM | IGP_F_CTA)
_device.plan_device(w2, hv, 32, r2, flags=IGP_F_FAST)
del os.environ["IGP_FAST_DELTA"]
_device.plan_device(w2, hv, 32, r2, flags=IGP_F_FAST)
igp.select_gpu_type([s for s, _ in inst], [hw, make_v100(gpu_type="b", r_unit=0.05)],
                    {"v100": {s.name: c for s, c in inst}, "b": {s.name: c for s, c in inst}})
print("sanitize workload done")
