"""Ad-hoc timing of prepare+place (device-resident inputs, CUDA events).

usage: python tools/quick_time.py S,m,flags [S,m,flags ...]   (IGP_LIB selects a variant; S=0: batch slots)"""
import ctypes, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np, torch
from paper_2211_01713_b200 import _device, _native, synth
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.model import HardwareProfile
from paper_2211_01713_b200.planner import name_ranks

hw = HardwareProfile("v100", 300.0, 1530.0, 53.5, 10.0, -1.025, 0.00475, -0.00902, r_unit=0.025, price_per_hour=3.06)
hv = np.array(hw_vector(hw))
lib = _native.lib_for_compute()
dev = torch.device("cuda", 0)
P = _device._ptr
cfgs = [tuple(int(v) for v in c.split(",")) for c in sys.argv[1:]] or [(2368, 10000, 0)]
for S, m, flags in cfgs:
    if S == 0:  # one scenario per resident slot of this build
        S = _device.batch_slots(m, hv, 32, flags)
    wl, names = synth.scenarios(S, m, hw, seed=2211)
    d_wl = torch.from_numpy(wl).to(dev)
    d_rk = torch.from_numpy(name_ranks(list(names))).to(dev)
    i32 = torch.empty((5, S, m), dtype=torch.int32, device=dev)
    d_gc = torch.empty(S, dtype=torch.int32, device=dev)
    d_st = torch.empty((S, 6), dtype=torch.int64, device=dev)
    d_err = torch.empty((S, 40), dtype=torch.uint8, device=dev)
    ws = torch.empty(_device.plan_workspace_bytes(S, m, hv, 32, flags), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    def call(fn):
        rc = fn(P(d_wl), S, m, _device._np_ptr(hv), 32, P(d_rk), 0, P(i32[0]), P(i32[1]), P(i32[2]), P(i32[3]),
                P(i32[4]), ctypes.c_void_p(0), P(d_gc), P(d_st), P(d_err), P(ws), ws.numel(), flags,
                ctypes.c_void_p(st.cuda_stream))
        assert rc == 0
    call(lib.igp_plan_batch_device); torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); call(lib.igp_plan_prepare_device); e[1].record(); call(lib.igp_plan_place_device); e[2].record()
    torch.cuda.synchronize()
    place = e[1].elapsed_time(e[2]); prep = e[0].elapsed_time(e[1])
    stats = d_st.cpu().numpy()
    print(f"[{os.path.basename(_native.LIB_PATH)}] S={S} m={m} fl={flags}: place {place:.1f} ms prep {prep:.1f} ms "
          f"-> {S/((place+prep)/1e3):.1f} plans/s; evals_run/scen={stats[:,3].mean():.0f} "
          f"cands_run/scen={stats[:,5].mean():.0f} exact_fallback/scen={stats[:,4].mean():.1f} "
          f"gpus={d_gc[:3].tolist()} err={np.unique(d_err.cpu().numpy().view(_native.err_dtype())['code'])}", flush=True)
    del ws, d_wl, i32
    torch.cuda.empty_cache()
