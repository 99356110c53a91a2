"""Per-phase cycles of one plan's steps (build with -DIGP_TIMING=1; IGP_LIB selects it).
usage: IGP_LIB=build/timing.so python tools/step_timing.py m r_unit b_max flags [S]
(S > 1: a batch of S scenarios, phases of scenario 0 under the batch's load; S=0: one wave)"""
import ctypes, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
import numpy as np, torch
from paper_2211_01713_b200 import _device, _native, synth
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.planner import name_ranks
from instances import make_v100
m, ru, bm, fl = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
S = int(sys.argv[5]) if len(sys.argv) > 5 else 1
hw = make_v100(r_unit=ru)
kw = dict(slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128) if bm == 128 else {}
hv = np.array(hw_vector(hw)); lib = _native.lib_for_compute(); P = _device._ptr
if S == 0:
    S = _device.batch_slots(m, hv, bm, fl)
wl, names = synth.scenarios(S, m, hw, seed=2211, **kw)
d_wl = torch.from_numpy(wl).cuda(); d_rk = torch.from_numpy(name_ranks(list(names))).cuda()
i32 = torch.empty((5, S, m), dtype=torch.int32, device="cuda")
gc = torch.empty(S, dtype=torch.int32, device="cuda"); st = torch.zeros(6 * S + 12, dtype=torch.int64, device="cuda")
er = torch.empty((S, 40), dtype=torch.uint8, device="cuda")
ws = torch.empty(_device.plan_workspace_bytes(S, m, hv, bm, fl), dtype=torch.uint8, device="cuda")
for rep in range(2):
    st.zero_()
    rc = lib.igp_plan_batch_device(P(d_wl), S, m, _device._np_ptr(hv), bm, P(d_rk), 0, P(i32[0]), P(i32[1]),
                                   P(i32[2]), P(i32[3]), P(i32[4]), ctypes.c_void_p(0), P(gc), P(st), P(er),
                                   P(ws), ws.numel(), fl, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
t = st.cpu().numpy()[6 * S:6 * S + 4] / m
extra = (st.cpu().numpy()[6 * S + 4:6 * S + 7] / m).round().tolist()
print(f"S={S} m={m} flags={fl}: cycles/step start+newcomer {t[0]:.0f} | candidates {t[1]:.0f} | "
      f"post-candidates {t[2]:.0f} | commit {t[3]:.0f} | total {t.sum():.0f} ({t.sum()/1.965e3:.2f} us @1.965GHz)"
      f" | extra per step {extra}")
