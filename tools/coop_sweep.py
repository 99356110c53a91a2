"""Single-plan latency of the cooperative kernel vs CTA count (flags bits 16..27).
usage: python tools/coop_sweep.py m r_unit b_max ctas,ctas,...   (0 = default heuristic)"""
import ctypes, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
import numpy as np, torch
from paper_2211_01713_b200 import _device, _native, synth
from paper_2211_01713_b200.layout import hw_vector
from paper_2211_01713_b200.planner import IGP_F_COOP, IGP_F_CTA, name_ranks
from instances import make_v100
m, ru, bm = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
ctas = [int(c) for c in sys.argv[4].split(",")]
hw = make_v100(r_unit=ru)
kw = dict(slo=(20.0, 100.0), rate=(50.0, 6000.0), b_max=128) if bm == 128 else {}
wl, names = synth.scenarios(1, m, hw, seed=2211, **kw)
hv = np.array(hw_vector(hw)); lib = _native.lib_for_compute(); P = _device._ptr
d_wl = torch.from_numpy(wl).cuda(); d_rk = torch.from_numpy(name_ranks(list(names))).cuda()
i32 = torch.empty((5, 1, m), dtype=torch.int32, device="cuda")
gc = torch.empty(1, dtype=torch.int32, device="cuda"); st = torch.empty((1, 6), dtype=torch.int64, device="cuda")
er = torch.empty((1, 40), dtype=torch.uint8, device="cuda")
ws = torch.empty(_device.plan_workspace_bytes(1, m, hv, bm, IGP_F_COOP | IGP_F_CTA), dtype=torch.uint8, device="cuda")
ref = None
for c in ctas + [-1]:
    fl = IGP_F_CTA if c < 0 else (IGP_F_COOP | IGP_F_CTA | (c << 16))
    def run():
        rc = lib.igp_plan_batch_device(P(d_wl), 1, m, _device._np_ptr(hv), bm, P(d_rk), 0, P(i32[0]), P(i32[1]),
                                       P(i32[2]), P(i32[3]), P(i32[4]), ctypes.c_void_p(0), P(gc), P(st), P(er),
                                       P(ws), ws.numel(), fl, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
    run(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    reps = 3 if m <= 20000 else 1
    a.record()
    for _ in range(reps): run()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    u = i32[2].cpu().numpy().copy()
    same = ref is None or np.array_equal(u, ref)
    ref = u if ref is None else ref
    print(f"m={m} r={ru} ctas={c if c >= 0 else 'CTA-mode'}: {ms:.2f} ms ({ms*1e3/m:.2f} us/step) same={same} "
          f"cands_run={int(st[0,5])}", flush=True)
