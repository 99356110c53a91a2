import collections, re, subprocess
lib = "paper_2211_01713_b200/_lib/libigniter_b200.so"
kerns = ["_ZN3igp7k_placeILi48ELi1ELb0ELb0ELi5EEEvNS_10PlanParamsE",
         "_ZN3igp11k_plan_smemILi48ELb0EEEvNS_10PlanParamsE",
         "_ZN3igp12k_place_fastILi48EEEvNS_10PlanParamsE",
         "_ZN3igp11k_solo_gridEPKdiNS_2HwEPiS3_S3_Py"]
print("# SASS evidence, round 2 final build (nvcc 12.9, -gencode arch=compute_100a,code=sm_100a -fmad=false)")
print("# cuobjdump -sass -fun <mangled> paper_2211_01713_b200/_lib/libigniter_b200.so")
print("# No tensor-core instructions (no HMMA/UTCMMA/UTC*): nothing on this path is a contraction.")
print("# Tile staging is per-thread LDGSTS + LDGDEPBAR / DEPBAR (cp.async commit/wait_group); the")
print("# newcomer's solo row is one UBLKCP (cp.async.bulk, one elected lane) on an mbarrier (SYNCS).")
print("# DFMA appear only inside IEEE division / reciprocal sequences; model multiplies and adds are")
print("# separately rounded DMUL/DADD (-fmad=false).")
for k in kerns:
    out = subprocess.run(["cuobjdump", "-sass", "-fun", k, lib], capture_output=True, text=True).stdout
    ins = [l for l in out.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
    if not ins:
        print(f"\n## {k}: not found"); continue
    ops = collections.Counter()
    for l in ins:
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
        if m: ops[m.group(2).split('.')[0]] += 1
    print(f"\n## {k}\ninstructions: {len(ins)}")
    print("opcode histogram (top 20):")
    for o, c in ops.most_common(20): print(f"  {c:6d} {o}")
    keys = ("LDGSTS", "LDGDEPBAR", "DEPBAR", "UBLKCP", "SYNCS", "HMMA", "UTC", "MUFU.RCP64H", "ATOMS", "VOTE", "SHFL", "LDL", "STL")
    print("selected opcode counts: " + ", ".join(f"{x} {sum(1 for l in ins if x in l)}" for x in keys))
    ex = [l.strip() for l in ins if any(x in l for x in ("LDGSTS", "DEPBAR", "UBLKCP", "SYNCS"))][:8]
    if ex:
        print("excerpt:")
        for l in ex: print("  " + l[:110])
