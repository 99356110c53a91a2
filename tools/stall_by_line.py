"""Aggregate ncu SASS-level stall samples by CUDA source line.

usage: python tools/stall_by_line.py <report.ncu-rep> <kernel mangled name> <lib.so> [topN]
Maps each SASS instruction offset (ncu source page, SASS view) to the
//## File/line annotation emitted by `nvdisasm -g` on the kernel's cubin."""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, kern, lib = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, stdout=subprocess.DEVNULL)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
sec = sass.split(f".text.{kern} ")[1] if f".text.{kern} " in sass else sass.split(f".text.{kern}")[1]
line_of = {}
cur = None
for ln in sec.splitlines():
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
    if ln.startswith("//-----") and line_of:
        break
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 2 and r[0] == "Address")
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
base = int(data[0]["Address"], 16)
key = "Warp Stall Sampling (All Samples)"
agg = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for d in data:
    off = int(d["Address"], 16) - base
    k = line_of.get(off, ("?", 0))
    agg[k] += float(d[key] or 0)
    for c in stall_cols:
        reasons[k][c] += float(d[c] or 0)
tot = sum(agg.values())
print(f"total samples {tot:.0f}")
for (f, l), v in agg.most_common(top):
    r = ", ".join(f"{c[6:]}={n/v*100:.0f}%" for c, n in reasons[(f, l)].most_common(3) if n)
    print(f"{v/tot*100:5.1f}%  {f}:{l}  [{r}]")

# instructions executed per line
ie = collections.Counter()
for d in data:
    off = int(d["Address"], 16) - base
    ie[line_of.get(off, ("?", 0))] += float(d["Instructions Executed"] or 0)
tot_i = sum(ie.values())
print(f"\ninstructions executed {tot_i:.3e}")
for (f, l), v in ie.most_common(top):
    print(f"{v/tot_i*100:5.1f}%  {f}:{l}")
