"""Top SASS instructions of an ncu capture by stall samples, with their CUDA
source line (nvdisasm -g line table of the library the capture ran).

usage: python tools/top_sass.py <report.ncu-rep> <kernel mangled name> <lib.so> [topN] [file:line]"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, kern, lib = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
only = sys.argv[5] if len(sys.argv) > 5 else None
tmp = tempfile.mkdtemp()
subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp,
                      stdout=subprocess.DEVNULL)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True,
                      text=True).stdout
sec = sass.split(f".text.{kern}:")[1].split(".section")[0]
line_of, cur = {}, None
for ln in sec.splitlines():
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 2 and r[0] == "Address")
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
base = int(data[0]["Address"], 16)
key = "Warp Stall Sampling (All Samples)"
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(d[key] or 0) for d in data)
items = []
for d in data:
    off = int(d["Address"], 16) - base
    ln = line_of.get(off, "?")
    if only and ln != only:
        continue
    v = float(d[key] or 0)
    rs = sorted(((float(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    items.append((v, off, ln, d.get("Source", ""), float(d["Instructions Executed"] or 0), rs))
if only:
    items.sort(key=lambda x: x[1])
else:
    items.sort(reverse=True)
for v, off, ln, src, ie, rs in items[:top] if not only else items:
    r = ", ".join(f"{c}={n/v*100:.0f}%" for n, c in rs if n) if v else ""
    print(f"{v/tot*100:5.2f}% {off:06x} {ln:24s} ie={ie:.2e} {src.strip()[:70]}  [{r}]")
