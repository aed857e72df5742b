"""Per-source-line stall samples of one kernel: maps the SASS addresses of an ncu --page source
(sass) CSV to CUDA source lines with nvdisasm -g line info (development diagnostic).
usage: python tools/ncu_lines.py <report.ncu-rep> <kernel regex> <object.o> [top]"""
import csv, io, re, subprocess, sys, tempfile, os, glob
rep, kre, obj = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = glob.glob(d + "/*.cubin")[0]
txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                       "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
name = rows[0][1]
hdr, data = rows[1], rows[2:]
# find the function in the nvdisasm text whose mangled name appears in the kernel name
fun_start = None
lines = txt.split("\n")
for i, l in enumerate(lines):
    if l.startswith("//--------------------- .text.") and re.search(kre, l):
        fun_start = i
        break
cur, amap = None, {}
for l in lines[fun_start + 1:]:
    if l.startswith("//--------------------- .text"):
        break
    mm = re.search(r'//## File "(.*)", line (\d+)', l)
    if mm:
        cur = (os.path.basename(mm.group(1)), int(mm.group(2)))
        continue
    ma = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if ma and cur:
        amap[int(ma.group(1), 16)] = cur
ia = hdr.index("Address"); isamp = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
T = sum(int(r[isamp] or 0) for r in data); E = sum(int(r[iex] or 0) for r in data)
agg = {}
for r in data:
    k = amap.get(int(r[ia], 16) - base, ("?", 0))
    s, e = agg.get(k, (0, 0))
    agg[k] = (s + int(r[isamp] or 0), e + int(r[iex] or 0))
src = {}
for (f, ln) in agg:
    if f not in src and f != "?":
        p = glob.glob(f"paper_2501_06838_b200/csrc/{f}")
        src[f] = open(p[0]).read().split("\n") if p else []
print(name[:100])
for (f, ln), (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    code = src.get(f, [])[ln - 1].strip()[:70] if f in src and 0 < ln <= len(src[f]) else ""
    print(f"{f}:{ln:<5} samples {s / T:6.3f} inst {e / E:6.3f}  {code}")
