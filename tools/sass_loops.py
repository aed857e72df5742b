"""Per-loop breakdown of an ncu source page (--page source --csv --print-source sass):
samples, executed instructions, FP32x2 / MUFU counts per loop body (development diagnostic).
usage: python tools/sass_loops.py source.csv"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
ith = hdr.index("Avg. Threads Executed")
base = int(data[0][ia], 16)
ins = [(int(r[ia], 16) - base, r[isrc].strip(), int(r[isamp] or 0), int(r[iex] or 0),
        float(r[ith] or 0)) for r in data]
tot_s = sum(x[2] for x in ins)
tot_e = sum(x[3] for x in ins)
print("total samples", tot_s, "inst", tot_e)
idx = {a: i for i, (a, *_) in enumerate(ins)}
for i, (a, s, *_) in enumerate(ins):
    if "BRA" not in s:
        continue
    m = re.search(r"(0x[0-9a-f]+)", s)
    if not m:
        continue
    t = int(m.group(1), 16) - base
    if t < a and t in idx:
        body = ins[idx[t]:i + 1]
        if len(body) > 400:
            continue
        S = sum(x[2] for x in body)
        E = sum(x[3] for x in body)
        fp2 = sum(x[3] for x in body if re.search(r"F(FMA|MUL|ADD)2", x[1]))
        mufu = sum(x[3] for x in body if "MUFU" in x[1])
        print(f"loop {hex(t)}-{hex(a)} n={len(body)} samples {S / tot_s:.1%} inst {E / tot_e:.1%} "
              f"fp2 {fp2:.3e} mufu {mufu:.3e} iters {ins[idx[t]][3]:.3e}")
fp2 = sum(x[3] for x in ins if re.search(r"F(FMA|MUL|ADD)2", x[1]))
print("all fp2 %.3e mufu %.3e" % (fp2, sum(x[3] for x in ins if "MUFU" in x[1])))
