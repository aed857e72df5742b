"""profiles/ncu_traffic.json from an ncu --set full report of the bench workload:
dram bytes (read + write) per launch of each render kernel. usage: make_traffic.py rep workload"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, wl = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
res = {}
for r in data:
    name = r[ix["Kernel Name"]]
    k = "render_fwd" if "k_render_fwd" in name else "render_bwd" if "k_render_bwd" in name else None
    if not k:
        continue
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        u = units[ix[m]]
        tot += float(r[ix[m]].replace(",", "")) * mult.get(u, 1)
    res[k] = {"dram_bytes_per_launch": tot, "source": rep,
              "duration_ns_under_ncu": float(r[ix["gpu__time_duration.sum"]].replace(",", ""))
              * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
                 "second": 1e9, "s": 1e9}.get(
                  units[ix["gpu__time_duration.sum"]], 1)}
p = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
d = json.loads(p.read_text()) if p.exists() else {}
d[wl] = res
p.parent.mkdir(exist_ok=True)
p.write_text(json.dumps(d, indent=1))
print(json.dumps(d, indent=1))
