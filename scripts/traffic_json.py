"""Fold ncu traffic captures (scripts/gpu.sh traffic) into profiles/traffic.json:
{"config<C>": {"fwd_main": bytes, "inv_main": bytes, ...}} -- dram__bytes_read.sum +
dram__bytes_write.sum per launch, averaged over the captured launches of each kernel."""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

out = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
data = json.loads(out.read_text()) if out.exists() else {}
for arg in sys.argv[1:]:                       # cfg=path.csv
    cfg, path = arg.split("=", 1)
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if "Metric Name" in r)
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    idi = hdr.index("ID")
    per = defaultdict(dict)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= vi:
            continue
        name = "fwd_main" if "fwd_main" in r[ki] else "inv_main" if "inv_main" in r[ki] else \
            "tiny_fwd" if "tiny_fwd" in r[ki] else "tiny_inv" if "tiny_inv" in r[ki] else None
        if name is None:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        per[(name, r[idi])][r[mi]] = v
    agg = defaultdict(list)
    for (name, _), m in per.items():
        agg[name].append((m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0),
                          m.get("gpu__time_duration.sum", 0)))
    entry = data.setdefault(f"config{cfg}", {})
    for name, vals in agg.items():
        entry[name] = sum(v[0] for v in vals) / len(vals)
        entry[name + "_ms_ncu"] = sum(v[1] for v in vals) / len(vals)
data["source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                  "--clock-control none (scripts/gpu.sh traffic), bytes per launch, final round-2 code")
out.write_text(json.dumps(data, indent=1) + "\n")
print(json.dumps(data, indent=1))
