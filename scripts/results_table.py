"""DESIGN.md results table from bench lines: python scripts/results_table.py profiles/<dir>
(bench_c<C>.json per config; DRAM traffic from profiles/traffic.json)."""
import json
import sys
from pathlib import Path

d = Path(sys.argv[1])
traffic = json.loads((Path(__file__).resolve().parents[1] / "profiles" / "traffic.json").read_text())
SHAPE = {1: "64, 1, f64", 2: "256, 16, f32", 3: "512, 64, f32", 4: "1024, 32, f32", 5: "4096, 1, f32"}
print("| cfg | n, B, dtype | images/s | ms/step | fwd / inv kernels (ms) | dominant kernel, HBM frac | step HBM frac | "
      "DRAM traffic / cube bytes (fwd / inv) | compact format images/s | e2e images/s (streamed / one step at a time) | "
      "cuFFT line images/s | oracle images/s |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for c in range(1, 6):
    f = d / f"bench_c{c}.json"
    if not f.exists():
        continue
    b = json.loads(f.read_text())
    r = b["roofline"]; k = r["kernel_ms"]; t = traffic.get(f"config{c}", {})
    fk, ik = ("tiny_fwd", "tiny_inv") if r.get("path") != "persistent" and "tiny_fwd" in t else ("fwd_main", "inv_main")
    cube = r["bytes_per_launch"]
    tr = "%.2f / %.2f" % (t[fk] / cube, t[ik] / cube) if fk in t and ik in t else "--"
    e = b.get("e2e") or {}
    es = "%.4g / %.4g" % ((e.get("streamed") or {}).get("value", float("nan")), (e.get("serial") or {}).get("value", float("nan")))
    cf = b.get("cufft_line") or {}; cp = b.get("compact_line") or {}; cb = b.get("cpu_baseline") or {}
    fwd = k.get("fwd_main", k.get("tiny_fwd", float("nan"))); inv = k.get("inv_main", k.get("tiny_inv", float("nan")))
    print("| %d | %s | %.5g | %.4f | %.3f / %.3f | %s %.3f | %.3f | %s | %s | %s | %s | %s (%s cores) |" % (
        c, SHAPE[c], b["value"], b["ms_per_step"], fwd, inv, r["kernel"], r["frac"], b["hbm_frac_step"], tr,
        ("%.5g" % cp["value"]) if cp else "--", es, ("%.4g" % cf["value"]) if cf else "--",
        ("%.3g" % cb["value"]) if cb else "--", cb.get("cores", "?")))
