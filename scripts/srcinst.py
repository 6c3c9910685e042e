"""Per-source-line executed warp instructions from an ncu source CSV (scripts/gpu.sh prof):
   python scripts/srcinst.py <source.csv.gz> [kernel-substring] [top]"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = csv.reader(gzip.open(path, "rt") if path.endswith(".gz") else open(path))
fname = func = None
agg = collections.defaultdict(collections.Counter)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No" or want not in (func or ""):
        continue
    if r[0].strip().isdigit() and r[2] == "-":      # source row: aggregated over its SASS
        key = (fname, int(r[0]), r[1].strip()[:80])
        agg[func][key] += int(r[7] or 0)
for f, c in agg.items():
    tot = sum(c.values())
    print(f"== {f}: {tot / 1e6:.1f} M warp instructions")
    for (fn, ln, src), v in c.most_common(top):
        print(f"  {100 * v / tot:5.1f}%  {fn}:{ln}  {src}")
