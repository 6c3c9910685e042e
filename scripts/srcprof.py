"""Aggregate an ncu 'source --print-source cuda,sass' CSV by CUDA source line."""
import csv, gzip, sys, collections
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fh = gzip.open(path, 'rt') if path.endswith('.gz') else open(path)
rows = list(csv.reader(fh))
cur_file = cur_func = None
agg = collections.defaultdict(lambda: [0, 0, ''])   # (func, file, line) -> [samples, inst, src]
hdr = None
line_no = None
line_src = ''
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name':
        cur_func = r[1]; continue
    if r[0] == 'Line No':
        hdr = r; continue
    if hdr is None:
        continue
    # rows: either a CUDA source line (Line No set) or SASS (Address set)
    d = dict(zip(hdr, r))
    if r[0] and r[0].strip().isdigit():
        line_no = int(r[0]); line_src = r[1].strip()
        continue
    try:
        samp = int(r[hdr.index('Warp Stall Sampling (All Samples)')])
        inst = int(r[hdr.index('Instructions Executed')])
    except Exception:
        continue
    key = (cur_func, cur_file, line_no)
    a = agg[key]; a[0] += samp; a[1] += inst; a[2] = line_src
funcs = collections.defaultdict(lambda: [0, 0])
for (f, fl, ln), (s, i, src) in agg.items():
    funcs[f][0] += s; funcs[f][1] += i
for f, (s, i) in funcs.items():
    print(f"== {f[:70]}  samples={s} warp-inst={i}")
    items = sorted(((v[0], v[1], fl, ln, v[2]) for (ff, fl, ln), v in agg.items() if ff == f), reverse=True)
    for s2, i2, fl, ln, src in items[:top]:
        print(f"  {100.0*s2/max(s,1):5.1f}%smp {100.0*i2/max(i,1):5.1f}%ins  {fl}:{ln}  {src[:90]}")
