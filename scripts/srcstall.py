"""Per-source-line stall breakdown from an ncu 'source --print-source cuda,sass' CSV (SASS rows)."""
import csv, gzip, sys, collections, re
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
want = sys.argv[3].split(',') if len(sys.argv) > 3 else ['stall_long_sb', 'stall_short_sb', 'stall_no_inst', 'stall_wait', 'stall_selected']
rows = list(csv.reader(gzip.open(path, 'rt') if path.endswith('.gz') else open(path)))
hdr = None; func = None; cur = None; src = ''; fname = ''
agg = collections.defaultdict(lambda: collections.Counter())
srcs = {}
for r in rows:
    if not r: continue
    if r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': func = r[1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None: continue
    if r[0].strip().isdigit() and r[1]:
        cur = (func, fname + ':' + r[0]); srcs[cur] = r[1].strip()[:80]; continue
    d = dict(zip(hdr, r))
    if not d.get('Address'): continue
    for k in hdr:
        if k.startswith('stall_') or k == 'Warp Stall Sampling (All Samples)':
            try: agg[cur][k] += int(d[k] or 0)
            except ValueError: pass
for f in sorted(set(k[0] for k in agg)):
    keys = [k for k in agg if k[0] == f]
    tot = sum(agg[k]['Warp Stall Sampling (All Samples)'] for k in keys) or 1
    print('==', f[:70], 'samples', tot)
    for w in want:
        wt = sum(agg[k][w] for k in keys)
        print(f'  -- {w}: {100*wt/tot:.1f}% of samples')
        for k in sorted(keys, key=lambda k: -agg[k][w])[:top]:
            if agg[k][w] == 0: break
            print(f'     {100*agg[k][w]/tot:5.1f}%  L{k[1]:>5} {srcs.get(k, "")}')
