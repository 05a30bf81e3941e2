"""Instruction / stall-sample breakdown by basic-block-like regions of one kernel in an ncu report.
  python tools/ncu_regions.py report.ncu-rep kernel_regex [threshold_pct] [name_substring]"""
import csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
sub = sys.argv[4] if len(sys.argv) > 4 else ""
blocks, cur = [], None
for ln in raw.splitlines():
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
blk = [b for b in blocks if sub in b[0]][0]
print(blk[0][:120])
rows = list(csv.reader(blk))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
cols = [c for c in hdr if c.startswith('stall_') and 'Not Issued' not in c]
ci = [hdr.index(c) for c in cols]
ie = hdr.index('Instructions Executed')
reg = []
for i, r in enumerate(data):
    n = int(r[ie]); st = [int(r[k]) for k in ci]
    if reg and reg[-1][2] == n:
        reg[-1][1] = i; reg[-1][3] = [x + y for x, y in zip(reg[-1][3], st)]
    else:
        reg.append([i, i, n, st, r[1].strip()[:38]])
tot = sum(sum(x[3]) for x in reg) or 1
ti = sum(x[2] * (x[1] - x[0] + 1) for x in reg) or 1
print(f"total warp inst {ti:.3e}, stall samples {tot}")
for a, b, n, st, src in reg:
    s = sum(st)
    if s > tot * thr / 100 or n * (b - a + 1) > ti * thr / 100:
        top = sorted(zip(cols, st), key=lambda x: -x[1])[:3]
        print(f"[{a:4d}-{b:4d}] x{n:10d} inst {100*n*(b-a+1)/ti:5.1f}% stall {100*s/tot:5.1f}% {src:38s}",
              ' '.join(f"{k[6:]}={100*v/tot:.1f}" for k, v in top))
