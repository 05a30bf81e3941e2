"""Per-instruction execution counts / stall samples of one kernel from an ncu report."""
import csv, subprocess, sys
rep, pat = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blocks = []; cur = None
for ln in raw.split('\n'):
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    if pat not in b[0]:
        continue
    rows = list(csv.reader(b[1:])); hdr = rows[0]; data = [r for r in rows[1:] if len(r) == len(hdr)]
    ie = hdr.index('Instructions Executed'); src = hdr.index('Source'); st = hdr.index('Warp Stall Sampling (All Samples)')
    tot = sum(int(r[ie]) for r in data); totst = sum(int(r[st]) for r in data) or 1
    print(b[0][:100], 'total warp inst %.3e' % tot)
    # regions: consecutive instructions with the same execution count
    reg = []
    for i, r in enumerate(data):
        n = int(r[ie])
        if reg and reg[-1][2] == n:
            reg[-1][1] = i; reg[-1][3] += int(r[st])
        else:
            reg.append([i, i, n, int(r[st]), r[src].strip()[:50]])
    for a, z, n, s, first in reg:
        inst = n * (z - a + 1)
        if inst >= tot * thr / 100 or s >= totst * thr / 100:
            print(f"[{a:4d}-{z:4d}] len {z-a+1:3d} x{n:11d} = {100*inst/tot:5.1f}% inst, {100*s/totst:5.1f}% stall  {first}")
