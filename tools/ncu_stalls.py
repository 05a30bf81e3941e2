"""Hot instructions of one kernel in an ncu report: execution count, stall samples and the
dominant stall reasons per SASS line.
  python tools/ncu_stalls.py REP KERNEL_REGEX [first_line last_line] [--min 0.2]"""
import csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
pos = [a for a in sys.argv[3:] if a.lstrip("-").isdigit() and not a.startswith("--")]
rng = [int(x) for x in pos[:2]] if len(pos) >= 2 else None
mn = float(sys.argv[sys.argv.index("--min") + 1]) if "--min" in sys.argv else 0.2
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
hdr = rows[h]
data = []
for r in rows[h + 1:]:
    if "Source" in r and "Instructions Executed" in r:
        break  # next kernel
    if len(r) == len(hdr):
        data.append(r)
ie, src, st = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
sc = [i for i, c in enumerate(hdr) if c.startswith("stall_")]
tot = sum(int(r[st]) for r in data) or 1
agg = {hdr[i]: sum(float(r[i] or 0) for r in data) for i in sc}
print("total stall samples", tot, " top reasons:",
      ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for k, r in enumerate(data):
    if rng and not (rng[0] <= k <= rng[1]):
        continue
    s = int(r[st])
    if s >= tot * mn / 100:
        rs = sorted(((float(r[i] or 0), hdr[i][6:]) for i in sc), reverse=True)[:2]
        print(f"{k:5d} x{int(r[ie]):10d} {100*s/tot:5.2f}%  {r[src].strip()[:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in rs))
