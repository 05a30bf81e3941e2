"""Per-pass dominant-kernel DRAM traffic and counters from an ncu --set full report -> JSON
(read by bench.py for the roofline line's `traffic`).

  python tools/make_traffic.py gpurun_out/prof_full.ncu-rep profiles/r01/ncu_traffic.json
"""
import csv, json, subprocess, sys

PASS_OF = [("grav_pipe_kernel", "gravity"), ("grav_warp_kernel", "gravity"), ("grav_sym_kernel", "gravity"),
           ("GeoPass", "geometry"), ("list_kernel2", "corrections_extras"), ("AccPass", "accel_dudt")]
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
col = lambda d, k: d[hdr.index(k)]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "second": 1}
num = lambda d, k: float(col(d, k).replace(",", "")) * scale.get(units[hdr.index(k)], 1)
res = {}
for d in data:
    name = col(d, "Kernel Name")
    ps = next((p for key, p in PASS_OF if key in name), None)
    if ps is None:
        continue
    t = num(d, "gpu__time_duration.sum")
    if ps in res and res[ps]["duration_s"] >= t:
        continue
    res[ps] = {"kernel": name, "duration_s": t,
               "dram_bytes": num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum"),
               "fma_pipe_pct": float(col(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active")),
               "issue_active_pct": float(col(d, "smsp__issue_active.avg.pct_of_peak_sustained_active")),
               "warps_active_pct": float(col(d, "sm__warps_active.avg.pct_of_peak_sustained_active")),
               "warp_inst": float(col(d, "smsp__inst_executed.sum").replace(",", ""))}
json.dump({"source": f"ncu --set full --clock-control none, one c4 (2x256^3) substep (tools/profile_step.py): {rep}",
           "kernels": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
