"""Executed FP32 work per kernel from an ncu capture (SURVEY.md §8(d) "% FP32 peak, executed"):
flops = 2 FFMA + 4 FFMA2 + FADD + 2 FADD2 + FMUL + 2 FMUL2 thread instructions (predicated on),
divided by the kernel's gpu__time_duration, against 148 SMs x 128 lanes x 2 x f (f the SM clock
ncu saw, sm__cycles_elapsed.avg.per_second, and the 1965 MHz max).  Also DRAM bytes per launch
(the bench's roofline `traffic`).  Writes JSON keyed by the bench's pass names.

  ncu --metrics <METRICS> --clock-control none --profile-from-start off -o rep python tools/profile_step.py
  python tools/ncu_fp32.py rep.ncu-rep profiles/r02/ncu_fp32.json
"""
import csv
import json
import subprocess
import sys

METRICS = ",".join([
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
])
PASS_OF = {"grav_pipe_kernel": "gravity", "GeoPass": "geometry", "list_kernel2": "corrections_extras", "CorExtPass": "corrections_extras",
           "AccPass": "accel_dudt"}
N_SM, LANES, F_MAX = 148, 128, 1965e6


def _num(v):
    return float(v.replace(",", "")) if v not in ("", "n/a") else 0.0


_SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
          "second": 1.0, "hz": 1.0, "khz": 1e3, "mhz": 1e6, "ghz": 1e9, "byte": 1.0, "kbyte": 1e3, "mbyte": 1e6,
          "gbyte": 1e9, "tbyte": 1e12}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    res = {}
    for d in data:
        name = d[col["Kernel Name"]]
        pas = next((p for k, p in PASS_OF.items() if k in name), None)
        if pas is None:
            continue
        t = _num(d[col["gpu__time_duration.sum"]]) * _SCALE[units[col["gpu__time_duration.sum"]].lower()]
        g = lambda m: _num(d[col["smsp__sass_thread_inst_executed_op_" + m + "_pred_on.sum"]])  # noqa: E731
        flops = 2 * g("ffma") + 4 * g("ffma2") + g("fadd") + 2 * g("fadd2") + g("fmul") + 2 * g("fmul2")
        f = _num(d[col["sm__cycles_elapsed.avg.per_second"]]) * _SCALE[units[col["sm__cycles_elapsed.avg.per_second"]].lower()]
        dram = sum(_num(d[col[m]]) * _SCALE[units[col[m]].lower()] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        if pas in res and res[pas]["ms"] >= t * 1e3:
            continue  # keep the dominant launch of the pass
        res[pas] = {"kernel": name[:120], "ms": t * 1e3, "executed_fp32_flop": flops,
                    "executed_tflops": flops / t / 1e12,
                    "frac_of_peak_at_ncu_clock": flops / t / (N_SM * LANES * 2 * f) if f else None,
                    "frac_of_peak_at_max_clock": flops / t / (N_SM * LANES * 2 * F_MAX),
                    "sm_clock_mhz": f / 1e6, "dram_bytes": dram,
                    "fma_pipe_pct": _num(d[col["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]]),
                    "issue_active_pct": _num(d[col["smsp__issue_active.avg.pct_of_peak_sustained_active"]])}
    json.dump({"source": rep, "note": "ncu, one substep of c4, --clock-control none (cold, serialised)",
               "passes": res}, open(out, "w"), indent=1)
    for k, v in res.items():
        print(f"{k:20s} {v['ms']:8.2f} ms  executed {v['executed_tflops']:6.2f} TFLOP/s  "
              f"{100 * v['frac_of_peak_at_max_clock']:5.1f}% of peak  DRAM {v['dram_bytes'] / 1e9:.2f} GB")


if __name__ == "__main__":
    if sys.argv[1] == "--metrics":
        print(METRICS)
    else:
        main(sys.argv[1], sys.argv[2])
