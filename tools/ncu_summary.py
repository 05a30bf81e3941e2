"""Summarise an ncu --set full report (raw page) for the pair kernels."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ['Kernel Name', 'gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'smsp__inst_executed.sum',
        'smsp__sass_thread_inst_executed_op_ffma_pred_on.sum', 'smsp__sass_thread_inst_executed_op_fadd_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_fmul_pred_on.sum',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'smsp__average_warp_latency_issue_stalled_barrier.ratio', 'smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio',
        'smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio', 'smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio',
        'smsp__average_warp_latency_issue_stalled_wait.ratio', 'smsp__average_warp_latency_issue_stalled_mio_throttle.ratio',
        'smsp__average_warp_latency_issue_stalled_not_selected.ratio', 'smsp__average_warp_latency_issue_stalled_selected.ratio']
for d in data:
    print('----')
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:75s} {d[i][:70]} {units[i]}")
    # executed fp32 flops
    try:
        ff = float(d[hdr.index('smsp__sass_thread_inst_executed_op_ffma_pred_on.sum')].replace(',', ''))
        fa = float(d[hdr.index('smsp__sass_thread_inst_executed_op_fadd_pred_on.sum')].replace(',', ''))
        fm = float(d[hdr.index('smsp__sass_thread_inst_executed_op_fmul_pred_on.sum')].replace(',', ''))
        t = float(d[hdr.index('gpu__time_duration.sum')].replace(',', ''))
        tu = units[hdr.index('gpu__time_duration.sum')]
        t = t * {'nsecond': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3, 'second': 1}[tu]
        print(f"  executed FP32 TFLOP/s (2 FFMA + FADD + FMUL) = {(2*ff+fa+fm)/t/1e12:.2f}")
    except Exception as e:
        print('  (no flop counters)', e)
