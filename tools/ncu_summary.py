"""Summarise an ncu --set full report (raw page) into the metrics we track."""
import csv
import io
import json
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_op_tmem_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__grid_size',
        'smsp__inst_executed.avg.per_cycle_active', 'lts__t_bytes.sum',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__average_warp_latency_issue_stalled_long_scoreboard', 'sm__cycles_elapsed.avg.per_second']


def summarise(path):
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[2:]:
        d = {'kernel': r[idx['Kernel Name']][:120]}
        for w in WANT:
            if w in idx:
                d[w] = f"{r[idx[w]]} {units[idx[w]]}".strip()
        out.append(d)
    return out


if __name__ == '__main__':
    res = {p: summarise(p) for p in sys.argv[1:]}
    print(json.dumps(res, indent=1))
