"""Summarise an ncu --set full report of the search kernel (dev tool)."""
import csv, json, subprocess, sys
rep, nodes = sys.argv[1], float(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(raw))
hdr, units, vals = r[0], r[1], r[2]
d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
def f(k):
    try: return float(d[k].replace(',', ''))
    except Exception: return None
keys = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.per_cycle_active',
        'smsp__warps_eligible.avg.per_cycle_active', 'launch__registers_per_thread',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__cycles_elapsed.avg']
out = {k: f(k) for k in keys}
out['unit'] = {k: u.get(k) for k in keys}
pipes = {k: f(k) for k in hdr if k.startswith('sm__inst_executed_pipe_') and k.endswith('.avg.pct_of_peak_sustained_active')}
stalls = {k.replace('smsp__pcsamp_warps_issue_stalled_', ''): f(k) for k in hdr
          if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued')}
tot = sum(v for v in stalls.values() if v)
out['warp_inst_per_node'] = out['smsp__inst_executed.sum'] / nodes
SCALE = {'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
def nbytes(k):  # each metric carries its own unit
    return (out[k] or 0.0) * SCALE.get(out['unit'].get(k), 1.0)
out['dram_bytes_per_launch'] = nbytes('dram__bytes_read.sum') + nbytes('dram__bytes_write.sum')
out['nodes_per_launch'] = nodes
out['stall_pct'] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0)) if v}
out['pipes_pct'] = {k.replace('sm__inst_executed_pipe_', '').replace('.avg.pct_of_peak_sustained_active', ''): v
                    for k, v in sorted(pipes.items(), key=lambda x: -(x[1] or 0)) if v}
# the machine code the profile belongs to: the SHA-1 of the profiled kernel's
# SASS in the built library (bench.py recomputes it and reports
# profile_matches_kernel); run this against the same libmcsg.so that was profiled
import os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_key import kernel_sass_sha1, U32_THROUGHPUT  # noqa: E402
kernel = sys.argv[3] if len(sys.argv) > 3 else U32_THROUGHPUT
lib = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1908_06418_b200", "libmcsg.so")
out['kernel'] = kernel
out['kernel_sass_sha1'] = kernel_sass_sha1(lib, kernel)
print(json.dumps(out, indent=1))
