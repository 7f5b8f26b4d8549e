#!/bin/bash
# Round-2 final captures for profiles/ (one B200; the kernel SASS these stamp is the shipped one)
set -x
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:mcs_search -s 3 -c 1 -o gpurun_out/r2f_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --configs '' > gpurun_out/r2f_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --configs '' > gpurun_out/r2f_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mcs_search -c 1 -o gpurun_out/r2f_c3 python tools/prof_c3.py > gpurun_out/r2f_c3.log 2>&1
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,sm__icc_requests.sum,sm__icc_requests_lookup_miss.sum,smsp__warp_issue_stalled_no_instruction_per_warp_active.pct --clock-control none -k regex:mcs_search -c 1 --csv python tools/prof_c4.py 2.0 > gpurun_out/r2f_c4.csv 2>&1
python - <<'PY' > gpurun_out/c4_witness.json
import json, sys
sys.path.insert(0, ".")
import paper_1908_06418_b200 as M
g, h = M.random_graph(45, 0.5, 45000), M.random_graph(45, 0.5, 45001)
r = M.solve(g, h, M.SolveConfig(mode=M.MODE_THROUGHPUT, budget_seconds=120))
print(json.dumps({"status": r.status.name, "size": r.size, "witness": [list(p) for p in r.best],
                  "kernel_s": r.stats.kernel_seconds, "nodes": r.stats.recursions}))
PY
cat gpurun_out/c4_witness.json
