#!/bin/bash
# Instruction-cache evidence for the 64-bit kernel (dev tool): ICC (L1.5 I$)
# request/miss counters and issue activity on one C3 launch with and without
# compacted subtrees, next to the 32-bit kernel on C2 pairs.
M=sm__icc_requests.sum,sm__icc_requests_lookup_hit.sum,sm__icc_requests_lookup_miss.sum,sm__icc_requests_lookup_miss_tag_miss.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__warp_issue_stalled_no_instruction_per_warp_active.pct,smsp__warp_issue_stalled_branch_resolving_per_warp_active.pct
mkdir -p gpurun_out
ncu --metrics $M --clock-control none -k regex:mcs_search -c 1 --csv python tools/prof_c3.py > gpurun_out/icc_c3.csv 2>&1
MCSG_DEBUG_NO_COMPACT=1 ncu --metrics $M --clock-control none -k regex:mcs_search -c 1 --csv python tools/prof_c3.py > gpurun_out/icc_c3_nocompact.csv 2>&1
ncu --metrics $M --clock-control none -k regex:mcs_search -c 1 --csv python tools/prof_c2.py 30 > gpurun_out/icc_c2.csv 2>&1
