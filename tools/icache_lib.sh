#!/bin/bash
# ICC counters + issue on one C3 launch for each library given (dev tool)
M=sm__icc_requests.sum,sm__icc_requests_lookup_miss.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for L in "$@"; do
  MCSG_LIB=$PWD/$L ncu --metrics $M --clock-control none -k regex:mcs_search -c 1 --csv python tools/prof_c3.py 2>/dev/null | grep -E '^"[0-9]' | awk -F'","' -v L=$L '{printf "%s %s %s\n", L, $(NF-2), $NF}'
done
