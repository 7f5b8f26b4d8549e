#!/bin/bash
# Full ncu capture of the undirected 64-bit kernel on a C4-like tree without a
# deadline: kernel replay first; application replay if that fails
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 120 python tools/prof_u64.py 2 40 0.5 > gpurun_out/u64s_plain.log 2>&1; cat gpurun_out/u64s_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mcs_search -c 1 -o gpurun_out/u64s_kr python tools/prof_u64.py 2 40 0.5 > gpurun_out/u64s_kr.log 2>&1
echo "kernel replay rc=$?"; tail -3 gpurun_out/u64s_kr.log
if [ ! -f gpurun_out/u64s_kr.ncu-rep ]; then
  timeout 1800 ncu --set full --replay-mode application --clock-control none --import-source on -k regex:mcs_search -c 1 -o gpurun_out/u64s_ar python tools/prof_u64.py 2 40 0.5 > gpurun_out/u64s_ar.log 2>&1
  echo "application replay rc=$?"; tail -3 gpurun_out/u64s_ar.log
fi
ls -la gpurun_out/*.ncu-rep
