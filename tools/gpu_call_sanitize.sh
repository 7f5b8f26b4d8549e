#!/bin/bash
# compute-sanitizer on the shipped kernels (incl. the undirected 64-bit kernel's PEXT nests and HiSlot)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/san2
for tool in racecheck synccheck memcheck; do
  MCSG_DEBUG_POLL_INTERVAL=16 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/race_drive.py all 64 > gpurun_out/san2/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san2/rc.txt
done
tail -4 gpurun_out/san2/san_*.log; cat gpurun_out/san2/rc.txt
