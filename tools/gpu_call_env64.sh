#!/bin/bash
# Host-side knobs of the 64-bit kernels re-checked on the final build: poll interval (C4, C3) and the directed nest slack (C3)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
L=paper_1908_06418_b200/libmcsg.so
for rep in 1 2; do
  timeout 300 python tools/ab.py $L --reps 1 --only c3,c4 | sed "s/^/default /" >> gpurun_out/env64.txt
  for pi in 256 512; do MCSG_DEBUG_POLL_INTERVAL=$pi timeout 300 python tools/ab.py $L --reps 1 --only c3,c4 | sed "s/^/poll$pi /" >> gpurun_out/env64.txt; done
  MCSG_DEBUG_COMPACT_SLACK=3 timeout 300 python tools/ab.py $L --reps 1 --only c3 | sed "s/^/slack3 /" >> gpurun_out/env64.txt
done
cat gpurun_out/env64.txt
