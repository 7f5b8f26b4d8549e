#!/bin/bash
# Ring capacity re-check (host knob): 4096 / 8192 / default on C2, C5, C4
mkdir -p gpurun_out
L=paper_1908_06418_b200/libmcsg.so
for rep in 1 2; do
  timeout 300 python tools/ab.py $L --reps 1 --only c2,c5,c4 | sed "s/^/default /" >> gpurun_out/ringcap.txt
  for rc in 4096 8192; do MCSG_DEBUG_RING_CAP=$rc timeout 300 python tools/ab.py $L --reps 1 --only c2,c5,c4 | sed "s/^/ring$rc /" >> gpurun_out/ringcap.txt; done
done
cat gpurun_out/ringcap.txt
