#!/bin/bash
# Poll interval re-check at 9 CTAs/SM (32-bit kernel): 256 / 384 (default) / 512 on C2 and C5
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for rep in 1 2; do for pi in 256 384 512; do MCSG_DEBUG_POLL_INTERVAL=$pi timeout 300 python tools/ab.py paper_1908_06418_b200/libmcsg.so --reps 1 --only c2,c5 | sed "s/^/poll$pi /" >> gpurun_out/poll9.txt 2>&1; done; done
cat gpurun_out/poll9.txt
