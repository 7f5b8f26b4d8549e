#!/bin/bash
# A/B: 32-bit kernel at 9 CTAs/SM (56 registers, no spill) and 10 (48, small spill) against 8 (64)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1500 python tools/ab.py ablibs/libmcsg_head2.so ablibs/libmcsg_c9.so ablibs/libmcsg_c10.so --reps 3 --only c2,c5,c4 > gpurun_out/ab_c9.jsonl 2>&1
cat gpurun_out/ab_c9.jsonl
