#!/bin/bash
# A/B: undirected 64-bit kernel at 9 CTAs/SM (56 registers, 64 B spill) against 8 (64 registers)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 python tools/ab.py ablibs/libmcsg_head3.so ablibs/libmcsg_u9.so --reps 3 --only c4 > gpurun_out/ab_u9.jsonl 2>&1
cat gpurun_out/ab_u9.jsonl
