#!/bin/bash
# A/B: directed 64-bit kernel at 7 CTAs/SM (72 registers, 16 B stack; more shared memory per warp for nests) against 8
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 python tools/ab.py ablibs/libmcsg_head5.so ablibs/libmcsg_d7.so --reps 3 --only c3 > gpurun_out/ab_d7.jsonl 2>&1
cat gpurun_out/ab_d7.jsonl
