#!/bin/bash
# A/B: directed 64-bit kernel with compacted subtrees in shared memory only
# (no HBM fallback; the s0 room bound makes most fit) against the shipped build
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 python tools/ab.py ablibs/libmcsg_head4.so ablibs/libmcsg_dsm.so --reps 3 --only c3 > gpurun_out/ab_dsm.jsonl 2>&1
cat gpurun_out/ab_dsm.jsonl
