#!/bin/bash
# Session validation of the shipped build: GPU suite, smoke, both bench arms,
# profiles re-captured for the shipped SASS, nest slack re-check (C4)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
bash tools/gpu_call_r2_validate.sh
for sl in 2 4; do MCSG_DEBUG_COMPACT_SLACK=$sl timeout 300 python tools/ab.py paper_1908_06418_b200/libmcsg.so --reps 2 --only c4 | sed "s/^/slack$sl /" >> gpurun_out/slack.txt 2>&1; done
cat gpurun_out/slack.txt
