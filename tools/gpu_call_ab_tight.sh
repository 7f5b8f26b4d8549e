#!/bin/bash
# A/B: nest stack bound from the level's Σ min (s0) instead of m; compaction
# and golden suites on the new build (in-tree)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compaction.py tests/test_gpu_golden.py tests/test_gpu_robustness.py -q -x > gpurun_out/tight_tests.log 2>&1; tail -3 gpurun_out/tight_tests.log
timeout 1200 python tools/ab.py ablibs/libmcsg_head.so ablibs/libmcsg_tight.so --reps 3 --only c3,c4 > gpurun_out/ab_tight.jsonl 2>&1
cat gpurun_out/ab_tight.jsonl
