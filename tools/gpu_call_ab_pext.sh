#!/bin/bash
# A/B: PEXT compaction (HD §7-4 move masks) against the previous build; the
# compaction suite on the new build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compaction.py tests/test_gpu_golden.py -q -x > gpurun_out/ab_tests.log 2>&1; tail -3 gpurun_out/ab_tests.log
timeout 900 python tools/ab.py ablibs/libmcsg_base.so ablibs/libmcsg_pext.so --reps 3 --only c2,c3,c4 > gpurun_out/ab_pext.jsonl 2>&1
MCSG_DEBUG_COMPACT_SLACK=2 timeout 300 python tools/ab.py ablibs/libmcsg_pext.so --reps 2 --only c4 > gpurun_out/ab_pext_slack2.jsonl 2>&1
cat gpurun_out/ab_pext.jsonl gpurun_out/ab_pext_slack2.jsonl
