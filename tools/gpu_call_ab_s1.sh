#!/bin/bash
# A/B: the 64-bit policy's second class slot read from the level's stack copy
# (one class per lane in registers) at 7 and 8 CTAs/SM, against PEXT
# compaction alone; the full GPU suite on the in-tree build (s1_8)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s1_tests.log 2>&1; tail -3 gpurun_out/s1_tests.log
timeout 1500 python tools/ab.py ablibs/libmcsg_pext.so ablibs/libmcsg_s1_7.so ablibs/libmcsg_s1_8.so ablibs/libmcsg_s1_8h.so --reps 3 --only c2,c3,c4 > gpurun_out/ab_s1.jsonl 2>&1
cat gpurun_out/ab_s1.jsonl
# undirected 64-bit kernel, C4-like trees without a deadline (replay-safe): full ncu capture of the PEXT build
MCSG_LIB=$PWD/ablibs/libmcsg_pext.so timeout 300 python tools/prof_u64.py 8 40 0.5 > gpurun_out/u64_plain.log 2>&1; cat gpurun_out/u64_plain.log
MCSG_LIB=$PWD/ablibs/libmcsg_pext.so timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mcs_search -c 1 -o gpurun_out/u64_pext python tools/prof_u64.py 8 40 0.5 > gpurun_out/u64_ncu.log 2>&1; tail -2 gpurun_out/u64_ncu.log
