#!/bin/bash
# Round-2 end-of-session validation on one B200: the GPU suite, smoke, both
# bench arms, and the profiles for the shipped SASS (tools/gpu_call_r2_final.sh)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/val_gputest.log 2>&1; tail -3 gpurun_out/val_gputest.log
python -c "import __graft_entry__ as E; E.smoke()" > gpurun_out/val_smoke.log 2>&1; cat gpurun_out/val_smoke.log
timeout 900 python bench.py > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/val_bench_ref.json 2> gpurun_out/val_bench_ref.err
bash tools/gpu_call_r2_final.sh > gpurun_out/val_final.log 2>&1
bash tools/icache_lib.sh paper_1908_06418_b200/libmcsg.so > gpurun_out/val_icc.txt 2>&1
tail -c 400 gpurun_out/val_bench.json; tail -c 400 gpurun_out/val_bench_ref.json
