#!/bin/bash
# Final: GPU suite, smoke, both bench arms, and the C3 capture for the directed kernel at 7 CTAs/SM
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin_gputest.log 2>&1; tail -3 gpurun_out/fin_gputest.log
python -c "import __graft_entry__ as E; E.smoke()" > gpurun_out/fin_smoke.log 2>&1; cat gpurun_out/fin_smoke.log
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mcs_search -c 1 -o gpurun_out/fin_c3 python tools/prof_c3.py > gpurun_out/fin_c3.log 2>&1
tail -c 300 gpurun_out/fin_bench.json
