#!/bin/bash
# GPU suite, smoke and the bench (both arms) on the current build
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/lean_gputest.log 2>&1; tail -3 gpurun_out/lean_gputest.log
python -c "import __graft_entry__ as E; E.smoke()" > gpurun_out/lean_smoke.log 2>&1; cat gpurun_out/lean_smoke.log
timeout 900 python bench.py > gpurun_out/lean_bench.json 2> gpurun_out/lean_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/lean_bench_ref.json 2> gpurun_out/lean_bench_ref.err
tail -c 300 gpurun_out/lean_bench.json
