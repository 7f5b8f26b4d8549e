set -x
export PATH=/usr/local/cuda/bin:$PATH
ncu --set full --clock-control none --import-source on -k regex:mcs_search -c 1 -o gpurun_out/r2_c3 python tools/prof_c3.py > gpurun_out/r2_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mcs_search -s 3 -c 1 -o gpurun_out/r2_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --configs '' --no-c4 > gpurun_out/r2_c2.log 2>&1
for tool in racecheck synccheck memcheck; do
  MCSG_DEBUG_POLL_INTERVAL=16 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/race_drive.py all 64 > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_rc.txt
done
tail -5 gpurun_out/san_*.log
cat gpurun_out/san_rc.txt
