#!/bin/bash
# A/B node rates of two builds of libmcsg.so, interleaved (dev tool):
#   tools/ab.sh build/libA.so build/libB.so [rounds]
A=$1; B=$2; R=${3:-2}
for i in $(seq $R); do
  for L in $A $B; do
    echo -n "$L C2 "; MCSG_LIB=$PWD/$L python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), 'G nodes/s', round(d['ms_per_step'],1), 'ms')"
    echo -n "$L C4 "; MCSG_LIB=$PWD/$L python tools/exp_c4.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['rate']/1e9,3), 'G nodes/s', round(d['kernel_s'],2), 's')"
  done
done
