#!/bin/bash
# C1 / C2 / C4 under builds that differ only in the fan-out threshold (dev tool)
for L in "$@"; do
  echo -n "$L C1(ms): "; MCSG_LIB=$PWD/$L python tools/configs.py --only c1 | python -c "
import sys,json
print(' '.join(str(round(1e3*json.loads(l).get('throughput_kernel_s', json.loads(l).get('kernel_s',0)),3)) for l in sys.stdin))"
  echo -n "$L C2: "; MCSG_LIB=$PWD/$L python bench.py --no-cpu-baseline --no-c4 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), 'G nodes/s', round(d['ms_per_step'],1), 'ms')"
  echo -n "$L C4: "; MCSG_LIB=$PWD/$L python tools/exp_c4.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['rate']/1e9,3), 'G nodes/s', round(d['kernel_s'],2), 's')"
done
