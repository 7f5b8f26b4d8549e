#!/bin/bash
# 64-bit kernel builds: C3 batch and C4 (dev tool)
for i in 1 2; do for L in "$@"; do
  echo -n "$L C3: "; MCSG_LIB=$PWD/$L python tools/exp_c3.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['c3_s'],3), 's', round(d['c3_rate'],2))"
  echo -n "$L C4: "; MCSG_LIB=$PWD/$L python tools/exp_c4.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['kernel_s'],2), 's', round(d['rate']/1e9,3))"
done; done
