#!/bin/bash
# C5 (10,000 pairs) time and node count under two builds, interleaved (dev tool)
for i in 1 2; do for L in "$@"; do echo -n "$L "; MCSG_LIB=$PWD/$L python tools/configs.py --only c5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['kernel_s'],3), 's', round(d['nodes']/1e9,2), 'G nodes')"; done; done
