for rep in 1 2; do for PI in 256 384 512; do echo "interval $PI"; MCSG_DEBUG_POLL_INTERVAL=$PI python tools/ab.py paper_1908_06418_b200/libmcsg.so --reps 1 --only c2,c3,c4; MCSG_DEBUG_POLL_INTERVAL=$PI python tools/configs.py --only c5,c1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d.get('config')=='C5': print('c5', round(d['kernel_s'],3), round(d['nodes']/1e9,2))
    if d.get('config')=='C1-batch': print('c1batch', round(d['kernel_s']*1e3,3))"; done; done
