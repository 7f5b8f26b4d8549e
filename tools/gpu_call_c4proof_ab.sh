#!/bin/bash
# One call: the C4 proof's remaining pieces on the box's host cores (15
# workers, background) while the GPU runs the PEXT A/B; then wait for the proof
mkdir -p gpurun_out
cp tests/golden/c4_pieces.jsonl gpurun_out/c4_pieces_box.jsonl
nice -n 5 python tools/c4_split_proof.py 12 15 gpurun_out/c4_pieces_box.jsonl > gpurun_out/c4_box.log 2>&1 &
PROOF=$!
bash tools/gpu_call_ab_pext.sh
for i in $(seq 1 200); do kill -0 $PROOF 2>/dev/null || break; sleep 10; done
kill $PROOF 2>/dev/null
wc -l gpurun_out/c4_pieces_box.jsonl; tail -2 gpurun_out/c4_box.log
