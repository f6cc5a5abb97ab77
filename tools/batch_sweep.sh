#!/bin/bash
# headline step vs ciphertexts per step (same box, alternating): bench.py --batch B, no micro rows
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do
for B in 16 32 24 48; do
  timeout 600 python bench.py --batch $B --no-micro --no-cpu-baseline --steps 8 --warmup 3 2> /dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('B=$B', round(d['value']), round(d['ms_per_step'],2), round(d['e2e']['value']), d['roofline']['frac'], d['clocks']['sm_mhz'])" >> gpurun_out/batch_sweep.txt 2>&1
done
done
