#!/bin/bash
# base-conversion tiles per CTA (wave quantisation of the 512-tile polynomials over 296 CTA slots), same box, alternating
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3; do
for T in 16 30 26 22; do
  SECPE_TC_TPC=$T timeout 600 python bench.py --no-micro --no-cpu-baseline --steps 10 --warmup 3 2> /dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('TPC=$T', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> gpurun_out/tpc_sweep.txt 2>&1
done
done
