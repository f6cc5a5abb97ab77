#!/bin/bash
# headline step under the library's environment switches, same box, alternating with the default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
one() {
  env "$@" timeout 600 python bench.py --no-micro --no-cpu-baseline --steps 10 --warmup 3 2> /dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$*', round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> gpurun_out/env_sweep.txt 2>&1
}
for r in 1 2; do
  one X=0
  one SECPE_NTT_FUSED=1
  one SECPE_NTT_FUSED_ROWS=256
  one SECPE_STREAMS=3
  one SECPE_KS_FUSE=0
done
