#!/bin/bash
# The GPU parity suite under the library's development switches (every mode must stay word-for-word equal to the
# oracle): one pytest run per mode, results in gpurun_out/modes_*.log.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # name, env assignments...
  name=$1; shift
  env "$@" timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/modes_$name.log 2>&1; echo "rc=$? env: $*" >> gpurun_out/modes_$name.log
}
run ntt_fused1 SECPE_NTT_FUSED=1
run ntt_fused3 SECPE_NTT_FUSED=3
run ks_fuse0 SECPE_KS_FUSE=0
run no_fpb SECPE_NO_FPB=1
run no_tc SECPE_NO_TC=1
run streams1_nograph SECPE_STREAMS=1 SECPE_GRAPH=0
for f in gpurun_out/modes_*.log; do echo "$f: $(tail -2 $f | tr '\n' ' ')"; done > gpurun_out/modes_summary.txt
