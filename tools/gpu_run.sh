cd $GRAFT_REPO_ROOT
SECPE_TC_V=2 timeout 900 python -m pytest tests -q -m gpu -x -k "fused_keyswitch or ks_config or small_ring or config5_full or rotate" > gpurun_out/t19.log 2>&1; echo rc=$? >> gpurun_out/t19.log
for i in 1 2 3; do for cfg in "1 16" "2 16" "2 8" "2 32"; do set -- $cfg
ms=$(SECPE_TC_V=$1 SECPE_TC2_TPC=$2 SECPE_BATCH=16 timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.')
echo "v=$1 tpc=$2 $ms" >> gpurun_out/ab19.log
done; done
for v in 1 2; do SECPE_TC_V=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bconv -s 10 -c 2 python tools/relin_bench.py 2>&1 | grep -E "bconv|duration" >> gpurun_out/ab19.log; done
