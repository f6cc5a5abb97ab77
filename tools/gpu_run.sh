cd $GRAFT_REPO_ROOT
run() { ms=$(env "$@" SECPE_BATCH=16 timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.'); echo "$* $ms" >> gpurun_out/ab24.log; }
for i in 1 2 3; do
run SECPE_TC_TPC=16
run SECPE_TC_TPC=16 SECPE_LIB=paper_2502_00847_b200/libsecpe_wpi.so
run SECPE_TC_TPC=32
run SECPE_TC_TPC=64
done
