cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -q -m gpu -x -k "ks_config or small_ring or config5 or digit_counts or other_ring" > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log
for i in 1 2 3; do
for cfg in "1 libsecpe.so" "1 libsecpe_cpb1.so" "0 libsecpe.so"; do set -- $cfg
ms=$(SECPE_LIB=paper_2502_00847_b200/$2 SECPE_KS_FUSE=$1 SECPE_BATCH=16 timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.')
echo "fuse=$1 $2 $ms" >> gpurun_out/ab11.log
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ntt_ks_inner -s 20 -c 1 python tools/relin_bench.py > gpurun_out/ncu_ksi11.log 2>&1
