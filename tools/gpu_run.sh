cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -k "fused_keyswitch or ks_config or small_ring or config5_full" > gpurun_out/t20.log 2>&1; echo rc=$? >> gpurun_out/t20.log
for i in 1 2 3; do for lib in libsecpe.so libsecpe_prev.so; do
ms=$(SECPE_LIB=paper_2502_00847_b200/$lib SECPE_BATCH=16 timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.')
echo "$lib $ms" >> gpurun_out/ab20.log
done; done
for lib in libsecpe.so libsecpe_prev.so; do SECPE_LIB=paper_2502_00847_b200/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ntt_ks_inner -s 20 -c 1 python tools/relin_bench.py 2>&1 | grep -E "duration" >> gpurun_out/ab20.log; done
