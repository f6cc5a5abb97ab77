cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -k "fused_keyswitch or ks_config or small_ring or config5_full or rotate or digit_counts" > gpurun_out/t22.log 2>&1; echo rc=$? >> gpurun_out/t22.log
for i in 1 2 3; do for lib in libsecpe.so libsecpe_dpb1.so libsecpe_pb2.so; do
ms=$(SECPE_LIB=paper_2502_00847_b200/$lib SECPE_BATCH=16 timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.')
echo "$lib $ms" >> gpurun_out/ab22.log
done; done
