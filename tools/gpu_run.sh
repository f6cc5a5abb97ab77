cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -k "fused_keyswitch or digit_counts or ks_config or small_ring or config5 or rotate or toy or other_ring or k16_shape or degenerate or linear_transform" > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
for i in 1 2 3; do for lib in libsecpe.so libsecpe_nointt.so; do
ms=$(SECPE_LIB=paper_2502_00847_b200/$lib SECPE_BATCH=16 timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.')
echo "$lib $ms" >> gpurun_out/ab15.log
done; done
