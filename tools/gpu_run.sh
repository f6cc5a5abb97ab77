cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log
for i in 1 2 3; do for lib in libsecpe.so libsecpe_prev.so; do
ms=$(SECPE_LIB=paper_2502_00847_b200/$lib SECPE_BATCH=16 timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.')
echo "$lib $ms" >> gpurun_out/ab13.log
done; done
for lib in libsecpe.so libsecpe_prev.so; do echo $lib >> gpurun_out/ab13.log; SECPE_LIB=paper_2502_00847_b200/$lib timeout 300 python tools/microbench.py ntt45 --reps 10 2>/dev/null | grep -i "us_per_limb" >> gpurun_out/ab13.log; done
