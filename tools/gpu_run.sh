cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -q -m gpu -x -k "ks_config or small_ring or dnum or relin or config5_full or rescale or bootstrap_bit_exact or argmax49" > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
for lib in libsecpe.so libsecpe_head.so libsecpe.so libsecpe_head.so; do echo "== $lib" >> gpurun_out/ab2.log; SECPE_LIB=paper_2502_00847_b200/$lib B=8 timeout 300 python tools/relin_bench.py >> gpurun_out/ab2.log 2>&1; done
bash tools/ab.sh head 3 16 2 >> gpurun_out/ab2.log 2>&1
