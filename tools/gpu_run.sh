cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/t26.log 2>&1; echo rc=$? >> gpurun_out/t26.log
SECPE_KS_FUSE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench26_f1.log 2>&1
SECPE_KS_FUSE=2 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench26_f2.log 2>&1
