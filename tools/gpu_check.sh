cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/g_tests.log 2>&1; echo rc=$? >> gpurun_out/g_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/g_smoke.log 2>&1; echo rc=$? >> gpurun_out/g_smoke.log
timeout 900 python bench.py > gpurun_out/g_bench.log 2>&1; echo rc=$? >> gpurun_out/g_bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/g_ref.log 2>&1; echo rc=$? >> gpurun_out/g_ref.log
