# round-2 final evidence: GPU parity suite, smoke, headline bench, ncu launch list, ncu --set full of the top kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f_tests.log 2>&1; echo rc=$? >> gpurun_out/f_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/f_smoke.log 2>&1; echo rc=$? >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1; echo rc=$? >> gpurun_out/f_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/f_launches.csv python bench.py --ncu --no-cpu-baseline --no-micro --steps 1 --warmup 3 > gpurun_out/f_ncu_launch.log 2>&1; echo rc=$? >> gpurun_out/f_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:ntt_ks_inner_kernel -c 1 -o gpurun_out/f_ksi python bench.py --ncu --no-cpu-baseline --no-micro --steps 1 --warmup 3 > gpurun_out/f_ncu_full.log 2>&1; echo rc=$? >> gpurun_out/f_ncu_full.log
