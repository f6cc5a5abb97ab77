#!/bin/bash
# compute-sanitizer passes over the small-ring paths (development evidence; summaries go to profiles/):
#   memcheck : toy smoke + the small-ring parity tests that reach every kernel family
#   racecheck / synccheck / initcheck : toy smoke (shared-memory hazards of the NTT / fused key-switch / tcgen05 kernels)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
# the torchrun / NCCL code path of bench.py with one rank (init, barriers, max-over-ranks all-reduce)
SECPE_DIST_SINGLE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-micro --no-cpu-baseline > gpurun_out/nccl1.log 2>&1; echo rc=$? >> gpurun_out/nccl1.log
# configs[1] NTT launches (60-bit rows, IntA): integer-pipe utilisation for DESIGN section 6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt --launch-skip 8 -c 6 -o gpurun_out/c1_ntt python tools/microbench.py ntt --reps 2 > gpurun_out/c1_ncu.log 2>&1; echo rc=$? >> gpurun_out/c1_ncu.log
K="test_ntt_bit_exact or test_ops_bit_exact_toy or test_argmax_small_ring_bit_exact or test_argmax_small49_bit_exact or test_key_switching_digit_counts or test_fused_keyswitch_digit_counts or test_rotate_hoisted_bit_exact or test_empty_inputs or test_cluster_ntt_path or test_fused_ntt_matches_two_pass_and_oracle or test_integer_base_conversion_fallback"
timeout 1200 $CS --tool memcheck --error-exitcode 9 --log-file gpurun_out/san_mem_smoke.txt python __graft_entry__.py smoke > gpurun_out/san_mem_smoke.log 2>&1; echo rc=$? >> gpurun_out/san_mem_smoke.log
timeout 1500 $CS --tool memcheck --error-exitcode 9 --log-file gpurun_out/san_mem_tests.txt python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$K" > gpurun_out/san_mem_tests.log 2>&1; echo rc=$? >> gpurun_out/san_mem_tests.log
timeout 1200 $CS --tool racecheck --error-exitcode 9 --log-file gpurun_out/san_race_smoke.txt python __graft_entry__.py smoke > gpurun_out/san_race_smoke.log 2>&1; echo rc=$? >> gpurun_out/san_race_smoke.log
timeout 900 $CS --tool synccheck --error-exitcode 9 --log-file gpurun_out/san_sync_smoke.txt python __graft_entry__.py smoke > gpurun_out/san_sync_smoke.log 2>&1; echo rc=$? >> gpurun_out/san_sync_smoke.log
timeout 900 $CS --tool initcheck --error-exitcode 9 --log-file gpurun_out/san_init_smoke.txt python __graft_entry__.py smoke > gpurun_out/san_init_smoke.log 2>&1; echo rc=$? >> gpurun_out/san_init_smoke.log
for f in gpurun_out/san_*.txt; do echo "== $f"; grep -c "=========" $f; tail -3 $f; done > gpurun_out/san_summary.txt 2>&1
# keep the logs small enough to travel
for f in gpurun_out/san_*.txt; do head -c 2000000 $f > $f.cut; mv $f.cut $f; done
