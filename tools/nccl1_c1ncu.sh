#!/bin/bash
# single-rank NCCL run of bench.py and the ncu --set full capture of the configs[1] (60-bit, IntA) NTT launches
# (compute-sanitizer is closed on this pool, so no sanitizer pass)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# the torchrun / NCCL code path of bench.py with one rank (init, barriers, max-over-ranks all-reduce)
SECPE_DIST_SINGLE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-micro --no-cpu-baseline > gpurun_out/nccl1.log 2>&1; echo rc=$? >> gpurun_out/nccl1.log
# configs[1] NTT launches (60-bit rows, IntA): integer-pipe utilisation for DESIGN section 6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ntt --launch-skip 8 -c 6 -o gpurun_out/c1_ntt python tools/microbench.py ntt --reps 2 > gpurun_out/c1_ncu.log 2>&1; echo rc=$? >> gpurun_out/c1_ncu.log
