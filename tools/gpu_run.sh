cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -k "small49 or argmax49 or fused_keyswitch or config5_full or ks_config or boot_k16 or bootstrap_n16_bit_exact" > gpurun_out/t25.log 2>&1; echo rc=$? >> gpurun_out/t25.log
for i in 1 2; do for f in 1 2; do
r=$(SECPE_KS_FUSE=$f timeout 300 python tools/argmax49_probe.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2))")
echo "49bit fuse=$f $r" >> gpurun_out/ab25.log
done; done
for i in 1 2; do for f in 1 2; do
ms=$(SECPE_KS_FUSE=$f SECPE_BATCH=16 timeout 300 python tools/microbench.py argmax --reps 6 2>/dev/null | grep ms_per_batch | tr -dc '0-9.')
echo "45bit fuse=$f $ms" >> gpurun_out/ab25.log
done; done
