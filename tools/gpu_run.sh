cd $GRAFT_REPO_ROOT
for i in 1 2; do for lib in libsecpe.so libsecpe_nors.so libsecpe_head.so; do
r=$(SECPE_LIB=paper_2502_00847_b200/$lib timeout 300 python tools/argmax49_probe.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2))")
echo "49bit $lib $r" >> gpurun_out/ab10.log
done; done
