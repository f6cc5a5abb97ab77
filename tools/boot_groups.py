import os, sys, time, statistics
sys.path.insert(0, "/root/repo")
import numpy as np, torch, synth
from paper_2502_00847_b200 import secpe
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = secpe.Context(synth.PARAM_SETS["boot16"], stream=stream.cuda_stream)
z = np.random.default_rng(1).uniform(-1, 1, ctx.N // 2)
for groups in [[int(x) for x in g.split(",")] for g in os.environ.get("BOOT_GROUPS", "5,5,5;4,5,6;4,4,4,3;3,4,4,4").split(";")]:
    boot = ctx.boot_create_fft(ctx.L, 16, 7, groups, ctx.scale, bsgs=True)
    keys = ctx.keygen(5, boot.steps(), h=64)
    c0 = ctx.new_ct(0)
    ctx.encrypt_coeffs(keys, ctx.encode(z, ctx.scale), 0, ctx.scale, 7, out=c0)
    c0.level, c0.scale = 0, ctx.scale
    for _ in range(2): r = ctx.bootstrap_boot(keys, c0, boot)
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); r = ctx.bootstrap_boot(keys, c0, boot); b.record(stream); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    err = float(np.abs(ctx.decrypt(keys, r) - z).max())
    print(groups, "ms %.2f" % statistics.median(ts), "keys", len(boot.steps()), "level_out", r.level, "err 2^%.1f" % np.log2(err), flush=True)
    del boot, keys, r
