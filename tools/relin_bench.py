#!/usr/bin/env python
"""mul_relin_rescale and rotate on the configs[4] parameters (45-bit rows), batch B at the top level
(development tool): CUDA-event medians."""
import os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2502_00847_b200 import build, secpe  # noqa: E402

build.build()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = secpe.Context(synth.PARAM_SETS["argmax"], stream=stream.cuda_stream)
keys = ctx.keygen(synth.KEY_SEED_BASE + 3, [1])
B = int(os.environ.get("B", "8"))
g = synth.rng(1)
a = ctx.new_ct(ctx.L, B)
for i in range(B):
    ctx.encrypt_coeffs(keys, ctx.encode(g.uniform(-1, 1, ctx.N // 2), ctx.scale), ctx.L, ctx.scale, i + 1,
                       out=secpe.Ct(a.t[i:i + 1], ctx.L, ctx.scale))
a.level, a.scale = ctx.L, ctx.scale
o = ctx.new_ct(ctx.L - 1, B)
ro = ctx.new_ct(ctx.L, B)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


print("mul_relin_rescale B=%d: %.3f ms" % (B, t(lambda: ctx.mul_relin_rescale(keys, a, a, out=o))))
print("rotate B=%d: %.3f ms" % (B, t(lambda: ctx.rotate_batch(keys, a, 1, out=ro))))
