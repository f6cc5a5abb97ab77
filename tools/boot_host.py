"""Host enqueue time vs device time of one N = 2^16 bootstrap (is the single-ciphertext path launch bound?)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_00847_b200 import secpe  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = secpe.Context(synth.PARAM_SETS["boot16"], stream=stream.cuda_stream)
boot = ctx.boot_create_fft(ctx.L, 16, 7, [5, 5, 5], ctx.scale, bsgs=True)
keys = ctx.keygen(5, boot.steps(), h=64)
z = np.random.default_rng(1).uniform(-1, 1, ctx.N // 2)
c0 = ctx.new_ct(0)
ctx.encrypt_coeffs(keys, ctx.encode(z, ctx.scale), 0, ctx.scale, 7, out=c0)
c0.level, c0.scale = 0, ctx.scale
for B in (1, 4):
    batch = secpe.Ct(c0.t.repeat(B, 1, 1, 1), 0, ctx.scale)
    for _ in range(3):
        r = ctx.bootstrap_boot(keys, batch if B > 1 else c0, boot) if B == 1 else None
    torch.cuda.synchronize()
    if B > 1:
        break
    hs, ds = [], []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        t0 = time.perf_counter()
        r = ctx.bootstrap_boot(keys, c0, boot)
        t1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize()
        hs.append((t1 - t0) * 1e3)
        ds.append(e0.elapsed_time(e1))
    print("B=1 host enqueue ms", np.median(hs), "device ms", np.median(ds))
