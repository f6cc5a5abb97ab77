"""Eight N = 2^16 bootstraps through one plan (secpe_bootstrap_boot_batch, groups 4/5/6) inside an NVTX range
"bootb" (for ncu --nvtx --nvtx-include bootb/ launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_00847_b200 import secpe  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = secpe.Context(synth.PARAM_SETS["boot16"], stream=stream.cuda_stream)
groups = [4, 5, 6]
boot = ctx.boot_create_fft(ctx.L, 16, 7, groups, ctx.scale, bsgs=True)
keys = ctx.keygen(5, boot.steps(), h=64)
B = 8
zs = [np.random.default_rng(i).uniform(-1, 1, ctx.N // 2) for i in range(B)]
cb = ctx.new_ct(0, B)
for i in range(B):
    ctx.encrypt_coeffs(keys, ctx.encode(zs[i], ctx.scale), 0, ctx.scale, 7 + i, out=secpe.Ct(cb.t[i:i + 1], 0, ctx.scale))
cb.level, cb.scale = 0, ctx.scale
r = ctx.bootstrap_boot(keys, cb, boot)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("bootb")
r = ctx.bootstrap_boot(keys, cb, boot)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("err", max(float(np.abs(ctx.decrypt(keys, r, i) - zs[i]).max()) for i in range(B)))
