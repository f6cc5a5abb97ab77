"""One N = 2^16 bootstrap inside an NVTX range "boot" (for ncu --nvtx --nvtx-include boot/)."""
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
boot = ctx.boot_create_fft(ctx.L, 16, 7, [5, 5, 5], ctx.scale, bsgs=True)
keys = ctx.keygen(5, boot.steps(), h=64)
z = np.random.default_rng(1).uniform(-1, 1, ctx.N // 2)
c0 = ctx.new_ct(0)
ctx.encrypt_coeffs(keys, ctx.encode(z, ctx.scale), 0, ctx.scale, 7, out=c0)
c0.level, c0.scale = 0, ctx.scale
r = ctx.bootstrap_boot(keys, c0, boot)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("boot")
r = ctx.bootstrap_boot(keys, c0, boot)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("err", float(np.abs(ctx.decrypt(keys, r) - z).max()))
