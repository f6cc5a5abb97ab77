"""Bootstrap precision over many keys and inputs at N = 2^16 (library-built 4/5/6 BSGS material): the
worst refresh error and its distribution.  python tools/boot_sweep.py [n_keys] [n_inputs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_00847_b200 import secpe  # noqa: E402

nk = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ni = int(sys.argv[2]) if len(sys.argv) > 2 else 20
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = secpe.Context(synth.PARAM_SETS["boot16"], stream=stream.cuda_stream)
boot = ctx.boot_create_fft(ctx.L, 16, 7, [4, 5, 6], ctx.scale, bsgs=True)
steps = boot.steps()
errs = []
for ks in range(nk):
    keys = ctx.keygen(1000 + ks, steps, h=64)
    for i in range(ni):
        g = np.random.default_rng(100 * ks + i)
        z = g.uniform(-1, 1, ctx.N // 2)
        c0 = ctx.new_ct(0)
        ctx.encrypt_coeffs(keys, ctx.encode(z, ctx.scale), 0, ctx.scale, 7 + i, out=c0)
        c0.level, c0.scale = 0, ctx.scale
        out = ctx.bootstrap_boot(keys, c0, boot)
        errs.append(float(np.abs(ctx.decrypt(keys, out) - z).max()))
    del keys
e = np.array(errs)
print("bootstraps %d  max err %.3g (2^%.2f)  median %.3g (2^%.2f)  p99 %.3g" % (
    len(e), e.max(), np.log2(e.max()), np.median(e), np.log2(np.median(e)), np.quantile(e, 0.99)))
