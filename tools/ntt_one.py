#!/usr/bin/env python
"""One NTT shape, forward then inverse, a few times (for ncu captures): python tools/ntt_one.py [P] [L] [reps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2502_00847_b200 import secpe  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = int(sys.argv[2]) if len(sys.argv) > 2 else 29
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
pset = sys.argv[4] if len(sys.argv) > 4 else "argmax"
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = secpe.Context(synth.PARAM_SETS[pset], stream=stream.cuda_stream)
x = torch.from_numpy(synth.uniform_residues(7, ctx.q[1:1 + L], P, ctx.logn)).cuda()
for _ in range(reps):
    ctx.ntt(x, 1, L)
    ctx.ntt(x, 1, L, inverse=True)
torch.cuda.synchronize()
print("ok")
