#!/usr/bin/env python
"""NTT per-limb time versus launch size (development tool): forward/inverse over P polys x L limbs of
the configs[4] 45-bit rows, CUDA-event medians."""
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
for P, L in ((1, 10), (2, 10), (4, 10), (8, 10), (8, 20), (8, 30), (16, 30), (64, 29)):
    x = torch.from_numpy(synth.uniform_residues(7, ctx.q[0:L], P, ctx.logn)).cuda()
    for inv in (False, True):
        for _ in range(3):
            ctx.ntt(x, 0, L, inverse=inv)
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.ntt(x, 0, L, inverse=inv)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        print("P=%3d L=%2d rows=%4d %s %.3f us/limb (%.1f us)" % (P, L, P * L, "inv" if inv else "fwd", 1000 * ms / (P * L), 1000 * ms))
