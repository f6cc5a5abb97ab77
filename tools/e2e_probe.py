#!/usr/bin/env python
"""Development probe: where does the end-to-end (host buffer) argmax step lose time vs the device call?"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_00847_b200 import build, secpe  # noqa: E402


def main():
    build.build()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = secpe.Context(synth.PARAM_SETS["argmax"], stream=stream.cuda_stream)
    lay = synth.LAYOUTS["argmax_k2"]
    st = [list(map(float, c)) for c in json.load(open(os.path.join(ROOT, "data", "sign_7_15_15.json")))["coeffs"]]
    keys = ctx.keygen(synth.KEY_SEED_BASE + 5, secpe.argmax_rotations(lay))
    B = 8
    ins = [ctx.new_ct(ctx.L, B) for _ in range(2)]
    for k in range(2):
        for i in range(B):
            s = synth.softmax_scores(5000 + i, lay["queries"], lay["prompts"], lay["classes"])
            c = secpe.Ct(ins[k].t[i:i + 1], ctx.L, ctx.scale)
            ctx.encrypt_coeffs(keys, ctx.encode(secpe.pack(s, lay, ctx.N // 2), ctx.scale), ctx.L, ctx.scale,
                               700 + i, out=c)
        ins[k].level, ins[k].scale = ctx.L, ctx.scale
    ol, _ = ctx.argmax_info(lay, st, ctx.L)
    outs = [ctx.new_ct(ol, B) for _ in range(2)]
    h_in = ins[0].t.cpu().pin_memory()
    h_out = torch.empty(outs[0].t.shape, dtype=torch.uint64).pin_memory()

    def timed(name, fn, reps=5):
        for _ in range(3):
            fn(0)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        for r in range(reps):
            fn(r)
        b.record(stream)
        torch.cuda.synchronize()
        print("%-34s %8.2f ms/step (host %.2f)" % (name, a.elapsed_time(b) / reps, (time.perf_counter() - t0) * 1e3 / reps),
              flush=True)

    timed("device same buffers", lambda r: ctx.enc_argmax(keys, ins[0], lay, st, out=outs[0]))
    timed("device alternating buffers", lambda r: ctx.enc_argmax(keys, ins[r & 1], lay, st, out=outs[r & 1]))

    def cp_then(r):
        ins[0].t.copy_(h_in, non_blocking=True)
        ctx.enc_argmax(keys, ins[0], lay, st, out=outs[0])
        h_out.copy_(outs[0].t, non_blocking=True)
    timed("device + torch copies same stream", cp_then)
    timed("host API chunk 8", lambda r: ctx.enc_argmax_host(keys, h_in, ctx.L, ctx.scale, lay, st, h_out=h_out))
    timed("host API chunk 4", lambda r: ctx.enc_argmax_host(keys, h_in, ctx.L, ctx.scale, lay, st, h_out=h_out,
                                                            chunk=4))
    timed("device same buffers (again)", lambda r: ctx.enc_argmax(keys, ins[0], lay, st, out=outs[0]))


if __name__ == "__main__":
    main()
