#!/usr/bin/env python
"""Determinism / race check (development tool): the configs[4] argmax over 16 ciphertexts on a non-default
stream (two sub-batch streams, CUDA graph) repeated R times; every output must equal the first word for word."""
import hashlib, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2502_00847_b200 import build, secpe  # noqa: E402

build.build()
R = int(os.environ.get("R", "20"))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
desc = synth.PARAM_SETS["argmax"]
lay = synth.LAYOUTS["argmax_k2"]
st = [list(map(float, c)) for c in json.load(open(os.path.join(ROOT, "data", "sign_7_15_15.json")))["coeffs"]]
ctx = secpe.Context(desc, stream=stream.cuda_stream)
keys = ctx.keygen(synth.KEY_SEED_BASE + 5, secpe.argmax_rotations(lay))
B = 16
inp = ctx.new_ct(ctx.L, B)
for i in range(B):
    s = synth.softmax_scores(7000 + i, lay["queries"], lay["prompts"], lay["classes"])
    ctx.encrypt_coeffs(keys, ctx.encode(secpe.pack(s, lay, ctx.N // 2), ctx.scale), ctx.L, ctx.scale, 70 + i,
                       out=secpe.Ct(inp.t[i:i + 1], ctx.L, ctx.scale))
inp.level, inp.scale = ctx.L, ctx.scale
ol, _ = ctx.argmax_info(lay, st, ctx.L)
out = ctx.new_ct(ol, B)
digests = []
for r in range(R):
    out.t.zero_()
    ctx.enc_argmax(keys, inp, lay, st, out=out)
    torch.cuda.synchronize()
    digests.append(hashlib.sha256(out.t.cpu().numpy().tobytes()).hexdigest())
print("runs", R, "distinct outputs", len(set(digests)))
sys.exit(0 if len(set(digests)) == 1 else 1)
