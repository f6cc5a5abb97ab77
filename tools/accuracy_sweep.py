#!/usr/bin/env python
"""Label accuracy at scale (development tool): R batches of 16 configs[4] ciphertexts (16 x 2048 queries,
P = 8 prompts, K = 2 classes, logits N(0, 2) through softmax), each encrypted, run through
secpe_enc_argmax, decrypted and decoded; labels compared with the plaintext argmax of the mean scores."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
from paper_2502_00847_b200 import build, secpe  # noqa: E402

build.build()
R = int(os.environ.get("R", "32"))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
lay = synth.LAYOUTS["argmax_k2"]
st = [list(map(float, c)) for c in json.load(open(os.path.join(ROOT, "data", "sign_7_15_15.json")))["coeffs"]]
ctx = secpe.Context(synth.PARAM_SETS["argmax"], stream=stream.cuda_stream)
keys = ctx.keygen(synth.KEY_SEED_BASE + 5, secpe.argmax_rotations(lay))
B = 16
inp = ctx.new_ct(ctx.L, B)
ol, _ = ctx.argmax_info(lay, st, ctx.L)
out = ctx.new_ct(ol, B)
n = ok = n_in = ok_in = 0
worst = 1.0
for r in range(R):
    scores = [synth.softmax_scores(900000 + r * B + i, lay["queries"], lay["prompts"], lay["classes"]) for i in range(B)]
    for i in range(B):
        ctx.encrypt_coeffs(keys, ctx.encode(secpe.pack(scores[i], lay, ctx.N // 2), ctx.scale), ctx.L, ctx.scale,
                           100000 + r * B + i, out=secpe.Ct(inp.t[i:i + 1], ctx.L, ctx.scale))
    inp.level, inp.scale = ctx.L, ctx.scale
    ctx.enc_argmax(keys, inp, lay, st, out=out)
    torch.cuda.synchronize()
    for i in range(B):
        dec = ctx.decrypt(keys, out, i)
        got = secpe.labels(dec, lay)
        mean = scores[i].mean(axis=1)
        srt = np.sort(mean, axis=1)
        gap = srt[:, -1] - srt[:, -2]
        truth = np.argmax(mean, axis=1)
        good = got == truth
        inside = gap < 2.0 ** -7
        n += len(truth)
        ok += int(good.sum())
        n_in += int(inside.sum())
        ok_in += int(good[inside].sum())
        if (~good).any():
            worst = min(worst, float(gap[~good].max()))
print(json.dumps({"queries": n, "labels_exact": ok / n, "in_margin_queries": n_in,
                  "in_margin_exact": ok_in / max(1, n_in), "wrong_above_margin": int(((n - ok) - (n_in - ok_in))),
                  "largest_gap_of_a_wrong_label": None if worst == 1.0 else worst}))
