#!/usr/bin/env python
"""Kernel microbenchmarks on one B200 (development tool; bench.py is the contract line).

    python tools/microbench.py [ntt] [relin] [rot] [argmax] [--reps R]

ntt    : BASELINE configs[1] -- 64 polys x 24 limbs x 2^16, forward + inverse round trip
relin  : configs[2]-shaped -- mul_relin + rescale on one ciphertext at 24 limbs (dnum 3)
rot    : configs[3]-shaped -- one rotation at 24 limbs
argmax : configs[4] -- secpe_enc_argmax over a batch of 8 ciphertexts
Times are CUDA-event medians after warm-up; inputs > L2 where it matters.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2502_00847_b200 import build, secpe  # noqa: E402


def timeit(fn, reps, stream):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def bench_ntt(reps, stream, out):
    ctx = secpe.Context(synth.PARAM_SETS["ntt"], stream=stream.cuda_stream)
    P, L, N = 64, 24, ctx.N
    x = torch.from_numpy(synth.uniform_residues(2001, ctx.q, P, ctx.logn)).cuda()
    ms_f = timeit(lambda: ctx.ntt(x, 0, L), reps, stream)
    ms_i = timeit(lambda: ctx.ntt(x, 0, L, inverse=True), reps, stream)
    limbs = P * L
    out["ntt"] = dict(fwd_ms=ms_f, inv_ms=ms_i, us_per_limb_fwd=1000 * ms_f / limbs, us_per_limb_inv=1000 * ms_i / limbs,
                      alg_gbs_fwd=16 * N * limbs / (ms_f / 1000) / 1e9, alg_gbs_inv=16 * N * limbs / (ms_i / 1000) / 1e9)


def bench_ntt45(reps, stream, out):
    """configs[4] chain: 64 polys x 29 limbs of the ~2^45 primes q_1..q_29 (exact-FP64 butterflies)."""
    ctx = secpe.Context(synth.PARAM_SETS["argmax"], stream=stream.cuda_stream)
    P, L, N = 64, 29, ctx.N
    x = torch.from_numpy(synth.uniform_residues(2002, ctx.q[1:30], P, ctx.logn)).cuda()
    ms_f = timeit(lambda: ctx.ntt(x, 1, L), reps, stream)
    ms_i = timeit(lambda: ctx.ntt(x, 1, L, inverse=True), reps, stream)
    limbs = P * L
    out["ntt45"] = dict(fwd_ms=ms_f, inv_ms=ms_i, us_per_limb_fwd=1000 * ms_f / limbs,
                        us_per_limb_inv=1000 * ms_i / limbs,
                        alg_gbs_fwd=16 * N * limbs / (ms_f / 1000) / 1e9, alg_gbs_inv=16 * N * limbs / (ms_i / 1000) / 1e9)


def bench_ks(reps, stream, out):
    ctx = secpe.Context(synth.PARAM_SETS["ks"], stream=stream.cuda_stream)
    keys = ctx.keygen(synth.KEY_SEED_BASE + 3, [1])
    L = ctx.L
    g = synth.rng(3001)
    z1 = g.uniform(-1, 1, ctx.N // 2)
    z2 = g.uniform(-1, 1, ctx.N // 2)
    a = ctx.encrypt(keys, z1, L, ctx.scale, 1)
    b = ctx.encrypt(keys, z2, L, ctx.scale, 2)
    out["relin_ms"] = timeit(lambda: ctx.mul_relin(keys, a, b), reps, stream)
    m = ctx.mul_relin(keys, a, b)
    out["rescale_ms"] = timeit(lambda: ctx.rescale(m), reps, stream)
    out["rot_ms"] = timeit(lambda: ctx.rotate(keys, a, 1), reps, stream)


def bench_argmax(reps, stream, out, B=8):
    ctx = secpe.Context(synth.PARAM_SETS[os.environ.get("SECPE_PSET", "argmax")], stream=stream.cuda_stream)
    lay = synth.LAYOUTS["argmax_k2"]
    st = [list(map(float, c)) for c in json.load(open(os.path.join(ROOT, "data", "sign_7_15_15.json")))["coeffs"]]
    keys = ctx.keygen(synth.KEY_SEED_BASE + 5, secpe.argmax_rotations(lay))
    inp = ctx.new_ct(ctx.L, B)
    for i in range(B):
        s = synth.softmax_scores(5000 + i, lay["queries"], lay["prompts"], lay["classes"])
        c = secpe.Ct(inp.t[i:i + 1], ctx.L, ctx.scale)
        ctx.encrypt_coeffs(keys, ctx.encode(secpe.pack(s, lay, ctx.N // 2), ctx.scale), ctx.L, ctx.scale, 700 + i,
                           out=c)
    inp.level, inp.scale = ctx.L, ctx.scale
    ol, _ = ctx.argmax_info(lay, st, ctx.L)
    o = ctx.new_ct(ol, B)
    ms = timeit(lambda: ctx.enc_argmax(keys, inp, lay, st, out=o), max(2, reps // 4), stream)
    ctx.profile_begin()
    ctx.enc_argmax(keys, inp, lay, st, out=o)
    torch.cuda.synchronize()
    pr = ctx.profile_end()
    out["argmax"] = dict(ms_per_batch=ms, batch=B, query_argmax_per_s=B * lay["queries"] / (ms / 1000),
                         ms_per_ct=ms / B, ntt_ms=pr["ntt"]["ms"], ks_ms=pr["keyswitch"]["ms"],
                         rescale_ms=pr["rescale"]["ms"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="*", default=["ntt", "relin", "argmax"])
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    build.build()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    out = {}
    if "ntt" in a.what:
        bench_ntt(a.reps, stream, out)
    if "ntt45" in a.what:
        bench_ntt45(a.reps, stream, out)
    if "relin" in a.what or "rot" in a.what:
        bench_ks(a.reps, stream, out)
    if "argmax" in a.what:
        bench_argmax(a.reps, stream, out, B=int(os.environ.get("SECPE_BATCH", "8")))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
