#!/usr/bin/env python
"""A/B of the fused TMA NTT (ntt_fused.cu) against the two-pass kernels (development tool).

    python tools/ntt_fused_ab.py            # runs itself with SECPE_NTT_FUSED=0 and =1, compares, prints times

Every shape's forward and inverse outputs must be word-for-word identical between the two paths (both are
pinned to the oracle by tests/test_gpu_parity.py); times are CUDA-event medians (us per limb transform).
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(1, 1, 3), (1, 30, 0), (2, 10, 5), (3, 7, 1), (8, 30, 0), (16, 30, 0), (64, 29, 1), (32, 40, 0)]
if os.environ.get("AB_PSET") == "ntt":  # configs[1]: 24 x 60-bit primes
    SHAPES = [(1, 1, 3), (2, 10, 5), (8, 24, 0), (16, 24, 0), (64, 24, 0)]


def child(tag):
    import numpy as np
    import torch
    import synth
    from paper_2502_00847_b200 import secpe
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = secpe.Context(synth.PARAM_SETS[os.environ.get("AB_PSET", "argmax")], stream=stream.cuda_stream)
    res, outs = {}, {}
    for P, L, first in SHAPES:
        x0 = torch.from_numpy(synth.uniform_residues(11 + P + L, ctx.q[first:first + L] if first + L <= ctx.nq else
                                                    (ctx.q + ctx.p)[first:first + L], P, ctx.logn)).cuda()
        for inv in (False, True):
            x = x0.clone()
            ctx.ntt(x, first, L, inverse=inv)
            torch.cuda.synchronize()
            import hashlib
            outs["%d_%d_%d_%d" % (P, L, first, inv)] = hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()
            for _ in range(3):
                ctx.ntt(x, first, L, inverse=inv)
            ts = []
            for _ in range(15):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.ntt(x, first, L, inverse=inv)
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res["%d_%d_%d_%d" % (P, L, first, inv)] = 1000 * statistics.median(ts) / (P * L)
    json.dump({"t": res, "h": outs}, open(os.path.join(ROOT, "gpurun_out", "ntt_ab_%s.json" % tag), "w"))


def main():
    if len(sys.argv) > 1:
        child(sys.argv[1])
        return
    import numpy as np
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    # extra args: variant libraries "tag=path/to/libsecpe_x.so" (fused on), compared with the default build
    fm = os.environ.get("AB_MODE", "1")
    runs = [("twopass", {"SECPE_NTT_FUSED": "0"}), ("fused", {"SECPE_NTT_FUSED": fm})]
    for v in sys.argv[1:] if False else os.environ.get("AB_VARIANTS", "").split():
        tag, lib = v.split("=")
        runs.append((tag, {"SECPE_NTT_FUSED": fm, "SECPE_LIB": lib}))
    res = {}
    for tag, ev in runs:
        env = dict(os.environ, **ev)
        r = subprocess.run([sys.executable, __file__, tag], env=env)
        if r.returncode:
            print("child %s failed rc=%d" % (tag, r.returncode))
            sys.exit(1)
        res[tag] = json.load(open(os.path.join(ROOT, "gpurun_out", "ntt_ab_%s.json" % tag)))
    A = res["twopass"]
    bad = 0
    print("shape".ljust(26) + "".join(t.rjust(10) for t, _ in runs))
    for k in A["h"]:
        P, L, first, inv = map(int, k.split("_"))
        same = all(res[t]["h"][k] == A["h"][k] for t, _ in runs)
        bad += not same
        print(("P=%d L=%d f=%d %s%s" % (P, L, first, "inv" if inv else "fwd", "" if same else " MISMATCH")).ljust(26) +
              "".join(("%.3f" % res[t]["t"][k]).rjust(10) for t, _ in runs))
    print("MISMATCHES", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
