#!/usr/bin/env python
"""SecPE encrypted aggregate-then-Argmax benchmark on B200 (BASELINE.json metric and configs[4]).

One step = the whole hot path (prompt aggregation, mask/normalise, duplicate, QuickMax, final Sign + 1;
SURVEY.md 8(a) H1-H6, i.e. PAPER.md:141-142 + Algorithm 1) over a batch of B packed ciphertexts,
each holding 2048 queries x P=8 prompts x K=2 classes at N = 2^16 (30 limbs, scale 2^45, dnum 3).
value = query-argmax/s over all ranks (weak scaling: B ciphertexts per rank, no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl secpe|reference]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted argmax/s at N=2^16; NTT & key-switch HBM GB/s vs peak"
UNIT = "query-argmax/s"
WORKLOAD = "configs[4]: SecPE encrypted prompt-ensemble aggregation + Argmax, N=2^16, L=30 (30 x 45-bit primes), " \
           "scale 2^45, dnum=3 (10 x 46-bit special), 2048 queries x P=8 x K=2 per ciphertext, Sign (7,15,15) eps=2^-7"


def peaks():
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_sign(name):
    d = json.load(open(os.path.join(ROOT, "data", name)))
    return [list(map(float, c)) for c in d["coeffs"]]


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.p = index, None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        rows = [l.split(",") for l in out.strip().splitlines() if l.count(",") >= 6]
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[3 + i] and "Not" not in r[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------------------------
# reference arm / cpu baseline: the CPU oracle as it stands
# ------------------------------------------------------------------------------------------------
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# 60-bit (IntA) NTT: warp instructions per N = 2^16 limb transform, mean of forward (384.98 M + 452.20 M) and inverse
# (395.97 M + 465.96 M) over 1536 rows -- ncu smsp__inst_executed.sum, profiles/r02_ncu_configs1_ntt_summary.txt
INTA_WARP_INSTR_PER_LIMB = (384.98e6 + 452.20e6 + 395.97e6 + 465.96e6) / 2 / 1536
SM_MAX_MHZ = 1965.0  # B200 max SM clock (MEASURED_PEAKS.json sm_max_mhz)


def workload_config(B, ws, queries, ct_words, n_rot, nq, np_, alpha, N):
    """`config` of the JSON line (both arms print the same dict for the same --batch / world size)."""
    return {"workload": WORKLOAD, "ciphertexts_per_rank_per_step": B, "queries_per_ciphertext": queries,
            "parallelism": "ciphertexts sharded over ranks (replicated keys)" if ws > 1 else "single GPU",
            "l2": "inputs larger than L2 (%.0f MB ciphertexts + %.0f MB keys per rank)" % (
                B * ct_words * 8 / 1e6, (n_rot + 1) * -(-nq // alpha) * 2 * (nq + np_) * N * 8 / 1e6)}


class OracleArgmax:
    """The CPU oracle's full argmax of ONE configs[4] ciphertext (2048 queries); keys and the input are
    built once, run() times plan.argmax only.  Returns (seconds, queries, threads actually used)."""

    def __init__(self, seed_base=1):
        import synth
        from oracle import ckks, plan
        self.plan = plan
        prm = ckks.Params(synth.PARAM_SETS["argmax"])
        self.lay = synth.LAYOUTS["argmax_k2"]
        self.st = load_sign("sign_7_15_15.json")
        self.ev = ckks.Oracle(prm)
        self.keys = self.ev.keygen(synth.KEY_SEED_BASE + 5, plan.argmax_rotations(self.lay))
        scores = synth.softmax_scores(1000 * 5 + seed_base, self.lay["queries"], self.lay["prompts"],
                                      self.lay["classes"])
        self.ct = self.ev.encrypt(self.keys, plan.pack(scores, self.lay, prm.N // 2), prm.scale, 11)

    def run(self):
        from oracle import ckks
        threads = ckks.lib().o_set_threads(0)  # the OpenMP team size the oracle's parallel loops run with
        t0 = time.perf_counter()
        self.plan.argmax(self.ev, self.keys, self.ct, self.lay, self.st)
        dt = time.perf_counter() - t0
        return dt, self.lay["queries"], threads

    def h1_seconds(self, threads):
        """Oracle time of the circuit's first stage (H1: log2 P = 3 rotations + additions at the top level, the
        key-switch-bound op the whole circuit is made of) with `threads` OpenMP threads."""
        from oracle import ckks
        lib = ckks.lib()
        prev = lib.o_set_threads(0)
        used = lib.o_set_threads(threads)
        try:
            y = self.ct
            t0 = time.perf_counter()
            for t in range(3):
                y = self.ev.add(y, self.ev.rot(self.keys, y, self.lay["classes"] << t))
            return time.perf_counter() - t0, used
        finally:
            lib.o_set_threads(prev)


def cpu_baseline_line(ora, dt, q, cores):
    """the oracle on all host cores (one full ciphertext) and single-threaded.  The
    single-thread figure is the all-core value scaled by the single/all-core time ratio measured on the H1
    sample (a full single-thread ciphertext would take minutes)."""
    t1, _ = ora.h1_seconds(1)
    tn, used = ora.h1_seconds(cores)
    v = q / dt
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "logical_cpus": os.cpu_count(),
            "sample": "1 ciphertext of the same workload (2048 queries, full argmax circuit) on %d OpenMP threads, "
                      "%.1f s" % (cores, dt),
            "single_thread_value": v * tn / t1,
            "single_thread_sample": "H1 stage (3 top-level rotations) timed on 1 thread (%.2f s) and on %d threads "
                                    "(%.2f s); single-thread value = all-core value x %.3f" % (t1, used, tn, tn / t1)}


def oracle_argmax_once(seed_base=1):
    return OracleArgmax(seed_base).run()


REF_CAP_S = 600.0  # safety cap on the reference arm's timed region (a default-sized run never reaches it)


def run_reference(a):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    ora = OracleArgmax()
    for _ in range(a.warmup if a.ref_warmup else 0):
        ora.run()
    # each step is one full ciphertext of the workload (2048 queries, ~13 s on 16 cores): --steps 20 ends in
    # about 4.5 minutes.  The cap only guards against a much slower host or a very large --steps.
    times, q, cores = [], 0, 1
    for _ in range(a.steps):
        dt, q, cores = ora.run()
        times.append(dt)
        if sum(times) > REF_CAP_S:
            break
    n = len(times)
    T = sum(times)
    v = q * n / T
    sample = ("1 ciphertext (2048 queries x P=8 x K=2, full argmax circuit) per step, %d of %d requested steps "
              "timed%s; warm-up steps %s" % (n, a.steps, "" if n == a.steps else " (capped at %.0f s)" % REF_CAP_S,
                                             "run" if a.ref_warmup else "skipped (CPU oracle has no warm-up state)"))
    prm, lay = ora.ev.prm, ora.lay
    cfg = workload_config(a.batch, ws, lay["queries"], 2 * prm.nq * prm.N, len(ora.plan.argmax_rotations(lay)),
                          prm.nq, prm.np_, prm.alpha, prm.N)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": n,
            "steps_requested": a.steps, "warmup": a.warmup, "ms_per_step": 1000 * T / n, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues mod 45/60-bit primes)", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model(), "logical_cpus": os.cpu_count()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
def micro_configs(stream, reps=5):
    """BASELINE configs[1]-[3] on one GPU (reported beside the headline; CUDA events, median of reps):
    [1] 64 polys x 24 limbs NTT + INTT round trip; [2] 32 ciphertext pairs mul + relinearise + rescale
    (one batched call); [3] 128 ciphertexts rotated by each of the 15 keys 2^k (one batched call per key)."""
    import torch
    import synth
    from paper_2502_00847_b200 import secpe
    peak, _ = peaks()

    def t_ms(fn):
        for _ in range(2):
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

    out = {}
    ctx = secpe.Context(synth.PARAM_SETS["ntt"], stream=stream.cuda_stream)
    x = torch.from_numpy(synth.uniform_residues(2001, ctx.q, 64, ctx.logn)).cuda()
    ms = t_ms(lambda: (ctx.ntt(x, 0, 24), ctx.ntt(x, 0, 24, inverse=True)))
    gbs = 2 * 16 * ctx.N * 64 * 24 / (ms / 1000) / 1e9
    out["configs[1]_ntt"] = {"ms_round_trip": ms, "limb_transforms_per_s": 2 * 64 * 24 / (ms / 1000),
                             "alg_gbs": gbs, "frac_of_hbm": gbs / peak,
                             # the 60-bit rows are bound by the integer instruction stream, not HBM:
                             # issue-slot roofline = warp instructions per limb transform (ncu smsp__inst_executed.sum of
                             # the four IntA passes / 1536 rows, profiles/r02_ncu_configs1_ntt_summary.txt) x transforms/s
                             # over 148 SMs x 4 schedulers x 1 warp instruction per clock at the max SM clock
                             "bound": "alu", "warp_instr_per_limb_transform": INTA_WARP_INSTR_PER_LIMB,
                             "alu_achieved_ginstr_s": INTA_WARP_INSTR_PER_LIMB * 2 * 64 * 24 / (ms / 1000) / 1e9,
                             "alu_peak_ginstr_s": 148 * 4 * SM_MAX_MHZ * 1e6 / 1e9,
                             "frac_of_issue_slots": INTA_WARP_INSTR_PER_LIMB * 2 * 64 * 24 / (ms / 1000)
                                                    / (148 * 4 * SM_MAX_MHZ * 1e6),
                             "note": "60-bit primes: integer Shoup path; ncu: ALU pipe 46-56 %, FMA pipe 23-28 %, issue "
                                     "51-60 %, DRAM 27-31 % of peak"}
    del ctx, x
    ctx = secpe.Context(synth.PARAM_SETS["ks"], stream=stream.cuda_stream)
    keys = ctx.keygen(synth.KEY_SEED_BASE + 3, [1 << k for k in range(15)])
    g = synth.rng(3001)
    B = 32
    a = ctx.new_ct(ctx.L, B)
    b = ctx.new_ct(ctx.L, B)
    for i in range(B):
        for c, seed in ((a, 2 * i + 1), (b, 2 * i + 2)):
            m = ctx.encode(g.uniform(-1, 1, ctx.N // 2), ctx.scale)
            ctx.encrypt_coeffs(keys, m, ctx.L, ctx.scale, seed, out=secpe.Ct(c.t[i:i + 1], ctx.L, ctx.scale))
    a.level = b.level = ctx.L
    a.scale = b.scale = ctx.scale
    o = ctx.new_ct(ctx.L - 1, B)
    ms = t_ms(lambda: ctx.mul_relin_rescale(keys, a, b, out=o))
    # algorithmic bytes per op (SURVEY 8(d) cfg 3): inputs 2 x 2 x (L+1) limbs, output 2 L limbs, the
    # relinearisation key (dnum x 2 x (L+1+k) limbs) once per batch
    limb = ctx.N * 8
    dnum = -(-ctx.nq // ctx.alpha)
    key_limbs = dnum * 2 * (ctx.nq + ctx.np_)
    b2 = (4 * ctx.nq + 2 * (ctx.nq - 1) + key_limbs / B) * limb
    gb2 = B * b2 / (ms / 1000) / 1e9
    out["configs[2]_mul_relin_rescale"] = {"ms_per_batch": ms, "batch": B, "ops_per_s": B / (ms / 1000),
                                           "alg_bytes_per_op": b2, "alg_gbs": gb2, "frac_of_hbm": gb2 / peak}
    R = 128
    r = ctx.new_ct(ctx.L, R)
    for i in range(R):
        r.t[i].copy_(a.t[i % B])
    r.level, r.scale = ctx.L, ctx.scale
    ro = ctx.new_ct(ctx.L, R)
    ms = t_ms(lambda: [ctx.rotate_batch(keys, r, 1 << k, out=ro) for k in range(15)])
    del ro
    # N2: the 15 rotations of each ciphertext share one ModUp (secpe_rotate_hoisted, reading R29)
    steps = [1 << k for k in range(15)]
    outs = [None]
    def hoisted():
        outs[0] = None  # free the previous call's 15 output batches first (48 GB)
        outs[0] = ctx.rotate_hoisted(keys, r, steps)
    ms_h = t_ms(hoisted)
    outs[0] = None
    # per rotation (SURVEY 8(d) cfg 4): input 2 (L+1) limbs + output 2 (L+1) limbs + the Galois key / R
    b3 = (4 * ctx.nq + key_limbs / R) * limb
    gb3 = 15 * R * b3 / (ms_h / 1000) / 1e9
    gb3n = 15 * R * b3 / (ms / 1000) / 1e9
    out["configs[3]_rotation"] = {"ms_per_15_keys": ms_h, "cts": R, "rotations_per_s": 15 * R / (ms_h / 1000),
                                  "hoisted": True, "alg_bytes_per_rotation": b3, "alg_gbs": gb3,
                                  "frac_of_hbm": gb3 / peak,
                                  "not_hoisted": {"ms_per_15_keys": ms, "rotations_per_s": 15 * R / (ms / 1000),
                                                  "alg_gbs": gb3n, "frac_of_hbm": gb3n / peak}}
    del ctx, keys, a, b, r, o
    nxt = {"N3_bootstrap": bootstrap_bench(stream, t_ms), "N4_argmax_k16": argmax_k16_bench(stream, t_ms),
           "N4_argmax_n256": argmax_boot_bench(stream, t_ms, "argmax_n256", 8, 6.0),
           "N4_clip_80x1000": clip_bench(stream, t_ms)}
    return out, nxt


def bootstrap_bench(stream, t_ms):
    """one CKKS bootstrap (readings R32-R37) of a level-0 ciphertext, sparse secret h = 64,
    K = 16, r = 7, library-built material: N = 2^12 with dense BSGS 64 x 32 transforms (secpe_boot_create) and
    N = 2^16 with the factorised special-FFT transforms (secpe_boot_create_fft).  Latency of one call on one
    GPU, CUDA events, median."""
    import torch
    import synth
    from paper_2502_00847_b200 import secpe
    ctx = secpe.Context(synth.PARAM_SETS["boot"], stream=stream.cuda_stream)
    n1, n2, K, r, h = 64, 32, 16, 7, 64
    rot = list(range(1, n1)) + [j * n1 for j in range(1, n2)] + [secpe.CONJ]
    keys = ctx.keygen(synth.KEY_SEED_BASE + 23, rot, h=h)
    t0 = time.time()
    boot = ctx.boot_create(ctx.L, K, r, n1, n2, ctx.scale)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    z = synth.rng(4001).uniform(-1, 1, ctx.N // 2)
    c0 = ctx.new_ct(0)
    ctx.encrypt_coeffs(keys, ctx.encode(z, ctx.scale), 0, ctx.scale, 77, out=c0)
    c0.level, c0.scale = 0, ctx.scale
    res = [None]

    def one():
        res[0] = ctx.bootstrap_with(keys, c0, boot)
    ms = t_ms(one)
    err = float(abs(ctx.decrypt(keys, res[0]) - z).max())
    ks = 2 * (n1 - 1 + n2 - 1) * 2 + 2 + 2 * (7 + r)
    out = {"N=2^12_dense": {"ms_per_bootstrap": ms, "logn": ctx.logn, "slots": ctx.N // 2, "level_in": 0,
                            "raised_to": ctx.L, "level_out": res[0].level, "key_switches": ks, "max_abs_err": err,
                            "setup_s": setup_s, "transforms": "dense BSGS 64 x 32 (R34)"}}
    del boot, keys, res, c0, ctx
    # the paper's ring: factorised special-FFT transforms (R37), groups 5/5/5
    ctx = secpe.Context(synth.PARAM_SETS["boot16"], stream=stream.cuda_stream)
    groups = [4, 5, 6]
    t0 = time.time()
    boot = ctx.boot_create_fft(ctx.L, K, r, groups, ctx.scale, bsgs=True)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    steps = boot.steps()
    keys = ctx.keygen(synth.KEY_SEED_BASE + 31, steps, h=h)
    z = synth.rng(4002).uniform(-1, 1, ctx.N // 2)
    c0 = ctx.new_ct(0)
    ctx.encrypt_coeffs(keys, ctx.encode(z, ctx.scale), 0, ctx.scale, 78, out=c0)
    c0.level, c0.scale = 0, ctx.scale
    res = [ctx.new_ct(ctx.L - (2 * len(groups) + 6 + r))]  # one output buffer: the call replays a CUDA graph

    def one16():
        res[0] = ctx.bootstrap_boot(keys, c0, boot, out=res[0])
    ms = t_ms(one16)
    err = float(abs(ctx.decrypt(keys, res[0]) - z).max())
    # where one bootstrap's time goes (the library's CUDA-event profiler, one extra untimed call)
    torch.cuda.synchronize()
    ctx.opcounts(reset=True)
    ctx.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    one16()
    e1.record(stream)
    prof = ctx.profile_end()
    torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    cnt = ctx.opcounts(reset=True)
    breakdown = {"keyswitch_share": prof["keyswitch"]["ms"] / tot, "rescale_share": prof["rescale"]["ms"] / tot,
                 "ntt_share": prof["ntt"]["ms"] / tot, "profiled_ms": tot, "key_switches": cnt["keyswitch"],
                 "ntt_limbs": cnt["ntt_limbs"], "launches": cnt["launches"]}
    # throughput: 8 distinct ciphertexts through one plan (secpe_bootstrap_boot_batch); every output checked
    B = 8
    zb = [synth.rng(4100 + i).uniform(-1, 1, ctx.N // 2) for i in range(B)]
    cb = ctx.new_ct(0, B)
    for i in range(B):
        ctx.encrypt_coeffs(keys, ctx.encode(zb[i], ctx.scale), 0, ctx.scale, 90 + i,
                           out=secpe.Ct(cb.t[i:i + 1], 0, ctx.scale))
    cb.level, cb.scale = 0, ctx.scale
    rb = [ctx.new_ct(ctx.L - (2 * len(groups) + 6 + r), B)]

    def batch():
        rb[0] = ctx.bootstrap_boot(keys, cb, boot, out=rb[0])
    ms_b = t_ms(batch)
    errs = [float(abs(ctx.decrypt(keys, rb[0], i) - zb[i]).max()) for i in range(B)]
    out["N=2^16_fft_batch8"] = {"ms_per_call": ms_b, "ciphertexts": B, "bootstraps_per_s": B / (ms_b / 1000),
                                "max_abs_err": max(errs), "inputs": "8 distinct ciphertexts, every output decrypted"}
    out["N=2^16_fft"] = {"breakdown": breakdown, "ms_per_bootstrap": ms, "logn": ctx.logn, "slots": ctx.N // 2, "level_in": 0,
                         "raised_to": ctx.L, "level_out": res[0].level, "galois_keys": len(steps),
                         "max_abs_err": err, "setup_s": setup_s,
                         "transforms": "special-FFT groups 4/5/6, baby-step giant-step form (R37, R39)"}
    return out


def clip_bench(stream, t_ms, G=2, prompts=80, classes=1000):
    """SURVEY 8(f) N4 CLIP scale: `prompts` prompts x `classes` classes (padded to 1024 with
    zero scores), 16 queries per query set at N = 2^16, 2 prompts per ciphertext and prompts / 2 ciphertexts
    per query set summed first (prompt_cts), ten bootstraps per query set; G query sets per call."""
    import torch
    import synth
    from paper_2502_00847_b200 import secpe
    ctx = secpe.Context(synth.PARAM_SETS["boot_argmax16_g4"], stream=stream.cuda_stream)
    lay = synth.LAYOUTS["clip"]
    st = load_sign("sign_7_15_15.json")
    bs = 2.0 ** 50
    boot = ctx.boot_create_fft(ctx.L, 16, 7, [3, 4, 4, 4], bs, bsgs=True)
    P, K, Q, blk = lay["prompts"], lay["classes"], lay["queries"], lay["block"]
    pc = prompts // P
    rot = [K << t for t in range(P.bit_length() - 1)] + [-K] + [1 << i for i in range(K.bit_length() - 1)]
    keys = ctx.keygen(synth.KEY_SEED_BASE + 45, sorted(set(rot)) + boot.steps(), h=64)
    scores, cts = [], []
    for gi in range(G):
        sc = np.zeros((Q, prompts, K))
        sc[:, :, :classes] = synth.ensemble_scores(61 + gi, Q, prompts, classes)
        scores.append(sc)
        for i in range(pc):
            z = np.zeros(ctx.N // 2)
            for qi in range(Q):
                for p in range(P):
                    z[qi * blk + p * K: qi * blk + (p + 1) * K] = sc[qi, i * P + p]
            cts.append(ctx.encrypt(keys, z, 16, ctx.scale, 1000 * gi + i))
    batch = secpe.Ct(torch.cat([c.t for c in cts]), 16, ctx.scale)
    del cts
    res = [None]

    def run():
        res[0] = ctx.enc_argmax_boot(keys, batch, lay, st, boot, bs, prompt_cts=pc)
    ms = t_ms(run)
    good = tot = 0
    for gi in range(G):
        lab = secpe.labels(ctx.decrypt(keys, res[0], gi), lay)
        mean = scores[gi].mean(axis=1)
        srt = np.sort(mean, axis=1)
        ok = srt[:, -1] - srt[:, -2] >= 2.0 ** -7
        good += int((lab[ok] == np.argmax(mean, axis=1)[ok]).sum())
        tot += int(ok.sum())
    return {"ms_per_call": ms, "query_sets_per_call": G, "queries_per_set": Q, "prompts": prompts,
            "classes": classes, "prompt_ciphertexts_per_set": pc, "query_argmax_per_s": G * Q / (ms / 1000),
            "bootstraps_per_set": K.bit_length() - 1, "labels_exact_above_margin": good / max(tot, 1),
            "above_margin": tot, "logn": ctx.logn}


def argmax_k16_bench(stream, t_ms, B=8):
    return argmax_boot_bench(stream, t_ms, "argmax_k16", B, 2.0)


def argmax_boot_bench(stream, t_ms, lname, B, sigma, pname="boot_argmax16_g4", groups=(3, 4, 4, 4)):
    """SURVEY 8(f) N4 (reading R38): Algorithm 1 with K = 16 classes at N = 2^16 (256 queries x 8 prompts per
    ciphertext), refreshed by four factorised bootstraps per ciphertext (secpe_enc_argmax_boot); one
    ciphertext per call, CUDA events, median.  Labels checked against the plaintext argmax above the margin."""
    import torch
    import synth
    from paper_2502_00847_b200 import secpe
    ctx = secpe.Context(synth.PARAM_SETS[pname], stream=stream.cuda_stream)
    lay = synth.LAYOUTS[lname]
    st = load_sign("sign_7_15_15.json")
    bs = 2.0 ** 50
    boot = ctx.boot_create_fft(ctx.L, 16, 7, list(groups), bs, bsgs=True)
    P, K = lay["prompts"], lay["classes"]
    rot = [K << t for t in range(P.bit_length() - 1)] + [-K] + [1 << i for i in range(K.bit_length() - 1)]
    keys = ctx.keygen(synth.KEY_SEED_BASE + 39, sorted(set(rot)) + boot.steps(), h=64)
    # B ciphertexts per call: one plan, keys and transform plaintexts read once per op for the batch
    scores = [synth.softmax_scores(47 + i, lay["queries"], P, K, sigma=sigma) for i in range(B)]
    cts = []
    for i in range(B):
        z = np.zeros(ctx.N // 2)
        for qi in range(lay["queries"]):
            for p in range(P):
                z[qi * lay["block"] + p * K: qi * lay["block"] + (p + 1) * K] = scores[i][qi, p]
        cts.append(ctx.encrypt(keys, z, 16, ctx.scale, 49 + i))
    batch = secpe.Ct(torch.cat([c.t for c in cts]), 16, ctx.scale)
    res = [None]

    def run():
        res[0] = ctx.enc_argmax_boot(keys, batch, lay, st, boot, bs)
    ms = t_ms(run)
    good, tot, inm = 0, 0, 0
    for i in range(B):
        lab = secpe.labels(ctx.decrypt(keys, res[0], i), lay)
        mean = scores[i].mean(axis=1)
        srt = np.sort(mean, axis=1)
        ok = srt[:, -1] - srt[:, -2] >= 2.0 ** -7
        good += int((lab[ok] == np.argmax(mean, axis=1)[ok]).sum())
        tot += int(ok.sum())
        inm += int((~ok).sum())
    return {"ms_per_call": ms, "ciphertexts_per_call": B, "queries_per_ciphertext": lay["queries"], "classes": K,
            "prompts": P, "query_argmax_per_s": B * lay["queries"] / (ms / 1000),
            "bootstraps_per_ciphertext": K.bit_length() - 1, "logit_sigma": sigma,
            "labels_exact_above_margin": good / tot, "in_margin_fraction": inm / (B * lay["queries"]),
            "logn": ctx.logn, "chain": pname + ": q0 60 + 16 x 45 + 21 x 50 bit", "groups": list(groups)}

def argmax_accuracy(ctx, keys, out, all_scores, lay):
    """Client side, outside every timed region: decrypt the step's outputs and decode the labels (argmax over each
    query's K window slots, reading R19) against the plaintext argmax of the mean scores."""
    from paper_2502_00847_b200 import secpe
    n_ok = n_ok_margin = n_margin = n_q = 0
    for i in range(len(all_scores)):
        dec = ctx.decrypt(keys, out, i)
        got = secpe.labels(dec, lay)
        mean = all_scores[i].mean(axis=1)
        srt = np.sort(mean, axis=1)
        above = srt[:, -1] - srt[:, -2] >= 2.0 ** -7  # the Sign margin of the (7,15,15) design
        truth = np.argmax(mean, axis=1)
        n_q += len(truth)
        n_ok += int((got == truth).sum())
        n_ok_margin += int((got == truth)[above].sum())
        n_margin += int(above.sum())
    return {"queries": n_q, "labels_exact": n_ok / n_q, "labels_exact_above_margin": n_ok_margin / max(1, n_margin),
            "in_margin_fraction": 1.0 - n_margin / n_q,
            "note": "decrypted one-hot decoded by argmax over each query's window vs argmax of the plaintext "
                    "mean scores; 'above margin' = top-1 gap >= 2^-7"}


def argmax49_bench(stream, B=16, steps=5, warmup=3):
    """configs[4]'s workload on the paper's prime size (reading R41: 30 x 49-bit chain primes at scale 2^49, 10 x
    50-bit special primes): every row takes the FP64 NTT with reductions (FpB).  Same batch, layout, circuit and
    timing as the headline (device time of `steps` steps after `warmup`), plus the NTT's HBM roofline from one
    profiled step."""
    import torch

    import synth
    from paper_2502_00847_b200 import secpe, shard
    lay = synth.LAYOUTS["argmax_k2"]
    st = load_sign("sign_7_15_15.json")
    ctx = secpe.Context(synth.PARAM_SETS["argmax49"], stream=stream.cuda_stream)
    keys = ctx.keygen(synth.KEY_SEED_BASE + 49, secpe.argmax_rotations(lay))
    L = ctx.L
    inp = ctx.new_ct(L, B)
    all_scores = []
    for i in range(B):
        scores = synth.softmax_scores(shard.input_seed(49, i), lay["queries"], lay["prompts"], lay["classes"])
        all_scores.append(scores)
        ctx.encrypt_coeffs(keys, ctx.encode(secpe.pack(scores, lay, ctx.N // 2), ctx.scale), L, ctx.scale, 900 + i,
                           out=secpe.Ct(inp.t[i:i + 1], L, ctx.scale))
    inp.level, inp.scale = L, ctx.scale
    ol, _ = ctx.argmax_info(lay, st, L)
    out = ctx.new_ct(ol, B)
    for _ in range(warmup):
        ctx.enc_argmax(keys, inp, lay, st, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        ctx.enc_argmax(keys, inp, lay, st, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ctx.profile_begin()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    ctx.enc_argmax(keys, inp, lay, st, out=out)
    p1.record(stream)
    torch.cuda.synchronize()
    prof = ctx.profile_end()
    ms_prof = p0.elapsed_time(p1)
    peak, _ = peaks()
    ntt, ks = prof["ntt_fp"], prof["keyswitch"]
    gbs = lambda d: d["bytes"] / (d["ms"] / 1000.0) / 1e9 if d["ms"] > 0 else 0.0
    ops = prof.get("ntt_fp_operands", {"bytes": 0.0})
    nttop = (ntt["bytes"] + ops["bytes"]) / (ntt["ms"] / 1000.0) / 1e9 if ntt["ms"] > 0 else 0.0
    r = {"workload": "configs[4] with 30 x 49-bit chain primes nearest 2^49, scale 2^49, 10 x 50-bit special "
                     "primes (R41; the paper's log Q / L, PAPER.md:327)",
         "ciphertexts_per_step": B, "ms_per_step": ms, "query_argmax_per_s": lay["queries"] * B / (ms / 1000.0),
         "ntt_rows": "FpB (FP64 with reductions)" if ntt["ms"] > 0 and prof["ntt_int"]["ms"] == 0 else "mixed",
         "ntt_gbs": nttop, "ntt_frac": nttop / peak, "ntt_gbs_transform_only": gbs(ntt),
         "ntt_frac_transform_only": gbs(ntt) / peak, "ntt_share_of_step": ntt["ms"] / ms_prof,
         "keyswitch_gbs": gbs(ks), "keyswitch_frac": gbs(ks) / peak,
         "accuracy": argmax_accuracy(ctx, keys, out, all_scores, lay)}
    del keys, inp, out, ctx
    torch.cuda.empty_cache()
    return r


def run_secpe(a):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2502_00847_b200 import build, secpe, shard

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    # NCCL plumbing (barriers + max-over-ranks) for N > 1; SECPE_DIST_SINGLE=1 runs the same path with one rank
    # (the 1-GPU box's check that the torchrun / NCCL code path executes)
    use_dist = ws > 1 or (os.environ.get("SECPE_DIST_SINGLE") == "1" and "MASTER_ADDR" in os.environ)
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    build.build()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    desc = synth.PARAM_SETS["argmax"]
    lay = synth.LAYOUTS["argmax_k2"]
    st = load_sign("sign_7_15_15.json")
    ctx = secpe.Context(desc, stream=stream.cuda_stream)
    steps_rot = secpe.argmax_rotations(lay)
    # evaluation keys: every rank derives the same keys from the same client seed (replicated, no transfer)
    keys = ctx.keygen(synth.KEY_SEED_BASE + 5, steps_rot)
    B = a.batch
    L = ctx.L
    inp = ctx.new_ct(L, B)
    all_scores = []
    for i in range(B):
        # rank r owns global ciphertexts [r B, (r + 1) B): the sharded job draws the single-rank job's inputs
        scores = synth.softmax_scores(shard.input_seed(5, rank * B + i), lay["queries"], lay["prompts"],
                                      lay["classes"])
        all_scores.append(scores)
        z = secpe.pack(scores, lay, ctx.N // 2)
        m = ctx.encode(z, ctx.scale)
        c = secpe.Ct(inp.t[i:i + 1], L, ctx.scale)
        ctx.encrypt_coeffs(keys, m, L, ctx.scale, 700 + i, out=c)
    inp.level, inp.scale = L, ctx.scale
    ol, _ = ctx.argmax_info(lay, st, L)
    out = ctx.new_ct(ol, B)
    torch.cuda.synchronize()

    def step():
        ctx.enc_argmax(keys, inp, lay, st, out=out)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if a.ncu:
        # exactly one step inside cudaProfilerStart/Stop (ncu --profile-from-start off)
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(json.dumps({"ncu_step": True, "batch": B, "launches": ctx.opcounts(reset=True)["launches"]}))
        return
    if use_dist:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    ctx.opcounts(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    counts = ctx.opcounts(reset=True)
    clk = clocks.stop()
    ms = shard.max_over_ranks(e0.elapsed_time(e1), device="cuda")  # slowest rank's device time
    if use_dist:
        dist.barrier()
    # roofline: the same K steps again with CUDA events recorded on the launching stream around every
    # NTT / key-switch / rescale span (kept out of the headline timing above)
    ctx.profile_begin()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(a.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof = ctx.profile_end()
    ms_prof = p0.elapsed_time(p1)
    queries = lay["queries"] * B * ws * a.steps
    value = shard.job_throughput(lay["queries"] * B * a.steps, ws, ms)

    # end to end through the public C-ABI host-buffer call (secpe_enc_argmax_host): pinned host inputs,
    # host->device copies (on the library's copy stream, overlapping the previous step's compute) and
    # the device->host result copy inside the timed region
    h_in = inp.t.cpu().pin_memory()
    h_out = torch.empty(out.t.shape, dtype=torch.uint64).pin_memory()
    for _ in range(max(4, a.warmup)):  # both staging slots captured and replayed once
        ctx.enc_argmax_host(keys, h_in, L, ctx.scale, lay, st, h_out=h_out, chunk=B)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    fe = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    f0, f1 = fe[0], fe[-1]
    t_host = time.perf_counter()
    f0.record(stream)
    for i in range(a.steps):
        ctx.enc_argmax_host(keys, h_in, L, ctx.scale, lay, st, h_out=h_out, chunk=B)
        fe[i + 1].record(stream)
    t_host = time.perf_counter() - t_host
    torch.cuda.synchronize()
    print("e2e steps ms", [round(fe[i].elapsed_time(fe[i + 1]), 2) for i in range(a.steps)],
          "host enqueue ms %.1f" % (1e3 * t_host), file=sys.stderr)
    ms_e2e = shard.max_over_ranks(f0.elapsed_time(f1), device="cuda")
    e2e = shard.job_throughput(lay["queries"] * B * a.steps, ws, ms_e2e)

    accuracy = argmax_accuracy(ctx, keys, out, all_scores, lay)

    if rank != 0:
        if use_dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    ntt, ntt_int, ks = prof["ntt_fp"], prof["ntt_int"], prof["keyswitch"]
    gbs = lambda d: d["bytes"] / (d["ms"] / 1000.0) / 1e9 if d["ms"] > 0 else 0.0
    # algorithmic bytes of the NTT launches: the transform's 16 N per limb (split over its passes) plus the operand
    # limbs their fused prologues / epilogues read (and, for the fused ModUp pass 2 + key inner product, the key,
    # tensor inputs and acc rows it reads and writes instead of the digits' NTT form)
    ops = prof.get("ntt_fp_operands", {"bytes": 0.0})
    ach_t, ks_ach = gbs(ntt), gbs(ks)
    ach = (ntt["bytes"] + ops["bytes"]) / (ntt["ms"] / 1000.0) / 1e9 if ntt["ms"] > 0 else 0.0
    traffic, tsrc, t_over_a, step_dram = None, None, None, {}
    tp = os.path.join(ROOT, "profiles", "ntt_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic, tsrc = tj["dram_bytes_per_limb_transform"], tj.get("source")
            t_over_a = tj.get("traffic_over_algorithmic")
            # every launch of the step: the real DRAM bytes (same ncu list) over the measured step time
            if tj.get("step_ciphertexts") == B and tj.get("step_dram_bytes"):
                step_dram = {"step_dram_bytes": tj["step_dram_bytes"],
                             "step_dram_gbs": tj["step_dram_bytes"] / (ms / a.steps / 1000.0) / 1e9,
                             "step_dram_source": tj.get("step_source")}
        except Exception:
            traffic = None
    # FP64-pipe roof of the same kernels: (N/2) log2 N butterflies per limb transform, 8 FP64-pipe
    # instructions each in the exact-FP64 formulation; peak = 148 SMs x 64 FP64
    # lanes/clk x the SM clock sampled under load
    clk_mhz = clk.get("sm_mhz") or 1965.0
    fp64_peak = 148 * 64 * clk_mhz * 1e6 / 1e12
    fp64_ach = (ctx.N // 2) * ctx.logn * 8 * ntt["units"] / (ntt["ms"] / 1000.0) / 1e12 if ntt["ms"] > 0 else 0.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64 (RNS residues mod 45/60-bit primes)", "data": "synthetic",
        "config": workload_config(B, ws, lay["queries"], inp.t[0].numel(), len(steps_rot), ctx.nq, ctx.np_,
                                  ctx.alpha, ctx.N),
        "roofline": {"bound": "hbm", "kernel": "ntt family on the 45-bit (FP64) rows: every forward/inverse launch in the "
                                                "profiled region incl. the fused ModUp pass 2 + key inner product "
                                                "(ntt_ks_inner_kernel) and the fused prologues/epilogues (%.0f limb "
                                                "transforms per step)" % (ntt["units"] / a.steps),
                     "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                     "traffic_source": tsrc, "traffic_over_algorithmic": t_over_a, "peak_source": peak_src,
                     "algorithmic_bytes": "per launch: 16 N per limb transform (split over its passes) + the operand "
                                          "limbs of its fused prologue / epilogue (%.1f MB per step of the %.1f MB)" % (
                                              ops["bytes"] / a.steps / 1e6,
                                              (ntt["bytes"] + ops["bytes"]) / a.steps / 1e6),
                     "algorithmic_bytes_per_limb_transform": 16 * ctx.N,
                     "achieved_transform_only": ach_t, "frac_transform_only": ach_t / peak,
                     "share_of_step": ntt["ms"] / ms_prof,
                     "fp64_pipe": {"achieved": fp64_ach, "peak": fp64_peak, "unit": "T FP64 instr/s",
                                   "frac": fp64_ach / fp64_peak,
                                   "peak_source": "148 SMs x 64 FP64 lanes/clk x %.0f MHz (sampled)" % clk_mhz},
                     "profiled_region": "second timed region of the same %d steps, one stream, CUDA events around "
                                        "every NTT launch and key-switch / rescale span" % a.steps,
                     "ntt_integer_rows": ({"achieved": gbs(ntt_int), "frac": gbs(ntt_int) / peak,
                                           "share_of_step": ntt_int["ms"] / ms_prof, "unit": "GB/s",
                                           "bound": "integer FMA pipe (quarter-rate IMAD.WIDE)"}
                                          if ntt_int["ms"] > 0 else "none: every prime of Q u P is < 2^46 (R24)"),
                     "keyswitch": {"achieved": ks_ach, "frac": ks_ach / peak, "share_of_step": ks["ms"] / ms_prof,
                                   "unit": "GB/s"},
                     # the same figures as flat fields (nested objects are not kept by every reader)
                     "keyswitch_achieved_gbs": ks_ach, "keyswitch_frac": ks_ach / peak,
                     "keyswitch_share_of_step": ks["ms"] / ms_prof,
                     "fp64_pipe_frac": fp64_ach / fp64_peak,
                     "rescale_share_of_step": prof["rescale"]["ms"] / ms_prof,
                     # whole step: real DRAM bytes of all its launches (ncu) over the measured step time
                     **({**step_dram, "step_dram_frac": step_dram["step_dram_gbs"] / peak} if step_dram else {})},
        "stage_share_of_step": {k[6:]: v["ms"] / ms_prof for k, v in prof.items() if k.startswith("stage_")},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h_in.numel() * 8),
                "d2h_bytes_per_step": int(h_out.numel() * 8)},
        "gpu_launches": int(counts["launches"]),
        "accuracy": accuracy,
        "op_counts_per_step": {k: v / a.steps for k, v in counts.items()},
        "clocks": clk,
    }
    if ws == 1 and not a.no_micro:
        # BASELINE configs[1]-[3] and the SURVEY 8(f) rows built beyond the hot path (N3 bootstrapping, N4
        # argmax with bootstrapping), each with its own parity tests
        line["configs_1_to_3"], line["next_rows"] = micro_configs(stream)
        c = line["configs_1_to_3"]
        rf = line["roofline"]
        rf["configs1_ntt_gbs"] = c["configs[1]_ntt"]["alg_gbs"]
        rf["configs1_ntt_frac"] = c["configs[1]_ntt"]["frac_of_hbm"]
        rf["configs1_ntt_bound"] = "alu"
        rf["configs1_ntt_issue_slot_frac"] = c["configs[1]_ntt"]["frac_of_issue_slots"]
        rf["configs2_mul_relin_rescale_gbs"] = c["configs[2]_mul_relin_rescale"]["alg_gbs"]
        rf["configs2_mul_relin_rescale_frac"] = c["configs[2]_mul_relin_rescale"]["frac_of_hbm"]
        rf["configs3_rotation_gbs"] = c["configs[3]_rotation"]["alg_gbs"]
        rf["configs3_rotation_frac"] = c["configs[3]_rotation"]["frac_of_hbm"]
        line["configs4_49bit"] = argmax49_bench(stream)
    if ws == 1 and not a.no_cpu_baseline:
        ora = OracleArgmax()
        dt, q, cores = ora.run()
        line["cpu_baseline"] = cpu_baseline_line(ora, dt, q, cores)
    print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=16, help="ciphertexts per rank per step")
    ap.add_argument("--impl", default="secpe", choices=["secpe", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-micro", action="store_true", help="skip the configs[1]-[3] lines")
    ap.add_argument("--ncu", action="store_true", help="run one profiled step (for ncu --profile-from-start off)")
    ap.add_argument("--ref-warmup", action="store_true", help="also run oracle warm-up steps (reference arm)")
    a = ap.parse_args()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_secpe(a)


if __name__ == "__main__":
    main()
