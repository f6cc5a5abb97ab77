"""Seeded synthetic workloads shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method: only workload shapes (BASELINE.json
configs, restated as data) and numpy PCG64 random draws.  Prime chains, NTT tables,
encodings, packing and every homomorphic step are implemented separately by
``oracle/`` and by ``paper_2502_00847_b200/``.

Recipe: per-prompt logits ~ N(0, sigma=2) iid per
(query, prompt, class), softmax over classes -> scores in [0, 1]; the toy config draws
scores ~ U[0,1] and keeps a query only if its mean-over-prompts top-1 gap is >= 0.1.
"""
import numpy as np

# Parameter sets.  Prime segments: (mode, bits, count); mode "nearest" = primes == 1 mod 2N
# closest to 2^bits alternating above/below; "below" = largest primes below 2^bits,
# descending.  Every segment excludes the primes generated before it (q first, then p).
PARAM_SETS = {
    # BASELINE configs[0]: 8 x 40-bit primes + 1 special 50-bit prime, scale 2^40, N = 2^12.
    "toy": dict(logn=12, q=[("nearest", 40, 8)], p=[("below", 50, 1)], alpha=1, log_scale=40),
    # Same ring with a 17-prime chain for the end-to-end toy argmax (reading R20).
    "toy_argmax": dict(logn=12, q=[("nearest", 40, 17)], p=[("below", 50, 1)], alpha=1, log_scale=40),
    # Tiny ring for fast CPU pins of every primitive (not a BASELINE config).
    "tiny": dict(logn=6, q=[("nearest", 30, 4)], p=[("below", 31, 2)], alpha=2, log_scale=25),
    "tiny_deep": dict(logn=8, q=[("below", 60, 1), ("nearest", 40, 16)], p=[("below", 61, 2)],
                      alpha=3, log_scale=40),
    # configs[4]'s prime structure on a 2^12 ring: CPU-sized check of the (7,15,15) circuit numerics.
    "argmax_small": dict(logn=12, q=[("nearest", 45, 30)], p=[("below", 46, 10)],
                         alpha=10, log_scale=45),
    # Bootstrapping (readings R32-R35): q_0 ~ 2^60 over scale 2^50 (R = q_0 / S ~ 2^10),
    # a 50-bit chain long enough for one bootstrap (8 + r levels) plus a few, 8 special primes below 2^50
    # (alpha = 7: P ~ 2^400 > every 7-prime digit <= 2^360; reading R40: ~50-bit special primes keep every
    # key-switching row except q_0 on the exact-FP64 NTT).  boot_tiny: CPU-sized (oracle pins); boot: the smallest ring the
    # library takes (N = 2^12, 2048 slots, BSGS 64 x 32).
    "boot_tiny": dict(logn=8, q=[("below", 60, 1), ("nearest", 50, 18)], p=[("below", 50, 8)],
                      alpha=7, log_scale=50),
    "boot": dict(logn=12, q=[("below", 60, 1), ("nearest", 50, 20)], p=[("below", 50, 8)],
                 alpha=7, log_scale=50),
    # N4 (reading R38): argmax with bootstrapping.  Levels 1..16 are 45-bit primes at the nominal scale 2^45
    # (the Sign polynomials' constants, up to 2^14.8, need Delta_c ~ q <= 2^47); the 19 levels above are
    # 50-bit primes for the bootstrap (ModRaise to the top, EvalMod at scale 2^50).  A refresh lands at
    # level 16: one normalisation, one Max (14 levels), one level left for the next refresh's scale-up.
    "boot_argmax_tiny": dict(logn=8, q=[("below", 60, 1), ("nearest", 45, 16), ("nearest", 50, 17)],
                             p=[("below", 50, 8)], alpha=7, log_scale=45),
    "boot_argmax": dict(logn=12, q=[("below", 60, 1), ("nearest", 45, 16), ("nearest", 50, 19)],
                        p=[("below", 50, 8)], alpha=7, log_scale=45),
    "boot_argmax16": dict(logn=16, q=[("below", 60, 1), ("nearest", 45, 16), ("nearest", 50, 19)],
                          p=[("below", 50, 8)], alpha=7, log_scale=45),
    # the same with two more bootstrap levels, for four stage groups (3/4/4/4: fewer key switches per group)
    "boot_argmax16_g4": dict(logn=16, q=[("below", 60, 1), ("nearest", 45, 16), ("nearest", 50, 21)],
                             p=[("below", 50, 8)], alpha=7, log_scale=45),
    # N = 2^12 analogues of the four-group chains (groups 2/3/3/3: depth 21): a standalone bootstrap chain and
    # boot_argmax16_g4's structure on the small ring (word-for-word parity of the bench's four-group plans)
    "boot_g4": dict(logn=12, q=[("below", 60, 1), ("nearest", 50, 22)], p=[("below", 50, 8)],
                    alpha=7, log_scale=50),
    "boot_argmax_g4": dict(logn=12, q=[("below", 60, 1), ("nearest", 45, 16), ("nearest", 50, 21)],
                           p=[("below", 50, 8)], alpha=7, log_scale=45),
    # the paper's ring (N = 2^16, 32768 slots) with the factorised transforms (R37, groups 5/5/5: depth 20)
    "boot16": dict(logn=16, q=[("below", 60, 1), ("nearest", 50, 22)], p=[("below", 50, 8)],
                   alpha=7, log_scale=50),
    # configs[4] at the paper's prime size (log Q = 1763 over L = 35 levels, ~49-bit primes; reading
    # R41): 30 chain primes nearest 2^49 at scale 2^49, 10 special primes below 2^50 (P ~ 2^500 > every 10-prime
    # digit ~ 2^490); every row of Q u P takes the FP64 NTT with reductions (FpB) at N >= 2^15
    "argmax49": dict(logn=16, q=[("nearest", 49, 30)], p=[("below", 50, 10)], alpha=10, log_scale=49),
    "argmax_small49": dict(logn=12, q=[("nearest", 49, 30)], p=[("below", 50, 10)], alpha=10, log_scale=49),
    # BASELINE configs[1]: NTT microbench, 24 x 60-bit primes, N = 2^16.
    "ntt": dict(logn=16, q=[("below", 60, 24)], p=[], alpha=8, log_scale=50),
    # BASELINE configs[2]/[3]: 24 x 60-bit q, dnum = 3 -> alpha = 8, 8 special 60-bit primes, scale 2^50.
    "ks": dict(logn=16, q=[("below", 60, 24)], p=[("below", 60, 8)], alpha=8, log_scale=50),
    # BASELINE configs[4]: q_0..q_29 ~ 2^45 (reading R23), dnum = 3 (alpha = 10), scale 2^45, 10 special
    # primes below 2^46 (reading R24: P ~ 2^460 > every 10-prime digit ~ 2^450, and every row of Q u P
    # takes the exact-FP64 NTT).
    "argmax": dict(logn=16, q=[("nearest", 45, 30)], p=[("below", 46, 10)],
                   alpha=10, log_scale=45),
}

# SecPE layouts ("2n slots per argmax"; BASELINE configs[4]):
# query q, prompt p, class k -> slot q*block + p*K + k.
LAYOUTS = {
    "toy": dict(queries=1, prompts=4, classes=4, block=16),
    "argmax_k2": dict(queries=2048, prompts=8, classes=2, block=16),
    "argmax_k16": dict(queries=256, prompts=8, classes=16, block=128),
    "argmax_small_k2": dict(queries=128, prompts=8, classes=2, block=16),
    "tiny_k16": dict(queries=1, prompts=8, classes=16, block=128),
    "boot_k16": dict(queries=16, prompts=8, classes=16, block=128),
    # SURVEY 8(f) N4 "n = 256 with 64 per ciphertext" (2n slots per argmax): 256 classes, 2 prompts
    "argmax_n256": dict(queries=64, prompts=2, classes=256, block=512),
    "boot_n256": dict(queries=4, prompts=2, classes=256, block=512),
    # CLIP scale (80 / 247 prompts, 1000 classes padded to 1024): 2 prompts per
    # ciphertext, the rest spread over several ciphertexts summed first (prompt_cts)
    "clip": dict(queries=16, prompts=2, classes=1024, block=2048),
    "boot_clip": dict(queries=1, prompts=2, classes=1024, block=2048),
}

KEY_SEED_BASE = 0x5EC9E000


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def softmax_scores(seed, queries, prompts, classes, sigma=2.0):
    """Per-prompt class scores: logits ~ N(0, sigma) iid, softmax over classes. Shape (q, P, K)."""
    g = rng(seed)
    logits = g.normal(0.0, sigma, size=(queries, prompts, classes))
    e = np.exp(logits - logits.max(axis=2, keepdims=True))
    return e / e.sum(axis=2, keepdims=True)


def ensemble_scores(seed, queries, prompts, classes, sigma_class=4.0, sigma_prompt=1.0):
    """Prompt-ensemble scores with agreeing prompts (the CLIP setting): logits = a per-(query,
    class) consensus ~ N(0, sigma_class) + per-prompt noise ~ N(0, sigma_prompt), softmax over classes."""
    g = rng(seed)
    base = g.normal(0.0, sigma_class, size=(queries, 1, classes))
    logits = base + g.normal(0.0, sigma_prompt, size=(queries, prompts, classes))
    e = np.exp(logits - logits.max(axis=2, keepdims=True))
    return e / e.sum(axis=2, keepdims=True)


def toy_scores(seed, queries, prompts, classes, gap=0.1):
    """Scores ~ U[0,1]; keep a query only if its mean-over-prompts top-1 gap >= gap (rejection)."""
    g = rng(seed)
    out = np.empty((queries, prompts, classes))
    i = 0
    while i < queries:
        s = g.uniform(0.0, 1.0, size=(prompts, classes))
        m = np.sort(s.mean(axis=0))
        if m[-1] - m[-2] >= gap:
            out[i] = s
            i += 1
    return out


def uniform_residues(seed, primes, n_polys, logn):
    """uint64 array (n_polys, len(primes), 2^logn), limb l uniform in [0, primes[l])."""
    g = rng(seed)
    n = 1 << logn
    out = np.empty((n_polys, len(primes), n), dtype=np.uint64)
    for l, q in enumerate(primes):
        out[:, l, :] = g.integers(0, int(q), size=(n_polys, n), dtype=np.uint64)
    return out


def uniform_slots(seed, n, lo=-1.0, hi=1.0):
    return rng(seed).uniform(lo, hi, size=n)
