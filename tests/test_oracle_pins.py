"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU needed).

Every check here recomputes the expected value by an independent route (Python big integers,
sympy/mpmath, schoolbook products, closed forms, brute force on tiny inputs) -- never by
re-calling the oracle routine under test.
"""
import json
import math
import os

import numpy as np
import pytest
import sympy
import mpmath

import synth
from oracle import ckks, plan

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "paper_examples.json")))


@pytest.fixture(scope="module")
def tiny():
    return ckks.Params(synth.PARAM_SETS["tiny"])


@pytest.fixture(scope="module")
def toy():
    return ckks.Params(synth.PARAM_SETS["toy"])


def brv(x, bits):
    return int(format(x, "0%db" % bits)[::-1], 2)


# ---------------------------------------------------------------------------------------------
# O-1 primes, O-3 psi
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tiny", "toy", "toy_argmax", "ks", "argmax"])
def test_prime_chain(name):
    d = synth.PARAM_SETS[name]
    logn = d["logn"]
    two_n = 2 << logn
    primes = []
    for segs in (d["q"], d["p"]):
        for mode, bits, cnt in segs:
            # independent walk with sympy primality
            base, got, k = 1 << bits, [], 0
            while len(got) < cnt:
                cands = [base + 1 + k * two_n, base + 1 - (k + 1) * two_n] if mode == "nearest" else \
                        [base + 1 - (k + 1) * two_n]
                for c in cands:
                    if len(got) < cnt and sympy.isprime(c) and c not in primes and c not in got:
                        got.append(c)
                k += 1
            primes += got
    assert ckks.Params(d).primes == primes
    for q in primes:
        assert q % two_n == 1 and q < 2 ** 62


@pytest.mark.parametrize("q,logn", [(7681, 8), (12289, 10), (257, 7), (65537, 12)])
def test_psi_is_smallest_root_bruteforce(q, logn):
    n = 1 << logn
    want = min(x for x in range(2, q) if pow(x, n, q) == q - 1)
    assert ckks.lib().o_find_psi(q, logn) == want


def test_psi_real_primes(toy):
    for q, psi in zip(toy.primes[:3], toy.psi[:3]):
        n = toy.N
        assert pow(psi, n, q) == q - 1
        g = sympy.primitive_root(q)
        r = pow(g, (q - 1) // (2 * n), q)
        r2 = r * r % q
        roots, cur = [], r
        for _ in range(n):
            roots.append(cur)
            cur = cur * r2 % q
        assert psi == min(roots)


# ---------------------------------------------------------------------------------------------
# O-3 NTT
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("logn", [3, 4, 6])
def test_ntt_definition_bigint(logn):
    q = 7681 if logn <= 7 else 12289
    n = 1 << logn
    psi = ckks.lib().o_find_psi(q, logn)
    a = np.random.default_rng(logn).integers(0, q, n).astype(np.uint64)
    want = [sum(int(a[k]) * pow(psi, (2 * brv(i, logn) + 1) * k, q) for k in range(n)) % q for i in range(n)]
    assert [int(v) for v in ckks.ntt(a, q, psi, logn)] == want


def test_ntt_roundtrip_and_convolution(toy):
    rng = np.random.default_rng(5)
    for logn, q in [(6, 7681), (8, 7681)]:
        n = 1 << logn
        psi = ckks.lib().o_find_psi(q, logn)
        a = rng.integers(0, q, n).astype(np.uint64)
        b = rng.integers(0, q, n).astype(np.uint64)
        assert np.array_equal(ckks.intt(ckks.ntt(a, q, psi, logn), q, psi, logn), a)
        # schoolbook negacyclic product mod (X^N + 1, q)
        c = [0] * n
        for i in range(n):
            for j in range(n):
                v = int(a[i]) * int(b[j])
                if i + j < n:
                    c[i + j] += v
                else:
                    c[i + j - n] -= v
        c = [x % q for x in c]
        A, B = ckks.ntt(a, q, psi, logn), ckks.ntt(b, q, psi, logn)
        prod = np.array([(int(x) * int(y)) % q for x, y in zip(A, B)], dtype=np.uint64)
        assert [int(v) for v in ckks.intt(prod, q, psi, logn)] == c
    # full-size round trip on a 40-bit toy prime
    q, psi = toy.primes[0], toy.psi[0]
    a = rng.integers(0, q, toy.N).astype(np.uint64)
    assert np.array_equal(ckks.intt(ckks.ntt(a, q, psi, toy.logn), q, psi, toy.logn), a)


# ---------------------------------------------------------------------------------------------
# O-6 sampler
# ---------------------------------------------------------------------------------------------
CHACHA = json.load(open(os.path.join(HERE, "golden", "chacha20.json")))


def _keystream(key_words, counter, nonce, nbytes=64):
    """Independent ChaCha20 (the `cryptography` package): its 16-byte nonce is state words 12-15."""
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms
    iv = int(counter).to_bytes(8, "little") + int(nonce).to_bytes(8, "little")
    key = np.asarray(key_words, dtype="<u4").tobytes()
    return Cipher(algorithms.ChaCha20(key, iv), mode=None).encryptor().update(bytes(nbytes))


def test_chacha20_block_vectors():
    """R6 sampler core: the oracle's ChaCha20 block equals the RFC 7539 test vectors
    (tests/golden/chacha20.json) and an independent implementation on random keys/counters/nonces."""
    for v in CHACHA["vectors"]:
        key = np.frombuffer(bytes.fromhex(v["key_hex"]), dtype="<u4")
        got = ckks.chacha20_block(key, v["counter"], v["nonce"]).astype("<u4").tobytes()
        assert got.hex() == v["block_hex"], v["source"]
    rng = np.random.default_rng(5)
    for _ in range(8):
        key = rng.integers(0, 1 << 32, 8, dtype=np.uint64).astype(np.uint32)
        ctr, nonce = int(rng.integers(0, 1 << 63)), int(rng.integers(0, 1 << 63))
        got = ckks.chacha20_block(key, ctr, nonce).astype("<u4").tobytes()
        assert got == _keystream(key, ctr, nonce)


def test_chacha_streams_and_key_domains():
    """draw ctr = 64-bit word ctr mod 8 of block ctr / 8 of the object's stream (nonce = tag); object keys are
    the first 32 bytes of block 0 under the master seed with nonce DOM_SK (secret material: s, e; tags 1, 3, 5),
    DOM_PK (public material: the uniform a of pk / switching keys; tags 2, 4) or DOM_ENC (encryption)."""
    L = ckks.lib()
    master = ckks.seed_key(0x1234567890ABCDEF)
    assert list(master[:2]) == [0x90ABCDEF, 0x12345678] and not master[2:].any()
    assert np.array_equal(ckks.seed_key(bytes(range(32))), np.frombuffer(bytes(range(32)), dtype="<u4"))
    doms = {1: 0x5345435045534B31, 3: 0x5345435045534B31, 5: 0x5345435045534B31,
            2: 0x5345435045504B31, 4: 0x5345435045504B31}
    for kind, dom in doms.items():
        tag = L.o_tag(kind, 5, 2)
        assert tag == (kind << 48) ^ (5 << 8) ^ 2
        k = ckks.object_key(master, tag)
        assert k.astype("<u4").tobytes() == _keystream(master, 0, dom)[:32], kind
        ks = _keystream(k, 0, tag, 128)
        for ctr in range(16):
            want = int.from_bytes(ks[8 * ctr: 8 * ctr + 8], "little")
            assert L.o_draw(k.ctypes.data_as(ckks.u32p), tag, ctr) == want
    ke = np.zeros(8, dtype=np.uint32)
    L.o_encrypt_key(master.ctypes.data_as(ckks.u32p), ke.ctypes.data_as(ckks.u32p))
    assert ke.astype("<u4").tobytes() == _keystream(master, 0, 0x5345435045454E31)[:32]
    # public and secret material never share a stream key
    assert not np.array_equal(ckks.object_key(master, L.o_tag(1, 0, 0)), ckks.object_key(master, L.o_tag(2, 0, 0)))


def test_cdt_table_mpmath():
    mpmath.mp.prec = 200
    sigma = mpmath.mpf(16) / 5
    rho = [mpmath.exp(-mpmath.mpf(j * j) / (2 * sigma ** 2)) for j in range(20)]
    tot = rho[0] + 2 * sum(rho[1:])
    acc, want = mpmath.mpf(0), []
    for m in range(20):
        acc += rho[m] if m == 0 else 2 * rho[m]
        want.append(int(mpmath.floor(mpmath.mpf(2) ** 63 * acc / tot)))
    want[-1] = 1 << 63
    assert [int(v) for v in ckks.cdt_table()] == want


def test_sampler_moments(toy):
    L = ckks.lib()
    n = 1 << 16
    k7 = ckks.seed_key(7)
    K = k7.ctypes.data_as(ckks.u32p)
    t = np.zeros(n, dtype=np.int64)
    L.o_sample_ternary(K, 99, 16, ckks.P(t))
    counts = np.bincount(t + 1, minlength=3)
    chi2 = ((counts - n / 3) ** 2 / (n / 3)).sum()
    assert set(np.unique(t)) <= {-1, 0, 1} and chi2 < 20
    e = np.zeros(n, dtype=np.int64)
    L.o_sample_gauss(K, 98, 16, ckks.P(toy.cdt), len(toy.cdt), ckks.P(e))
    assert abs(e.mean()) < 0.05 and abs(e.std() - 3.2) < 0.05 and np.abs(e).max() <= 19
    # exact discrete Gaussian pmf vs histogram (chi^2 over |e| <= 8)
    rho = np.exp(-np.arange(-19, 20) ** 2 / (2 * 3.2 ** 2))
    p = rho / rho.sum()
    hist = np.array([(e == v).sum() for v in range(-8, 9)])
    exp = n * p[19 - 8: 19 + 9]
    assert ((hist - exp) ** 2 / exp).sum() < 60
    # uniform mod q: mean and bucket chi^2
    q = toy.primes[0]
    u = np.array([L.o_uniform(K, 5, 0, k, 12, q) for k in range(4096)], dtype=np.float64)
    assert u.max() < q and abs(u.mean() / q - 0.5) < 0.02
    h = np.histogram(u / q, bins=16, range=(0, 1))[0]
    assert ((h - 256) ** 2 / 256).sum() < 45


# ---------------------------------------------------------------------------------------------
# O-7 keys, O-8 encryption
# ---------------------------------------------------------------------------------------------
def ntt_def(vals, q, psi, logn):
    n = 1 << logn
    return [sum(int(vals[k]) * pow(psi, (2 * brv(i, logn) + 1) * k, q) for k in range(n)) % q for i in range(n)]


def test_switching_key_gadget_identity(tiny):
    """b_j + a_j s - e_j == [P]_t s' [t in D_j]   (Python big ints, NTT by definition)."""
    prm, ev = tiny, ckks.Oracle(tiny)
    keys = ev.keygen(11, [1])
    L = ckks.lib()
    N, ne = prm.N, prm.nq + prm.np_
    # the secret itself: ternary stream, NTT by definition
    master = ckks.seed_key(11)
    ks = ckks.object_key(master, L.o_tag(1, 0, 0))
    s = np.zeros(N, dtype=np.int64)
    L.o_sample_ternary(ks.ctypes.data_as(ckks.u32p), L.o_tag(1, 0, 0), prm.logn, ckks.P(s))
    for t in range(ne):
        q = prm.primes[t]
        assert [int(v) for v in keys.s_ntt[t]] == ntt_def([int(x) % q for x in s], q, prm.psi[t], prm.logn)
    P_ = 1
    for p in prm.p:
        P_ *= p
    for j in range(prm.beta(prm.L)):
        e = np.zeros(N, dtype=np.int64)
        ke = ckks.object_key(master, L.o_tag(5, 0, j))
        L.o_sample_gauss(ke.ctypes.data_as(ckks.u32p), L.o_tag(5, 0, j), prm.logn, ckks.P(prm.cdt), len(prm.cdt),
                         ckks.P(e))
        for t in range(ne):
            q = prm.primes[t]
            en = ntt_def([int(x) % q for x in e], q, prm.psi[t], prm.logn)
            b, a = keys.rlk[j, 0, t], keys.rlk[j, 1, t]
            lhs = [(int(b[k]) + int(a[k]) * int(keys.s_ntt[t, k]) - en[k]) % q for k in range(N)]
            in_digit = t < prm.nq and t // prm.alpha == j
            rhs = [((P_ % q) * int(keys.s_ntt[t, k]) ** 2) % q if in_digit else 0 for k in range(N)]
            assert lhs == rhs


def test_encrypt_decrypt(toy):
    ev = ckks.Oracle(toy)
    keys = ev.keygen(3)
    z = synth.uniform_slots(1, toy.N // 2)
    ct = ev.encrypt(keys, z, toy.scale, 9)
    assert np.abs(ev.decrypt(keys, ct).real - z).max() < 2 ** -20
    # bit-level: decrypt_int - m is the small encryption noise
    m = ckks.encode(toy, z, toy.scale)
    noise = ev.decrypt_int(keys, ct) - m.astype(object)
    assert max(abs(int(v)) for v in noise) < 2 ** 14


# ---------------------------------------------------------------------------------------------
# O-9..O-12 homomorphic ops
# ---------------------------------------------------------------------------------------------
def test_rescale_exact_bigint(tiny):
    prm = tiny
    rng = np.random.default_rng(2)
    nl = prm.nq
    data = np.stack([np.stack([rng.integers(0, q, prm.N).astype(np.uint64) for q in prm.q]) for _ in range(2)])
    ct = ckks.Ct(data, 1.0)
    out = ckks.Oracle(prm).rescale(ct)
    ids = list(range(nl))
    coef = ckks.ntt_limbs(data, prm, ids, inverse=True)
    coef_out = ckks.ntt_limbs(out.data, prm, ids[:-1], inverse=True)
    Q = 1
    for q in prm.q:
        Q *= q
    ql = prm.q[-1]
    Qd = Q // ql
    for b in range(2):
        for k in range(prm.N):
            c = 0
            for i in range(nl):  # CRT, independent of the oracle's crt_centered
                Qi = Q // prm.q[i]
                c += int(coef[b, i, k]) * Qi * pow(Qi, -1, prm.q[i])
            c %= Q
            want = ((c + ql // 2) // ql) % Qd
            for i in range(nl - 1):
                assert int(coef_out[b, i, k]) == want % prm.q[i]


def _centered(x, Q):
    x %= Q
    return x - Q if x > Q // 2 else x


def test_keyswitch_bigint_bound(tiny):
    """<KS(d), (1, s)> - d s^2 is small mod Q_l (reading R10/R11), checked with big ints."""
    prm, ev = tiny, ckks.Oracle(tiny)
    keys = ev.keygen(4)
    rng = np.random.default_rng(8)
    for level in (prm.L, prm.L - 1):
        nl = level + 1
        d = np.stack([rng.integers(0, q, prm.N).astype(np.uint64) for q in prm.q[:nl]])
        ks = ev.keyswitch(d, keys.rlk)
        Q = 1
        for q in prm.q[:nl]:
            Q *= q
        ids = list(range(nl))
        # err = ks0 + ks1 s - d s^2  in NTT form, then back to coefficients
        err = np.zeros((nl, prm.N), dtype=np.uint64)
        for i, q in enumerate(prm.q[:nl]):
            s = [int(v) for v in keys.s_ntt[i]]
            err[i] = [(int(ks[0, i, k]) + int(ks[1, i, k]) * s[k] - int(d[i, k]) * s[k] * s[k]) % q
                      for k in range(prm.N)]
        ec = ckks.ntt_limbs(err, prm, ids, inverse=True)
        for k in range(prm.N):
            x = 0
            for i in range(nl):
                Qi = Q // prm.q[i]
                x += int(ec[i, k]) * Qi * pow(Qi, -1, prm.q[i])
            assert abs(_centered(x, Q)) < 2 ** 20


def test_wide_constants_big_int(tiny):
    """Constant products and additions with |C| >= 2^63 (reading R41: C = rha(c Delta_c) ~ 2^64 at 49-bit
    primes): every residue equals Python's big-int a C mod q and (a + C) mod q; wide_int splits into two's
    complement words; constants at the 2^120 limit raise."""
    prm, ev = tiny, ckks.Oracle(tiny)
    rng = np.random.default_rng(41)
    nl = prm.L + 1
    a = ckks.Ct(np.stack([np.stack([rng.integers(0, q, prm.N).astype(np.uint64) for q in prm.q[:nl]])
                          for _ in range(2)]), prm.scale)
    for C in (2 ** 64 + 12345, -(2 ** 64) - 7, 2 ** 100 - 3, -(2 ** 119), 2 ** 63, -(2 ** 63) - 1, 5, -5):
        hi, lo = ckks.wide_int(C)
        assert hi * 2 ** 64 + lo == C and 0 <= lo < 2 ** 64 and -(2 ** 63) <= hi < 2 ** 63
        m = ev.mul_int_raw(a, C)
        s = ev.add_int_raw(a, C)
        for l, q in enumerate(prm.q[:nl]):
            for k in (0, 1, prm.N - 1):
                for p_ in (0, 1):
                    assert int(m[p_, l, k]) == int(a.data[p_, l, k]) * C % q
                assert int(s[0, l, k]) == (int(a.data[0, l, k]) + C) % q
                assert int(s[1, l, k]) == int(a.data[1, l, k])
    with pytest.raises(OverflowError):
        ev.mul_int_raw(a, 2 ** 120)


def test_ops_against_slots(toy):
    ev = ckks.Oracle(toy)
    keys = ev.keygen(5, [1, -1, 3])
    z1 = synth.uniform_slots(11, toy.N // 2)
    z2 = synth.uniform_slots(12, toy.N // 2)
    a = ev.encrypt(keys, z1, toy.scale, 1)
    b = ev.encrypt(keys, z2, toy.scale, 2)
    tol = 2 ** -10
    assert np.abs(ev.decrypt(keys, ev.add_raw(a, b)).real - (z1 + z2)).max() < tol
    assert np.abs(ev.decrypt(keys, ev.sub_raw(a, b)).real - (z1 - z2)).max() < tol
    m = ev.rescale(ev.mul_relin(keys, a, b))
    assert np.abs(ev.decrypt(keys, m).real - z1 * z2).max() < tol
    # planned product with a linear term joined before the rescale (R13): a b + 0.25 a
    f = ev.mul_ct(keys, a, b, toy.scale, a.level - 1, lin=(a, 0.25))
    assert f.level == a.level - 1 and f.scale == toy.scale
    assert np.abs(ev.decrypt(keys, f).real - (z1 * z2 + 0.25 * z1)).max() < tol
    # two summed products with one relinearisation and rescale (R13b): a b + b b - 0.5 a
    f2 = ev.mul_ct(keys, a, b, toy.scale, a.level - 1, lin=(a, -0.5), prod2=(b, b))
    assert f2.level == a.level - 1 and f2.scale == toy.scale
    assert np.abs(ev.decrypt(keys, f2).real - (z1 * z2 + z2 * z2 - 0.5 * z1)).max() < tol
    # ... and its integers equal the relinearisation of the summed tensors written out (O-10 on d + d')
    lv = a.level
    d = ev.tensor(a, b)
    dd = ev.tensor(b, b)
    dsum = ((d.astype(object) + dd.astype(object)) % np.array(toy.primes[:lv + 1], dtype=object)[None, :, None]).astype(np.uint64)
    C = ckks.round_half_away(-0.5 * ((toy.scale * float(toy.primes[lv])) / a.scale))
    ca = ev.mul_int_raw(a, C)
    dsum[:2] = ((dsum[:2].astype(object) + ca.astype(object)) % np.array(toy.primes[:lv + 1], dtype=object)[None, :, None]).astype(np.uint64)
    manual = ev.rescale(ev.mul_relin(keys, a, b, dsum), toy.scale)
    assert np.array_equal(manual.data, f2.data)
    for s in (1, -1, 3):
        r = ev.rotate_raw(keys, a, s)
        assert np.abs(ev.decrypt(keys, r).real - np.roll(z1, -s)).max() < tol
    # RotL o RotR = id and additive composition RotL(RotL(a,1),... )
    back = ev.rotate_raw(keys, ev.rotate_raw(keys, a, 1), -1)
    assert np.abs(ev.decrypt(keys, back).real - z1).max() < tol
    # golden: RotL([a0..a3], 1) = [a1, a2, a3, a0]
    g = GOLD["rotation_direction"]
    v = np.zeros(toy.N // 2)
    v[:4] = g["vector"]
    v[4:] = 0
    v4 = np.array(g["vector"], dtype=float)
    full = np.tile(v4, toy.N // 8)
    r = ev.rotate_raw(keys, ev.encrypt(keys, full, toy.scale, 3), g["steps"])
    assert np.allclose(ev.decrypt(keys, r).real[:4], g["rotl"], atol=tol)
    # planned ops: mul_const lands exactly on the target scale and level
    y = ev.mul_const(a, 0.75, toy.scale, a.level - 2)
    assert y.level == a.level - 2 and y.scale == toy.scale
    assert np.abs(ev.decrypt(keys, y).real - 0.75 * z1).max() < tol
    w = ev.add_const(a, -0.5)
    assert np.abs(ev.decrypt(keys, w).real - (z1 - 0.5)).max() < tol


def _ntt_sigma(vals, g, logn):
    """NTT-domain sigma_g by the evaluation-point identity NTT(sigma_g a)[i] = NTT(a)[j] with
    2 brv(j) + 1 = g (2 brv(i) + 1) mod 2N (R4 ordering), independent of o_automorph."""
    n = 1 << logn
    out = [0] * n
    for i in range(n):
        e = (g * (2 * brv(i, logn) + 1)) % (2 * n)
        out[i] = int(vals[brv((e - 1) // 2, logn)])
    return out


def test_hoisted_keyswitch_bigint_bound(tiny):
    """N2 hoisted key switch (reading R29): <KS_g(d), (1, s)> - sigma_g(d) sigma_g(s) is small mod Q_l,
    with sigma_g taken by its evaluation-point definition and the CRT lift in Python big ints; and the
    integers differ from the non-hoisted KS(sigma_g(d)) (O-12: ModUp does not commute with sigma_g)."""
    prm, ev = tiny, ckks.Oracle(tiny)
    keys = ev.keygen(4, [1, 3])
    L = ckks.lib()
    rng = np.random.default_rng(18)
    for steps in (1, 3):
        g = ckks.galois_elt(prm, steps)
        for level in (prm.L, prm.L - 1):
            nl = level + 1
            d = np.stack([rng.integers(0, q, prm.N).astype(np.uint64) for q in prm.q[:nl]])
            ks = np.zeros((2, nl, prm.N), dtype=np.uint64)
            L.o_keyswitch_g(prm.cptr, ckks.P(np.ascontiguousarray(d)), nl, ckks.P(keys.gk[g]), g, ckks.P(ks))
            Q = 1
            for q in prm.q[:nl]:
                Q *= q
            err = np.zeros((nl, prm.N), dtype=np.uint64)
            for i, q in enumerate(prm.q[:nl]):
                s = [int(v) for v in keys.s_ntt[i]]
                sg, dg = _ntt_sigma(keys.s_ntt[i], g, prm.logn), _ntt_sigma(d[i], g, prm.logn)
                err[i] = [(int(ks[0, i, k]) + int(ks[1, i, k]) * s[k] - dg[k] * sg[k]) % q for k in range(prm.N)]
            ec = ckks.ntt_limbs(err, prm, list(range(nl)), inverse=True)
            for k in range(prm.N):
                x = 0
                for i in range(nl):
                    Qi = Q // prm.q[i]
                    x += int(ec[i, k]) * Qi * pow(Qi, -1, prm.q[i])
                assert abs(_centered(x, Q)) < 2 ** 20
            dsig = np.stack([np.array(_ntt_sigma(d[i], g, prm.logn), dtype=np.uint64) for i in range(nl)])
            assert not np.array_equal(ks, ev.keyswitch(dsig, keys.gk[g]))


def test_hoisted_rotations_against_slots(toy):
    """N2: one ModUp shared by several rotation steps; every output decrypts to RotL(z, step)."""
    ev = ckks.Oracle(toy)
    steps = [1, 2, 4, -1, 0]
    keys = ev.keygen(5, [s for s in steps if s])
    z = synth.uniform_slots(31, toy.N // 2)
    a = ev.encrypt(keys, z, toy.scale, 1)
    outs = ev.rotate_hoisted_raw(keys, a, steps)
    for s, r in zip(steps, outs):
        assert r.level == a.level and r.scale == a.scale
        assert np.abs(ev.decrypt(keys, r).real - np.roll(z, -s)).max() < 2 ** -10
    assert np.array_equal(outs[-1].data, a.data)  # step 0: identity


def test_linear_transform_against_matrix(toy):
    """R30: the hoisted diagonal-form linear transform decrypts to the plaintext matrix-vector product
    y[t] = sum_i d_i[t] z[t + s_i] (numpy, independent of the oracle's arithmetic) within 2^-10."""
    ev = ckks.Oracle(toy)
    steps = [0, 1, 2, 5, -3]
    keys = ev.keygen(21, [s for s in steps if s])
    n = toy.N // 2
    rng = np.random.default_rng(4)
    z = rng.uniform(-1, 1, n)
    diags = [rng.uniform(-1, 1, n) for _ in steps]
    ct = ev.encrypt(keys, z, toy.scale, 3)
    pt_scale = float(toy.primes[ct.level])  # one rescale returns the ciphertext's own scale
    pts = [ev.plain_ntt(ckks.encode(toy, d, pt_scale), ct.level) for d in diags]
    out = ev.linear_transform(keys, ct, pts, steps, pt_scale)
    assert out.level == ct.level - 1 and out.scale == ct.scale * pt_scale / float(toy.primes[ct.level])
    want = sum(d * np.roll(z, -s) for d, s in zip(diags, steps))
    assert np.abs(ev.decrypt(keys, out).real - want).max() < 2 ** -10


def test_linear_transform_bsgs_against_matrix(toy):
    """R31: the baby-step giant-step transform with pre-rotated diagonals decrypts to
    y = sum_{i < n1 n2} d_i (.) RotL(z, i) (numpy) within 2^-10."""
    ev = ckks.Oracle(toy)
    n1, n2 = 4, 3
    keys = ev.keygen(23, list(range(1, n1)) + [g * n1 for g in range(1, n2)])
    n = toy.N // 2
    rng = np.random.default_rng(6)
    z = rng.uniform(-1, 1, n)
    d = [rng.uniform(-1, 1, n) for _ in range(n1 * n2)]
    ct = ev.encrypt(keys, z, toy.scale, 5)
    pt_scale = float(toy.primes[ct.level])
    pts = [[ev.plain_ntt(ckks.encode(toy, np.roll(d[g * n1 + j], g * n1), pt_scale), ct.level) for j in range(n1)]
           for g in range(n2)]
    out = ev.linear_transform_bsgs(keys, ct, pts, n1, n2, pt_scale)
    want = sum(d[i] * np.roll(z, -i) for i in range(n1 * n2))
    assert np.abs(ev.decrypt(keys, out).real - want).max() < 2 ** -10


def test_automorph_is_sigma_g(tiny):
    """o_automorph == coefficient map X^k -> X^{gk} applied by definition (Python)."""
    prm, ev = tiny, ckks.Oracle(tiny)
    rng = np.random.default_rng(1)
    nl = prm.nq
    data = np.stack([np.stack([rng.integers(0, q, prm.N).astype(np.uint64) for q in prm.q]) for _ in range(2)])
    g = ckks.galois_elt(prm, 3)
    out = ev.automorph_poly(data[0], g)
    coef = ckks.ntt_limbs(data[0], prm, list(range(nl)), inverse=True)
    for i, q in enumerate(prm.q):
        want = [0] * prm.N
        for k in range(prm.N):
            e = k * g % (2 * prm.N)
            if e < prm.N:
                want[e] = int(coef[i, k])
            else:
                want[e - prm.N] = (q - int(coef[i, k])) % q
        assert [int(v) for v in ntt_def(want, q, prm.psi[i], prm.logn)] == [int(v) for v in out[i]]


# ---------------------------------------------------------------------------------------------
# O-5 encoding
# ---------------------------------------------------------------------------------------------
def test_encode_fft_vs_definition(toy):
    z = synth.uniform_slots(4, toy.N // 2)
    a = ckks.encode(toy, z, toy.scale)
    b = ckks.encode_naive(toy, z, toy.scale)
    assert np.abs(a - b).max() <= 1
    assert np.abs(ckks.decode(toy, a.astype(float), toy.scale).real - z).max() < 2 ** -25


def test_mask_encoding_quantised(toy):
    lay = synth.LAYOUTS["toy"]
    m = plan.mask_slots(lay, toy.N // 2)
    M = ckks.mask_coeffs(toy, m, 2.0 ** 40)
    back = ckks.decode(toy, M.astype(float), 2.0 ** 40).real
    assert np.abs(back - m).max() < 2 ** -14


# ---------------------------------------------------------------------------------------------
# O-13 sign plan, O-14 argmax (plaintext mirror)
# ---------------------------------------------------------------------------------------------
def load_sign(name):
    d = json.load(open(os.path.join(os.path.dirname(__file__), "..", "data", name)))
    return [list(map(float, c)) for c in d["coeffs"]]


def horner(stages, x):
    for c in stages:
        y = np.zeros_like(x)
        for cf in reversed(c):
            y = y * x + cf
        x = y
    return x


class _Flat:
    """Mirror inputs at a given level/scale."""


@pytest.mark.parametrize("sname", ["sign_7_15_15.json", "sign_f1_f1.json"])
def test_sign_plan_equals_horner(sname):
    prm = ckks.Params(synth.PARAM_SETS["argmax"]) if sname.startswith("sign_7") else \
        ckks.Params(synth.PARAM_SETS["toy_argmax"])
    st = load_sign(sname)
    mir = ckks.Mirror(prm)
    x = np.linspace(-1, 1, 2001)
    out = plan.sign(mir, None, ckks.MirrorCt(x, prm.L, prm.scale), st, prm.scale)
    assert np.abs(out.v - horner(st, x)).max() < 1e-9
    assert out.level == prm.L - plan.sign_depth(st)
    # depth law (ceil(log2(d+1)) for a BSGS plan), except degree 15 whose
    # Paterson-Stockmeyer plan (R13) trades one level for three fewer ct x ct products
    assert plan.sign_depth(st) == sum(math.ceil(math.log2(len(c))) + (len(c) == 16) for c in st)
    nprod = {4: 2, 8: 5, 16: 7}  # ct x ct products (tensors) per stage: deg 3, 7 (BSGS), 15 (PS)
    nks = {4: 2, 8: 4, 16: 6}    # relinearisations: two summed products share one (reading R13b)
    single = sum(1 for l in mir.log if l.startswith("MULCT "))
    summed = sum(1 for l in mir.log if l.startswith("MULCT2 "))
    assert single + 2 * summed == sum(nprod[len(c)] for c in st)
    assert single + summed == sum(nks[len(c)] for c in st)
    # odd symmetry S(-x) = -S(x)
    assert np.abs(horner(st, -x) + horner(st, x)).max() < 1e-9
    # every planned addition saw identical scales, constants fit 62 bits
    assert all(abs(int(l.split()[4])) < 2 ** 62 for l in mir.log if l.startswith("MULC "))
    assert all(abs(int(v)) < 2 ** 62 for l in mir.log if l.startswith(("LINC ", "MULCT ", "MULCT2 ")) and len(l.split()) > 4
               for v in l.split()[4].split(","))


def test_sign_certificate_7_15_15():
    """Certifier: max |1 - S| over >= 10^6 grid points on [2^-7, 1] (+1e5 random)."""
    st = load_sign("sign_7_15_15.json")
    x = np.concatenate([np.linspace(2.0 ** -7, 1, 1_000_001),
                        np.random.default_rng(0).uniform(2.0 ** -7, 1, 100_000)])
    err = np.abs(1 - horner(st, x)).max()
    assert err < 1.2e-4
    # range preservation on [-1, 1]
    assert np.abs(horner(st, np.linspace(-1, 1, 200001))).max() < 1 + 1.2e-4


def test_paper_layout_and_op_law():
    g = GOLD["batching"]
    assert g["slots"] // (2 * g["n"]) == g["argmax_per_ct"]
    lay = dict(queries=g["argmax_per_ct"], prompts=1, classes=g["n"], block=2 * g["n"])
    plan.check_layout(lay, g["slots"])
    # op-count law through the mirror: log n + 1 Sign, log n + 1 rotations
    prm = ckks.Params(synth.PARAM_SETS["argmax"])
    for n in (2, 4, 16, 256):
        mir = ckks.Mirror(prm)
        lay = dict(queries=1, prompts=1, classes=n, block=2 * n)
        calls = {"sign": 0}
        orig = plan.sign

        def counting(ev, keys, x, stages, s):
            calls["sign"] += 1
            return orig(ev, keys, x, stages, s)

        plan.sign = counting
        try:
            # a 1-stage degree-3 sign keeps the depth within the 30-level chain for n <= 256
            st = [[0.0, 1.5, 0.0, -0.5]]
            plan.argmax(mir, None, ckks.MirrorCt(np.zeros(prm.N // 2), prm.L, prm.scale), lay, st)
        except ValueError:
            pass
        finally:
            plan.sign = orig
        if n <= 4:
            assert calls["sign"] == int(math.log2(n)) + 1
            assert mir.counts["ROT"] == int(math.log2(n)) + 1


def _count_argmax_boot(n, prompts):
    """Sign calls, ROT ops and refreshes of plan.argmax_boot on the plaintext mirror (the op list the oracle
    and the library both run), with a mirror bootstrap that returns its input at the post-bootstrap level."""
    prm = ckks.Params(synth.PARAM_SETS["boot_argmax"])
    st = json.load(open(os.path.join(HERE, "..", "data", "sign_7_15_15.json")))["coeffs"]
    st = [list(map(float, c)) for c in st]
    mir = ckks.Mirror(prm)
    lay = dict(queries=1, prompts=prompts, classes=n, block=2 * n * prompts)
    out_level = prm.L - plan.fft_boot_depth([4, 4, 3], 7)
    calls = {"sign": 0, "boot": 0}
    orig = plan.sign

    def counting(ev, keys, x, stages, s):
        calls["sign"] += 1
        return orig(ev, keys, x, stages, s)

    def boot(c):
        calls["boot"] += 1
        assert c.level == 0
        return ckks.MirrorCt(c.v.copy(), out_level, c.scale)
    z = np.zeros(prm.N // 2)
    z[: n * prompts] = np.linspace(0, 1, n * prompts)
    plan.sign = counting
    try:
        plan.argmax_boot(mir, None, ckks.MirrorCt(z, 16, prm.scale), lay, st, boot, 2.0 ** 50)
    finally:
        plan.sign = orig
    return calls["sign"], mir.counts.get("ROT", 0), calls["boot"]


@pytest.mark.parametrize("n,prompts", [(2, 1), (16, 1), (256, 1), (16, 8), (256, 2)])
def test_op_law_counts(n, prompts):
    """PAPER.md:419 (Sec. 4.5): Algorithm 1 on a length-n input needs (log n + 1) Sign operations and
    (log n + 1) rotations; n = 256 -> 9 Sign, 9 rotations.  Counted through the planned circuit
    (plan.argmax_boot on the mirror, refreshes included where the level budget runs out); the prompt
    aggregation adds log2 P rotations on top."""
    signs, rots, boots = _count_argmax_boot(n, prompts)
    ln = int(math.log2(n))
    assert signs == ln + 1
    assert rots == ln + 1 + int(math.log2(prompts))
    if n == 256 and prompts == 1:
        assert (signs, rots) == (GOLD["op_law"]["sign_ops"], GOLD["op_law"]["rotations"])
    assert boots >= (1 if n >= 16 else 0)


def test_argmax_mirror_examples():
    """SPEC.md:246, :259-260, :326 examples through the planned circuit on doubles."""
    prm = ckks.Params(synth.PARAM_SETS["argmax"])
    st = load_sign("sign_7_15_15.json")
    mir = ckks.Mirror(prm)
    # Eq. 6 example Max(0.2, 0.8) = 0.8
    g = GOLD["max_example"]
    r = ckks.MirrorCt(np.full(4, g["a"]), prm.L, prm.scale)
    y = ckks.MirrorCt(np.full(4, g["b"]), prm.L, prm.scale)
    assert abs(plan.hom_max(mir, None, r, y, st).v[0] - g["max"]) < 1e-3
    for key in ("argmax_window", "argmax_ties"):
        g = GOLD[key]
        lay = dict(queries=1, prompts=1, classes=4, block=8)
        z = np.zeros(prm.N // 2)
        z[:4] = g["window"]
        out = plan.argmax(ckks.Mirror(prm), None, ckks.MirrorCt(z, prm.L, prm.scale), lay, st)
        # the polynomial Sign is not exact: y_max undershoots the max by ~|S - 1| |a - b| / 2,
        # which the steep Sign near 0 turns into a ~1e-2 deficit on the winning slot
        assert np.abs(out.v[:4] - np.array(g["one_hot"])).max() < 2e-2
    # vote example: 3 prompts is not a power of two -> pad prompts with zeros (reading R17)
    g = GOLD["vote_example"]
    logits = np.array(g["logits"], dtype=float)
    norm = (logits - g["d_min"]) / (g["d_max"] - g["d_min"])  # Eq. 5
    scores = np.zeros((1, 4, 2))
    scores[0, :3] = norm
    lay = dict(queries=1, prompts=4, classes=2, block=8)
    z = plan.pack(scores, lay, prm.N // 2)
    out = plan.argmax(ckks.Mirror(prm), None, ckks.MirrorCt(z, prm.L, prm.scale), lay, st)
    assert plan.labels(out.v, lay)[0] == g["label"]
    assert np.allclose(logits.mean(axis=0), g["mean"])


def test_argmax_mirror_random_labels():
    prm = ckks.Params(synth.PARAM_SETS["argmax"])
    st = load_sign("sign_7_15_15.json")
    lay = synth.LAYOUTS["argmax_k2"]
    scores = synth.softmax_scores(1000 * 5 + 1, lay["queries"], lay["prompts"], lay["classes"])
    z = plan.pack(scores, lay, prm.N // 2)
    out = plan.argmax(ckks.Mirror(prm), None, ckks.MirrorCt(z, prm.L, prm.scale), lay, st)
    mean = scores.mean(axis=1)
    gap = np.abs(mean[:, 0] - mean[:, 1])
    ok = gap >= 2.0 ** -7
    assert (plan.labels(out.v, lay)[ok] == plan.true_labels(scores)[ok]).all()
    assert out.level == prm.L - plan.argmax_depth(lay, st) == 1  # 1 + (13 + 1) + 13 = 28 of 29 levels


@pytest.mark.slow
def test_toy_argmax_end_to_end_oracle():
    """Full toy argmax on oracle ciphertexts: labels exact, values within 2^-10 of the mirror."""
    prm = ckks.Params(synth.PARAM_SETS["toy_argmax"])
    st = load_sign("sign_f1_f1.json")
    lay = dict(synth.LAYOUTS["toy"])
    lay["queries"] = 8
    scores = synth.toy_scores(1001, lay["queries"], lay["prompts"], lay["classes"])
    z = plan.pack(scores, lay, prm.N // 2)
    ev = ckks.Oracle(prm)
    keys = ev.keygen(synth.KEY_SEED_BASE + 1, plan.argmax_rotations(lay))
    ct = ev.encrypt(keys, z, prm.scale, 77)
    out = plan.argmax(ev, keys, ct, lay, st)
    mir = ckks.Mirror(prm)
    ref = plan.argmax(mir, None, ckks.MirrorCt(z, prm.L, prm.scale), lay, st)
    assert ev.log == mir.log
    dec = ev.decrypt(keys, out).real
    assert np.abs(dec - ref.v).max() < 2 ** -10
    assert (plan.labels(dec, lay) == plan.true_labels(scores)).all()


@pytest.mark.slow
def test_argmax_small_ring_7_15_15_oracle():
    """configs[4] circuit (30 x 45-bit, dnum 3, (7,15,15) Sign, K=2, P=8) on a 2^12 ring."""
    prm = ckks.Params(synth.PARAM_SETS["argmax_small"])
    st = load_sign("sign_7_15_15.json")
    lay = synth.LAYOUTS["argmax_small_k2"]
    scores = synth.softmax_scores(5001, lay["queries"], lay["prompts"], lay["classes"])
    z = plan.pack(scores, lay, prm.N // 2)
    ev = ckks.Oracle(prm)
    keys = ev.keygen(synth.KEY_SEED_BASE + 5, plan.argmax_rotations(lay))
    ct = ev.encrypt(keys, z, prm.scale, 55)
    out = plan.argmax(ev, keys, ct, lay, st)
    mir = ckks.Mirror(prm)
    ref = plan.argmax(mir, None, ckks.MirrorCt(z, prm.L, prm.scale), lay, st)
    assert ev.log == mir.log and out.level == 1
    dec = ev.decrypt(keys, out).real
    assert np.abs(dec - ref.v).max() < 2 ** -10
    mean = scores.mean(axis=1)
    ok = np.abs(mean[:, 0] - mean[:, 1]) >= 2.0 ** -7
    assert (plan.labels(dec, lay)[ok] == plan.true_labels(scores)[ok]).all()


# ---------------------------------------------------------------------------------------------
# O-20 bootstrapping building blocks (readings R32-R35)
# ---------------------------------------------------------------------------------------------
BOOT_TINY = dict(n1=16, n2=8, K=16, r=8, h=64)


@pytest.fixture(scope="module")
def boot_tiny():
    prm = ckks.Params(synth.PARAM_SETS["boot_tiny"])
    ev = ckks.Oracle(prm)
    keys = ev.keygen(7, plan.boot_rotations(BOOT_TINY["n1"], BOOT_TINY["n2"]), h=BOOT_TINY["h"])
    return prm, ev, keys


def test_sparse_secret(boot_tiny):
    """R36: the sparse secret has exactly h nonzeros, all +-1, is a function of the seed alone, and its first
    nonzero sits where the first draw's top log N bits point (the sampler's definition, recomputed here
    with an independent ChaCha20)."""
    prm, ev, keys = boot_tiny
    s = keys.s
    assert np.count_nonzero(s) == BOOT_TINY["h"] and set(np.unique(s)) <= {-1, 0, 1}
    assert np.array_equal(ev.keygen(7, (), h=BOOT_TINY["h"]).s, s)
    assert not np.array_equal(ev.keygen(8, (), h=BOOT_TINY["h"]).s, s)
    tag = 1 << 48
    k = ckks.object_key(ckks.seed_key(7), tag)
    x = int.from_bytes(_keystream(k, 0, tag)[:8], "little")
    assert s[x >> (64 - prm.logn)] == (-1 if x & 1 else 1)


def test_conjugation_is_complex_conjugate(boot_tiny):
    """R32: sigma_{2N-1} (step CONJ) maps the slots of a complex message to their complex conjugates."""
    prm, ev, keys = boot_tiny
    n = prm.N // 2
    rng = np.random.default_rng(8)
    z = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    ct = ev.encrypt(keys, z, prm.scale, 3, level=4)
    assert ckks.galois_elt(prm, ckks.CONJ) == 2 * prm.N - 1
    out = ev.rotate_raw(keys, ct, ckks.CONJ)
    m = np.array([float(v) for v in ev.decrypt_int(keys, out)])
    got = ckks.decode(prm, m, out.scale)
    assert np.abs(got - np.conj(z)).max() < 2 ** -30


def test_mod_raise_adds_multiple_of_q0(boot_tiny):
    """R33: the raised ciphertext decrypts to t = m + q_0 I over the integers, |I_k| <= (h + 1)/2 with h the
    secret's Hamming weight (|c0 + c1 s| <= q_0 (1 + h) / 2 for centred c0, c1)."""
    prm, ev, keys = boot_tiny
    ct = ev.encrypt(keys, np.linspace(-1, 1, prm.N // 2), prm.scale, 4, level=0)
    up = ev.mod_raise(ct, prm.L)
    assert up.level == prm.L and up.scale == ct.scale
    t, m = ev.decrypt_int(keys, up), ev.decrypt_int(keys, ct)
    q0, h = prm.primes[0], int(np.count_nonzero(keys.s))
    assert all((a - b) % q0 == 0 for a, b in zip(t, m))
    I = [(a - b) // q0 for a, b in zip(t, m)]
    assert max(abs(i) for i in I) <= (h + 1) // 2
    assert any(i != 0 for i in I)  # a non-trivial raise


def test_boot_matrices_invert_decoding(boot_tiny):
    """R34: for a real polynomial t, the slots z_j = sum_k t_k zeta^{5^j k} (the definition, written out here)
    satisfy A z = t_lo + i t_hi and U (t_lo + i t_hi) = z."""
    prm = boot_tiny[0]
    N, n = prm.N, prm.N // 2
    rng = np.random.default_rng(2)
    t = rng.integers(-1000, 1000, N).astype(np.float64)
    z = np.array([sum(t[k] * np.exp(1j * np.pi * (pow(5, j, 2 * N) * k % (2 * N)) / N) for k in range(N))
                  for j in range(n)])
    M = plan.boot_matrices(prm, 1.0)
    A = 2 * M["cts_re"]
    w = A @ z
    assert np.abs(w - (t[:n] + 1j * t[n:])).max() < 1e-8
    U = M["stc_re"] * 4 * np.pi
    assert np.abs(U @ (t[:n] + 1j * t[n:]) - z).max() < 1e-7
    assert np.allclose(M["cts_im"], -1j * M["cts_re"]) and np.allclose(M["stc_im"], 1j * M["stc_re"])


def test_boot_poly_is_doubled_cosine():
    """R35: the degree-15 Taylor coefficients match 2 cos((2 pi K x - pi/2) / 2^r) on [-1, 1] (closed form),
    and r double-angle steps d <- d^2 - 2 turn it into 2 sin(2 pi K x)."""
    K, r = 16, 8
    c = plan.boot_poly(K, r)
    x = np.linspace(-1, 1, 2001)
    d = np.polynomial.polynomial.polyval(x, c)
    assert np.abs(d - 2 * np.cos((2 * np.pi * K * x - np.pi / 2) / 2 ** r)).max() < 1e-14
    for _ in range(r):
        d = d * d - 2
    assert np.abs(d - 2 * np.sin(2 * np.pi * K * x)).max() < 1e-9


def test_eval_poly15_general(boot_tiny):
    """R35: the general degree-15 plan decrypts to sum_i c_i x^i (numpy polyval) and uses 5 levels."""
    prm, ev, keys = boot_tiny
    n = prm.N // 2
    rng = np.random.default_rng(12)
    z = rng.uniform(-1, 1, n)
    c = list(rng.uniform(-1, 1, 16) / np.arange(1, 17))
    ct = ev.encrypt(keys, z, prm.scale, 9, level=8)
    out = plan.eval_poly15(ev, keys, ct, c, prm.scale)
    assert out.level == 3 and out.scale == prm.scale
    assert np.abs(ev.decrypt(keys, out).real - np.polynomial.polynomial.polyval(z, c)).max() < 2 ** -30


def test_bootstrap_refreshes_levels(boot_tiny):
    """N3 end to end: a level-0 ciphertext bootstraps to level L - (8 + r) and still decrypts to its slots
    (within 2^-14; the precision budget of DESIGN.md R35)."""
    prm, ev, keys = boot_tiny
    n = prm.N // 2
    rng = np.random.default_rng(3)
    z = rng.uniform(-1, 1, n)
    ct = ev.encrypt(keys, z, prm.scale, 5, level=0)
    cfg = plan.boot_config(ev, ct.scale, prm.L, BOOT_TINY["K"], BOOT_TINY["r"], BOOT_TINY["n1"], BOOT_TINY["n2"])
    out = plan.bootstrap(ev, keys, ct, cfg)
    assert out.level == prm.L - plan.boot_depth(BOOT_TINY["r"])
    assert np.abs(ev.decrypt(keys, out).real - z).max() < 2 ** -14
    # and it computes on: one more product after the refresh
    sq = ev.mul_ct(keys, out, out, None, out.level - 1)
    assert np.abs(ev.decrypt(keys, sq).real - z * z).max() < 2 ** -13


def test_special_fft_stages_factor_decoding():
    """R37: the butterfly stages applied to the bit-reversed coefficient vector give U w with U[j][k] =
    zeta^{5^j k} (the decoding definition, written out); the inverse stages undo it; merged groups in
    diagonal form equal the stages applied one by one."""
    for logn in (4, 6, 8):
        N, n = 1 << logn, 1 << (logn - 1)
        e = [pow(5, j, 2 * N) for j in range(n)]
        U = np.array([[np.exp(1j * np.pi * ((e[j] * k) % (2 * N)) / N) for k in range(n)] for j in range(n)])
        rng = np.random.default_rng(logn)
        w = rng.normal(size=n) + 1j * rng.normal(size=n)
        br = plan.bitrev_perm(n)
        assert sorted(br) == list(range(n)) and all(br[br[i]] == i for i in range(n))
        v = w[br]
        for S in plan.dft_stages(N):
            assert len(S) <= 3
            v = plan.diag_apply(S, v)
        assert np.abs(v - U @ w).max() < 1e-12
        z = U @ w
        for S in plan.dft_stages_inv(N)[::-1]:
            z = plan.diag_apply(S, z)
        assert np.abs(z - w[br]).max() < 1e-12
        groups = [logn - 3, 2]
        stc, cts = plan.fft_groups(N, groups)
        assert [len(D) for D in stc] == [2 ** (g + 1) - 1 if i < len(groups) - 1 else 2 ** g
                                         for i, g in enumerate(groups)]
        v = w[br]
        for D in stc:
            v = plan.diag_apply(D, v)
        assert np.abs(v - U @ w).max() < 1e-12
        z = U @ w
        for D in cts:
            z = plan.diag_apply(D, z)
        assert np.abs(z - w[br]).max() < 1e-12


def test_bootstrap_fft_refreshes():
    """R37 end to end (N = 2^8, groups 3 + 4): decrypts to the input slots within 2^-14 at level
    L - (2 * 2 + 6 + r)."""
    prm = ckks.Params(synth.PARAM_SETS["boot_tiny"])
    ev = ckks.Oracle(prm)
    groups, K, r = [3, 4], 16, 8
    keys = ev.keygen(9, plan.fft_boot_rotations(prm.N, groups), h=64)
    z = np.random.default_rng(10).uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(keys, z, prm.scale, 5, level=0)
    cfg = plan.fft_boot_config(ev, ct.scale, prm.L, K, r, groups)
    out = plan.bootstrap_fft(ev, keys, ct, cfg)
    assert out.level == prm.L - plan.fft_boot_depth(groups, r)
    assert np.abs(ev.decrypt(keys, out).real - z).max() < 2 ** -14


def test_argmax_boot_k16_one_hot():
    """N4 (reading R38): Algorithm 1 with K = 16 classes (four Max steps + the final Sign, more levels than the
    chain holds) refreshes with four bootstraps and still returns the one-hot of the true label."""
    prm = ckks.Params(synth.PARAM_SETS["boot_argmax_tiny"])
    ev = ckks.Oracle(prm)
    lay = synth.LAYOUTS["tiny_k16"]
    d = json.load(open(os.path.join(os.path.dirname(__file__), "..", "data", "sign_7_15_15.json")))
    st = [list(map(float, c)) for c in d["coeffs"]]
    groups = [4, 3]
    rot = plan.argmax_rotations(lay) + plan.fft_boot_rotations(prm.N, groups)
    keys = ev.keygen(11, rot, h=64)
    cfg = plan.fft_boot_config(ev, 2.0 ** 50, prm.L, 16, 7, groups)
    nb = [0]

    def boot(c):
        nb[0] += 1
        assert c.level == 0 and c.scale == 2.0 ** 50
        return plan.bootstrap_fft(ev, keys, c, cfg)
    scores = synth.softmax_scores(5, lay["queries"], lay["prompts"], lay["classes"])
    ct = ev.encrypt(keys, plan.pack(scores, lay, prm.N // 2), prm.scale, 3, level=16)
    out = plan.argmax_boot(ev, keys, ct, lay, st, boot, 2.0 ** 50)
    assert nb[0] == 4 and out.scale == prm.scale
    dec = ev.decrypt(keys, out).real
    want = np.zeros(lay["classes"])
    want[plan.true_labels(scores)[0]] = 1.0
    assert np.abs(dec[: lay["classes"]] - want).max() < 2 ** -5


def test_bsgs_split_equals_diagonal_form():
    """R39: every merged special-FFT group in baby-step giant-step form,
    sum_g RotL(sum_j RotR(d_{b_j + G_g}, G_g) (.) RotL(v, b_j), G_g), equals its diagonal form on a plaintext
    vector; baby / giant counts about sqrt(#diagonals)."""
    N = 1 << 8
    n = N // 2
    v = np.random.default_rng(3).normal(size=n) + 0j
    for groups in ([3, 4], [2, 2, 3], [7]):
        stc, cts = plan.fft_groups(N, groups)
        for D in stc + cts:
            baby, giant, where = plan.bsgs_split(D, n)
            assert len(baby) * len(giant) >= len(D) and len(baby) < 2 * math.sqrt(len(D)) + 1
            acc = 0
            for g, G in enumerate(giant):
                inner = 0
                for j, b in enumerate(baby):
                    k = where[(g, j)]
                    d = D[k] if k is not None else np.zeros(n)
                    inner = inner + np.roll(d, G) * np.roll(v, -b)
                acc = acc + np.roll(inner, -G)
            assert np.abs(acc - plan.diag_apply(D, v)).max() < 1e-9


def test_bootstrap_fft_bsgs_refreshes():
    """R39 end to end (N = 2^8): the baby-step giant-step bootstrap needs fewer keys and still refreshes within
    2^-14."""
    prm = ckks.Params(synth.PARAM_SETS["boot_tiny"])
    ev = ckks.Oracle(prm)
    groups, K, r = [3, 4], 16, 7
    rot = plan.fft_boot_rotations(prm.N, groups, bsgs=True)
    assert len(rot) < len(plan.fft_boot_rotations(prm.N, groups))
    keys = ev.keygen(9, rot, h=64)
    z = np.random.default_rng(10).uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(keys, z, prm.scale, 5, level=0)
    cfg = plan.fft_boot_config(ev, ct.scale, prm.L, K, r, groups, bsgs=True)
    out = plan.bootstrap_fft(ev, keys, ct, cfg)
    assert out.level == prm.L - plan.fft_boot_depth(groups, r)
    assert np.abs(ev.decrypt(keys, out).real - z).max() < 2 ** -14


def test_argmax_boot_prompt_groups_equal_one_ciphertext():
    """N4 prompt groups (PAPER.md:141 y* = sum y_i across ciphertexts): splitting 8 prompts into two ciphertexts
    of 4 (prompt_cts = 2) decrypts to the same one-hot as the true label of the mean over all 8 prompts."""
    prm = ckks.Params(synth.PARAM_SETS["boot_argmax_tiny"])
    ev = ckks.Oracle(prm)
    lay = dict(queries=1, prompts=4, classes=16, block=128)
    d = json.load(open(os.path.join(os.path.dirname(__file__), "..", "data", "sign_7_15_15.json")))
    st = [list(map(float, c)) for c in d["coeffs"]]
    groups = [4, 3]
    keys = ev.keygen(13, plan.argmax_rotations(lay) + plan.fft_boot_rotations(prm.N, groups, bsgs=True), h=64)
    cfg = plan.fft_boot_config(ev, 2.0 ** 50, prm.L, 16, 7, groups, bsgs=True)
    scores = synth.ensemble_scores(7, 1, 8, 16)
    cts = [ev.encrypt(keys, plan.pack(scores[:, 4 * i:4 * i + 4], lay, prm.N // 2), prm.scale, 20 + i, level=16)
           for i in range(2)]
    out = plan.argmax_boot(ev, keys, cts, lay, st, lambda c: plan.bootstrap_fft(ev, keys, c, cfg), 2.0 ** 50,
                           prompt_cts=2)
    dec = ev.decrypt(keys, out).real[:16]
    want = np.zeros(16)
    want[plan.true_labels(scores)[0]] = 1.0
    assert np.abs(dec - want).max() < 2 ** -5
