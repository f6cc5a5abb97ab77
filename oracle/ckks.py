"""Oracle RNS-CKKS + SecPE Argmax -- TEST INFRASTRUCTURE ONLY.

Python orchestration over the plain-C core ``ckks_oracle.c``.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  Shares no code with paper_2502_00847_b200/.

What each part follows (PAPER.md line numbers; readings R* are listed in DESIGN.md sec. 3):
  Params / primes ........ PAPER.md:89-93 (R_Q, Q = prod q_i), reading R1
  encode / decode ........ PAPER.md:98 (SIMD packing), reading R5 (slot j <-> zeta^{5^j})
  sampler / keygen ....... reading R6/R7 (BASELINE configs[0]: Gaussian sigma=3.2, ternary secret)
  encrypt / decrypt ...... PAPER.md:139, :143 (Steps 1 and 4)
  add / sub / mul / rot .. PAPER.md:101-105
  scale planning ......... reading R9
  Sign plan .............. PAPER.md:189-195 (Eq. 4 composite, BSGS), reading R13
  Max .................... PAPER.md:208-210 (Eq. 6)
  Argmax ................. PAPER.md:214-235 (Algorithm 1), :141 (aggregation), :197-204 (Eq. 5),
                           :239 (2n slots per argmax)
  Bootstrapping .......... SURVEY 8(f) N3 (PAPER.md:94-96, :327 bootstraps at L = 35): conjugation
                           (R32), ModRaise (R33), CoeffToSlot / SlotToCoeff (R34), EvalMod (R35);
                           the plan is in plan.py
"""
import ctypes
import math
import os
import struct
import subprocess
from decimal import Decimal, getcontext

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "ckks_oracle.c")

u64p = ctypes.POINTER(ctypes.c_uint64)
i64p = ctypes.POINTER(ctypes.c_int64)
u32p = ctypes.POINTER(ctypes.c_uint32)
intp = ctypes.POINTER(ctypes.c_int)


def seed_key(seed):
    """256-bit master seed as 8 little-endian uint32 words (R6): 32 bytes are taken as they are;
    an integer 0 <= seed < 2^64 is the TEST-ONLY deterministic mode, bytes = LE64(seed) followed by 24 zeros."""
    if isinstance(seed, (bytes, bytearray)):
        if len(seed) != 32:
            raise ValueError("a seed is 32 bytes")
        return np.frombuffer(bytes(seed), dtype="<u4").astype(np.uint32)
    seed = int(seed)
    if not 0 <= seed < 1 << 64:
        raise ValueError("integer seeds are 64-bit")
    return np.array([seed & 0xFFFFFFFF, seed >> 32, 0, 0, 0, 0, 0, 0], dtype=np.uint32)


def chacha20_block(key, counter, nonce):
    """One ChaCha20 block (16 uint32 words) of the oracle core."""
    out = np.zeros(16, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    lib().o_chacha20_block(k.ctypes.data_as(u32p), counter, nonce, out.ctypes.data_as(u32p))
    return out


def object_key(master, tag):
    out = np.zeros(8, dtype=np.uint32)
    lib().o_object_key(master.ctypes.data_as(u32p), tag, out.ctypes.data_as(u32p))
    return out


def build():
    """Compile the oracle core (plain C, -O2, no fast-math)."""
    if os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(_SRC):
        return _SO
    cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
           "-o", _SO, _SRC]
    subprocess.check_call(cmd)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        U, I = ctypes.c_uint64, ctypes.c_int
        sig = {
            "o_set_threads": (I, [I]),
            "o_is_prime": (I, [U]),
            "o_gen_primes": (I, [I, I, U, I, u64p, I, u64p]),
            "o_find_psi": (U, [U, I]),
            "o_mulmod": (U, [U, U, U]),
            "o_powmod": (U, [U, U, U]),
            "o_ntt": (None, [u64p, I, U, U]),
            "o_intt": (None, [u64p, I, U, U]),
            "o_ntt_naive": (None, [u64p, u64p, I, U, U]),
            "o_ntt_limbs": (None, [u64p, I, I, u64p, u64p, intp]),
            "o_intt_limbs": (None, [u64p, I, I, u64p, u64p, intp]),
            "o_chacha20_block": (None, [u32p, U, U, u32p]),
            "o_derive": (None, [u32p, U, u32p]),
            "o_object_key": (None, [u32p, U, u32p]),
            "o_encrypt_key": (None, [u32p, u32p]),
            "o_draw": (U, [u32p, U, U]),
            "o_tag": (U, [U, U, U]),
            "o_uniform": (U, [u32p, U, U, U, I, U]),
            "o_sample_uniform": (None, [u32p, U, I, I, u64p, intp, u64p]),
            "o_sample_ternary": (None, [u32p, U, I, i64p]),
            "o_sample_sparse": (None, [u32p, U, I, I, i64p]),
            "o_sample_gauss": (None, [u32p, U, I, u64p, I, i64p]),
            "o_int_to_ntt": (None, [ctypes.c_void_p, i64p, I, intp, u64p]),
            "o_keygen_pk": (None, [ctypes.c_void_p, u32p, u64p, u64p, I, u64p]),
            "o_keygen_swk": (None, [ctypes.c_void_p, u32p, U, u64p, u64p, u64p, I, u64p]),
            "o_encrypt": (None, [ctypes.c_void_p, u32p, u64p, i64p, I, u64p, I, u64p]),
            "o_decrypt_residues": (None, [ctypes.c_void_p, u64p, u64p, I, u64p]),
            "o_add": (None, [ctypes.c_void_p, u64p, u64p, I, I, u64p]),
            "o_sub": (None, [ctypes.c_void_p, u64p, u64p, I, I, u64p]),
            "o_mul_int": (None, [ctypes.c_void_p, u64p, I, ctypes.c_int64, ctypes.c_uint64, u64p]),
            "o_add_int": (None, [ctypes.c_void_p, u64p, I, ctypes.c_int64, ctypes.c_uint64, u64p]),
            "o_mul_plain": (None, [ctypes.c_void_p, u64p, I, u64p, u64p]),
            "o_tensor": (None, [ctypes.c_void_p, u64p, u64p, I, u64p]),
            "o_keyswitch": (None, [ctypes.c_void_p, u64p, I, u64p, u64p]),
            "o_keyswitch_g": (None, [ctypes.c_void_p, u64p, I, u64p, ctypes.c_uint64, u64p]),
            "o_rescale": (None, [ctypes.c_void_p, u64p, I, u64p]),
            "o_mul_vec": (None, [u64p, u64p, U, U, u64p]),
            "o_automorph": (None, [ctypes.c_void_p, u64p, I, I, U, u64p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def P(a):
    """numpy uint64 array -> pointer (array must be C-contiguous)."""
    assert a.flags["C_CONTIGUOUS"]
    if a.dtype == np.uint64:
        return a.ctypes.data_as(u64p)
    if a.dtype == np.int64:
        return a.ctypes.data_as(i64p)
    if a.dtype == np.int32:
        return a.ctypes.data_as(intp)
    raise TypeError(a.dtype)


class _OCtx(ctypes.Structure):
    _fields_ = [("logn", ctypes.c_int), ("nq", ctypes.c_int), ("np", ctypes.c_int),
                ("alpha", ctypes.c_int), ("primes", u64p), ("psi", u64p)]


# ---------------------------------------------------------------------------
# exact rounding helpers
# ---------------------------------------------------------------------------
# Plan constants C = rha(c Delta_c) are integers below 2^120 in magnitude, passed to the C oracle as two words
# (two's complement 128-bit); with Delta_c ~ q ~ 2^49 the Sign coefficients (up to 2^14.8) give C ~ 2^64.
CONST_LIMIT = 2 ** 120


def wide_int(C):
    """(c_hi, c_lo) with C = c_hi 2^64 + c_lo, c_lo in [0, 2^64)."""
    C = int(C)
    if abs(C) >= CONST_LIMIT:
        raise OverflowError("constant too large")
    return C >> 64, C & ((1 << 64) - 1)


def round_half_away(x):
    """Exact round-half-away-from-zero of a Python float -> int."""
    a = abs(x)
    f = math.floor(a)
    r = f + (1 if a - f >= 0.5 else 0)  # a - f is exact (Sterbenz)
    return int(r) if x >= 0 else -int(r)


def round_half_away_np(x):
    a = np.abs(x)
    f = np.floor(a)
    r = f + (a - f >= 0.5)
    return np.where(x >= 0, r, -r)


def dbits(x):
    """IEEE-754 bit pattern of a double as 16 hex digits (used in op logs)."""
    return "%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


# ---------------------------------------------------------------------------
# Parameters (reading R1: prime chains; O-3 psi)
# ---------------------------------------------------------------------------
def gen_primes(bits, count, logn, mode, exclude=()):
    ex = np.array(list(exclude) or [0], dtype=np.uint64)
    out = np.zeros(count, dtype=np.uint64)
    got = lib().o_gen_primes(bits, count, 2 << logn, 0 if mode == "nearest" else 1, P(ex),
                             len(exclude), P(out))
    if got != count:
        raise RuntimeError("prime generation failed")
    return [int(v) for v in out]


def cdt_table(sigma=Decimal("3.2"), tail=19):
    """CDT thresholds T[m] = floor(2^63 F(m)), F = CDF of |X|, X ~ D_{Z,sigma} cut at |X| <= tail.
    Computed with 60-digit decimal arithmetic (reading R6)."""
    getcontext().prec = 60
    sigma = Decimal(sigma)
    rho = [(-(Decimal(j * j)) / (2 * sigma * sigma)).exp() for j in range(tail + 1)]
    tot = rho[0] + 2 * sum(rho[1:])
    out, acc = [], rho[0]
    two63 = Decimal(2) ** 63
    for m in range(tail + 1):
        if m > 0:
            acc += 2 * rho[m]
        out.append(int((two63 * acc / tot).to_integral_value(rounding="ROUND_FLOOR")))
    out[-1] = 1 << 63
    return np.array(out, dtype=np.uint64)


class Params:
    """RNS-CKKS parameters: ring degree N = 2^logn, chain q_0..q_L, special primes p, digit size alpha."""

    def __init__(self, desc):
        self.desc = desc
        self.logn = desc["logn"]
        self.N = 1 << self.logn
        primes = []
        for mode, bits, cnt in desc["q"]:
            primes += gen_primes(bits, cnt, self.logn, mode, primes)
        self.nq = len(primes)
        for mode, bits, cnt in desc["p"]:
            primes += gen_primes(bits, cnt, self.logn, mode, primes)
        self.np_ = len(primes) - self.nq
        self.primes = primes
        self.q = primes[: self.nq]
        self.p = primes[self.nq:]
        self.alpha = desc["alpha"]
        self.scale = float(2 ** desc["log_scale"])
        self.psi = [int(lib().o_find_psi(q, self.logn)) for q in primes]
        self.primes_np = np.array(primes, dtype=np.uint64)
        self.psi_np = np.array(self.psi, dtype=np.uint64)
        self.cdt = cdt_table()
        self._c = _OCtx(self.logn, self.nq, self.np_, self.alpha, P(self.primes_np), P(self.psi_np))
        self.cptr = ctypes.cast(ctypes.pointer(self._c), ctypes.c_void_p)

    @property
    def L(self):
        return self.nq - 1

    def beta(self, level):
        return (level + 1 + self.alpha - 1) // self.alpha


# ---------------------------------------------------------------------------
# NTT helpers
# ---------------------------------------------------------------------------
def ntt(a, q, psi, logn):
    a = np.ascontiguousarray(a, dtype=np.uint64).copy()
    lib().o_ntt(P(a), logn, q, psi)
    return a


def intt(a, q, psi, logn):
    a = np.ascontiguousarray(a, dtype=np.uint64).copy()
    lib().o_intt(P(a), logn, q, psi)
    return a


def ntt_limbs(a, prm, pids, inverse=False):
    """In-place-free batched NTT of array [..., nl, N] with limb l under prime index pids[l]."""
    a = np.ascontiguousarray(a, dtype=np.uint64).copy()
    nl = a.shape[-2]
    flat = a.reshape(-1, nl, prm.N)
    ids = np.array(pids, dtype=np.int32)
    f = lib().o_intt_limbs if inverse else lib().o_ntt_limbs
    for b in range(flat.shape[0]):
        blk = np.ascontiguousarray(flat[b])
        f(P(blk), prm.logn, nl, P(prm.primes_np), P(prm.psi_np), P(ids))
        flat[b] = blk
    return flat.reshape(a.shape)


# ---------------------------------------------------------------------------
# Encoding (reading R5): slot j <-> evaluation at zeta^{5^j mod 2N}, zeta = e^{i pi / N}
# m_k = round_half_away((2 Delta / N) Re sum_j z_j zeta^{-5^j k})
# ---------------------------------------------------------------------------
def _rot_group(N):
    e = np.empty(N // 2, dtype=np.int64)
    v = 1
    for j in range(N // 2):
        e[j] = v
        v = (v * 5) % (2 * N)
    return e


def encode_real(prm, z, scale):
    """Real coefficients (before rounding) of the scaled encoding, via numpy's FFT (a library step)."""
    N = prm.N
    z = np.zeros(N // 2, dtype=np.complex128) if z is None else np.asarray(z, dtype=np.complex128)
    zz = np.zeros(N // 2, dtype=np.complex128)
    zz[: len(z)] = z
    e = _rot_group(N)
    w = np.zeros(2 * N, dtype=np.complex128)
    w[e] = zz
    w[(2 * N - e) % (2 * N)] = np.conj(zz)
    W = w[1::2]  # W[t] = w[2t+1]
    k = np.arange(N)
    zeta_mk = np.exp(-1j * np.pi * k / N)
    m = zeta_mk * np.fft.fft(W) / N
    return m.real * scale


def encode(prm, z, scale):
    """Integer plaintext coefficients (int64) of slot vector z at the given scale."""
    r = round_half_away_np(encode_real(prm, z, scale))
    if np.max(np.abs(r)) >= 2.0 ** 62:
        raise OverflowError("encoded coefficient exceeds 2^62")
    return r.astype(np.int64)


def encode_naive(prm, z, scale):
    """O(N^2) evaluation of the encoding definition (pins only, small N)."""
    N = prm.N
    zz = np.zeros(N // 2, dtype=np.complex128)
    zz[: len(z)] = z
    e = _rot_group(N)
    k = np.arange(N)
    M = np.exp(-1j * np.pi * np.outer(e, k) / N)  # zeta^{-5^j k}
    s = (zz[:, None] * M).sum(axis=0)
    return round_half_away_np(2.0 * scale / N * s.real).astype(np.int64)


def decode(prm, m, scale):
    """z_j = (1/scale) sum_k m_k zeta^{5^j k}; m real/integer coefficients (float array)."""
    N = prm.N
    m = np.asarray(m, dtype=np.float64)
    k = np.arange(N)
    v = np.fft.ifft(m * np.exp(1j * np.pi * k / N)) * N  # v[t] = sum_k m_k zeta^k omega^{tk}
    e = _rot_group(N)
    return v[(e - 1) // 2] / scale


def mask_coeffs(prm, mask_slots, delta_m, quant_bits=24):
    """Quantised plaintext-mask encoding (reading R16): M_k = rha(delta_m * rha(m_k 2^24) / 2^24),
    m_k the unit-scale real coefficients of the mask."""
    mk = encode_real(prm, mask_slots, 1.0)
    qk = round_half_away_np(mk * float(2 ** quant_bits)) / float(2 ** quant_bits)
    return round_half_away_np(delta_m * qk).astype(np.int64)


# ---------------------------------------------------------------------------
# CRT (O-4): centered lift of residues [nl][N]
# ---------------------------------------------------------------------------
def crt_centered(res, primes):
    nl = res.shape[0]
    Q = 1
    for q in primes[:nl]:
        Q *= q
    acc = np.zeros(res.shape[1], dtype=object)
    for i in range(nl):
        qi = primes[i]
        Qi = Q // qi
        c = pow(Qi % qi, -1, qi)
        r = res[i].astype(object)
        acc = acc + ((r * c) % qi) * Qi
    acc = acc % Q
    return np.where(acc > Q // 2, acc - Q, acc)


# ---------------------------------------------------------------------------
# Ciphertexts and keys
# ---------------------------------------------------------------------------
class Ct:
    __slots__ = ("data", "scale")

    def __init__(self, data, scale):
        self.data = np.ascontiguousarray(data, dtype=np.uint64)
        self.scale = float(scale)

    @property
    def level(self):
        return self.data.shape[1] - 1

    def copy(self):
        return Ct(self.data.copy(), self.scale)


# Step value meaning complex conjugation of the slots (reading R32): sigma_g with g = 2N - 1 (X -> X^-1)
CONJ = -(2 ** 31)


def galois_elt(prm, steps):
    """RotL(s): g = 5^s mod 2N; RotR(s) = RotL(N/2 - s) (reading R2); CONJ: g = 2N - 1 (R32)."""
    N = prm.N
    if steps == CONJ:
        return 2 * N - 1
    s = steps % (N // 2)
    return pow(5, s, 2 * N)


class Keys:
    pass


class Oracle:
    """Oracle evaluator: plain CKKS ops on Ct objects (every op logged for plan comparison)."""

    def __init__(self, prm):
        self.prm = prm
        self.log = []
        self.counts = {}

    # ---- keys ----------------------------------------------------------------
    def keygen(self, seed, rot_steps=(), h=0):
        """h = 0: uniform ternary secret (R6); h > 0: sparse ternary secret of Hamming weight h (R36)."""
        prm = self.prm
        L = lib()
        N, ne = prm.N, prm.nq + prm.np_
        k = Keys()
        k.seed = seed
        master = seed_key(seed)
        mk = master.ctypes.data_as(u32p)
        ks = object_key(master, L.o_tag(1, 0, 0))
        s = np.zeros(N, dtype=np.int64)
        if h:
            if not 0 < h <= N:
                raise ValueError("Hamming weight out of range")
            L.o_sample_sparse(ks.ctypes.data_as(u32p), L.o_tag(1, 0, 0), prm.logn, h, P(s))
        else:
            L.o_sample_ternary(ks.ctypes.data_as(u32p), L.o_tag(1, 0, 0), prm.logn, P(s))
        k.s = s
        k.s_ntt = np.zeros((ne, N), dtype=np.uint64)
        L.o_int_to_ntt(prm.cptr, P(s), ne, P(np.arange(ne, dtype=np.int32)), P(k.s_ntt))
        k.pk = np.zeros((2, prm.nq, N), dtype=np.uint64)
        L.o_keygen_pk(prm.cptr, mk, P(k.s_ntt), P(prm.cdt), len(prm.cdt), P(k.pk))
        # relinearisation key: s' = s^2
        s2 = np.zeros((prm.nq, N), dtype=np.uint64)
        for t in range(prm.nq):
            q = prm.primes[t]
            lib().o_mul_vec(P(np.ascontiguousarray(k.s_ntt[t])), P(np.ascontiguousarray(k.s_ntt[t])), N, q, P(s2[t]))
        k.rlk = self._swk(master, 0, k.s_ntt, s2)
        k.gk = {}
        for st in rot_steps:
            g = galois_elt(prm, st)
            if g in k.gk:
                continue
            sg = self.automorph_poly(k.s_ntt[: prm.nq], g)
            k.gk[g] = self._swk(master, g, k.s_ntt, sg)
        return k

    def _swk(self, master, g, s_ntt, sp_ntt):
        prm = self.prm
        beta = prm.beta(prm.L)
        out = np.zeros((beta, 2, prm.nq + prm.np_, prm.N), dtype=np.uint64)
        sp = np.ascontiguousarray(sp_ntt, dtype=np.uint64)
        lib().o_keygen_swk(prm.cptr, master.ctypes.data_as(u32p), g, P(s_ntt), P(sp), P(prm.cdt), len(prm.cdt),
                           P(out))
        return out

    def automorph_poly(self, poly_ntt, g):
        """sigma_g of a single polynomial [nl][N] in NTT form (via the coefficient domain)."""
        nl = poly_ntt.shape[0]
        src = np.ascontiguousarray(poly_ntt[None], dtype=np.uint64)
        out = np.zeros_like(src)
        lib().o_automorph(self.prm.cptr, P(src), nl, 1, g, P(out))
        return out[0]

    # ---- encrypt / decrypt -----------------------------------------------------
    def encrypt_int(self, keys, m, level, scale, seed):
        prm = self.prm
        m = np.ascontiguousarray(m, dtype=np.int64)
        ct = np.zeros((2, level + 1, prm.N), dtype=np.uint64)
        lib().o_encrypt(prm.cptr, seed_key(seed).ctypes.data_as(u32p), P(keys.pk), P(m), level, P(prm.cdt),
                        len(prm.cdt), P(ct))
        return Ct(ct, scale)

    def encrypt(self, keys, z, scale, seed, level=None):
        level = self.prm.L if level is None else level
        return self.encrypt_int(keys, encode(self.prm, z, scale), level, scale, seed)

    def decrypt_int(self, keys, ct):
        """Centered integer coefficients of c0 + c1 s mod Q_level (Python ints)."""
        prm = self.prm
        out = np.zeros((ct.level + 1, prm.N), dtype=np.uint64)
        lib().o_decrypt_residues(prm.cptr, P(keys.s_ntt), P(ct.data), ct.level, P(out))
        return crt_centered(out, prm.primes)

    def decrypt(self, keys, ct):
        m = self.decrypt_int(keys, ct)
        return decode(self.prm, np.array([float(v) for v in m]), ct.scale)

    # ---- logging ------------------------------------------------------------------
    def _log(self, kind, lin, lout, scale, extra=""):
        self.log.append("%s %d %d %s %s" % (kind, lin, lout, dbits(scale), extra))
        self.counts[kind] = self.counts.get(kind, 0) + 1

    # ---- primitive ops (no logging; used by the planned ops below and by tests) ----------
    def drop(self, ct, level):
        if level > ct.level:
            raise ValueError("cannot raise level")
        return Ct(ct.data[:, : level + 1].copy(), ct.scale)

    def _align(self, a, b):
        lv = min(a.level, b.level)
        if a.scale != b.scale:
            raise ValueError("scale mismatch %r vs %r" % (a.scale, b.scale))
        return self.drop(a, lv), self.drop(b, lv)

    def add_raw(self, a, b):
        a, b = self._align(a, b)
        out = np.zeros_like(a.data)
        lib().o_add(self.prm.cptr, P(a.data), P(b.data), a.level + 1, 2, P(out))
        return Ct(out, a.scale)

    def sub_raw(self, a, b):
        a, b = self._align(a, b)
        out = np.zeros_like(a.data)
        lib().o_sub(self.prm.cptr, P(a.data), P(b.data), a.level + 1, 2, P(out))
        return Ct(out, a.scale)

    def mul_int_raw(self, a, C):
        out = np.zeros_like(a.data)
        lib().o_mul_int(self.prm.cptr, P(a.data), a.level + 1, *wide_int(C), P(out))
        return out

    def add_int_raw(self, a, C):
        out = np.zeros_like(a.data)
        lib().o_add_int(self.prm.cptr, P(a.data), a.level + 1, *wide_int(C), P(out))
        return out

    def mul_plain_raw(self, a, pt_ntt):
        out = np.zeros_like(a.data)
        pt = np.ascontiguousarray(pt_ntt[: a.level + 1])
        lib().o_mul_plain(self.prm.cptr, P(a.data), a.level + 1, P(pt), P(out))
        return out

    def tensor(self, a, b):
        nl = a.level + 1
        d = np.zeros((3, nl, self.prm.N), dtype=np.uint64)
        lib().o_tensor(self.prm.cptr, P(a.data), P(b.data), nl, P(d))
        return d

    def keyswitch(self, d, swk):
        nl = d.shape[0]
        ks = np.zeros((2, nl, self.prm.N), dtype=np.uint64)
        dd = np.ascontiguousarray(d)
        lib().o_keyswitch(self.prm.cptr, P(dd), nl, P(swk), P(ks))
        return ks

    def mul_relin(self, keys, a, b, d=None):
        """ct x ct -> tensor -> relinearise (no rescale); scale S_a S_b.  d: a precomputed
        (possibly augmented) tensor of a and b."""
        if a.level != b.level:
            raise ValueError("level mismatch")
        if d is None:
            d = self.tensor(a, b)
        ks = self.keyswitch(np.ascontiguousarray(d[2]), keys.rlk)
        out = np.zeros((2, a.level + 1, self.prm.N), dtype=np.uint64)
        lib().o_add(self.prm.cptr, P(np.ascontiguousarray(d[:2])), P(ks), a.level + 1, 2, P(out))
        return Ct(out, a.scale * b.scale)

    def rescale(self, ct, new_scale=None):
        nl = ct.level + 1
        out = np.zeros((2, nl - 1, self.prm.N), dtype=np.uint64)
        lib().o_rescale(self.prm.cptr, P(ct.data), nl, P(out))
        s = ct.scale / float(self.prm.primes[ct.level]) if new_scale is None else new_scale
        return Ct(out, s)

    def rotate_raw(self, keys, ct, steps):
        g = galois_elt(self.prm, steps)
        if g == 1:
            return ct.copy()
        if g not in keys.gk:
            raise KeyError("no Galois key for step %d" % steps)
        nl = ct.level + 1
        sig = np.zeros_like(ct.data)
        lib().o_automorph(self.prm.cptr, P(ct.data), nl, 2, g, P(sig))
        ks = self.keyswitch(np.ascontiguousarray(sig[1]), keys.gk[g])
        out = np.zeros_like(ct.data)
        o0 = np.zeros((nl, self.prm.N), dtype=np.uint64)
        lib().o_add(self.prm.cptr, P(np.ascontiguousarray(sig[0])), P(np.ascontiguousarray(ks[0])), nl, 1, P(o0))
        out[0] = o0
        out[1] = ks[1]
        return Ct(out, ct.scale)

    def rotate_hoisted_raw(self, keys, ct, steps_list):
        """N2: rotations of ONE ciphertext by several steps sharing one ModUp of c1
        (PAPER.md:237 applies rotations to the same ciphertext; the hoisting itself is this build's
        reading R29): for each step with Galois element g,
            ks = ModDown( sum_j sigma_g(ModUp_j(c1)) * gk_g[j] ),   out = (sigma_g(c0) + ks0, ks1).
        sigma_g is applied to the integer polynomials ModUp_j(c1), so the integers differ from
        rotate_raw (ModUp of sigma_g(c1), O-12) by key-switching noise only."""
        prm = self.prm
        nl = ct.level + 1
        c1 = np.ascontiguousarray(ct.data[1])
        outs = []
        for st in steps_list:
            g = galois_elt(prm, st)
            if g == 1:
                outs.append(ct.copy())
                continue
            if g not in keys.gk:
                raise KeyError("no Galois key for step %d" % st)
            sig0 = np.zeros((1, nl, prm.N), dtype=np.uint64)
            lib().o_automorph(prm.cptr, P(np.ascontiguousarray(ct.data[:1])), nl, 1, g, P(sig0))
            ks = np.zeros((2, nl, prm.N), dtype=np.uint64)
            lib().o_keyswitch_g(prm.cptr, P(c1), nl, P(keys.gk[g]), g, P(ks))
            out = np.zeros_like(ct.data)
            o0 = np.zeros((nl, prm.N), dtype=np.uint64)
            lib().o_add(prm.cptr, P(np.ascontiguousarray(sig0[0])), P(np.ascontiguousarray(ks[0])), nl, 1, P(o0))
            out[0] = o0
            out[1] = ks[1]
            outs.append(Ct(out, ct.scale))
        return outs

    def plain_ntt(self, m, level):
        """NTT-form residues [level+1][N] of a signed integer plaintext m (int64[N])."""
        prm = self.prm
        pt = np.zeros((level + 1, prm.N), dtype=np.uint64)
        lib().o_int_to_ntt(prm.cptr, P(np.ascontiguousarray(m, dtype=np.int64)), level + 1,
                           P(np.arange(level + 1, dtype=np.int32)), P(pt))
        return pt

    def linear_transform(self, keys, ct, pts, steps, pt_scale):
        """Homomorphic diagonal-form matrix-vector product (reading R30; the linear transforms of CKKS
        bootstrapping's CoeffToSlot / SlotToCoeff, are products of these):
            out = Rescale( sum_i pt_i (.) RotL(ct, steps[i]) ),
        the rotations hoisted (R29, one ModUp), pt_i integer plaintexts in NTT form (encoded at pt_scale),
        the products summed exactly mod q, one rescale (R12).  Output scale (S_ct pt_scale) / q_level."""
        prm = self.prm
        if len(pts) != len(steps) or not steps:
            raise ValueError("one plaintext per step")
        rots = self.rotate_hoisted_raw(keys, ct, steps)
        nl = ct.level + 1
        acc = np.zeros((2, nl, prm.N), dtype=np.uint64)
        for r, pt in zip(rots, pts):
            prod = self.mul_plain_raw(r, pt)
            nxt = np.zeros_like(acc)
            lib().o_add(prm.cptr, P(acc), P(prod), nl, 2, P(nxt))
            acc = nxt
        return self.rescale(Ct(acc, ct.scale * pt_scale))

    def linear_transform_bsgs(self, keys, ct, pts, n1, n2, pt_scale):
        """Baby-step giant-step form of linear_transform (reading R31; how bootstrapping evaluates its
        dense CoeffToSlot / SlotToCoeff factors with about 2 sqrt(n) rotations instead of n):
            out = Rescale( sum_{g < n2} RotL( sum_{j < n1} pts[g][j] (.) RotL(ct, j), g n1 ) )
        the baby rotations hoisted (R29), the giant ones plain (O-12), every product and sum exact mod q,
        one rescale.  With pts[g][j] = encode(RotR(d_{g n1 + j}, g n1)) this is sum_i d_i (.) RotL(ct, i)."""
        prm = self.prm
        if len(pts) != n2 or any(len(r) != n1 for r in pts):
            raise ValueError("pts must be n2 lists of n1 plaintexts")
        nl = ct.level + 1
        baby = self.rotate_hoisted_raw(keys, ct, list(range(n1)))
        acc = None
        for g in range(n2):
            inner = np.zeros((2, nl, prm.N), dtype=np.uint64)
            for j in range(n1):
                prod = self.mul_plain_raw(baby[j], pts[g][j])
                nxt = np.zeros_like(inner)
                lib().o_add(prm.cptr, P(inner), P(prod), nl, 2, P(nxt))
                inner = nxt
            term = Ct(inner, ct.scale * pt_scale)
            if g:
                term = self.rotate_raw(keys, term, g * n1)
            if acc is None:
                acc = term.data
            else:
                nxt = np.zeros_like(acc)
                lib().o_add(prm.cptr, P(acc), P(term.data), nl, 2, P(nxt))
                acc = nxt
        return self.rescale(Ct(acc, ct.scale * pt_scale))

    def mod_raise(self, ct, level):
        """ModRaise (reading R33, the first step of CKKS bootstrapping): a level-0
        ciphertext (c0, c1) mod q_0 is read as the integer polynomials with centred coefficients in
        (-q_0/2, q_0/2] and reduced mod every prime of Q_level.  It then decrypts to
        t = c0 + c1 s = m + q_0 I over the integers, I a small integer polynomial (|I| <= (h+1)/2)."""
        if ct.level != 0:
            raise ValueError("mod_raise takes a level-0 ciphertext")
        prm = self.prm
        q0 = prm.primes[0]
        out = np.zeros((2, level + 1, prm.N), dtype=np.uint64)
        for i in range(2):
            coef = ntt_limbs(ct.data[i, :1], prm, [0], inverse=True)[0]
            v = np.array([int(c) - q0 if int(c) > (q0 - 1) // 2 else int(c) for c in coef], dtype=np.int64)
            out[i] = self.plain_ntt(v, level)
        r = Ct(out, ct.scale)
        self._log("MODRAISE", 0, level, ct.scale)
        return r

    def linear_transform_bsgs_gen(self, keys, ct, pts, baby, giant, pt_scale):
        """General baby-step giant-step transform (reading R39):
            out = Rescale( sum_g RotL( sum_j pts[g][j] (.) RotL(ct, baby[j]), giant[g] ) ),
        the baby rotations hoisted (R29), the giant ones plain (a zero giant step is no rotation), every
        product and sum exact mod q, the terms accumulated in g order.  With
        pts[g][j] = encode(RotR(d_{baby[j] + giant[g]}, giant[g])) this is sum_o d_o (.) RotL(ct, o)."""
        prm = self.prm
        if len(pts) != len(giant) or any(len(r) != len(baby) for r in pts):
            raise ValueError("pts must be len(giant) lists of len(baby) plaintexts")
        nl = ct.level + 1
        bab = self.rotate_hoisted_raw(keys, ct, list(baby))
        acc = None
        for g, G in enumerate(giant):
            inner = np.zeros((2, nl, prm.N), dtype=np.uint64)
            for j in range(len(baby)):
                prod = self.mul_plain_raw(bab[j], pts[g][j])
                nxt = np.zeros_like(inner)
                lib().o_add(prm.cptr, P(inner), P(prod), nl, 2, P(nxt))
                inner = nxt
            term = Ct(inner, ct.scale * pt_scale)
            if G:
                term = self.rotate_raw(keys, term, G)
            if acc is None:
                acc = term.data
            else:
                nxt = np.zeros_like(acc)
                lib().o_add(prm.cptr, P(acc), P(term.data), nl, 2, P(nxt))
                acc = nxt
        return self.rescale(Ct(acc, ct.scale * pt_scale))

    # ---- planned ops (logged; reading R9 scale planning) ------------------------------------
    def lt_gen(self, keys, x, pts, baby, giant, pt_scale):
        out = self.linear_transform_bsgs_gen(keys, x, pts, baby, giant, pt_scale)
        self._log("LTG", x.level, out.level, out.scale,
                  ",".join(str(s) for s in baby) + ";" + ",".join(str(s) for s in giant))
        return out

    def lt(self, keys, x, pts, steps, pt_scale):
        out = self.linear_transform(keys, x, pts, steps, pt_scale)
        self._log("LT", x.level, out.level, out.scale, ",".join(str(s) for s in steps))
        return out

    def lt_bsgs(self, keys, x, pts, n1, n2, pt_scale):
        out = self.linear_transform_bsgs(keys, x, pts, n1, n2, pt_scale)
        self._log("LTB", x.level, out.level, out.scale, "%dx%d" % (n1, n2))
        return out

    def rot(self, keys, x, steps):
        g = galois_elt(self.prm, steps)
        out = self.rotate_raw(keys, x, steps)
        self._log("ROT", x.level, out.level, out.scale, str(g))
        return out

    def add(self, a, b):
        out = self.add_raw(a, b)
        self._log("ADD", max(a.level, b.level), out.level, out.scale)
        return out

    def sub(self, a, b):
        out = self.sub_raw(a, b)
        self._log("SUB", max(a.level, b.level), out.level, out.scale)
        return out

    def mul_const(self, x, c, target_scale, target_level):
        """c * x landing at (target_scale, target_level): drop x to target_level + 1,
        Delta_c = (S_t * q_{l}) / S_x, C = rha(c * Delta_c), multiply, rescale, scale := S_t."""
        lv = target_level + 1
        x = self.drop(x, lv)
        dc = (target_scale * float(self.prm.primes[lv])) / x.scale
        C = round_half_away(c * dc)
        if abs(C) >= CONST_LIMIT:
            raise OverflowError("constant too large")
        y = Ct(self.mul_int_raw(x, C), x.scale * dc)
        out = self.rescale(y, target_scale)
        self._log("MULC", lv, target_level, target_scale, str(C))
        return out

    def lincomb(self, terms, target_scale, target_level):
        """sum_i c_i x_i landing at (target_scale, target_level) with ONE rescale (reading R13): every
        x_i dropped to l = target_level + 1, C_i = rha(c_i Delta_i), Delta_i = (S_t q_l) / S_{x_i},
        integer products summed mod q, rescale, scale := S_t."""
        lv = target_level + 1
        acc, Cs = None, []
        for x, c in terms:
            x = self.drop(x, lv)
            dc = (target_scale * float(self.prm.primes[lv])) / x.scale
            C = round_half_away(c * dc)
            if abs(C) >= CONST_LIMIT:
                raise OverflowError("constant too large")
            cx = self.mul_int_raw(x, C)
            if acc is None:
                acc = cx
            else:
                out = np.zeros_like(acc)
                lib().o_add(self.prm.cptr, P(acc), P(cx), lv + 1, 2, P(out))
                acc = out
            Cs.append(str(C))
        out = self.rescale(Ct(acc, target_scale * float(self.prm.primes[lv])), target_scale)
        self._log("LINC", lv, target_level, target_scale, ",".join(Cs))
        return out

    def mul_ct(self, keys, a, b, target_scale, target_level, lin=None, prod2=None):
        """a (x) b [+ a2 (x) b2] [+ sum c x]: drop the inputs to target_level + 1 = l, tensor, optionally add
        a second tensor a2 (x) b2 (prod2 = (a2, b2); reading R13b: two products summed share ONE
        relinearisation and rescale; needs a planned target scale), optionally add the constant products
        C x to (d0, d1) with C = rha(c Delta_c), Delta_c = (S_t q_l) / S_x (lin = (x, c) or a list of such
        terms; R9, R13), relinearise, rescale.  Output scale := target_scale if given else (S_a * S_b) / q_l."""
        lv = target_level + 1
        a = self.drop(a, lv)
        b = self.drop(b, lv)
        s = (a.scale * b.scale) / float(self.prm.primes[lv]) if target_scale is None else target_scale
        d = self.tensor(a, b)
        kind = "MULCT"
        if prod2 is not None:
            if target_scale is None:
                raise ValueError("a summed product needs a planned target scale")
            d2 = self.tensor(self.drop(prod2[0], lv), self.drop(prod2[1], lv))
            dsum = np.zeros_like(d)
            lib().o_add(self.prm.cptr, P(np.ascontiguousarray(d)), P(np.ascontiguousarray(d2)), lv + 1, 3, P(dsum))
            d = dsum
            kind = "MULCT2"
        extra = ""
        if lin is not None:
            terms = lin if isinstance(lin, list) else [lin]
            Cs = []
            for x, c in terms:
                x = self.drop(x, lv)
                dc = (s * float(self.prm.primes[lv])) / x.scale
                C = round_half_away(c * dc)
                if abs(C) >= CONST_LIMIT:
                    raise OverflowError("constant too large")
                cx = self.mul_int_raw(x, C)
                d01 = np.zeros((2, lv + 1, self.prm.N), dtype=np.uint64)
                lib().o_add(self.prm.cptr, P(np.ascontiguousarray(d[:2])), P(cx), lv + 1, 2, P(d01))
                d[:2] = d01
                Cs.append(str(C))
            extra = ",".join(Cs)
        out = self.rescale(self.mul_relin(keys, a, b, d), s)
        self._log(kind, lv, target_level, s, extra)
        return out

    def mul_mask(self, x, mask_slots, target_scale):
        """x * mask (plaintext), Delta_m = (S_t * q_l) / S_x, quantised encoding (R16), rescale."""
        prm = self.prm
        lv = x.level
        dm = (target_scale * float(prm.primes[lv])) / x.scale
        M = mask_coeffs(prm, mask_slots, dm)
        pt = np.zeros((lv + 1, prm.N), dtype=np.uint64)
        lib().o_int_to_ntt(prm.cptr, P(M), lv + 1, P(np.arange(lv + 1, dtype=np.int32)), P(pt))
        y = Ct(self.mul_plain_raw(x, pt), x.scale * dm)
        out = self.rescale(y, target_scale)
        self._log("MULP", lv, lv - 1, target_scale, dbits(dm))
        return out

    def add_const(self, x, c):
        C = round_half_away(c * x.scale)
        out = Ct(self.add_int_raw(x, C), x.scale)
        self._log("ADDC", x.level, x.level, x.scale, str(C))
        return out


# ---------------------------------------------------------------------------
# Plaintext mirror: the same planned ops on float slot vectors (O-16)
# ---------------------------------------------------------------------------
class MirrorCt:
    __slots__ = ("v", "level", "scale")

    def __init__(self, v, level, scale):
        self.v, self.level, self.scale = v, level, scale


class Mirror:
    """Executes the plan on doubles with identical level/scale bookkeeping; exact slot semantics."""

    def __init__(self, prm):
        self.prm = prm
        self.log = []
        self.counts = {}

    _log = Oracle._log

    def _check(self, a, b):
        if a.scale != b.scale:
            raise ValueError("scale mismatch")
        return min(a.level, b.level)

    def rot(self, keys, x, steps):
        out = MirrorCt(np.roll(x.v, -steps), x.level, x.scale)
        self._log("ROT", x.level, x.level, x.scale, str(galois_elt(self.prm, steps)))
        return out

    def add(self, a, b):
        lv = self._check(a, b)
        self._log("ADD", max(a.level, b.level), lv, a.scale)
        return MirrorCt(a.v + b.v, lv, a.scale)

    def sub(self, a, b):
        lv = self._check(a, b)
        self._log("SUB", max(a.level, b.level), lv, a.scale)
        return MirrorCt(a.v - b.v, lv, a.scale)

    def mul_const(self, x, c, target_scale, target_level):
        lv = target_level + 1
        if x.level < lv:
            raise ValueError("level")
        dc = (target_scale * float(self.prm.primes[lv])) / x.scale
        C = round_half_away(c * dc)
        self._log("MULC", lv, target_level, target_scale, str(C))
        return MirrorCt(c * x.v, target_level, target_scale)

    def lincomb(self, terms, target_scale, target_level):
        lv = target_level + 1
        v, Cs = 0.0, []
        for x, c in terms:
            if x.level < lv:
                raise ValueError("level")
            Cs.append(str(round_half_away(c * ((target_scale * float(self.prm.primes[lv])) / x.scale))))
            v = v + c * x.v
        self._log("LINC", lv, target_level, target_scale, ",".join(Cs))
        return MirrorCt(v, target_level, target_scale)

    def mul_ct(self, keys, a, b, target_scale, target_level, lin=None, prod2=None):
        lv = target_level + 1
        if a.level < lv or b.level < lv:
            raise ValueError("level")
        s = (a.scale * b.scale) / float(self.prm.primes[lv]) if target_scale is None else target_scale
        v = a.v * b.v
        kind = "MULCT"
        if prod2 is not None:
            if target_scale is None or prod2[0].level < lv or prod2[1].level < lv:
                raise ValueError("prod2")
            v = v + prod2[0].v * prod2[1].v
            kind = "MULCT2"
        extra = ""
        if lin is not None:
            terms = lin if isinstance(lin, list) else [lin]
            Cs = []
            for x, c in terms:
                if x.level < lv:
                    raise ValueError("level")
                Cs.append(str(round_half_away(c * ((s * float(self.prm.primes[lv])) / x.scale))))
                v = v + c * x.v
            extra = ",".join(Cs)
        self._log(kind, lv, target_level, s, extra)
        return MirrorCt(v, target_level, s)

    def mul_mask(self, x, mask_slots, target_scale):
        lv = x.level
        dm = (target_scale * float(self.prm.primes[lv])) / x.scale
        self._log("MULP", lv, lv - 1, target_scale, dbits(dm))
        return MirrorCt(x.v * mask_slots, lv - 1, target_scale)

    def add_const(self, x, c):
        C = round_half_away(c * x.scale)
        self._log("ADDC", x.level, x.level, x.scale, str(C))
        return MirrorCt(x.v + c, x.level, x.scale)
