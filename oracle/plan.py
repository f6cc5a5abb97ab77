"""Oracle circuit plans: composite Sign (Eq. 4 + BSGS), Max (Eq. 6), Algorithm 1 Argmax.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The plan is written once here and
executed by either ``ckks.Oracle`` (ciphertexts) or ``ckks.Mirror`` (plaintext doubles);
both log the same op list, which tests diff against the CUDA library's own planner.

Reading R13: odd polynomials in the power basis, evaluated with the fixed
BSGS plans below (degrees 3, 7, 15).  A linear term c x that is summed with a ct x ct
product enters that product before its rescale (one rescale instead of two).  Every sub-expression is requested at a target
(scale, level) and computed as low as possible: a constant product drops its input to
target+1 first; a ct x ct product drops both inputs to target+1.  Emission order is
"first operand first" exactly as written here.
"""
import math

import numpy as np

CONJ_STEP = -(2 ** 31)  # = ckks.CONJ: slot conjugation (reading R32)


def poly_depth(deg):
    """Multiplicative depth of the plan for an odd degree-`deg` polynomial: ceil(log2(deg+1)) for the
    BSGS plans of degree 3 and 7, one more for degree 15 (Paterson-Stockmeyer with a shared x^3:
    7 ct x ct products instead of 10, reading R13)."""
    return 5 if deg == 15 else int(math.ceil(math.log2(deg + 1)))


def eval_odd_poly(ev, keys, x, coeffs, target_scale):
    """p(x) = sum_i c_i x^i (odd, degree 3, 7 or 15) landing at level x.level - depth, scale target_scale.

    PAPER.md:195 ("we evaluate the polynomials using the Baby-Step-Giant-Step algorithm").
    Powers x^2, x^4, x^8 carry their natural scales; the constants absorb every deviation
    (reading R9) so each sum has bit-identical operand scales.
    """
    deg = len(coeffs) - 1
    if deg not in (3, 7, 15):
        raise ValueError("supported odd degrees: 3, 7, 15")
    for i in range(0, deg + 1, 2):
        if coeffs[i] != 0.0:
            raise ValueError("sign polynomials must be odd")
    prm = ev.prm
    q = lambda lv: float(prm.primes[lv])
    l = x.level
    x2 = ev.mul_ct(keys, x, x, None, l - 1)
    x4 = ev.mul_ct(keys, x2, x2, None, l - 2) if deg >= 7 else None
    x8 = ev.mul_ct(keys, x4, x4, None, l - 3) if deg >= 15 else None

    def A(i, S, L):
        # A_i = (c_{4i+3} x) * x^2 + c_{4i+1} x  at (S, L); the linear term joins the product
        # before its (fused) rescale (reading R13)
        inner = ev.mul_const(x, coeffs[4 * i + 3], (S * q(L + 1)) / x2.scale, L + 1)
        return ev.mul_ct(keys, inner, x2, S, L, lin=(x, coeffs[4 * i + 1]))

    def B(i, S, L):
        # B_i = x^4 A_{2i+1} + A_{2i}  at (S, L); A_{2i} = (c x) x^2 + c' x is a second product summed
        # with the first: both tensors share ONE relinearisation and rescale (reading R13b)
        hi = A(2 * i + 1, (S * q(L + 1)) / x4.scale, L + 1)
        inner = ev.mul_const(x, coeffs[8 * i + 3], (S * q(L + 1)) / x2.scale, L + 1)
        return ev.mul_ct(keys, hi, x4, S, L, lin=(x, coeffs[8 * i + 1]), prod2=(inner, x2))

    if deg == 3:
        return A(0, target_scale, l - 2)
    if deg == 7:
        return B(0, target_scale, l - 3)
    # degree 15, Paterson-Stockmeyer (R13): baby steps x, x^3 (shared), giant steps x^4, x^8;
    # q_k = c_{4k+1} x + c_{4k+3} x^3 are linear combinations (one rescale each, or folded into the
    # product they are summed with); p = (q_1 x^4 + q_0) + (q_3 x^4 + q_2) x^8 at depth 5
    T, Lo = target_scale, l - 5
    x3 = ev.mul_ct(keys, x, x2, None, l - 2)
    c = coeffs
    S_b1 = (T * q(l - 4)) / x8.scale
    q3 = ev.lincomb([(x, c[13]), (x3, c[15])], (S_b1 * q(l - 3)) / x4.scale, l - 3)
    b1 = ev.mul_ct(keys, q3, x4, S_b1, l - 4, lin=[(x, c[9]), (x3, c[11])])
    q1 = ev.lincomb([(x, c[5]), (x3, c[7])], (T * q(l - 4)) / x4.scale, l - 4)
    # q_1 x^4 + q_0 + b_1 x^8: the two products share one relinearisation and rescale (reading R13b)
    return ev.mul_ct(keys, q1, x4, T, Lo, lin=[(x, c[1]), (x3, c[3])], prod2=(b1, x8))


def sign(ev, keys, x, stages, target_scale):
    """Composite Sign = p_r o ... o p_1 (Eq. 4).  Every stage lands at the
    nominal scale except the last, which lands at target_scale."""
    for i, c in enumerate(stages):
        s = target_scale if i == len(stages) - 1 else ev.prm.scale
        x = eval_odd_poly(ev, keys, x, c, s)
    return x


def sign_depth(stages):
    return sum(poly_depth(len(c) - 1) for c in stages)


def hom_max(ev, keys, r, y, stages):
    """Max(r, y) = (r + y)/2 + (r - y)/2 * Sign(r - y)  (Eq. 6).
    The halves are constant products (reading R8); output scale = y's scale."""
    Sy = y.scale
    d = ev.sub(r, y)
    s = sign(ev, keys, d, stages, ev.prm.scale)
    Ls = s.level
    g = ev.mul_const(d, 0.5, (Sy * float(ev.prm.primes[Ls])) / s.scale, Ls)
    ry = ev.add(r, y)
    # (r - y)/2 * Sign(r - y) + (r + y)/2: the half-sum joins the product before its rescale
    return ev.mul_ct(keys, g, s, Sy, Ls - 1, lin=(ry, 0.5))


def mask_slots(layout, n_slots):
    """Plaintext mask of H2: 1/P on slot q*block + k (k < K), 0 elsewhere (Eq. 5 with D_min = 0,
    D_max = P folded in; reading R15)."""
    m = np.zeros(n_slots)
    P, K, b, nq = layout["prompts"], layout["classes"], layout["block"], layout["queries"]
    for qi in range(nq):
        m[qi * b: qi * b + K] = 1.0 / P
    return m


def check_layout(layout, n_slots):
    P, K, b, nq = layout["prompts"], layout["classes"], layout["block"], layout["queries"]
    for v in (P, K):
        if v < 1 or v & (v - 1):
            raise ValueError("prompts and classes must be powers of two (pad, reading R17)")
    if P * K > b or 2 * K > b or nq * b > n_slots:
        raise ValueError("layout does not fit")


def argmax(ev, keys, y, layout, stages):
    """SecPE private voting on one packed ciphertext (Algorithm 1 :214-235).

    H1  y <- sum over prompts by rotate-and-sum, RotL(y, K 2^t)
    H2  y <- y * mask/P (Eq. 5 normalisation, zero the non-window slots)
    H3  y <- y + RotR(y, K)                                  (Alg. 1 line 2)
    H4  for i < log2 K: y <- Max(RotL(y, 2^i), y)            (QuickMax, lines 9-16)
    H6  z <- Sign(y_dup - y_max) + 1                         (lines 3-6, Eq. 2)
    """
    P, K = layout["prompts"], layout["classes"]
    n_slots = ev.prm.N // 2
    check_layout(layout, n_slots)
    for t in range(int(math.log2(P))):
        y = ev.add(y, ev.rot(keys, y, K << t))
    y = ev.mul_mask(y, mask_slots(layout, n_slots), ev.prm.scale)
    y = ev.add(y, ev.rot(keys, y, -K))
    ydup = y
    for i in range(int(math.log2(K))):
        y = hom_max(ev, keys, ev.rot(keys, y, 1 << i), y, stages)
    d = ev.sub(ydup, y)
    z = sign(ev, keys, d, stages, ev.prm.scale)
    return ev.add_const(z, 1.0)


def argmax_rotations(layout):
    """Rotation steps the argmax circuit needs (keys to generate)."""
    P, K = layout["prompts"], layout["classes"]
    steps = [K << t for t in range(int(math.log2(P)))] + [-K] + [1 << i for i in range(int(math.log2(K)))]
    return sorted(set(steps))


def argmax_depth(layout, stages):
    K = layout["classes"]
    return 1 + int(math.log2(K)) * (sign_depth(stages) + 1) + sign_depth(stages)


def pack(scores, layout, n_slots):
    """H0 client packing: score[q, p, k] -> slot q*block + p*K + k."""
    P, K, b = layout["prompts"], layout["classes"], layout["block"]
    z = np.zeros(n_slots)
    nq = scores.shape[0]
    for qi in range(nq):
        for p in range(P):
            z[qi * b + p * K: qi * b + p * K + K] = scores[qi, p]
    return z


def labels(z, layout):
    """Client decode (reading R5/A5): argmax over each query's K window slots, first index on ties."""
    K, b, nq = layout["classes"], layout["block"], layout["queries"]
    return np.array([int(np.argmax(np.real(z[qi * b: qi * b + K]))) for qi in range(nq)])


def true_labels(scores):
    """Plaintext truth: argmax of the mean-over-prompts scores, first index on ties."""
    return np.argmax(scores.mean(axis=1), axis=1)


# ---------------------------------------------------------------------------------------------
# CKKS bootstrapping (the paper bootstraps with L = 35, K = 14, PAPER.md:94-96,
# :327).  Readings R32-R35: conjugation, ModRaise, dense CoeffToSlot / SlotToCoeff as
# baby-step giant-step linear transforms (R31), EvalMod as 2 cos((2 pi K x - pi/2) / 2^r) followed
# by r double-angle steps d <- d^2 - 2.
# ---------------------------------------------------------------------------------------------
def eval_poly15(ev, keys, x, c, target_scale):
    """General degree-15 p(x) = sum_i c_i x^i landing at level x.level - 5, scale target_scale (R35).

    The odd plan's Paterson-Stockmeyer shape (R13) with the even terms added: baby steps x, x^2, x^3,
    giant steps x^4, x^8; q_k = c_{4k} + c_{4k+1} x + c_{4k+2} x^2 + c_{4k+3} x^3 (a two-term linear
    combination, a one-term one and a constant); p = (q_0 + q_1 x^4) + (q_2 + q_3 x^4) x^8."""
    if len(c) != 16:
        raise ValueError("degree-15 coefficients c_0..c_15")
    prm = ev.prm
    q = lambda lv: float(prm.primes[lv])
    l = x.level
    T, Lo = target_scale, l - 5
    x2 = ev.mul_ct(keys, x, x, None, l - 1)
    x3 = ev.mul_ct(keys, x, x2, None, l - 2)
    x4 = ev.mul_ct(keys, x2, x2, None, l - 2)
    x8 = ev.mul_ct(keys, x4, x4, None, l - 3)
    S_b1 = (T * q(l - 4)) / x8.scale
    S_q3 = (S_b1 * q(l - 3)) / x4.scale
    q3 = ev.lincomb([(x, c[13]), (x3, c[15])], S_q3, l - 3)
    q3 = ev.add_const(ev.add(q3, ev.lincomb([(x2, c[14])], S_q3, l - 3)), c[12])
    b1 = ev.mul_ct(keys, q3, x4, S_b1, l - 4, lin=[(x, c[9]), (x3, c[11])])
    b1 = ev.add_const(ev.add(b1, ev.lincomb([(x2, c[10])], S_b1, l - 4)), c[8])
    S_q1 = (T * q(l - 4)) / x4.scale
    q1 = ev.lincomb([(x, c[5]), (x3, c[7])], S_q1, l - 4)
    q1 = ev.add_const(ev.add(q1, ev.lincomb([(x2, c[6])], S_q1, l - 4)), c[4])
    p = ev.mul_ct(keys, q1, x4, T, Lo, lin=[(x, c[1]), (x3, c[3])], prod2=(b1, x8))
    return ev.add_const(ev.add(p, ev.lincomb([(x2, c[2])], T, Lo)), c[0])


def boot_poly(K, r):
    """Power-basis coefficients c_0..c_15 of 2 cos(a x + b), a = 2 pi K / 2^r, b = -pi / 2^(r+1), on
    [-1, 1] (R35): its Taylor series at 0, c_i = 2 a^i cos(b + i pi / 2) / i!, truncated after x^15
    (remainder <= 2 a^16 / 16!; every coefficient exact to a double's rounding)."""
    a = 2.0 * math.pi * K / 2.0 ** r
    b = -math.pi / 2.0 ** (r + 1)
    return [2.0 * a ** i * math.cos(b + i * math.pi / 2) / math.factorial(i) for i in range(16)]


def boot_depth(r):
    """Levels one bootstrap consumes: CoeffToSlot 1, normalisation 1, polynomial 5, r doublings,
    SlotToCoeff 1."""
    return 8 + r


def boot_rotations(n1, n2):
    """Galois keys bootstrapping needs: baby steps 1..n1-1, giant steps n1, 2 n1, ..., conjugation."""
    return list(range(1, n1)) + [g * n1 for g in range(1, n2)] + [CONJ_STEP]


def boot_matrices(prm, R):
    """Slot-domain matrices (R34), n = N/2, e_j = 5^j mod 2N, zeta = e^{i pi / N}:
    A[k, j] = zeta^{-e_j k} / n (encode's inverse: (A z)_k = t_k + i t_{k+n} for the real integer
    polynomial t behind the slots z, both divided by the scale), U[j, k] = zeta^{e_j k} (decode).
    CoeffToSlot: A/2 and -i A/2 (u + conj(u) then gives Re and Im of A z);
    SlotToCoeff: c U and i c U with c = R / (4 pi) (the doubled cosine's 2 and EvalMod's R / 2 pi)."""
    from oracle.ckks import _rot_group
    N, n = prm.N, prm.N // 2
    e = _rot_group(N).astype(np.int64)
    k = np.arange(n, dtype=np.int64)
    # zeta^m with the exponent m = e_j k reduced mod 2N exactly (zeta^{2N} = 1) before the angle is formed
    A = np.exp(-1j * np.pi * (np.outer(k, e) % (2 * N)).astype(np.float64) / N) / n
    U = np.exp(1j * np.pi * (np.outer(e, k) % (2 * N)).astype(np.float64) / N)
    c = R / (4.0 * np.pi)
    return dict(cts_re=A / 2, cts_im=-0.5j * A, stc_re=c * U, stc_im=1j * c * U)


def bsgs_pts(ev, M, n1, n2, level, pt_scale):
    """pts[g][j] = NTT(encode(RotR(d_{g n1 + j}, g n1), pt_scale)) at `level`, d_i[t] = M[t, (t + i) mod n]
    (R30/R31)."""
    from oracle.ckks import encode
    n = M.shape[0]
    if n1 * n2 != n:
        raise ValueError("n1 n2 must equal the slot count")
    t = np.arange(n)
    out = []
    for g in range(n2):
        row = []
        for j in range(n1):
            i = g * n1 + j
            d = M[t, (t + i) % n]
            row.append(ev.plain_ntt(encode(ev.prm, np.roll(d, g * n1), pt_scale), level))
        out.append(row)
    return out


def boot_config(ev, in_scale, level, K, r, n1, n2):
    """Everything the bootstrap plan takes besides the ciphertext: the EvalMod range K and doublings r,
    the BSGS split, the polynomial and the four encoded matrices at their levels and scales."""
    prm = ev.prm
    R = float(prm.primes[0]) / in_scale
    Ms = boot_matrices(prm, R)
    l_stc = level - 7 - r
    cts_scale, stc_scale = float(prm.primes[level]), float(prm.primes[l_stc])
    cfg = dict(level=level, K=float(K), r=r, n1=n1, n2=n2, poly=boot_poly(K, r), cts_scale=cts_scale,
               stc_scale=stc_scale, stc_level=l_stc)
    for name in ("cts_re", "cts_im"):
        cfg[name] = bsgs_pts(ev, Ms[name], n1, n2, level, cts_scale)
    for name in ("stc_re", "stc_im"):
        cfg[name] = bsgs_pts(ev, Ms[name], n1, n2, l_stc, stc_scale)
    return cfg


def bootstrap(ev, keys, ct, cfg):
    """CKKS bootstrapping of a level-0 ciphertext (readings R32-R35):
      ModRaise to cfg level L                          t = m + q_0 I
      CoeffToSlot (two BSGS transforms)                u = A z / 2, u' = -i A z / 2
      x = u + conj(u), x' = u' + conj(u')              slots t_k / S and t_{k+n} / S
      normalise x / (K R), R = q_0 / S                 in [-1, 1]
      d = 2 cos((2 pi K x - pi/2) / 2^r), r times d <- d^2 - 2    d = 2 sin(2 pi t / q_0)
      SlotToCoeff (two BSGS transforms, summed)        z = U (d_re + i d_im) R / (4 pi)
    The output decrypts to the input's slots at a higher level."""
    prm = ev.prm
    L, K, r, n1, n2 = cfg["level"], cfg["K"], cfg["r"], cfg["n1"], cfg["n2"]
    S0 = ct.scale
    z = ev.mod_raise(ct, L)
    us = [ev.lt_bsgs(keys, z, cfg[nm], n1, n2, cfg["cts_scale"]) for nm in ("cts_re", "cts_im")]
    inv = 1.0 / (K * (float(prm.primes[0]) / S0))
    ds = []
    for u in us:
        x = ev.add(u, ev.rot(keys, u, CONJ_STEP))
        xn = ev.mul_const(x, inv, S0, x.level - 1)  # EvalMod runs at the input's scale (R38)
        d = eval_poly15(ev, keys, xn, cfg["poly"], S0)
        for _ in range(r):
            d = ev.add_const(ev.mul_ct(keys, d, d, None, d.level - 1), -2.0)  # natural scale (R9)
        ds.append(d)
    o_re = ev.lt_bsgs(keys, ds[0], cfg["stc_re"], n1, n2, cfg["stc_scale"])
    o_im = ev.lt_bsgs(keys, ds[1], cfg["stc_im"], n1, n2, cfg["stc_scale"])
    return ev.add(o_re, o_im)


# ---------------------------------------------------------------------------------------------
# Factorised CoeffToSlot / SlotToCoeff (reading R37): the decoding matrix U as log2(n) butterfly stages
# (the special FFT) in slot-domain diagonal form, consecutive stages merged into groups; the slots then
# hold the coefficients in bit-reversed order, which EvalMod (slot-wise) does not see.
# ---------------------------------------------------------------------------------------------
def bitrev_perm(n):
    b = n.bit_length() - 1
    return np.array([int(format(i, "0%db" % b)[::-1], 2) for i in range(n)])


def dft_stages(N):
    """Butterfly stage s = 1..log2 n of the special FFT as {offset: diagonal} (slot-domain, cyclic offsets
    mod n), len = 2^s, h = len/2, for block start i and j < h:
        out[i+j] = v[i+j] + w_j v[i+j+h],  out[i+j+h] = v[i+j] - w_j v[i+j+h],
        w_j = zeta^{(e_j mod 4 len) 2N / (4 len)}, e_j = 5^j mod 2N.
    U w = S_log2n ... S_1 (w in bit-reversed order) (pinned in the tests)."""
    from oracle.ckks import _rot_group
    n = N // 2
    e = _rot_group(N)
    out = []
    ln = 2
    while ln <= n:
        h = ln // 2
        d0, dp, dm = np.zeros(n, complex), np.zeros(n, complex), np.zeros(n, complex)
        for i in range(0, n, ln):
            for j in range(h):
                m = (int(e[j]) % (4 * ln)) * (2 * N // (4 * ln))
                w = np.exp(1j * np.pi * m / N)
                d0[i + j], dp[i + j] = 1.0, w          # out[i+j] = v[i+j] + w v[i+j+h]
                dm[i + j + h], d0[i + j + h] = 1.0, -w  # out[i+j+h] = v[i+j] - w v[i+j+h]
        out.append({0: d0, h % n: dp, (n - h) % n: dm} if h != n - h else {0: d0, h: dp + dm})
        ln *= 2
    return out


def dft_stages_inv(N):
    """Inverses of dft_stages: in[i+j] = (o[i+j] + o[i+j+h]) / 2, in[i+j+h] = (o[i+j] - o[i+j+h]) / (2 w_j)."""
    from oracle.ckks import _rot_group
    n = N // 2
    e = _rot_group(N)
    out = []
    ln = 2
    while ln <= n:
        h = ln // 2
        d0, dp, dm = np.zeros(n, complex), np.zeros(n, complex), np.zeros(n, complex)
        for i in range(0, n, ln):
            for j in range(h):
                m = (int(e[j]) % (4 * ln)) * (2 * N // (4 * ln))
                wi = np.exp(-1j * np.pi * m / N)
                d0[i + j], dp[i + j] = 0.5, 0.5
                dm[i + j + h], d0[i + j + h] = 0.5 * wi, -0.5 * wi
        out.append({0: d0, h % n: dp, (n - h) % n: dm} if h != n - h else {0: d0, h: dp + dm})
        ln *= 2
    return out


def diag_mul(A, B, n):
    """Diagonal form of the product A B (A applied last): (A B) v = sum_{a,b} (alpha_a (.) RotL(beta_b, a))
    (.) RotL(v, a + b), offsets mod n."""
    out = {}
    for a, al in A.items():
        for b, be in B.items():
            k = (a + b) % n
            out[k] = out.get(k, 0) + al * np.roll(be, -a)
    return out


def diag_apply(D, v):
    """sum_i d_i (.) RotL(v, i) (plaintext, for pins)."""
    return sum(d * np.roll(v, -i) for i, d in D.items())


def fft_groups(N, groups):
    """Merged stage groups.  groups: stage counts summing to log2(n), in the order SlotToCoeff applies them
    (S_1 first).  Returns (stc, cts): stc[g] = product of its stages (later stages applied last);
    cts = inverses in the reverse order (CoeffToSlot applies cts[0] first)."""
    n = N // 2
    st, si = dft_stages(N), dft_stages_inv(N)
    if sum(groups) != len(st):
        raise ValueError("groups must cover log2(N/2) stages")
    stc, cts, pos = [], [], 0
    for g in groups:
        D = {0: np.ones(n, complex)}
        Di = {0: np.ones(n, complex)}
        for s in range(pos, pos + g):
            D = diag_mul({k: v for k, v in st[s].items()}, D, n)     # S_s applied after the previous ones
            Di = diag_mul(Di, {k: v for k, v in si[s].items()}, n)   # S_s^-1 applied before the previous
        stc.append(D)
        cts.append(Di)
        pos += g
    return stc, cts[::-1]


def _signed(k, n):
    return k - n if k > n // 2 else k


def lt_pts(ev, D, level, pt_scale):
    """(steps, pts) of a diagonal-form transform for linear_transform (R30): steps the signed offsets
    (sorted), pts[i] = NTT(encode(d_i, pt_scale)) at `level`."""
    from oracle.ckks import encode
    n = ev.prm.N // 2
    keys = sorted(D, key=lambda k: _signed(k, n))
    steps = [_signed(k, n) for k in keys]
    pts = [ev.plain_ntt(encode(ev.prm, D[k], pt_scale), level) for k in keys]
    return steps, pts


def bsgs_split(D, n):
    """Baby-step giant-step split of a diagonal set whose signed offsets are the multiples u k,
    k_min <= k <= k_max, of one step u (every merged special-FFT group is, R39): n1 = the power of two
    >= sqrt(count), baby u j (j < n1), giant u (k_min + n1 g) (g < ceil(count / n1)).  Returns
    (baby, giant, {(g, j): offset key or None}) -- None where k > k_max (a zero diagonal)."""
    offs = sorted(_signed(k, n) for k in D)
    nz = [abs(o) for o in offs if o]
    u = 0
    for o in nz:
        u = math.gcd(u, o)
    u = u or 1
    ks = [o // u for o in offs]
    kmin, kmax = ks[0], ks[-1]
    if ks != list(range(kmin, kmax + 1)):
        raise ValueError("offsets are not a contiguous progression")
    cnt = kmax - kmin + 1
    n1 = 1
    while n1 * n1 < cnt:
        n1 *= 2
    n2 = -(-cnt // n1)
    baby = [u * j for j in range(n1)]
    giant = [u * (kmin + n1 * g) for g in range(n2)]
    where = {}
    for g in range(n2):
        for j in range(n1):
            k = kmin + n1 * g + j
            where[(g, j)] = (u * k) % n if k <= kmax else None
    return baby, giant, where


def lt_bsgs_pts(ev, D, level, pt_scale):
    """(baby, giant, pts) of a diagonal-form transform for linear_transform_bsgs_gen (R39):
    pts[g][j] = NTT(encode(RotR(d_{baby_j + giant_g}, giant_g), pt_scale)), zero where no diagonal."""
    from oracle.ckks import encode
    n = ev.prm.N // 2
    baby, giant, where = bsgs_split(D, n)
    pts = []
    for g, G in enumerate(giant):
        row = []
        for j in range(len(baby)):
            k = where[(g, j)]
            d = D[k] if k is not None else np.zeros(n, complex)
            row.append(ev.plain_ntt(encode(ev.prm, np.roll(d, G), pt_scale), level))
        pts.append(row)
    return baby, giant, pts


def fft_boot_config(ev, in_scale, level, K, r, groups, bsgs=False):
    """Factorised bootstrapping material (R37): CoeffToSlot stages (the last one in a Re (x 1/2) and an Im
    (x -i/2) variant), SlotToCoeff stages (the first one in a Re (x c) and an Im (x i c) variant, c = R/(4 pi)),
    each encoded at q of its level."""
    prm = ev.prm
    n = prm.N // 2
    R = float(prm.primes[0]) / in_scale
    c = R / (4.0 * np.pi)
    stc, cts = fft_groups(prm.N, groups)
    mc, ms = len(cts), len(stc)
    cfg = dict(level=level, K=float(K), r=r, poly=boot_poly(K, r), groups=list(groups), cts=[], stc=[])
    enc = lt_bsgs_pts if bsgs else lt_pts
    lv = level
    for i, D in enumerate(cts):
        sc = float(prm.primes[lv])
        if i < mc - 1:
            cfg["cts"].append((*enc(ev, D, lv, sc), sc))
        else:
            cfg["cts"].append((*enc(ev, {k: 0.5 * v for k, v in D.items()}, lv, sc), sc))
            cfg["cts_im"] = (*enc(ev, {k: -0.5j * v for k, v in D.items()}, lv, sc), sc)
        lv -= 1
    lv = level - mc - 6 - r
    cfg["stc_level"] = lv
    for i, D in enumerate(stc):
        sc = float(prm.primes[lv])
        if i == 0:
            cfg["stc"].append((*enc(ev, {k: c * v for k, v in D.items()}, lv, sc), sc))
            cfg["stc_im"] = (*enc(ev, {k: 1j * c * v for k, v in D.items()}, lv, sc), sc)
        else:
            cfg["stc"].append((*enc(ev, D, lv, sc), sc))
        lv -= 1
    return cfg


def fft_boot_depth(groups, r):
    return 2 * len(groups) + 6 + r


def fft_boot_rotations(N, groups, bsgs=False):
    """Galois keys the factorised bootstrap needs: every nonzero offset of every group (diagonal form) or
    every nonzero baby and giant step (R39), and conjugation."""
    n = N // 2
    stc, cts = fft_groups(N, groups)
    s = set()
    for D in stc + cts:
        if bsgs:
            baby, giant, _ = bsgs_split(D, n)
            s |= {x for x in baby + giant if x % n}
        else:
            s |= {_signed(k, n) for k in D if k % n}
    return sorted(s) + [CONJ_STEP]


def _lt_stage(ev, keys, x, t):
    """A stage of bootstrap_fft: (steps, pts, scale) diagonal form (R30) or (baby, giant, pts, scale) (R39)."""
    if len(t) == 3:
        return ev.lt(keys, x, t[1], t[0], t[2])
    return ev.lt_gen(keys, x, t[2], t[0], t[1], t[3])


def bootstrap_fft(ev, keys, ct, cfg):
    """Bootstrapping with the factorised transforms (R37; otherwise as `bootstrap`, R32-R36):
    ModRaise; CoeffToSlot stages (hoisted diagonal transforms, R30), the last in Re / Im variants;
    x = u + conj(u); x / (K R); doubled cosine; r doublings; SlotToCoeff's first stage on d_re and d_im,
    summed; the remaining SlotToCoeff stages."""
    prm = ev.prm
    L, K, r = cfg["level"], cfg["K"], cfg["r"]
    S0 = ct.scale
    v = ev.mod_raise(ct, L)
    for t in cfg["cts"][:-1]:
        v = _lt_stage(ev, keys, v, t)
    us = [_lt_stage(ev, keys, v, cfg["cts"][-1]), _lt_stage(ev, keys, v, cfg["cts_im"])]
    inv = 1.0 / (K * (float(prm.primes[0]) / S0))
    ds = []
    for u in us:
        x = ev.add(u, ev.rot(keys, u, CONJ_STEP))
        xn = ev.mul_const(x, inv, S0, x.level - 1)  # EvalMod runs at the input's scale (R38)
        d = eval_poly15(ev, keys, xn, cfg["poly"], S0)
        for _ in range(r):
            d = ev.add_const(ev.mul_ct(keys, d, d, None, d.level - 1), -2.0)
        ds.append(d)
    o = _lt_stage(ev, keys, ds[0], cfg["stc"][0])
    o = ev.add(o, _lt_stage(ev, keys, ds[1], cfg["stc_im"]))
    for t in cfg["stc"][1:]:
        o = _lt_stage(ev, keys, o, t)
    return o


# ---------------------------------------------------------------------------------------------
# N4: Argmax over K classes when the level budget runs out (K = 16 needs 4 comparisons of
# 12 levels each plus the final Sign), with a bootstrap (R37) before every comparison
# that would not fit (reading R38).
# ---------------------------------------------------------------------------------------------
def argmax_boot(ev, keys, y, layout, stages, boot, boot_scale, prompt_cts=1):
    """Algorithm 1 as `argmax`, refreshing y (before a Max) or y_dup - y_max (before the final Sign) when
    fewer levels remain than the step needs (a Max keeps one level for the next refresh): one constant
    product by 1 landing at level 0 and scale boot_scale (the scale the bootstrap material expects),
    boot(ct), then one constant product by 1 back to the nominal scale (so that y_dup - y_max sees
    bit-identical scales).

    prompt_cts > 1 (CLIP-scale prompt counts): y is a list of prompt_cts ciphertexts holding
    disjoint prompt sets in the same layout; H1 first sums them in list order (y* = sum y_i),
    and the mask normalises by prompts x prompt_cts (Eq. 5 with D_max = the total prompt count)."""
    P, K = layout["prompts"], layout["classes"]
    n_slots = ev.prm.N // 2
    check_layout(layout, n_slots)
    if prompt_cts > 1:
        if len(y) != prompt_cts:
            raise ValueError("one ciphertext per prompt group")
        acc = y[0]
        for c in y[1:]:
            acc = ev.add(acc, c)
        y = acc
    for t in range(int(math.log2(P))):
        y = ev.add(y, ev.rot(keys, y, K << t))
    y = ev.mul_mask(y, mask_slots(layout, n_slots) / prompt_cts, ev.prm.scale)
    y = ev.add(y, ev.rot(keys, y, -K))
    ydup = y
    sd = sign_depth(stages)

    def refresh(x):
        b = boot(ev.mul_const(x, 1.0, boot_scale, 0))
        return ev.mul_const(b, 1.0, ev.prm.scale, b.level - 1)
    for i in range(int(math.log2(K))):
        if y.level < sd + 2:
            y = refresh(y)
        y = hom_max(ev, keys, ev.rot(keys, y, 1 << i), y, stages)
    d = ev.sub(ydup, y)
    if d.level < sd:
        d = refresh(d)
    z = sign(ev, keys, d, stages, ev.prm.scale)
    return ev.add_const(z, 1.0)
