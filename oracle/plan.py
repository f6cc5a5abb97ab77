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
