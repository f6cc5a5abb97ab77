// ks.cu -- hybrid key switching (ModUp fast base conversion, key inner product, ModDown)
// and rescale kernels.  Readings R10/R11/R12 in DESIGN.md; PAPER.md:103-105 (relinearisation
// and rotation need key switching), PAPER.md:90-94 (leveled modulus chain / rescale).
//
// Base conversions accumulate the alpha (or k) 120-bit products lazily in 128 bits and
// reduce once with Barrett; the per-source factor [x (Q'/q_i)^-1]_{q_i} is a Shoup product.
#include "common.cuh"
#include "kernels.h"
#include "fpk.cuh"

namespace {
constexpr int TPB = 256;
constexpr int MAXA = 16;  // max primes per digit / special primes

// Split-30 multiply-accumulate for base conversion.  Every residue is < 2^60, so writing
// y = yh 2^30 + yl and c = ch 2^30 + cl (all halves < 2^30) gives four 32x32->64 partial products
// < 2^60 each; up to 16 of them accumulate in a 64-bit register without overflow (IMAD.WIDE.U32 with
// a 64-bit addend, one instruction each).  V = s3 2^60 + (s1 + s2) 2^30 + s0 < 2^125 is then reduced
// once with Barrett.  Constants are stored packed as (ch << 32) | cl.
struct Acc4 {
    u64 s0, s1, s2, s3;
};
__device__ __forceinline__ void acc4_zero(Acc4 &a) { a.s0 = a.s1 = a.s2 = a.s3 = 0; }
__device__ __forceinline__ void acc4_mac(Acc4 &a, uint32_t yl, uint32_t yh, u64 cpk) {
    const uint32_t cl = (uint32_t)cpk, ch = (uint32_t)(cpk >> 32);
    a.s0 += (u64)yl * cl;
    a.s1 += (u64)yl * ch;
    a.s2 += (u64)yh * cl;
    a.s3 += (u64)yh * ch;
}
__device__ __forceinline__ u64 acc4_reduce(const Acc4 &a, u64 q, u64 r0, u64 r1) {
    const u128 m = (u128)a.s1 + a.s2;
    const u128 v = ((u128)a.s3 << 60) + (m << 30) + a.s0;
    return barrett128(U128{(u64)v, (u64)(v >> 64)}, q, r0, r1);
}
constexpr uint32_t M30 = (1u << 30) - 1;

__device__ __forceinline__ ulonglong2 ldv2(const u64 *p) { return *reinterpret_cast<const ulonglong2 *>(p); }
__device__ __forceinline__ void stv2(u64 *p, u64 a, u64 b) { *reinterpret_cast<ulonglong2 *>(p) = make_ulonglong2(a, b); }

// ModUp (R10).  grid: x = coefficient chunks (two coefficients per thread), y = ct * beta + j.
// The digit's packed constants [Q'_j/q_i]_{t_e} sit in shared memory as sc[e][a] (A words per e).
template <int A>
__global__ void __launch_bounds__(TPB) modup_kernel(Tab tab, int logn, const u64 *__restrict__ dc, long dcs,
                                                    u64 *__restrict__ ext, long exts, int nl, int np, int nq_total,
                                                    int alpha, int beta, const u64 *__restrict__ hatpk) {
    static_assert(A % 2 == 0, "A even (16-byte constant pairs)");
    __shared__ __align__(16) u64 sc[MAXL * A];
    const int ct = blockIdx.y / beta, j = blockIdx.y % beta;
    const long N = 1L << logn;
    const int i0 = j * alpha, i1 = min(i0 + alpha, nl), na = i1 - i0;
    const int ne = nl + np;
    for (int t = threadIdx.x; t < ne * A; t += TPB) {
        const int e = t / A, a = t % A;
        sc[t] = a < na ? hatpk[((long)j * MAXA + a) * ne + e] : 0;
    }
    const long k = 2L * ((long)blockIdx.x * TPB + threadIdx.x);
    uint32_t yl[A][2], yh[A][2];
#pragma unroll
    for (int a = 0; a < A; a++) {
        if (a < na) {
            const int i = i0 + a;
            const ulonglong2 x = ldv2(dc + ct * dcs + i * N + k);
            // the factor (Q'_j/q_i)^{-1} is folded into the INTT: the input already is y
            const u64 y0 = x.x, y1 = x.y;
            yl[a][0] = (uint32_t)y0 & M30, yh[a][0] = (uint32_t)(y0 >> 30);
            yl[a][1] = (uint32_t)y1 & M30, yh[a][1] = (uint32_t)(y1 >> 30);
        } else {
            yl[a][0] = yh[a][0] = yl[a][1] = yh[a][1] = 0;
        }
    }
    __syncthreads();
    u64 *out = ext + ct * exts + (long)j * ne * N + k;
    for (int e = 0; e < ne; e++) {
        if (e >= i0 && e < i1) continue;
        const int pr = e < nl ? e : nq_total + (e - nl);
        Acc4 s0, s1;
        acc4_zero(s0);
        acc4_zero(s1);
        const ulonglong2 *cp = reinterpret_cast<const ulonglong2 *>(sc + e * A);
#pragma unroll
        for (int a2 = 0; a2 < A / 2; a2++) {
            if (2 * a2 < na) {
                const ulonglong2 c = cp[a2];
                acc4_mac(s0, yl[2 * a2][0], yh[2 * a2][0], c.x);
                acc4_mac(s1, yl[2 * a2][1], yh[2 * a2][1], c.x);
                acc4_mac(s0, yl[2 * a2 + 1][0], yh[2 * a2 + 1][0], c.y);
                acc4_mac(s1, yl[2 * a2 + 1][1], yh[2 * a2 + 1][1], c.y);
            }
        }
        const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
        stv2(out + e * N, acc4_reduce(s0, q, r0, r1), acc4_reduce(s1, q, r0, r1));
    }
}

// Key inner product (R10).  grid: x = coefficient chunks (two coefficients per thread, 16-byte vectors),
// y = extended limb e.  Loops over the n_ct ciphertexts so each key word is read from HBM once per
// launch (held in registers across the batch); the next ciphertext's inputs are loaded before the
// current one is reduced (two register sets), so twice the bytes are in flight.  MAXB = beta exactly
// (beta <= 4); larger dnum uses the scalar ks_inner_kernel below.
template <int MAXB>
struct KsIn {
    ulonglong2 x[MAXB];
};
// Hoisted rotation (R29): the key inner product reads sigma_g(x) instead of x.  In the NTT domain
// sigma_g is the permutation NTT(sigma_g a)[i] = NTT(a)[pi(i)], 2 brv(pi(i)) + 1 = g (2 brv(i) + 1) mod 2N;
// for even k, pi(k + 1) = pi(k) ^ 1, so the output pair (k, k+1) reads one aligned source pair (swapped
// when pi(k) is odd), and aligned blocks of 2^m map onto aligned blocks (coalesced gathers).
__device__ __forceinline__ long gal_src(long k, int logn, u64 g, bool &swap) {
    const unsigned e = 2u * (__brev((unsigned)k) >> (32 - logn)) + 1u;
    const unsigned e2 = (unsigned)(((u64)e * g) & ((2ull << logn) - 1));
    const unsigned j = __brev((e2 - 1u) >> 1) >> (32 - logn);
    swap = j & 1u;
    return (long)(j & ~1u);
}

// digit j's value at (e, pair kx): the input itself for the digit containing e, else its ModUp
template <int MAXB>
__device__ __forceinline__ void ks_load(KsIn<MAXB> &in, int c, const u64 *__restrict__ d, long ds,
                                        const u64 *__restrict__ ext, long exts, int e, int jd, int ne, int beta,
                                        long N, long kx, bool swap) {
#pragma unroll
    for (int j = 0; j < MAXB; j++)
        if (j < beta) {
            in.x[j] = ldv2((j == jd) ? d + c * ds + e * N + kx : ext + c * exts + ((long)j * ne + e) * N + kx);
            if (swap) in.x[j] = make_ulonglong2(in.x[j].y, in.x[j].x);
        }
}


__device__ __forceinline__ void tensor1_fp(u64 a0, u64 a1, u64 b0, u64 b1, bool lin, u64 x0, u64 x1, u64 c,
                                           bool lin2, u64 y0, u64 y1, u64 c2, double qd, double qinv, u64 &d0,
                                           u64 &d1, u64 &d2, bool p2 = false, u64 u0 = 0, u64 u1 = 0, u64 w0 = 0,
                                           u64 w1 = 0) {
    const double A0 = fpt::d(a0), A1 = fpt::d(a1), B0 = fpt::d(b0), B1 = fpt::d(b1);
    const double B0q = __dmul_rn(B0, qinv), B1q = __dmul_rn(B1, qinv);
    double e0 = fpt::mm(A0, B0, B0q, qd);
    double e1 = __dadd_rn(fpt::mm(A0, B1, B1q, qd), fpt::mm(A1, B0, B0q, qd));
    double e2 = fpt::mm(A1, B1, B1q, qd);
    if (p2) {  // second product (R13b): |e| stays below 4 * 0.75 q + linear terms < 2^51
        const double U0 = fpt::d(u0), U1 = fpt::d(u1), W0 = fpt::d(w0), W1 = fpt::d(w1);
        const double W0q = __dmul_rn(W0, qinv), W1q = __dmul_rn(W1, qinv);
        e0 = __dadd_rn(e0, fpt::mm(U0, W0, W0q, qd));
        e1 = __dadd_rn(e1, __dadd_rn(fpt::mm(U0, W1, W1q, qd), fpt::mm(U1, W0, W0q, qd)));
        e2 = __dadd_rn(e2, fpt::mm(U1, W1, W1q, qd));
    }
    if (lin) {
        const double C = fpt::d(c), Cq = __dmul_rn(C, qinv);
        e0 = __dadd_rn(e0, fpt::mm(fpt::d(x0), C, Cq, qd));
        e1 = __dadd_rn(e1, fpt::mm(fpt::d(x1), C, Cq, qd));
    }
    if (lin2) {
        const double C = fpt::d(c2), Cq = __dmul_rn(C, qinv);
        e0 = __dadd_rn(e0, fpt::mm(fpt::d(y0), C, Cq, qd));
        e1 = __dadd_rn(e1, fpt::mm(fpt::d(y1), C, Cq, qd));
    }
    d0 = fpt::canon(e0, qd, qinv);
    d1 = fpt::canon(e1, qd, qinv);
    d2 = fpt::canon(e2, qd, qinv);
}

// Plain key inner product (rotations): two coefficients per thread (16-byte vectors), the key words in
// registers across the ciphertext batch, the next ciphertext's inputs double-buffered.
template <int MAXB>
__global__ void __launch_bounds__(TPB, 3) ks_inner_vec_kernel(Tab tab, int logn, const u64 *__restrict__ d, long ds,
                                                            const u64 *__restrict__ ext, long exts,
                                                            const u64 *__restrict__ key, int nq_total, int np,
                                                            u64 *__restrict__ acc, long accs, int n_ct, int nl,
                                                            int alpha, int beta, u64 galois) {
    const int e = blockIdx.y;
    const long N = 1L << logn;
    const long k = 2L * ((long)blockIdx.x * TPB + threadIdx.x);
    bool swap = false;
    const long kx = galois > 1 ? gal_src(k, logn, galois, swap) : k;  // hoisted rotation gather
    const int ne = nl + np, nk = nq_total + np;
    const int pr = e < nl ? e : nq_total + (e - nl);
    const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
    ulonglong2 kb[MAXB], ka[MAXB];
#pragma unroll
    for (int j = 0; j < MAXB; j++)
        if (j < beta) {
            kb[j] = ldv2(key + (((long)j * 2 + 0) * nk + pr) * N + k);
            ka[j] = ldv2(key + (((long)j * 2 + 1) * nk + pr) * N + k);
        }
    const int jd = e < nl ? e / alpha : -1;  // digit containing e (Q limbs only)
    pdl_wait();
    KsIn<MAXB> cur, nxt;
    ks_load<MAXB>(cur, 0, d, ds, ext, exts, e, jd, ne, beta, N, kx, swap);
    // exact-FP64 products for q < 2^52 / 3.5 (the FpA and FpB rows): with canonical inputs |mm| <= 0.79 q,
    // beta <= 4 terms stay below 3.2 q < 2^52 and k = rint(s / q) <= 4 keeps k q exact
    const bool fp = q < FP_KS_LIMIT;
    const double qd = tab.qd[pr], qinv = tab.qinv[pr];
    for (int c = 0; c < n_ct; c++) {
        if (c + 1 < n_ct) ks_load<MAXB>(nxt, c + 1, d, ds, ext, exts, e, jd, ne, beta, N, kx, swap);
        if (fp) {
            // exact-FP64 products (as ks_inner_ten1_kernel): |sum of beta terms| <= 3 q -> canonical
            double s0 = 0, t0 = 0, s1 = 0, t1 = 0;
#pragma unroll
            for (int j = 0; j < MAXB; j++)
                if (j < beta) {
                    const double X = fpt::d(cur.x[j].x), Y = fpt::d(cur.x[j].y);
                    const double B0 = fpt::d(kb[j].x), B1 = fpt::d(kb[j].y), A0 = fpt::d(ka[j].x), A1 = fpt::d(ka[j].y);
                    s0 = __dadd_rn(s0, fpt::mm(X, B0, __dmul_rn(B0, qinv), qd));
                    t0 = __dadd_rn(t0, fpt::mm(Y, B1, __dmul_rn(B1, qinv), qd));
                    s1 = __dadd_rn(s1, fpt::mm(X, A0, __dmul_rn(A0, qinv), qd));
                    t1 = __dadd_rn(t1, fpt::mm(Y, A1, __dmul_rn(A1, qinv), qd));
                }
            stv2(acc + c * accs + (long)e * N + k, fp_canon4(s0, q, qd, qinv), fp_canon4(t0, q, qd, qinv));
            stv2(acc + c * accs + (long)(ne + e) * N + k, fp_canon4(s1, q, qd, qinv), fp_canon4(t1, q, qd, qinv));
            cur = nxt;
            continue;
        }
        U128 s0{0, 0}, s1{0, 0}, t0{0, 0}, t1{0, 0};  // (poly 0, poly 1) x (coefficient k, k + 1)
#pragma unroll
        for (int j = 0; j < MAXB; j++)
            if (j < beta) {
                mac_wide(s0, cur.x[j].x, kb[j].x);
                mac_wide(t0, cur.x[j].y, kb[j].y);
                mac_wide(s1, cur.x[j].x, ka[j].x);
                mac_wide(t1, cur.x[j].y, ka[j].y);
            }
        stv2(acc + c * accs + (long)e * N + k, barrett128(s0, q, r0, r1), barrett128(t0, q, r0, r1));
        stv2(acc + c * accs + (long)(ne + e) * N + k, barrett128(s1, q, r0, r1), barrett128(t1, q, r0, r1));
        cur = nxt;
    }
}

// Relinearise-and-rescale key inner product, one coefficient per thread: about half the registers of the
// two-coefficient kernel (which holds 16-byte vectors of every tensor input), so three CTAs fit per SM
// without spills.  Same integers (tensor1_fp / tensor1, 128-bit MACs, one Barrett per output).
#ifndef KS_TEN1_MINB
#define KS_TEN1_MINB 3  // (two ciphertexts per iteration at 2 CTAs/SM measured 1.3 % slower)
#endif
template <int MAXB>
__global__ void __launch_bounds__(TPB, KS_TEN1_MINB) ks_inner_ten1_kernel(Tab tab, int logn, const u64 *__restrict__ ext,
                                                                       long exts, const u64 *__restrict__ key,
                                                                       int nq_total, int np, u64 *__restrict__ acc,
                                                                       long accs, int n_ct, int nl, int alpha,
                                                                       int beta, TensorSrc ten,
                                                                       const u64 *__restrict__ pmod) {
    const int e = blockIdx.y;
    const long N = 1L << logn;
    const long k = (long)blockIdx.x * TPB + threadIdx.x;
    const int ne = nl + np, nk = nq_total + np;
    const int pr = e < nl ? e : nq_total + (e - nl);
    const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
    u64 kb[MAXB], ka[MAXB];
#pragma unroll
    for (int j = 0; j < MAXB; j++)
        if (j < beta) {
            kb[j] = __ldg(key + (((long)j * 2 + 0) * nk + pr) * N + k);
            ka[j] = __ldg(key + (((long)j * 2 + 1) * nk + pr) * N + k);
        }
    const int jd = e < nl ? e / alpha : -1;
    const bool qrow = e < nl;
    const u64 pm = qrow ? pmod[e] : 0;
    pdl_wait();  // the key words above are not produced by the previous kernel
    const bool lin = ten.x.p != nullptr, lin2 = ten.x2.p != nullptr, p2 = ten.a2.p != nullptr;
    const u64 cc = lin && qrow ? ten.C.c[e] : 0, ccsh = lin && qrow ? ten.C.csh[e] : 0;
    const u64 c2 = lin2 && qrow ? ten.C2.c[e] : 0, c2sh = lin2 && qrow ? ten.C2.csh[e] : 0;
    const double qd = tab.qd[pr], qinv = tab.qinv[pr];
    const long o = e * N + k;
    struct In {
        u64 x[MAXB], a0, a1, b0, b1, x0, x1, y0, y1, u0, u1, w0, w1;
    };
    auto load = [&](int c, In &in) {
#pragma unroll
        for (int j = 0; j < MAXB; j++)
            if (j < beta && j != jd) in.x[j] = ext[c * exts + ((long)j * ne + e) * N + k];
        if (qrow) {
            in.a0 = ten.a.p[c * ten.a.cs + o];
            in.a1 = ten.a.p[c * ten.a.cs + ten.a.ps + o];
            in.b0 = ten.b.p[c * ten.b.cs + o];
            in.b1 = ten.b.p[c * ten.b.cs + ten.b.ps + o];
            in.x0 = lin ? ten.x.p[c * ten.x.cs + o] : 0;
            in.x1 = lin ? ten.x.p[c * ten.x.cs + ten.x.ps + o] : 0;
            in.y0 = lin2 ? ten.x2.p[c * ten.x2.cs + o] : 0;
            in.y1 = lin2 ? ten.x2.p[c * ten.x2.cs + ten.x2.ps + o] : 0;
            in.u0 = p2 ? ten.a2.p[c * ten.a2.cs + o] : 0;
            in.u1 = p2 ? ten.a2.p[c * ten.a2.cs + ten.a2.ps + o] : 0;
            in.w0 = p2 ? ten.b2.p[c * ten.b2.cs + o] : 0;
            in.w1 = p2 ? ten.b2.p[c * ten.b2.cs + ten.b2.ps + o] : 0;
        }
    };
    auto compute = [&](int c, In &in) {
        if (q < (1ULL << 46)) {
            // exact-FP64 products on the FP64 pipe (the integer path's 128-bit MACs and Barrett reductions are
            // its dominant instructions): sum_j mm(x_j, key_j) [+ mm(d_b, [P])] -> |s| <= 3 q -> canonical
            double e0 = 0, e1 = 0, e2 = 0;
            if (qrow)
                tensor1_fp_raw(in.a0, in.a1, in.b0, in.b1, lin, in.x0, in.x1, cc, lin2, in.y0, in.y1, c2, qd, qinv, e0,
                               e1, e2, p2, in.u0, in.u1, in.w0, in.w1);
            double s0 = 0, s1 = 0;
#pragma unroll
            for (int j = 0; j < MAXB; j++)
                if (j < beta) {
                    const double X = j == jd ? e2 : fpt::d(in.x[j]);
                    const double KB = fpt::d(kb[j]), KA = fpt::d(ka[j]);
                    s0 = __dadd_rn(s0, fpt::mm(X, KB, __dmul_rn(KB, qinv), qd));
                    s1 = __dadd_rn(s1, fpt::mm(X, KA, __dmul_rn(KA, qinv), qd));
                }
            if (qrow) {
                const double PM = fpt::d(pm), PMq = __dmul_rn(PM, qinv);
                s0 = __dadd_rn(s0, fpt::mm(e0, PM, PMq, qd));
                s1 = __dadd_rn(s1, fpt::mm(e1, PM, PMq, qd));
            }
            acc[c * accs + (long)e * N + k] = fp_canon4(s0, q, qd, qinv);
            acc[c * accs + (long)(ne + e) * N + k] = fp_canon4(s1, q, qd, qinv);
            return;
        }
        u64 d0 = 0, d1 = 0;
        if (qrow) {
            u64 d2;
            if (q < (1ULL << 46))
                tensor1_fp(in.a0, in.a1, in.b0, in.b1, lin, in.x0, in.x1, cc, lin2, in.y0, in.y1, c2, qd, qinv, d0, d1,
                           d2, p2, in.u0, in.u1, in.w0, in.w1);
            else
                tensor1(in.a0, in.a1, in.b0, in.b1, lin, in.x0, in.x1, cc, ccsh, lin2, in.y0, in.y1, c2, c2sh, q, r0, r1,
                        d0, d1, d2, p2, in.u0, in.u1, in.w0, in.w1);
#pragma unroll
            for (int j = 0; j < MAXB; j++)
                if (j == jd) in.x[j] = d2;
        }
        U128 s0{0, 0}, s1{0, 0};
#pragma unroll
        for (int j = 0; j < MAXB; j++)
            if (j < beta) {
                mac_wide(s0, in.x[j], kb[j]);
                mac_wide(s1, in.x[j], ka[j]);
            }
        if (qrow) {
            mac_wide(s0, d0, pm);
            mac_wide(s1, d1, pm);
        }
        acc[c * accs + (long)e * N + k] = barrett128(s0, q, r0, r1);
        acc[c * accs + (long)(ne + e) * N + k] = barrett128(s1, q, r0, r1);
    };
    for (int c = 0; c < n_ct; c++) {
        In A;
        load(c, A);
        compute(c, A);
    }
}

// The same relinearise-and-rescale inner product with the ciphertext inputs staged by bulk asynchronous
// copies (cp.async.bulk, one 2 KB row slice per input array and ciphertext) into a KB_STAGES-deep shared
// memory ring: thread 0 issues the copies of ciphertext c + KB_STAGES while the block computes c, so the
// loads of the next ciphertexts are in flight during the arithmetic (the per-thread version waits on each
// ciphertext's loads).  Identical integers: the arithmetic is ks_inner_ten1_kernel's, reading its operands
// from shared memory.
#ifndef KB_STAGES
#define KB_STAGES 3
#endif
constexpr int KB_MAXARR = 14;  // ext digits (<= 4) + a0 a1 b0 b1 + x0 x1 + y0 y1 + u0 u1 w0 w1
__device__ __forceinline__ uint32_t ks_su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MAXB>
__global__ void __launch_bounds__(TPB, 2) ks_inner_ten1_bulk_kernel(Tab tab, int logn, const u64 *__restrict__ ext,
                                                                  long exts, const u64 *__restrict__ key,
                                                                  int nq_total, int np, u64 *__restrict__ acc,
                                                                  long accs, int n_ct, int nl, int alpha, int beta,
                                                                  TensorSrc ten, const u64 *__restrict__ pmod,
                                                                  int narr_max) {
    extern __shared__ __align__(16) u64 kbuf[];  // [KB_STAGES][narr_max][TPB]
    __shared__ __align__(8) uint64_t kfull[KB_STAGES];
    const int e = blockIdx.y, tid = threadIdx.x;
    const long N = 1L << logn;
    const long k0 = (long)blockIdx.x * TPB, k = k0 + tid;
    const int ne = nl + np, nk = nq_total + np;
    const int pr = e < nl ? e : nq_total + (e - nl);
    const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
    u64 kb[MAXB], ka[MAXB];
#pragma unroll
    for (int j = 0; j < MAXB; j++)
        if (j < beta) {
            kb[j] = __ldg(key + (((long)j * 2 + 0) * nk + pr) * N + k);
            ka[j] = __ldg(key + (((long)j * 2 + 1) * nk + pr) * N + k);
        }
    const int jd = e < nl ? e / alpha : -1;
    const bool qrow = e < nl;
    const u64 pm = qrow ? pmod[e] : 0;
    const bool lin = ten.x.p != nullptr, lin2 = ten.x2.p != nullptr, p2 = ten.a2.p != nullptr;
    const u64 cc = lin && qrow ? ten.C.c[e] : 0, ccsh = lin && qrow ? ten.C.csh[e] : 0;
    const u64 c2 = lin2 && qrow ? ten.C2.c[e] : 0, c2sh = lin2 && qrow ? ten.C2.csh[e] : 0;
    const double qd = tab.qd[pr], qinv = tab.qinv[pr];
    const long o0 = e * N + k0;
    // this row's input slices: slot -> (base, per-ciphertext stride); ext digits first (slot j = digit j)
    const int next_ = qrow ? beta - 1 : beta;
    const int narr = next_ + (qrow ? 4 + (lin ? 2 : 0) + (lin2 ? 2 : 0) + (p2 ? 4 : 0) : 0);
    auto slot_src = [&](int i, int c) -> const u64 * {
        if (i < next_) {
            const int j = (qrow && i >= jd) ? i + 1 : i;
            return ext + c * exts + ((long)j * ne + e) * N + k0;
        }
        int t = i - next_;
        if (t < 4) {
            const CRows &r = t < 2 ? ten.a : ten.b;
            return r.p + c * r.cs + (t & 1) * r.ps + o0;
        }
        t -= 4;
        if (lin) {
            if (t < 2) return ten.x.p + c * ten.x.cs + t * ten.x.ps + o0;
            t -= 2;
        }
        if (lin2) {
            if (t < 2) return ten.x2.p + c * ten.x2.cs + t * ten.x2.ps + o0;
            t -= 2;
        }
        const CRows &r = t < 2 ? ten.a2 : ten.b2;
        return r.p + c * r.cs + (t & 1) * r.ps + o0;
    };
    auto issue = [&](int c) {
        const int st = c % KB_STAGES;
        const uint32_t bar = ks_su32(&kfull[st]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(narr * TPB * 8)
                     : "memory");
        for (int i = 0; i < narr; i++)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             ks_su32(kbuf + ((long)st * narr_max + i) * TPB)),
                         "l"(slot_src(i, c)), "r"(TPB * 8), "r"(bar)
                         : "memory");
    };
    if (tid == 0) {
        for (int st = 0; st < KB_STAGES; st++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ks_su32(&kfull[st])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();  // the key words above are not produced by the previous kernel; the inputs are
    if (tid == 0)
        for (int c = 0; c < KB_STAGES && c < n_ct; c++) issue(c);
    for (int c = 0; c < n_ct; c++) {
        const int st = c % KB_STAGES;
        {
            const uint32_t bar = ks_su32(&kfull[st]), par = (c / KB_STAGES) & 1;
            asm volatile(
                "{\n\t.reg .pred p;\n\tKBW%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra KBW%=;\n\t}" ::"r"(bar),
                "r"(par)
                : "memory");
        }
        const u64 *sl = kbuf + (long)st * narr_max * TPB + tid;
        u64 x[MAXB];
#pragma unroll
        for (int j = 0; j < MAXB; j++)
            if (j < beta && j != jd) x[j] = sl[(qrow && j > jd ? j - 1 : j) * TPB];
        u64 d0 = 0, d1 = 0;
        if (qrow) {
            const u64 *tp = sl + next_ * TPB;
            const u64 a0 = tp[0], a1 = tp[TPB], b0 = tp[2 * TPB], b1 = tp[3 * TPB];
            int t = 4;
            u64 x0 = 0, x1 = 0, y0 = 0, y1 = 0, u0 = 0, u1 = 0, w0 = 0, w1 = 0;
            if (lin) {
                x0 = tp[t * TPB];
                x1 = tp[(t + 1) * TPB];
                t += 2;
            }
            if (lin2) {
                y0 = tp[t * TPB];
                y1 = tp[(t + 1) * TPB];
                t += 2;
            }
            if (p2) {
                u0 = tp[t * TPB];
                u1 = tp[(t + 1) * TPB];
                w0 = tp[(t + 2) * TPB];
                w1 = tp[(t + 3) * TPB];
            }
            u64 d2;
            if (q < (1ULL << 46))
                tensor1_fp(a0, a1, b0, b1, lin, x0, x1, cc, lin2, y0, y1, c2, qd, qinv, d0, d1, d2, p2, u0, u1, w0, w1);
            else
                tensor1(a0, a1, b0, b1, lin, x0, x1, cc, ccsh, lin2, y0, y1, c2, c2sh, q, r0, r1, d0, d1, d2, p2, u0,
                        u1, w0, w1);
#pragma unroll
            for (int j = 0; j < MAXB; j++)
                if (j == jd) x[j] = d2;
        }
        U128 s0{0, 0}, s1{0, 0};
#pragma unroll
        for (int j = 0; j < MAXB; j++)
            if (j < beta) {
                mac_wide(s0, x[j], kb[j]);
                mac_wide(s1, x[j], ka[j]);
            }
        if (qrow) {
            mac_wide(s0, d0, pm);
            mac_wide(s1, d1, pm);
        }
        acc[c * accs + (long)e * N + k] = barrett128(s0, q, r0, r1);
        acc[c * accs + (long)(ne + e) * N + k] = barrett128(s1, q, r0, r1);
        __syncthreads();  // every thread is done with stage st
        if (tid == 0 && c + KB_STAGES < n_ct) issue(c + KB_STAGES);
    }
}

// scalar variant for dnum > 4 (small primes only: the toy ring): one coefficient per thread
template <int MAXB>
__global__ void ks_inner_kernel(Tab tab, int logn, const u64 *__restrict__ d, long ds, const u64 *__restrict__ ext,
                                long exts, const u64 *__restrict__ key, int nq_total, int np,
                                u64 *__restrict__ acc, long accs, int n_ct, int nl, int alpha, int beta,
                                TensorSrc ten, const u64 *__restrict__ pmod, u64 galois) {
    const int e = blockIdx.y;
    const long N = 1L << logn;
    const long k = (long)blockIdx.x * TPB + threadIdx.x;
    long kx = k;
    if (galois > 1) {
        bool sw;
        const long base = gal_src(k & ~1L, logn, galois, sw);  // sets sw: sequenced before its use
        kx = base + ((k & 1) ^ (sw ? 1 : 0));
    }
    const bool qrow = ten.a.p && e < nl;
    const int ne = nl + np, nk = nq_total + np;
    const int pr = e < nl ? e : nq_total + (e - nl);
    const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
    const int jd = e < nl ? e / alpha : -1;
    for (int c = 0; c < n_ct; c++) {
        U128 s0{0, 0}, s1{0, 0};
        u64 d0 = 0, d1 = 0, d2 = 0;
        if (qrow) {
            const long o = e * N + k;
            const bool lin = ten.x.p != nullptr, lin2 = ten.x2.p != nullptr;
            tensor1(ten.a.p[c * ten.a.cs + o], ten.a.p[c * ten.a.cs + ten.a.ps + o], ten.b.p[c * ten.b.cs + o],
                    ten.b.p[c * ten.b.cs + ten.b.ps + o], lin, lin ? ten.x.p[c * ten.x.cs + o] : 0,
                    lin ? ten.x.p[c * ten.x.cs + ten.x.ps + o] : 0, lin ? ten.C.c[e] : 0, lin ? ten.C.csh[e] : 0,
                    lin2, lin2 ? ten.x2.p[c * ten.x2.cs + o] : 0, lin2 ? ten.x2.p[c * ten.x2.cs + ten.x2.ps + o] : 0,
                    lin2 ? ten.C2.c[e] : 0, lin2 ? ten.C2.csh[e] : 0, q, r0, r1, d0, d1, d2, ten.a2.p != nullptr,
                    ten.a2.p ? ten.a2.p[c * ten.a2.cs + o] : 0, ten.a2.p ? ten.a2.p[c * ten.a2.cs + ten.a2.ps + o] : 0,
                    ten.a2.p ? ten.b2.p[c * ten.b2.cs + o] : 0, ten.a2.p ? ten.b2.p[c * ten.b2.cs + ten.b2.ps + o] : 0);
        }
        for (int j = 0; j < beta; j++) {
            const u64 x = (j == jd) ? (qrow ? d2 : d[c * ds + e * N + kx]) : ext[c * exts + ((long)j * ne + e) * N + kx];
            mac_wide(s0, x, __ldg(key + (((long)j * 2 + 0) * nk + pr) * N + k));
            mac_wide(s1, x, __ldg(key + (((long)j * 2 + 1) * nk + pr) * N + k));
        }
        if (qrow) {
            const u64 pm = pmod[e];
            mac_wide(s0, d0, pm);
            mac_wide(s1, d1, pm);
        }
        acc[c * accs + (long)e * N + k] = barrett128(s0, q, r0, r1);
        acc[c * accs + (long)(ne + e) * N + k] = barrett128(s1, q, r0, r1);
    }
}

// ModDown conversion (R11).  grid: x = coefficient chunks (two per thread), y = ct * 2 + b.
// Sources: ns rows starting at row0 of each acc polynomial (already holding [r_s (B/s)^{-1}]_s: the
// factor is folded into the INTT); targets: q_0..q_{nt-1}.  Packed constants [B/s]_{q_i} at
// hatpk[s * hstride + i], staged in shared memory as sc[i][s] (NS words per i).
template <int NS>
__global__ void __launch_bounds__(TPB) moddown_conv_kernel(Tab tab, int logn, const u64 *__restrict__ acc, long accs,
                                                           int ne, int row0, int ns, u64 *__restrict__ T, long Ts,
                                                           int nt, const u64 *__restrict__ hatpk, int hstride) {
    static_assert(NS % 2 == 0, "NS even");
    __shared__ __align__(16) u64 sc[MAXL * NS];
    const int ct = blockIdx.y / 2, b = blockIdx.y % 2;
    const long N = 1L << logn;
    for (int t = threadIdx.x; t < nt * NS; t += TPB) {
        const int i = t / NS, p = t % NS;
        sc[t] = p < ns ? hatpk[(long)p * hstride + i] : 0;
    }
    const long k = 2L * ((long)blockIdx.x * TPB + threadIdx.x);
    const u64 *src = acc + ct * accs + ((long)b * ne + row0) * N + k;
    uint32_t yl[NS][2], yh[NS][2];
#pragma unroll
    for (int p = 0; p < NS; p++) {
        if (p < ns) {
            const ulonglong2 x = ldv2(src + p * N);
            yl[p][0] = (uint32_t)x.x & M30, yh[p][0] = (uint32_t)(x.x >> 30);
            yl[p][1] = (uint32_t)x.y & M30, yh[p][1] = (uint32_t)(x.y >> 30);
        } else {
            yl[p][0] = yh[p][0] = yl[p][1] = yh[p][1] = 0;
        }
    }
    __syncthreads();
    u64 *dst = T + ct * Ts + (long)b * nt * N + k;
    for (int i = 0; i < nt; i++) {
        Acc4 s0, s1;
        acc4_zero(s0);
        acc4_zero(s1);
        const ulonglong2 *cp = reinterpret_cast<const ulonglong2 *>(sc + i * NS);
#pragma unroll
        for (int p2 = 0; p2 < NS / 2; p2++) {
            if (2 * p2 < ns) {
                const ulonglong2 c = cp[p2];
                acc4_mac(s0, yl[2 * p2][0], yh[2 * p2][0], c.x);
                acc4_mac(s1, yl[2 * p2][1], yh[2 * p2][1], c.x);
                acc4_mac(s0, yl[2 * p2 + 1][0], yh[2 * p2 + 1][0], c.y);
                acc4_mac(s1, yl[2 * p2 + 1][1], yh[2 * p2 + 1][1], c.y);
            }
        }
        stv2(dst + i * N, acc4_reduce(s0, tab.q[i], tab.br0[i], tab.br1[i]),
             acc4_reduce(s1, tab.q[i], tab.br0[i], tab.br1[i]));
    }
}
// Fused ModDown + rescale conversion (ev_mul_relin_rescale).  grid: x = coefficient chunks (two
// per thread), y = ct * 2 + b.  Rows l .. l + np of each acc polynomial hold, in coefficient form,
// xc = INTT(x_l) and y_p = [INTT(x_p) (P/p)^{-1}]_p, where x = acc + [P] d.  Per coefficient:
//   Y_l = (xc - sum_p y_p [P/p]_{q_l}) P^{-1} mod q_l        (the q_l limb of the ModDown output)
//   r   = [Y_l + floor(q_l/2)]_{q_l}                           (R12)
//   T_i = sum_p y_p [P/p]_{q_i} + r [P]_{q_i} - [P floor(q_l/2)]_{q_i}   for i < l
// so that (x_i - NTT(T_i)) (P q_l)^{-1} equals ModDown followed by the rescale, exactly.
template <int NS>
__global__ void __launch_bounds__(TPB) rr_conv_kernel(Tab tab, int logn, const u64 *__restrict__ acc, long accs,
                                                      int ne, int l, int np, u64 *__restrict__ T, long Ts,
                                                      const u64 *__restrict__ hatpk, const u64 *__restrict__ hl,
                                                      u64 pinv_l, u64 pinv_l_sh) {
    static_assert(NS % 2 == 0, "NS even");
    __shared__ __align__(16) u64 sc[MAXL * NS];
    __shared__ u64 shl[MAXA];
    const int ct = blockIdx.y / 2, b = blockIdx.y % 2;
    const long N = 1L << logn;
    const int ns = np + 2;
    for (int t = threadIdx.x; t < l * NS; t += TPB) {
        const int i = t / NS, p = t % NS;
        sc[t] = p < ns ? hatpk[(long)p * l + i] : 0;
    }
    for (int t = threadIdx.x; t < np; t += TPB) shl[t] = hl[t];
    const long k = 2L * ((long)blockIdx.x * TPB + threadIdx.x);
    const u64 *src = acc + ct * accs + ((long)b * ne + l) * N + k;
    uint32_t yl[NS][2], yh[NS][2];
#pragma unroll
    for (int p = 0; p < NS; p++) {
        if (p < np) {
            const ulonglong2 x = ldv2(src + (p + 1) * N);
            yl[p][0] = (uint32_t)x.x & M30, yh[p][0] = (uint32_t)(x.x >> 30);
            yl[p][1] = (uint32_t)x.y & M30, yh[p][1] = (uint32_t)(x.y >> 30);
        } else {
            yl[p][0] = yh[p][0] = yl[p][1] = yh[p][1] = 0;
        }
    }
    __syncthreads();
    {
        const ulonglong2 xc = ldv2(src);
        const u64 ql = tab.q[l], half = ql >> 1;
        Acc4 s0, s1;
        acc4_zero(s0);
        acc4_zero(s1);
#pragma unroll
        for (int p = 0; p < NS; p++)
            if (p < np) {
                acc4_mac(s0, yl[p][0], yh[p][0], shl[p]);
                acc4_mac(s1, yl[p][1], yh[p][1], shl[p]);
            }
        const u64 t0 = acc4_reduce(s0, ql, tab.br0[l], tab.br1[l]), t1 = acc4_reduce(s1, ql, tab.br0[l], tab.br1[l]);
        const u64 r0 = csub(mul_shoup(submod(xc.x, t0, ql), pinv_l, pinv_l_sh, ql) + half, ql);
        const u64 r1 = csub(mul_shoup(submod(xc.y, t1, ql), pinv_l, pinv_l_sh, ql) + half, ql);
        // sources np (r) and np + 1 (the constant 1)
#pragma unroll
        for (int p = 0; p < NS; p++)
            if (p == np) {
                yl[p][0] = (uint32_t)r0 & M30, yh[p][0] = (uint32_t)(r0 >> 30);
                yl[p][1] = (uint32_t)r1 & M30, yh[p][1] = (uint32_t)(r1 >> 30);
            } else if (p == np + 1) {
                yl[p][0] = yl[p][1] = 1;
                yh[p][0] = yh[p][1] = 0;
            }
    }
    u64 *dst = T + ct * Ts + (long)b * l * N + k;
    for (int i = 0; i < l; i++) {
        Acc4 s0, s1;
        acc4_zero(s0);
        acc4_zero(s1);
        const ulonglong2 *cp = reinterpret_cast<const ulonglong2 *>(sc + i * NS);
#pragma unroll
        for (int p2 = 0; p2 < NS / 2; p2++) {
            if (2 * p2 < ns) {
                const ulonglong2 c = cp[p2];
                acc4_mac(s0, yl[2 * p2][0], yh[2 * p2][0], c.x);
                acc4_mac(s1, yl[2 * p2][1], yh[2 * p2][1], c.x);
                acc4_mac(s0, yl[2 * p2 + 1][0], yh[2 * p2 + 1][0], c.y);
                acc4_mac(s1, yl[2 * p2 + 1][1], yh[2 * p2 + 1][1], c.y);
            }
        }
        stv2(dst + i * N, acc4_reduce(s0, tab.q[i], tab.br0[i], tab.br1[i]),
             acc4_reduce(s1, tab.q[i], tab.br0[i], tab.br1[i]));
    }
}
}  // namespace

static inline unsigned chunks(int logn) { return (unsigned)((1L << logn) / TPB); }
static inline unsigned chunks2(int logn) { return (unsigned)((1L << logn) / (2 * TPB)); }

void k_modup(const Tab &tab, int logn, const u64 *dc, long dcs, u64 *ext, long exts, int n_ct, int nl, int np,
             int nq_total, int alpha, const u64 *hat, cudaStream_t st) {
    const int beta = (nl + alpha - 1) / alpha;
    if (alpha > MAXA) throw SecpeError{-1, "alpha > 16 not supported"};
    const dim3 grid(chunks2(logn), n_ct * beta);
#define MODUP(A_)                                                                                          \
    modup_kernel<A_><<<grid, TPB, 0, st>>>(tab, logn, dc, dcs, ext, exts, nl, np, nq_total, alpha, beta, hat)
    if (alpha <= 2)
        MODUP(2);
    else if (alpha <= 4)
        MODUP(4);
    else if (alpha <= 8)
        MODUP(8);
    else if (alpha <= 10)
        MODUP(10);
    else
        MODUP(16);
#undef MODUP
    LAUNCH_CHECK();
}
void k_ks_inner(const Tab &tab, int logn, const u64 *d, long ds, const u64 *ext, long exts, const u64 *key,
                int nq_total, int np, u64 *acc, long accs, int n_ct, int nl, int alpha, cudaStream_t st,
                const TensorSrc *ten, const u64 *pmod, u64 galois) {
    const int beta = (nl + alpha - 1) / alpha;
    if (ten && galois > 1) throw SecpeError{-1, "ks_inner: the galois gather is for plain key switching only"};
    // 128-bit accumulation of beta + 1 products < 2^120 stays below the Barrett input bound 2^125
    // (checked at context creation against the actual prime sizes).
    const dim3 g2(chunks2(logn), nl + np), g1(chunks(logn), nl + np);
    static const TensorSrc none{};
    const TensorSrc &T = ten ? *ten : none;
    // bulk-staged relinearisation inner product (ks_inner_ten1_bulk_kernel): slices per ciphertext
    const int narr_max = ten ? std::max(beta, beta - 1 + 4 + (T.x.p ? 2 : 0) + (T.x2.p ? 2 : 0) + (T.a2.p ? 4 : 0)) : 0;
    const size_t kb_smem = (size_t)KB_STAGES * narr_max * TPB * 8;
    static int kb_mode = -1;
    if (kb_mode < 0) {
        const char *e = getenv("SECPE_KS_BULK");  // development switch: 0 = per-thread loads
        kb_mode = e ? atoi(e) : 0;  // measured slower than the per-thread kernel (profiles/r02_notes.md)
    }
#define KSV(B_)                                                                                                   \
    do {                                                                                                          \
        if (ten && kb_mode) {                                                                                     \
            static bool attr = false;                                                                             \
            if (!attr) {                                                                                          \
                CUDA_CHECK(cudaFuncSetAttribute(ks_inner_ten1_bulk_kernel<B_>,                                    \
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,                      \
                                                KB_STAGES * KB_MAXARR * TPB * 8));                                \
                attr = true;                                                                                      \
            }                                                                                                     \
            launch_pdl_k(ks_inner_ten1_bulk_kernel<B_>, g1, dim3(TPB), kb_smem, st, tab, logn, ext, exts, key,    \
                         nq_total, np, acc, accs, n_ct, nl, alpha, beta, T, pmod, narr_max);                      \
        } else if (ten)                                                                                           \
            launch_pdl_k(ks_inner_ten1_kernel<B_>, g1, dim3(TPB), 0, st, tab, logn, ext, exts, key, nq_total, np, \
                         acc, accs, n_ct, nl, alpha, beta, T, pmod);                                              \
        else                                                                                                      \
            launch_pdl_k(ks_inner_vec_kernel<B_>, g2, dim3(TPB), 0, st, tab, logn, d, ds, ext, exts, key, nq_total, \
                         np, acc, accs, n_ct, nl, alpha, beta, galois);                                           \
    } while (0)
    if (beta == 1)
        KSV(1);
    else if (beta == 2)
        KSV(2);
    else if (beta == 3)
        KSV(3);
    else if (beta == 4)
        KSV(4);
    else
        ks_inner_kernel<0><<<g1, TPB, 0, st>>>(tab, logn, d, ds, ext, exts, key, nq_total, np, acc, accs, n_ct, nl,
                                               alpha, beta, T, pmod, galois);
#undef KSV
    LAUNCH_CHECK();
}
void k_moddown_conv(const Tab &tab, int logn, const u64 *acc, long accs, int ne, int row0, int ns, u64 *T,
                    long Ts, int nt, int n_ct, const u64 *hatpk, int hstride, cudaStream_t st) {
    if (ns > MAXA) throw SecpeError{-1, "more than 16 conversion sources not supported"};
    const dim3 grid(chunks2(logn), n_ct * 2);
#define MDC(P_) \
    moddown_conv_kernel<P_><<<grid, TPB, 0, st>>>(tab, logn, acc, accs, ne, row0, ns, T, Ts, nt, hatpk, hstride)
    if (ns <= 2)
        MDC(2);
    else if (ns <= 4)
        MDC(4);
    else if (ns <= 8)
        MDC(8);
    else if (ns <= 10)
        MDC(10);
    else
        MDC(16);
#undef MDC
    LAUNCH_CHECK();
}

void k_rr_conv(const Tab &tab, int logn, const u64 *acc, long accs, int ne, int l, int np, u64 *T, long Ts, int n_ct,
               const u64 *hatpk, const u64 *hl, u64 pinv_l, u64 pinv_l_sh, cudaStream_t st) {
    if (np + 2 > MAXA) throw SecpeError{-1, "more than 14 special primes not supported"};
    const dim3 grid(chunks2(logn), n_ct * 2);
#define RRC(P_) \
    rr_conv_kernel<P_><<<grid, TPB, 0, st>>>(tab, logn, acc, accs, ne, l, np, T, Ts, hatpk, hl, pinv_l, pinv_l_sh)
    if (np + 2 <= 4)
        RRC(4);
    else if (np + 2 <= 10)
        RRC(10);
    else
        RRC(16);
#undef RRC
    LAUNCH_CHECK();
}
