// fpk.cuh -- exact-FP64 modular products for primes < 2^46 shared by the key inner products (ks.cu) and the
// fused ModUp-NTT + key inner product kernel (ntt.cu).
#pragma once
#include "common.cuh"

namespace {

// Exact-FP64 tensor for primes < 2^46 (the configs[4] chain): operands < 2^46 are exact doubles;
// w y mod q = fma(y, w, -k q) with k = rint(y w / q) (the ntt.cu FpA product), |r| <= 0.75 q, so the
// FP64 pipe takes the products and the integer pipes keep only the key MACs.
namespace fpt {
constexpr double MAGIC = 6755399441055744.0, TWO52 = 4503599627370496.0;
__device__ __forceinline__ double d(u64 x) {
    return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ULL)), TWO52);
}
__device__ __forceinline__ double mm(double y, double w, double wq, double qd) {
    const double k = __dsub_rn(__fma_rn(y, wq, MAGIC), MAGIC);
    const double ph = __dmul_rn(k, qd);
    const double pl = __fma_rn(k, qd, -ph);
    return __dsub_rn(__fma_rn(y, w, -ph), pl);
}
// canonical integer of an exact double |v| < 2^51
__device__ __forceinline__ u64 canon(double v, double qd, double qinv) {
    const double k = __dsub_rn(__dadd_rn(__dmul_rn(v, qinv), MAGIC), MAGIC);
    double t = __fma_rn(-k, qd, v);
    if (t < 0) t = __dadd_rn(t, qd);
    return (u64)__double_as_longlong(__dadd_rn(t, TWO52)) & ((1ULL << 52) - 1);
}
}  // namespace fpt

// the same tensor left as exact doubles (|e| <= 4.5 q < 2^49, not canonicalised): the FP64 key inner product
// below multiplies them directly
__device__ __forceinline__ void tensor1_fp_raw(u64 a0, u64 a1, u64 b0, u64 b1, bool lin, u64 x0, u64 x1, u64 c,
                                               bool lin2, u64 y0, u64 y1, u64 c2, double qd, double qinv, double &e0,
                                               double &e1, double &e2, bool p2, u64 u0, u64 u1, u64 w0, u64 w1) {
    const double A0 = fpt::d(a0), A1 = fpt::d(a1), B0 = fpt::d(b0), B1 = fpt::d(b1);
    const double B0q = __dmul_rn(B0, qinv), B1q = __dmul_rn(B1, qinv);
    e0 = fpt::mm(A0, B0, B0q, qd);
    e1 = __dadd_rn(fpt::mm(A0, B1, B1q, qd), fpt::mm(A1, B0, B0q, qd));
    e2 = fpt::mm(A1, B1, B1q, qd);
    if (p2) {
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
}
// Rows whose plain (rotation) key inner products run on the FP64 pipe: q < 2^52 / 3.5.  With canonical inputs
// the quotient estimate of fpt::mm is off by at most 1 + q / 2^52 <= 1.29, so |mm| <= 1.29 q and beta <= 4
// products sum to |s| <= 5.2 q < 2^52.5: every partial sum is an exact double, and the canonicalisation's
// fma(-k, q, s) is exact whatever k.  The relinearisation kernel sums up to six raw tensor products before its
// [P] product, which for ~50-bit q could pass 2^53: it keeps the FP64 path to q < 2^46.
constexpr u64 FP_KS_LIMIT = 1286742750677284ULL;
// canonical residue of an exact double |v| <= 6 q (four FP64 operations, the sign fix on the integer pipe)
__device__ __forceinline__ u64 fp_canon4(double v, u64 q, double qd, double qinv) {
    const double k = __dsub_rn(__fma_rn(v, qinv, fpt::MAGIC), fpt::MAGIC);
    const double r = __fma_rn(-k, qd, v);
    const long long ri = __double_as_longlong(__dadd_rn(r, fpt::MAGIC)) - __double_as_longlong(fpt::MAGIC);
    return (u64)(ri + ((ri >> 63) & (long long)q));
}


// one coefficient of the tensor: (d0, d1, d2) mod q, with the optional linear term C x
__device__ __forceinline__ void tensor1(u64 a0, u64 a1, u64 b0, u64 b1, bool lin, u64 x0, u64 x1, u64 c, u64 csh,
                                        bool lin2, u64 y0, u64 y1, u64 c2, u64 c2sh, u64 q, u64 r0, u64 r1, u64 &d0,
                                        u64 &d1, u64 &d2, bool p2 = false, u64 u0 = 0, u64 u1 = 0, u64 w0 = 0,
                                        u64 w1 = 0) {
    U128 t0 = mul_wide(a0, b0), t2 = mul_wide(a1, b1);
    U128 t = mul_wide(a0, b1);
    mac_wide(t, a1, b0);
    if (p2) {  // second product (R13b); four 120-bit products stay below the Barrett bound 2^125
        mac_wide(t0, u0, w0);
        mac_wide(t2, u1, w1);
        mac_wide(t, u0, w1);
        mac_wide(t, u1, w0);
    }
    d0 = barrett128(t0, q, r0, r1);
    d1 = barrett128(t, q, r0, r1);
    d2 = barrett128(t2, q, r0, r1);
    if (lin) {
        d0 = addmod(d0, mul_shoup(x0, c, csh, q), q);
        d1 = addmod(d1, mul_shoup(x1, c, csh, q), q);
    }
    if (lin2) {
        d0 = addmod(d0, mul_shoup(y0, c2, c2sh, q), q);
        d1 = addmod(d1, mul_shoup(y1, c2, c2sh, q), q);
    }
}

}  // namespace
