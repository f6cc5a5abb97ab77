// ntt_core.cuh -- the butterfly arithmetic shared by the NTT kernels (ntt.cu: two-pass and cluster
// kernels; ntt_fused.cu: the persistent TMA-pipelined kernel).  See ntt.cu for the decomposition and the
// two arithmetic policies (FpA: exact FP64 for primes < 2^46; IntA: Harvey/Shoup for primes < 2^60).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace {

#ifndef NTT_MINB
#define NTT_MINB 3  // resident CTAs per SM the register allocation targets (measured: 3 ~ 4 > 2)
#endif
#ifndef NTT_MINB_FP
#define NTT_MINB_FP 4  // FP rows: 64 registers, no spills
#endif
#ifndef NTT_STREAMING
#define NTT_STREAMING 1  // data loads/stores with the streaming (evict-first) cache hint: L1 kept for twiddles
#endif
#if NTT_STREAMING
#define NTT_LD(p) __ldcs(p)
#define NTT_LD2(p) __ldcs(p)
#define NTT_ST(p, v) __stcs(p, v)
#define NTT_ST2(p, v) __stcs(p, v)
#else
#define NTT_LD(p) (*(p))
#define NTT_LD2(p) (*(p))
#define NTT_ST(p, v) (*(p) = (v))
#define NTT_ST2(p, v) (*(p) = (v))
#endif
#ifndef NTT_PDL
#define NTT_PDL 1  // programmatic dependent launch of the NTT passes
#endif
#ifndef NTT_WAVE_PREFETCH
#define NTT_WAVE_PREFETCH 1  // first forward pass: the next wave's input tiles prefetched into L2
                             // (isolated forward NTT 0.451 -> 0.420 us/limb; the same for the first
                             // inverse pass measured +2 %, not used)
#endif
#ifndef NTT_EPI_PREFETCH
#define NTT_EPI_PREFETCH 1  // L2 prefetch of the rescale / ModDown epilogue operands at kernel start
#endif
#ifndef NTT_APPROX_HI
#define NTT_APPROX_HI 1  // approximate Shoup quotient in the butterflies (measured: inverse -4%)
#endif
constexpr int RB = 4;        // bits held per thread
constexpr int NV = 1 << RB;  // values per thread
constexpr int SC = 16;       // columns per CTA in strided passes (16 x 8 B = one 128-B line)
constexpr int CT = 256;      // threads per CTA in contiguous passes

#if NTT_APPROX_HI
// floor(y s / 2^64) - delta, delta in {0, 1}: the yl*sl partial product is dropped
__device__ __forceinline__ u64 mulhi_approx(u64 y, u64 s) {
    const uint32_t yl = (uint32_t)y, yh = (uint32_t)(y >> 32), sl = (uint32_t)s, sh = (uint32_t)(s >> 32);
    u64 r;
    asm("{\n\t.reg .u32 t0, t1, m0, m1, c;\n\t"
        "mul.lo.u32 t0, %1, %4;\n\t"
        "mul.hi.u32 t1, %1, %4;\n\t"
        "mad.lo.cc.u32 m0, %2, %3, t0;\n\t"
        "madc.hi.cc.u32 m1, %2, %3, t1;\n\t"
        "addc.u32 c, 0, 0;\n\t"
        "mov.b64 %0, {m1, c};\n\t"
        "mad.wide.u32 %0, %1, %3, %0;\n\t"
        "}"
        : "=l"(r)
        : "r"(yh), "r"(yl), "r"(sh), "r"(sl));
    return r;
}
// T = y w - qhat' q in [0, 3q)
__device__ __forceinline__ u64 shoup_bfly(u64 y, u64 w, u64 wsh, u64 q) { return y * w - mulhi_approx(y, wsh) * q; }
// forward: corrected stages fold x >= 8q (inputs < 14q), outputs < 11q; uncorrected: inputs < 11q -> < 14q
constexpr int FWD_FOLD = 8, FWD_T = 3;
#else
__device__ __forceinline__ u64 shoup_bfly(u64 y, u64 w, u64 wsh, u64 q) { return mul_shoup_lazy(y, w, wsh, q); }
constexpr int FWD_FOLD = 4, FWD_T = 2;
#endif

// ---------------------------------------------------------------------------------------------
// Arithmetic policies.  Values travel in 64-bit registers; a row (one prime) uses one policy for
// both passes, so the intermediate buffer between the passes holds that policy's representation.
// ---------------------------------------------------------------------------------------------
struct PrimeC {
    u64 q;
    double qd, qinv;
};

// Integer Shoup path (any prime < 2^60).  Forward CT, lazy every other stage: T = y w in [0, 3q)
// (approximate quotient) or [0, 2q); x' = X + T, y' = X - T + FWD_T q.  Corrected stages (odd global
// stage) fold X = x >= FWD_FOLD q ? x - FWD_FOLD q : x.  Inverse GS keeps values < 4q (< 2q exact).
struct IntA {
    template <bool CORR>
    static __device__ __forceinline__ void ct(u64 &x, u64 &y, ulonglong2 w, const PrimeC &P) {
        const u64 q = P.q;
        u64 X = x;
        if (CORR) X = X >= FWD_FOLD * q ? X - FWD_FOLD * q : X;
        const u64 T = shoup_bfly(y, w.x, w.y, q);
        x = X + T;
        y = X - T + FWD_T * q;
    }
    template <bool RED>
    static __device__ __forceinline__ void gs(u64 &x, u64 &y, ulonglong2 w, const PrimeC &P) {
        constexpr int B = NTT_APPROX_HI ? 4 : 2;
        const u64 q = P.q, X = x, Y = y, T = X + Y;
        x = T >= B * q ? T - B * q : T;
        y = shoup_bfly(X - Y + B * q, w.x, w.y, q);
    }
    static __device__ __forceinline__ u64 in(u64 x, const PrimeC &) { return x; }
    // {w, Shoup companion} (16-byte interleaved table)
    static constexpr bool PAIRS = false;
    static __device__ __forceinline__ ulonglong2 twiddle(const ulonglong2 *tw, int i, const PrimeC &) {
        return __ldg(tw + i);
    }
    static __device__ __forceinline__ void twiddle2(const ulonglong2 *, int, const PrimeC &, ulonglong2 &,
                                                    ulonglong2 &) {}
    // forward output (< 11q or < 6q) -> [0, q)
    static __device__ __forceinline__ u64 out_fwd(u64 x, const PrimeC &P) {
        const u64 q = P.q;
        if (NTT_APPROX_HI) x = csub(x, 8 * q);
        return csub(csub(csub(x, 4 * q), 2 * q), q);
    }
    // inverse output times a per-limb factor k (Shoup companion ksh) -> [0, q)
    static __device__ __forceinline__ u64 out_scaled(u64 x, u64 k, u64 ksh, const PrimeC &P) {
        return mul_shoup(x, k, ksh, P.q);
    }
};

// Exact FP64 path (primes < 2^46, i.e. the 45-bit chain of configs[4]).  Values are signed integers
// held exactly in IEEE doubles (|v| < 2^51).  w y mod q with w_q = RN(w / q):
//   k = rint(y w_q) (fma with the 1.5 2^52 magic constant), (ph, pl) = TwoProduct(k, q),
//   r = fma(y, w, -ph) - pl  =  y w - k q  exactly,  |r| <= 0.75 q.
// Forward CT needs no corrections at all (|v| <= q + 16 * 0.75 q); inverse GS reduces the sum on
// every fourth stage (|v| <= 12 q; the product input X - Y <= 16 q keeps |y w / q| < 2^51).  All operations are on the FP64 pipe, which the integer path leaves
// idle; the explicit _rn intrinsics keep the compiler from contracting or reassociating.
constexpr double FP_MAGIC = 6755399441055744.0;  // 1.5 * 2^52
constexpr double TWO52 = 4503599627370496.0;
struct FpA {
    static __device__ __forceinline__ double D(u64 b) { return __longlong_as_double((long long)b); }
    static __device__ __forceinline__ u64 B(double d) { return (u64)__double_as_longlong(d); }
    static __device__ __forceinline__ double rint_(double x) { return __dsub_rn(__dadd_rn(x, FP_MAGIC), FP_MAGIC); }
    static __device__ __forceinline__ double mm(double y, double w, double wq, double qd) {
        const double k = __dsub_rn(__fma_rn(y, wq, FP_MAGIC), FP_MAGIC);
        const double ph = __dmul_rn(k, qd);
        const double pl = __fma_rn(k, qd, -ph);
        return __dsub_rn(__fma_rn(y, w, -ph), pl);
    }
    // centred representative, |result| <= q/2 (for |x| < 2^51)
    static __device__ __forceinline__ double red(double x, const PrimeC &P) {
        const double k = rint_(__dmul_rn(x, P.qinv));
        return __fma_rn(-k, P.qd, x);
    }
    template <bool CORR>
    static __device__ __forceinline__ void ct(u64 &x, u64 &y, ulonglong2 w, const PrimeC &P) {
        const double X = D(x), T = mm(D(y), D(w.x), D(w.y), P.qd);
        x = B(__dadd_rn(X, T));
        y = B(__dsub_rn(X, T));
    }
    template <bool RED>
    static __device__ __forceinline__ void gs(u64 &x, u64 &y, ulonglong2 w, const PrimeC &P) {
        const double X = D(x), Y = D(y);
        double s = __dadd_rn(X, Y);
        if (RED) s = red(s, P);
        y = B(mm(__dsub_rn(X, Y), D(w.x), D(w.y), P.qd));
        x = B(s);
    }
    // dense table of doubles w (the prime's 2N-word table region holds N doubles); w_q = RN(w RN(1/q))
    // has relative error <= 2^-52, so |y w_q - y w / q| <= 13 q 2^-52 < 0.2 and |r| <= 0.7 q still holds
    static __device__ __forceinline__ ulonglong2 twiddle(const ulonglong2 *tw, int i, const PrimeC &P) {
        const double w = __ldg(reinterpret_cast<const double *>(tw) + i);
        return make_ulonglong2(B(w), B(__dmul_rn(w, P.qinv)));
    }
    // entries i, i + 1 (i even) with one 16-byte load
    static constexpr bool PAIRS = true;
    static __device__ __forceinline__ void twiddle2(const ulonglong2 *tw, int i, const PrimeC &P, ulonglong2 &w0,
                                                    ulonglong2 &w1) {
        const double2 w = __ldg(reinterpret_cast<const double2 *>(reinterpret_cast<const double *>(tw) + i));
        w0 = make_ulonglong2(B(w.x), B(__dmul_rn(w.x, P.qinv)));
        w1 = make_ulonglong2(B(w.y), B(__dmul_rn(w.y, P.qinv)));
    }
    // canonical integer (< 2^52) -> exact double
    static __device__ __forceinline__ u64 in(u64 x, const PrimeC &) {
        return B(__dsub_rn(D(x | 0x4330000000000000ULL), TWO52));
    }
    // exact integer t (|t| < 2^51) -> two's complement int64 (t + 1.5 2^52 has t in its low mantissa bits)
    static __device__ __forceinline__ i64 to_int(double t) {
        return (i64)B(__dadd_rn(t, FP_MAGIC)) - (i64)B(FP_MAGIC);
    }
    // canonical residue: r = t - rint(t / q) q in [-q/2, q/2] (exact), then + q when negative on the
    // integer pipe (4 FP64 operations)
    static __device__ __forceinline__ u64 canon(double t, const PrimeC &P) {
        const double k = __dsub_rn(__fma_rn(t, P.qinv, FP_MAGIC), FP_MAGIC);
        const i64 r = to_int(__fma_rn(-k, P.qd, t));
        return (u64)(r + ((r >> 63) & (i64)P.q));
    }
    static __device__ __forceinline__ u64 out_fwd(u64 x, const PrimeC &P) { return canon(D(x), P); }
    // mm's result already lies in [-0.75 q, 0.75 q]: one conditional add of q (integer pipe) makes it
    // canonical (no second quotient)
    static __device__ __forceinline__ u64 out_scaled(u64 x, u64 k, u64, const PrimeC &P) {
        const double kd = D(in(k, P)), kq = __dmul_rn(kd, P.qinv);
        const i64 r = to_int(mm(D(x), kd, kq, P.qd));
        return (u64)(r + ((r >> 63) & (i64)P.q));
    }
};

// Exact FP64 path for the ~50-bit primes (2^46 <= q < 2^52 / 3.5 ~ 2^50.19: the bootstrap chains' 50-bit primes,
// the paper's ~49-bit primes).  Same exact product as FpA.  With y up to a few q the quotient k = rint(y w / q) is
// formed as fma(y, w/q, 1.5 2^52) - 1.5 2^52; once |y w / q| passes 2^51 that sum's ulp is 2, so with the w/q
// rounding |k - y w / q| <= 1 + |y| / 2^52 and |mm| <= q (1 + c 0.287) for |y| = c q (q / 2^52 <= 0.287).  mm
// stays exact while |r + pl| < 2^53 (pl <= ulp(y w) / 2 <= 2^50).  Bounds, worst case over the stages: forward CT
// folds X to [-q/2, q/2] on every other stage (the CORR stages, as IntA): outputs settle below 2.8 q after a
// folding stage and 4.6 q after the next (the multiplied input of 4.6 q gives |mm| <= 2.3 q); inverse GS folds the
// sum on every stage: |v| <= 2.35 q, differences <= 4.7 q.  Everything stays below 4.7 q < 2^52.4, an exact
// double integer.  red(x) = x - rint(x / q) q with rint by fma + the 1.5 2^52 magic (k <= 5: one fma gives the
// exact remainder).
struct FpB : FpA {
    static __device__ __forceinline__ double redB(double x, const PrimeC &P) {
        const double k = __dsub_rn(__fma_rn(x, P.qinv, FP_MAGIC), FP_MAGIC);
        return __fma_rn(-k, P.qd, x);
    }
    template <bool CORR>
    static __device__ __forceinline__ void ct(u64 &x, u64 &y, ulonglong2 w, const PrimeC &P) {
        double X = D(x);
        if (CORR) X = redB(X, P);
        const double T = mm(D(y), D(w.x), D(w.y), P.qd);
        x = B(__dadd_rn(X, T));
        y = B(__dsub_rn(X, T));
    }
    template <bool RED>
    static __device__ __forceinline__ void gs(u64 &x, u64 &y, ulonglong2 w, const PrimeC &P) {
        const double X = D(x), Y = D(y);
        y = B(mm(__dsub_rn(X, Y), D(w.x), D(w.y), P.qd));
        x = B(redB(__dadd_rn(X, Y), P));
    }
    // |mm| <= 2.4 q: a full canonicalisation
    static __device__ __forceinline__ u64 out_scaled(u64 x, u64 k, u64, const PrimeC &P) {
        const double kd = D(in(k, P)), kq = __dmul_rn(kd, P.qinv);
        return canon(mm(D(x), kd, kq, P.qd), P);
    }
};
constexpr u64 FPB_LIMIT = 1286742750677284ULL;  // floor(2^52 / 3.5)

// the arithmetic policy A reading its twiddles as 16-byte {w, w'} pairs (FpA: {w, w/q} of Tab::twp)
template <class A>
struct PairTw : A {
    static constexpr bool PAIRS = false;
    static __device__ __forceinline__ ulonglong2 twiddle(const ulonglong2 *tw, int i, const PrimeC &) {
        return __ldg(tw + i);
    }
    static __device__ __forceinline__ void twiddle2(const ulonglong2 *, int, const PrimeC &, ulonglong2 &,
                                                    ulonglong2 &) {}
};
#ifndef NTT_STRIDED_PAIRS
#define NTT_STRIDED_PAIRS 0  // measured: isolated 0.420 vs 0.412 us/limb, in-step neutral (profiles/r02_notes.md)
#endif

// [C]_q for a signed constant |C| < 2^62 (R9 constants), with the prime's Barrett constants
__device__ __forceinline__ u64 smod_dev(i128 C, u64 q, u64 br0, u64 br1) {
    const u128 a = (u128)(C < 0 ? -C : C);  // |C| < 2^120: within barrett128's 2^125
    const u64 m = barrett128(U128{(u64)a, (u64)(a >> 64)}, q, br0, br1);
    return (C < 0 && m) ? q - m : m;
}

// local index of held value v of thread tau when the held bits start at LO
template <int LO>
__device__ __forceinline__ int held(int tau, int v) {
    return ((tau >> LO) << (LO + RB)) | (v << LO) | (tau & ((1 << LO) - 1));
}

// Round k of a pass of S stages.  Forward rounds pair local bits hi = S-1-4k downwards, inverse
// rounds pair lo = 4k upwards; the held window [LO, LO+4) is clipped into [0, S).
template <int S, bool INV>
struct Rnd {
    static constexpr int NR = (S + RB - 1) / RB;
    __host__ __device__ static constexpr int first(int k) { return INV ? RB * k : S - 1 - RB * k; }
    __host__ __device__ static constexpr int nb(int k) {
        return INV ? (S - RB * k < RB ? S - RB * k : RB) : (S - RB * k < RB ? S - RB * k : RB);
    }
    __host__ __device__ static constexpr int lo(int k) {
        return INV ? (RB * k < S - RB ? RB * k : S - RB) : (S - 1 - RB * k - (RB - 1) > 0 ? S - RB * k - RB : 0);
    }
};

// One round of butterflies on the 16 held values.  Twiddle of the pair whose lower element has
// local index r, paired bit b: tw[2^sg + (g << (S-1-b)) + (r >> (b+1))] where sg is the global
// stage (strided: S-1-b, g = 0; contiguous: LOGN-1-b, g = group).  It depends only on the held bits
// above the paired one, so each distinct twiddle is loaded once.
template <int S, bool INV, int K, bool CONTIG, int LOGN, class A>
__device__ __forceinline__ void do_round(u64 (&v)[NV], int tau, int g, const ulonglong2 *__restrict__ tw,
                                         const PrimeC &P) {
    using R = Rnd<S, INV>;
    constexpr int LO = R::lo(K);
#pragma unroll
    for (int st = 0; st < R::nb(K); st++) {
        const int b = INV ? R::first(K) + st : R::first(K) - st;
        const int vb = b - LO;
        const int sg = CONTIG ? LOGN - 1 - b : S - 1 - b;
        const int gterm = CONTIG ? (g << (S - 1 - b)) : 0;
        // the distinct twiddles of this stage are consecutive table entries idx0 + u
        const int NTW = 1 << (RB - 1 - vb);  // compile-time after unrolling
        ulonglong2 ws[1 << (RB - 1)];
        {
            const int idx0 = (1 << sg) + gterm + (held<LO>(tau, 0) >> (b + 1));
            if (A::PAIRS && NTW >= 2) {
#pragma unroll
                for (int u = 0; u < NTW; u += 2) A::twiddle2(tw, idx0 + u, P, ws[u], ws[u + 1]);
            } else {
#pragma unroll
                for (int u = 0; u < NTW; u++) ws[u] = A::twiddle(tw, idx0 + u, P);
            }
        }
#pragma unroll
        for (int u = 0; u < NTW; u++) {
            const int v0b = u << (vb + 1);
            const ulonglong2 w = ws[u];
#pragma unroll
            for (int l = 0; l < (1 << vb); l++) {
                const int i0 = v0b | l, i1 = i0 | (1 << vb);
                if (INV) {
                    // FpA reduces the GS sum on every fourth stage only (|v| <= 12 q in between); IntA
                    // ignores the flag (its Harvey bounds reduce every stage)
                    if (sg & 3)
                        A::template gs<false>(v[i0], v[i1], w, P);
                    else
                        A::template gs<true>(v[i0], v[i1], w, P);
                } else if (sg & 1) {
                    A::template ct<true>(v[i0], v[i1], w, P);
                } else {
                    A::template ct<false>(v[i0], v[i1], w, P);
                }
            }
        }
    }
}


__device__ __forceinline__ PrimeC prime_consts(const Tab &tab, int prime) {
    PrimeC P;
    P.q = tab.q[prime];
    P.qd = tab.qd[prime];
    P.qinv = tab.qinv[prime];
    return P;
}

// Fused prologue / epilogue modes (NttFusion in kernels.h)
enum { IN_PLAIN = 0, IN_SRC = 1, IN_BCAST = 2, IN_MUL = 3, IN_MUL2 = 4, IN_LIN = 5 };
enum { OUT_PLAIN = 0, OUT_RESCALE = 1, OUT_MODDOWN = 2 };

}  // namespace
