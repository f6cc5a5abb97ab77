// ntt.cu -- batched multi-limb negacyclic NTT / INTT for sm_100a.
//
// Definition (R4): NTT(a)[i] = sum_k a_k psi^{(2 brv(i)+1) k} mod q, computed with the
// merged Cooley-Tukey network (twiddle psi^{brv(m+i)} at stage m) and its Gentleman-Sande inverse.
//
// Decomposition: N = 2^LOGN = G1 * G2 (G = 2^S, S1 = LOGN/2, S2 = LOGN - S1).  Two passes over a limb:
//   forward : pass 1 = stages 0..S1-1 on "columns" {c + (N/G1) r}   (strided groups)
//             pass 2 = stages S1..LOGN-1 on contiguous blocks of G2
//   inverse : pass A = GS stages LOGN-1..S1 on contiguous blocks, pass B = stages S1-1..0 on columns
// Radix-16 register rounds: a group of G elements is held by G/16 threads, 16 values each, so one
// round runs four butterfly stages on registers (LOGN = 16: two rounds per pass, one shared-memory
// exchange).  A round needs 1 + 2 + 4 + 8 = 15 distinct twiddles per thread, loaded once each as a
// 16-byte {w, w'} pair (interleaved Shoup table).
// Global access: strided passes put 16 consecutive columns in one CTA, so every load/store
// instruction of a half-warp covers one full 128-byte line; contiguous passes read (forward) or
// write (inverse) straight from registers in a lane-consecutive layout and stage the other side
// through padded shared memory with 16-byte vectors.
// Arithmetic (per row, by prime class): primes < 2^46 use exact-FP64 butterflies (FpA: signed integers
// held exactly in doubles, TwoProduct remainders, no forward corrections); larger primes (< 2^60) use
// Harvey lazy butterflies with Shoup twiddles (IntA: forward values below 8q with a correction on every
// other stage, inverse in [0, 4q)).  The last pass reduces to [0, q) (the inverse folds in N^{-1} or a
// caller-supplied per-limb factor).  Launch level: programmatic dependent launch, an L2 prefetch of the
// next wave's tiles in the first forward pass and of the epilogue operands in the fused epilogues,
// batched-segment launches of independent transforms (ntt_segments), and an optional single-pass
// thread-block-cluster kernel (ntt_cluster, SECPE_NTT_CLUSTER).
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "ntt_core.cuh"
#include "fpk.cuh"

#ifndef NTT_WAVE_PREFETCH_INV
#define NTT_WAVE_PREFETCH_INV 0  // the same next-wave L2 prefetch in the inverse's last (strided) pass
#endif
#ifndef NTT_KSI_MINB
#define NTT_KSI_MINB 3  // resident CTAs per SM of the fused ModUp pass 2 + key inner product kernel
#endif
#ifndef KSI_CPB
#define KSI_CPB 1  // ciphertexts per CTA of the fused kernel (2: one key load serves two tiles -- measured slower: partial sums
                   // spill from L2 to DRAM, 71.8 vs 68.0 ms per argmax step)
#endif
#ifndef NTT_KSI_PREFETCH
#define NTT_KSI_PREFETCH 1  // per digit: L2 prefetch of its key tiles and the next digit's tile (all tiles at kernel start: evicted before use, slower)
#endif

namespace {


// A launch covers one row range of one buffer, or (nseg > 0, plain transforms only) up to MAXSEG
// independent row ranges of several buffers: small transforms batched into one grid (a transform of a
// few rows costs about one CTA latency per pass, ~10 us, whatever its size).
constexpr int MAXSEG = 8;
struct Seg {
    RowsArg d;
    LimbMap lm;
    int limb0, nsub;  // limbs [limb0, limb0 + nsub) of every polynomial of the segment
    int row0;         // first grid row (blockIdx.y) of the segment
};
struct PassArgs {
    RowsArg d;  // transform buffer rows (row = poly * nl + limb)
    LimbMap lm;
    Tab tab;
    NttFusion f;
    int limb0, nsub;  // this launch covers limbs [limb0, limb0 + nsub) of every polynomial (one prime class)
    int poly0;        // ... of polynomials poly0, poly0 + 1, ... (L2-sized chunks, see run())
    int nseg = 0;     // > 0: the rows come from seg[0 .. nseg) instead (d, lm, limb0, nsub, poly0 unused)
    int wave = 0;     // CTAs resident at once (grid-linear distance of the tile prefetched one wave ahead)
    Seg seg[MAXSEG];
};

// grid row y -> buffer, polynomial, limb, prime
__device__ __forceinline__ void locate(const PassArgs &a, int y, RowsArg &d, int &poly, int &limb, int &prime) {
    if (a.nseg == 0) {
        d = a.d;
        poly = a.poly0 + y / a.nsub;
        limb = a.limb0 + y % a.nsub;
        prime = prime_of(a.lm, limb);
        return;
    }
    int si = 0;
#pragma unroll
    for (int i = 1; i < MAXSEG; i++)
        if (i < a.nseg && y >= a.seg[i].row0) si = i;
    const Seg &g = a.seg[si];
    const int local = y - g.row0;
    d = g.d;
    poly = local / g.nsub;
    limb = g.limb0 + local % g.nsub;
    prime = prime_of(g.lm, limb);
}

// ---------------------------------------------------------------------------------------------
// strided pass: group = column c, elements c + (N >> S) r, SC columns per CTA
//   forward: stages 0..S-1 (first pass);  inverse: stages S-1..0 (last pass, * N^{-1})
// ---------------------------------------------------------------------------------------------
template <int LOGN, bool INV, int IN, class A>
__device__ __forceinline__ void strided_body(const PassArgs &a, const RowsArg &d, u64 *sm, int poly, int limb,
                                             int prime, const PrimeC &P) {
    constexpr int S = LOGN / 2;
    constexpr long N = 1L << LOGN;
    constexpr int STRIDE = (int)(N >> S);
    using R = Rnd<S, INV>;
    const int cl = threadIdx.x % SC, tau = threadIdx.x / SC;
    const int c = blockIdx.x * SC + cl;
    u64 *base = d.p + poly_off(d.cs, d.ps, poly) + limb * N + c;
    const u64 q = P.q;
#if NTT_STRIDED_PAIRS
    // column stages: 255 twiddles per prime, L1-resident -- the {w, w/q} pair table saves the per-twiddle DMUL
    using AT = typename std::conditional<std::is_same<A, FpA>::value, PairTw<A>, A>::type;
    const ulonglong2 *tw = (std::is_same<A, FpA>::value ? (INV ? a.tab.itwp : a.tab.twp) : (INV ? a.tab.itw2 : a.tab.tw2)) +
                           prime * N;
#else
    using AT = A;
    const ulonglong2 *tw = (INV ? a.tab.itw2 : a.tab.tw2) + prime * N;
#endif
    u64 v[NV];
    constexpr int LO0 = R::lo(0);
    if constexpr (IN == IN_BCAST) {
        // rescale (R12): T_i = [floor(q_l/2)]_{q_i} - [r]_{q_i}, r = [c_l + floor(q_l/2)]_{q_l};
        // the source row is the coefficient-form last limb of the same polynomial
        const u64 *src = a.f.src.p + poly_off(a.f.src.cs, a.f.src.ps, poly) + c;
        const u64 ql = a.tab.q[a.f.lp], hl = ql >> 1, hi = a.f.half[limb], one_sh = a.tab.br1[prime];
        if (std::is_same<A, FpA>::value && ql < (1ULL << 47)) {
            // exact-FP64 rows: [floor(q_l/2)]_{q_i} - r as an exact double, |v| < 2^47 (the forward stages need no
            // reduction of r mod q_i: their bound grows from 4 q instead of q, 16 q < 2^51)
            const double hd = FpA::D(FpA::in(hi, P));
#pragma unroll
            for (int k = 0; k < NV; k++) {
                const u64 r = csub(src[STRIDE * held<LO0>(tau, k)] + hl, ql);
                v[k] = FpA::B(__dsub_rn(hd, FpA::D(FpA::in(r, P))));
            }
        } else {
#pragma unroll
            for (int k = 0; k < NV; k++) {
                const u64 r = csub(src[STRIDE * held<LO0>(tau, k)] + hl, ql);
                v[k] = A::in(submod(hi, mul_shoup(r, 1, one_sh, q), q), P);
            }
        }
    } else if (!INV) {
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = A::in(NTT_LD(base + STRIDE * held<LO0>(tau, k)), P);
    } else {
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = base[STRIDE * held<LO0>(tau, k)];  // intermediate representation
    }
    do_round<S, INV, 0, false, LOGN, AT>(v, tau, 0, tw, P);
    if constexpr (R::NR > 1) {
#pragma unroll
        for (int k = 0; k < NV; k++) sm[held<R::lo(0)>(tau, k) * SC + cl] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = sm[held<R::lo(1)>(tau, k) * SC + cl];
        do_round<S, INV, 1, false, LOGN, AT>(v, tau, 0, tw, P);
    }
    static_assert(R::NR <= 2, "strided pass: at most two rounds");
    constexpr int LOL = R::lo(R::NR - 1);
    if (INV) {
        // last inverse pass: * N^{-1} (or a caller-supplied per-limb factor that includes it)
        const u64 ni = a.f.k ? a.f.k[limb] : a.tab.ninv[prime];
        const u64 nish = a.f.k ? a.f.ksh[limb] : a.tab.ninvsh[prime];
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = A::out_scaled(v[k], ni, nish, P);
    }
#pragma unroll
    for (int k = 0; k < NV; k++) NTT_ST(base + STRIDE * held<LOL>(tau, k), v[k]);
}


// resident CTAs per SM the register allocation targets: FP rows fit 64 registers (4 CTAs), the
// integer Shoup path needs 80 (3 CTAs)
template <class A>
struct MinB {
    static constexpr int v = NTT_MINB;
};
template <>
struct MinB<FpA> {
    static constexpr int v = NTT_MINB_FP;
};

template <int LOGN, bool INV, int IN, class A>
__global__ void __launch_bounds__(SC *(1 << (LOGN / 2 - RB)), MinB<A>::v) ntt_strided(PassArgs a) {
    __shared__ u64 sm[(1 << (LOGN / 2)) * SC];
    RowsArg d;
    int poly, limb, prime;
#if NTT_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
#if NTT_WAVE_PREFETCH
    if ((!INV || NTT_WAVE_PREFETCH_INV) && IN == IN_PLAIN && a.wave > 0) {
        // the tile a CTA of the next wave will read: one 128-byte row segment per thread into L2
        constexpr int S = LOGN / 2;
        constexpr long N = 1L << LOGN;
        static_assert((1 << S) == SC * (1 << (S - RB)), "one row segment per thread");
        const long t = (long)blockIdx.y * gridDim.x + blockIdx.x + a.wave;
        if (t < (long)gridDim.x * gridDim.y) {
            RowsArg d2;
            int p2, l2, pr2;
            locate(a, (int)(t / gridDim.x), d2, p2, l2, pr2);
            const u64 *g = d2.p + poly_off(d2.cs, d2.ps, p2) + l2 * N + (t % gridDim.x) * SC + (N >> S) * threadIdx.x;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(g));
        }
    }
#endif
    locate(a, blockIdx.y, d, poly, limb, prime);
    const PrimeC P = prime_consts(a.tab, prime);
    strided_body<LOGN, INV, IN, A>(a, d, sm, poly, limb, prime, P);
}

// ---------------------------------------------------------------------------------------------
// contiguous pass: group = block of G consecutive elements, CT / (G/16) groups per CTA
//   forward: stages S1..LOGN-1 (last pass, reduce to [0, q));  inverse: stages LOGN-1..S1 (first)
// ---------------------------------------------------------------------------------------------
template <int LOGN>
struct ContigCfg {
    static constexpr int S = LOGN - LOGN / 2;
    static constexpr int G = 1 << S;
    static constexpr int TPG = G / NV;
    static constexpr int CG = CT / TPG;
    static constexpr int PITCH = G + G / 16;  // one pad word per 16: conflict-free both layouts
};
__device__ __forceinline__ int padr(int r) { return r + (r >> 4); }

template <int LOGN, bool INV, int IO, class A>
__device__ __forceinline__ void contig_body(const PassArgs &a, const RowsArg &d, u64 *sm, int poly, int limb,
                                            int prime, const PrimeC &P) {
    // IO: inverse -> IN_PLAIN | IN_SRC | IN_MUL (first pass reads f.src rows);  forward -> OUT_* epilogue
    using CF = ContigCfg<LOGN>;
    constexpr int S = CF::S, G = CF::G, TPG = CF::TPG, CG = CF::CG, PITCH = CF::PITCH;
    constexpr long N = 1L << LOGN;
    using R = Rnd<S, INV>;
    static_assert(R::NR == 2, "contiguous pass: two rounds");
    const long boff = limb * N + (long)blockIdx.x * CG * G;  // tile offset inside the polynomial
    u64 *blk = d.p + poly_off(d.cs, d.ps, poly) + boff;
    const u64 q = P.q;
#if NTT_EPI_PREFETCH
    if (!INV && IO != OUT_PLAIN) {
        // the epilogue operands do not depend on the transform: start pulling this tile's lines into L2
        // now (one 128-byte line per thread) so the epilogue does not wait on DRAM latency
        static_assert(CG * G * 8 == CT * 128, "one line per thread");
        const char *p1 = reinterpret_cast<const char *>(a.f.e1.p + poly_off(a.f.e1.cs, a.f.e1.ps, poly) + boff);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p1 + threadIdx.x * 128));
        if (IO == OUT_RESCALE && a.f.lin == 2) {
            const char *pb = reinterpret_cast<const char *>(a.f.e1b.p + poly_off(a.f.e1b.cs, a.f.e1b.ps, poly) + boff);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + threadIdx.x * 128));
        }
        if (IO == OUT_MODDOWN && (poly & 1) < a.f.e2_polys) {
            const char *p2 = reinterpret_cast<const char *>(a.f.e2.p + poly_off(a.f.e2.cs, a.f.e2.ps, poly) + boff);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p2 + threadIdx.x * 128));
        }
        if (IO == OUT_MODDOWN && a.f.e3.p) {
            const char *p3 = reinterpret_cast<const char *>(a.f.e3.p + poly_off(a.f.e3.cs, a.f.e3.ps, poly) + boff);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p3 + threadIdx.x * 128));
        }
    }
#endif
    const ulonglong2 *tw = (INV ? a.tab.itw2 : a.tab.tw2) + prime * N;
    const int gl = threadIdx.x / TPG, tau = threadIdx.x % TPG;
    const int g = blockIdx.x * CG + gl;
    u64 *smg = sm + gl * PITCH;
    u64 v[NV];
    constexpr int LO0 = R::lo(0), LO1 = R::lo(1);
    if (!INV) {
        // forward round 0 holds r = 16 k + tau: lane-consecutive, load straight from global
        const u64 *src = blk + gl * G;
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = NTT_LD(src + held<LO0>(tau, k));  // intermediate representation
    } else {
        const u64 *sp = (IO == IN_SRC || IO == IN_MUL || IO == IN_MUL2 || IO == IN_LIN)
                            ? a.f.src.p + poly_off(a.f.src.cs, a.f.src.ps, poly) + boff
                            : blk;
        const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(sp);
        const ulonglong2 *src2 = nullptr, *src3 = nullptr, *src4 = nullptr;
        if (IO == IN_MUL || IO == IN_MUL2 || (IO == IN_LIN && a.f.lin == 2))
            src2 = reinterpret_cast<const ulonglong2 *>(a.f.src2.p + poly_off(a.f.src2.cs, a.f.src2.ps, poly) + boff);
        if (IO == IN_MUL2) {
            src3 = reinterpret_cast<const ulonglong2 *>(a.f.src3.p + poly_off(a.f.src3.cs, a.f.src3.ps, poly) + boff);
            src4 = reinterpret_cast<const ulonglong2 *>(a.f.src4.p + poly_off(a.f.src4.cs, a.f.src4.ps, poly) + boff);
        }
        const u64 br0 = a.tab.br0[prime], br1 = a.tab.br1[prime];
        const u64 lc1 = IO == IN_LIN ? smod_dev(a.f.C1, q, br0, br1) : 0;
        const u64 lc2 = IO == IN_LIN && a.f.lin == 2 ? smod_dev(a.f.C2, q, br0, br1) : 0;
        constexpr bool FPX = std::is_same<A, FpA>::value && (IO == IN_MUL || IO == IN_MUL2 || IO == IN_LIN);
        if (FPX) {
            // exact-FP64 rows: the fused products as FpA exact products of canonical operands (the sum of up to
            // two products, |v| <= 1.5 q, enters the GS stages as it is: their bound analysis holds up to 24 q)
            const double c1d = FpA::D(FpA::in(lc1, P)), c1q = __dmul_rn(c1d, P.qinv);
            const double c2d = FpA::D(FpA::in(lc2, P)), c2q = __dmul_rn(c2d, P.qinv);
            auto fd = [&](u64 x) { return FpA::D(FpA::in(x, P)); };
#pragma unroll 4
            for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
                const ulonglong2 x = NTT_LD2(src + i);
                double r0, r1;
                if (IO == IN_LIN) {
                    r0 = FpA::mm(fd(x.x), c1d, c1q, P.qd);
                    r1 = FpA::mm(fd(x.y), c1d, c1q, P.qd);
                    if (src2) {
                        const ulonglong2 y = src2[i];
                        r0 = __dadd_rn(r0, FpA::mm(fd(y.x), c2d, c2q, P.qd));
                        r1 = __dadd_rn(r1, FpA::mm(fd(y.y), c2d, c2q, P.qd));
                    }
                } else {
                    const ulonglong2 y = src2[i];
                    const double y0 = fd(y.x), y1 = fd(y.y);
                    r0 = FpA::mm(fd(x.x), y0, __dmul_rn(y0, P.qinv), P.qd);
                    r1 = FpA::mm(fd(x.y), y1, __dmul_rn(y1, P.qinv), P.qd);
                    if (IO == IN_MUL2) {
                        const ulonglong2 z = src3[i], w = src4[i];
                        const double w0 = fd(w.x), w1 = fd(w.y);
                        r0 = __dadd_rn(r0, FpA::mm(fd(z.x), w0, __dmul_rn(w0, P.qinv), P.qd));
                        r1 = __dadd_rn(r1, FpA::mm(fd(z.y), w1, __dmul_rn(w1, P.qinv), P.qd));
                    }
                }
                const int e = 2 * i, gg = e / G, r = e % G;
                sm[gg * PITCH + padr(r)] = FpA::B(r0);
                sm[gg * PITCH + padr(r + 1)] = FpA::B(r1);
            }
        } else
#pragma unroll 4
        for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
            ulonglong2 x = NTT_LD2(src + i);
            if (IO == IN_LIN) {
                U128 t0 = mul_wide(x.x, lc1), t1 = mul_wide(x.y, lc1);
                if (src2) {
                    const ulonglong2 y = src2[i];
                    mac_wide(t0, y.x, lc2);
                    mac_wide(t1, y.y, lc2);
                }
                x.x = barrett128(t0, q, br0, br1);
                x.y = barrett128(t1, q, br0, br1);
            } else if (IO == IN_MUL) {
                const ulonglong2 y = src2[i];
                x.x = mulmod(x.x, y.x, q, br0, br1);
                x.y = mulmod(x.y, y.y, q, br0, br1);
            } else if (IO == IN_MUL2) {
                const ulonglong2 y = src2[i], z = src3[i], w = src4[i];
                U128 t0 = mul_wide(x.x, y.x), t1 = mul_wide(x.y, y.y);
                mac_wide(t0, z.x, w.x);
                mac_wide(t1, z.y, w.y);
                x.x = barrett128(t0, q, br0, br1);
                x.y = barrett128(t1, q, br0, br1);
            }
            const int e = 2 * i, gg = e / G, r = e % G;
            sm[gg * PITCH + padr(r)] = A::in(x.x, P);
            sm[gg * PITCH + padr(r + 1)] = A::in(x.y, P);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = smg[padr(held<LO0>(tau, k))];
        // no barrier: each thread rewrites exactly the words it just read (same layout)
    }
    do_round<S, INV, 0, true, LOGN, A>(v, tau, g, tw, P);
#pragma unroll
    for (int k = 0; k < NV; k++) smg[padr(held<LO0>(tau, k))] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; k++) v[k] = smg[padr(held<LO1>(tau, k))];
    do_round<S, INV, 1, true, LOGN, A>(v, tau, g, tw, P);
    // exact-FP64 rows with a fused epilogue: the transform's doubles (|v| <= 13 q) go into the epilogue as they
    // are and its products are FpA exact products (one canonicalisation per output instead of Shoup / Barrett)
    constexpr bool FPE = std::is_same<A, FpA>::value && !INV && (IO == OUT_RESCALE || IO == OUT_MODDOWN);
    if (!INV) {
        if (!FPE) {
#pragma unroll
            for (int k = 0; k < NV; k++) v[k] = A::out_fwd(v[k], P);
        }
        // no barrier: each thread rewrites exactly the words it read for round 1
#pragma unroll
        for (int k = 0; k < NV; k++) smg[padr(held<LO1>(tau, k))] = v[k];
        __syncthreads();
        // epilogue on 16-byte vectors; element e of the tile is at boff + e in its polynomial
        const ulonglong2 *e1 = nullptr, *e2 = nullptr, *e3 = nullptr, *e1b = nullptr;
        ulonglong2 *dst;
        u64 kc = 0, kcsh = 0, lc1 = 0, lc2 = 0, br0e = 0, br1e = 0;
        if (IO == OUT_PLAIN) {
            dst = reinterpret_cast<ulonglong2 *>(blk);
        } else {
            const int P = poly;
            e1 = reinterpret_cast<const ulonglong2 *>(a.f.e1.p + poly_off(a.f.e1.cs, a.f.e1.ps, P) + boff);
            if (IO == OUT_RESCALE && a.f.lin) {
                br0e = a.tab.br0[prime];
                br1e = a.tab.br1[prime];
                lc1 = smod_dev(a.f.C1, q, br0e, br1e);
                if (a.f.lin == 2) {
                    lc2 = smod_dev(a.f.C2, q, br0e, br1e);
                    e1b = reinterpret_cast<const ulonglong2 *>(a.f.e1b.p + poly_off(a.f.e1b.cs, a.f.e1b.ps, P) + boff);
                }
            }
            if (IO == OUT_MODDOWN && (P & 1) < a.f.e2_polys)
                e2 = reinterpret_cast<const ulonglong2 *>(a.f.e2.p + poly_off(a.f.e2.cs, a.f.e2.ps, P) + boff);
            if (IO == OUT_MODDOWN && a.f.e3.p)
                e3 = reinterpret_cast<const ulonglong2 *>(a.f.e3.p + poly_off(a.f.e3.cs, a.f.e3.ps, P) + boff);
            dst = reinterpret_cast<ulonglong2 *>(a.f.out.p + poly_off(a.f.out.cs, a.f.out.ps, P) + boff);
            kc = a.f.k[limb];
            kcsh = a.f.ksh[limb];
        }
        if (FPE) {
            const double kd = FpA::D(FpA::in(kc, P)), kq = __dmul_rn(kd, P.qinv);
            const double c1d = FpA::D(FpA::in(lc1, P)), c1q = __dmul_rn(c1d, P.qinv);
            const double c2d = FpA::D(FpA::in(lc2, P)), c2q = __dmul_rn(c2d, P.qinv);
            auto fd = [&](u64 x) { return FpA::D(FpA::in(x, P)); };
            // mm result in [-0.75 q, 0.75 q] -> canonical with one conditional add (integer pipe)
            auto fix = [&](double t) {
                const i64 r = FpA::to_int(t);
                return (u64)(r + ((r >> 63) & (i64)q));
            };
#pragma unroll 4
            for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
                const int e = 2 * i, gg = e / G, r = e % G;
                const double x0 = FpA::D(sm[gg * PITCH + padr(r)]), x1 = FpA::D(sm[gg * PITCH + padr(r + 1)]);
                const ulonglong2 c = e1[i];
                u64 o0, o1;
                if (IO == OUT_RESCALE) {
                    // (C1 e1 [+ C2 e1b] + NTT(T)) q_l^{-1}
                    double c0d = fd(c.x), c1v = fd(c.y);
                    if (a.f.lin) {
                        c0d = FpA::mm(c0d, c1d, c1q, P.qd);
                        c1v = FpA::mm(c1v, c1d, c1q, P.qd);
                        if (e1b) {
                            const ulonglong2 y = e1b[i];
                            c0d = __dadd_rn(c0d, FpA::mm(fd(y.x), c2d, c2q, P.qd));
                            c1v = __dadd_rn(c1v, FpA::mm(fd(y.y), c2d, c2q, P.qd));
                        }
                    }
                    o0 = fix(FpA::mm(__dadd_rn(c0d, x0), kd, kq, P.qd));
                    o1 = fix(FpA::mm(__dadd_rn(c1v, x1), kd, kq, P.qd));
                } else {
                    // (acc - NTT(T)) P^{-1} (+ addends): |sum| <= 2.75 q -> canonical
                    double t0 = FpA::mm(__dsub_rn(fd(c.x), x0), kd, kq, P.qd);
                    double t1 = FpA::mm(__dsub_rn(fd(c.y), x1), kd, kq, P.qd);
                    if (e2) {
                        const ulonglong2 d = e2[i];
                        t0 = __dadd_rn(t0, fd(d.x));
                        t1 = __dadd_rn(t1, fd(d.y));
                    }
                    if (e3) {
                        const ulonglong2 d = e3[i];
                        t0 = __dadd_rn(t0, fd(d.x));
                        t1 = __dadd_rn(t1, fd(d.y));
                    }
                    o0 = FpA::canon(t0, P);
                    o1 = FpA::canon(t1, P);
                }
                NTT_ST2(dst + i, make_ulonglong2(o0, o1));
            }
        } else
#pragma unroll 4
        for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
            const int e = 2 * i, gg = e / G, r = e % G;
            u64 x0 = sm[gg * PITCH + padr(r)], x1 = sm[gg * PITCH + padr(r + 1)];
            if (IO == OUT_RESCALE) {
                // (c_i + NTT(T)_i) * q_l^{-1};  c_i = C1 e1_i (+ C2 e1b_i) for a fused constant product
                ulonglong2 c = e1[i];
                if (a.f.lin) {
                    U128 t0 = mul_wide(c.x, lc1), t1 = mul_wide(c.y, lc1);
                    if (e1b) {
                        const ulonglong2 y = e1b[i];
                        mac_wide(t0, y.x, lc2);
                        mac_wide(t1, y.y, lc2);
                    }
                    c.x = barrett128(t0, q, br0e, br1e);
                    c.y = barrett128(t1, q, br0e, br1e);
                }
                x0 = mul_shoup(addmod(c.x, x0, q), kc, kcsh, q);
                x1 = mul_shoup(addmod(c.y, x1, q), kc, kcsh, q);
            } else if (IO == OUT_MODDOWN) {
                // (acc_i - NTT(T)_i) * P^{-1} (+ addend)
                const ulonglong2 c = e1[i];
                x0 = mul_shoup(submod(c.x, x0, q), kc, kcsh, q);
                x1 = mul_shoup(submod(c.y, x1, q), kc, kcsh, q);
                if (e2) {
                    const ulonglong2 d = e2[i];
                    x0 = addmod(x0, d.x, q);
                    x1 = addmod(x1, d.y, q);
                }
                if (e3) {
                    const ulonglong2 d = e3[i];
                    x0 = addmod(x0, d.x, q);
                    x1 = addmod(x1, d.y, q);
                }
            }
            NTT_ST2(dst + i, make_ulonglong2(x0, x1));
        }
    } else {
        // inverse round 1 holds r = 16 k + tau (LO = S - 4): store straight to global
        u64 *dst = blk + gl * G;
#pragma unroll
        for (int k = 0; k < NV; k++) NTT_ST(dst + held<LO1>(tau, k), v[k]);
    }
}

template <int LOGN, bool INV, int IO, class A>
__global__ void __launch_bounds__(CT, MinB<A>::v) ntt_contig(PassArgs a) {
    using CF = ContigCfg<LOGN>;
    __shared__ __align__(16) u64 sm[CF::CG * CF::PITCH];
    RowsArg d;
    int poly, limb, prime;
#if NTT_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif

    locate(a, blockIdx.y, d, poly, limb, prime);
    const PrimeC P = prime_consts(a.tab, prime);
    contig_body<LOGN, INV, IO, A>(a, d, sm, poly, limb, prime, P);
}

// ---------------------------------------------------------------------------------------------
// Fused ModUp forward pass 2 + relinearise-and-rescale key inner product (R10/R11 key switching, every row
// exact-FP64).  CTA = (row e, ciphertext c, tile of CG G words): for each digit j with e outside I_j, the tile of
// ext[c][j][e] (after the first forward pass) runs stages S..LOGN-1 (the contiguous pass) and lands in shared
// memory as raw transform doubles (|v| <= 13 q, as the FPE epilogues); each word is multiplied with the key words
// key_j[0/1][e] (FpA exact products, |mm| <= 0.75 q).  The partial sums stay exact doubles and are parked in the
// acc rows between digits (the same thread re-reads its own words: L2-resident); the Q rows then add the
// tensor's terms (d2 = a1 b1 (+ a2_1 b2_1) with the own digit's key, [P] d0 / [P] d1) and every output is
// canonicalised once.  At most beta + 1 <= 5 terms: |s| <= 3.75 q, an exact double.  The same canonical
// residues as ks_inner_ten1_kernel (sums of exact products mod q), so the key-switch integers are unchanged.
// Rows are ordered e-major (ciphertexts of one row adjacent) so a key tile is read from HBM once per batch.
// ---------------------------------------------------------------------------------------------
// the ModDown's INTT rows (e >= f.intt_row0): the inverse NTT's first pass (GS stages LOGN-1..S, the contiguous pass
// with a plain input) on the tile this CTA just finished (canonical, L2-resident), written back in place in the
// inverse's intermediate representation -- the same words the separate first-pass launch would write
template <int LOGN, class A>
__device__ __forceinline__ void ksi_intt_rows(const Tab &tab, const KsFuse &f, int e, int pr, const PrimeC &P, long boff,
                                              int c0, int nc, long a1off, u64 *sm) {
    if (f.intt_row0 < 0 || e < f.intt_row0) return;
    using CF = ContigCfg<LOGN>;
    constexpr int S = CF::S, G = CF::G, TPG = CF::TPG, CG = CF::CG, PITCH = CF::PITCH;
    constexpr long N = 1L << LOGN;
    using R = Rnd<S, true>;
    constexpr int LO0 = R::lo(0), LO1 = R::lo(1);
    const ulonglong2 *itw = tab.itw2 + pr * N;
    const int gl = threadIdx.x / TPG, tau = threadIdx.x % TPG;
    const int g = blockIdx.x * CG + gl;
    u64 *smg = sm + gl * PITCH;
    for (int u = 0; u < nc; u++)
        for (int b = 0; b < 2; b++) {
            u64 *row = f.acc + (c0 + u) * f.accs + (long)e * N + boff + b * a1off;
            __syncthreads();  // this CTA's writes of the row (and the shared tile's previous use) are complete
            const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(row);
            for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
                const ulonglong2 x = src[i];
                const int el = 2 * i, gg = el / G, r = el % G;
                sm[gg * PITCH + padr(r)] = A::in(x.x, P);
                sm[gg * PITCH + padr(r + 1)] = A::in(x.y, P);
            }
            __syncthreads();
            u64 v[NV];
#pragma unroll
            for (int k = 0; k < NV; k++) v[k] = smg[padr(held<LO0>(tau, k))];
            do_round<S, true, 0, true, LOGN, A>(v, tau, g, itw, P);
#pragma unroll
            for (int k = 0; k < NV; k++) smg[padr(held<LO0>(tau, k))] = v[k];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NV; k++) v[k] = smg[padr(held<LO1>(tau, k))];
            do_round<S, true, 1, true, LOGN, A>(v, tau, g, itw, P);
            u64 *dst = row + gl * G;
#pragma unroll
            for (int k = 0; k < NV; k++) NTT_ST(dst + held<LO1>(tau, k), v[k]);
        }
}

// iterations of the digit epilogue in flight per thread: their key and partial-sum loads overlap (1 exposes every
// load's latency: measured 497 vs 442 us per launch at 8 ciphertexts)
constexpr int ksi_epi_unroll = KSI_CPB == 1 ? 4 : 1;
template <int LOGN, class A>
__device__ __forceinline__ void ksi_body(const Tab &tab, const KsFuse &f) {
    // A = the row's policy.  FpA (q < 2^46): raw transform doubles |v| <= 13 q go into the products, partial sums
    // unreduced.  FpB (~50-bit rows): every transform value centred first, |y| <= q/2 + 1, products |mm| <= 1.29 q,
    // partial sums centred per digit, the tensor formed canonically on the integer pipe -- every sum < 2^52.
    // IntA (larger primes): the transform canonicalised, 128-bit products (+ the parked canonical partial sum) and
    // one Barrett reduction per digit, the integer tensor -- the arithmetic of ks_inner_ten1_kernel's integer path.
    constexpr bool FB = std::is_same<A, FpB>::value;
    constexpr bool IA = std::is_same<A, IntA>::value;
    extern __shared__ __align__(16) u64 ksi_sm[];  // [KSI_CPB][CG * PITCH]
    using CF = ContigCfg<LOGN>;
    constexpr int S = CF::S, G = CF::G, TPG = CF::TPG, CG = CF::CG, PITCH = CF::PITCH;
    constexpr long N = 1L << LOGN;
    using R = Rnd<S, false>;
    constexpr int LO0 = R::lo(0), LO1 = R::lo(1);
    // KSI_CPB ciphertexts per CTA (one padded tile each): every key word loaded serves all of them
    const int ncg = (f.n_ct + KSI_CPB - 1) / KSI_CPB;
    const int e = f.e0 + blockIdx.y / ncg, c0 = (blockIdx.y % ncg) * KSI_CPB;
    const int nc = min(KSI_CPB, f.n_ct - c0);
    const int ne = f.nl + f.np, nk = f.nq_total + f.np;
    const bool qrow = e < f.nl;
    const int pr = qrow ? e : f.nq_total + (e - f.nl);
    const int jd = qrow ? e / f.alpha : -1;
    const PrimeC P = prime_consts(tab, pr);
    const double qd = P.qd, qinv = P.qinv;
    // centred residue of an exact double |v| < 2^52.5: |result| <= q/2 (+1)
    auto cen = [&](double v) { return __fma_rn(-__dsub_rn(__fma_rn(v, qinv, FP_MAGIC), FP_MAGIC), qd, v); };
    const long boff = (long)blockIdx.x * CG * G;
    const ulonglong2 *tw = tab.tw2 + pr * N;
    const int gl = threadIdx.x / TPG, tau = threadIdx.x % TPG;
    const int g = blockIdx.x * CG + gl;
    // acc rows of ciphertext c0 + u: b = 0 at accb(u), b = 1 at accb(u) + ne N
    auto accb = [&](int u) { return f.acc + (c0 + u) * f.accs + (long)e * N + boff; };
    const long a1off = (long)ne * N;
    const u64 *keyrow = f.key + (long)pr * N + boff;  // key_j[b] row of this prime: + (2 j + b) nk N
    auto fx = [](u64 x) { return fpt::d(x); };
#if NTT_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    const int ndig = qrow ? f.beta - 1 : f.beta;
    auto next_digit = [&](int j) {
        for (j = j + 1; j < f.beta; j++)
            if (j != jd) return j;
        return -1;
    };
    const long lo = (long)threadIdx.x * 16;  // this thread's 128-byte line of a tile (L2 prefetches)
    int nd = 0;
    {
    for (int j = next_digit(-1); j >= 0; j = next_digit(j)) {
        const bool fin = nd == ndig - 1 && !qrow;  // the last term of a special row: canonicalise
#if NTT_KSI_PREFETCH
        // this digit's key tiles into L2 while the rounds run
        asm volatile("prefetch.global.L2 [%0];" ::"l"(keyrow + (long)(2 * j) * nk * N + lo));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(keyrow + (long)(2 * j + 1) * nk * N + lo));
#endif
#pragma unroll 1
        for (int u = 0; u < nc; u++) {
            u64 *const smg = ksi_sm + u * CG * PITCH + gl * PITCH;
            const u64 *src = f.ext + (c0 + u) * f.exts + ((long)j * ne + e) * N + boff + gl * G;
            // opaque copy of the twiddle pointer: the twiddle loads stay inside the loop (hoisting them out of it
            // keeps 30 twiddle pairs live across the rounds and spills)
            const ulonglong2 *twu;
            asm volatile("mov.b64 %0, %1;" : "=l"(twu) : "l"(tw));
            u64 v[NV];
#pragma unroll
            for (int k = 0; k < NV; k++) v[k] = NTT_LD(src + held<LO0>(tau, k));  // first-pass representation
            do_round<S, false, 0, true, LOGN, A>(v, tau, g, twu, P);
#pragma unroll
            for (int k = 0; k < NV; k++) smg[padr(held<LO0>(tau, k))] = v[k];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NV; k++) v[k] = smg[padr(held<LO1>(tau, k))];
            do_round<S, false, 1, true, LOGN, A>(v, tau, g, twu, P);
            // no barrier: each thread rewrites exactly the words it read for round 1
#pragma unroll
            for (int k = 0; k < NV; k++) smg[padr(held<LO1>(tau, k))] = v[k];
        }
        __syncthreads();
        const ulonglong2 *kb = reinterpret_cast<const ulonglong2 *>(keyrow + (long)(2 * j) * nk * N);
        const ulonglong2 *ka = reinterpret_cast<const ulonglong2 *>(keyrow + (long)(2 * j + 1) * nk * N);
        if constexpr (IA) {
            const u64 r0 = tab.br0[pr], r1 = tab.br1[pr];
#pragma unroll 2
            for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
                const int el = 2 * i, gg = el / G, r = el % G;
                const ulonglong2 KB = __ldg(kb + i), KA = __ldg(ka + i);
#pragma unroll
                for (int u = 0; u < KSI_CPB; u++) {
                    if (u >= nc) break;
                    const u64 *sm = ksi_sm + u * CG * PITCH;
                    const u64 x0 = IntA::out_fwd(sm[gg * PITCH + padr(r)], P), x1 = IntA::out_fwd(sm[gg * PITCH + padr(r + 1)], P);
                    U128 t00 = mul_wide(x0, KB.x), t01 = mul_wide(x1, KB.y), t10 = mul_wide(x0, KA.x), t11 = mul_wide(x1, KA.y);
                    ulonglong2 *acc0 = reinterpret_cast<ulonglong2 *>(accb(u)), *acc1 = reinterpret_cast<ulonglong2 *>(accb(u) + a1off);
                    if (nd > 0) {
                        const ulonglong2 p0 = acc0[i], p1 = acc1[i];
                        add_wide(t00, U128{p0.x, 0});
                        add_wide(t01, U128{p0.y, 0});
                        add_wide(t10, U128{p1.x, 0});
                        add_wide(t11, U128{p1.y, 0});
                    }
                    acc0[i] = make_ulonglong2(barrett128(t00, P.q, r0, r1), barrett128(t01, P.q, r0, r1));
                    acc1[i] = make_ulonglong2(barrett128(t10, P.q, r0, r1), barrett128(t11, P.q, r0, r1));
                }
            }
        } else
#pragma unroll (ksi_epi_unroll)
        for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
            const int el = 2 * i, gg = el / G, r = el % G;
            const ulonglong2 KB = __ldg(kb + i), KA = __ldg(ka + i);
            const double B0 = fx(KB.x), B1 = fx(KB.y), A0 = fx(KA.x), A1 = fx(KA.y);
            const double B0q = __dmul_rn(B0, qinv), B1q = __dmul_rn(B1, qinv), A0q = __dmul_rn(A0, qinv),
                         A1q = __dmul_rn(A1, qinv);
#pragma unroll
            for (int u = 0; u < KSI_CPB; u++) {
                if (u >= nc) break;
                const u64 *sm = ksi_sm + u * CG * PITCH;
                double x0 = FpA::D(sm[gg * PITCH + padr(r)]), x1 = FpA::D(sm[gg * PITCH + padr(r + 1)]);
                if (FB) {
                    x0 = cen(x0);
                    x1 = cen(x1);
                }
                double s00 = fpt::mm(x0, B0, B0q, qd), s01 = fpt::mm(x1, B1, B1q, qd);
                double s10 = fpt::mm(x0, A0, A0q, qd), s11 = fpt::mm(x1, A1, A1q, qd);
                ulonglong2 *acc0 = reinterpret_cast<ulonglong2 *>(accb(u)), *acc1 = reinterpret_cast<ulonglong2 *>(accb(u) + a1off);
                if (nd > 0) {
                    const ulonglong2 p0 = acc0[i], p1 = acc1[i];
                    s00 = __dadd_rn(s00, FpA::D(p0.x));
                    s01 = __dadd_rn(s01, FpA::D(p0.y));
                    s10 = __dadd_rn(s10, FpA::D(p1.x));
                    s11 = __dadd_rn(s11, FpA::D(p1.y));
                }
                if (fin) {
                    acc0[i] = make_ulonglong2(fp_canon4(s00, P.q, qd, qinv), fp_canon4(s01, P.q, qd, qinv));
                    acc1[i] = make_ulonglong2(fp_canon4(s10, P.q, qd, qinv), fp_canon4(s11, P.q, qd, qinv));
                } else if (FB) {
                    acc0[i] = make_ulonglong2(FpA::B(cen(s00)), FpA::B(cen(s01)));
                    acc1[i] = make_ulonglong2(FpA::B(cen(s10)), FpA::B(cen(s11)));
                } else {
                    acc0[i] = make_ulonglong2(FpA::B(s00), FpA::B(s01));
                    acc1[i] = make_ulonglong2(FpA::B(s10), FpA::B(s11));
                }
            }
        }
        __syncthreads();  // the next digit's round 0 rewrites the shared tiles
        nd++;
    }
    }
    if (!qrow) {
        ksi_intt_rows<LOGN, A>(tab, f, e, pr, P, boff, c0, nc, a1off, ksi_sm);
        return;
    }
    if (!f.ten.a.p) {
        // plain key switch: the own digit's term is d_e (NTT form) times its key
        const ulonglong2 *kb = reinterpret_cast<const ulonglong2 *>(keyrow + (long)(2 * jd) * nk * N);
        const ulonglong2 *ka = reinterpret_cast<const ulonglong2 *>(keyrow + (long)(2 * jd + 1) * nk * N);
#pragma unroll 1
        for (int u = 0; u < nc; u++) {
            const ulonglong2 *dp = reinterpret_cast<const ulonglong2 *>(f.d + (c0 + u) * f.d_stride + (long)e * N + boff);
            ulonglong2 *acc0 = reinterpret_cast<ulonglong2 *>(accb(u)), *acc1 = reinterpret_cast<ulonglong2 *>(accb(u) + a1off);
            if constexpr (IA) {
                const u64 r0 = tab.br0[pr], r1 = tab.br1[pr];
#pragma unroll 2
                for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
                    const ulonglong2 X = dp[i], KB = __ldg(kb + i), KA = __ldg(ka + i);
                    U128 t00 = mul_wide(X.x, KB.x), t01 = mul_wide(X.y, KB.y), t10 = mul_wide(X.x, KA.x),
                         t11 = mul_wide(X.y, KA.y);
                    if (nd > 0) {
                        const ulonglong2 p0 = acc0[i], p1 = acc1[i];
                        add_wide(t00, U128{p0.x, 0});
                        add_wide(t01, U128{p0.y, 0});
                        add_wide(t10, U128{p1.x, 0});
                        add_wide(t11, U128{p1.y, 0});
                    }
                    acc0[i] = make_ulonglong2(barrett128(t00, P.q, r0, r1), barrett128(t01, P.q, r0, r1));
                    acc1[i] = make_ulonglong2(barrett128(t10, P.q, r0, r1), barrett128(t11, P.q, r0, r1));
                }
            } else
#pragma unroll 2
            for (int i = threadIdx.x; i < CG * G / 2; i += CT) {
                const ulonglong2 X = dp[i], KB = __ldg(kb + i), KA = __ldg(ka + i);
                const double x0 = fx(X.x), x1 = fx(X.y);
                const double B0 = fx(KB.x), B1 = fx(KB.y), A0 = fx(KA.x), A1 = fx(KA.y);
                double s00 = fpt::mm(x0, B0, __dmul_rn(B0, qinv), qd), s01 = fpt::mm(x1, B1, __dmul_rn(B1, qinv), qd);
                double s10 = fpt::mm(x0, A0, __dmul_rn(A0, qinv), qd), s11 = fpt::mm(x1, A1, __dmul_rn(A1, qinv), qd);
                if (nd > 0) {
                    const ulonglong2 p0 = acc0[i], p1 = acc1[i];
                    s00 = __dadd_rn(s00, FpA::D(p0.x));
                    s01 = __dadd_rn(s01, FpA::D(p0.y));
                    s10 = __dadd_rn(s10, FpA::D(p1.x));
                    s11 = __dadd_rn(s11, FpA::D(p1.y));
                }
                acc0[i] = make_ulonglong2(fp_canon4(s00, P.q, qd, qinv), fp_canon4(s01, P.q, qd, qinv));
                acc1[i] = make_ulonglong2(fp_canon4(s10, P.q, qd, qinv), fp_canon4(s11, P.q, qd, qinv));
            }
        }
        ksi_intt_rows<LOGN, A>(tab, f, e, pr, P, boff, c0, nc, a1off, ksi_sm);
        return;
    }
    // Q rows: the tensor (formed on the fly, tensor1_fp_raw) -- d2 with the own digit's key, [P] d0 / [P] d1
    const TensorSrc &T = f.ten;
    const bool lin = T.x.p != nullptr, lin2 = T.x2.p != nullptr, p2 = T.a2.p != nullptr;
    const u64 cc = lin ? T.C.c[e] : 0, c2 = lin2 ? T.C2.c[e] : 0;
    const u64 ccsh = lin ? T.C.csh[e] : 0, c2sh = lin2 ? T.C2.csh[e] : 0, br0 = tab.br0[pr], br1 = tab.br1[pr];
    const double PM = fx(f.pmod[e]), PMq = __dmul_rn(PM, qinv);
    const u64 *kb1 = keyrow + (long)(2 * jd) * nk * N, *ka1 = keyrow + (long)(2 * jd + 1) * nk * N;
    const long o = (long)e * N + boff;
#pragma unroll 1
    for (int i = threadIdx.x; i < CG * G; i += CT) {
        const double KBd = fx(__ldg(kb1 + i)), KAd = fx(__ldg(ka1 + i));
        const double KBq = __dmul_rn(KBd, qinv), KAq = __dmul_rn(KAd, qinv);
#pragma unroll 1
        for (int u = 0; u < nc; u++) {
            const int c = c0 + u;
            auto at = [&](const CRows &rr, int poly) { return rr.p[c * rr.cs + poly * rr.ps + o + i]; };
            const u64 x0 = lin ? at(T.x, 0) : 0, x1 = lin ? at(T.x, 1) : 0;
            const u64 y0 = lin2 ? at(T.x2, 0) : 0, y1 = lin2 ? at(T.x2, 1) : 0;
            const u64 u0 = p2 ? at(T.a2, 0) : 0, u1 = p2 ? at(T.a2, 1) : 0;
            const u64 w0 = p2 ? at(T.b2, 0) : 0, w1 = p2 ? at(T.b2, 1) : 0;
            if constexpr (IA) {
                u64 d0, d1, d2;
                tensor1(at(T.a, 0), at(T.a, 1), at(T.b, 0), at(T.b, 1), lin, x0, x1, cc, ccsh, lin2, y0, y1, c2, c2sh, P.q,
                        br0, br1, d0, d1, d2, p2, u0, u1, w0, w1);
                const u64 KBw = __ldg(kb1 + i), KAw = __ldg(ka1 + i), pm = f.pmod[e];
                U128 t0 = mul_wide(d2, KBw), t1 = mul_wide(d2, KAw);
                mac_wide(t0, d0, pm);
                mac_wide(t1, d1, pm);
                u64 *o0p = accb(u), *o1p = accb(u) + a1off;
                if (nd > 0) {
                    add_wide(t0, U128{o0p[i], 0});
                    add_wide(t1, U128{o1p[i], 0});
                }
                o0p[i] = barrett128(t0, P.q, br0, br1);
                o1p[i] = barrett128(t1, P.q, br0, br1);
                continue;
            }
            double e0, e1, e2;
            if (FB) {
                // ~50-bit rows: up to six raw products could pass 2^53, so the tensor is formed canonically (128-bit
                // MACs + Barrett, the integer kernels' arithmetic)
                u64 d0, d1, d2;
                tensor1(at(T.a, 0), at(T.a, 1), at(T.b, 0), at(T.b, 1), lin, x0, x1, cc, ccsh, lin2, y0, y1, c2, c2sh, P.q,
                        br0, br1, d0, d1, d2, p2, u0, u1, w0, w1);
                e0 = fx(d0);
                e1 = fx(d1);
                e2 = fx(d2);
            } else {
                tensor1_fp_raw(at(T.a, 0), at(T.a, 1), at(T.b, 0), at(T.b, 1), lin, x0, x1, cc, lin2, y0, y1, c2, qd, qinv,
                               e0, e1, e2, p2, u0, u1, w0, w1);
            }
            double s0 = __dadd_rn(fpt::mm(e2, KBd, KBq, qd), fpt::mm(e0, PM, PMq, qd));
            double s1 = __dadd_rn(fpt::mm(e2, KAd, KAq, qd), fpt::mm(e1, PM, PMq, qd));
            u64 *o0p = accb(u), *o1p = accb(u) + a1off;
            if (nd > 0) {
                s0 = __dadd_rn(s0, FpA::D(o0p[i]));
                s1 = __dadd_rn(s1, FpA::D(o1p[i]));
            }
            o0p[i] = fp_canon4(s0, P.q, qd, qinv);
            o1p[i] = fp_canon4(s1, P.q, qd, qinv);
        }
    }
    ksi_intt_rows<LOGN, A>(tab, f, e, pr, P, boff, c0, nc, a1off, ksi_sm);
}

// one launch per run of rows of one class (the ModUp digits of a level can mix the ~50-bit FpB rows with a 60-bit q_0,
// as the bootstrapping chains do): rows [f.e0, f.e1) of the level, each CTA with its class's policy
template <class A>
struct KsiMinB {
    static constexpr int v = NTT_KSI_MINB;
};
template <>
struct KsiMinB<IntA> {
    static constexpr int v = 2;  // 128-bit products and Barrett reductions: 80 registers spill
};
template <int LOGN, class A>
__global__ void __launch_bounds__(CT, KsiMinB<A>::v) ntt_ks_inner_kernel(Tab tab, KsFuse f) {
    ksi_body<LOGN, A>(tab, f);
}

// ---------------------------------------------------------------------------------------------
// single-pass cluster NTT (LOGN = 16): one thread-block cluster of CL CTAs per limb.  The limb is
// read from HBM once and written once; the transpose between the column stages and the row stages
// goes through distributed shared memory instead of a second HBM round trip.
//   forward: CTA j runs stages 0..S1-1 on columns [j CC, (j+1) CC) (loaded straight from HBM) and
//            parks them in its shared memory as [r][col]; after a cluster barrier it gathers rows
//            [j RR, (j+1) RR) from all CL CTAs (ld.shared::cluster), runs stages S1..LOGN-1 and
//            writes the rows with the contiguous pass's epilogue (rescale / ModDown fusions).
//   inverse: mirror image: rows first (prologue fusions: copy-in, tensor product), parked as
//            [r_local][col], columns gathered from all CTAs, GS stages S1-1..0, * N^{-1} (or k).
// Each CTA's buffer is read remotely only between the two cluster barriers; the second one is
// split (arrive after the gather, wait before the buffer is reused) so round 0 of the second half
// overlaps the other CTAs' gathers.
// ---------------------------------------------------------------------------------------------
#ifndef NTT_CLUSTER_CTAS
#define NTT_CLUSTER_CTAS 16  // CTAs per cluster (16 = non-portable maximum: 256-thread CTAs, 4 per SM)
#endif
constexpr int CL = NTT_CLUSTER_CTAS;
template <int LOGN>
struct ClusterCfg {
    static constexpr int S1 = LOGN / 2, S2 = LOGN - S1;
    static constexpr int G1 = 1 << S1, G2 = 1 << S2;  // column length, row length
    static constexpr int NCOL = G2, NROW = G1;
    static constexpr int CC = NCOL / CL, RR = NROW / CL;  // columns / rows per CTA
    static constexpr int THREADS = CC * (G1 / NV);
    static_assert(THREADS == RR * (G2 / NV), "cluster NTT: column and row halves need the same thread count");
    static constexpr int PITCH = G2 + G2 / 16;
    static constexpr int XW = (1 << LOGN) / CL;  // exchange block words
    static constexpr int SMEM_WORDS = XW > RR * PITCH ? XW : RR * PITCH;
};

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ u64 ld_dsmem(uint32_t a) {
    u64 v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

template <class A>
struct MinBC {
    static constexpr int v = 48 / CL;  // integer Shoup rows: ~80 registers
};
template <>
struct MinBC<FpA> {
    static constexpr int v = 64 / CL;  // FP rows: 64 registers
};

template <int LOGN, bool INV, int IN, int OUT, class A>
__global__ void __launch_bounds__(ClusterCfg<LOGN>::THREADS, MinBC<A>::v) ntt_cluster(PassArgs a) {
    using CF = ClusterCfg<LOGN>;
    constexpr int S1 = CF::S1, S2 = CF::S2, G2 = CF::G2, NCOL = CF::NCOL, CC = CF::CC, RR = CF::RR;
    constexpr int PITCH = CF::PITCH;
    constexpr long N = 1L << LOGN;
    constexpr int TPR = G2 / NV;
    extern __shared__ __align__(16) u64 xs[];
    const int rank = blockIdx.x;  // == %cluster_ctarank (cluster dims (CL,1,1), gridDim.x == CL)
    const int poly = a.poly0 + blockIdx.y / a.nsub, limb = a.limb0 + blockIdx.y % a.nsub;
    const int prime = prime_of(a.lm, limb);
    const PrimeC P = prime_consts(a.tab, prime);
    const u64 q = P.q;
    const ulonglong2 *tw = (INV ? a.tab.itw2 : a.tab.tw2) + prime * N;
    u64 *const limb_base = a.d.p + poly_off(a.d.cs, a.d.ps, poly) + limb * N;
    const uint32_t xs_local = smem_addr(xs);
    u64 v[NV];
    // row half: row gl of this CTA's RR rows, tau = thread within the row
    const int rgl = threadIdx.x / TPR, rtau = threadIdx.x % TPR;
    const int grow = rank * RR + rgl;  // global row (= contiguous block index)
    u64 *const smg = xs + rgl * PITCH;
    // column half: column ccl of this CTA's CC columns
    const int ccl = threadIdx.x % CC, ctau = threadIdx.x / CC;
    const int gcol = rank * CC + ccl;

    if (!INV) {
        using R = Rnd<S1, false>;
        static_assert(R::NR == 2, "cluster NTT: two rounds per half");
        constexpr int LO0 = R::lo(0), LO1 = R::lo(1);
        // ---- columns: stages 0..S1-1 ----
        u64 *cb = limb_base + gcol;
        if constexpr (IN == IN_BCAST) {
            const u64 *src = a.f.src.p + poly_off(a.f.src.cs, a.f.src.ps, poly) + gcol;
            const u64 ql = a.tab.q[a.f.lp], hl = ql >> 1, hi = a.f.half[limb], one_sh = a.tab.br1[prime];
#pragma unroll
            for (int k = 0; k < NV; k++) {
                const u64 r = csub(src[NCOL * held<LO0>(ctau, k)] + hl, ql);
                v[k] = A::in(submod(hi, mul_shoup(r, 1, one_sh, q), q), P);
            }
        } else {
#pragma unroll
            for (int k = 0; k < NV; k++) v[k] = A::in(cb[NCOL * held<LO0>(ctau, k)], P);
        }
        do_round<S1, false, 0, false, LOGN, A>(v, ctau, 0, tw, P);
#pragma unroll
        for (int k = 0; k < NV; k++) xs[held<LO0>(ctau, k) * CC + ccl] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = xs[held<LO1>(ctau, k) * CC + ccl];
        do_round<S1, false, 1, false, LOGN, A>(v, ctau, 0, tw, P);
        // park [r][col]: each thread rewrites exactly the words it read
#pragma unroll
        for (int k = 0; k < NV; k++) xs[held<LO1>(ctau, k) * CC + ccl] = v[k];
        cluster_arrive();
        cluster_wait();
        // ---- rows: stages S1..LOGN-1 on row grow ----
        using RB2 = Rnd<S2, false>;
        constexpr int RLO0 = RB2::lo(0), RLO1 = RB2::lo(1);
#pragma unroll
        for (int k = 0; k < NV; k++) {
            const int c = held<RLO0>(rtau, k);
            v[k] = ld_dsmem(mapa_rank(xs_local + 8u * (uint32_t)(grow * CC + (c % CC)), (uint32_t)(c / CC)));
        }
        cluster_arrive();
        do_round<S2, false, 0, true, LOGN, A>(v, rtau, grow, tw, P);
        cluster_wait();
#pragma unroll
        for (int k = 0; k < NV; k++) smg[padr(held<RLO0>(rtau, k))] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = smg[padr(held<RLO1>(rtau, k))];
        do_round<S2, false, 1, true, LOGN, A>(v, rtau, grow, tw, P);
#pragma unroll
        for (int k = 0; k < NV; k++) smg[padr(held<RLO1>(rtau, k))] = A::out_fwd(v[k], P);
        __syncthreads();
        // epilogue on 16-byte vectors over this CTA's RR contiguous rows
        const long boff = limb * N + (long)rank * RR * G2;
        const ulonglong2 *e1 = nullptr, *e2 = nullptr, *e3 = nullptr;
        ulonglong2 *dst;
        u64 kc = 0, kcsh = 0;
        if (OUT == OUT_PLAIN) {
            dst = reinterpret_cast<ulonglong2 *>(a.d.p + poly_off(a.d.cs, a.d.ps, poly) + boff);
        } else {
            e1 = reinterpret_cast<const ulonglong2 *>(a.f.e1.p + poly_off(a.f.e1.cs, a.f.e1.ps, poly) + boff);
            if (OUT == OUT_MODDOWN && (poly & 1) < a.f.e2_polys)
                e2 = reinterpret_cast<const ulonglong2 *>(a.f.e2.p + poly_off(a.f.e2.cs, a.f.e2.ps, poly) + boff);
            if (OUT == OUT_MODDOWN && a.f.e3.p)
                e3 = reinterpret_cast<const ulonglong2 *>(a.f.e3.p + poly_off(a.f.e3.cs, a.f.e3.ps, poly) + boff);
            dst = reinterpret_cast<ulonglong2 *>(a.f.out.p + poly_off(a.f.out.cs, a.f.out.ps, poly) + boff);
            kc = a.f.k[limb];
            kcsh = a.f.ksh[limb];
        }
#pragma unroll 4
        for (int i = threadIdx.x; i < RR * G2 / 2; i += CF::THREADS) {
            const int e = 2 * i, gg = e / G2, r = e % G2;
            u64 x0 = xs[gg * PITCH + padr(r)], x1 = xs[gg * PITCH + padr(r + 1)];
            if (OUT == OUT_RESCALE) {
                const ulonglong2 c = e1[i];
                x0 = mul_shoup(addmod(c.x, x0, q), kc, kcsh, q);
                x1 = mul_shoup(addmod(c.y, x1, q), kc, kcsh, q);
            } else if (OUT == OUT_MODDOWN) {
                const ulonglong2 c = e1[i];
                x0 = mul_shoup(submod(c.x, x0, q), kc, kcsh, q);
                x1 = mul_shoup(submod(c.y, x1, q), kc, kcsh, q);
                if (e2) {
                    const ulonglong2 d = e2[i];
                    x0 = addmod(x0, d.x, q);
                    x1 = addmod(x1, d.y, q);
                }
                if (e3) {
                    const ulonglong2 d = e3[i];
                    x0 = addmod(x0, d.x, q);
                    x1 = addmod(x1, d.y, q);
                }
            }
            dst[i] = make_ulonglong2(x0, x1);
        }
    } else {
        using RB2 = Rnd<S2, true>;
        static_assert(RB2::NR == 2, "cluster NTT: two rounds per half");
        constexpr int RLO0 = RB2::lo(0), RLO1 = RB2::lo(1);
        // ---- rows: GS stages LOGN-1..S1 on this CTA's RR rows (prologue fusions) ----
        const long boff = limb * N + (long)rank * RR * G2;
        const u64 *sp = (IN == IN_SRC || IN == IN_MUL || IN == IN_MUL2)
                            ? a.f.src.p + poly_off(a.f.src.cs, a.f.src.ps, poly) + boff
                            : limb_base + (long)rank * RR * G2;
        const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(sp);
        const ulonglong2 *src2 = nullptr, *src3 = nullptr, *src4 = nullptr;
        if (IN == IN_MUL || IN == IN_MUL2)
            src2 = reinterpret_cast<const ulonglong2 *>(a.f.src2.p + poly_off(a.f.src2.cs, a.f.src2.ps, poly) + boff);
        if (IN == IN_MUL2) {
            src3 = reinterpret_cast<const ulonglong2 *>(a.f.src3.p + poly_off(a.f.src3.cs, a.f.src3.ps, poly) + boff);
            src4 = reinterpret_cast<const ulonglong2 *>(a.f.src4.p + poly_off(a.f.src4.cs, a.f.src4.ps, poly) + boff);
        }
        const u64 br0 = a.tab.br0[prime], br1 = a.tab.br1[prime];
#pragma unroll 4
        for (int i = threadIdx.x; i < RR * G2 / 2; i += CF::THREADS) {
            ulonglong2 x = src[i];
            if (IN == IN_MUL) {
                const ulonglong2 y = src2[i];
                x.x = mulmod(x.x, y.x, q, br0, br1);
                x.y = mulmod(x.y, y.y, q, br0, br1);
            } else if (IN == IN_MUL2) {
                const ulonglong2 y = src2[i], z = src3[i], w = src4[i];
                U128 t0 = mul_wide(x.x, y.x), t1 = mul_wide(x.y, y.y);
                mac_wide(t0, z.x, w.x);
                mac_wide(t1, z.y, w.y);
                x.x = barrett128(t0, q, br0, br1);
                x.y = barrett128(t1, q, br0, br1);
            }
            const int e = 2 * i, gg = e / G2, r = e % G2;
            xs[gg * PITCH + padr(r)] = A::in(x.x, P);
            xs[gg * PITCH + padr(r + 1)] = A::in(x.y, P);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = smg[padr(held<RLO0>(rtau, k))];
        do_round<S2, true, 0, true, LOGN, A>(v, rtau, grow, tw, P);
#pragma unroll
        for (int k = 0; k < NV; k++) smg[padr(held<RLO0>(rtau, k))] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = smg[padr(held<RLO1>(rtau, k))];
        do_round<S2, true, 1, true, LOGN, A>(v, rtau, grow, tw, P);
        __syncthreads();  // the padded row layout is dead: park [r_local][col]
#pragma unroll
        for (int k = 0; k < NV; k++) xs[rgl * NCOL + held<RLO1>(rtau, k)] = v[k];
        cluster_arrive();
        cluster_wait();
        // ---- columns: GS stages S1-1..0 on column gcol ----
        using R = Rnd<S1, true>;
        constexpr int LO0 = R::lo(0), LO1 = R::lo(1);
#pragma unroll
        for (int k = 0; k < NV; k++) {
            const int r = held<LO0>(ctau, k);
            v[k] = ld_dsmem(mapa_rank(xs_local + 8u * (uint32_t)((r % RR) * NCOL + gcol), (uint32_t)(r / RR)));
        }
        cluster_arrive();
        do_round<S1, true, 0, false, LOGN, A>(v, ctau, 0, tw, P);
        cluster_wait();
#pragma unroll
        for (int k = 0; k < NV; k++) xs[held<LO0>(ctau, k) * CC + ccl] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < NV; k++) v[k] = xs[held<LO1>(ctau, k) * CC + ccl];
        do_round<S1, true, 1, false, LOGN, A>(v, ctau, 0, tw, P);
        const u64 ni = a.f.k ? a.f.k[limb] : a.tab.ninv[prime];
        const u64 nish = a.f.k ? a.f.ksh[limb] : a.tab.ninvsh[prime];
        u64 *cb = limb_base + gcol;
#pragma unroll
        for (int k = 0; k < NV; k++) cb[NCOL * held<LO1>(ctau, k)] = A::out_scaled(v[k], ni, nish, P);
    }
}

template <typename K>
void max_smem_carveout(K kern) {
    static bool done = false;  // per instantiation
    if (!done) {
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        done = true;
    }
}

// Programmatic dependent launch (NTT_PDL): the kernel may be scheduled while its predecessor on the
// stream drains; griddepcontrol.wait at its top blocks until the predecessor has completed and its
// writes are visible, so only the launch latency and CTA rasterisation overlap the predecessor's tail.
template <typename K>
void launch_pdl(K kern, dim3 grid, dim3 block, cudaStream_t st, const PassArgs &a) {
    if (!NTT_PDL) {
        kern<<<grid, block, 0, st>>>(a);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
}

// CTAs of a kernel resident at once on the device (occupancy x SMs), cached per kernel
template <typename K>
int resident_ctas(K kern, int threads) {
    static int v = 0;  // per instantiation
    if (!v) {
        int dev = 0, sms = 0, per = 0;
        CUDA_CHECK(cudaGetDevice(&dev));
        CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, 0));
        v = sms * std::max(per, 1);
    }
    return v;
}

template <int LOGN, bool INV, int IN, class A>
void launch_strided_a(const PassArgs &a0, int n_polys, cudaStream_t st) {
    constexpr int S = LOGN / 2;
    max_smem_carveout(ntt_strided<LOGN, INV, IN, A>);
    PassArgs a = a0;
    a.wave = resident_ctas(ntt_strided<LOGN, INV, IN, A>, SC * (1 << (S - RB)));
    dim3 grid((unsigned)((1L << (LOGN - S)) / SC), n_polys * a.nsub);
    launch_pdl(ntt_strided<LOGN, INV, IN, A>, grid, dim3(SC * (1 << (S - RB))), st, a);
}
template <int LOGN, bool INV, int IO, class A>
void launch_contig_a(const PassArgs &a0, int n_polys, cudaStream_t st) {
    using CF = ContigCfg<LOGN>;
    max_smem_carveout(ntt_contig<LOGN, INV, IO, A>);
    const PassArgs &a = a0;
    dim3 grid((unsigned)((1L << (LOGN - CF::S)) / CF::CG), n_polys * a.nsub);
    launch_pdl(ntt_contig<LOGN, INV, IO, A>, grid, dim3(CT), st, a);
}
// one launch per run of consecutive limbs of the same prime class: 0 exact FP64 (tab.fp_mask: q < 2^46, FpA),
// 1 exact FP64 with reductions (tab.fpb_mask: ~50-bit q, FpB), 2 integer Shoup (IntA)
enum { CLS_FPA = 0, CLS_FPB = 1, CLS_INT = 2 };
inline int prime_cls(const Tab &t, int p) {
    if (p < 64 && ((t.fp_mask >> p) & 1)) return CLS_FPA;
    if (p < 64 && ((t.fpb_mask >> p) & 1)) return CLS_FPB;
    return CLS_INT;
}
inline int limb_cls(const PassArgs &a, int limb) { return prime_cls(a.tab, prime_of(a.lm, limb)); }
// calls f(policy) with a value of the arithmetic policy of class cls
template <class F>
void with_policy(int cls, F f) {
    if (cls == CLS_FPA)
        f(FpA{});
    else if (cls == CLS_FPB)
        f(FpB{});
    else
        f(IntA{});
}
thread_local const NttProfHook *g_hook = nullptr;

// calls launch(a, cls) once per run of same-class limbs; `passes` = launches per limb transform that
// this call makes (2: one of the two passes, 1: single-pass cluster kernel) for the profiling hook (which
// sees the FP64 classes as one)
// operand limbs the fused modes of a launch read per limb on top of the transform's own input (prologue: the
// inverse's first pass; epilogue: the forward's last pass)
inline double prologue_limbs(const NttFusion &f) {
    if (f.in_mode == IN_MUL) return 1;
    if (f.in_mode == IN_MUL2) return 3;
    if (f.in_mode == IN_LIN) return f.lin == 2 ? 1 : 0;
    return 0;
}
inline double epilogue_limbs(const NttFusion &f) {
    if (f.out_mode == OUT_RESCALE) return 1 + (f.lin == 2 ? 1 : 0);
    if (f.out_mode == OUT_MODDOWN) return 1 + 0.5 * (f.e2.p ? f.e2_polys : 0) + (f.e3.p ? 1 : 0);
    return 0;
}
template <class F>
void for_runs(const PassArgs &a0, int n_polys, int passes, long N, F launch, double op_limbs = 0) {
    int l = 0;
    while (l < a0.lm.nl) {
        const int cls = limb_cls(a0, l);
        const bool fp = cls != CLS_INT;
        int e = l + 1;
        while (e < a0.lm.nl && limb_cls(a0, e) == cls) e++;
        PassArgs a = a0;
        a.limb0 = l;
        a.nsub = e - l;
        // per launch: its share of the limb transforms (a two-pass transform counts half in each pass)
        const double limbs = (double)n_polys * a.nsub / passes;
        const double bytes = 16.0 * limbs * (double)N;  // N words read + written once per transform
        const double opb = 8.0 * op_limbs * (double)n_polys * a.nsub * (double)N;
        if (g_hook) g_hook->mark(g_hook->ctx, 0, fp, bytes, limbs, opb);
        launch(a, cls);
        if (g_hook) g_hook->mark(g_hook->ctx, 1, fp, bytes, limbs, opb);
        l = e;
    }
}
template <int LOGN, bool INV, int IN>
void launch_strided(const PassArgs &a0, int n_polys, cudaStream_t st) {
    for_runs(a0, n_polys, 2, 1L << LOGN, [&](const PassArgs &a, int cls) {
        with_policy(cls, [&](auto pol) { launch_strided_a<LOGN, INV, IN, decltype(pol)>(a, n_polys, st); });
    });
}
template <int LOGN, bool INV, int IO>
void launch_contig(const PassArgs &a0, int n_polys, cudaStream_t st) {
    for_runs(
        a0, n_polys, 2, 1L << LOGN,
        [&](const PassArgs &a, int cls) {
            with_policy(cls, [&](auto pol) { launch_contig_a<LOGN, INV, IO, decltype(pol)>(a, n_polys, st); });
        },
        INV ? prologue_limbs(a0.f) : epilogue_limbs(a0.f));
}

template <int LOGN>
void run_chunk(const PassArgs &a, int rows, bool inverse, cudaStream_t st);

// (an L2-chunked variant -- both passes over ~56 MB of rows at a time so the intermediate is re-read
// from L2 -- was measured no faster and removed: profiles/r01_notes.md)
template <int LOGN>
void run(const PassArgs &a0, int n_polys, bool inverse, cudaStream_t st) {
    PassArgs a = a0;
    a.poly0 = 0;
    run_chunk<LOGN>(a, n_polys, inverse, st);
}

// Tab::ntt_cluster (SECPE_NTT_CLUSTER at context creation): 0 = two-pass everywhere (default; the FP rows
// are FP64-pipe bound and the cluster barriers cost more than the saved HBM pass), 1 = single-pass
// cluster kernel for FP rows, 2 = for every row
inline int cluster_mode(const PassArgs &a) { return a.tab.ntt_cluster; }

template <int LOGN, bool INV, int IN, int OUT, class A>
void launch_cluster_a(const PassArgs &a, int n_polys, cudaStream_t st) {
    using CF = ClusterCfg<LOGN>;
    auto kern = ntt_cluster<LOGN, INV, IN, OUT, A>;
    static bool done = false;  // per instantiation
    if (!done) {
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM_WORDS * 8));
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        if (CL > 8) CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        done = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CL, n_polys * a.nsub);
    cfg.blockDim = dim3(CF::THREADS);
    cfg.dynamicSmemBytes = CF::SMEM_WORDS * 8;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
}

template <int LOGN, bool INV, int IN, int OUT>
void launch_cluster_or_split(const PassArgs &a0, int n_polys, cudaStream_t st) {
    const int mode = cluster_mode(a0);
    for_runs(a0, n_polys, 1, 1L << LOGN, [&](const PassArgs &a, int cls) {
        if (cls == CLS_FPA && mode >= 1) {
            launch_cluster_a<LOGN, INV, IN, OUT, FpA>(a, n_polys, st);
        } else if (cls == CLS_INT && mode >= 2) {
            launch_cluster_a<LOGN, INV, IN, OUT, IntA>(a, n_polys, st);
        } else {
            with_policy(cls, [&](auto pol) {
                using A = decltype(pol);
                if (!INV) {
                    launch_strided_a<LOGN, false, IN, A>(a, n_polys, st);
                    launch_contig_a<LOGN, false, OUT, A>(a, n_polys, st);
                } else {
                    launch_contig_a<LOGN, true, IN, A>(a, n_polys, st);
                    launch_strided_a<LOGN, true, IN_PLAIN, A>(a, n_polys, st);
                }
            });
        }
        LAUNCH_CHECK();
    });
}

// the two-pass kernels on one run of same-class limbs (fallback of the fused kernel)
template <int LOGN, class A>
void two_pass_run_a(const PassArgs &a, int rows, bool inverse, cudaStream_t st) {
    const NttFusion &f = a.f;
    if (!inverse) {
        if (f.in_mode == IN_BCAST)
            launch_strided_a<LOGN, false, IN_BCAST, A>(a, rows, st);
        else
            launch_strided_a<LOGN, false, IN_PLAIN, A>(a, rows, st);
        LAUNCH_CHECK();
        if (f.out_mode == OUT_RESCALE)
            launch_contig_a<LOGN, false, OUT_RESCALE, A>(a, rows, st);
        else if (f.out_mode == OUT_MODDOWN)
            launch_contig_a<LOGN, false, OUT_MODDOWN, A>(a, rows, st);
        else
            launch_contig_a<LOGN, false, OUT_PLAIN, A>(a, rows, st);
    } else {
        if (f.in_mode == IN_SRC)
            launch_contig_a<LOGN, true, IN_SRC, A>(a, rows, st);
        else if (f.in_mode == IN_MUL)
            launch_contig_a<LOGN, true, IN_MUL, A>(a, rows, st);
        else if (f.in_mode == IN_MUL2)
            launch_contig_a<LOGN, true, IN_MUL2, A>(a, rows, st);
        else if (f.in_mode == IN_LIN)
            launch_contig_a<LOGN, true, IN_LIN, A>(a, rows, st);
        else
            launch_contig_a<LOGN, true, IN_PLAIN, A>(a, rows, st);
        LAUNCH_CHECK();
        launch_strided_a<LOGN, true, IN_PLAIN, A>(a, rows, st);
    }
    LAUNCH_CHECK();
}

template <int LOGN>
void run_chunk(const PassArgs &a, int rows, bool inverse, cudaStream_t st) {
    const NttFusion &f = a.f;
    if constexpr (LOGN == 16) {
        if (cluster_mode(a) == 0 && ntt_fused_enabled()) {
            // one persistent TMA-pipelined launch per run of exact-FP64 rows (ntt_fused.cu)
            for_runs(
                a, rows, 1, 1L << LOGN,
                [&](const PassArgs &r, int cls) {
                    if (ntt_fused_run(r.tab, LOGN, r.d, rows, r.lm, r.limb0, r.nsub, cls, inverse, r.f, st))
                        return;
                    with_policy(cls, [&](auto pol) { two_pass_run_a<LOGN, decltype(pol)>(r, rows, inverse, st); });
                },
                inverse ? prologue_limbs(f) : epilogue_limbs(f));
            return;
        }
        if (cluster_mode(a) > 0 && !f.lin) {  // (fused constant products: two-pass kernels only)
            if (!inverse) {
                const bool bc = f.in_mode == IN_BCAST;
                if (f.out_mode == OUT_RESCALE)
                    bc ? launch_cluster_or_split<LOGN, false, IN_BCAST, OUT_RESCALE>(a, rows, st)
                       : launch_cluster_or_split<LOGN, false, IN_PLAIN, OUT_RESCALE>(a, rows, st);
                else if (f.out_mode == OUT_MODDOWN)
                    bc ? launch_cluster_or_split<LOGN, false, IN_BCAST, OUT_MODDOWN>(a, rows, st)
                       : launch_cluster_or_split<LOGN, false, IN_PLAIN, OUT_MODDOWN>(a, rows, st);
                else
                    bc ? launch_cluster_or_split<LOGN, false, IN_BCAST, OUT_PLAIN>(a, rows, st)
                       : launch_cluster_or_split<LOGN, false, IN_PLAIN, OUT_PLAIN>(a, rows, st);
            } else {
                if (f.in_mode == IN_SRC)
                    launch_cluster_or_split<LOGN, true, IN_SRC, OUT_PLAIN>(a, rows, st);
                else if (f.in_mode == IN_MUL)
                    launch_cluster_or_split<LOGN, true, IN_MUL, OUT_PLAIN>(a, rows, st);
                else if (f.in_mode == IN_MUL2)
                    launch_cluster_or_split<LOGN, true, IN_MUL2, OUT_PLAIN>(a, rows, st);
                else if (f.in_mode == IN_LIN)
                    launch_cluster_or_split<LOGN, true, IN_LIN, OUT_PLAIN>(a, rows, st);
                else
                    launch_cluster_or_split<LOGN, true, IN_PLAIN, OUT_PLAIN>(a, rows, st);
            }
            return;
        }
    }
    if (!inverse) {
        if (f.in_mode == IN_BCAST)
            launch_strided<LOGN, false, IN_BCAST>(a, rows, st);
        else
            launch_strided<LOGN, false, IN_PLAIN>(a, rows, st);
        LAUNCH_CHECK();
        if (f.out_mode == OUT_RESCALE)
            launch_contig<LOGN, false, OUT_RESCALE>(a, rows, st);
        else if (f.out_mode == OUT_MODDOWN)
            launch_contig<LOGN, false, OUT_MODDOWN>(a, rows, st);
        else
            launch_contig<LOGN, false, OUT_PLAIN>(a, rows, st);
        LAUNCH_CHECK();
    } else {
        if (f.in_mode == IN_SRC)
            launch_contig<LOGN, true, IN_SRC>(a, rows, st);
        else if (f.in_mode == IN_MUL)
            launch_contig<LOGN, true, IN_MUL>(a, rows, st);
        else if (f.in_mode == IN_MUL2)
            launch_contig<LOGN, true, IN_MUL2>(a, rows, st);
        else if (f.in_mode == IN_LIN)
            launch_contig<LOGN, true, IN_LIN>(a, rows, st);
        else
            launch_contig<LOGN, true, IN_PLAIN>(a, rows, st);
        LAUNCH_CHECK();
        launch_strided<LOGN, true, IN_PLAIN>(a, rows, st);
        LAUNCH_CHECK();
    }
}

void dispatch(int logn, const PassArgs &a, int rows, bool inverse, cudaStream_t st) {
    switch (logn) {
        case 12: run<12>(a, rows, inverse, st); break;
        case 13: run<13>(a, rows, inverse, st); break;
        case 14: run<14>(a, rows, inverse, st); break;
        case 15: run<15>(a, rows, inverse, st); break;
        case 16: run<16>(a, rows, inverse, st); break;
        default: throw SecpeError{-1, "NTT: log N must be in [12, 16]"};
    }
}

}  // namespace

void ntt_set_prof_hook(const NttProfHook *h) { g_hook = h; }

namespace {
// several independent plain forward transforms in as few launches as possible (MAXSEG row ranges per
// launch, one launch pair per prime class)
template <int LOGN>
void run_segs(const Tab &tab, const NttSeg *segs, int nseg, bool inverse, cudaStream_t st, bool pass1_only = false) {
    struct Run {
        Seg g;
        int cls;
        int rows;
    };
    std::vector<Run> runs;
    for (int i = 0; i < nseg; i++) {
        const NttSeg &x = segs[i];
        if (x.n_polys <= 0 || x.lm.nl <= 0) continue;
        int l = 0;
        while (l < x.lm.nl) {
            const int cls = prime_cls(tab, prime_of(x.lm, l));
            int e = l + 1;
            while (e < x.lm.nl && prime_cls(tab, prime_of(x.lm, e)) == cls) e++;
            runs.push_back(Run{Seg{x.d, x.lm, l, e - l, 0}, cls, x.n_polys * (e - l)});
            l = e;
        }
    }
    constexpr long N = 1L << LOGN;
    for (int cls = 0; cls < 3; cls++) {
        const bool fp = cls != CLS_INT;
        PassArgs a{};
        a.tab = tab;
        a.nseg = 0;
        int rows = 0;
        auto flush = [&] {
            if (!a.nseg) return;
            a.nsub = rows;  // grid rows (n_polys = 1 below)
            const double bytes = 16.0 * rows * (double)N / 2;
            for (int pass = 0; pass < (pass1_only ? 1 : 2); pass++) {
                if (g_hook) g_hook->mark(g_hook->ctx, 0, fp, bytes, rows / 2.0, 0.0);
                const bool first = pass == 0;
                with_policy(cls, [&](auto pol) {
                    using A = decltype(pol);
                    if (!inverse) {
                        if (first)
                            launch_strided_a<LOGN, false, IN_PLAIN, A>(a, 1, st);
                        else
                            launch_contig_a<LOGN, false, OUT_PLAIN, A>(a, 1, st);
                    } else {
                        if (first)
                            launch_contig_a<LOGN, true, IN_PLAIN, A>(a, 1, st);
                        else
                            launch_strided_a<LOGN, true, IN_PLAIN, A>(a, 1, st);
                    }
                });
                LAUNCH_CHECK();
                if (g_hook) g_hook->mark(g_hook->ctx, 1, fp, bytes, rows / 2.0, 0.0);
            }
            a.nseg = 0;
            rows = 0;
        };
        for (auto &r : runs) {
            if (r.cls != cls) continue;
            if (a.nseg == MAXSEG) flush();
            r.g.row0 = rows;
            a.seg[a.nseg++] = r.g;
            rows += r.rows;
        }
        flush();
    }
}
}  // namespace

void ntt_segments(const Tab &tab, int logn, const NttSeg *segs, int nseg, bool inverse, cudaStream_t st) {
    switch (logn) {
        case 12: run_segs<12>(tab, segs, nseg, inverse, st); break;
        case 13: run_segs<13>(tab, segs, nseg, inverse, st); break;
        case 14: run_segs<14>(tab, segs, nseg, inverse, st); break;
        case 15: run_segs<15>(tab, segs, nseg, inverse, st); break;
        case 16: run_segs<16>(tab, segs, nseg, inverse, st); break;
        default: throw SecpeError{-1, "NTT: log N must be in [12, 16]"};
    }
}

void ntt_inverse_last_pass(const Tab &tab, int logn, RowsArg data, int n_polys, LimbMap lm, cudaStream_t st,
                           const NttFusion &f) {
    if (n_polys <= 0 || lm.nl <= 0) return;
    const PassArgs a{data, lm, tab, f, 0, lm.nl, 0};
    switch (logn) {
        case 12: launch_strided<12, true, IN_PLAIN>(a, n_polys, st); break;
        case 13: launch_strided<13, true, IN_PLAIN>(a, n_polys, st); break;
        case 14: launch_strided<14, true, IN_PLAIN>(a, n_polys, st); break;
        case 15: launch_strided<15, true, IN_PLAIN>(a, n_polys, st); break;
        case 16: launch_strided<16, true, IN_PLAIN>(a, n_polys, st); break;
        default: throw SecpeError{-1, "NTT: log N must be in [12, 16]"};
    }
    LAUNCH_CHECK();
}

void ntt_segments_pass1(const Tab &tab, int logn, const NttSeg *segs, int nseg, cudaStream_t st) {
    switch (logn) {
        case 12: run_segs<12>(tab, segs, nseg, false, st, true); break;
        case 13: run_segs<13>(tab, segs, nseg, false, st, true); break;
        case 14: run_segs<14>(tab, segs, nseg, false, st, true); break;
        case 15: run_segs<15>(tab, segs, nseg, false, st, true); break;
        case 16: run_segs<16>(tab, segs, nseg, false, st, true); break;
        default: throw SecpeError{-1, "NTT: log N must be in [12, 16]"};
    }
}

namespace {
template <int LOGN, class A>
void launch_ks_inner_a(const Tab &tab, const KsFuse &f, cudaStream_t st) {
    using CF = ContigCfg<LOGN>;
    const dim3 grid((unsigned)((1L << LOGN) / (CF::CG * CF::G)),
                    (unsigned)((f.e1 - f.e0) * ((f.n_ct + KSI_CPB - 1) / KSI_CPB)));
    auto kern = ntt_ks_inner_kernel<LOGN, A>;
    const int smem = KSI_CPB * CF::CG * CF::PITCH * 8;
    static bool done = false;
    if (!done) {
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        done = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(CT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = NTT_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, tab, f));
}
template <int LOGN>
void launch_ks_inner(const Tab &tab, const KsFuse &f0, cudaStream_t st) {
    // rows e of the level in order (Q rows 0..nl-1, then the special rows), split into runs of one prime class
    const int ne = f0.nl + f0.np;
    auto cls_of = [&](int e) {
        const int pr = e < f0.nl ? e : f0.nq_total + (e - f0.nl);
        return prime_cls(tab, pr);
    };
    int e0 = 0;
    while (e0 < ne) {
        const int cls = cls_of(e0);
        int e1 = e0 + 1;
        while (e1 < ne && cls_of(e1) == cls) e1++;
        KsFuse f = f0;
        f.e0 = e0;
        f.e1 = e1;
        if (cls == CLS_FPA)
            launch_ks_inner_a<LOGN, FpA>(tab, f, st);
        else if (cls == CLS_FPB)
            launch_ks_inner_a<LOGN, FpB>(tab, f, st);
        else
            launch_ks_inner_a<LOGN, IntA>(tab, f, st);
        e0 = e1;
    }
}
}  // namespace

void ntt_ks_inner(const Tab &tab, int logn, const KsFuse &f0, cudaStream_t st) {
    if (f0.n_ct <= 0) return;
    KsFuse f = f0;
    // profiling: the second half of every digit row's transform (8 N per limb) plus the operands the fused inner
    // product reads and writes (key once per batch, tensor inputs of the Q rows, the acc rows)
    const double N = (double)(1L << logn);
    const int ne = f.nl + f.np;
    double drows = 0;
    for (int e = 0; e < ne; e++) drows += e < f.nl ? f.beta - 1 : f.beta;
    drows *= f.n_ct;
    const TensorSrc &T = f.ten;
    const int tin = T.a.p ? 4 + (T.x.p ? 2 : 0) + (T.x2.p ? 2 : 0) + (T.a2.p ? 4 : 0) : 1;
    // the ModDown's INTT rows get the inverse's first pass here too: half a transform each, 2 polys per ciphertext
    if (f.intt_row0 >= 0) drows += 2.0 * f.n_ct * (ne - f.intt_row0);
    const double opb = 8.0 * N * (2.0 * f.beta * ne + (double)f.n_ct * (tin * f.nl + 2.0 * ne));
    if (g_hook) g_hook->mark(g_hook->ctx, 0, true, 8.0 * N * drows, drows / 2, opb);
    switch (logn) {
        case 12: launch_ks_inner<12>(tab, f, st); break;
        case 13: launch_ks_inner<13>(tab, f, st); break;
        case 14: launch_ks_inner<14>(tab, f, st); break;
        case 15: launch_ks_inner<15>(tab, f, st); break;
        case 16: launch_ks_inner<16>(tab, f, st); break;
        default: throw SecpeError{-1, "NTT: log N must be in [12, 16]"};
    }
    LAUNCH_CHECK();
    if (g_hook) g_hook->mark(g_hook->ctx, 1, true, 8.0 * N * drows, drows / 2, opb);
}

void ntt_forward(const Tab &tab, int logn, RowsArg data, int n_polys, LimbMap lm, cudaStream_t st,
                 const NttFusion &f) {
    if (n_polys <= 0 || lm.nl <= 0) return;
    if (f.in_mode != IN_PLAIN && f.in_mode != IN_BCAST) throw SecpeError{-1, "ntt_forward: bad input mode"};
    dispatch(logn, PassArgs{data, lm, tab, f, 0, lm.nl, 0}, n_polys, false, st);
}

void ntt_inverse(const Tab &tab, int logn, RowsArg data, int n_polys, LimbMap lm, cudaStream_t st,
                 const NttFusion &f) {
    if (n_polys <= 0 || lm.nl <= 0) return;
    if ((f.in_mode != IN_PLAIN && f.in_mode != IN_SRC && f.in_mode != IN_MUL && f.in_mode != IN_MUL2 &&
         f.in_mode != IN_LIN) ||
        f.out_mode != OUT_PLAIN)
        throw SecpeError{-1, "ntt_inverse: bad fusion mode"};
    dispatch(logn, PassArgs{data, lm, tab, f, 0, lm.nl, 0}, n_polys, true, st);
}
