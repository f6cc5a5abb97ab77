// bconv_tc.cu -- RNS fast base conversion on the 5th-generation tensor cores (tcgen05, kind::i8).
//
// A base conversion (ModUp R10, ModDown R11, and the fused ModDown + rescale of
// ev_mul_relin_rescale) is a dense contraction: for every coefficient m and target prime t,
//     z_t(m) = sum_s y_s(m) c_{s,t}  mod t          (y_s, c_{s,t} < 2^60, up to 12 sources s).
// Byte-slicing both operands turns it into an exact unsigned 8-bit GEMM:
//     y_s = sum_a y_{s,a} 256^a,   C'_{(s,a),t} = 256^a c_{s,t} mod t = sum_b C'_{(s,a),t,b} 256^b,
//     G_{t,b}(m) = sum_{(s,a)} y_{s,a}(m) C'_{(s,a),t,b}        (A: 128 x 96 u8, B: 96 x 8T u8, D: s32)
//     z_t(m) = (sum_b G_{t,b}(m) 256^b) mod t                   (< 2^80 before the Barrett reduction)
// G < 96 * 255 * 255 < 2^23, so the s32 accumulators never overflow and the result is exact.  One
// tcgen05.mma (M = 128, N = 8T <= 256, K = 32) per 32 bytes of K replaces the 4 quarter-rate
// IMAD.WIDE per source and target of the integer kernels; the epilogue (TMEM -> registers,
// 128-bit recombination, one Barrett per output) is what remains on the integer pipes.
//
// CTA: 512 threads.  Four threads per coefficient row stage the byte slices of 128 coefficients into shared memory
// in the canonical K-major no-swizzle UMMA layout (8 x 16-byte core matrices); one thread issues the
// MMAs and commits to an mbarrier; then warp w reads TMEM lanes 32 (w % 4) .. +31 and handles the
// targets t = w / 4, w / 4 + 4, ...  The B matrix of a conversion group is precomputed on the host
// (already in canonical layout) and copied to shared memory once per CTA.
#include "context.h"

#include <cstdlib>

namespace {

constexpr int TC_THREADS = 512;  // 16 warps: 4 groups of 4 warps share the targets in the epilogue
constexpr int TC_M = 128;
constexpr int TC_K = 96;               // bytes of K (12 sources x 8 bytes)
constexpr int LBO = 128;               // bytes between the two 16-byte K chunks of one MMA K-step
constexpr int SBO = (TC_K / 16) * 128; // bytes between consecutive 8-row groups
constexpr int TMEM_COLS = 256;

__host__ __device__ __forceinline__ int canon(int row, int k) {
    return ((row & 7) * 16) + (row >> 3) * SBO + (k >> 4) * LBO + (k & 15);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((LBO >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((SBO >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, legacy LBO mode, SWIZZLE_NONE
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr double TC_MAGIC = 6755399441055744.0;  // 1.5 2^52
constexpr double TC_TWO52 = 4503599627370496.0;

__global__ void __launch_bounds__(TC_THREADS) bconv_tc_kernel(TcArgs a) {
    extern __shared__ __align__(128) uint8_t tsm[];
    uint8_t *sA = tsm;                      // TC_M * TC_K
    uint8_t *sB = tsm + TC_M * TC_K;        // 8 * TC_TMAX * TC_K
    uint8_t *sR = sB + 8 * TC_TMAX * TC_K;  // TC_M * TC_K: the r source of the fused ModDown + rescale, zero elsewhere
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tslot;
    // per-target constants staged once per CTA: prime, output row offset, 1/q, [P]_{q_t} (+ Shoup)
    __shared__ u64 sq[TC_TMAX], spm[TC_TMAX], spmsh[TC_TMAX];
    __shared__ double sqinv[TC_TMAX];
    __shared__ long soff[TC_TMAX];
    // the same per-target constants packed for the 6-plane epilogue: {q, -q, 2^16/q, byte offset of the row}
    __shared__ __align__(16) ulonglong2 spk[TC_TMAX][2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int p = blockIdx.y;
    const TcGroup &G = a.groups[a.grouped ? p % a.pdiv : 0];
    const int nt = G.nt, ns = G.ns + (a.const1 ? 1 : 0);
    const int ncols = G.ncols, planes = G.planes;  // MMA N (multiple of 16), byte planes per target
    const int ksteps = (8 * ns + 31) / 32;
    const long N = 1L << a.logn;
    // fused ModDown + rescale with r as a third source: a second MMA adds r [P]_{q_i} once r is known, so every
    // target's epilogue is the plain conversion epilogue
    const bool rr2 = a.rr && G.rslot >= 0;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tslot)),
                     "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid < nt) {
        const u64 q = a.tab.q[G.prime[tid]];
        sq[tid] = q;
        sqinv[tid] = G.qinv[tid];
        spm[tid] = G.pmod[tid];
        spmsh[tid] = G.pmodsh[tid];
        soff[tid] = (long)G.out_row[tid] << a.logn;
        spk[tid][0] = make_ulonglong2(q, (u64)0 - q);
        spk[tid][1] = make_ulonglong2((u64)__double_as_longlong(G.qinv[tid] * 65536.0),
                                      (u64)(((long)G.out_row[tid] << a.logn) * 8));
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    {  // B (canonical, 8 ntp rows x TC_K bytes) and a zeroed A (the constant-1 source written once) and R
        const uint4 *gb = reinterpret_cast<const uint4 *>(G.B);
        uint4 *b4 = reinterpret_cast<uint4 *>(sB);
        for (int i = tid; i < ncols * TC_K / 16; i += TC_THREADS) b4[i] = gb[i];
        uint4 *a4 = reinterpret_cast<uint4 *>(sA);
        for (int i = tid; i < TC_M * TC_K / 16; i += TC_THREADS) a4[i] = make_uint4(0, 0, 0, 0);
        if (rr2) {
            uint4 *r4 = reinterpret_cast<uint4 *>(sR);
            for (int i = tid; i < TC_M * TC_K / 16; i += TC_THREADS) r4[i] = make_uint4(0, 0, 0, 0);
        }
    }
    __syncthreads();
    if (a.const1 && tid < TC_M) *reinterpret_cast<u64 *>(sA + canon(tid, 8 * G.ns)) = 1;
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tslot;
    const uint32_t idesc = (2u << 4) | ((uint32_t)(ncols >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
    const u64 *src = a.src + (long)(p / a.pdiv) * a.s_cs + (long)(p % a.pdiv) * a.s_ps + (long)G.src_row0 * N;
    u64 *dst = a.dst + (long)(p / a.pdiv) * a.d_cs + (long)(p % a.pdiv) * a.d_ps;
    const int lq = warp & 3, tpar = warp >> 2;  // TMEM lane quarter, target group (0..3)
    const int m = 32 * lq + lane;  // the coefficient (TMEM lane) this thread reads in the epilogue
    const int ntiles = (int)(N / TC_M);
    // staging: thread (row, half) holds sources s = half, half + 2, ... of coefficient row; the next
    // tile's values are loaded into registers before the current tile's epilogue
    const int srow = tid & (TC_M - 1), shalf = tid >> 7;  // 4 threads per coefficient row
    u64 pre[3], prexc = 0;
    // rr: the coefficient-form row x_l the prelude needs, fetched with the sources (warps 0-3: m == srow)
    const bool xc_here = a.rr && (!rr2 || tpar == 0);
    auto fetch = [&](int tile) {
        const long k0 = (long)tile * TC_M;
#pragma unroll
        for (int u = 0; u < 3; u++) {
            const int s = shalf + 4 * u;
            if (s < G.ns) pre[u] = src[(long)s * N + k0 + srow];
        }
        if (xc_here) prexc = src[(long)(-1) * N + k0 + m];
    };
    pdl_wait();  // TMEM, constants and the B matrix above do not depend on the previous kernel
    if ((int)blockIdx.x < ntiles) fetch(blockIdx.x);
    uint32_t phase = 0;  // mbarrier phase (one or two MMA commits per tile)
    auto mma_wait = [&]() {
        uint32_t done = 0;
        const uint32_t mb = smem_u32(&mbar);
        while (!done)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(done)
                : "r"(mb), "r"(phase));
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    };
    u64 rrv = 0;  // fused ModDown + rescale: r of this thread's coefficient
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long k0 = (long)tile * TC_M;
#pragma unroll
        for (int u = 0; u < 3; u++) {
            const int s = shalf + 4 * u;
            if (s < G.ns) *reinterpret_cast<u64 *>(sA + canon(srow, 8 * s)) = pre[u];
        }
        asm volatile("fence.proxy.async.shared::cta;\n");
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (tid == 0) {
            const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
            for (int s = 0; s < ksteps; s++) {
                const uint64_t da = smem_desc(a0 + s * 2 * LBO), db = smem_desc(b0 + s * 2 * LBO);
                const uint32_t acc = s > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(&mbar)));
        }
        mma_wait();
        const u64 xc = prexc;
        if (tile + (int)gridDim.x < ntiles) fetch(tile + gridDim.x);  // overlaps the epilogue below
        // epilogue: per target, the byte-plane sums G_b (< 96 * 255^2 < 2^23) -> V = sum_b G_b 256^b -> V mod t.
        const uint32_t lane_base = tmem + ((uint32_t)(32 * lq) << 16);
        auto v6 = [](const uint32_t *g) -> u64 {
            u64 v = (u64)g[0] + (u64)g[1] * 256u;
            v += (u64)g[2] * 65536u;
            v += (u64)g[3] * 16777216u;
            return v + ((u64)(g[4] + g[5] * 256u) << 32);
        };
        auto to_d = [](u64 x) -> double {  // exact for x < 2^52
            return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ULL)), TC_TWO52);
        };
        // V given as lo + hi 2^32 (hi < 2^32 for 6 planes, < 2^47 for 8), V mod 2^64 = vw.  6 planes: V < 2^64
        // and t > 2^40, so k < 2^24 (32-bit product); 8 planes: V < 2^79, k < 2^39 (64-bit product)
        auto reduce = [&](u64 lo, u64 hi, u64 vw, int t, bool wide) -> u64 {
            const u64 q = sq[t];
            const double vd = __fma_rn(to_d(hi), 4294967296.0, to_d(lo));
            const double kb = __fma_rn(vd, sqinv[t], TC_MAGIC);  // k + 1.5 2^52
            const u64 kq = wide ? ((u64)__double_as_longlong(kb) & ((1ULL << 51) - 1)) * q
                                : (u64)(uint32_t)__double_as_longlong(kb) * q;
            const long long r = (long long)(vw - kq);
            return (u64)(r + ((r >> 63) & (long long)q));
        };
        auto emit = [&](u64 z, int t) {
            if (a.rr && !rr2) z = addmod(z, csub(mul_shoup(rrv, spm[t], spmsh[t], sq[t]), sq[t]), sq[t]);
            dst[soff[t] + k0 + m] = z;
        };
        if (a.rr && xc_here) {
            // fused ModDown + rescale prelude (target 0 = q_l): Y_l = (xc - T_l) P^{-1}, r = [Y_l + floor(q_l/2)]
            const u64 ql = sq[0];
            uint32_t g[8];
            if (planes == 6) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]) : "r"(lane_base));
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n"
                             : "=r"(g[4]), "=r"(g[5]) : "r"(lane_base + 4));
            } else {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                             : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]),
                               "=r"(g[7])
                             : "r"(lane_base));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            u64 tl;
            if (planes == 6) {
                const u64 v = v6(g);
                tl = reduce(v & 0xFFFFFFFFULL, v >> 32, v, 0, false);
            } else {
                const u64 lo = (u64)g[0] + (u64)g[1] * 256u + (u64)g[2] * 65536u + (u64)g[3] * 16777216u;
                const u64 hi = (u64)g[4] + (u64)g[5] * 256u + (u64)g[6] * 65536u + (u64)g[7] * 16777216u;
                tl = reduce(lo, hi, lo + (hi << 32), 0, true);
            }
            rrv = csub(mul_shoup(submod(xc, tl, ql), a.pinv_l, a.pinv_l_sh, ql) + (ql >> 1), ql);
            if (rr2) *reinterpret_cast<u64 *>(sR + canon(m, 8 * G.rslot)) = rrv;
        }
        if (rr2) {
            // second MMA: the accumulators += r [P]_{q_i} (the K-step of sR holding r; its other bytes are zero)
            asm volatile("fence.proxy.async.shared::cta;\n");
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            if (tid == 0) {
                const int ks = (8 * G.rslot) / 32;
                const uint64_t da = smem_desc(smem_u32(sR) + ks * 2 * LBO), db = smem_desc(smem_u32(sB) + ks * 2 * LBO);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(1));
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&mbar)));
            }
            mma_wait();
        }
        const int t0 = a.rr ? 1 : 0;
        const int per = (nt - t0 + 3) >> 2;  // targets per warp group (contiguous)
        const int tb = t0 + tpar * per, te = min(nt, tb + per);
        if (planes == 6 && (!a.rr || rr2)) {
            // lean path: A = G0 + 256 G1, B = G2 + 256 G3, C = G4 + 256 G5 (each < 2^31), V = A + B 2^16 + C 2^32
            // (< 2^61: V < 96 * 255 t).  k = rint((V - A) / t) = rint((C 2^16 + B) * RN(2^16 / t)) from one FP64
            // product (A / t < 2^-13), so V - k t lies in (-t/2 - 1, t/2 + 2^32): one conditional add of t.  V - k t
            // is formed exactly mod 2^64 from the two 32-bit words of V and k (-t).
            uint8_t *const obase = reinterpret_cast<uint8_t *>(dst + k0 + m);
            auto lean = [&](const uint32_t *x, int t) {
                const ulonglong2 c0 = spk[t][0], c1 = spk[t][1];
                const uint32_t A = x[0] + (x[1] << 8), B = x[2] + (x[3] << 8), C = x[4] + (x[5] << 8);
                const double cb = __fma_rn(__dsub_rn(__hiloint2double(0x43300000, (int)C), TC_TWO52), 65536.0,
                                           __dsub_rn(__hiloint2double(0x43300000, (int)B), TC_TWO52));
                const uint32_t k =
                    (uint32_t)__double_as_longlong(__fma_rn(cb, __longlong_as_double((long long)c1.x), TC_MAGIC));
                uint32_t lo, hi;
                asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
                    : "=r"(lo), "=r"(hi)
                    : "r"(A), "r"(B << 16), "r"(C), "r"(B >> 16));
                u64 r = (((u64)hi << 32) | lo) + (u64)k * c0.y;
                asm("{\n\t.reg .pred p;\n\t.reg .u32 rl, rh, tl, th;\n\t"
                    "mov.b64 {rl, rh}, %0;\n\tmov.b64 {tl, th}, %1;\n\t"
                    "setp.lt.s32 p, rh, 0;\n\t"
                    "@p add.cc.u32 rl, rl, tl;\n\t@p addc.u32 rh, rh, th;\n\t"
                    "mov.b64 %0, {rl, rh};\n\t}"
                    : "+l"(r)
                    : "l"(c0.x));  // + t when negative (predicated, 3 instructions)
                *reinterpret_cast<u64 *>(obase + c1.y) = r;
            };
            for (int t = tb; t < te; t += 2) {
                uint32_t g[12];
                const uint32_t c = lane_base + (uint32_t)(6 * t);
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                             : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]),
                               "=r"(g[7])
                             : "r"(c));
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(g[8]), "=r"(g[9]), "=r"(g[10]), "=r"(g[11]) : "r"(c + 8));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                lean(g, t);
                if (t + 1 < te) lean(g + 6, t + 1);
            }
        } else if (planes == 6) {
            for (int t = tb; t < te; t += 2) {
                uint32_t g[12];
                const uint32_t c = lane_base + (uint32_t)(6 * t);
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                             : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]),
                               "=r"(g[7])
                             : "r"(c));
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                             : "=r"(g[8]), "=r"(g[9]), "=r"(g[10]), "=r"(g[11]) : "r"(c + 8));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                {
                    const u64 v = v6(g);
                    emit(reduce(v & 0xFFFFFFFFULL, v >> 32, v, t, false), t);
                }
                if (t + 1 < te) {
                    const u64 v = v6(g + 6);
                    emit(reduce(v & 0xFFFFFFFFULL, v >> 32, v, t + 1, false), t + 1);
                }
            }
        } else {
            for (int t = tb; t < te; t += 2) {
                uint32_t g[16];
                const uint32_t c = lane_base + (uint32_t)(8 * t);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                    "[%16];\n"
                    : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]), "=r"(g[7]),
                      "=r"(g[8]), "=r"(g[9]), "=r"(g[10]), "=r"(g[11]), "=r"(g[12]), "=r"(g[13]), "=r"(g[14]),
                      "=r"(g[15])
                    : "r"(c));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    if (h == 1 && t + 1 >= te) break;
                    const uint32_t *x = g + 8 * h;
                    const u64 lo = (u64)x[0] + (u64)x[1] * 256u + (u64)x[2] * 65536u + (u64)x[3] * 16777216u;
                    const u64 hi = (u64)x[4] + (u64)x[5] * 256u + (u64)x[6] * 65536u + (u64)x[7] * 16777216u;
                    emit(reduce(lo, hi, lo + (hi << 32), t + h, true), t + h);
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
}


// ---------------------------------------------------------------------------------------------
// Pipelined variant (default): one CTA per SM with warp roles, two A stages and two TMEM accumulators,
// so the staging of tile i + 1 and its MMAs overlap the epilogue of tile i (the round-1 kernel ran the
// phases of a tile one after another, separated by block barriers).
//   warps 0-3  : producers -- thread = coefficient row; load the row's sources of the tile, store them
//                into A[i % 2] (canonical K-major layout), arrive a_full[i % 2]
//   warp 4     : lane 0 issues the tile's MMAs into accumulator i % 2 and commits to acc_full[i % 2]
//   warps 5-28 : epilogue, six warps per TMEM lane quarter, each a contiguous block of targets; arrive
//                acc_empty[i % 2] when done with the accumulator
// Same integers as bconv_tc_kernel (the same GEMM and epilogue arithmetic).
// ---------------------------------------------------------------------------------------------
#ifndef TC2_EPI
#define TC2_EPI 24  // epilogue warps (a multiple of 4: TMEM lane quarters)
#endif
constexpr int TC2_PROD = 128, TC2_EPI_WARPS = TC2_EPI;
constexpr int TC2_THREADS = TC2_PROD + 32 + 32 * TC2_EPI_WARPS;  // 544
constexpr int TC2_TMEM_COLS = 512;                                // two accumulators of up to 256 columns

__device__ __forceinline__ void tc2_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tTC2W%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TC2W%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tc2_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(TC2_THREADS, 1) bconv_tc2_kernel(TcArgs a, int tiles_per_cta) {
    extern __shared__ __align__(128) uint8_t tsm[];
    uint8_t *sA0 = tsm;                        // 2 x TC_M * TC_K
    uint8_t *sB = tsm + 2 * TC_M * TC_K;       // 8 * TC_TMAX * TC_K
    __shared__ __align__(8) uint64_t a_full[2], acc_full[2], acc_empty[2];
    __shared__ uint32_t tslot;
    __shared__ u64 sq[TC_TMAX], spm[TC_TMAX], spmsh[TC_TMAX];
    __shared__ double sqinv[TC_TMAX];
    __shared__ long soff[TC_TMAX];
    __shared__ __align__(16) ulonglong2 spk[TC_TMAX][2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int p = blockIdx.y;
    const TcGroup &G = a.groups[a.grouped ? p % a.pdiv : 0];
    const int nt = G.nt, ns = G.ns;
    const int ncols = G.ncols, planes = G.planes;
    const int ksteps = (8 * (ns + (a.const1 ? 1 : 0)) + 31) / 32;
    const long N = 1L << a.logn;
    const int ntiles = (int)(N / TC_M);
    const int tile0 = blockIdx.x * tiles_per_cta;
    const int T = min(tiles_per_cta, ntiles - tile0);

    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tslot)),
                     "n"(TC2_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid < nt) {
        const u64 q = a.tab.q[G.prime[tid]];
        sq[tid] = q;
        sqinv[tid] = G.qinv[tid];
        spm[tid] = G.pmod[tid];
        spmsh[tid] = G.pmodsh[tid];
        soff[tid] = (long)G.out_row[tid] << a.logn;
        spk[tid][0] = make_ulonglong2(q, (u64)0 - q);
        spk[tid][1] = make_ulonglong2((u64)__double_as_longlong(G.qinv[tid] * 65536.0),
                                      (u64)(((long)G.out_row[tid] << a.logn) * 8));
    }
    if (tid == 0) {
        for (int b = 0; b < 2; b++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&a_full[b])), "r"(TC2_PROD));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&acc_full[b])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&acc_empty[b])),
                         "r"(TC2_EPI_WARPS));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    {  // B (canonical) and both A stages zeroed (the constant-1 source is written once)
        const uint4 *gb = reinterpret_cast<const uint4 *>(G.B);
        uint4 *b4 = reinterpret_cast<uint4 *>(sB);
        for (int i = tid; i < ncols * TC_K / 16; i += TC2_THREADS) b4[i] = gb[i];
        uint4 *a4 = reinterpret_cast<uint4 *>(sA0);
        for (int i = tid; i < 2 * TC_M * TC_K / 16; i += TC2_THREADS) a4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    if (a.const1 && tid < TC_M)
        for (int b = 0; b < 2; b++) *reinterpret_cast<u64 *>(sA0 + b * TC_M * TC_K + canon(tid, 8 * ns)) = 1;
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tslot;
    const u64 *src = a.src + (long)(p / a.pdiv) * a.s_cs + (long)(p % a.pdiv) * a.s_ps + (long)G.src_row0 * N;
    u64 *dst = a.dst + (long)(p / a.pdiv) * a.d_cs + (long)(p % a.pdiv) * a.d_ps;
    pdl_wait();  // TMEM, constants and B do not depend on the previous kernel; the sources do

    if (warp < 4) {
        // ---------------- producers ----------------
        const int row = tid;
        for (int i = 0; i < T; i++) {
            const int b = i & 1;
            const long k0 = (long)(tile0 + i) * TC_M;
            u64 v[12];
#pragma unroll
            for (int s = 0; s < 12; s++)
                if (s < ns) v[s] = src[(long)s * N + k0 + row];
            if (i >= 2) tc2_wait(&acc_full[b], ((i - 2) >> 1) & 1);  // MMAs of tile i - 2 have read A[b]
            uint8_t *sA = sA0 + b * TC_M * TC_K;
#pragma unroll
            for (int s = 0; s < 12; s++)
                if (s < ns) *reinterpret_cast<u64 *>(sA + canon(row, 8 * s)) = v[s];
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            tc2_arrive(&a_full[b]);
        }
    } else if (warp == 4) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            const uint32_t idesc = (2u << 4) | ((uint32_t)(ncols >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
            for (int i = 0; i < T; i++) {
                const int b = i & 1;
                tc2_wait(&a_full[b], (i >> 1) & 1);
                if (i >= 2) tc2_wait(&acc_empty[b], ((i - 2) >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint32_t a0 = smem_u32(sA0 + b * TC_M * TC_K), b0 = smem_u32(sB);
                const uint32_t acc = tmem + (uint32_t)(b * 256);
                for (int s = 0; s < ksteps; s++) {
                    const uint64_t da = smem_desc(a0 + s * 2 * LBO), db = smem_desc(b0 + s * 2 * LBO);
                    const uint32_t accum = s > 0;
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(acc),
                        "l"(da), "l"(db), "r"(idesc), "r"(accum));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                    smem_u32(&acc_full[b])));
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue ----------------
        const int ew = warp - 5;                // 0 .. TC2_EPI_WARPS - 1
        constexpr int TGS = TC2_EPI_WARPS / 4;  // warps per lane quarter
        const int lq = warp & 3, tg = ew / 4;   // TMEM lane quarter, target block (0 .. TGS - 1)
        const int m = 32 * lq + lane;
        const int t0 = a.rr ? 1 : 0;
        const int per = (nt - t0 + TGS - 1) / TGS;
        const int tb = t0 + tg * per, te = min(nt, tb + per);
        for (int i = 0; i < T; i++) {
            const int b = i & 1;
            const long k0 = (long)(tile0 + i) * TC_M;
            tc2_wait(&acc_full[b], (i >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t lane_base = tmem + (uint32_t)(b * 256) + ((uint32_t)(32 * lq) << 16);
            auto v6 = [](const uint32_t *g) -> u64 {
                u64 v = (u64)g[0] + (u64)g[1] * 256u;
                v += (u64)g[2] * 65536u;
                v += (u64)g[3] * 16777216u;
                return v + ((u64)(g[4] + g[5] * 256u) << 32);
            };
            auto to_d = [](u64 x) -> double {
                return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ULL)), 4503599627370496.0);
            };
            auto reduce = [&](u64 lo, u64 hi, u64 vw, int t, bool wide) -> u64 {
                const u64 q = sq[t];
                const double vd = __fma_rn(to_d(hi), 4294967296.0, to_d(lo));
                const double kb = __fma_rn(vd, sqinv[t], 6755399441055744.0);
                const u64 kq = wide ? ((u64)__double_as_longlong(kb) & ((1ULL << 51) - 1)) * q
                                    : (u64)(uint32_t)__double_as_longlong(kb) * q;
                const long long r = (long long)(vw - kq);
                return (u64)(r + ((r >> 63) & (long long)q));
            };
            u64 rrv = 0;
            if (a.rr) {
                const u64 ql = sq[0];
                uint32_t g[8];
                if (planes == 6) {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                                 : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]) : "r"(lane_base));
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n"
                                 : "=r"(g[4]), "=r"(g[5]) : "r"(lane_base + 4));
                } else {
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                                 : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]),
                                   "=r"(g[7])
                                 : "r"(lane_base));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                u64 tl;
                if (planes == 6) {
                    const u64 v = v6(g);
                    tl = reduce(v & 0xFFFFFFFFULL, v >> 32, v, 0, false);
                } else {
                    const u64 lo = (u64)g[0] + (u64)g[1] * 256u + (u64)g[2] * 65536u + (u64)g[3] * 16777216u;
                    const u64 hi = (u64)g[4] + (u64)g[5] * 256u + (u64)g[6] * 65536u + (u64)g[7] * 16777216u;
                    tl = reduce(lo, hi, lo + (hi << 32), 0, true);
                }
                const u64 xc = src[(long)(-1) * N + k0 + m];
                rrv = csub(mul_shoup(submod(xc, tl, ql), a.pinv_l, a.pinv_l_sh, ql) + (ql >> 1), ql);
            }
            auto emit = [&](u64 z, int t) {
                if (a.rr) z = addmod(z, csub(mul_shoup(rrv, spm[t], spmsh[t], sq[t]), sq[t]), sq[t]);
                dst[soff[t] + k0 + m] = z;
            };
            if (planes == 6 && !a.rr) {
                uint8_t *const obase = reinterpret_cast<uint8_t *>(dst + k0 + m);
                auto lean = [&](const uint32_t *x, int t) {  // bconv_tc_kernel's lean epilogue (same integers)
                    const ulonglong2 c0 = spk[t][0], c1 = spk[t][1];
                    const uint32_t A = x[0] + (x[1] << 8), B = x[2] + (x[3] << 8), C = x[4] + (x[5] << 8);
                    const double cb = __fma_rn(__dsub_rn(__hiloint2double(0x43300000, (int)C), TC_TWO52), 65536.0,
                                               __dsub_rn(__hiloint2double(0x43300000, (int)B), TC_TWO52));
                    const uint32_t k =
                        (uint32_t)__double_as_longlong(__fma_rn(cb, __longlong_as_double((long long)c1.x), TC_MAGIC));
                    uint32_t lo, hi;
                    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;"
                        : "=r"(lo), "=r"(hi)
                        : "r"(A), "r"(B << 16), "r"(C), "r"(B >> 16));
                    u64 r = (((u64)hi << 32) | lo) + (u64)k * c0.y;
                    asm("{\n\t.reg .pred p;\n\t.reg .u32 rl, rh, tl, th;\n\t"
                        "mov.b64 {rl, rh}, %0;\n\tmov.b64 {tl, th}, %1;\n\t"
                        "setp.lt.s32 p, rh, 0;\n\t"
                        "@p add.cc.u32 rl, rl, tl;\n\t@p addc.u32 rh, rh, th;\n\t"
                        "mov.b64 %0, {rl, rh};\n\t}"
                        : "+l"(r)
                        : "l"(c0.x));
                    *reinterpret_cast<u64 *>(obase + c1.y) = r;
                };
                for (int t = tb; t < te; t += 2) {
                    uint32_t g[12];
                    const uint32_t c = lane_base + (uint32_t)(6 * t);
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                                 : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]),
                                   "=r"(g[7])
                                 : "r"(c));
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                                 : "=r"(g[8]), "=r"(g[9]), "=r"(g[10]), "=r"(g[11]) : "r"(c + 8));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    lean(g, t);
                    if (t + 1 < te) lean(g + 6, t + 1);
                }
            } else if (planes == 6) {
                for (int t = tb; t < te; t += 2) {
                    uint32_t g[12];
                    const uint32_t c = lane_base + (uint32_t)(6 * t);
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                                 : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]),
                                   "=r"(g[7])
                                 : "r"(c));
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                                 : "=r"(g[8]), "=r"(g[9]), "=r"(g[10]), "=r"(g[11]) : "r"(c + 8));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    {
                        const u64 v = v6(g);
                        emit(reduce(v & 0xFFFFFFFFULL, v >> 32, v, t, false), t);
                    }
                    if (t + 1 < te) {
                        const u64 v = v6(g + 6);
                        emit(reduce(v & 0xFFFFFFFFULL, v >> 32, v, t + 1, false), t + 1);
                    }
                }
            } else {
                for (int t = tb; t < te; t += 2) {
                    uint32_t g[16];
                    const uint32_t c = lane_base + (uint32_t)(8 * t);
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                        "[%16];\n"
                        : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]), "=r"(g[7]),
                          "=r"(g[8]), "=r"(g[9]), "=r"(g[10]), "=r"(g[11]), "=r"(g[12]), "=r"(g[13]), "=r"(g[14]),
                          "=r"(g[15])
                        : "r"(c));
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        if (h == 1 && t + 1 >= te) break;
                        const uint32_t *x = g + 8 * h;
                        const u64 lo = (u64)x[0] + (u64)x[1] * 256u + (u64)x[2] * 65536u + (u64)x[3] * 16777216u;
                        const u64 hi = (u64)x[4] + (u64)x[5] * 256u + (u64)x[6] * 65536u + (u64)x[7] * 16777216u;
                        emit(reduce(lo, hi, lo + (hi << 32), t + h, true), t + h);
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncwarp();
            if (lane == 0) tc2_arrive(&acc_empty[b]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TC2_TMEM_COLS));
}

}  // namespace

// host: a conversion group's B matrix in canonical layout.  c[s][t] = the constant of source s for
// target t (mod prime t); rows 8 t + b, columns 8 s + a hold byte b of (c 256^a mod t).
std::vector<uint8_t> tc_bmatrix(const std::vector<std::vector<u64>> &c, const std::vector<u64> &tprimes, int planes,
                                int ncols) {
    const int ns = (int)c.size(), nt = (int)tprimes.size();
    std::vector<uint8_t> B((size_t)ncols * TC_K, 0);
    for (int t = 0; t < nt; t++) {
        const u64 q = tprimes[t];
        for (int s = 0; s < ns; s++) {
            u64 v = c[s][t] % q;
            for (int aa = 0; aa < 8; aa++) {
                for (int b = 0; b < planes; b++) B[canon(planes * t + b, 8 * s + aa)] = (uint8_t)(v >> (8 * b));
                v = h_mulmod(v, 256, q);
            }
        }
    }
    return B;
}

// dynamic shared memory per CTA: A + B need 36 KB; 80 KB caps residency at two CTAs per SM, which is
// what the 512 TMEM columns hold (256 each), so no CTA ever blocks in tcgen05.alloc
int tc_smem_bytes() { return 80 * 1024; }

void k_bconv_tc(const TcArgs &a, int n_polys, cudaStream_t st) {
    static int ver = -1, tpc2 = 0;
    if (ver < 0) {
        const char *e = getenv("SECPE_TC_V");  // development switch: 1 = the round-1 kernel layout
        ver = e ? atoi(e) : 1;  // the pipelined kernel measured slower in the step (profiles/r02_notes.md)
        const char *t = getenv("SECPE_TC2_TPC");
        tpc2 = t ? std::max(1, atoi(t)) : 16;
    }
    if (ver == 2 && !a.rr) {  // (the fused ModDown + rescale keeps the second-MMA kernel below)
        // 2 A stages (24 KB) + B (24 KB); > 114 KB requested so one CTA (512 TMEM columns) per SM
        constexpr int smem2 = 120 * 1024;
        static bool attr2 = false;
        if (!attr2) {
            CUDA_CHECK(cudaFuncSetAttribute(bconv_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
            attr2 = true;
        }
        const int ntiles = (int)((1L << a.logn) / TC_M);
        const dim3 grid((ntiles + tpc2 - 1) / tpc2, n_polys);
        launch_pdl_k(bconv_tc2_kernel, grid, dim3(TC2_THREADS), smem2, st, a, tpc2);
        LAUNCH_CHECK();
        return;
    }
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(bconv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes()));
        attr = true;
    }
    const int ntiles = (int)((1L << a.logn) / TC_M);
    static int tiles_per_cta = 0;
    if (!tiles_per_cta) {
        const char *e = getenv("SECPE_TC_TPC");  // development switch
        tiles_per_cta = e ? atoi(e) : 16;  // measured (round 2) 4: 78.6, 8: 77.6, 16: 77.6; (session 3) 4: 68.0,
                                           // 8: 66.8, 16: 66.5, 32: 66.5, 64: 69.5 ms per argmax step
        if (tiles_per_cta < 1) tiles_per_cta = 1;
    }
    const dim3 grid((ntiles + tiles_per_cta - 1) / tiles_per_cta, n_polys);
    launch_pdl_k(bconv_tc_kernel, grid, dim3(TC_THREADS), tc_smem_bytes(), st, a);
    LAUNCH_CHECK();
}
