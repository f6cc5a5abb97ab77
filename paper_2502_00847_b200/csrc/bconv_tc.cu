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

__global__ void __launch_bounds__(TC_THREADS) bconv_tc_kernel(TcArgs a) {
    extern __shared__ __align__(128) uint8_t tsm[];
    uint8_t *sA = tsm;                      // TC_M * TC_K
    uint8_t *sB = tsm + TC_M * TC_K;        // 8 * TC_TMAX * TC_K
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tslot;
    // per-target constants staged once per CTA: prime, output row offset, 1/q, [P]_{q_t} (+ Shoup)
    __shared__ u64 sq[TC_TMAX], spm[TC_TMAX], spmsh[TC_TMAX];
    __shared__ double sqinv[TC_TMAX];
    __shared__ long soff[TC_TMAX];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int p = blockIdx.y;
    const TcGroup &G = a.groups[a.grouped ? p % a.pdiv : 0];
    const int nt = G.nt, ns = G.ns + (a.const1 ? 1 : 0);
    const int ncols = G.ncols, planes = G.planes;  // MMA N (multiple of 16), byte planes per target
    const int ksteps = (8 * ns + 31) / 32;
    const long N = 1L << a.logn;

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
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    {  // B (canonical, 8 ntp rows x TC_K bytes) and a zeroed A (the constant-1 source written once)
        const uint4 *gb = reinterpret_cast<const uint4 *>(G.B);
        uint4 *b4 = reinterpret_cast<uint4 *>(sB);
        for (int i = tid; i < ncols * TC_K / 16; i += TC_THREADS) b4[i] = gb[i];
        uint4 *a4 = reinterpret_cast<uint4 *>(sA);
        for (int i = tid; i < TC_M * TC_K / 16; i += TC_THREADS) a4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    if (a.const1 && tid < TC_M) *reinterpret_cast<u64 *>(sA + canon(tid, 8 * G.ns)) = 1;
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
    u64 pre[3];
    auto fetch = [&](int tile) {
        const long k0 = (long)tile * TC_M;
#pragma unroll
        for (int u = 0; u < 3; u++) {
            const int s = shalf + 4 * u;
            if (s < G.ns) pre[u] = src[(long)s * N + k0 + srow];
        }
    };
    pdl_wait();  // TMEM, constants and the B matrix above do not depend on the previous kernel
    if ((int)blockIdx.x < ntiles) fetch(blockIdx.x);
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, it++) {
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
        {
            uint32_t done = 0;
            const uint32_t mb = smem_u32(&mbar), par = it & 1;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, p;\n\t}\n"
                    : "=r"(done)
                    : "r"(mb), "r"(par));
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (tile + (int)gridDim.x < ntiles) fetch(tile + gridDim.x);  // overlaps the epilogue below
        // epilogue: 8 int32 byte-plane sums per target -> value < 2^80 -> reduced with an FP64 quotient
        // V = lo + hi 2^32 with lo, hi < 2^48; k = floor(V / t) from doubles is off by at most one, so
        // r = V - k t (exact, mod 2^64) lies in [-t, 2t) and two corrections make it canonical.
        auto tld = [&](int t, uint32_t (&g)[8]) {
            const uint32_t lane_base = tmem + ((uint32_t)(32 * lq) << 16);
            if (planes == 8) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                             : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]),
                               "=r"(g[7])
                             : "r"(lane_base + (uint32_t)(8 * t)));
            } else {
                const uint32_t a6 = lane_base + (uint32_t)(6 * t);
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n"
                             : "=r"(g[0]), "=r"(g[1]) : "r"(a6));
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n"
                             : "=r"(g[2]), "=r"(g[3]) : "r"(a6 + 2));
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n"
                             : "=r"(g[4]), "=r"(g[5]) : "r"(a6 + 4));
                g[6] = g[7] = 0;
            }
        };
        auto tld_wait = [] { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); };
        // 6-plane epilogue (constants < 2^48): the same quotient reduction with the two zero planes
        // dropped (hi = G4 + G5 2^8 < 2^32 is a plain 32-bit value)
        auto reduce6 = [&](const uint32_t (&g)[8], int t) -> u64 {
            const u64 q = sq[t];
            const u64 lo = (u64)g[0] + ((u64)g[1] << 8) + ((u64)g[2] << 16) + ((u64)g[3] << 24);
            const uint32_t hi = g[4] + (g[5] << 8);
            const double two52 = 4503599627370496.0;
            const double lod = __dsub_rn(__longlong_as_double((long long)(lo | 0x4330000000000000ULL)), two52);
            const double hid = __dsub_rn(__hiloint2double(0x43300000, (int)hi), two52);
            const double vd = __fma_rn(hid, 4294967296.0, lod);
            const double kd = floor(__dmul_rn(vd, sqinv[t]));
            const u64 k = (u64)__double_as_longlong(__dadd_rn(kd, two52)) & ((1ULL << 52) - 1);
            long long r = (long long)(lo + ((u64)hi << 32) - k * q);
            if (r < 0) r += (long long)q;
            if ((u64)r >= q) r -= (long long)q;
            return (u64)r;
        };
        auto reduce_g = [&](const uint32_t (&g)[8], u64 q, double qinv) -> u64 {
            const u64 lo = (u64)g[0] + ((u64)g[1] << 8) + ((u64)g[2] << 16) + ((u64)g[3] << 24);
            const u64 hi = (u64)g[4] + ((u64)g[5] << 8) + ((u64)g[6] << 16) + ((u64)g[7] << 24);
            const double two52 = 4503599627370496.0;
            const double lod = __dsub_rn(__longlong_as_double((long long)(lo | 0x4330000000000000ULL)), two52);
            const double hid = __dsub_rn(__longlong_as_double((long long)(hi | 0x4330000000000000ULL)), two52);
            const double vd = __fma_rn(hid, 4294967296.0, lod);
            const double kd = floor(__dmul_rn(vd, qinv));
            const u64 k = (u64)__double_as_longlong(__dadd_rn(kd, two52)) & ((1ULL << 52) - 1);
            long long r = (long long)(lo + (hi << 32) - k * q);
            if (r < 0) r += (long long)q;
            if ((u64)r >= q) r -= (long long)q;
            return (u64)r;
        };
        int t0 = 0;
        u64 r = 0;
        if (a.rr) {
            // fused ModDown + rescale prelude (target 0 = q_l): Y_l = (xc - T_l) P^{-1}, r = [Y_l + floor(q_l/2)]
            const u64 ql = sq[0];
            uint32_t g[8];
            tld(0, g);
            tld_wait();
            const u64 tl = planes == 6 ? reduce6(g, 0) : reduce_g(g, ql, sqinv[0]);
            const u64 xc = src[(long)(-1) * N + k0 + m];
            r = csub(mul_shoup(submod(xc, tl, ql), a.pinv_l, a.pinv_l_sh, ql) + (ql >> 1), ql);
            t0 = 1;
        }
        // two targets per TMEM wait: both loads are in flight together
        for (int t = t0 + tpar; t < nt; t += 8) {
            const int t2 = t + 4;
            uint32_t g[8], h[8];
            tld(t, g);
            if (t2 < nt) tld(t2, h);
            tld_wait();
            {
                const u64 q = sq[t];
                u64 z = planes == 6 ? reduce6(g, t) : reduce_g(g, q, sqinv[t]);
                if (a.rr) z = addmod(z, csub(mul_shoup(r, spm[t], spmsh[t], q), q), q);
                dst[soff[t] + k0 + m] = z;
            }
            if (t2 < nt) {
                const u64 q = sq[t2];
                u64 z = planes == 6 ? reduce6(h, t2) : reduce_g(h, q, sqinv[t2]);
                if (a.rr) z = addmod(z, csub(mul_shoup(r, spm[t2], spmsh[t2], q), q), q);
                dst[soff[t2] + k0 + m] = z;
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
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
    static bool attr = false;
    if (!attr) {
        CUDA_CHECK(cudaFuncSetAttribute(bconv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes()));
        attr = true;
    }
    const int ntiles = (int)((1L << a.logn) / TC_M);
    static int tiles_per_cta = 0;
    if (!tiles_per_cta) {
        const char *e = getenv("SECPE_TC_TPC");  // development switch
        tiles_per_cta = e ? atoi(e) : 4;
        if (tiles_per_cta < 1) tiles_per_cta = 1;
    }
    const dim3 grid((ntiles + tiles_per_cta - 1) / tiles_per_cta, n_polys);
    launch_pdl_k(bconv_tc_kernel, grid, dim3(TC_THREADS), tc_smem_bytes(), st, a);
    LAUNCH_CHECK();
}
