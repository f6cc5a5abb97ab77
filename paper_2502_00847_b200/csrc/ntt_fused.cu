// ntt_fused.cu -- the N = 2^16 negacyclic NTT / INTT as ONE persistent, TMA-pipelined launch per call.
//
// Same transform, decomposition and butterfly arithmetic as the two-pass kernels of ntt.cu (R4; the
// limb viewed as a 256 x 256 matrix, stages 0..7 on columns, 8..15 on rows, radix-16 register rounds,
// ntt_core.cuh), so every output word is identical; what changes is the data movement:
//   * work items are 32 KB tiles: phase A (forward: 16 columns x 256 rows, inverse: 16 rows x 256) and
//     phase B (the other orientation) of every limb row of the call, 16 tiles per limb and phase;
//   * CTAs are persistent (2 per SM) and claim items in a fixed order from a global counter: phase-A
//     tiles of limb r + LAG are claimed right after the phase-B tiles of limb r, so the intermediate
//     (written by phase A, read by phase B) is re-read from L2 while it is hot -- HBM sees one read and
//     one write per limb instead of two of each (the two-pass design's 2.08 MB per limb);
//   * a phase-B tile of limb r waits on a per-limb counter that phase-A tiles of r release after their
//     TMA store has completed (the TMA reads and writes are performed in L2); items are claimed in order by running CTAs, so every item a
//     claimed item waits on is held by a running CTA (no deadlock, whatever else shares the GPU);
//   * warp-specialised CTA: warp 0 claims items and issues the TMA tensor loads (cp.async.bulk.tensor,
//     5-D maps over (element, line, limb, c0/c1, ciphertext)) into a 3-stage shared-memory ring with
//     mbarrier completion; warps 2..9 compute; warp 1 issues the TMA stores and releases the counters.
//     Row tiles use the 128-byte hardware swizzle, so both radix-16 round layouts read shared memory
//     conflict-free (16-byte vectors for the 16-consecutive-element layout);
//   * operands of the fused prologues / epilogues (tensor products, rescale / ModDown combinations)
//     are pulled into L2 by bulk prefetches issued with the tile's load;
//   * the counters clean themselves up (the last user of each resets it), so no memset precedes a launch
//     and the launch can be captured in a CUDA graph and replayed.
#include <cuda.h>

#include <map>
#include <mutex>

#include "ntt_core.cuh"

namespace {

constexpr int FL = 16;                 // log N of the fused kernel
constexpr long FN = 1L << FL;
constexpr int FS = 8;                  // stages per phase (256-point transforms)
constexpr int FT_CONS = 256;           // consumer threads per group (8 warps: one tile)
#ifndef FT_NGROUPS
#define FT_NGROUPS 2                   // consumer groups per CTA (one CTA per SM; 72 registers per thread)
#endif
#ifndef FT_NSTAGES
#define FT_NSTAGES 4                   // shared-memory ring: tile (32 KB) + its column twiddles (4 KB)
#endif
#ifndef FT_CLAIM
#define FT_CLAIM 1                     // items claimed per atomic
#endif
#ifndef FT_PEND
#define FT_PEND 2                      // store groups in flight before the storer completes the older half
#endif
constexpr int FT_NG = FT_NGROUPS;
// every stage is used by one consumer group only (iteration it -> stage it % FT_STAGES, group it % FT_NG):
// otherwise a group could reach a stage whose previous load (another group's, still in flight -- TMA loads
// complete out of order) is one phase behind and pass its parity wait early
static_assert(FT_NSTAGES % FT_NGROUPS == 0, "stages must be a multiple of the consumer groups");
constexpr int FT_THREADS = FT_NG * FT_CONS + 64;
constexpr int FT_STAGES = FT_NSTAGES;
constexpr int TILE_WORDS = 4096;       // 32 KB
constexpr int TILE_BYTES = TILE_WORDS * 8;
// column twiddles of a stage (stages 0..7 use table entries 1..255 only): the 256 {w, w/q} (FpA) or
// {w, w'} (IntA) pairs of the prime's pair table, copied with the tile
constexpr int TW_BYTES = 4096;
constexpr int STAGE_BYTES = TILE_BYTES + TW_BYTES;
constexpr int TILES_PER_LIMB = 16;
constexpr int FT_MAXROWS = 16384;      // limb rows per launch (larger calls are split)
#ifndef NTT_FUSED_LAG
#define NTT_FUSED_LAG 32               // limb rows between a limb's phase-A and phase-B tiles in claim order
#endif

struct FtSync {
    uint32_t work, exit;
    uint32_t pad[30];
    uint32_t flag[FT_MAXROWS];  // phase-A tiles done (0..16), then phase-B loads passed (16..32) -> reset
#ifdef FT_DEBUG_HANG
    int dbg[160][8];
#endif
};
#ifdef FT_DEBUG_HANG
#define DBG(i, v) (((volatile int *)sy->dbg[blockIdx.x])[i] = (v))
#else
#define DBG(i, v)
#endif

struct __align__(64) FtArgs {
    CUtensorMap a_in, a_out, b_in, b_out;
    Tab tab;
    NttFusion f;
    LimbMap lm;
    int limb0, nsub, rows, lag;
    long d_cs, d_ps;  // data rows (polynomial addressing of the fused operands)
    FtSync *sync;
};

// ---------------------------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *b, uint32_t parity);
#ifdef FT_DEBUG_HANG
__device__ __forceinline__ void mbar_wait_dbg(uint64_t *b, uint32_t parity, int role, int it) {
    long n = 0;
    while (!mbar_test(b, parity)) {
        if (++n == (1L << 26)) {
            printf("HANG block %d role %d it %d parity %u\n", blockIdx.x, role, it, parity);
            asm volatile("trap;");
        }
    }
}
#define MBAR_WAIT(b, p, role, it) mbar_wait_dbg(b, p, role, it)
#else
#define MBAR_WAIT(b, p, role, it) mbar_wait(b, p)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT%=;\n\t}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2,
                                         int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap *m, const void *src, int c0, int c1, int c2, int c3,
                                          int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(m)),
        "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
// the arithmetic policy A with its twiddles read as {w, w'} pairs from shared memory (column tiles)
template <class A>
struct SmemTw : A {
    static constexpr bool PAIRS = false;
    static __device__ __forceinline__ ulonglong2 twiddle(const ulonglong2 *tw, int i, const PrimeC &) {
        ulonglong2 w;
        asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(w.x), "=l"(w.y) : "r"(su32(tw + i)));
        return w;
    }
    static __device__ __forceinline__ void twiddle2(const ulonglong2 *, int, const PrimeC &, ulonglong2 &,
                                                    ulonglong2 &) {}
};
__device__ __forceinline__ void l2_prefetch(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// relaxed (not acquire) poll: an acquire load or a global proxy fence invalidates the SM's L1 (CCTL.IVALL),
// which would evict the consumers' twiddles; the data it guards is read by TMA from L2 only, after the loop
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release(uint32_t *p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// claim order: LAG phase-A limbs first, then (A of r + LAG, B of r) pairs, then the remaining B limbs
__device__ __forceinline__ void decode_item(int item, int rows, int lag, bool &phase_b, int &row, int &tile) {
    const int slot = item / TILES_PER_LIMB;
    tile = item % TILES_PER_LIMB;
    const int dm = lag < rows ? lag : rows, inter = rows - dm;
    if (slot < dm) {
        phase_b = false;
        row = slot;
        return;
    }
    const int q = slot - dm;
    if (q < 2 * inter) {
        phase_b = q & 1;
        row = phase_b ? q >> 1 : dm + (q >> 1);
    } else {
        phase_b = true;
        row = inter + (q - 2 * inter);
    }
}

// swizzled (128-byte TMA swizzle) byte offset of element e of row gl in a row tile (16 rows x 256)
__device__ __forceinline__ uint32_t swz(int gl, int e) {
    const int L = gl * 16 + (e >> 4);
    return (uint32_t)(L * 128 + ((((e & 15) >> 1) ^ (L & 7)) << 4) + ((e & 1) << 3));
}

template <class A, bool INV, int IN, int OUT>
__global__ void __launch_bounds__(FT_THREADS, 1) ntt_fused_kernel(const __grid_constant__ FtArgs a) {
    extern __shared__ uint8_t fsm_raw[];
    // 1024-byte alignment (128-byte swizzle), by pointer arithmetic so the compiler keeps shared-space accesses
    uint8_t *fsm = fsm_raw + ((1024 - (su32(fsm_raw) & 1023)) & 1023);
    __shared__ __align__(8) uint64_t full[FT_STAGES], computed[FT_STAGES], empty_[FT_STAGES];
    __shared__ int items[FT_STAGES];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < FT_STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&computed[s], FT_CONS);  // one consumer group per item
            mbar_init(&empty_[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    FtSync *sy = a.sync;
    const int total = a.rows * 2 * TILES_PER_LIMB;

    if (warp == 0) {
        // ---------------- producer: claim, wait for dependencies, TMA load ----------------
        if (lane == 0) {
            // items are claimed FT_CLAIM at a time (contiguous ranges keep the claim order deadlock-free: a
            // blocked item only waits on smaller items, the smallest unfinished one is always being worked on),
            // and the next range is claimed one range ahead so the atomic's latency is off the critical path
            int next = (int)atomicAdd(&sy->work, (unsigned)FT_CLAIM), cur = 0, left = 0;
            for (int it = 0;; it++) {
                const int s = it % FT_STAGES;
                if (it >= FT_STAGES) MBAR_WAIT(&empty_[s], ((it / FT_STAGES) - 1) & 1, 0, it);
                if (left == 0) {
                    cur = next;
                    left = FT_CLAIM;
                    if (cur < total) next = (int)atomicAdd(&sy->work, (unsigned)FT_CLAIM);
                }
                const int item = cur++;
                left--;
                DBG(0, it);
                DBG(1, item);
                DBG(2, next);
                if (item >= total) {
                    // one end marker per consumer group (groups take iterations round-robin)
                    for (int j = 0; j < FT_NG; j++) {
                        const int sj = (it + j) % FT_STAGES;
                        if (j > 0 && it + j >= FT_STAGES) mbar_wait(&empty_[sj], (((it + j) / FT_STAGES) - 1) & 1);
                        items[sj] = -1;
                        mbar_arrive(&full[sj]);
                    }
                    break;
                }
                bool pb;
                int row, tile;
                decode_item(item, a.rows, a.lag, pb, row, tile);
                const int poly = row / a.nsub, limb = row % a.nsub;
                if (pb) {
                    uint32_t *fl = &sy->flag[row];
#ifdef FT_DEBUG_HANG
                    long nspin = 0;
                    while (ld_relaxed(fl) < TILES_PER_LIMB) {
                        if (++nspin == (1L << 22)) {
                            printf("HANG flag block %d it %d item %d row %d flag %u\n", blockIdx.x, it, item, row, ld_relaxed(fl));
                            for (int b = 0; b < (int)gridDim.x; b++) {
                                volatile int *d = sy->dbg[b];
                                printf("  blk %d prod it %d item %d next %d | stor it %d item %d np %d | grp %d\n", b, d[0],
                                       d[1], d[2], d[3], d[4], d[5], d[6]);
                            }
                            asm volatile("trap;");
                        }
                        __nanosleep(64);
                    }
#else
                    while (ld_relaxed(fl) < TILES_PER_LIMB) __nanosleep(64);
#endif
                    if (atomicAdd(fl, 1u) == 2 * TILES_PER_LIMB - 1) *fl = 0;  // last phase-B claim resets it
                }
                items[s] = item;
                uint8_t *dst = fsm + (size_t)s * STAGE_BYTES;
                const bool col = INV == pb;  // forward: A = columns; inverse: B = columns
                const int c0 = col ? tile * 16 : 0, c1 = col ? 0 : tile * 256;
                const bool bcast = !pb && IN == IN_BCAST;
                if (col) {
                    // the 255 twiddles of stages 0..7 (table entries 1..255) with the tile
                    const int prime = prime_of(a.lm, a.limb0 + limb);
                    const ulonglong2 *tw = (INV ? a.tab.itwp : a.tab.twp) + (long)prime * FN;
                    mbar_arrive_tx(&full[s], TILE_BYTES + TW_BYTES);
                    bulk_load(dst + TILE_BYTES, tw, TW_BYTES, &full[s]);
                } else {
                    mbar_arrive_tx(&full[s], TILE_BYTES);
                }
                tma_load(dst, pb ? &a.b_in : &a.a_in, &full[s], c0, c1, bcast ? 0 : limb, poly & 1, poly >> 1);
                // operands of the fused prologue (inverse phase A) / epilogue (forward phase B): into L2 now
                const long toff = (long)(a.limb0 + limb) * FN + (long)tile * TILE_WORDS;
                if (!INV && pb && OUT != OUT_PLAIN) {
                    const NttFusion &f = a.f;
                    l2_prefetch(f.e1.p + poly_off(f.e1.cs, f.e1.ps, poly) + toff, TILE_BYTES);
                    if (OUT == OUT_RESCALE && f.lin == 2)
                        l2_prefetch(f.e1b.p + poly_off(f.e1b.cs, f.e1b.ps, poly) + toff, TILE_BYTES);
                    if (OUT == OUT_MODDOWN && (poly & 1) < f.e2_polys)
                        l2_prefetch(f.e2.p + poly_off(f.e2.cs, f.e2.ps, poly) + toff, TILE_BYTES);
                    if (OUT == OUT_MODDOWN && f.e3.p) l2_prefetch(f.e3.p + poly_off(f.e3.cs, f.e3.ps, poly) + toff, TILE_BYTES);
                }
                if (INV && !pb && (IN == IN_MUL || IN == IN_MUL2 || (IN == IN_LIN && a.f.lin == 2))) {
                    const NttFusion &f = a.f;
                    l2_prefetch(f.src2.p + poly_off(f.src2.cs, f.src2.ps, poly) + toff, TILE_BYTES);
                    if (IN == IN_MUL2) {
                        l2_prefetch(f.src3.p + poly_off(f.src3.cs, f.src3.ps, poly) + toff, TILE_BYTES);
                        l2_prefetch(f.src4.p + poly_off(f.src4.cs, f.src4.ps, poly) + toff, TILE_BYTES);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- storer: TMA store, free the stage, release the per-limb counters ----------------
        // A stage is freed as soon as the store has READ it; the phase-A counters are released once the
        // writes are complete, which is checked lazily (wait_group on all but the newest groups) so the
        // storer never blocks on a write round trip; before it would idle, it completes and releases all
        if (lane == 0) {
            constexpr int PEND = FT_PEND;
            int prow[PEND];  // phase-A rows of the pending (uncompleted) store groups, oldest first; -1: phase B
            int np = 0;
            auto release_all = [&]() {
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                for (int i = 0; i < np; i++)
                    if (prow[i] >= 0) red_release(&sy->flag[prow[i]], 1u);
                np = 0;
            };
            for (int it = 0;; it++) {
                const int s = it % FT_STAGES;
                const uint32_t par = (it / FT_STAGES) & 1;
                if (np > 0 && !mbar_test(&computed[s], par)) release_all();
                MBAR_WAIT(&computed[s], par, 1, it);
                const int item = items[s];
                DBG(3, it);
                DBG(4, item);
                DBG(5, np);
                if (item < 0) break;
                bool pb;
                int row, tile;
                decode_item(item, a.rows, a.lag, pb, row, tile);
                const int poly = row / a.nsub, limb = row % a.nsub;
                const bool col = INV == pb;
                const int c0 = col ? tile * 16 : 0, c1 = col ? 0 : tile * 256;
                tma_store(pb ? &a.b_out : &a.a_out, fsm + (size_t)s * STAGE_BYTES, c0, c1, limb, poly & 1, poly >> 1);
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                mbar_arrive(&empty_[s]);
                if (np == PEND) {
                    // the oldest half is complete once at most PEND / 2 newer groups are pending
                    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(PEND / 2) : "memory");
                    for (int i = 0; i < PEND / 2; i++)
                        if (prow[i] >= 0) red_release(&sy->flag[prow[i]], 1u);
                    for (int i = PEND / 2; i < PEND; i++) prow[i - PEND / 2] = prow[i];
                    np = PEND / 2;
                }
                prow[np++] = pb ? -1 : row;
            }
            release_all();
        }
    } else {
        // ---------------- consumers: two radix-16 rounds per tile ----------------
        const int grp = (tid - 64) / FT_CONS, ct = (tid - 64) % FT_CONS;
        const int bar = 1 + grp;                // the group's named barrier
        const int tau = ct >> 4, cl = ct & 15;  // column tiles: row group tau, column cl
        const int gl = ct >> 4, rt = ct & 15;   // row tiles: row gl of the tile, thread rt within the row
        for (int it = grp;; it += FT_NG) {
            const int s = it % FT_STAGES;
            if (ct == 0) DBG(6, it);
            MBAR_WAIT(&full[s], (it / FT_STAGES) & 1, 2, it);
            const int item = items[s];
            if (item < 0) {
                mbar_arrive(&computed[s]);
                break;
            }
            bool pb;
            int row, tile;
            decode_item(item, a.rows, a.lag, pb, row, tile);
            const int poly = row / a.nsub, limb = a.limb0 + row % a.nsub;
            const int prime = prime_of(a.lm, limb);
            const PrimeC P = prime_consts(a.tab, prime);
            const u64 q = P.q;
            // row-tile twiddles: FpA dense doubles (w/q formed by one DMUL; a 16-byte {w, w/q} pair table
            // doubles the L2 traffic of these loads and measured 20 % slower), IntA {w, w'} pairs
            const ulonglong2 *tw = (INV ? a.tab.itw2 : a.tab.tw2) + (long)prime * FN;
            uint8_t *t8 = fsm + (size_t)s * STAGE_BYTES;
            u64 *tc = reinterpret_cast<u64 *>(t8);
            const long toff = (long)limb * FN + (long)tile * TILE_WORDS;  // tile offset inside the polynomial
            u64 v[NV];
            const bool col = INV == pb;
#ifdef FT_NOCOMPUTE
            if (true) {
            } else
#endif
            if (col) {
                // ---- column tile: element (r, cl) at tc[r * 16 + cl] ----
                using R = Rnd<FS, INV>;
                constexpr int LO0 = R::lo(0), LO1 = R::lo(1);
                const ulonglong2 *ctw = reinterpret_cast<const ulonglong2 *>(t8 + TILE_BYTES);

                if (!INV && IN == IN_BCAST) {
                    // rescale broadcast (R12): [floor(q_l/2)]_{q_i} - [[x + floor(q_l/2)]_{q_l}]_{q_i}
                    const u64 ql = a.tab.q[a.f.lp], hl = ql >> 1, hi = a.f.half[limb], one_sh = a.tab.br1[prime];
#pragma unroll
                    for (int k = 0; k < NV; k++) {
                        const u64 r = csub(tc[held<LO0>(tau, k) * 16 + cl] + hl, ql);
                        v[k] = A::in(submod(hi, mul_shoup(r, 1, one_sh, q), q), P);
                    }
                } else if (!INV) {
#pragma unroll
                    for (int k = 0; k < NV; k++) v[k] = A::in(tc[held<LO0>(tau, k) * 16 + cl], P);
                } else {
#pragma unroll
                    for (int k = 0; k < NV; k++) v[k] = tc[held<LO0>(tau, k) * 16 + cl];
                }
                do_round<FS, INV, 0, false, FL, SmemTw<A>>(v, tau, 0, ctw, P);
#pragma unroll
                for (int k = 0; k < NV; k++) tc[held<LO0>(tau, k) * 16 + cl] = v[k];
                named_sync(bar, FT_CONS);
#pragma unroll
                for (int k = 0; k < NV; k++) v[k] = tc[held<LO1>(tau, k) * 16 + cl];
                do_round<FS, INV, 1, false, FL, SmemTw<A>>(v, tau, 0, ctw, P);
                if (INV) {
                    const u64 ni = a.f.k ? a.f.k[limb] : a.tab.ninv[prime];
                    const u64 nish = a.f.k ? a.f.ksh[limb] : a.tab.ninvsh[prime];
#pragma unroll
                    for (int k = 0; k < NV; k++) v[k] = A::out_scaled(v[k], ni, nish, P);
                }
#pragma unroll
                for (int k = 0; k < NV; k++) tc[held<LO1>(tau, k) * 16 + cl] = v[k];
            } else {
                // ---- row tile (swizzled): element e of row gl at byte swz(gl, e) ----
                using R = Rnd<FS, INV>;
                constexpr int LO0 = R::lo(0), LO1 = R::lo(1);
                static_assert(INV ? (LO0 == 0 && LO1 == 4) : (LO0 == 4 && LO1 == 0), "row tile layouts");
                const int g = tile * 16 + gl;  // row of the 256 x 256 matrix
                if (INV && (IN == IN_MUL || IN == IN_MUL2 || IN == IN_LIN)) {
                    // fused prologue on 16-byte vectors: vector i = elements 2i, 2i + 1 of the tile
                    const NttFusion &f = a.f;
                    const u64 br0 = a.tab.br0[prime], br1 = a.tab.br1[prime];
                    const u64 lc1 = IN == IN_LIN ? smod_dev(f.C1, q, br0, br1) : 0;
                    const u64 lc2 = IN == IN_LIN && f.lin == 2 ? smod_dev(f.C2, q, br0, br1) : 0;
                    const ulonglong2 *s2 = nullptr, *s3 = nullptr, *s4 = nullptr;
                    if (IN == IN_MUL || IN == IN_MUL2 || (IN == IN_LIN && f.lin == 2))
                        s2 = reinterpret_cast<const ulonglong2 *>(f.src2.p + poly_off(f.src2.cs, f.src2.ps, poly) + toff);
                    if (IN == IN_MUL2) {
                        s3 = reinterpret_cast<const ulonglong2 *>(f.src3.p + poly_off(f.src3.cs, f.src3.ps, poly) + toff);
                        s4 = reinterpret_cast<const ulonglong2 *>(f.src4.p + poly_off(f.src4.cs, f.src4.ps, poly) + toff);
                    }
#pragma unroll 4
                    for (int i = ct; i < TILE_WORDS / 2; i += FT_CONS) {
                        const int e = 2 * i;
                        ulonglong2 *sp = reinterpret_cast<ulonglong2 *>(t8 + swz(e >> 8, e & 255));
                        ulonglong2 x = *sp;
                        if (IN == IN_LIN) {
                            U128 t0 = mul_wide(x.x, lc1), t1 = mul_wide(x.y, lc1);
                            if (s2) {
                                const ulonglong2 y = s2[i];
                                mac_wide(t0, y.x, lc2);
                                mac_wide(t1, y.y, lc2);
                            }
                            x.x = barrett128(t0, q, br0, br1);
                            x.y = barrett128(t1, q, br0, br1);
                        } else if (IN == IN_MUL) {
                            const ulonglong2 y = s2[i];
                            x.x = mulmod(x.x, y.x, q, br0, br1);
                            x.y = mulmod(x.y, y.y, q, br0, br1);
                        } else {
                            const ulonglong2 y = s2[i], z = s3[i], w = s4[i];
                            U128 t0 = mul_wide(x.x, y.x), t1 = mul_wide(x.y, y.y);
                            mac_wide(t0, z.x, w.x);
                            mac_wide(t1, z.y, w.y);
                            x.x = barrett128(t0, q, br0, br1);
                            x.y = barrett128(t1, q, br0, br1);
                        }
                        *sp = x;
                    }
                    named_sync(bar, FT_CONS);
                }
                if (INV) {
                    // round 0 holds elements 16 rt + k: 16-byte pairs
#pragma unroll
                    for (int k = 0; k < NV; k += 2) {
                        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(t8 + swz(gl, 16 * rt + k));
                        v[k] = A::in(x.x, P);
                        v[k + 1] = A::in(x.y, P);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < NV; k++) v[k] = *reinterpret_cast<const u64 *>(t8 + swz(gl, held<LO0>(rt, k)));
                }
                do_round<FS, INV, 0, true, FL, A>(v, rt, g, tw, P);
                if (INV) {
#pragma unroll
                    for (int k = 0; k < NV; k += 2)
                        *reinterpret_cast<ulonglong2 *>(t8 + swz(gl, 16 * rt + k)) = make_ulonglong2(v[k], v[k + 1]);
                } else {
#pragma unroll
                    for (int k = 0; k < NV; k++) *reinterpret_cast<u64 *>(t8 + swz(gl, held<LO0>(rt, k))) = v[k];
                }
                named_sync(bar, FT_CONS);
                if (INV) {
#pragma unroll
                    for (int k = 0; k < NV; k++) v[k] = *reinterpret_cast<const u64 *>(t8 + swz(gl, held<LO1>(rt, k)));
                } else {
#pragma unroll
                    for (int k = 0; k < NV; k += 2) {
                        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(t8 + swz(gl, 16 * rt + k));
                        v[k] = x.x;
                        v[k + 1] = x.y;
                    }
                }
                do_round<FS, INV, 1, true, FL, A>(v, rt, g, tw, P);
                if (INV) {
#pragma unroll
                    for (int k = 0; k < NV; k++) *reinterpret_cast<u64 *>(t8 + swz(gl, held<LO1>(rt, k))) = v[k];
                } else {
#pragma unroll
                    for (int k = 0; k < NV; k += 2)
                        *reinterpret_cast<ulonglong2 *>(t8 + swz(gl, 16 * rt + k)) =
                            make_ulonglong2(A::out_fwd(v[k], P), A::out_fwd(v[k + 1], P));
                }
                if (!INV && OUT != OUT_PLAIN) {
                    // fused epilogue on 16-byte vectors (rescale R12 / ModDown R11), as ntt.cu contig_body
                    named_sync(bar, FT_CONS);
                    const NttFusion &f = a.f;
                    const ulonglong2 *e1 = reinterpret_cast<const ulonglong2 *>(f.e1.p + poly_off(f.e1.cs, f.e1.ps, poly) + toff);
                    const ulonglong2 *e1b = nullptr, *e2 = nullptr, *e3 = nullptr;
                    u64 lc1 = 0, lc2 = 0, br0e = 0, br1e = 0;
                    if (OUT == OUT_RESCALE && f.lin) {
                        br0e = a.tab.br0[prime];
                        br1e = a.tab.br1[prime];
                        lc1 = smod_dev(f.C1, q, br0e, br1e);
                        if (f.lin == 2) {
                            lc2 = smod_dev(f.C2, q, br0e, br1e);
                            e1b = reinterpret_cast<const ulonglong2 *>(f.e1b.p + poly_off(f.e1b.cs, f.e1b.ps, poly) + toff);
                        }
                    }
                    if (OUT == OUT_MODDOWN && (poly & 1) < f.e2_polys)
                        e2 = reinterpret_cast<const ulonglong2 *>(f.e2.p + poly_off(f.e2.cs, f.e2.ps, poly) + toff);
                    if (OUT == OUT_MODDOWN && f.e3.p)
                        e3 = reinterpret_cast<const ulonglong2 *>(f.e3.p + poly_off(f.e3.cs, f.e3.ps, poly) + toff);
                    const u64 kc = f.k[limb], kcsh = f.ksh[limb];
#pragma unroll 4
                    for (int i = ct; i < TILE_WORDS / 2; i += FT_CONS) {
                        const int e = 2 * i;
                        ulonglong2 *sp = reinterpret_cast<ulonglong2 *>(t8 + swz(e >> 8, e & 255));
                        ulonglong2 x = *sp;
                        if (OUT == OUT_RESCALE) {
                            ulonglong2 c = e1[i];
                            if (f.lin) {
                                U128 t0 = mul_wide(c.x, lc1), t1 = mul_wide(c.y, lc1);
                                if (e1b) {
                                    const ulonglong2 y = e1b[i];
                                    mac_wide(t0, y.x, lc2);
                                    mac_wide(t1, y.y, lc2);
                                }
                                c.x = barrett128(t0, q, br0e, br1e);
                                c.y = barrett128(t1, q, br0e, br1e);
                            }
                            x.x = mul_shoup(addmod(c.x, x.x, q), kc, kcsh, q);
                            x.y = mul_shoup(addmod(c.y, x.y, q), kc, kcsh, q);
                        } else {
                            const ulonglong2 c = e1[i];
                            x.x = mul_shoup(submod(c.x, x.x, q), kc, kcsh, q);
                            x.y = mul_shoup(submod(c.y, x.y, q), kc, kcsh, q);
                            if (e2) {
                                const ulonglong2 d = e2[i];
                                x.x = addmod(x.x, d.x, q);
                                x.y = addmod(x.y, d.y, q);
                            }
                            if (e3) {
                                const ulonglong2 d = e3[i];
                                x.x = addmod(x.x, d.x, q);
                                x.y = addmod(x.y, d.y, q);
                            }
                        }
                        *sp = x;
                    }
                }
            }
            // generic-proxy writes -> the TMA store (async proxy) of this stage
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&computed[s]);
        }
    }
    // the last CTA out resets the claim counter (self-cleaning: the next launch on the stream starts at 0)
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(&sy->exit, 1u) == gridDim.x - 1) {
            sy->work = 0;
            sy->exit = 0;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 5-D view (element, line, limb, c0/c1, ciphertext) of nsub limbs of every polynomial at base:
// column view (col): 256 x 256 elements per limb, box 16 columns x 256 rows;
// row view: 16-element (128-byte) lines, 4096 per limb, box 256 lines (16 matrix rows), 128-byte swizzle
bool make_map(CUtensorMap *m, const u64 *base, bool col, int nsub, long cs, long ps, int n_polys) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const int nct = (n_polys + 1) / 2, nb = n_polys > 1 ? 2 : 1;
    if (((ps * 8) % 16) || ((cs * 8) % 16) || (reinterpret_cast<uintptr_t>(base) % 16)) return false;
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5] = {16, 256, 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    if (col) {
        dims[0] = 256;
        dims[1] = 256;
        strides[0] = 256 * 8;
    } else {
        dims[0] = 16;
        dims[1] = FN / 16;
        strides[0] = 128;
    }
    dims[2] = (cuuint64_t)nsub;
    dims[3] = (cuuint64_t)nb;
    dims[4] = (cuuint64_t)nct;
    strides[1] = (cuuint64_t)FN * 8;
    strides[2] = (cuuint64_t)(ps > 0 ? ps : FN) * 8;
    strides[3] = (cuuint64_t)(cs > 0 ? cs : 2 * FN) * 8;
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, const_cast<u64 *>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, col ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// per-stream self-cleaning counters (allocated zeroed on first use, outside any capture)
FtSync *stream_sync(cudaStream_t st) {
    static std::mutex mu;
    static std::map<cudaStream_t, FtSync *> m;
    std::lock_guard<std::mutex> g(mu);
    auto it = m.find(st);
    if (it != m.end()) return it->second;
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    CUDA_CHECK(cudaThreadExchangeStreamCaptureMode(&mode));
    FtSync *p = nullptr;
    cudaStream_t z = nullptr;
    cudaError_t e = cudaMalloc(&p, sizeof(FtSync));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&z, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, sizeof(FtSync), z);
    if (e == cudaSuccess) e = cudaStreamSynchronize(z);
    if (z) cudaStreamDestroy(z);
    cudaThreadExchangeStreamCaptureMode(&mode);
    CUDA_CHECK(e);
    m[st] = p;
    return p;
}

// SECPE_NTT_FUSED: 0 off; 1 every exact-FP64 run; 2 (default) plain transforms of at least FT_AUTO_ROWS rows
// only.  Measured (tools/ntt_fused_ab.py, profiles/r02_notes.md): the fused kernel moves 1.1 MB per limb
// instead of 2.08 MB but the transform is FP64-pipe bound, so it wins only where the two-pass kernels'
// extra HBM pass is not hidden (large launches, 3-4 %); inside the argmax step (100-700 rows per launch,
// fused prologues / epilogues) its pipeline fill and drain cost more than the saved traffic
int g_fused_mode = -1;
int ft_auto_rows() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SECPE_NTT_FUSED_ROWS");  // development switch
        v = e ? atoi(e) : 1024;
    }
    return v;
}

template <class A, bool INV, int IN, int OUT>
void launch_k(const FtArgs &a, cudaStream_t st) {
    auto kern = ntt_fused_kernel<A, INV, IN, OUT>;
    constexpr int smem = FT_STAGES * STAGE_BYTES + 1024;
    static int ctas = 0;  // per instantiation
    if (!ctas) {
        CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int dev = 0, sms = 0, per = 0;
        CUDA_CHECK(cudaGetDevice(&dev));
        CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, FT_THREADS, smem));
        ctas = sms * std::max(per, 1);
    }
    const int items = a.rows * 2 * TILES_PER_LIMB;
    const int grid = std::min(ctas, items);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(FT_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
}

template <class A, bool INV>
void dispatch_modes(const FtArgs &a, cudaStream_t st) {
    const NttFusion &f = a.f;
    if (!INV) {
        const bool bc = f.in_mode == IN_BCAST;
        if (f.out_mode == OUT_RESCALE)
            bc ? launch_k<A, false, IN_BCAST, OUT_RESCALE>(a, st) : launch_k<A, false, IN_PLAIN, OUT_RESCALE>(a, st);
        else if (f.out_mode == OUT_MODDOWN)
            bc ? launch_k<A, false, IN_BCAST, OUT_MODDOWN>(a, st) : launch_k<A, false, IN_PLAIN, OUT_MODDOWN>(a, st);
        else
            bc ? launch_k<A, false, IN_BCAST, OUT_PLAIN>(a, st) : launch_k<A, false, IN_PLAIN, OUT_PLAIN>(a, st);
    } else {
        switch (f.in_mode) {
            case IN_SRC: launch_k<A, true, IN_SRC, OUT_PLAIN>(a, st); break;
            case IN_MUL: launch_k<A, true, IN_MUL, OUT_PLAIN>(a, st); break;
            case IN_MUL2: launch_k<A, true, IN_MUL2, OUT_PLAIN>(a, st); break;
            case IN_LIN: launch_k<A, true, IN_LIN, OUT_PLAIN>(a, st); break;
            default: launch_k<A, true, IN_PLAIN, OUT_PLAIN>(a, st); break;
        }
    }
}

}  // namespace

int ntt_fused_mode(int mode) {
    ntt_fused_enabled();
    const int prev = g_fused_mode;
    if (mode >= 0) g_fused_mode = mode;
    return prev;
}

bool ntt_fused_enabled() {
    if (g_fused_mode < 0) {
        const char *e = getenv("SECPE_NTT_FUSED");
        g_fused_mode = e ? atoi(e) : 2;
    }
    return g_fused_mode > 0 && encode_fn() != nullptr;
}

// one run of same-class limbs [limb0, limb0 + nsub) of n_polys polynomials; false: not handled (caller
// falls back to the two-pass kernels)
bool ntt_fused_run(const Tab &tab, int logn, RowsArg d, int n_polys, LimbMap lm, int limb0, int nsub, int cls,
                   bool inverse, const NttFusion &f, cudaStream_t st) {
    if (logn != FL || !ntt_fused_enabled()) return false;
    if ((g_fused_mode == 2 || (g_fused_mode == 3 && cls == 0)) && (f.in_mode != IN_PLAIN || f.out_mode != OUT_PLAIN || (long)n_polys * nsub < ft_auto_rows()))
        return false;
    // classes (ntt.cu): 0 exact FP64 (FpA), 1 FP64 with reductions (FpB: two-pass kernels), 2 integer (IntA)
    if (cls == 1) return false;
    if (cls == 2 && g_fused_mode < 3) return false;  // integer rows: opt-in (mode 3)
    if ((long)n_polys * nsub > FT_MAXROWS) return false;
    FtArgs a{};
    a.tab = tab;
    a.f = f;
    a.lm = lm;
    a.limb0 = limb0;
    a.nsub = nsub;
    a.lag = NTT_FUSED_LAG;
    a.d_cs = d.cs;
    a.d_ps = d.ps;
    const u64 *dbase = d.p + (long)limb0 * FN;
    const bool colA = !inverse;
    bool ok = true;
    // phase A load: data, or the fused source (inverse prologues; forward rescale broadcast)
    if (!inverse && f.in_mode == IN_BCAST)
        ok &= make_map(&a.a_in, f.src.p, true, 1, f.src.cs, f.src.ps, n_polys);
    else if (inverse && f.in_mode != IN_PLAIN)
        ok &= make_map(&a.a_in, f.src.p + (long)limb0 * FN, colA, nsub, f.src.cs, f.src.ps, n_polys);
    else
        ok &= make_map(&a.a_in, dbase, colA, nsub, d.cs, d.ps, n_polys);
    ok &= make_map(&a.a_out, dbase, colA, nsub, d.cs, d.ps, n_polys);
    ok &= make_map(&a.b_in, dbase, !colA, nsub, d.cs, d.ps, n_polys);
    if (!inverse && f.out_mode != OUT_PLAIN)
        ok &= make_map(&a.b_out, f.out.p + (long)limb0 * FN, !colA, nsub, f.out.cs, f.out.ps, n_polys);
    else
        ok &= make_map(&a.b_out, dbase, !colA, nsub, d.cs, d.ps, n_polys);
    if (!ok) return false;
    a.sync = stream_sync(st);
    a.rows = n_polys * nsub;
    if (cls == 0) {
        if (inverse)
            dispatch_modes<FpA, true>(a, st);
        else
            dispatch_modes<FpA, false>(a, st);
    } else {
        if (inverse)
            dispatch_modes<IntA, true>(a, st);
        else
            dispatch_modes<IntA, false>(a, st);
    }
    LAUNCH_CHECK();
    return true;
}
