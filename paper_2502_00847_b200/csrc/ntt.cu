// ntt.cu -- batched multi-limb negacyclic NTT / INTT for sm_100a.
//
// Definition (R4): NTT(a)[i] = sum_k a_k psi^{(2 brv(i)+1) k} mod q, computed with the
// merged Cooley-Tukey network (twiddle psi^{brv(m+i)} at stage m) and its Gentleman-Sande inverse.
//
// Decomposition: N = 2^logN = G1 * G2 (G = 2^S).  Each transform is two passes over HBM:
//   forward : pass 1 = the first S1 stages on "columns" {c + (N/G1) r}  (strided groups)
//             pass 2 = the last  S2 stages on contiguous blocks of G2
//   inverse : pass A = the first S2 GS stages on contiguous blocks, pass B = the last S1 on columns
// Within a pass a group of G elements is held by G/8 threads, 8 values per thread (radix-8 register
// rounds of up to three butterfly stages), exchanging through shared memory between rounds.
// Strided passes put 16 consecutive columns in one CTA so every global access is a full 128-byte
// line; contiguous passes stage their loads/stores through shared memory with 16-byte vectors.
// Arithmetic: Harvey lazy butterflies with Shoup twiddles; forward values stay in [0, 4q),
// inverse in [0, 2q); the last pass reduces to [0, q) (and the inverse folds in N^{-1}).
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int STRIDED_C = 16;  // columns per CTA in strided passes (16 x 8 B = one 128-B line)

__device__ __forceinline__ void bfly_ct(u64 &x, u64 &y, u64 w, u64 wsh, u64 q, u64 q2) {
    u64 X = x >= q2 ? x - q2 : x;
    u64 T = mul_shoup_lazy(y, w, wsh, q);
    x = X + T;
    y = X - T + q2;
}
__device__ __forceinline__ void bfly_gs(u64 &x, u64 &y, u64 w, u64 wsh, u64 q, u64 q2) {
    u64 X = x, Y = y;
    u64 T = X + Y;
    x = T >= q2 ? T - q2 : T;
    y = mul_shoup_lazy(X - Y + q2, w, wsh, q);
}

// index of value v (3 bits) held by thread tau when the held bits start at LO
template <int LO>
__device__ __forceinline__ int held_index(int tau, int v) {
    return ((tau >> LO) << (LO + 3)) | (v << LO) | (tau & ((1 << LO) - 1));
}

// Rounds: forward round k pairs local bits hi = S-1-3k, hi-1, hi-2 (clipped at 0),
// holding bits LO = max(hi-2, 0).  Inverse round k pairs bits lo = 3k .. min(lo+2, S-1),
// holding LO = min(lo, S-3).
template <int S, bool INV>
struct RoundInfo {
    static constexpr int NR = (S + 2) / 3;
    __host__ __device__ static constexpr int first_bit(int k) { return INV ? 3 * k : S - 1 - 3 * k; }
    __host__ __device__ static constexpr int nbits(int k) {
        return INV ? ((3 * k + 2 <= S - 1) ? 3 : S - 3 * k) : ((S - 1 - 3 * k - 2 >= 0) ? 3 : S - 3 * k);
    }
    __host__ __device__ static constexpr int lo(int k) {
        return INV ? ((3 * k < S - 3) ? 3 * k : S - 3) : ((S - 1 - 3 * k - 2 > 0) ? S - 1 - 3 * k - 2 : 0);
    }
};

// One round of butterflies on the 8 values held by this thread.
// gidx(r) maps a local index to the global index within the limb.
template <int S, bool INV, int K, typename GIdx>
__device__ __forceinline__ void do_round(u64 (&v)[8], int tau, GIdx gidx, int logn, int sg0,
                                         const u64 *__restrict__ tw, const u64 *__restrict__ twsh,
                                         u64 q, u64 q2) {
    using R = RoundInfo<S, INV>;
    constexpr int LO = R::lo(K);
    constexpr int NB = R::nbits(K);
#pragma unroll
    for (int st = 0; st < NB; st++) {
        const int b = INV ? R::first_bit(K) + st : R::first_bit(K) - st;  // local bit paired
        const int vb = b - LO;
        const int s_local = INV ? b : (S - 1 - b);
        const int sg = INV ? sg0 - s_local : sg0 + s_local;  // global stage
        const int shift = logn - sg;
#pragma unroll
        for (int p = 0; p < 4; p++) {
            // p enumerates the 4 pairs: insert a 0 bit at position vb
            const int v0 = ((p >> vb) << (vb + 1)) | (p & ((1 << vb) - 1));
            const int v1 = v0 | (1 << vb);
            const int r0 = held_index<LO>(tau, v0);
            const int j0 = gidx(r0);
            const int ti = (1 << sg) + (j0 >> shift);
            const u64 w = __ldg(tw + ti), wsh = __ldg(twsh + ti);
            if (INV)
                bfly_gs(v[v0], v[v1], w, wsh, q, q2);
            else
                bfly_ct(v[v0], v[v1], w, wsh, q, q2);
        }
    }
}

template <int LO, typename Phys>
__device__ __forceinline__ void smem_store(u64 *sm, const u64 (&v)[8], int tau, Phys phys) {
#pragma unroll
    for (int k = 0; k < 8; k++) sm[phys(held_index<LO>(tau, k))] = v[k];
}
template <int LO, typename Phys>
__device__ __forceinline__ void smem_load(const u64 *sm, u64 (&v)[8], int tau, Phys phys) {
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = sm[phys(held_index<LO>(tau, k))];
}

struct PassArgs {
    u64 *data;
    long cs, ps;  // polynomial addressing (see RowsArg)
    LimbMap lm;
    Tab tab;
    int logn;
    int sg0;     // global stage of local stage 0
    int final_;  // last pass of the transform: reduce to [0, q) (inverse: also * N^{-1})
};

// ---------------------------------------------------------------------------------------------
// strided pass: group = column c, elements c + stride * r, 16 columns per CTA
// ---------------------------------------------------------------------------------------------
template <int S, bool INV>
__global__ void __launch_bounds__(STRIDED_C *(1 << S) / 8)
    ntt_strided(PassArgs a) {
    constexpr int G = 1 << S, C = STRIDED_C;
    __shared__ u64 sm[G * C];
    const int nl = a.lm.nl;
    const int poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const int prime = prime_of(a.lm, limb);
    const long N = 1L << a.logn;
    u64 *base = a.data + poly_off(a.cs, a.ps, poly) + limb * N;
    const u64 q = a.tab.q[prime], q2 = 2 * q;
    const u64 *tw = (INV ? a.tab.itw : a.tab.tw) + prime * N;
    const u64 *twsh = (INV ? a.tab.itwsh : a.tab.twsh) + prime * N;
    const int cl = threadIdx.x % C, tau = threadIdx.x / C;
    const int c = blockIdx.x * C + cl;
    const int stride = (int)(N >> S);
    auto gidx = [&](int r) { return c + stride * r; };
    auto phys = [&](int r) { return r * C + cl; };
    using R = RoundInfo<S, INV>;
    u64 v[8];
    constexpr int LO0 = R::lo(0);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = base[gidx(held_index<LO0>(tau, k))];
    do_round<S, INV, 0>(v, tau, gidx, a.logn, a.sg0, tw, twsh, q, q2);
    if constexpr (R::NR > 1) {
        smem_store<R::lo(0)>(sm, v, tau, phys);
        __syncthreads();
        smem_load<R::lo(1)>(sm, v, tau, phys);
        do_round<S, INV, 1>(v, tau, gidx, a.logn, a.sg0, tw, twsh, q, q2);
    }
    if constexpr (R::NR > 2) {
        __syncthreads();
        smem_store<R::lo(1)>(sm, v, tau, phys);
        __syncthreads();
        smem_load<R::lo(2)>(sm, v, tau, phys);
        do_round<S, INV, 2>(v, tau, gidx, a.logn, a.sg0, tw, twsh, q, q2);
    }
    constexpr int LOL = R::lo(R::NR - 1);
    if (a.final_) {
        if (INV) {
            const u64 ni = a.tab.ninv[prime], nish = a.tab.ninvsh[prime];
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = mul_shoup(v[k], ni, nish, q);
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = csub(csub(v[k], q2), q);
        }
    }
#pragma unroll
    for (int k = 0; k < 8; k++) base[gidx(held_index<LOL>(tau, k))] = v[k];
}

// ---------------------------------------------------------------------------------------------
// contiguous pass: group = block of G consecutive elements, CG groups per CTA
// ---------------------------------------------------------------------------------------------
template <int S>
struct ContigCfg {
    static constexpr int G = 1 << S;
    static constexpr int TPG = G / 8;
    static constexpr int CG = (256 / TPG) > 0 ? 256 / TPG : 1;  // 256 threads per CTA
    static constexpr int PITCH = G + G / 8;                     // padded group pitch in smem
};

template <int S, bool INV>
__global__ void __launch_bounds__(256) ntt_contig(PassArgs a) {
    using CF = ContigCfg<S>;
    constexpr int G = CF::G, TPG = CF::TPG, CG = CF::CG, PITCH = CF::PITCH;
    __shared__ __align__(16) u64 sm[CG * PITCH];
    const int nl = a.lm.nl;
    const int poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const int prime = prime_of(a.lm, limb);
    const long N = 1L << a.logn;
    u64 *base = a.data + poly_off(a.cs, a.ps, poly) + limb * N + (long)blockIdx.x * CG * G;
    const u64 q = a.tab.q[prime], q2 = 2 * q;
    const u64 *tw = (INV ? a.tab.itw : a.tab.tw) + prime * N;
    const u64 *twsh = (INV ? a.tab.itwsh : a.tab.twsh) + prime * N;
    const int gl = threadIdx.x / TPG, tau = threadIdx.x % TPG;
    const int g = blockIdx.x * CG + gl;
    auto gidx = [&](int r) { return g * G + r; };
    u64 *smg = sm + gl * PITCH;
    auto phys = [&](int r) { return r + (r >> 3); };
    // coalesced load of CG*G elements (16-byte vectors) into padded smem
    {
        const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(base);
        for (int i = threadIdx.x; i < CG * G / 2; i += 256) {
            ulonglong2 x = src[i];
            const int e = 2 * i, gg = e / G, r = e % G;
            sm[gg * PITCH + phys(r)] = x.x;
            sm[gg * PITCH + phys(r + 1)] = x.y;
        }
    }
    __syncthreads();
    using R = RoundInfo<S, INV>;
    u64 v[8];
    smem_load<R::lo(0)>(smg, v, tau, phys);
    do_round<S, INV, 0>(v, tau, gidx, a.logn, a.sg0, tw, twsh, q, q2);
    if constexpr (R::NR > 1) {
        __syncthreads();
        smem_store<R::lo(0)>(smg, v, tau, phys);
        __syncthreads();
        smem_load<R::lo(1)>(smg, v, tau, phys);
        do_round<S, INV, 1>(v, tau, gidx, a.logn, a.sg0, tw, twsh, q, q2);
    }
    if constexpr (R::NR > 2) {
        __syncthreads();
        smem_store<R::lo(1)>(smg, v, tau, phys);
        __syncthreads();
        smem_load<R::lo(2)>(smg, v, tau, phys);
        do_round<S, INV, 2>(v, tau, gidx, a.logn, a.sg0, tw, twsh, q, q2);
    }
    if (a.final_) {
        if (INV) {
            const u64 ni = a.tab.ninv[prime], nish = a.tab.ninvsh[prime];
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = mul_shoup(v[k], ni, nish, q);
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = csub(csub(v[k], q2), q);
        }
    }
    __syncthreads();
    smem_store<R::lo(R::NR - 1)>(smg, v, tau, phys);
    __syncthreads();
    {
        ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(base);
        for (int i = threadIdx.x; i < CG * G / 2; i += 256) {
            const int e = 2 * i, gg = e / G, r = e % G;
            dst[i] = make_ulonglong2(sm[gg * PITCH + phys(r)], sm[gg * PITCH + phys(r + 1)]);
        }
    }
}

template <int S, bool INV>
void launch_strided(const PassArgs &a, int n_rows, cudaStream_t st) {
    const long N = 1L << a.logn;
    const int ncols = (int)(N >> S);
    dim3 grid(ncols / STRIDED_C, n_rows);
    ntt_strided<S, INV><<<grid, STRIDED_C * (1 << S) / 8, 0, st>>>(a);
}
template <int S, bool INV>
void launch_contig(const PassArgs &a, int n_rows, cudaStream_t st) {
    const long N = 1L << a.logn;
    const int nblocks = (int)(N >> S);
    dim3 grid(nblocks / ContigCfg<S>::CG, n_rows);
    ntt_contig<S, INV><<<grid, 256, 0, st>>>(a);
}

template <bool INV>
void dispatch_strided(int S, const PassArgs &a, int rows, cudaStream_t st) {
    switch (S) {
        case 5: launch_strided<5, INV>(a, rows, st); break;
        case 6: launch_strided<6, INV>(a, rows, st); break;
        case 7: launch_strided<7, INV>(a, rows, st); break;
        case 8: launch_strided<8, INV>(a, rows, st); break;
        default: throw SecpeError{-1, "unsupported NTT split"};
    }
}
template <bool INV>
void dispatch_contig(int S, const PassArgs &a, int rows, cudaStream_t st) {
    switch (S) {
        case 5: launch_contig<5, INV>(a, rows, st); break;
        case 6: launch_contig<6, INV>(a, rows, st); break;
        case 7: launch_contig<7, INV>(a, rows, st); break;
        case 8: launch_contig<8, INV>(a, rows, st); break;
        case 9: launch_contig<9, INV>(a, rows, st); break;
        default: throw SecpeError{-1, "unsupported NTT split"};
    }
}

}  // namespace

// logN = S1 + S2 with S1 = logN / 2 (strided part), S2 = logN - S1 (contiguous part)
void ntt_forward(const Tab &tab, int logn, RowsArg data, int n_polys, LimbMap lm, cudaStream_t st) {
    if (n_polys <= 0 || lm.nl <= 0) return;
    const int S1 = logn / 2, S2 = logn - S1;
    const int rows = n_polys * lm.nl;
    PassArgs a{data.p, data.cs, data.ps, lm, tab, logn, 0, 0};
    dispatch_strided<false>(S1, a, rows, st);
    LAUNCH_CHECK();
    a.sg0 = S1;
    a.final_ = 1;
    dispatch_contig<false>(S2, a, rows, st);
    LAUNCH_CHECK();
}

void ntt_inverse(const Tab &tab, int logn, RowsArg data, int n_polys, LimbMap lm, cudaStream_t st) {
    if (n_polys <= 0 || lm.nl <= 0) return;
    const int S1 = logn / 2, S2 = logn - S1;
    const int rows = n_polys * lm.nl;
    PassArgs a{data.p, data.cs, data.ps, lm, tab, logn, logn - 1, 0};
    dispatch_contig<true>(S2, a, rows, st);
    LAUNCH_CHECK();
    a.sg0 = S1 - 1;
    a.final_ = 1;
    dispatch_strided<true>(S1, a, rows, st);
    LAUNCH_CHECK();
}
