// common.cuh -- internal definitions of libsecpe (product path; shares nothing with oracle/).
//
// 64-bit modular arithmetic on the sm_100a integer pipes:
//   * Shoup multiplication by a precomputed constant w (w' = floor(w 2^64 / q)):
//       a*w - umulhi(a, w') q  in [0, 2q) for any a < 2^64   (lazy, Harvey-style)
//   * Barrett reduction of a 128-bit value with r = floor(2^128 / q) = (r1, r0):
//       qhat = hi r1 + hi64(hi r0 + lo r1 + hi64(lo r0)) = floor(z r / 2^128),  z - qhat q in [0, 2q)
// All primes are < 2^62 so 4q fits in a word.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;
typedef __int128 i128;  // plan constants C = rha(c Delta_c), |C| < 2^120 (plan.cu CONST_LIMIT)

#define SECPE_HD __host__ __device__ __forceinline__

// ----------------------------------------------------------------------------------------
// device arithmetic
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ u64 csub(u64 a, u64 q) { return a >= q ? a - q : a; }

__device__ __forceinline__ u64 mul_shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) {
    return a * w - __umul64hi(a, wsh) * q;
}
__device__ __forceinline__ u64 mul_shoup(u64 a, u64 w, u64 wsh, u64 q) {
    return csub(mul_shoup_lazy(a, w, wsh, q), q);
}

struct U128 {
    u64 lo, hi;
};
__device__ __forceinline__ U128 mul_wide(u64 a, u64 b) {
    U128 r;
    r.lo = a * b;
    r.hi = __umul64hi(a, b);
    return r;
}
__device__ __forceinline__ void add_wide(U128 &acc, U128 v) {
    u64 lo = acc.lo + v.lo;
    acc.hi += v.hi + (lo < v.lo ? 1 : 0);
    acc.lo = lo;
}
__device__ __forceinline__ void mac_wide(U128 &acc, u64 a, u64 b) { add_wide(acc, mul_wide(a, b)); }

// z mod q for z < 2^125 and 2^32 < q < 2^62 (exact result in [0, q))
__device__ __forceinline__ u64 barrett128(U128 z, u64 q, u64 r0, u64 r1) {
    // t = hi*r0 + lo*r1 + hi64(lo*r0)   (128-bit)
    U128 t = mul_wide(z.hi, r0);
    add_wide(t, mul_wide(z.lo, r1));
    add_wide(t, U128{__umul64hi(z.lo, r0), 0});
    u64 qhat = z.hi * r1 + t.hi;
    return csub(z.lo - qhat * q, q);  // qhat = floor(z r / 2^128) >= floor(z/q) - 1 -> [0, 2q)
}
__device__ __forceinline__ u64 mulmod(u64 a, u64 b, u64 q, u64 r0, u64 r1) {
    return barrett128(mul_wide(a, b), q, r0, r1);
}
__device__ __forceinline__ u64 addmod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
__device__ __forceinline__ u64 submod(u64 a, u64 b, u64 q) { return csub(a + q - b, q); }

// ----------------------------------------------------------------------------------------
// device tables (struct of arrays indexed by global prime index: q_0..q_L, p_0..p_{k-1})
// ----------------------------------------------------------------------------------------
struct Tab {
    const u64 *q;      // [P]
    const u64 *br0;    // [P] Barrett floor(2^128/q) low word
    const u64 *br1;    // [P] high word
    const ulonglong2 *tw2;   // [P][N] {psi^{brv(i)}, Shoup companion}   (forward CT twiddles)
    const ulonglong2 *itw2;  // [P][N] {psi^{-brv(i)}, Shoup companion}  (inverse GS twiddles)
    const u64 *ninv;   // [P] N^{-1} mod q
    const u64 *ninvsh; // [P]
    u64 fp_mask;       // host-visible: bit i set when prime i < 2^46 (exact-FP64 NTT rows, ntt.cu FpA)
    const double *qd;  // [P] (double) q and RN(1 / q): no per-CTA int->double conversion or division
    const double *qinv;
    int ntt_cluster;   // host-visible: single-pass cluster NTT for 0 none, 1 FP rows, 2 all rows (SECPE_NTT_CLUSTER)
    // [P][N] {w, RN(w RN(1/q))} as doubles for the exact-FP64 rows (fused kernel, ntt_fused.cu); integer rows:
    // the same pointer as tw2 / itw2 ({w, Shoup companion})
    const ulonglong2 *twp = nullptr, *itwp = nullptr;
    // host-visible: bit i set when 2^46 <= prime i < 2^52 / 3.5 (~50-bit rows: exact-FP64 NTT with reductions,
    // ntt_core.cuh FpB; dense double twiddle tables like the FpA rows)
    u64 fpb_mask = 0;
};

// limb l of a polynomial -> global prime index
struct LimbMap {
    int nl;      // limbs per polynomial
    int nq_part; // first nq_part limbs are ciphertext primes q0 + l
    int q0;
    int p0;      // remaining limbs are primes p0 + (l - nq_part)
};
SECPE_HD int prime_of(const LimbMap &m, int l) { return l < m.nq_part ? m.q0 + l : m.p0 + (l - m.nq_part); }

// ----------------------------------------------------------------------------------------
// host-side helpers shared inside the library
// ----------------------------------------------------------------------------------------
struct SecpeError {
    int code;
    std::string msg;
};
void set_error(const std::string &m);
#define CUDA_CHECK(x)                                                                       \
    do {                                                                                    \
        cudaError_t e__ = (x);                                                              \
        if (e__ != cudaSuccess)                                                             \
            throw SecpeError{-7, std::string("CUDA: ") + cudaGetErrorString(e__) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__)};            \
    } while (0)
#define LAUNCH_CHECK() CUDA_CHECK(cudaGetLastError())

#ifndef SECPE_PDL
#define SECPE_PDL 1  // development switch
#endif
// Programmatic dependent launch: the kernel may be scheduled while its stream predecessor drains; it
// calls pdl_wait() before touching the predecessor's outputs (setup that reads only constants, keys or
// tables can come first).  Without the launch attribute pdl_wait() is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
void launch_pdl_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = SECPE_PDL ? 1 : 0;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}
