// sample.cu -- counter-based randomness and key/encryption assembly kernels (client side).
//
// Reading R6: stream(seed, tag) = SplitMix64 started at s0 = mix(seed ^ mix(tag + gamma));
// its ctr-th output is mix(s0 + (ctr + 1) gamma), so every coefficient is drawn independently on
// the GPU.  Uniform residues (NTT domain): floor(X q / 2^128) with X = draws 2c, 2c+1 where
// c = prime_index * N + k.  Ternary: floor(x 3 / 2^64) -> {0, 1, -1}.  Gaussian sigma = 3.2:
// cumulative table over |e| <= 19 on the low 63 bits, sign = top bit.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace {
constexpr int TPB = 256;
constexpr u64 GAMMA = 0x9E3779B97F4A7C15ULL;
__constant__ u64 c_cdt[32];
__constant__ int c_ncdt;

__device__ __forceinline__ u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ u64 stream_state(u64 seed, u64 tag) { return mix64(seed ^ mix64(tag + GAMMA)); }
__device__ __forceinline__ u64 draw(u64 s0, u64 ctr) { return mix64(s0 + (ctr + 1) * GAMMA); }

__global__ void uniform_kernel(Tab tab, int logn, u64 s0, u64 *out, LimbMap lm) {
    const int limb = blockIdx.y;
    const int pr = prime_of(lm, limb);
    const u64 q = tab.q[pr];
    const u64 k = (u64)blockIdx.x * TPB + threadIdx.x;
    const u64 ctr = 2 * (((u64)pr << logn) + k);
    const u64 xh = draw(s0, ctr), xl = draw(s0, ctr + 1);
    // floor((xh 2^64 + xl) q / 2^128) = hi64(xh q + hi64(xl q))
    const u64 c1 = __umul64hi(xl, q);
    const u64 lo = xh * q + c1;
    const u64 carry = lo < c1 ? 1 : 0;
    out[((long)limb << logn) + k] = __umul64hi(xh, q) + carry;
}

__global__ void small_kernel(int logn, u64 s0, int kind, i64 *out) {
    const u64 k = (u64)blockIdx.x * TPB + threadIdx.x;
    const u64 x = draw(s0, k);
    i64 v;
    if (kind == 0) {
        const u64 t = __umul64hi(x, 3);
        v = t == 0 ? 0 : (t == 1 ? 1 : -1);
    } else {
        const u64 u = x & 0x7FFFFFFFFFFFFFFFULL;
        int m = 0;
        while (m < c_ncdt - 1 && u >= c_cdt[m]) m++;
        v = (x >> 63) ? -(i64)m : (i64)m;
    }
    out[k] = v;
}

__global__ void int_to_rows_kernel(Tab tab, int logn, const i64 *__restrict__ m, u64 *out, LimbMap lm) {
    const int limb = blockIdx.y;
    const int pr = prime_of(lm, limb);
    const u64 q = tab.q[pr];
    const u64 k = (u64)blockIdx.x * TPB + threadIdx.x;
    const i64 v = m[k];
    const u64 a = (u64)(v < 0 ? -v : v);
    u64 r = barrett128(U128{a, 0}, q, tab.br0[pr], tab.br1[pr]);
    if (v < 0 && r) r = q - r;
    out[((long)limb << logn) + k] = r;
}

// out = -a s + e (+ g_l * sp on flagged limbs)
__global__ void key_combine_kernel(Tab tab, int logn, const u64 *__restrict__ a, const u64 *__restrict__ s,
                                   const u64 *__restrict__ e, const u64 *__restrict__ sp, LimbConst g, int use_g,
                                   u64 *out, LimbMap lm) {
    const int limb = blockIdx.y;
    const int pr = prime_of(lm, limb);
    const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
    const long i = ((long)limb << logn) + (long)blockIdx.x * TPB + threadIdx.x;
    const long is = ((long)pr << logn) + (long)blockIdx.x * TPB + threadIdx.x;  // s indexed by prime
    u64 v = submod(e[i], mulmod(a[i], s[is], q, r0, r1), q);
    if (use_g && g.c[limb]) v = addmod(v, mul_shoup(sp[i], g.c[limb], g.csh[limb], q), q);
    out[i] = v;
}

__global__ void encrypt_kernel(Tab tab, int logn, const u64 *__restrict__ v, const u64 *__restrict__ pk, long pks,
                               const u64 *__restrict__ e0, const u64 *__restrict__ e1, const u64 *__restrict__ m,
                               u64 *ct, int nl) {
    const int limb = blockIdx.y;
    const u64 q = tab.q[limb], r0 = tab.br0[limb], r1 = tab.br1[limb];
    const long i = ((long)limb << logn) + (long)blockIdx.x * TPB + threadIdx.x;
    const long P = (long)nl << logn;
    ct[i] = addmod(addmod(mulmod(v[i], pk[i], q, r0, r1), e0[i], q), m[i], q);
    ct[P + i] = addmod(mulmod(v[i], pk[pks + i], q, r0, r1), e1[i], q);
}

__global__ void decrypt_kernel(Tab tab, int logn, const u64 *__restrict__ ct, const u64 *__restrict__ s, u64 *out,
                               int nl) {
    const int limb = blockIdx.y;
    const u64 q = tab.q[limb], r0 = tab.br0[limb], r1 = tab.br1[limb];
    const long i = ((long)limb << logn) + (long)blockIdx.x * TPB + threadIdx.x;
    const long P = (long)nl << logn;
    out[i] = addmod(ct[i], mulmod(ct[P + i], s[i], q, r0, r1), q);
}

__global__ void square_kernel(Tab tab, int logn, const u64 *__restrict__ a, u64 *out, LimbMap lm) {
    const int limb = blockIdx.y;
    const int pr = prime_of(lm, limb);
    const long i = ((long)limb << logn) + (long)blockIdx.x * TPB + threadIdx.x;
    out[i] = mulmod(a[i], a[i], tab.q[pr], tab.br0[pr], tab.br1[pr]);
}

// host mirror of stream_state for the launch parameter
u64 host_mix(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
u64 host_state(u64 seed, u64 tag) { return host_mix(seed ^ host_mix(tag + GAMMA)); }
inline dim3 g1(int logn, int rows) { return dim3((unsigned)((1L << logn) / TPB), rows); }
}  // namespace

// sparse ternary secret of Hamming weight h (R36), host side (key generation is client work): the ctr-th
// draw's top logn bits pick a coefficient; a still-zero one becomes -1 (odd draw) or +1; h nonzeros
void h_sample_sparse(u64 seed, u64 tag, int logn, int h, i64 *out) {
    const u64 s0 = host_state(seed, tag);
    std::fill(out, out + (1L << logn), (i64)0);
    int cnt = 0;
    for (u64 ctr = 0; cnt < h; ctr++) {
        const u64 x = host_mix(s0 + (ctr + 1) * GAMMA);
        const u64 pos = x >> (64 - logn);
        if (out[pos] == 0) {
            out[pos] = (x & 1) ? -1 : 1;
            cnt++;
        }
    }
}

void set_cdt(const u64 *cdt, int n) {
    CUDA_CHECK(cudaMemcpyToSymbol(c_cdt, cdt, sizeof(u64) * n));
    CUDA_CHECK(cudaMemcpyToSymbol(c_ncdt, &n, sizeof(int)));
}
void k_sample_uniform(const Tab &tab, int logn, u64 seed, u64 tag, u64 *out, LimbMap lm, cudaStream_t st) {
    uniform_kernel<<<g1(logn, lm.nl), TPB, 0, st>>>(tab, logn, host_state(seed, tag), out, lm);
    LAUNCH_CHECK();
}
void k_sample_small(int logn, u64 seed, u64 tag, int kind, i64 *out, cudaStream_t st) {
    small_kernel<<<g1(logn, 1), TPB, 0, st>>>(logn, host_state(seed, tag), kind, out);
    LAUNCH_CHECK();
}
void k_int_to_rows(const Tab &tab, int logn, const i64 *m, u64 *out, LimbMap lm, cudaStream_t st) {
    int_to_rows_kernel<<<g1(logn, lm.nl), TPB, 0, st>>>(tab, logn, m, out, lm);
    LAUNCH_CHECK();
}
// ModRaise (R33): coefficient-form residues mod q_0 (coef[P][N], P = polynomial) centred into
// (-q_0/2, q_0/2] and reduced mod every ciphertext prime q_0..q_{nl-1} (coefficient form out)
__global__ void mod_raise_kernel(Tab tab, int logn, const u64 *__restrict__ coef, RowsArg out, int nl) {
    const int limb = blockIdx.y, P = blockIdx.z;
    const u64 k = (u64)blockIdx.x * TPB + threadIdx.x;
    const u64 q0 = tab.q[0], q = tab.q[limb];
    const u64 a = coef[((long)P << logn) + k];
    const bool neg = a > (q0 - 1) / 2;
    const u64 mag = neg ? q0 - a : a;  // |centred value| < q_0 / 2
    u64 r = barrett128(U128{mag, 0}, q, tab.br0[limb], tab.br1[limb]);
    if (neg && r) r = q - r;
    out.p[poly_off(out.cs, out.ps, P) + ((long)limb << logn) + k] = r;
}
void k_mod_raise(const Tab &tab, int logn, const u64 *coef, RowsArg out, int n_polys, int nl, cudaStream_t st) {
    dim3 g = g1(logn, nl);
    g.z = n_polys;
    mod_raise_kernel<<<g, TPB, 0, st>>>(tab, logn, coef, out, nl);
    LAUNCH_CHECK();
}
void k_key_combine(const Tab &tab, int logn, const u64 *a, const u64 *s, const u64 *e, const u64 *sp,
                   const LimbConst *gadget, u64 *out, LimbMap lm, cudaStream_t st) {
    LimbConst g{};
    if (gadget) g = *gadget;
    key_combine_kernel<<<g1(logn, lm.nl), TPB, 0, st>>>(tab, logn, a, s, e, sp, g, gadget ? 1 : 0, out, lm);
    LAUNCH_CHECK();
}
void k_encrypt_combine(const Tab &tab, int logn, const u64 *v, const u64 *pk, long pks, const u64 *e0,
                       const u64 *e1, const u64 *m, u64 *ct, int nl, cudaStream_t st) {
    encrypt_kernel<<<g1(logn, nl), TPB, 0, st>>>(tab, logn, v, pk, pks, e0, e1, m, ct, nl);
    LAUNCH_CHECK();
}
void k_decrypt_combine(const Tab &tab, int logn, const u64 *ct, const u64 *s, u64 *out, int nl, cudaStream_t st) {
    decrypt_kernel<<<g1(logn, nl), TPB, 0, st>>>(tab, logn, ct, s, out, nl);
    LAUNCH_CHECK();
}
void k_square(const Tab &tab, int logn, const u64 *a, u64 *out, LimbMap lm, cudaStream_t st) {
    square_kernel<<<g1(logn, lm.nl), TPB, 0, st>>>(tab, logn, a, out, lm);
    LAUNCH_CHECK();
}
