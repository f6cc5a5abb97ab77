// sample.cu -- keystream randomness and key/encryption assembly kernels (client side).
//
// Reading R6: every random object is drawn from a ChaCha20 keystream (Bernstein's layout:
// 64-bit block counter in state words 12-13, 64-bit nonce in 14-15).  The caller's 256-bit master seed is
// never used directly: the secret material (s, e: tags of kind 1, 3, 5) is drawn under
// derive(master, DOM_SK), the public uniform polynomials (kind 2, 4) under derive(master, DOM_PK), and the
// encryption randomness (kind 6-8) under derive(encryption seed, DOM_ENC), with derive(K, d) = the first 32
// bytes of block 0 of (K, nonce d).  Stream (key, tag): draw ctr = 64-bit word ctr mod 8 of block ctr / 8.
// Uniform residues (NTT domain): floor(X q / 2^128) with X = draws 2c || 2c+1, c = prime_index * N + k.
// Ternary: floor(x 3 / 2^64) -> {0, 1, -1}.  Gaussian sigma = 3.2: cumulative table over |e| <= 19 on the
// low 63 bits, sign = top bit.  A thread computes one block: 4 uniform coefficients or 8 small ones.
#include <algorithm>
#include <sys/random.h>

#include "common.cuh"
#include "kernels.h"

namespace {
constexpr int TPB = 256;
__constant__ u64 c_cdt[32];
__constant__ int c_ncdt;

SECPE_HD uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }
SECPE_HD void quarter(uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    a += b; d ^= a; d = rotl32(d, 16);
    c += d; b ^= c; b = rotl32(b, 12);
    a += b; d ^= a; d = rotl32(d, 8);
    c += d; b ^= c; b = rotl32(b, 7);
}
SECPE_HD void chacha_block(const Key256 &k, u64 counter, u64 nonce, uint32_t out[16]) {
    uint32_t x[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, k.w[0], k.w[1], k.w[2], k.w[3],
                      k.w[4], k.w[5], k.w[6], k.w[7], (uint32_t)counter, (uint32_t)(counter >> 32),
                      (uint32_t)nonce, (uint32_t)(nonce >> 32)};
    uint32_t in[16];
#pragma unroll
    for (int i = 0; i < 16; i++) in[i] = x[i];
#pragma unroll 1
    for (int r = 0; r < 10; r++) {
        quarter(x[0], x[4], x[8], x[12]);
        quarter(x[1], x[5], x[9], x[13]);
        quarter(x[2], x[6], x[10], x[14]);
        quarter(x[3], x[7], x[11], x[15]);
        quarter(x[0], x[5], x[10], x[15]);
        quarter(x[1], x[6], x[11], x[12]);
        quarter(x[2], x[7], x[8], x[13]);
        quarter(x[3], x[4], x[9], x[14]);
    }
#pragma unroll
    for (int i = 0; i < 16; i++) out[i] = x[i] + in[i];
}
SECPE_HD u64 word64(const uint32_t *w, int j) { return (u64)w[2 * j] | ((u64)w[2 * j + 1] << 32); }

// one block per thread: coefficients 4b .. 4b+3 of the limb (draws 8b .. 8b+7 = block (pr N + 4b) / 4)
__global__ void uniform_kernel(Tab tab, int logn, Key256 key, u64 tag, u64 *out, LimbMap lm) {
    const int limb = blockIdx.y;
    const int pr = prime_of(lm, limb);
    const u64 q = tab.q[pr];
    const u64 k0 = 4 * ((u64)blockIdx.x * TPB + threadIdx.x);
    uint32_t w[16];
    chacha_block(key, (((u64)pr << logn) + k0) >> 2, tag, w);
    u64 r[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const u64 xh = word64(w, 2 * i), xl = word64(w, 2 * i + 1);
        // floor((xh 2^64 + xl) q / 2^128) = hi64(xh q + hi64(xl q))
        const u64 c1 = __umul64hi(xl, q);
        const u64 lo = xh * q + c1;
        const u64 carry = lo < c1 ? 1 : 0;
        r[i] = __umul64hi(xh, q) + carry;
    }
    ulonglong2 *o = reinterpret_cast<ulonglong2 *>(out + ((long)limb << logn) + k0);
    o[0] = make_ulonglong2(r[0], r[1]);
    o[1] = make_ulonglong2(r[2], r[3]);
}

// one block per thread: coefficients 8b .. 8b+7
__global__ void small_kernel(int logn, Key256 key, u64 tag, int kind, i64 *out) {
    const u64 b = (u64)blockIdx.x * TPB + threadIdx.x;
    uint32_t w[16];
    chacha_block(key, b, tag, w);
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const u64 x = word64(w, j);
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
        out[8 * b + j] = v;
    }
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

inline dim3 g1(int logn, int rows) { return dim3((unsigned)((1L << logn) / TPB), rows); }
}  // namespace

Key256 derive_key(const Key256 &master, u64 domain) {
    uint32_t w[16];
    chacha_block(master, 0, domain, w);
    Key256 k;
    for (int i = 0; i < 8; i++) k.w[i] = w[i];
    return k;
}
Key256 object_key(const Key256 &master, u64 tag) {
    const u64 kind = tag >> 48;
    return derive_key(master, kind == 2 || kind == 4 ? DOM_PK : DOM_SK);
}
Key256 os_entropy_key() {
    Key256 k;
    size_t got = 0;
    while (got < sizeof k.w) {
        const ssize_t r = getrandom(reinterpret_cast<char *>(k.w) + got, sizeof k.w - got, 0);
        if (r < 0) throw SecpeError{-1, "getrandom failed: no OS entropy for an unseeded call"};
        got += (size_t)r;
    }
    return k;
}

// sparse ternary secret of Hamming weight h (R36), host side (key generation is client work): the ctr-th
// draw's top logn bits pick a coefficient; a still-zero one becomes -1 (odd draw) or +1; h nonzeros
void h_sample_sparse(const Key256 &key, u64 tag, int logn, int h, i64 *out) {
    std::fill(out, out + (1L << logn), (i64)0);
    int cnt = 0;
    uint32_t w[16];
    u64 blk = ~0ULL;
    for (u64 ctr = 0; cnt < h; ctr++) {
        if ((ctr >> 3) != blk) {
            blk = ctr >> 3;
            chacha_block(key, blk, tag, w);
        }
        const u64 x = word64(w, (int)(ctr & 7));
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
void k_sample_uniform(const Tab &tab, int logn, const Key256 &key, u64 tag, u64 *out, LimbMap lm, cudaStream_t st) {
    uniform_kernel<<<dim3((unsigned)((1L << logn) / (4 * TPB)), lm.nl), TPB, 0, st>>>(tab, logn, key, tag, out, lm);
    LAUNCH_CHECK();
}
void k_sample_small(int logn, const Key256 &key, u64 tag, int kind, i64 *out, cudaStream_t st) {
    small_kernel<<<dim3((unsigned)((1L << logn) / (8 * TPB))), TPB, 0, st>>>(logn, key, tag, kind, out);
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
