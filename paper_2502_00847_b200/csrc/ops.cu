// ops.cu -- HBM-bound elementwise kernels: modular add/sub, constant and plaintext products,
// the ciphertext tensor product and the NTT-domain Galois automorphism
// (PAPER.md:104-105).  Every kernel streams limbs with 16-byte vector accesses, two
// coefficients per thread, grid.y = (polynomial, limb) row.
#include "common.cuh"
#include "kernels.h"

namespace {
constexpr int TPB = 256;

__device__ __forceinline__ ulonglong2 ld2(const u64 *p) { return *reinterpret_cast<const ulonglong2 *>(p); }
__device__ __forceinline__ void st2(u64 *p, ulonglong2 v) { *reinterpret_cast<ulonglong2 *>(p) = v; }

inline dim3 grid_rows(int logn, int rows) { return dim3((unsigned)((1L << logn) / (2 * TPB)), rows); }

__global__ void addsub_kernel(Tab tab, int logn, CRows a, CRows b, RowsArg out, LimbMap lm, int sub) {
    const int nl = lm.nl, poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const u64 q = tab.q[prime_of(lm, limb)];
    const long off = (long)limb << logn;
    const long k = 2L * (blockIdx.x * TPB + threadIdx.x);
    ulonglong2 x = ld2(a.p + poly_off(a.cs, a.ps, poly) + off + k), y = ld2(b.p + poly_off(b.cs, b.ps, poly) + off + k);
    ulonglong2 r;
    if (sub) {
        r.x = submod(x.x, y.x, q);
        r.y = submod(x.y, y.y, q);
    } else {
        r.x = addmod(x.x, y.x, q);
        r.y = addmod(x.y, y.y, q);
    }
    st2(out.p + poly_off(out.cs, out.ps, poly) + off + k, r);
}

__global__ void copy_kernel(int logn, CRows a, RowsArg out, int nl) {
    const int poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const long off = (long)limb << logn;
    const long k = 2L * (blockIdx.x * TPB + threadIdx.x);
    st2(out.p + poly_off(out.cs, out.ps, poly) + off + k, ld2(a.p + poly_off(a.cs, a.ps, poly) + off + k));
}

__global__ void mul_const_kernel(Tab tab, int logn, CRows a, RowsArg out, LimbMap lm, LimbConst c) {
    const int nl = lm.nl, poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const u64 q = tab.q[prime_of(lm, limb)];
    const u64 w = c.c[limb], wsh = c.csh[limb];
    const long off = (long)limb << logn;
    const long k = 2L * (blockIdx.x * TPB + threadIdx.x);
    ulonglong2 x = ld2(a.p + poly_off(a.cs, a.ps, poly) + off + k);
    x.x = mul_shoup(x.x, w, wsh, q);
    x.y = mul_shoup(x.y, w, wsh, q);
    st2(out.p + poly_off(out.cs, out.ps, poly) + off + k, x);
}

// out = C1 a + C2 b (per-limb constant residues, Shoup); b.p == nullptr: out = C1 a
__global__ void lincomb2_kernel(Tab tab, int logn, CRows a, CRows b, RowsArg out, LimbMap lm, LimbConst c1,
                                LimbConst c2) {
    const int nl = lm.nl, poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const u64 q = tab.q[prime_of(lm, limb)];
    const long off = (long)limb << logn;
    const long k = 2L * (blockIdx.x * TPB + threadIdx.x);
    ulonglong2 x = ld2(a.p + poly_off(a.cs, a.ps, poly) + off + k);
    x.x = mul_shoup(x.x, c1.c[limb], c1.csh[limb], q);
    x.y = mul_shoup(x.y, c1.c[limb], c1.csh[limb], q);
    if (b.p) {
        const ulonglong2 y = ld2(b.p + poly_off(b.cs, b.ps, poly) + off + k);
        x.x = addmod(x.x, mul_shoup(y.x, c2.c[limb], c2.csh[limb], q), q);
        x.y = addmod(x.y, mul_shoup(y.y, c2.c[limb], c2.csh[limb], q), q);
    }
    st2(out.p + poly_off(out.cs, out.ps, poly) + off + k, x);
}

__global__ void add_const_kernel(Tab tab, int logn, CRows a, RowsArg out, LimbMap lm, LimbConst c) {
    const int nl = lm.nl, poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const u64 q = tab.q[prime_of(lm, limb)];
    const u64 w = c.c[limb];
    const long off = (long)limb << logn;
    const long k = 2L * (blockIdx.x * TPB + threadIdx.x);
    ulonglong2 x = ld2(a.p + poly_off(a.cs, a.ps, poly) + off + k);
    x.x = addmod(x.x, w, q);
    x.y = addmod(x.y, w, q);
    st2(out.p + poly_off(out.cs, out.ps, poly) + off + k, x);
}

__global__ void mul_poly_kernel(Tab tab, int logn, CRows a, const u64 *__restrict__ b, RowsArg out, LimbMap lm) {
    const int nl = lm.nl, poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const int pr = prime_of(lm, limb);
    const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
    const long off = (long)limb << logn;
    const long k = 2L * (blockIdx.x * TPB + threadIdx.x);
    ulonglong2 x = ld2(a.p + poly_off(a.cs, a.ps, poly) + off + k), y = ld2(b + off + k);
    x.x = mulmod(x.x, y.x, q, r0, r1);
    x.y = mulmod(x.y, y.y, q, r0, r1);
    st2(out.p + poly_off(out.cs, out.ps, poly) + off + k, x);
}

// grid.y = ct * nl + limb
__global__ void tensor_kernel(Tab tab, int logn, CRows a, CRows b, u64 *__restrict__ d, long ds, int nl, CRows x,
                              LimbConst C) {
    const int ct = blockIdx.y / nl, limb = blockIdx.y % nl;
    const u64 q = tab.q[limb], r0 = tab.br0[limb], r1 = tab.br1[limb];
    const long N = 1L << logn, P = (long)nl * N;
    const long k = (long)limb * N + 2L * (blockIdx.x * TPB + threadIdx.x);
    const u64 *A = a.p + ct * a.cs, *B = b.p + ct * b.cs;
    u64 *D = d + ct * ds;
    ulonglong2 a0 = ld2(A + k), a1 = ld2(A + a.ps + k), b0 = ld2(B + k), b1 = ld2(B + b.ps + k);
    ulonglong2 d0, d1, d2;
    d0.x = mulmod(a0.x, b0.x, q, r0, r1);
    d0.y = mulmod(a0.y, b0.y, q, r0, r1);
    U128 t = mul_wide(a0.x, b1.x);
    mac_wide(t, a1.x, b0.x);
    d1.x = barrett128(t, q, r0, r1);
    t = mul_wide(a0.y, b1.y);
    mac_wide(t, a1.y, b0.y);
    d1.y = barrett128(t, q, r0, r1);
    d2.x = mulmod(a1.x, b1.x, q, r0, r1);
    d2.y = mulmod(a1.y, b1.y, q, r0, r1);
    if (x.p) {
        const u64 *X = x.p + ct * x.cs;
        const ulonglong2 x0 = ld2(X + k), x1 = ld2(X + x.ps + k);
        const u64 c = C.c[limb], csh = C.csh[limb];
        d0.x = addmod(d0.x, mul_shoup(x0.x, c, csh, q), q);
        d0.y = addmod(d0.y, mul_shoup(x0.y, c, csh, q), q);
        d1.x = addmod(d1.x, mul_shoup(x1.x, c, csh, q), q);
        d1.y = addmod(d1.y, mul_shoup(x1.y, c, csh, q), q);
    }
    st2(D + k, d0);
    st2(D + P + k, d1);
    st2(D + 2 * P + k, d2);
}

__device__ __forceinline__ unsigned brv_bits(unsigned x, int bits) { return __brev(x) >> (32 - bits); }

// out[i] = in[i'] with 2 brv(i') + 1 = g (2 brv(i) + 1) mod 2N
__global__ void automorph_kernel(int logn, CRows a, RowsArg out, int nl, u64 g) {
    pdl_wait();
    const int poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const long off = (long)limb << logn;
    const unsigned mask2n = (2u << logn) - 1;
    const unsigned i0 = 2u * (blockIdx.x * TPB + threadIdx.x);
    const u64 *src = a.p + poly_off(a.cs, a.ps, poly) + off;
    u64 r[2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const unsigned i = i0 + h;
        const unsigned e = 2u * brv_bits(i, logn) + 1u;
        const unsigned e2 = (unsigned)(((u64)e * g) & mask2n);
        r[h] = __ldg(src + brv_bits((e2 - 1u) >> 1, logn));
    }
    st2(out.p + poly_off(out.cs, out.ps, poly) + off + i0, make_ulonglong2(r[0], r[1]));
}
// out[P][l] = sum_s pt_s[l] * a_s[P][l] mod q_l (linear transform, R30): a_s = ciphertext s of a batch
// (stride as), pt_s at pt + s * ps_stride; 128-bit accumulation reduced every 16 products
__global__ void mac_plain_kernel(Tab tab, int logn, CRows a, long as, const u64 *__restrict__ pt, long pts, int n,
                                 RowsArg out, LimbMap lm) {
    const int nl = lm.nl, poly = blockIdx.y / nl, limb = blockIdx.y % nl;
    const int pr = prime_of(lm, limb);
    const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
    const long off = (long)limb << logn;
    const long k = 2L * ((long)blockIdx.x * TPB + threadIdx.x);
    U128 s0{0, 0}, s1{0, 0};
    for (int s = 0; s < n; s++) {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(a.p + s * as + poly_off(a.cs, a.ps, poly) + off + k);
        const ulonglong2 w = *reinterpret_cast<const ulonglong2 *>(pt + s * pts + off + k);
        mac_wide(s0, x.x, w.x);
        mac_wide(s1, x.y, w.y);
        if ((s & 15) == 15) {
            s0 = U128{barrett128(s0, q, r0, r1), 0};
            s1 = U128{barrett128(s1, q, r0, r1), 0};
        }
    }
    *reinterpret_cast<ulonglong2 *>(out.p + poly_off(out.cs, out.ps, poly) + off + k) =
        make_ulonglong2(barrett128(s0, q, r0, r1), barrett128(s1, q, r0, r1));
}
}  // namespace

void k_mac_plain(const Tab &tab, int logn, CRows a, long as, const u64 *pt, long pts, int n, RowsArg out, int n_polys,
                 LimbMap lm, cudaStream_t st) {
    mac_plain_kernel<<<grid_rows(logn, n_polys * lm.nl), TPB, 0, st>>>(tab, logn, a, as, pt, pts, n, out, lm);
    LAUNCH_CHECK();
}

void k_addsub(const Tab &tab, int logn, CRows a, CRows b, RowsArg out, int n_polys, LimbMap lm, bool sub,
              cudaStream_t st) {
    addsub_kernel<<<grid_rows(logn, n_polys * lm.nl), TPB, 0, st>>>(tab, logn, a, b, out, lm, sub ? 1 : 0);
    LAUNCH_CHECK();
}
void k_copy_rows(int logn, CRows a, RowsArg out, int n_polys, int nl, cudaStream_t st) {
    copy_kernel<<<grid_rows(logn, n_polys * nl), TPB, 0, st>>>(logn, a, out, nl);
    LAUNCH_CHECK();
}
void k_mul_const(const Tab &tab, int logn, CRows a, RowsArg out, int n_polys, LimbMap lm, const LimbConst &c,
                 cudaStream_t st) {
    mul_const_kernel<<<grid_rows(logn, n_polys * lm.nl), TPB, 0, st>>>(tab, logn, a, out, lm, c);
    LAUNCH_CHECK();
}
void k_lincomb2(const Tab &tab, int logn, CRows a, CRows b, RowsArg out, int n_polys, LimbMap lm,
                const LimbConst &c1, const LimbConst &c2, cudaStream_t st) {
    lincomb2_kernel<<<grid_rows(logn, n_polys * lm.nl), TPB, 0, st>>>(tab, logn, a, b, out, lm, c1, c2);
    LAUNCH_CHECK();
}
void k_add_const(const Tab &tab, int logn, CRows a, RowsArg out, int n_polys, LimbMap lm, const LimbConst &c,
                 cudaStream_t st) {
    add_const_kernel<<<grid_rows(logn, n_polys * lm.nl), TPB, 0, st>>>(tab, logn, a, out, lm, c);
    LAUNCH_CHECK();
}
void k_mul_poly(const Tab &tab, int logn, CRows a, const u64 *b, RowsArg out, int n_polys, LimbMap lm,
                cudaStream_t st) {
    mul_poly_kernel<<<grid_rows(logn, n_polys * lm.nl), TPB, 0, st>>>(tab, logn, a, b, out, lm);
    LAUNCH_CHECK();
}
void k_tensor(const Tab &tab, int logn, CRows a, CRows b, u64 *d, long ds, int n_ct, int nl, cudaStream_t st,
              CRows x, const LimbConst *C) {
    static const LimbConst zero{};
    tensor_kernel<<<grid_rows(logn, n_ct * nl), TPB, 0, st>>>(tab, logn, a, b, d, ds, nl, x, C ? *C : zero);
    LAUNCH_CHECK();
}
void k_automorph(int logn, CRows a, RowsArg out, int n_polys, int nl, u64 galois, cudaStream_t st) {
    launch_pdl_k(automorph_kernel, grid_rows(logn, n_polys * nl), dim3(TPB), 0, st, logn, a, out, nl, galois);
    LAUNCH_CHECK();
}
