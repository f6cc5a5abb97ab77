// ks.cu -- hybrid key switching (ModUp fast base conversion, key inner product, ModDown)
// and rescale kernels.  Readings R10/R11/R12 in DESIGN.md; PAPER.md:103-105 (relinearisation
// and rotation need key switching), PAPER.md:90-94 (leveled modulus chain / rescale).
//
// Base conversions accumulate the alpha (or k) 120-bit products lazily in 128 bits and
// reduce once with Barrett; the per-source factor [x (Q'/q_i)^-1]_{q_i} is a Shoup product.
#include "common.cuh"
#include "kernels.h"

namespace {
constexpr int TPB = 256;
constexpr int MAXA = 16;  // max primes per digit / special primes

// grid: x = coefficient chunks, y = ct * beta + j ; one coefficient per thread
__global__ void modup_kernel(Tab tab, int logn, const u64 *__restrict__ dc, long dcs, u64 *__restrict__ ext,
                             long exts, int nl, int np, int nq_total, int alpha, int beta,
                             const u64 *__restrict__ inv_hat, const u64 *__restrict__ inv_hat_sh,
                             const u64 *__restrict__ hat) {
    const int ct = blockIdx.y / beta, j = blockIdx.y % beta;
    const long N = 1L << logn;
    const long k = (long)blockIdx.x * TPB + threadIdx.x;
    const int i0 = j * alpha, i1 = min(i0 + alpha, nl), na = i1 - i0;
    const int ne = nl + np;
    u64 y[MAXA];
#pragma unroll
    for (int a = 0; a < MAXA; a++) {
        if (a < na) {
            const int i = i0 + a;
            y[a] = mul_shoup(dc[ct * dcs + i * N + k], inv_hat[i], inv_hat_sh[i], tab.q[i]);
        }
    }
    const u64 *hj = hat + (long)j * MAXA * ne;  // hat[j][a][e]
    u64 *out = ext + ct * exts + (long)j * ne * N + k;
    for (int e = 0; e < ne; e++) {
        if (e >= i0 && e < i1) continue;
        const int pr = e < nl ? e : nq_total + (e - nl);
        U128 acc{0, 0};
#pragma unroll
        for (int a = 0; a < MAXA; a++)
            if (a < na) mac_wide(acc, y[a], __ldg(hj + a * ne + e));
        out[e * N] = barrett128(acc, tab.q[pr], tab.br0[pr], tab.br1[pr]);
    }
}

// grid: x = coefficient chunks, y = extended limb e; loops over the n_ct ciphertexts so each key
// word is read from HBM once per launch (held in registers across the batch).  MAXB >= beta.
template <int MAXB>
__global__ void ks_inner_kernel(Tab tab, int logn, const u64 *__restrict__ d, long ds, const u64 *__restrict__ ext,
                                long exts, const u64 *__restrict__ key, int nq_total, int np,
                                u64 *__restrict__ acc, long accs, int n_ct, int nl, int alpha, int beta) {
    const int e = blockIdx.y;
    const long N = 1L << logn;
    const long k = (long)blockIdx.x * TPB + threadIdx.x;
    const int ne = nl + np, nk = nq_total + np;
    const int pr = e < nl ? e : nq_total + (e - nl);
    const u64 q = tab.q[pr], r0 = tab.br0[pr], r1 = tab.br1[pr];
    u64 kb[MAXB], ka[MAXB];
#pragma unroll
    for (int j = 0; j < MAXB; j++)
        if (j < beta) {
            kb[j] = __ldg(key + (((long)j * 2 + 0) * nk + pr) * N + k);
            ka[j] = __ldg(key + (((long)j * 2 + 1) * nk + pr) * N + k);
        }
    const int jd = e < nl ? e / alpha : -1;  // digit containing e (Q limbs only)
    for (int c = 0; c < n_ct; c++) {
        U128 s0{0, 0}, s1{0, 0};
#pragma unroll
        for (int j = 0; j < MAXB; j++)
            if (j < beta) {
                const u64 x = (j == jd) ? d[c * ds + e * N + k] : ext[c * exts + ((long)j * ne + e) * N + k];
                mac_wide(s0, x, kb[j]);
                mac_wide(s1, x, ka[j]);
            }
        acc[c * accs + (long)e * N + k] = barrett128(s0, q, r0, r1);
        acc[c * accs + (long)(ne + e) * N + k] = barrett128(s1, q, r0, r1);
    }
}

// grid: x = coefficient chunks, y = ct * 2 + b
__global__ void moddown_conv_kernel(Tab tab, int logn, const u64 *__restrict__ acc, long accs, u64 *__restrict__ T,
                                    long Ts, int nl, int np, int nq_total, const u64 *__restrict__ ihp,
                                    const u64 *__restrict__ ihp_sh, const u64 *__restrict__ hat_p) {
    const int ct = blockIdx.y / 2, b = blockIdx.y % 2;
    const long N = 1L << logn;
    const long k = (long)blockIdx.x * TPB + threadIdx.x;
    const int ne = nl + np;
    const u64 *src = acc + ct * accs + ((long)b * ne + nl) * N + k;
    u64 y[MAXA];
#pragma unroll
    for (int p = 0; p < MAXA; p++)
        if (p < np) {
            const int pr = nq_total + p;
            y[p] = mul_shoup(src[p * N], ihp[p], ihp_sh[p], tab.q[pr]);
        }
    u64 *dst = T + ct * Ts + (long)b * nl * N + k;
    for (int i = 0; i < nl; i++) {
        U128 s{0, 0};
#pragma unroll
        for (int p = 0; p < MAXA; p++)
            if (p < np) mac_wide(s, y[p], __ldg(hat_p + (long)p * nq_total + i));
        dst[i * N] = barrett128(s, tab.q[i], tab.br0[i], tab.br1[i]);
    }
}

// grid: x = coefficient chunks, y = (ct * 2 + b) * nl + i
__global__ void moddown_combine_kernel(Tab tab, int logn, const u64 *__restrict__ acc, long accs,
                                       const u64 *__restrict__ T, long Ts, const u64 *__restrict__ add, long adds,
                                       int add_polys, u64 *__restrict__ out, long outs, int nl, int ne,
                                       const u64 *__restrict__ pinv, const u64 *__restrict__ pinv_sh) {
    const int row = blockIdx.y;
    const int i = row % nl, b = (row / nl) % 2, ct = row / (2 * nl);
    const long N = 1L << logn;
    const long k = (long)blockIdx.x * TPB + threadIdx.x;
    const u64 q = tab.q[i];
    const u64 a = acc[ct * accs + ((long)b * ne + i) * N + k];
    const u64 t = T[ct * Ts + ((long)b * nl + i) * N + k];
    u64 v = mul_shoup(submod(a, t, q), pinv[i], pinv_sh[i], q);
    if (b < add_polys) v = addmod(v, add[ct * adds + ((long)b * nl + i) * N + k], q);
    out[ct * outs + ((long)b * nl + i) * N + k] = v;
}

// rescale, step 1 (coefficient domain): T[c][b][i] = [floor(q_l/2)]_{q_i} - [r]_{q_i} mod q_i with
// r = [c_l + floor(q_l/2)]_{q_l} per coefficient (the half is added to every coefficient).
// grid: y = (ct * 2 + b) * l + i
__global__ void rescale_bcast_kernel(Tab tab, int logn, const u64 *__restrict__ last, long lasts,
                                     u64 *__restrict__ T, long Ts, int l, const u64 *__restrict__ half) {
    const int row = blockIdx.y;
    const int i = row % l, b = (row / l) % 2, ct = row / (2 * l);
    const long N = 1L << logn;
    const long k = (long)blockIdx.x * TPB + threadIdx.x;
    const u64 ql = tab.q[l];
    const u64 r = csub(last[ct * lasts + (long)b * N + k] + (ql >> 1), ql);
    const u64 qi = tab.q[i];
    T[ct * Ts + ((long)b * l + i) * N + k] = submod(half[i], barrett128(U128{r, 0}, qi, tab.br0[i], tab.br1[i]), qi);
}

// rescale, step 2 (NTT domain): out = (in + NTT(T)) * q_l^{-1}
__global__ void rescale_combine_kernel(Tab tab, int logn, CRows in,
                                       const u64 *__restrict__ T, long Ts, u64 *__restrict__ out, long outs, int l,
                                       const u64 *__restrict__ qlinv,
                                       const u64 *__restrict__ qlinv_sh) {
    const int row = blockIdx.y;
    const int i = row % l, b = (row / l) % 2, ct = row / (2 * l);
    const long N = 1L << logn;
    const long k = (long)blockIdx.x * TPB + threadIdx.x;
    const u64 q = tab.q[i];
    const u64 x = in.p[poly_off(in.cs, in.ps, 2 * ct + b) + (long)i * N + k];
    const u64 t = T[ct * Ts + ((long)b * l + i) * N + k];
    const u64 v = addmod(x, t, q);
    out[ct * outs + ((long)b * l + i) * N + k] = mul_shoup(v, qlinv[i], qlinv_sh[i], q);
}
}  // namespace

static inline unsigned chunks(int logn) { return (unsigned)((1L << logn) / TPB); }

void k_modup(const Tab &tab, int logn, const u64 *dc, long dcs, u64 *ext, long exts, int n_ct, int nl, int np,
             int nq_total, int alpha, const u64 *inv_hat, const u64 *inv_hat_sh, const u64 *hat, cudaStream_t st) {
    const int beta = (nl + alpha - 1) / alpha;
    if (alpha > MAXA) throw SecpeError{-1, "alpha > 16 not supported"};
    modup_kernel<<<dim3(chunks(logn), n_ct * beta), TPB, 0, st>>>(tab, logn, dc, dcs, ext, exts, nl, np, nq_total,
                                                                   alpha, beta, inv_hat, inv_hat_sh, hat);
    LAUNCH_CHECK();
}
void k_ks_inner(const Tab &tab, int logn, const u64 *d, long ds, const u64 *ext, long exts, const u64 *key,
                int nq_total, int np, u64 *acc, long accs, int n_ct, int nl, int alpha, cudaStream_t st) {
    const int beta = (nl + alpha - 1) / alpha;
    const dim3 grid(chunks(logn), nl + np);
    // 128-bit accumulation of beta products < 2^124 each requires beta <= 16 per Barrett input bound
    // (2^125); larger dnum only occurs with small primes (toy: 40-bit, products < 2^80).
    if (beta <= 4)
        ks_inner_kernel<4><<<grid, TPB, 0, st>>>(tab, logn, d, ds, ext, exts, key, nq_total, np, acc, accs, n_ct, nl,
                                                 alpha, beta);
    else if (beta <= 8)
        ks_inner_kernel<8><<<grid, TPB, 0, st>>>(tab, logn, d, ds, ext, exts, key, nq_total, np, acc, accs, n_ct, nl,
                                                 alpha, beta);
    else if (beta <= 16)
        ks_inner_kernel<16><<<grid, TPB, 0, st>>>(tab, logn, d, ds, ext, exts, key, nq_total, np, acc, accs, n_ct, nl,
                                                  alpha, beta);
    else if (beta <= 32)
        ks_inner_kernel<32><<<grid, TPB, 0, st>>>(tab, logn, d, ds, ext, exts, key, nq_total, np, acc, accs, n_ct, nl,
                                                  alpha, beta);
    else
        throw SecpeError{-1, "dnum > 32 not supported"};
    LAUNCH_CHECK();
}
void k_moddown_conv(const Tab &tab, int logn, const u64 *acc, long accs, u64 *T, long Ts, int n_ct, int nl, int np,
                    int nq_total, const u64 *ihp, const u64 *ihp_sh, const u64 *hat_p, cudaStream_t st) {
    if (np > MAXA) throw SecpeError{-1, "more than 16 special primes not supported"};
    moddown_conv_kernel<<<dim3(chunks(logn), n_ct * 2), TPB, 0, st>>>(tab, logn, acc, accs, T, Ts, nl, np, nq_total,
                                                                       ihp, ihp_sh, hat_p);
    LAUNCH_CHECK();
}
void k_moddown_combine(const Tab &tab, int logn, const u64 *acc, long accs, const u64 *T, long Ts, const u64 *add,
                       long adds, int add_polys, u64 *out, long outs, int n_ct, int nl, int ne, const u64 *pinv,
                       const u64 *pinv_sh, cudaStream_t st) {
    moddown_combine_kernel<<<dim3(chunks(logn), n_ct * 2 * nl), TPB, 0, st>>>(tab, logn, acc, accs, T, Ts, add, adds,
                                                                               add_polys, out, outs, nl, ne, pinv,
                                                                               pinv_sh);
    LAUNCH_CHECK();
}
void k_rescale_bcast(const Tab &tab, int logn, const u64 *last, long lasts, u64 *T, long Ts, int n_ct, int l,
                     const u64 *half, cudaStream_t st) {
    rescale_bcast_kernel<<<dim3(chunks(logn), n_ct * 2 * l), TPB, 0, st>>>(tab, logn, last, lasts, T, Ts, l, half);
    LAUNCH_CHECK();
}
void k_rescale_combine(const Tab &tab, int logn, CRows in, const u64 *T, long Ts, u64 *out, long outs,
                       int n_ct, int l, const u64 *qlinv, const u64 *qlinv_sh, cudaStream_t st) {
    rescale_combine_kernel<<<dim3(chunks(logn), n_ct * 2 * l), TPB, 0, st>>>(tab, logn, in, T, Ts, out, outs, l,
                                                                              qlinv, qlinv_sh);
    LAUNCH_CHECK();
}
