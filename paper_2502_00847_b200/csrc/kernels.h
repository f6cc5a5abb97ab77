// kernels.h -- launchers of the sm_100a kernels (all enqueue on the given stream).
#pragma once
#include "common.cuh"

// ---- elementwise (ops.cu) -----------------------------------------------------------------
// Polynomial P (of a batch) lives at p + (P >> 1) * cs + (P & 1) * ps: P = 2 * ct + b for
// ciphertext batches (cs = ct stride, ps = c0 -> c1 offset); a plain array of polynomials with
// stride s uses cs = 2 s, ps = s.  Row r = P * nl + limb; element (r, k) at poly + limb * N + k.
struct RowsArg {
    u64 *p;
    long cs, ps;
};
struct CRows {
    const u64 *p;
    long cs, ps;
};
SECPE_HD long poly_off(long cs, long ps, int P) { return (long)(P >> 1) * cs + (long)(P & 1) * ps; }
constexpr int MAXL = 64;  // max limbs per polynomial (n_q + n_p)
struct LimbConst {
    u64 c[MAXL];
    u64 csh[MAXL];
};

// ---- NTT (ntt.cu) -------------------------------------------------------------------------
// data: n_polys polynomials (RowsArg addressing) of lm.nl limbs each; in place unless fused.
// Fusions (all optional; the default is a plain in-place transform):
//   in_mode  1 (inverse): the first pass reads polynomial P, limb i from src (copy fused in)
//   in_mode  3 (inverse): the first pass reads src[P] * src2[P] mod q_i (tensor term fused in)
//   in_mode  4 (inverse): ... src[P] * src2[P] + src3[P] * src4[P] mod q_i (two summed tensors, R13b)
//   in_mode  5 (inverse): ... C1 src[P] + C2 src2[P] mod q_i (src2 when lin == 2; constant products, R9)
//   in_mode  2 (forward): rescale broadcast (R12): the input of limb i is
//            [floor(q_l/2)]_{q_i} - [[x + floor(q_l/2)]_{q_l}]_{q_i}, x = src row of polynomial P
//            (one coefficient-form limb, prime lp); half[i] = [floor(q_l/2)]_{q_i}
//   out_mode 1 (forward): out = (e1 + NTT(x)) * k[i]            (rescale: e1 = ciphertext, k = q_l^-1)
//   out_mode 2 (forward): out = (e1 - NTT(x)) * k[i] (+ e2 for polys with (P & 1) < e2_polys)
//            (ModDown R11: e1 = acc, k = P^-1, e2 = tensor / sigma(c0) addend)
//   k/ksh on an inverse transform: per-limb final factor replacing N^{-1} (must include it)
struct NttFusion {
    int in_mode = 0, out_mode = 0;
    CRows src{nullptr, 0, 0};
    CRows src2{nullptr, 0, 0};  // in_mode 3 (inverse): the first pass reads src[P] * src2[P] mod q (tensor d2)
    CRows src3{nullptr, 0, 0}, src4{nullptr, 0, 0};  // in_mode 4: src*src2 + src3*src4 (two summed tensors' d2)
    int lp = 0;
    const u64 *half = nullptr;
    CRows e1{nullptr, 0, 0}, e2{nullptr, 0, 0};
    int e2_polys = 0;
    CRows e3{nullptr, 0, 0};  // out_mode 2: optional addend of every polynomial (a rotation's "y + RotL(y)")
    // constant products fused into a rescale (reading R9's MULC / LINC): the rescaled value is
    // C1 src + C2 src2 instead of src (in_mode 5 on the INTT of the top limb), and the rescale epilogue
    // (out_mode 1) uses C1 e1 + C2 e1b instead of e1; lin = number of terms (0: plain)
    int lin = 0;
    i128 C1 = 0, C2 = 0;
    CRows e1b{nullptr, 0, 0};
    RowsArg out{nullptr, 0, 0};
    const u64 *k = nullptr, *ksh = nullptr;
};
void ntt_forward(const Tab &tab, int logn, RowsArg data, int n_polys, LimbMap lm, cudaStream_t st,
                 const NttFusion &f = NttFusion());
// optional profiling hook (bench.py roofline): called before (phase 0) and after (phase 1) every launch
// with the row class of the launch (FP64 or integer rows) and its algorithmic bytes; thread-local
struct NttProfHook {
    void *ctx;
    // bytes: the transform's 16 N per limb transform (split over its passes); opbytes: the operand limbs the fused
    // prologue / epilogue of this launch reads on top (tensor factors, rescale / ModDown operands, addends)
    void (*mark)(void *ctx, int phase, bool fp, double bytes, double limbs, double opbytes);
};
void ntt_set_prof_hook(const NttProfHook *h);
// several independent plain in-place transforms (each: n_polys polynomials of lm.nl limbs in d) batched
// into as few launches as possible (ntt.cu MAXSEG row ranges per launch and prime class)
struct NttSeg {
    RowsArg d;
    int n_polys;
    LimbMap lm;
};
void ntt_segments(const Tab &tab, int logn, const NttSeg *segs, int nseg, bool inverse, cudaStream_t st);
void ntt_inverse(const Tab &tab, int logn, RowsArg data, int n_polys, LimbMap lm, cudaStream_t st,
                 const NttFusion &f = NttFusion());
// persistent TMA-pipelined single-launch transform (ntt_fused.cu, N = 2^16, exact-FP64 rows) of limbs
// [limb0, limb0 + nsub) of n_polys polynomials; returns false when it does not apply (caller falls back to
// the two-pass kernels).  SECPE_NTT_FUSED=0 disables it.
bool ntt_fused_enabled();
int ntt_fused_mode(int mode);  // sets SECPE_NTT_FUSED's mode (mode < 0: query); returns the previous one
bool ntt_fused_run(const Tab &tab, int logn, RowsArg d, int n_polys, LimbMap lm, int limb0, int nsub, int cls,
                   bool inverse, const NttFusion &f, cudaStream_t st);

void k_addsub(const Tab &tab, int logn, CRows a, CRows b, RowsArg out, int n_polys, LimbMap lm,
              bool sub, cudaStream_t st);
void k_copy_rows(int logn, CRows a, RowsArg out, int n_polys, int nl, cudaStream_t st);
// out = a * c_l (Shoup, per-limb constant residues)
void k_mul_const(const Tab &tab, int logn, CRows a, RowsArg out, int n_polys, LimbMap lm,
                 const LimbConst &c, cudaStream_t st);
// out = C1 a + C2 b (b.p == nullptr: C1 a); per-limb constant residues with Shoup companions
void k_lincomb2(const Tab &tab, int logn, CRows a, CRows b, RowsArg out, int n_polys, LimbMap lm,
                const LimbConst &c1, const LimbConst &c2, cudaStream_t st);
// out = a + c_l (only the rows given)
void k_add_const(const Tab &tab, int logn, CRows a, RowsArg out, int n_polys, LimbMap lm,
                 const LimbConst &c, cudaStream_t st);
// out[p][l] = a[p][l] * b[l]  (b one polynomial, broadcast over n_polys)
void k_mul_poly(const Tab &tab, int logn, CRows a, const u64 *b, RowsArg out, int n_polys, LimbMap lm,
                cudaStream_t st);
// tensor: d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 for n_ct ciphertexts (a, b: CRows views);
// d compact: ct c, poly p at d + c*d_ct_stride + p*nl*N.  With lin (x != nullptr): d0 += C x0,
// d1 += C x1 (C per-limb residues, the planned linear term of R13)
void k_tensor(const Tab &tab, int logn, CRows a, CRows b, u64 *d, long d_ct_stride, int n_ct, int nl,
              cudaStream_t st, CRows x = CRows{nullptr, 0, 0}, const LimbConst *C = nullptr);
// linear transform accumulation (R30): out[P][l] = sum_{s<n} pt[s][l] * a_s[P][l] mod q_l, ciphertext s of
// the batch at a.p + s * as (same CRows layout), plaintext s at pt + s * pts ([l][N] rows, NTT form)
void k_mac_plain(const Tab &tab, int logn, CRows a, long as, const u64 *pt, long pts, int n, RowsArg out, int n_polys,
                 LimbMap lm, cudaStream_t st);
// automorphism in the NTT domain: out[i] = in[perm_g(i)]
void k_automorph(int logn, CRows a, RowsArg out, int n_polys, int nl, u64 galois, cudaStream_t st);

// ---- key switching (keyswitch.cu) ------------------------------------------------------------
struct KsLevel;  // per-level constants (device pointers), see context.h
// ModUp base conversion (coefficient domain, R10): for every digit j and extended limb e not in I_j:
//   ext[c][j][e] = sum_{i in I_j} y_i [Q'_j/q_i]_{t_e}  mod t_e
// dc: [n_ct][nl][N] holding y_i = [INTT(d)_i (Q'_j/q_i)^-1]_{q_i} (the factor folded into the INTT);
// ext: [n_ct][beta][ne][N]; hat: split-30 packed constants [beta][16][ne]
void k_modup(const Tab &tab, int logn, const u64 *dc, long dc_ct_stride, u64 *ext, long ext_ct_stride,
             int n_ct, int nl, int np, int nq_total, int alpha, const u64 *hat, cudaStream_t st);
// key inner product: acc[c][b][e] = sum_j X_j[e] * key_j[b][prime(e)], X_j[e] = d[c][e] if e in I_j else ext[c][j][e]
// Relinearise-and-rescale (ten != nullptr): the tensor of a and b is formed on the fly on the Q limbs:
// d2 = a1 b1 replaces d, and pmod[e] * d_b is added with d0 = a0 b0 + C x0, d1 = a0 b1 + a1 b0 + C x1
// (the optional linear term x, C of R13).
struct TensorSrc {
    CRows a, b, x;  // ciphertext views (c0 at p + ct * cs, c1 at + ps); x.p == nullptr: no linear term
    CRows a2, b2;   // optional second product a2 (x) b2 summed before the relinearisation (R13b); a2.p == nullptr: none
    LimbConst C;    // per-limb residues of the linear term's integer constant (Shoup companions)
    CRows x2;       // optional second linear term C2 x2 (x2.p == nullptr: none)
    LimbConst C2;
};
void k_ks_inner(const Tab &tab, int logn, const u64 *d, long d_ct_stride, const u64 *ext, long ext_ct_stride,
                const u64 *key, int nq_total, int np, u64 *acc, long acc_ct_stride, int n_ct, int nl,
                int alpha, cudaStream_t st, const TensorSrc *ten = nullptr, const u64 *pmod = nullptr,
                u64 galois = 1);  // galois > 1: read sigma_g(X_j) (NTT-domain gather; hoisted rotation, R29)
// Fused ModUp forward pass 2 + key inner product (relinearise-and-rescale or plain; every row of Q_l u P exact-FP64,
// q < 2^46): ext[c][j][e] holds the ModUp digits after the FIRST forward pass (ntt_segments_pass1); for every
// (ciphertext, row e, tile) the kernel runs the second pass of each digit j with e outside I_j and multiplies the
// raw transform with key_j[b][e] on the fly, then adds the tensor terms of the Q rows (d2 = a1 b1 (+ a2_1 b2_1)
// for the own digit, [P] d_b) exactly as k_ks_inner with ten -- the digits never return to HBM in NTT form.
struct KsFuse {
    const u64 *ext;
    long exts;
    const u64 *key;  // [beta][2][nq_total + np][N]
    u64 *acc;        // [n_ct][2][nl + np][N]
    long accs;
    int n_ct, nl, np, nq_total, alpha, beta;
    TensorSrc ten;    // ten.a.p == nullptr: plain key switch of d (rotations), no tensor / [P] terms
    const u64 *pmod;  // [P]_{q_e} per Q row
    const u64 *d;     // plain key switch: the switched polynomial in NTT form, ct c row e at d + c d_stride + e N
    long d_stride;
    int intt_row0;    // >= 0: rows e >= intt_row0 (the ModDown's INTT rows) also get the inverse NTT's first pass,
                      // in place (finish them with ntt_inverse_last_pass); -1: none
    int e0 = 0, e1 = 0;  // set by ntt_ks_inner: the launch's rows (one run of one prime class: FpA, FpB or integer)
};
void ntt_ks_inner(const Tab &tab, int logn, const KsFuse &f, cudaStream_t st);
// the inverse NTT's last pass only (its first pass already ran, e.g. inside ntt_ks_inner): f.k / f.ksh factors
void ntt_inverse_last_pass(const Tab &tab, int logn, RowsArg data, int n_polys, LimbMap lm, cudaStream_t st,
                           const NttFusion &f);
// ntt_segments' first forward pass only (the fused kernel above runs the second)
void ntt_segments_pass1(const Tab &tab, int logn, const NttSeg *segs, int nseg, cudaStream_t st);
// ModDown conversion (R11): T[c][b][i] = sum_{s < ns} y_s [B/s]_{q_i} mod q_i for i < nt, with
// y_s = acc[c][b][row0 + s] (coefficient form, already times (B/s)^{-1}); hatpk[s * hstride + i]
// split-30 packed
void k_moddown_conv(const Tab &tab, int logn, const u64 *acc, long acc_ct_stride, int ne, int row0, int ns, u64 *T,
                    long T_ct_stride, int nt, int n_ct, const u64 *hatpk, int hstride, cudaStream_t st);
// fused ModDown + rescale conversion (see ks.cu rr_conv_kernel): acc rows l .. l+np hold INTT(x_l) and
// the folded P-limbs; T[c][b][i] for i < l
void k_rr_conv(const Tab &tab, int logn, const u64 *acc, long acc_ct_stride, int ne, int l, int np, u64 *T,
               long T_ct_stride, int n_ct, const u64 *hatpk, const u64 *hl, u64 pinv_l, u64 pinv_l_sh,
               cudaStream_t st);

// ---- sampling / keys (sample.cu) ----------------------------------------------------------------
// ChaCha20 keys (reading R6): a 256-bit master seed, keys derived per material domain
struct Key256 {
    uint32_t w[8];
};
constexpr u64 DOM_SK = 0x5345435045534B31ULL, DOM_PK = 0x5345435045504B31ULL, DOM_ENC = 0x5345435045454E31ULL;
Key256 derive_key(const Key256 &master, u64 domain);
Key256 object_key(const Key256 &master, u64 tag);  // DOM_PK for tags of kind 2, 4 (the uniform a), else DOM_SK
Key256 os_entropy_key();                             // 32 bytes from getrandom(2)
// uniform residues in the NTT domain: out[l][k] for prime ids map (formula lm), counter layout per R6
// (N must be a multiple of 1024)
void k_sample_uniform(const Tab &tab, int logn, const Key256 &key, u64 tag, u64 *out, LimbMap lm, cudaStream_t st);
// signed small polynomial: kind 0 ternary, 1 Gaussian (cdt in constant memory)
void k_sample_small(int logn, const Key256 &key, u64 tag, int kind, i64 *out, cudaStream_t st);
// host: sparse ternary secret of Hamming weight h (reading R36), out[N]
void h_sample_sparse(const Key256 &key, u64 tag, int logn, int h, i64 *out);
void set_cdt(const u64 *cdt, int n);
// residues of a signed int64 polynomial: out[l][k] = m[k] mod q_l (coefficient form)
void k_int_to_rows(const Tab &tab, int logn, const i64 *m, u64 *out, LimbMap lm, cudaStream_t st);
// ModRaise (R33): centred lift of coefficient-form rows mod q_0 (coef[n_polys][N]) to nl limbs
void k_mod_raise(const Tab &tab, int logn, const u64 *coef, RowsArg out, int n_polys, int nl, cudaStream_t st);
// out = -a*s + e  (+ gadget * sp on limbs with gadget flag) ; all NTT form, rows lm
void k_key_combine(const Tab &tab, int logn, const u64 *a, const u64 *s, const u64 *e, const u64 *sp,
                   const LimbConst *gadget, u64 *out, LimbMap lm, cudaStream_t st);
// ct0 = v*pk0 + e0 + m, ct1 = v*pk1 + e1  (all NTT, nl limbs)
void k_encrypt_combine(const Tab &tab, int logn, const u64 *v, const u64 *pk, long pk_stride, const u64 *e0,
                       const u64 *e1, const u64 *m, u64 *ct, int nl, cudaStream_t st);
// out = c0 + c1 * s
void k_decrypt_combine(const Tab &tab, int logn, const u64 *ct, const u64 *s, u64 *out, int nl, cudaStream_t st);
// elementwise square: out = a*a
void k_square(const Tab &tab, int logn, const u64 *a, u64 *out, LimbMap lm, cudaStream_t st);
