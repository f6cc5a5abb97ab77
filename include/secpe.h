/*
 * secpe.h -- C ABI of the B200-native SecPE private-voting library (libsecpe.so).
 *
 * SecPE (arXiv 2502.00847): the server aggregates encrypted per-prompt class scores and
 * evaluates an encrypted Argmax (Sec. 3.1; Algorithm 1)
 * over packed RNS-CKKS ciphertexts (Sec. 2.2).  Every homomorphic step
 * runs in hand-written sm_100a CUDA kernels on the stream given to secpe_ctx_create /
 * secpe_set_stream.  There is no CPU fallback: without a CUDA device every call that
 * computes returns SECPE_ECUDA.
 *
 * Conventions (DESIGN.md sections 3 and 5):
 *  - N = 2^log_n; a polynomial limb is N uint64 residues in [0, q); a ciphertext at level l
 *    is uint64[2][l+1][N] (c0 limbs then c1 limbs), limb i under prime q_i, NTT (evaluation)
 *    form, NTT(a)[i] = sum_k a_k psi^{(2 brv(i)+1) k}, psi the smallest primitive 2N-th root.
 *  - Slots: N/2 complex slots, slot j <-> evaluation at zeta^{5^j mod 2N}; real scores use the
 *    real parts (reading R5).  RotL(s) uses Galois element 5^s mod 2N and
 *    RotR(s) = RotL(N/2 - s) (reading R2).
 *  - Device pointers (marked "dev") are caller-owned, 16-byte aligned, and must stay valid
 *    until the enqueued work completes.  Host pointers ("host") are read or written before
 *    the call returns.  The library never frees caller memory.  Context and keys are
 *    library-owned.  Keys are immutable after generation.  A context is NOT safe to use from
 *    several threads at once: it keeps per-context caches (captured CUDA graphs, encoded masks,
 *    auxiliary streams, host staging buffers), op counters, the op log and the profiler; use one
 *    context per thread (each with its own keys), or serialise the calls.
 *  - Calls enqueue work on the context stream and return; secpe_decrypt*, secpe_key_export,
 *    secpe_sync and the host-returning calls synchronise.
 *  - Errors: a negative status; secpe_last_error() returns a thread-local message.
 *    Nothing throws across the ABI.
 */
#ifndef SECPE_H
#define SECPE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum {
    SECPE_OK = 0,
    SECPE_EINVAL = -1,    /* bad argument / shape */
    SECPE_ELEVEL = -2,    /* not enough levels left for the requested circuit */
    SECPE_ESCALE = -3,    /* add/sub of ciphertexts whose scales are not bit-identical (reading R9) */
    SECPE_ENOKEY = -4,    /* no Galois key generated for this rotation */
    SECPE_ELAYOUT = -5,   /* slot layout does not fit / not a power of two */
    SECPE_EOVERFLOW = -6, /* an encoded value does not fit the 62-bit integer range */
    SECPE_ECUDA = -7,     /* CUDA error (including: no device) */
    SECPE_ENOMEM = -8
};

/* Rotation "step" meaning complex conjugation of the slots (reading R32): the Galois element 2N - 1
 * (X -> X^-1).  Accepted wherever a rotation step is (secpe_keygen's rot_steps, secpe_rotate). */
#define SECPE_CONJ ((int32_t)(-2147483647 - 1))

typedef struct secpe_ctx secpe_ctx;   /* opaque: parameters + device tables + stream */
typedef struct secpe_keys secpe_keys; /* opaque: secret/public/relinearisation/Galois keys (device) */

/* RNS-CKKS parameters (R_Q = Z_Q[X]/(X^N+1), Q = prod q_i). */
typedef struct {
    uint32_t log_n;     /* 12..16 */
    uint32_t n_q;       /* ciphertext primes q_0..q_L (L = n_q - 1), each in (2^32, 2^60), == 1 mod 2N (all primes,
                           special ones included: the split-30 base-conversion MACs need < 2^60) */
    const uint64_t *q;  /* host[n_q] */
    uint32_t n_p;       /* special primes for hybrid key switching (>= 1 for keys; 0 = NTT-only context) */
    const uint64_t *p;  /* host[n_p] */
    uint32_t alpha;     /* primes per key-switching digit (<= 16); dnum = ceil(n_q / alpha) <= 32; the
                           products of two primes times max(dnum, alpha, n_p) must stay < 2^125 */
    double scale;       /* nominal scale Delta used by the planner for intermediate results */
} secpe_params;

/* A ciphertext: data = dev uint64[2][level+1][N] (NTT form), scale = its CKKS scale. */
typedef struct {
    uint64_t *data;
    int32_t level;
    double scale;
} secpe_ct;

/* Composite odd Sign approximation p_r o ... o p_1 (Eq. 4).
 * degrees: host[n_stages], each 3, 7 or 15.  coeffs: host, concatenated power-basis
 * coefficients c_0..c_d of every stage (even ones must be 0). */
typedef struct {
    int32_t n_stages;
    const int32_t *degrees;
    const double *coeffs;
} secpe_sign_cfg;

/* Packed slot layout: query q, prompt p, class k -> slot q*block + p*classes + k.
 * prompts and classes powers of two; prompts*classes <= block; 2*classes <= block;
 * queries*block <= N/2. */
typedef struct {
    int32_t queries;
    int32_t prompts;
    int32_t classes;
    int32_t block;
} secpe_layout;

/* ---- context ------------------------------------------------------------------------- */
const char *secpe_last_error(void);
const char *secpe_version(void);

/* Product-side prime chain generator (reading R1): primes == 1 mod 2^(log_n+1).
 * mode 0: nearest to 2^bits, alternating above/below (closest first); mode 1: largest below
 * 2^bits, descending.  Primes in exclude (host[n_exclude]) are skipped.  out: host[count]. */
int secpe_gen_primes(uint32_t bits, uint32_t count, uint32_t log_n, int32_t mode,
                     const uint64_t *exclude, uint32_t n_exclude, uint64_t *out);

/* Build the context: twiddle/Shoup tables, CRT and base-conversion constants (device).
 * stream: a cudaStream_t (NULL = legacy default stream). */
int secpe_ctx_create(const secpe_params *prm, void *stream, secpe_ctx **out);
void secpe_ctx_destroy(secpe_ctx *ctx);
int secpe_set_stream(secpe_ctx *ctx, void *stream);
int secpe_sync(secpe_ctx *ctx);
/* host[n_q + n_p] copies of the primes and of psi (the NTT root per prime). */
int secpe_ctx_info(const secpe_ctx *ctx, uint64_t *primes_out, uint64_t *psi_out);
size_t secpe_ct_bytes(const secpe_ctx *ctx, int32_t level);

/* ---- keys (client) ---------------------------------------------------------------------
 * Randomness (reading R6): a 256-bit master seed keys ChaCha20 keystreams.  The secret material (the
 * secret s, every Gaussian error) is drawn under derive(seed, DOM_SK), the public uniform polynomials
 * (pk.a, every switching key's a) under derive(seed, DOM_PK) -- so the public and evaluation keys
 * reveal nothing about the stream the secret came from -- and encryption randomness (v, e0, e1) under
 * derive(encryption seed, DOM_ENC); derive(K, d) = first 32 bytes of ChaCha20 block 0 of key K, nonce d.
 * seed == NULL: 32 bytes of OS entropy (getrandom(2)) -- the production mode.  A seed built by
 * secpe_seed_from_u64 is TEST-ONLY (deterministic, 64 bits of entropy at most): parity tests and
 * benchmarks use it so the oracle can regenerate the same keys. */
typedef struct {
    uint8_t bytes[32];
} secpe_seed;
/* TEST-ONLY deterministic seed: bytes = little-endian u64 followed by 24 zero bytes. */
void secpe_seed_from_u64(uint64_t s, secpe_seed *out);
/* Ternary secret, public key, relinearisation key (s^2) and one Galois key per distinct rotation step in
 * rot_steps (host[n_rot]; >0 RotL, <0 RotR).  Hybrid digits (reading R7). */
int secpe_keygen(secpe_ctx *ctx, const secpe_seed *seed, const int32_t *rot_steps, int32_t n_rot,
                 secpe_keys **out);
/* As secpe_keygen with a sparse ternary secret of Hamming weight `hamming` (reading R36, the secret
 * bootstrapping uses to keep |I| and the EvalMod range K small): draw x_ctr from the secret's stream
 * for ctr = 0, 1, ...; the top log_n bits pick a coefficient; a still-zero one becomes -1 (x odd) or
 * +1; stop at `hamming` nonzeros.  hamming = 0: the uniform ternary secret of secpe_keygen.
 * SECPE_EINVAL: hamming outside [0, N]. */
int secpe_keygen_sparse(secpe_ctx *ctx, const secpe_seed *seed, int32_t hamming, const int32_t *rot_steps,
                        int32_t n_rot, secpe_keys **out);
/* Frees the key material.  Synchronises the owning context's stream and destroys every CUDA graph
 * secpe_enc_argmax captured with these keys (a later keys object at the same address never replays
 * them).  Keys may be destroyed before or after their context; null is a no-op. */
void secpe_keys_destroy(secpe_keys *keys);
/* Copy key material to host (synchronises), for parity tests.
 * which 0: secret s, NTT form over all n_q+n_p primes, uint64[n_q+n_p][N]
 *       1: public key uint64[2][n_q][N]
 *       2: relinearisation key uint64[dnum][2][n_q+n_p][N]
 *       3: Galois key of element `galois` (same shape as 2)
 * n_words must equal the shape's size. */
int secpe_key_export(const secpe_ctx *ctx, const secpe_keys *keys, int32_t which, uint64_t galois,
                     uint64_t *host_out, size_t n_words);

/* ---- encoding / encryption (client, PAPER.md:139 Step 1 and :143 Step 4) ------------------ */
/* Integer plaintext of host slots[n] (real parts, n <= N/2) at `scale`:
 * m_k = round_half_away((2 scale / N) Re sum_j z_j zeta^{-5^j k}); host out int64[N]. */
int secpe_encode(secpe_ctx *ctx, const double *slots, size_t n, double scale, int64_t *coeffs_out);
/* Encrypt the integer plaintext host coeffs[N] at `level` with the public key; out->data must
 * hold secpe_ct_bytes(level); out->level/scale are set.  seed: the encryption randomness's master seed
 * (NULL: OS entropy; never reuse one for two messages). */
int secpe_encrypt_coeffs(secpe_ctx *ctx, const secpe_keys *keys, const int64_t *coeffs,
                         int32_t level, double scale, const secpe_seed *seed, secpe_ct *out);
int secpe_encrypt(secpe_ctx *ctx, const secpe_keys *keys, const double *slots, size_t n,
                  int32_t level, double scale, const secpe_seed *seed, secpe_ct *out);
/* host out uint64[level+1][N]: residues of c0 + c1 s in coefficient form (synchronises). */
int secpe_decrypt_residues(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *ct,
                           uint64_t *host_out);
/* host slots_out[n] (real parts) = decode(centered lift of c0 + c1 s) / scale (synchronises). */
int secpe_decrypt(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *ct, double *slots_out,
                  size_t n);

/* ---- primitives (server; all device buffers) ---------------------------------------------- */
/* In-place forward / inverse negacyclic NTT of polys dev uint64[n_polys][n_limbs][N] (R4; implied by
 * PAPER.md:92, arithmetic in R_Q); limb l uses prime index first_prime + l of the chain q_0..q_L,
 * p_0..p_{k-1}; inputs canonical residues, outputs canonical.  n_polys = 0 is a no-op (polys may be
 * null).  SECPE_EINVAL: null ctx, negative n_polys, or a limb range outside the chain. */
int secpe_ntt(secpe_ctx *ctx, uint64_t *polys, int32_t n_polys, int32_t first_prime, int32_t n_limbs);
int secpe_intt(secpe_ctx *ctx, uint64_t *polys, int32_t n_polys, int32_t first_prime, int32_t n_limbs);

/* a (+) b, a (-) b.  Levels are aligned by dropping top limbs; scales must be
 * bit-identical (SECPE_ESCALE).  out may alias a or b; out level = min level. */
int secpe_add(secpe_ctx *ctx, const secpe_ct *a, const secpe_ct *b, secpe_ct *out);
int secpe_sub(secpe_ctx *ctx, const secpe_ct *a, const secpe_ct *b, secpe_ct *out);
/* Add the real constant c: round_half_away(c * scale) on every NTT point of c0. */
int secpe_add_const(secpe_ctx *ctx, const secpe_ct *a, double c, secpe_ct *out);
/* c * a landing at (target_scale, target_level) (reading R9): a is dropped to target_level+1,
 * multiplied by C = round_half_away(c * Delta_c), Delta_c = target_scale * q_{l} / scale_a,
 * then rescaled.  out level = target_level. */
int secpe_mul_const(secpe_ctx *ctx, const secpe_ct *a, double c, double target_scale,
                    int32_t target_level, secpe_ct *out);
/* a * plaintext mask (host mask_slots[n] real), quantised encoding at
 * Delta_m = target_scale * q_l / scale_a (reading R16), then rescale; out level = a.level-1. */
int secpe_mul_mask(secpe_ctx *ctx, const secpe_ct *a, const double *mask_slots, size_t n,
                   double target_scale, secpe_ct *out);
/* Drop to a lower level (exact; scale unchanged). */
int secpe_drop(secpe_ctx *ctx, const secpe_ct *a, int32_t level, secpe_ct *out);
/* PAPER.md:103 a (x) b: tensor + relinearisation (hybrid key switching, reading R10/R11), no
 * rescale.  Same level required; out scale = scale_a * scale_b.  out must not alias. */
int secpe_mul_relin(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *a, const secpe_ct *b,
                    secpe_ct *out);
/* a (x) b relinearised and rescaled in ONE pass for a batch of n pairs (the form the argmax circuit
 * uses): the ModDown conversion (R11) and the rescale conversion (R12) share one INTT/NTT round trip
 * (ks.cu rr_conv_kernel + the NTT's rescale epilogue).  Bit-identical to secpe_mul_relin followed by
 * secpe_rescale (tests/test_gpu_parity.py test_ops_bit_exact_toy).  a[i], b[i]: same level
 * l >= 1 and scale within the batch; out[i]: level l - 1, scale (S_a S_b) / q_l, sized
 * secpe_ct_bytes(l - 1), must not alias.  Contiguous batches (data[i] = data[0] + i * ct words)
 * are used in place; others are staged.  The relinearisation key is streamed once per batch. */
int secpe_mul_relin_rescale(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *a, const secpe_ct *b,
                            int32_t n, secpe_ct *out);
/* Batched secpe_rotate: n ciphertexts (same level and scale) rotated by the same step with one
 * pass over the Galois key.  out[i] must not alias in[i]. */
int secpe_rotate_batch(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n, int32_t steps,
                       secpe_ct *out);
/* Hoisted rotations (reading R29; PAPER.md:237 rotates the same ciphertext by several
 * steps): the n ciphertexts in[0..n) (same level and scale) rotated by each of steps[0..n_steps) with
 * ONE ModUp of c1 shared by all steps: for Galois element g,
 *   out = (sigma_g(c0) + ks0, ks1),  ks = ModDown(sum_j sigma_g(ModUp_j(c1)) * gk_g[j]).
 * Not the same integers as secpe_rotate (ModUp does not commute with sigma_g); the same plaintext up
 * to key-switching noise.  out is [n_steps][n], row-major: out[s * n + i] receives step s of ct i,
 * level = out[0].level (<= input level; lower drops limbs), scale = input scale; must not alias in.
 * Steps with g = 1 copy.  Errors: SECPE_ENOKEY for a missing Galois key (checked before any work),
 * SECPE_EINVAL for null arguments, n < 1 or n_steps < 1. */
int secpe_rotate_hoisted(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n,
                         const int32_t *steps, int32_t n_steps, secpe_ct *out);
/* Diagonal-form homomorphic linear transform (reading R30; the matrix-vector products that CKKS
 * bootstrapping's CoeffToSlot / SlotToCoeff are built from):
 *   out = Rescale( sum_i pt_i (.) RotL(in, steps[i]) )
 * with the rotations hoisted (one ModUp, R29).  in: one ciphertext at level l >= 1.  pts: dev
 * uint64[n][l+1][N], pt_i's NTT-form residues (an integer plaintext encoded at scale pt_scale; rows
 * 0..l used), steps: host[n] (0 = identity).  out: level l - 1, scale (in.scale * pt_scale) / q_l,
 * must not alias in.  Errors: SECPE_EINVAL (null arguments, n < 1), SECPE_ELEVEL (l < 1),
 * SECPE_ENOKEY (a step without its Galois key). */
int secpe_linear_transform(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const uint64_t *pts,
                           const int32_t *steps, int32_t n, double pt_scale, secpe_ct *out);
/* Baby-step giant-step form (reading R31): with n1 baby and n2 giant steps,
 *   out = Rescale( sum_{g<n2} RotL( sum_{j<n1} pt_{g,j} (.) RotL(in, j), g n1 ) ),
 * the baby rotations hoisted (R29), the giant rotations plain (secpe_rotate's integers), one rescale;
 * with pt_{g,j} = encode(RotR(d_{g n1 + j}, g n1)) this is sum_i d_i (.) RotL(in, i) over n1 n2 diagonals
 * with n1 + n2 - 2 rotations instead of n1 n2 - 1.  pts: dev uint64[n2][n1][l+1][N] (NTT form); Galois
 * keys needed for 1..n1-1 and n1, 2 n1, ..., (n2-1) n1.  out: level l - 1, scale (in.scale pt_scale)/q_l,
 * must not alias in.  Errors: SECPE_EINVAL, SECPE_ELEVEL (l < 1), SECPE_ENOKEY. */
int secpe_linear_transform_bsgs(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const uint64_t *pts,
                                int32_t n1, int32_t n2, double pt_scale, secpe_ct *out);
/* Rescale by q_level: round(c / q_l) (round half up, reading R12).  out level = in level - 1,
 * out scale = scale / q_l.  out must not alias. */
/* ---- bootstrapping (the paper bootstraps at L = 35) ----
 * ModRaise (reading R33): a level-0 ciphertext (c0, c1) mod q_0, read as integer polynomials with
 * centred coefficients in (-q_0/2, q_0/2], reduced mod every prime of Q_level.  It then decrypts to
 * t = m + q_0 I, I a small integer polynomial.  out: level `level` (1 <= level <= L), in's scale,
 * out->data sized secpe_ct_bytes(level), must not alias in.  SECPE_EINVAL: in not at level 0. */
int secpe_mod_raise(secpe_ctx *ctx, const secpe_ct *in, int32_t level, secpe_ct *out);
/* CKKS bootstrapping (readings R32-R35), for full slot packing (N/2 slots):
 *   ModRaise to `level`; CoeffToSlot u = M_re z, u' = M_im z (BSGS transforms, R31);
 *   x = u + conj(u), x' = u' + conj(u') (the polynomial's coefficients t_k / S and t_{k+N/2} / S);
 *   x / (K R), R = q_0 / S; d = p(x) with p ~ 2 cos((2 pi K x - pi/2) / 2^r) (power basis, degree 15);
 *   r times d <- d^2 - 2 (so d = 2 sin(2 pi t / q_0)); SlotToCoeff out = W_re d + W_im d' (BSGS).
 * The caller encodes the four matrices' diagonals (NTT form, pts[g][j] = encode(RotR(diag_{g n1 + j},
 * g n1)) as for secpe_linear_transform_bsgs): M_re = A/2, M_im = -i A/2, A[k][j] = zeta^{-5^j k} / (N/2);
 * W_re = c U, W_im = i c U, U[j][k] = zeta^{5^j k}, c = R / (4 pi).  Keys: Galois keys for 1..n1-1,
 * n1, ..., (n2-1) n1 and SECPE_CONJ.  The input must decrypt to m with |I| + |m| / q_0 <= K. */
typedef struct {
    int32_t level;           /* ModRaise target L */
    int32_t n1, n2;          /* BSGS split of the N/2 diagonals: n1 * n2 == N/2 */
    double K;                /* EvalMod range (above) */
    int32_t r;               /* double-angle steps */
    const double *poly;      /* host[16]: c_0..c_15 */
    const uint64_t *cts_re;  /* dev uint64[n2][n1][level+1][N], encoded at cts_scale */
    const uint64_t *cts_im;
    double cts_scale;
    const uint64_t *stc_re;  /* dev uint64[n2][n1][level-7-r+1][N], encoded at stc_scale */
    const uint64_t *stc_im;
    double stc_scale;
} secpe_boot_cfg;
/* Library-built bootstrapping material (the caller-side encoding above done by the library, host
 * double precision + device NTT): the polynomial = Taylor coefficients of 2 cos(a x + b), a = 2 pi K / 2^r,
 * b = -pi / 2^(r+1), and the four matrices for inputs of scale in_scale, CoeffToSlot encoded at
 * q_level, SlotToCoeff at q_{level-7-r}.  Device memory: 2 n1 n2 ((level + 1) + (level - 6 - r)) N words.
 * secpe_boot_get_cfg fills *cfg with pointers into it (valid until secpe_boot_destroy).
 * Errors: SECPE_EINVAL (n1 n2 != N/2, K <= 0, r outside [0, 30]), SECPE_ELEVEL, SECPE_EOVERFLOW. */
typedef struct secpe_boot secpe_boot;
int secpe_boot_create(secpe_ctx *ctx, int32_t level, double K, int32_t r, int32_t n1, int32_t n2, double in_scale,
                      secpe_boot **out);
int secpe_boot_get_cfg(const secpe_boot *boot, secpe_boot_cfg *cfg);
/* Synchronises the owning context's stream and drops the CUDA graphs that read the material; may run
 * before or after the context's destruction; null is a no-op. */
void secpe_boot_destroy(secpe_boot *boot);
/* Copy matrix `which` (0 cts_re, 1 cts_im, 2 stc_re, 3 stc_im) to host uint64[n2][n1][limbs][N], for
 * parity tests (synchronises); n_words must equal that size. */
int secpe_boot_export(secpe_ctx *ctx, const secpe_boot *boot, int32_t which, uint64_t *host_out, size_t n_words);
/* Factorised bootstrapping (reading R37; what N = 2^16 needs): the decoding matrix U is the product of
 * log2(N/2) special-FFT butterfly stages S_s (3 slot-domain diagonals each: offsets 0, +-2^(s-1)); the
 * caller groups consecutive stages and each group becomes one hoisted diagonal transform (R30, one level).
 * CoeffToSlot applies the inverse groups (slots end up holding the coefficients in bit-reversed order,
 * invisible to the slot-wise EvalMod), its last group in a Re (x 1/2) and an Im (x -i/2) variant;
 * SlotToCoeff applies its first group to d_re (x c) and d_im (x i c), sums, then the other groups.
 * Depth 2 n_groups + 6 + r.  A stage: n_diag signed rotation steps (ascending) and pts dev
 * uint64[n_diag][stage level + 1][N] (NTT form, encoded at pt_scale); CoeffToSlot stage i sits at
 * level - i, SlotToCoeff stage j at level - n_cts - 6 - r - j. */
typedef struct {
    int32_t n_diag;
    const int32_t *steps;   /* host[n_diag] */
    const uint64_t *pts;    /* dev */
    double pt_scale;
    /* baby-step giant-step form (reading R39) when n_giant > 0: steps / n_diag unused, pts dev
     * uint64[n_giant][n_baby][stage level + 1][N] with pts[g][j] = encode(RotR(d_{baby_j + giant_g}, giant_g))
     * (zero where no diagonal); out = Rescale(sum_g RotL(sum_j pts[g][j] (.) RotL(x, baby_j), giant_g)) */
    int32_t n_baby;
    const int32_t *baby;    /* host[n_baby] */
    int32_t n_giant;
    const int32_t *giant;   /* host[n_giant] */
} secpe_lt_stage;
typedef struct {
    int32_t level;
    double K;
    int32_t r;
    const double *poly;            /* host[16] */
    int32_t n_cts;                 /* == n_stc */
    const secpe_lt_stage *cts;     /* host[n_cts]; cts[n_cts-1] is the Re variant of the last group */
    secpe_lt_stage cts_im;
    int32_t n_stc;
    const secpe_lt_stage *stc;     /* host[n_stc]; stc[0] is the Re variant of the first group */
    secpe_lt_stage stc_im;
} secpe_boot_fft_cfg;
int secpe_bootstrap_fft(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const secpe_boot_fft_cfg *cfg,
                        secpe_ct *out);
/* Library-built factorised material: groups host[n_groups] (stage counts, S_1 first, summing to
 * log2(N/2)); same polynomial and scales as secpe_boot_create; bsgs != 0: every group in baby-step
 * giant-step form (R39: n1 = the power of two >= sqrt(#diagonals) baby steps, about as many giant steps). */
int secpe_boot_create_fft(secpe_ctx *ctx, int32_t level, double K, int32_t r, const int32_t *groups,
                          int32_t n_groups, double in_scale, int32_t bsgs, secpe_boot **out);
/* Bootstrap with library-built material of either kind; out->data sized for level - secpe_boot_levels.
 * Factorised material on a non-default context stream: the call is captured as a CUDA graph the second
 * time the same (in, out, scale, material, keys) are seen and replayed afterwards (as secpe_enc_argmax);
 * secpe_boot_destroy and secpe_keys_destroy drop such graphs.  secpe_enc_argmax_boot does the same on
 * unstaged (contiguous) input and output batches. */
int secpe_bootstrap_boot(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const secpe_boot *boot,
                         secpe_ct *out);
/* A batch of n level-0 ciphertexts (one level and scale) through one bootstrap plan (every key and
 * transform plaintext read once per op for the batch; one ciphertext does not fill the GPU): in / out
 * host[n] as secpe_enc_argmax; factorised material only (SECPE_EINVAL otherwise: loop over
 * secpe_bootstrap_boot for dense material); no output may overlap any input (byte ranges checked);
 * CUDA graph as above on unstaged buffers. */
int secpe_bootstrap_boot_batch(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n,
                               const secpe_boot *boot, secpe_ct *out);
/* Rotation steps (SECPE_CONJ included) whose Galois keys a library-built bootstrap needs, ascending with
 * SECPE_CONJ last; returns their count, writes min(count, cap) of them to steps (may be null). */
int32_t secpe_boot_steps(const secpe_boot *boot, int32_t *steps, int32_t cap);
/* Depth of a library-built bootstrap; *raise_level (optional) receives its ModRaise level. */
int32_t secpe_boot_levels(const secpe_boot *boot, int32_t *raise_level);
/* A factorised stage for parity tests: kind 0 cts[idx], 1 cts_im, 2 stc[idx], 3 stc_im.  Writes *n_diag;
 * when steps / host_out are non-null also the steps and the pts (uint64[n_diag][limbs][N], n_words). */
int secpe_boot_stage_export(secpe_ctx *ctx, const secpe_boot *boot, int32_t kind, int32_t idx, int32_t *n_diag,
                            int32_t *steps, uint64_t *host_out, size_t n_words);
/* The same for a baby-step giant-step stage: *n_baby, *n_giant, and (when non-null) the steps and the pts
 * (uint64[n_giant][n_baby][limbs][N], n_words). */
int secpe_boot_stage_export_bsgs(secpe_ctx *ctx, const secpe_boot *boot, int32_t kind, int32_t idx, int32_t *n_baby,
                                 int32_t *n_giant, int32_t *baby, int32_t *giant, uint64_t *host_out, size_t n_words);
/* SURVEY 8(f) N4 (reading R38): secpe_enc_argmax (Algorithm 1) for layouts whose
 * comparisons do not fit the level budget (K = 16: four Max steps + the final Sign), refreshing with a
 * factorised bootstrap: before a Max when fewer than sign_depth + 2 levels remain (one is kept for the
 * next refresh) and before the final Sign when fewer than sign_depth remain.  A refresh is a constant
 * product by 1 onto level 0 at boot_scale (the input scale the bootstrap material was built for), the
 * bootstrap, and a constant product by 1 back to the context's nominal scale.  The batch runs as one
 * plan (every key and transform plaintext read once per op for all of it).  prompt_cts >= 1: the prompts
 * of one query set are spread over prompt_cts ciphertexts (CLIP-scale prompt counts),
 * in[g * prompt_cts + i] = member i of group g, all in the same layout; H1 first sums each group in member
 * order and the mask normalises by layout->prompts x prompt_cts.  n_in = groups x
 * prompt_cts inputs (one level and scale); out: host[groups].  Errors: SECPE_ELEVEL when a refresh cannot
 * fit, SECPE_ENOKEY, SECPE_EINVAL, SECPE_ELAYOUT. */
int secpe_argmax_boot_info(secpe_ctx *ctx, const secpe_layout *layout, const secpe_sign_cfg *cfg,
                           const secpe_boot *boot, int32_t in_level, int32_t *out_level);
int secpe_enc_argmax_boot(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n_in,
                          int32_t prompt_cts, const secpe_layout *layout, const secpe_sign_cfg *cfg,
                          const secpe_boot *boot, double boot_scale, secpe_ct *out);
/* The same with caller-encoded factorised material (parity tests). */
int secpe_enc_argmax_boot_cfg(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n_in,
                              int32_t prompt_cts, const secpe_layout *layout, const secpe_sign_cfg *cfg,
                              const secpe_boot_fft_cfg *bcfg, double boot_scale, secpe_ct *out);
/* Levels one bootstrap consumes (8 + r): out level = cfg->level - secpe_boot_depth(cfg). */
int32_t secpe_boot_depth(const secpe_boot_cfg *cfg);
/* in: level 0; out->data sized secpe_ct_bytes(cfg->level - secpe_boot_depth(cfg)); out->level / scale
 * set.  Errors: SECPE_EINVAL (shape, n1 n2 != N/2, level), SECPE_ENOKEY (a missing Galois key). */
int secpe_bootstrap(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const secpe_boot_cfg *cfg,
                    secpe_ct *out);

int secpe_rescale(secpe_ctx *ctx, const secpe_ct *in, secpe_ct *out);
/* PAPER.md:104-105 RotL(a, steps) (steps < 0: RotR(a, -steps)).  out must not alias. */
int secpe_rotate(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t steps,
                 secpe_ct *out);

/* ---- SecPE circuits --------------------------------------------------------------------- */
/* Composite Sign (Eq. 3-4) with the fixed BSGS plan of reading R13;
 * out level = in level - secpe_sign_depth(cfg); out scale = target_scale. */
/* Levels the plan of reading R13 consumes: the sum over stages of 2 (degree 3), 3 (degree 7) or 5
 * (degree 15, Paterson-Stockmeyer: x, x^2, x^3, x^4, x^8 then two giant products); 13 for (7, 15, 15).
 * Returns < 0 (SECPE_EINVAL) for an unsupported configuration. */
int32_t secpe_sign_depth(const secpe_sign_cfg *cfg);
int secpe_sign_poly(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in,
                    const secpe_sign_cfg *cfg, double target_scale, secpe_ct *out);
/* Level and scale of secpe_enc_argmax's outputs for inputs at in_level. */
int secpe_argmax_info(secpe_ctx *ctx, const secpe_layout *layout, const secpe_sign_cfg *cfg,
                      int32_t in_level, int32_t *out_level, double *out_scale);
/* SecPE private voting (PAPER.md:141-142 + Algorithm 1) on n_in packed ciphertexts:
 * aggregate prompts by rotate-and-sum, mask/normalise (Eq. 5), duplicate, QuickMax with
 * Eq. 6, Sign(y - y_max) + 1 (Eq. 2).  in: host[n_in] ciphertexts (same level and scale);
 * out: host[n_in], out[i].data sized for the level secpe_argmax_info reports.  The batch is
 * evaluated together so every key is read once per op for all n_in ciphertexts, as up to two
 * concurrent sub-batches on context-owned streams.  On a non-default context stream the call is
 * captured as a CUDA graph the second time the same (buffers, level, layout, Sign, keys) are seen and
 * replayed from the third time on (at most 16 graphs per context, oldest evicted; secpe_keys_destroy
 * drops the graphs of its keys).  No secret key is taken or needed.  No output ciphertext may overlap
 * any input ciphertext (the two sub-batches run concurrently; checked on the byte ranges).
 * Errors: SECPE_EINVAL (null arguments, n_in < 1, mixed levels/scales, overlapping in/out), SECPE_ELAYOUT, SECPE_ELEVEL
 * (not enough levels, e.g. K = 16 with the (7,15,15) Sign at L = 29), SECPE_ENOKEY, SECPE_ECUDA. */
int secpe_enc_argmax(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n_in,
                     const secpe_layout *layout, const secpe_sign_cfg *cfg, secpe_ct *out);
/* secpe_enc_argmax on ciphertexts held in HOST memory (the end-to-end server call).
 * h_in: uint64[n_in][2][level+1][N] (ciphertext i at h_in + i * secpe_ct_bytes(level) / 8, all at
 * `level` and `scale`); h_out: uint64[n_in][2][out_level+1][N], out_level / out_scale as
 * secpe_argmax_info reports (written to *out_level / *out_scale when non-null).  The batch runs
 * in chunks of `chunk` ciphertexts (<= 0: 16) through two device staging slots owned by the
 * context: the host-to-device copy of a chunk runs on a context-owned copy stream while the
 * previous chunk (possibly of the previous call) computes; each result is copied back on the
 * context stream.  Pinned host memory gives overlapped transfers (pageable memory is correct
 * but copies synchronously).  Enqueue-only: h_out is complete, and h_in may be reused, after
 * secpe_sync(ctx).  Needs an explicit (non-default) context stream (else SECPE_EINVAL). */
int secpe_enc_argmax_host(secpe_ctx *ctx, const secpe_keys *keys, const uint64_t *h_in, int32_t n_in,
                          int32_t level, double scale, const secpe_layout *layout,
                          const secpe_sign_cfg *cfg, uint64_t *h_out, int32_t chunk,
                          int32_t *out_level, double *out_scale);

/* ---- instrumentation ---------------------------------------------------------------------- */
/* Enable (1) / disable (0) the planned-op log; secpe_oplog_get copies it (NUL-terminated)
 * into host buf[cap] and returns its full length; secpe_oplog_clear empties it. */
int secpe_oplog_enable(secpe_ctx *ctx, int32_t on);
int64_t secpe_oplog_get(secpe_ctx *ctx, char *buf, size_t cap);
int secpe_oplog_clear(secpe_ctx *ctx);
/* CUDA-event profile of the NTT launches and the key-switch and rescale spans enqueued between begin
 * and end (events recorded on the context stream around each span; end synchronises).  out[12]:
 * per kind k (0 NTT launches on FP64 rows (primes < 2^46), 1 key switch, 2 rescale, 3 NTT launches
 * on integer rows): out[3k] total ms, out[3k+1] algorithmic bytes (NTT: 16 N per limb transform,
 * split evenly over its passes; key switch: (input + output limbs) per ciphertext + key once per
 * batch; rescale: 2(l+1) + 2l limbs per ciphertext), out[3k+2] units (limb transforms per launch,
 * summed / ciphertexts).  With n_out >= 27 also the argmax circuit stages as kinds 4..8 (H1
 * aggregation, H2 mask, H3 duplication, H4 QuickMax incl. its Sign, H6 final Sign + 1; ms in
 * out[3k], ciphertexts in out[3k+2]).  With n_out >= 30 also kind 9: the operand bytes the fused
 * prologues / epilogues of the FP64-row NTT launches read on top of their transforms (tensor factors,
 * rescale and ModDown operands, addends; out[28]), timed over the same launches (out[27]).
 * Returns SECPE_EINVAL when n_out < 12. */
int secpe_profile_begin(secpe_ctx *ctx);
int secpe_profile_end(secpe_ctx *ctx, double *out, int32_t n_out);
/* Development switch of the N = 2^16 exact-FP64 NTT implementation (process-wide; SECPE_NTT_FUSED sets the
 * initial value): 0 = the two-pass kernels everywhere, 1 = the persistent TMA-pipelined single-launch kernel
 * (ntt_fused.cu) for every exact-FP64 run, 2 (default) = the fused kernel for plain transforms of >= 1024
 * limb rows only.  Both give identical words.  mode < 0 queries.  Returns the previous mode. */
int32_t secpe_ntt_mode(int32_t mode);
/* host counts[8]: NTT limb-transforms, key switches, rescales, rotations, ct-ct products,
 * constant products, kernel launches, Sign evaluations. */
int secpe_opcounts(secpe_ctx *ctx, int64_t *counts, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif
