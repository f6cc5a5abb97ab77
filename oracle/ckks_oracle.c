/*
 * ckks_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the RNS-CKKS integer
 * arithmetic that SecPE's private voting step runs on (Sec. 2.2;
 * PAPER.md:141-142, Sec. 3.1 step 3; Algorithm 1).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code, header, table or
 * constant generator with paper_2502_00847_b200/ (the CUDA product path).
 *
 * Conventions followed literally (readings listed in DESIGN.md section 3):
 *   - every residue is canonical in [0, q); products use (unsigned __int128)a*b % q
 *     (no Barrett, Shoup, Montgomery or lazy reduction anywhere in this file);
 *   - NTT(a)[i] = sum_k a_k psi^{(2 brv(i) + 1) k} mod q  (bit-reversed evaluation
 *     order), psi = the smallest primitive 2N-th root of unity mod q;
 *     computed as  twist by psi^k  ->  textbook radix-2 cyclic DFT with omega = psi^2
 *     ->  read out in bit-reversed order;
 *   - sampler: ChaCha20 keystreams keyed by keys derived from a 256-bit master seed (R6);
 *   - key switching: hybrid, consecutive alpha-prime digits, ModDown without
 *     rounding correction (readings R10/R11);
 *   - rescale: round-half-up division by the last prime (R12);
 *   - rotation: sigma_g on coefficients X^k -> +-X^{kg mod 2N}, not hoisted.
 *
 * Parallelism: plain `omp parallel for` over independent limbs only; every
 * per-limb computation is sequential and identical with or without OpenMP.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;

/* thread control for the timed CPU baseline (bench.py): n > 0 sets the OpenMP team size; returns the
 * number of threads a parallel region actually runs with */
int o_set_threads(int n) {
    if (n > 0) omp_set_num_threads(n);
    int t = 1;
#pragma omp parallel
    {
#pragma omp single
        t = omp_get_num_threads();
    }
    return t;
}

/* ------------------------------------------------------------------ */
/* O-2 modular arithmetic: residues in [0,q), plain % reduction        */
/* ------------------------------------------------------------------ */
static inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static inline u64 addmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + b) % q); }
static inline u64 submod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + q - b) % q); }
static u64 powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}
/* inverse by Fermat (q prime) */
static u64 invmod(u64 a, u64 q) { return powmod(a % q, q - 2, q); }
/* signed integer -> residue */
static inline u64 smod(i64 v, u64 q) {
    if (v >= 0) return (u64)v % q;
    u64 m = ((u64)(-(v + 1)) + 1) % q; /* |v| mod q without overflow */
    return m ? q - m : 0;
}

/* signed 128-bit integer C = c_hi 2^64 + c_lo (two's complement) -> residue: the plan's constants
   C = rha(c Delta_c) pass 2^63 once Delta_c ~ q ~ 2^49 and |c| ~ 2^15 (the Sign coefficients) */
static inline u64 smod_wide(i64 c_hi, u64 c_lo, u64 q) {
    u128 v = ((u128)(u64)c_hi << 64) | c_lo;
    if (c_hi >= 0) return (u64)(v % q);
    u64 m = (u64)((~v + 1) % q); /* |C| mod q */
    return m ? q - m : 0;
}

u64 o_mulmod(u64 a, u64 b, u64 q) { return mulmod(a, b, q); }
u64 o_powmod(u64 a, u64 e, u64 q) { return powmod(a, e, q); }

/* ------------------------------------------------------------------ */
/* O-1 primes: deterministic Miller-Rabin with bases 2..37             */
/* ------------------------------------------------------------------ */
int o_is_prime(u64 n) {
    static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    u64 d = n - 1;
    int r = 0;
    while ((d & 1) == 0) { d >>= 1; r++; }
    for (int i = 0; i < 12; i++) {
        u64 x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int k = 1; k < r; k++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

static int excluded(u64 c, const u64 *ex, int nex) {
    for (int i = 0; i < nex; i++) if (ex[i] == c) return 1;
    return 0;
}

/*
 * Prime chain generator (reading R1 in DESIGN.md).
 * Candidates are c = 2^bits + 1 + k*2N (so c == 1 mod 2N).
 * mode 0 ("nearest"): visit candidates by increasing |c - 2^bits|, i.e.
 *         k = 0, -1, +1, -2, +2, ...  (above first on the k=0 / k=-1 tie: 1 < 2N-1).
 * mode 1 ("below"):   k = -1, -2, -3, ...  (largest primes below 2^bits, descending).
 * Primes listed in `ex` are skipped.  Returns the number written (== count on success).
 */
int o_gen_primes(int bits, int count, u64 two_n, int mode, const u64 *ex, int nex, u64 *out) {
    u64 base = ((u64)1) << bits;
    int got = 0;
    if (mode == 0) {
        for (u64 k = 0; got < count && k < (u64)1 << 40; k++) {
            /* k-th step of the alternating walk: above(k) then below(k+1) */
            u64 above = base + 1 + k * two_n;
            if (o_is_prime(above) && !excluded(above, ex, nex)) out[got++] = above;
            if (got >= count) break;
            u64 below = base + 1 - (k + 1) * two_n;
            if (o_is_prime(below) && !excluded(below, ex, nex)) out[got++] = below;
        }
    } else {
        for (u64 k = 1; got < count && k < (u64)1 << 40; k++) {
            u64 c = base + 1 - k * two_n;
            if (o_is_prime(c) && !excluded(c, ex, nex)) out[got++] = c;
        }
    }
    return got;
}

/*
 * O-3: psi = the smallest x in [2, q) with x^N == -1 (mod q), i.e. the smallest
 * primitive 2N-th root of unity.  Any primitive root r gives all of them as
 * r^(2j+1), j < N; we enumerate that set and take its minimum.
 */
u64 o_find_psi(u64 q, int logn) {
    u64 n = (u64)1 << logn, two_n = n << 1;
    u64 r = 0;
    for (u64 g = 2; g < q; g++) {
        u64 x = powmod(g, (q - 1) / two_n, q);
        if (powmod(x, n, q) == q - 1) { r = x; break; }
    }
    if (!r) return 0;
    u64 r2 = mulmod(r, r, q), cur = r, best = r;
    for (u64 j = 0; j < n; j++) {
        if (cur < best) best = cur;
        cur = mulmod(cur, r2, q);
    }
    return best;
}

/* ------------------------------------------------------------------ */
/* O-3 negacyclic NTT by definition                                    */
/* ------------------------------------------------------------------ */
static inline u64 brv(u64 x, int bits) {
    u64 r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* textbook iterative radix-2 cyclic DFT, natural order in and out:
   A[u] = sum_k a[k] w^{uk}, w a primitive n-th root of unity mod q */
static void cyclic_dft(u64 *a, int logn, u64 q, u64 w) {
    u64 n = (u64)1 << logn;
    for (u64 i = 0; i < n; i++) {
        u64 j = brv(i, logn);
        if (i < j) { u64 t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    for (u64 len = 2; len <= n; len <<= 1) {
        u64 wl = powmod(w, n / len, q);
        for (u64 s = 0; s < n; s += len) {
            u64 wk = 1;
            for (u64 j = 0; j < len / 2; j++) {
                u64 u = a[s + j], v = mulmod(a[s + j + len / 2], wk, q);
                a[s + j] = addmod(u, v, q);
                a[s + j + len / 2] = submod(u, v, q);
                wk = mulmod(wk, wl, q);
            }
        }
    }
}

/* NTT(a)[i] = sum_k a_k psi^{(2 brv(i)+1) k}: twist, cyclic DFT with omega = psi^2, bit-reverse read-out */
void o_ntt(u64 *a, int logn, u64 q, u64 psi) {
    u64 n = (u64)1 << logn;
    u64 *b = (u64 *)malloc(n * sizeof(u64));
    u64 pk = 1;
    for (u64 k = 0; k < n; k++) { b[k] = mulmod(a[k] % q, pk, q); pk = mulmod(pk, psi, q); }
    cyclic_dft(b, logn, q, mulmod(psi, psi, q));
    for (u64 i = 0; i < n; i++) a[i] = b[brv(i, logn)];
    free(b);
}

/* exact inverse of o_ntt */
void o_intt(u64 *a, int logn, u64 q, u64 psi) {
    u64 n = (u64)1 << logn;
    u64 *b = (u64 *)malloc(n * sizeof(u64));
    for (u64 u = 0; u < n; u++) b[u] = a[brv(u, logn)] % q;
    u64 psi_inv = invmod(psi, q);
    cyclic_dft(b, logn, q, mulmod(psi_inv, psi_inv, q));
    u64 ninv = invmod(n % q, q), pk = ninv;
    for (u64 k = 0; k < n; k++) { a[k] = mulmod(b[k], pk, q); pk = mulmod(pk, psi_inv, q); }
    free(b);
}

/* O(N^2) evaluation of the definition, for pins at small N */
void o_ntt_naive(const u64 *a, u64 *out, int logn, u64 q, u64 psi) {
    u64 n = (u64)1 << logn;
    for (u64 i = 0; i < n; i++) {
        u64 e = 2 * brv(i, logn) + 1, x = powmod(psi, e, q), xk = 1, acc = 0;
        for (u64 k = 0; k < n; k++) { acc = addmod(acc, mulmod(a[k] % q, xk, q), q); xk = mulmod(xk, x, q); }
        out[i] = acc;
    }
}

/* batched helpers: polys laid out [nl][N], limb l uses prime primes[pid[l]] */
void o_ntt_limbs(u64 *a, int logn, int nl, const u64 *primes, const u64 *psis, const int *pid) {
    u64 n = (u64)1 << logn;
#pragma omp parallel for schedule(dynamic, 1)
    for (int l = 0; l < nl; l++) o_ntt(a + (u64)l * n, logn, primes[pid[l]], psis[pid[l]]);
}
void o_intt_limbs(u64 *a, int logn, int nl, const u64 *primes, const u64 *psis, const int *pid) {
    u64 n = (u64)1 << logn;
#pragma omp parallel for schedule(dynamic, 1)
    for (int l = 0; l < nl; l++) o_intt(a + (u64)l * n, logn, primes[pid[l]], psis[pid[l]]);
}

/* ------------------------------------------------------------------ */
/* O-6 sampler: ChaCha20 keystreams (R6)                     */
/* ------------------------------------------------------------------ */
typedef uint32_t u32;
static inline u32 rotl32(u32 x, int r) { return (x << r) | (x >> (32 - r)); }
#define QR(a, b, c, d)                          \
    a += b; d ^= a; d = rotl32(d, 16);          \
    c += d; b ^= c; b = rotl32(b, 12);          \
    a += b; d ^= a; d = rotl32(d, 8);           \
    c += d; b ^= c; b = rotl32(b, 7);
/* the ChaCha20 block function (Bernstein's layout: words 12-13 a 64-bit block counter, 14-15 a 64-bit
 * nonce): 20 rounds on the state, then the input state added word by word */
void o_chacha20_block(const u32 *key, u64 counter, u64 nonce, u32 *out) {
    u32 x[16], in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u};
    for (int i = 0; i < 8; i++) in[4 + i] = key[i];
    in[12] = (u32)counter; in[13] = (u32)(counter >> 32);
    in[14] = (u32)nonce; in[15] = (u32)(nonce >> 32);
    for (int i = 0; i < 16; i++) x[i] = in[i];
    for (int r = 0; r < 10; r++) {
        QR(x[0], x[4], x[8], x[12]) QR(x[1], x[5], x[9], x[13])
        QR(x[2], x[6], x[10], x[14]) QR(x[3], x[7], x[11], x[15])
        QR(x[0], x[5], x[10], x[15]) QR(x[1], x[6], x[11], x[12])
        QR(x[2], x[7], x[8], x[13]) QR(x[3], x[4], x[9], x[14])
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + in[i];
}
/* key derivation: the first 8 words of the block (master, counter 0, nonce domain) */
void o_derive(const u32 *master, u64 domain, u32 *out) {
    u32 w[16];
    o_chacha20_block(master, 0, domain, w);
    for (int i = 0; i < 8; i++) out[i] = w[i];
}
/* stream (key, tag): draw ctr is the 64-bit word (w[2j], w[2j+1]) of block ctr / 8, j = ctr mod 8 */
u64 o_draw(const u32 *key, u64 tag, u64 ctr) {
    u32 w[16];
    o_chacha20_block(key, ctr >> 3, tag, w);
    int j = (int)(ctr & 7);
    return (u64)w[2 * j] | ((u64)w[2 * j + 1] << 32);
}
/* the same draws with the last block kept (sequential callers) */
typedef struct { const u32 *key; u64 tag, blk; u32 w[16]; } OStream;
static void os_init(OStream *s, const u32 *key, u64 tag) { s->key = key; s->tag = tag; s->blk = ~(u64)0; }
static u64 os_draw(OStream *s, u64 ctr) {
    if ((ctr >> 3) != s->blk) { s->blk = ctr >> 3; o_chacha20_block(s->key, s->blk, s->tag, s->w); }
    int j = (int)(ctr & 7);
    return (u64)s->w[2 * j] | ((u64)s->w[2 * j + 1] << 32);
}
/* object tags */
u64 o_tag(u64 kind, u64 g, u64 j) { return (kind << 48) ^ (g << 8) ^ j; }
/* key domains (nonces of o_derive): secret material (s, e), public material (the uniform a), encryption */
#define DOM_SK 0x5345435045534B31ULL
#define DOM_PK 0x5345435045504B31ULL
#define DOM_ENC 0x5345435045454E31ULL
static int kind_public(u64 tag) { u64 k = tag >> 48; return k == 2 || k == 4; }

/* uniform residue mod q for prime index t, coefficient k: floor(X*q / 2^128), X = draws 2c || 2c+1 */
static u64 uniform_from(u64 xh, u64 xl, u64 q) {
    u128 p1 = (u128)xl * q;
    u128 p2 = (u128)xh * q + (u64)(p1 >> 64);
    return (u64)(p2 >> 64);
}
u64 o_uniform(const u32 *key, u64 tag, u64 t, u64 k, int logn, u64 q) {
    u64 ctr = 2 * ((t << logn) + k);
    return uniform_from(o_draw(key, tag, ctr), o_draw(key, tag, ctr + 1), q);
}
/* uniform polynomial, sampled directly in the NTT domain, limbs [nl][N] for primes pid[] */
void o_sample_uniform(const u32 *key, u64 tag, int logn, int nl, const u64 *primes, const int *pid, u64 *out) {
    u64 n = (u64)1 << logn;
#pragma omp parallel for
    for (int l = 0; l < nl; l++) {
        OStream st;
        os_init(&st, key, tag);
        for (u64 k = 0; k < n; k++) {
            u64 ctr = 2 * (((u64)pid[l] << logn) + k);
            out[(u64)l * n + k] = uniform_from(os_draw(&st, ctr), os_draw(&st, ctr + 1), primes[pid[l]]);
        }
    }
}
/* ternary: v = floor(x*3 / 2^64) in {0,1,2} -> {0, 1, -1} */
void o_sample_ternary(const u32 *key, u64 tag, int logn, i64 *out) {
    u64 n = (u64)1 << logn;
    OStream st;
    os_init(&st, key, tag);
    for (u64 k = 0; k < n; k++) {
        u64 x = os_draw(&st, k);
        u64 v = (u64)(((u128)x * 3) >> 64);
        out[k] = v == 0 ? 0 : (v == 1 ? 1 : -1);
    }
}
/* sparse ternary secret of Hamming weight h (reading R36, bootstrapping's sparse secret): draw
 * x_ctr for ctr = 0, 1, ...; position = top logn bits of x; if that coefficient is still 0 it becomes
 * -1 when x is odd, else +1; stop after h nonzeros.  out must be zeroed; h <= N. */
void o_sample_sparse(const u32 *key, u64 tag, int logn, int h, i64 *out) {
    int cnt = 0;
    OStream st;
    os_init(&st, key, tag);
    for (u64 ctr = 0; cnt < h; ctr++) {
        u64 x = os_draw(&st, ctr);
        u64 pos = x >> (64 - logn);
        if (out[pos] == 0) {
            out[pos] = (x & 1) ? -1 : 1;
            cnt++;
        }
    }
}
/* discrete Gaussian via CDT: sign = top bit, u = low 63 bits, |e| = min{m : u < T[m]} */
void o_sample_gauss(const u32 *key, u64 tag, int logn, const u64 *cdt, int ncdt, i64 *out) {
    u64 n = (u64)1 << logn;
    OStream st;
    os_init(&st, key, tag);
    for (u64 k = 0; k < n; k++) {
        u64 x = os_draw(&st, k);
        u64 u = x & 0x7FFFFFFFFFFFFFFFULL;
        i64 m = 0;
        while (m < ncdt - 1 && u >= cdt[m]) m++;
        out[k] = (x >> 63) ? -m : m;
    }
}

/* ------------------------------------------------------------------ */
/* context + CKKS operations                                           */
/* ------------------------------------------------------------------ */
typedef struct {
    int logn;
    int nq;       /* number of ciphertext primes q_0..q_{nq-1} (top level L = nq-1) */
    int np;       /* number of special primes p_0..p_{np-1} */
    int alpha;    /* primes per key-switching digit */
    const u64 *primes; /* nq + np: q_0..q_{L}, p_0..p_{k-1} */
    const u64 *psi;    /* nq + np */
} OCtx;

#define NN(c) ((u64)1 << (c)->logn)

/* signed integer polynomial -> NTT residues for prime ids pid[0..nl) */
void o_int_to_ntt(const OCtx *c, const i64 *m, int nl, const int *pid, u64 *out) {
    u64 n = NN(c);
#pragma omp parallel for
    for (int l = 0; l < nl; l++) {
        u64 q = c->primes[pid[l]];
        for (u64 k = 0; k < n; k++) out[(u64)l * n + k] = smod(m[k], q);
        o_ntt(out + (u64)l * n, c->logn, q, c->psi[pid[l]]);
    }
}

static int *ids_range(int a, int cnt) {
    int *p = (int *)malloc(sizeof(int) * (cnt > 0 ? cnt : 1));
    for (int i = 0; i < cnt; i++) p[i] = a + i;
    return p;
}

/* O-7 public key: pk = (-a s + e, a) over Q_L, a uniform (NTT domain), e Gaussian */
/* the key of object `tag`'s stream under the 256-bit master seed: public-material objects (the uniform
 * a of pk and of every switching key) use derive(master, DOM_PK), all others derive(master, DOM_SK) */
void o_object_key(const u32 *master, u64 tag, u32 *out) { o_derive(master, kind_public(tag) ? DOM_PK : DOM_SK, out); }
void o_encrypt_key(const u32 *master, u32 *out) { o_derive(master, DOM_ENC, out); }

void o_keygen_pk(const OCtx *c, const u32 *master, const u64 *s_ntt, const u64 *cdt, int ncdt, u64 *pk) {
    u64 n = NN(c);
    int nq = c->nq;
    int *pid = ids_range(0, nq);
    u64 *a = pk + (u64)nq * n;
    u32 kp[8], ks[8];
    o_object_key(master, o_tag(2, 0, 0), kp);
    o_object_key(master, o_tag(3, 0, 0), ks);
    o_sample_uniform(kp, o_tag(2, 0, 0), c->logn, nq, c->primes, pid, a);
    i64 *e = (i64 *)malloc(n * sizeof(i64));
    o_sample_gauss(ks, o_tag(3, 0, 0), c->logn, cdt, ncdt, e);
    u64 *en = (u64 *)malloc((u64)nq * n * sizeof(u64));
    o_int_to_ntt(c, e, nq, pid, en);
    for (int l = 0; l < nq; l++) {
        u64 q = c->primes[l];
        for (u64 k = 0; k < n; k++) {
            u64 i = (u64)l * n + k;
            pk[i] = addmod(submod(0, mulmod(a[i], s_ntt[i], q), q), en[i], q);
        }
    }
    free(e); free(en); free(pid);
}

/*
 * O-7 switching key for s' (NTT form over Q_L, [nq][N]) under s (NTT form over Q_L u P, [nq+np][N]).
 * For digit j = 0..beta-1 with D_j = {j*alpha .. j*alpha+alpha-1} n [0, nq):
 *   a_j uniform over Q_L u P, e_j Gaussian,
 *   Q-limb t : b_j = -a_j s + e_j + [P]_t * s' * [t in D_j]
 *   P-limb   : b_j = -a_j s + e_j
 * layout out[j][0 = b, 1 = a][nq+np][N].  g = Galois element (0 for relinearization).
 */
void o_keygen_swk(const OCtx *c, const u32 *master, u64 g, const u64 *s_ntt, const u64 *sp_ntt,
                  const u64 *cdt, int ncdt, u64 *out) {
    u32 kp[8], ks[8];
    o_object_key(master, o_tag(4, g, 0), kp);
    o_object_key(master, o_tag(5, g, 0), ks);
    u64 n = NN(c);
    int nq = c->nq, np = c->np, ne = nq + np;
    int beta = (nq + c->alpha - 1) / c->alpha;
    int *pid = ids_range(0, ne);
    i64 *e = (i64 *)malloc(n * sizeof(i64));
    u64 *en = (u64 *)malloc((u64)ne * n * sizeof(u64));
    for (int j = 0; j < beta; j++) {
        u64 *b = out + (u64)j * 2 * ne * n;
        u64 *a = b + (u64)ne * n;
        o_sample_uniform(kp, o_tag(4, g, (u64)j), c->logn, ne, c->primes, pid, a);
        o_sample_gauss(ks, o_tag(5, g, (u64)j), c->logn, cdt, ncdt, e);
        o_int_to_ntt(c, e, ne, pid, en);
        for (int t = 0; t < ne; t++) {
            u64 q = c->primes[t];
            u64 Pt = 1; /* [P]_t */
            for (int p = 0; p < np; p++) Pt = mulmod(Pt, c->primes[nq + p] % q, q);
            int in_digit = (t < nq) && (t / c->alpha == j);
            for (u64 k = 0; k < n; k++) {
                u64 i = (u64)t * n + k;
                u64 v = addmod(submod(0, mulmod(a[i], s_ntt[i], q), q), en[i], q);
                if (in_digit) v = addmod(v, mulmod(Pt, sp_ntt[i], q), q);
                b[i] = v;
            }
        }
    }
    free(e); free(en); free(pid);
}

/* O-8 encryption at level `level` with the public key: ct = (v pk0 + e0 + m, v pk1 + e1) */
void o_encrypt(const OCtx *c, const u32 *master, const u64 *pk, const i64 *m, int level,
               const u64 *cdt, int ncdt, u64 *ct) {
    u32 ke[8];
    o_encrypt_key(master, ke);
    u64 n = NN(c);
    int nl = level + 1, nq = c->nq;
    int *pid = ids_range(0, nl);
    i64 *tmp = (i64 *)malloc(n * sizeof(i64));
    u64 *vn = (u64 *)malloc((u64)nl * n * sizeof(u64));
    u64 *e0 = (u64 *)malloc((u64)nl * n * sizeof(u64));
    u64 *e1 = (u64 *)malloc((u64)nl * n * sizeof(u64));
    u64 *mn = (u64 *)malloc((u64)nl * n * sizeof(u64));
    o_sample_ternary(ke, o_tag(6, 0, 0), c->logn, tmp);
    o_int_to_ntt(c, tmp, nl, pid, vn);
    o_sample_gauss(ke, o_tag(7, 0, 0), c->logn, cdt, ncdt, tmp);
    o_int_to_ntt(c, tmp, nl, pid, e0);
    o_sample_gauss(ke, o_tag(8, 0, 0), c->logn, cdt, ncdt, tmp);
    o_int_to_ntt(c, tmp, nl, pid, e1);
    o_int_to_ntt(c, m, nl, pid, mn);
    for (int l = 0; l < nl; l++) {
        u64 q = c->primes[l];
        const u64 *p0 = pk + (u64)l * n, *p1 = pk + (u64)(nq + l) * n;
        for (u64 k = 0; k < n; k++) {
            u64 i = (u64)l * n + k;
            ct[i] = addmod(addmod(mulmod(vn[i], p0[k], q), e0[i], q), mn[i], q);
            ct[(u64)nl * n + i] = addmod(mulmod(vn[i], p1[k], q), e1[i], q);
        }
    }
    free(pid); free(tmp); free(vn); free(e0); free(e1); free(mn);
}

/* O-8 decryption, up to the centered lift: out = INTT(c0 + c1 s) residues [nl][N] */
void o_decrypt_residues(const OCtx *c, const u64 *s_ntt, const u64 *ct, int level, u64 *out) {
    u64 n = NN(c);
    int nl = level + 1;
    for (int l = 0; l < nl; l++) {
        u64 q = c->primes[l];
        for (u64 k = 0; k < n; k++) {
            u64 i = (u64)l * n + k;
            out[i] = addmod(ct[i], mulmod(ct[(u64)nl * n + i], s_ntt[i], q), q);
        }
    }
    int *pid = ids_range(0, nl);
    o_intt_limbs(out, c->logn, nl, c->primes, c->psi, pid);
    free(pid);
}

/* M4: slot-wise add / sub (coefficient-wise mod q_i) on [npoly][nl][N] arrays */
void o_add(const OCtx *c, const u64 *a, const u64 *b, int nl, int npoly, u64 *out) {
    u64 n = NN(c);
    for (int p = 0; p < npoly; p++)
        for (int l = 0; l < nl; l++)
            for (u64 k = 0; k < n; k++) {
                u64 i = ((u64)p * nl + l) * n + k;
                out[i] = addmod(a[i], b[i], c->primes[l]);
            }
}
void o_sub(const OCtx *c, const u64 *a, const u64 *b, int nl, int npoly, u64 *out) {
    u64 n = NN(c);
    for (int p = 0; p < npoly; p++)
        for (int l = 0; l < nl; l++)
            for (u64 k = 0; k < n; k++) {
                u64 i = ((u64)p * nl + l) * n + k;
                out[i] = submod(a[i], b[i], c->primes[l]);
            }
}
/* multiply both polynomials by the integer constant C = c_hi 2^64 + c_lo (an integer plaintext with all NTT
   points = C) */
void o_mul_int(const OCtx *c, const u64 *a, int nl, i64 c_hi, u64 c_lo, u64 *out) {
    u64 n = NN(c);
    for (int p = 0; p < 2; p++)
        for (int l = 0; l < nl; l++) {
            u64 q = c->primes[l], cq = smod_wide(c_hi, c_lo, q);
            for (u64 k = 0; k < n; k++) {
                u64 i = ((u64)p * nl + l) * n + k;
                out[i] = mulmod(a[i], cq, q);
            }
        }
}
/* add the integer constant C to the message: c0 += C (the constant polynomial C has NTT points all = C) */
void o_add_int(const OCtx *c, const u64 *a, int nl, i64 c_hi, u64 c_lo, u64 *out) {
    u64 n = NN(c);
    memcpy(out, a, (u64)2 * nl * n * sizeof(u64));
    for (int l = 0; l < nl; l++) {
        u64 q = c->primes[l], cq = smod_wide(c_hi, c_lo, q);
        for (u64 k = 0; k < n; k++) out[(u64)l * n + k] = addmod(a[(u64)l * n + k], cq, q);
    }
}
/* multiply by a plaintext given in NTT form pt[nl][N] (limbs 0..nl-1) */
void o_mul_plain(const OCtx *c, const u64 *a, int nl, const u64 *pt, u64 *out) {
    u64 n = NN(c);
    for (int p = 0; p < 2; p++)
        for (int l = 0; l < nl; l++)
            for (u64 k = 0; k < n; k++) {
                u64 i = ((u64)p * nl + l) * n + k;
                out[i] = mulmod(a[i], pt[(u64)l * n + k], c->primes[l]);
            }
}

/* M5 tensor: d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 (NTT domain, pointwise) */
void o_tensor(const OCtx *c, const u64 *a, const u64 *b, int nl, u64 *d) {
    u64 n = NN(c), L = (u64)nl * n;
    for (int l = 0; l < nl; l++) {
        u64 q = c->primes[l];
        for (u64 k = 0; k < n; k++) {
            u64 i = (u64)l * n + k;
            u64 a0 = a[i], a1 = a[L + i], b0 = b[i], b1 = b[L + i];
            d[i] = mulmod(a0, b0, q);
            d[L + i] = addmod(mulmod(a0, b1, q), mulmod(a1, b0, q), q);
            d[2 * L + i] = mulmod(a1, b1, q);
        }
    }
}

/*
 * O-10 hybrid key switching of d (NTT form, [nl][N], level = nl-1) with switching key swk
 * ([beta_top][2][nq+np][N], limb index = global prime index).  Output ks[2][nl][N] with
 * ks0 + ks1 s ~= d s' (mod Q_level).
 *   ModUp  : for digit j with present primes I_j and Q'_j = prod_{i in I_j} q_i:
 *            y_i = [d_i (Q'_j/q_i)^{-1}]_{q_i};  ext_j[t] = sum_i y_i [Q'_j/q_i]_t mod t  (t not in I_j)
 *            ext_j[t] = d_t for t in I_j.
 *   inner  : acc_b[t] = sum_j ext_j[t] * swk_j[b][t]
 *   ModDown: r_p = INTT(acc_b[p]);  out_b,i = (acc_b,i - NTT(sum_p [r_p (P/p)^{-1}]_p [P/p]_{q_i})) [P^{-1}]_{q_i}
 */
/* ModUp + key inner product of O-10: returns acc[2][ne][N] (NTT form over Q_level u P, extended
 * index e < nl -> prime e, e >= nl -> special prime e - nl); *eid_out = extended index -> prime id */
/* sigma_g on one coefficient-form residue vector mod q: X^k -> X^{kg mod 2N}, negated when
 * kg mod 2N >= N (O-12) */
static void sigma_coeff(const u64 *in, u64 *out, u64 n, u64 g, u64 q) {
    u64 two_n = 2 * n;
    for (u64 k = 0; k < n; k++) {
        u64 e = (u64)(((u128)k * g) % two_n);
        if (e >= n) out[e - n] = submod(0, in[k], q);
        else out[e] = in[k];
    }
}

/* g > 1 (N2, hoisted rotation): every extended digit polynomial ModUp_j(d) is replaced by
 * sigma_g(ModUp_j(d)) -- the automorphism applied to the integer polynomial ModUp_j(d) limb by limb
 * in the coefficient domain -- before the inner product with the Galois key of g. */
static u64 *ks_acc(const OCtx *c, const u64 *d, int nl, const u64 *swk, u64 g, int **eid_out) {
    u64 n = NN(c);
    int nq = c->nq, np = c->np, ne = nl + np, nek = nq + np;
    (void)nq;
    int beta = (nl + c->alpha - 1) / c->alpha;
    /* extended basis: ext index e < nl -> prime e; e >= nl -> prime nq + (e - nl) */
    int *eid = (int *)malloc(sizeof(int) * ne);
    for (int e = 0; e < ne; e++) eid[e] = e < nl ? e : nq + (e - nl);
    u64 *dc = (u64 *)malloc((u64)nl * n * sizeof(u64));
    memcpy(dc, d, (u64)nl * n * sizeof(u64));
    o_intt_limbs(dc, c->logn, nl, c->primes, c->psi, eid);
    u64 *acc = (u64 *)calloc((u64)2 * ne * n, sizeof(u64));
    u64 *ext = (u64 *)malloc((u64)ne * n * sizeof(u64));
    for (int j = 0; j < beta; j++) {
        int i0 = j * c->alpha, i1 = i0 + c->alpha < nl ? i0 + c->alpha : nl;
        /* (Q'_j/q_i)^{-1} mod q_i for i in I_j */
        u64 inv_hat[64];
        for (int i = i0; i < i1; i++) {
            u64 qi = c->primes[i], h = 1;
            for (int i2 = i0; i2 < i1; i2++) if (i2 != i) h = mulmod(h, c->primes[i2] % qi, qi);
            inv_hat[i - i0] = invmod(h, qi);
        }
#pragma omp parallel for schedule(dynamic, 1)
        for (int e = 0; e < ne; e++) {
            u64 t = c->primes[eid[e]];
            u64 *x = ext + (u64)e * n;
            if (e >= i0 && e < i1) {
                if (g <= 1) { memcpy(x, d + (u64)e * n, n * sizeof(u64)); continue; }
                u64 *y = (u64 *)malloc(n * sizeof(u64));
                sigma_coeff(dc + (u64)e * n, y, n, g, t);
                memcpy(x, y, n * sizeof(u64));
                free(y);
                o_ntt(x, c->logn, t, c->psi[eid[e]]);
                continue;
            }
            u64 hat_t[64]; /* (Q'_j/q_i) mod t */
            for (int i = i0; i < i1; i++) {
                u64 h = 1;
                for (int i2 = i0; i2 < i1; i2++) if (i2 != i) h = mulmod(h, c->primes[i2] % t, t);
                hat_t[i - i0] = h;
            }
            for (u64 k = 0; k < n; k++) {
                u64 sum = 0;
                for (int i = i0; i < i1; i++) {
                    u64 y = mulmod(dc[(u64)i * n + k], inv_hat[i - i0], c->primes[i]);
                    sum = addmod(sum, mulmod(y % t, hat_t[i - i0], t), t);
                }
                x[k] = sum;
            }
            if (g > 1) {
                u64 *y = (u64 *)malloc(n * sizeof(u64));
                sigma_coeff(x, y, n, g, t);
                memcpy(x, y, n * sizeof(u64));
                free(y);
            }
            o_ntt(x, c->logn, t, c->psi[eid[e]]);
        }
        const u64 *kb = swk + (u64)j * 2 * nek * n;
        const u64 *ka = kb + (u64)nek * n;
        for (int e = 0; e < ne; e++) {
            u64 t = c->primes[eid[e]];
            for (u64 k = 0; k < n; k++) {
                u64 x = ext[(u64)e * n + k];
                u64 *a0 = acc + (u64)e * n + k, *a1 = acc + (u64)(ne + e) * n + k;
                *a0 = addmod(*a0, mulmod(x, kb[(u64)eid[e] * n + k], t), t);
                *a1 = addmod(*a1, mulmod(x, ka[(u64)eid[e] * n + k], t), t);
            }
        }
    }
    free(dc); free(ext);
    *eid_out = eid;
    return acc;
}

void o_keyswitch_g(const OCtx *c, const u64 *d, int nl, const u64 *swk, u64 g, u64 *ks);
void o_keyswitch(const OCtx *c, const u64 *d, int nl, const u64 *swk, u64 *ks) { o_keyswitch_g(c, d, nl, swk, 1, ks); }

/* O-10 key switching with the automorphism sigma_g hoisted past ModUp (N2): ks0 + ks1 s ~=
 * sigma_g(d) sigma_g(s) when swk is the Galois key of g -- ModUp of the un-rotated d, sigma_g on every
 * extended digit, inner product, ModDown.  g = 1 is plain O-10. */
void o_keyswitch_g(const OCtx *c, const u64 *d, int nl, const u64 *swk, u64 g, u64 *ks) {
    u64 n = NN(c);
    int nq = c->nq, np = c->np, ne = nl + np;
    int *eid;
    u64 *acc = ks_acc(c, d, nl, swk, g, &eid);
    /* ModDown */
    for (int b = 0; b < 2; b++) {
        u64 *ab = acc + (u64)b * ne * n;
        u64 *r = (u64 *)malloc((u64)np * n * sizeof(u64));
        memcpy(r, ab + (u64)nl * n, (u64)np * n * sizeof(u64));
        o_intt_limbs(r, c->logn, np, c->primes, c->psi, eid + nl);
#pragma omp parallel for schedule(dynamic, 1)
        for (int i = 0; i < nl; i++) {
            u64 qi = c->primes[i];
            u64 *conv = (u64 *)malloc(n * sizeof(u64));
            u64 Pinv = 1;
            for (int p = 0; p < np; p++) Pinv = mulmod(Pinv, c->primes[nq + p] % qi, qi);
            Pinv = invmod(Pinv, qi);
            u64 inv_hat_p[64], hat_q[64]; /* (P/p)^{-1} mod p and (P/p) mod q_i */
            for (int p = 0; p < np; p++) {
                u64 pp = c->primes[nq + p], hp = 1, hq = 1;
                for (int p2 = 0; p2 < np; p2++) if (p2 != p) {
                    hp = mulmod(hp, c->primes[nq + p2] % pp, pp);
                    hq = mulmod(hq, c->primes[nq + p2] % qi, qi);
                }
                inv_hat_p[p] = invmod(hp, pp);
                hat_q[p] = hq;
            }
            for (u64 k = 0; k < n; k++) {
                u64 sum = 0;
                for (int p = 0; p < np; p++) {
                    u64 y = mulmod(r[(u64)p * n + k], inv_hat_p[p], c->primes[nq + p]);
                    sum = addmod(sum, mulmod(y % qi, hat_q[p], qi), qi);
                }
                conv[k] = sum;
            }
            o_ntt(conv, c->logn, qi, c->psi[i]);
            for (u64 k = 0; k < n; k++)
                ks[((u64)b * nl + i) * n + k] = mulmod(submod(ab[(u64)i * n + k], conv[k], qi), Pinv, qi);
            free(conv);
        }
        free(r);
    }
    free(eid); free(acc);
}

/*
 * O-11 rescale by q_l (l = nl-1): c' = floor((c + floor(q_l/2)) / q_l) mod Q_{l-1}, in RNS:
 *   r = [c_l + floor(q_l/2)]_{q_l};  c'_i = (c_i + [floor(q_l/2)]_{q_i} - [r]_{q_i}) [q_l^{-1}]_{q_i}
 * computed in the coefficient domain; input/output in NTT form.  in [2][nl][N] -> out [2][nl-1][N].
 */
void o_rescale(const OCtx *c, const u64 *ct, int nl, u64 *out) {
    u64 n = NN(c);
    int lo = nl - 1;
    u64 ql = c->primes[lo], half = ql >> 1;
    int *pid = ids_range(0, nl);
    u64 *tmp = (u64 *)malloc((u64)nl * n * sizeof(u64));
    for (int b = 0; b < 2; b++) {
        memcpy(tmp, ct + (u64)b * nl * n, (u64)nl * n * sizeof(u64));
        o_intt_limbs(tmp, c->logn, nl, c->primes, c->psi, pid);
        const u64 *cl = tmp + (u64)lo * n;
        u64 *o = out + (u64)b * lo * n;
        for (int i = 0; i < lo; i++) {
            u64 qi = c->primes[i], qinv = invmod(ql % qi, qi);
            for (u64 k = 0; k < n; k++) {
                u64 r = addmod(cl[k], half, ql);
                u64 v = submod(addmod(tmp[(u64)i * n + k], half % qi, qi), r % qi, qi);
                o[(u64)i * n + k] = mulmod(v, qinv, qi);
            }
        }
        o_ntt_limbs(o, c->logn, lo, c->primes, c->psi, pid);
    }
    free(pid); free(tmp);
}

/*
 * O-12 automorphism sigma_g on both polynomials: coefficient X^k -> X^{kg mod 2N}, negated
 * when kg mod 2N >= N.  Done in the coefficient domain (INTT -> signed permutation -> NTT).
 */
void o_automorph(const OCtx *c, const u64 *ct, int nl, int npoly, u64 g, u64 *out) {
    u64 n = NN(c), two_n = 2 * n;
    int *pid = ids_range(0, nl);
    u64 *tmp = (u64 *)malloc((u64)nl * n * sizeof(u64));
    for (int b = 0; b < npoly; b++) {
        memcpy(tmp, ct + (u64)b * nl * n, (u64)nl * n * sizeof(u64));
        o_intt_limbs(tmp, c->logn, nl, c->primes, c->psi, pid);
        u64 *o = out + (u64)b * nl * n;
        for (int l = 0; l < nl; l++) {
            u64 q = c->primes[l];
            for (u64 k = 0; k < n; k++) {
                u64 e = (u64)(((u128)k * g) % two_n);
                u64 v = tmp[(u64)l * n + k];
                if (e >= n) o[(u64)l * n + (e - n)] = submod(0, v, q);
                else o[(u64)l * n + e] = v;
            }
        }
        o_ntt_limbs(o, c->logn, nl, c->primes, c->psi, pid);
    }
    free(pid); free(tmp);
}

/* pointwise product of two residue vectors mod q */
void o_mul_vec(const u64 *a, const u64 *b, u64 n, u64 q, u64 *out) {
    for (u64 k = 0; k < n; k++) out[k] = mulmod(a[k], b[k], q);
}
