// client.cu -- key generation, encryption and decryption on the GPU (PAPER.md:139 Step 1,
// :143 Step 4; readings R6/R7 of DESIGN.md).
//
// Object tags (kind << 48 ^ g << 8 ^ j): 1 secret, 2 pk.a, 3 pk.e, 4 swk.a, 5 swk.e (g = Galois
// element, 0 for relinearisation; j = digit), 6 enc.v, 7 enc.e0, 8 enc.e1; each drawn from a ChaCha20
// stream under a key derived from the caller's 256-bit seed (sample.cu, reading R6).
#include <cstring>

#include "context.h"

static inline u64 tag(u64 kind, u64 g, u64 j) { return (kind << 48) ^ (g << 8) ^ j; }
static inline LimbMap allmap(const Ctx &c) { return LimbMap{c.nprimes(), c.nq, 0, c.nq}; }
static inline LimbMap qmap(int nl) { return LimbMap{nl, nl, 0, 0}; }

// small signed polynomial (ternary / Gaussian) -> NTT residues on lm.nl limbs
static void small_to_ntt(Ctx &c, const Key256 &key, u64 tg, int kind, u64 *out, LimbMap lm) {
    DevBuf m(c.N, c.st);
    k_sample_small(c.logn, key, tg, kind, (i64 *)m.p, c.st);
    k_int_to_rows(c.tab, c.logn, (const i64 *)m.p, out, lm, c.st);
    ev_ntt(c, RowsArg{out, 2L * lm.nl * c.N, (long)lm.nl * c.N}, 1, lm, false);
}

// switching key for s' (NTT, nq limbs): out[j][0 = b, 1 = a][nq + np][N]
static void gen_swk(Ctx &c, const Keys &k, const Key256 &master, u64 g, const u64 *sp, DevBuf &out) {
    const Key256 kp = object_key(master, tag(4, g, 0)), ks = object_key(master, tag(5, g, 0));
    const int P = c.nprimes(), bt = c.beta(c.L());
    const long N = c.N;
    out = DevBuf((size_t)bt * 2 * P * N, c.st);
    DevBuf e((size_t)P * N, c.st);
    // [P]_t for every ciphertext prime t
    std::vector<u64> Pt(c.nq);
    for (int t = 0; t < c.nq; t++) {
        u64 v = 1;
        for (int a = 0; a < c.np; a++) v = h_mulmod(v, c.primes[c.nq + a] % c.primes[t], c.primes[t]);
        Pt[t] = v;
    }
    for (int j = 0; j < bt; j++) {
        u64 *b = out.p + (size_t)j * 2 * P * N;
        u64 *a = b + (size_t)P * N;
        k_sample_uniform(c.tab, c.logn, kp, tag(4, g, j), a, allmap(c), c.st);
        small_to_ntt(c, ks, tag(5, g, j), 1, e.p, allmap(c));
        LimbConst gad{};
        for (int t = j * c.alpha; t < std::min((j + 1) * c.alpha, c.nq); t++) {
            gad.c[t] = Pt[t];
            gad.csh[t] = h_shoup(Pt[t], c.primes[t]);
        }
        k_key_combine(c.tab, c.logn, a, k.s.p, e.p, sp, &gad, b, allmap(c), c.st);
    }
}

Keys *keygen(Ctx &c, const Key256 &master, const int *rot, int n_rot, int h) {
    const Key256 ksk = object_key(master, tag(1, 0, 0)), kpk = object_key(master, tag(2, 0, 0));
    auto k = std::make_unique<Keys>();
    const int P = c.nprimes();
    const long N = c.N;
    k->s = DevBuf((size_t)P * N, c.st);
    if (h > 0) {  // sparse secret (R36), sampled on the host
        std::vector<i64> sh(N);
        h_sample_sparse(ksk, tag(1, 0, 0), c.logn, h, sh.data());
        DevBuf m(N, c.st);
        CUDA_CHECK(cudaMemcpyAsync(m.p, sh.data(), N * 8, cudaMemcpyHostToDevice, c.st));
        k_int_to_rows(c.tab, c.logn, (const i64 *)m.p, k->s.p, allmap(c), c.st);
        ev_ntt(c, RowsArg{k->s.p, 2L * P * N, (long)P * N}, 1, allmap(c), false);
        CUDA_CHECK(cudaStreamSynchronize(c.st));  // sh is host memory of this frame
    } else {
        small_to_ntt(c, ksk, tag(1, 0, 0), 0, k->s.p, allmap(c));
    }
    // public key (-a s + e, a) over Q_L
    k->pk = DevBuf(2L * c.nq * N, c.st);
    {
        u64 *a = k->pk.p + (size_t)c.nq * N;
        k_sample_uniform(c.tab, c.logn, kpk, tag(2, 0, 0), a, qmap(c.nq), c.st);
        DevBuf e((size_t)c.nq * N, c.st);
        small_to_ntt(c, ksk, tag(3, 0, 0), 1, e.p, qmap(c.nq));
        k_key_combine(c.tab, c.logn, a, k->s.p, e.p, nullptr, nullptr, k->pk.p, qmap(c.nq), c.st);
    }
    // relinearisation key: s' = s^2
    {
        DevBuf s2((size_t)c.nq * N, c.st);
        k_square(c.tab, c.logn, k->s.p, s2.p, qmap(c.nq), c.st);
        gen_swk(c, *k, master, 0, s2.p, k->rlk);
    }
    // Galois keys: s' = sigma_g(s)
    for (int i = 0; i < n_rot; i++) {
        const u64 g = galois_elt(c, rot[i]);
        if (g == 1 || k->gk.count(g)) continue;
        DevBuf sg((size_t)c.nq * N, c.st);
        k_automorph(c.logn, CRows{k->s.p, 2L * P * N, (long)P * N}, RowsArg{sg.p, 2L * c.nq * N, (long)c.nq * N}, 1,
                    c.nq, g, c.st);
        DevBuf key;
        gen_swk(c, *k, master, g, sg.p, key);
        k->gk.emplace(g, std::move(key));
    }
    CUDA_CHECK(cudaStreamSynchronize(c.st));
    return k.release();
}

// ct = (v pk0 + e0 + m, v pk1 + e1) at `level`; coeffs = integer plaintext (host)
void encrypt_coeffs(Ctx &c, const Keys &k, const i64 *coeffs, int level, const Key256 &master, u64 *ct) {
    const Key256 ke = derive_key(master, DOM_ENC);
    const int nl = level + 1;
    const long N = c.N;
    DevBuf mi(N, c.st), m((size_t)nl * N, c.st), v((size_t)nl * N, c.st), e0((size_t)nl * N, c.st),
        e1((size_t)nl * N, c.st);
    CUDA_CHECK(cudaMemcpyAsync(mi.p, coeffs, N * 8, cudaMemcpyHostToDevice, c.st));
    k_int_to_rows(c.tab, c.logn, (const i64 *)mi.p, m.p, qmap(nl), c.st);
    ev_ntt(c, RowsArg{m.p, 2L * nl * N, (long)nl * N}, 1, qmap(nl), false);
    small_to_ntt(c, ke, tag(6, 0, 0), 0, v.p, qmap(nl));
    small_to_ntt(c, ke, tag(7, 0, 0), 1, e0.p, qmap(nl));
    small_to_ntt(c, ke, tag(8, 0, 0), 1, e1.p, qmap(nl));
    k_encrypt_combine(c.tab, c.logn, v.p, k.pk.p, (long)c.nq * N, e0.p, e1.p, m.p, ct, nl, c.st);
    CUDA_CHECK(cudaStreamSynchronize(c.st));  // coeffs is caller host memory
}

// residues of c0 + c1 s in coefficient form (host out [nl][N])
void decrypt_residues(Ctx &c, const Keys &k, const CtView &ct, u64 *host_out) {
    const int nl = ct.level + 1;
    const long N = c.N;
    DevBuf m((size_t)nl * N, c.st), cc(2L * nl * N, c.st);
    ev_copy(c, ct, compact_view(c, cc.p, 1, ct.level, ct.scale));
    k_decrypt_combine(c.tab, c.logn, cc.p, k.s.p, m.p, nl, c.st);
    ev_ntt(c, RowsArg{m.p, 2L * nl * N, (long)nl * N}, 1, qmap(nl), true);
    CUDA_CHECK(cudaMemcpyAsync(host_out, m.p, (size_t)nl * N * 8, cudaMemcpyDeviceToHost, c.st));
    CUDA_CHECK(cudaStreamSynchronize(c.st));
}

// centered lift from the first two limbs (exact whenever |m'| < q0 q1 / 2), then decode
void decrypt_slots(Ctx &c, const Keys &k, const CtView &ct, double *slots, size_t n) {
    const int nl = ct.level + 1;
    const long N = c.N;
    std::vector<u64> r((size_t)nl * N);
    decrypt_residues(c, k, ct, r.data());
    std::vector<double> coef(N);
    const u64 q0 = c.primes[0];
    if (nl == 1) {
        for (long i = 0; i < N; i++) coef[i] = r[i] > q0 / 2 ? -(double)(q0 - r[i]) : (double)r[i];
    } else {
        const u64 q1 = c.primes[1];
        const u128 Q = (u128)q0 * q1;
        const u64 inv = h_invmod(q0 % q1, q1);  // x = r0 + q0 * ((r1 - r0) q0^{-1} mod q1)
        for (long i = 0; i < N; i++) {
            const u64 r0 = r[i], r1 = r[N + i];
            const u64 t = h_mulmod((r1 + q1 - r0 % q1) % q1, inv, q1);
            const u128 x = (u128)r0 + (u128)q0 * t;
            coef[i] = x > Q / 2 ? -(double)(Q - x) : (double)x;
        }
    }
    decode_real(c, coef, ct.scale, slots, n);
}
