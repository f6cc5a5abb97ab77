// abi.cpp -- extern "C" entry points of libsecpe.so (declared in include/secpe.h).
// Exceptions never cross the boundary: every entry point maps them to a status code and a
// thread-local message (secpe_last_error).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/secpe.h"
#include "context.h"

Keys *keygen(Ctx &c, const Key256 &master, const int *rot, int n_rot, int h);
void encrypt_coeffs(Ctx &c, const Keys &k, const i64 *coeffs, int level, const Key256 &master, u64 *ct);
void decrypt_residues(Ctx &c, const Keys &k, const CtView &ct, u64 *host_out);
void decrypt_slots(Ctx &c, const Keys &k, const CtView &ct, double *slots, size_t n);

struct secpe_ctx {
    Ctx c;
};
struct secpe_keys {
    Keys *k;
};

static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }

template <typename F>
static int guard(F &&f) {
    try {
        f();
        return SECPE_OK;
    } catch (const SecpeError &e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc &) {
        g_err = "out of host memory";
        return SECPE_ENOMEM;
    } catch (const std::exception &e) {
        g_err = e.what();
        return SECPE_EINVAL;
    }
}
#define REQUIRE(cond, code, msg) \
    do {                         \
        if (!(cond)) throw SecpeError{code, msg}; \
    } while (0)

static CtView view_of(const Ctx &c, const secpe_ct *ct) {
    REQUIRE(ct && ct->data, SECPE_EINVAL, "null ciphertext");
    REQUIRE(ct->level >= 0 && ct->level < c.nq, SECPE_EINVAL, "ciphertext level out of range");
    return compact_view(c, ct->data, 1, ct->level, ct->scale);
}
// A batch of n caller ciphertexts as one CtView: the caller's memory when the batch is contiguous
// (data[i] = data[0] + i * ct_words), else a staged copy (`stage` receives the buffer).
// the byte ranges [data, data + words) of the n_out outputs must not overlap those of the n_in inputs
// (an output batch larger than the input batch can overlap it without sharing a start pointer)
static void no_overlap(const secpe_ct *in, int n_in, long in_words, const secpe_ct *out, int n_out, long out_words) {
    for (int i = 0; i < n_out; i++)
        for (int j = 0; j < n_in; j++) {
            const uint64_t *o0 = out[i].data, *o1 = o0 + out_words, *i0 = in[j].data, *i1 = i0 + in_words;
            REQUIRE(o1 <= i0 || i1 <= o0, SECPE_EINVAL, "out must not overlap in");
        }
}
static CtView batch_in(Ctx &c, const secpe_ct *in, int n, DevBuf &stage) {
    REQUIRE(in && n >= 1, SECPE_EINVAL, "empty batch");
    const int lv = in[0].level;
    REQUIRE(lv >= 0 && lv < c.nq, SECPE_EINVAL, "ciphertext level out of range");
    for (int i = 0; i < n; i++) {
        REQUIRE(in[i].data, SECPE_EINVAL, "null ciphertext data");
        REQUIRE(in[i].level == lv && in[i].scale == in[0].scale, SECPE_EINVAL, "batch must share level and scale");
    }
    const long cw = c.ct_words(lv);
    bool contiguous = true;
    for (int i = 1; i < n; i++) contiguous &= in[i].data == in[0].data + (long)i * cw;
    CtView v = compact_view(c, in[0].data, n, lv, in[0].scale);
    if (!contiguous) {
        stage = DevBuf((size_t)n * cw, c.st);
        for (int i = 0; i < n; i++)
            CUDA_CHECK(cudaMemcpyAsync(stage.p + (long)i * cw, in[i].data, cw * 8, cudaMemcpyDeviceToDevice, c.st));
        v.data = stage.p;
    }
    return v;
}
// Output batch at `level`: the caller's memory when contiguous, else a staging buffer copied back by
// batch_out_finish.
static CtView batch_out(Ctx &c, secpe_ct *out, int n, int level, double scale, DevBuf &stage) {
    const long ow = c.ct_words(level);
    bool contiguous = true;
    for (int i = 0; i < n; i++) REQUIRE(out[i].data, SECPE_EINVAL, "null output data");
    for (int i = 1; i < n; i++) contiguous &= out[i].data == out[0].data + (long)i * ow;
    CtView v = compact_view(c, out[0].data, n, level, scale);
    if (!contiguous) {
        stage = DevBuf((size_t)n * ow, c.st);
        v.data = stage.p;
    }
    return v;
}
static void batch_out_finish(Ctx &c, secpe_ct *out, int n, const CtView &v, const DevBuf &stage) {
    const long ow = c.ct_words(v.level);
    if (stage.p)
        for (int i = 0; i < n; i++)
            CUDA_CHECK(cudaMemcpyAsync(out[i].data, stage.p + (long)i * ow, ow * 8, cudaMemcpyDeviceToDevice, c.st));
    for (int i = 0; i < n; i++) {
        out[i].level = v.level;
        out[i].scale = v.scale;
    }
}

static void set_out(secpe_ct *out, const CtView &v) {
    out->level = v.level;
    out->scale = v.scale;
}
// CUDA-graph cache around a data-independent plan `run` writing vout: replay the graph captured for `key`
// if there is one, else run eagerly and capture on the key's second sighting (a caller allocating fresh
// buffers every call would otherwise pay a capture per call); at most kMaxGraphs graphs, oldest evicted.
// keys / aux: library-owned device memory the kernels read (destroying it drops the graph).
template <class F>
static void graphed(Ctx &c, bool graphable, const std::string &key, const void *keys, const void *aux, CtView &vout,
                    F run) {
    graphable = graphable && c.use_graphs && !c.log_on && !c.prof.on && c.st != nullptr && c.st != cudaStreamLegacy &&
                c.st != cudaStreamPerThread;
    auto git = graphable ? c.graphs.find(key) : c.graphs.end();
    if (git != c.graphs.end() && git->second.exec) {
        CUDA_CHECK(cudaGraphLaunch(git->second.exec, c.st));
        const Counters &d = git->second.cnt;
        c.cnt.ntt_limbs += d.ntt_limbs, c.cnt.keyswitch += d.keyswitch, c.cnt.rescale += d.rescale;
        c.cnt.rotate += d.rotate, c.cnt.mulct += d.mulct, c.cnt.mulconst += d.mulconst;
        c.cnt.launches += d.launches, c.cnt.sign += d.sign;
        vout.scale = git->second.out_scale;
        return;
    }
    run();
    if (!graphable) return;
    if (++c.graph_seen[key] < 2) {
        if (c.graph_seen.size() > 4 * Ctx::kMaxGraphs) c.graph_seen.clear();
        return;
    }
    if ((int)c.graphs.size() >= Ctx::kMaxGraphs && !c.graph_order.empty()) {
        CUDA_CHECK(cudaStreamSynchronize(c.st));  // the evicted graph may still be running
        auto old = c.graphs.find(c.graph_order.front());
        if (old != c.graphs.end()) {
            if (old->second.exec) cudaGraphExecDestroy(old->second.exec);
            c.graphs.erase(old);
        }
        c.graph_order.erase(c.graph_order.begin());
    }
    const Counters before = c.cnt;
    cudaGraph_t graph;
    CUDA_CHECK(cudaStreamBeginCapture(c.st, cudaStreamCaptureModeThreadLocal));
    try {
        run();
    } catch (...) {
        cudaStreamEndCapture(c.st, &graph);
        throw;
    }
    CUDA_CHECK(cudaStreamEndCapture(c.st, &graph));
    Ctx::Graph G;
    CUDA_CHECK(cudaGraphInstantiate(&G.exec, graph, 0));
    CUDA_CHECK(cudaGraphDestroy(graph));
    CUDA_CHECK(cudaGraphUpload(G.exec, c.st));  // pay the one-time upload now, not on the first replay
    G.keys = keys;
    G.aux = aux;
    G.cnt.ntt_limbs = c.cnt.ntt_limbs - before.ntt_limbs;
    G.cnt.keyswitch = c.cnt.keyswitch - before.keyswitch;
    G.cnt.rescale = c.cnt.rescale - before.rescale;
    G.cnt.rotate = c.cnt.rotate - before.rotate;
    G.cnt.mulct = c.cnt.mulct - before.mulct;
    G.cnt.mulconst = c.cnt.mulconst - before.mulconst;
    G.cnt.launches = c.cnt.launches - before.launches;
    G.cnt.sign = c.cnt.sign - before.sign;
    c.cnt = before;  // the capture executed nothing
    G.out_scale = vout.scale;
    c.graphs[key] = G;
    c.graph_order.push_back(key);
    c.graph_seen.erase(key);
}
static std::string dkey(double x) {
    u64 b;
    std::memcpy(&b, &x, 8);
    return std::to_string(b);
}
static SignCfg sign_cfg(const secpe_sign_cfg *cfg) {
    REQUIRE(cfg && cfg->n_stages > 0 && cfg->degrees && cfg->coeffs, SECPE_EINVAL, "bad sign config");
    SignCfg s;
    size_t off = 0;
    for (int i = 0; i < cfg->n_stages; i++) {
        const int d = cfg->degrees[i];
        REQUIRE(d == 3 || d == 7 || d == 15, SECPE_EINVAL, "sign stage degree must be 3, 7 or 15");
        std::vector<double> c(cfg->coeffs + off, cfg->coeffs + off + d + 1);
        for (int e = 0; e <= d; e += 2) REQUIRE(c[e] == 0.0, SECPE_EINVAL, "sign polynomials must be odd");
        s.stages.push_back(c);
        off += d + 1;
    }
    return s;
}
static Layout layout_of(const Ctx &c, const secpe_layout *l) {
    REQUIRE(l, SECPE_EINVAL, "null layout");
    auto pow2 = [](int v) { return v >= 1 && (v & (v - 1)) == 0; };
    REQUIRE(pow2(l->prompts) && pow2(l->classes), SECPE_ELAYOUT, "prompts and classes must be powers of two");
    REQUIRE(l->queries >= 1 && l->prompts * l->classes <= l->block && 2 * l->classes <= l->block &&
                (long)l->queries * l->block <= c.N / 2,
            SECPE_ELAYOUT, "layout does not fit the slots");
    return Layout{l->queries, l->prompts, l->classes, l->block};
}

extern "C" {

const char *secpe_last_error(void) { return g_err.c_str(); }
const char *secpe_version(void) { return "secpe-b200 0.1 (sm_100a)"; }

int secpe_gen_primes(uint32_t bits, uint32_t count, uint32_t log_n, int32_t mode, const uint64_t *exclude,
                     uint32_t n_exclude, uint64_t *out) {
    return guard([&] {
        REQUIRE(bits >= 20 && bits <= 62 && out && (mode == 0 || mode == 1), SECPE_EINVAL, "bad prime request");
        const int got = h_gen_primes((int)bits, (int)count, (int)log_n, mode, exclude, (int)n_exclude, out);
        REQUIRE(got == (int)count, SECPE_EINVAL, "not enough primes");
    });
}

int secpe_ctx_create(const secpe_params *prm, void *stream, secpe_ctx **out) {
    return guard([&] {
        REQUIRE(prm && out && prm->q && (prm->p || prm->n_p == 0), SECPE_EINVAL, "null argument");
        REQUIRE(prm->log_n >= 12 && prm->log_n <= 16, SECPE_EINVAL, "log_n must be in [12, 16]");
        REQUIRE(prm->n_q >= 1 && prm->n_q + prm->n_p <= MAXL, SECPE_EINVAL, "prime counts");
        REQUIRE(prm->alpha >= 1 && prm->alpha <= 16 && (prm->n_q + prm->alpha - 1) / prm->alpha <= 32 &&
                    prm->n_p <= 16,
                SECPE_EINVAL, "need alpha <= 16, dnum <= 32, special primes <= 16");
        const u64 two_n = (u64)2 << prm->log_n;
        // lazy 128-bit accumulations (key inner product: dnum terms, ModUp: alpha terms, ModDown: n_p terms)
        // must stay below 2^125 (Barrett input bound)
        {
            u64 mx = 0;
            for (uint32_t i = 0; i < prm->n_q; i++) mx = std::max(mx, prm->q[i]);
            for (uint32_t i = 0; i < prm->n_p; i++) mx = std::max(mx, prm->p[i]);
            const double lg = 2.0 * std::log2((double)mx);
            const int terms = (int)std::max({(prm->n_q + prm->alpha - 1) / prm->alpha, prm->alpha, prm->n_p});
            REQUIRE(lg + std::log2((double)terms) < 124.9, SECPE_EINVAL,
                    "prime sizes x dnum/alpha/n_p exceed the 128-bit lazy accumulation bound");
        }
        for (uint32_t i = 0; i < prm->n_q + prm->n_p; i++) {
            const u64 v = i < prm->n_q ? prm->q[i] : prm->p[i - prm->n_q];
            REQUIRE(v > (1ULL << 32) && v < (1ULL << 60) && v % two_n == 1 && h_is_prime(v), SECPE_EINVAL,
                    "primes must be NTT-friendly primes in (2^32, 2^60)");
        }
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw SecpeError{SECPE_ECUDA, "no CUDA device: libsecpe has no CPU fallback"};
        auto h = std::make_unique<secpe_ctx>();
        h->c.st = (cudaStream_t)stream;
        {
            // scratch comes from the device's stream-ordered pool: keep freed blocks cached instead of
            // returning them to the driver at every synchronisation (hot-path allocations are then free)
            int dev = 0;
            CUDA_CHECK(cudaGetDevice(&dev));
            cudaMemPool_t pool;
            CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, dev));
            uint64_t thr = ~0ULL;
            CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        }
        h->c.build(prm->q, (int)prm->n_q, prm->p, (int)prm->n_p, (int)prm->alpha, (int)prm->log_n, prm->scale);
        *out = h.release();
    });
}
void secpe_ctx_destroy(secpe_ctx *ctx) {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->c.st);
    delete ctx;
}
int secpe_set_stream(secpe_ctx *ctx, void *stream) {
    return guard([&] {
        REQUIRE(ctx, SECPE_EINVAL, "null ctx");
        CUDA_CHECK(cudaStreamSynchronize(ctx->c.st));
        ctx->c.st = (cudaStream_t)stream;
    });
}
int secpe_sync(secpe_ctx *ctx) {
    return guard([&] {
        REQUIRE(ctx, SECPE_EINVAL, "null ctx");
        CUDA_CHECK(cudaStreamSynchronize(ctx->c.st));
    });
}
int secpe_ctx_info(const secpe_ctx *ctx, uint64_t *primes_out, uint64_t *psi_out) {
    return guard([&] {
        REQUIRE(ctx, SECPE_EINVAL, "null ctx");
        if (primes_out) std::memcpy(primes_out, ctx->c.primes.data(), ctx->c.primes.size() * 8);
        if (psi_out) std::memcpy(psi_out, ctx->c.psi.data(), ctx->c.psi.size() * 8);
    });
}
size_t secpe_ct_bytes(const secpe_ctx *ctx, int32_t level) {
    if (!ctx || level < 0) return 0;
    return (size_t)ctx->c.ct_words(level) * 8;
}

// the 256-bit master seed (null: OS entropy), reading R6
static Key256 master_key(const secpe_seed *seed) {
    if (!seed) return os_entropy_key();
    Key256 k;
    for (int i = 0; i < 8; i++)
        k.w[i] = (uint32_t)seed->bytes[4 * i] | ((uint32_t)seed->bytes[4 * i + 1] << 8) |
                 ((uint32_t)seed->bytes[4 * i + 2] << 16) | ((uint32_t)seed->bytes[4 * i + 3] << 24);
    return k;
}
void secpe_seed_from_u64(uint64_t s, secpe_seed *out) {
    if (!out) return;
    for (int i = 0; i < 32; i++) out->bytes[i] = i < 8 ? (uint8_t)(s >> (8 * i)) : 0;
}
int secpe_keygen(secpe_ctx *ctx, const secpe_seed *seed, const int32_t *rot_steps, int32_t n_rot, secpe_keys **out) {
    return secpe_keygen_sparse(ctx, seed, 0, rot_steps, n_rot, out);
}
int secpe_keygen_sparse(secpe_ctx *ctx, const secpe_seed *seed, int32_t hamming, const int32_t *rot_steps,
                        int32_t n_rot,
                        secpe_keys **out) {
    return guard([&] {
        REQUIRE(ctx && out && (n_rot == 0 || rot_steps), SECPE_EINVAL, "null argument");
        REQUIRE(ctx->c.np >= 1, SECPE_EINVAL, "key generation needs at least one special prime");
        REQUIRE(hamming >= 0 && hamming <= ctx->c.N, SECPE_EINVAL, "Hamming weight out of range");
        auto h = std::make_unique<secpe_keys>();
        h->k = keygen(ctx->c, master_key(seed), rot_steps, n_rot, hamming);
        h->k->owner = &ctx->c;
        ctx->c.live_keys.insert(h->k);
        *out = h.release();
    });
}
void secpe_keys_destroy(secpe_keys *keys) {
    if (!keys) return;
    if (keys->k && keys->k->owner) {
        // captured argmax graphs read this key material: drop them before it is freed (a later keys
        // object at the same address must never replay them)
        Ctx &c = *keys->k->owner;
        if (c.st) cudaStreamSynchronize(c.st);
        c.drop_graphs(keys);
        c.live_keys.erase(keys->k);
    }
    delete keys->k;
    delete keys;
}
int secpe_key_export(const secpe_ctx *ctx, const secpe_keys *keys, int32_t which, uint64_t galois, uint64_t *host_out,
                     size_t n_words) {
    return guard([&] {
        REQUIRE(ctx && keys && host_out, SECPE_EINVAL, "null argument");
        const Ctx &c = ctx->c;
        const DevBuf *b = nullptr;
        if (which == 0) b = &keys->k->s;
        else if (which == 1) b = &keys->k->pk;
        else if (which == 2) b = &keys->k->rlk;
        else if (which == 3) {
            auto it = keys->k->gk.find(galois);
            REQUIRE(it != keys->k->gk.end(), SECPE_ENOKEY, "no Galois key for this element");
            b = &it->second;
        } else
            throw SecpeError{SECPE_EINVAL, "bad key selector"};
        REQUIRE(n_words == b->words, SECPE_EINVAL, "n_words does not match the key size");
        CUDA_CHECK(cudaMemcpyAsync(host_out, b->p, n_words * 8, cudaMemcpyDeviceToHost, c.st));
        CUDA_CHECK(cudaStreamSynchronize(c.st));
    });
}

int secpe_encode(secpe_ctx *ctx, const double *slots, size_t n, double scale, int64_t *coeffs_out) {
    return guard([&] {
        REQUIRE(ctx && coeffs_out && (n == 0 || slots), SECPE_EINVAL, "null argument");
        encode_int(ctx->c, slots, n, scale, coeffs_out);
    });
}
int secpe_encrypt_coeffs(secpe_ctx *ctx, const secpe_keys *keys, const int64_t *coeffs, int32_t level, double scale,
                         const secpe_seed *seed, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && coeffs && out && out->data, SECPE_EINVAL, "null argument");
        REQUIRE(level >= 0 && level < ctx->c.nq, SECPE_EINVAL, "level out of range");
        encrypt_coeffs(ctx->c, *keys->k, coeffs, level, master_key(seed), out->data);
        out->level = level;
        out->scale = scale;
    });
}
int secpe_encrypt(secpe_ctx *ctx, const secpe_keys *keys, const double *slots, size_t n, int32_t level, double scale,
                  const secpe_seed *seed, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && out && out->data && (n == 0 || slots), SECPE_EINVAL, "null argument");
        REQUIRE(level >= 0 && level < ctx->c.nq, SECPE_EINVAL, "level out of range");
        std::vector<i64> m(ctx->c.N);
        encode_int(ctx->c, slots, n, scale, m.data());
        encrypt_coeffs(ctx->c, *keys->k, m.data(), level, master_key(seed), out->data);
        out->level = level;
        out->scale = scale;
    });
}
int secpe_decrypt_residues(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *ct, uint64_t *host_out) {
    return guard([&] {
        REQUIRE(ctx && keys && host_out, SECPE_EINVAL, "null argument");
        decrypt_residues(ctx->c, *keys->k, view_of(ctx->c, ct), host_out);
    });
}
int secpe_decrypt(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *ct, double *slots_out, size_t n) {
    return guard([&] {
        REQUIRE(ctx && keys && slots_out, SECPE_EINVAL, "null argument");
        decrypt_slots(ctx->c, *keys->k, view_of(ctx->c, ct), slots_out, n);
    });
}

static int ntt_common(secpe_ctx *ctx, uint64_t *polys, int32_t n_polys, int32_t first, int32_t n_limbs, bool inv) {
    return guard([&] {
        REQUIRE(ctx && (polys || n_polys == 0), SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        REQUIRE(n_polys >= 0 && n_limbs >= 1 && first >= 0 && first + n_limbs <= c.nprimes(), SECPE_EINVAL,
                "limb range out of the prime chain");
        const long s = (long)n_limbs * c.N;
        LimbMap lm{n_limbs, std::max(0, std::min(n_limbs, c.nq - first)), first, first <= c.nq ? c.nq : first};
        if (first >= c.nq) lm = LimbMap{n_limbs, 0, 0, first};
        ev_ntt(c, RowsArg{polys, 2 * s, s}, n_polys, lm, inv);
    });
}
int secpe_ntt(secpe_ctx *ctx, uint64_t *polys, int32_t n_polys, int32_t first_prime, int32_t n_limbs) {
    return ntt_common(ctx, polys, n_polys, first_prime, n_limbs, false);
}
int secpe_intt(secpe_ctx *ctx, uint64_t *polys, int32_t n_polys, int32_t first_prime, int32_t n_limbs) {
    return ntt_common(ctx, polys, n_polys, first_prime, n_limbs, true);
}

int secpe_add(secpe_ctx *ctx, const secpe_ct *a, const secpe_ct *b, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && out && out->data, SECPE_EINVAL, "null argument");
        CtView va = view_of(ctx->c, a), vb = view_of(ctx->c, b);
        CtView vo = compact_view(ctx->c, out->data, 1, std::min(va.level, vb.level), va.scale);
        ev_addsub(ctx->c, va, vb, vo, false);
        set_out(out, vo);
    });
}
int secpe_sub(secpe_ctx *ctx, const secpe_ct *a, const secpe_ct *b, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && out && out->data, SECPE_EINVAL, "null argument");
        CtView va = view_of(ctx->c, a), vb = view_of(ctx->c, b);
        CtView vo = compact_view(ctx->c, out->data, 1, std::min(va.level, vb.level), va.scale);
        ev_addsub(ctx->c, va, vb, vo, true);
        set_out(out, vo);
    });
}
int secpe_add_const(secpe_ctx *ctx, const secpe_ct *a, double cval, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && out && out->data, SECPE_EINVAL, "null argument");
        CtView va = view_of(ctx->c, a);
        const double Cd = round_half_away(cval * va.scale);
        REQUIRE(std::fabs(Cd) < 4611686018427387904.0, SECPE_EOVERFLOW, "constant exceeds 2^62");
        CtView vo = compact_view(ctx->c, out->data, 1, va.level, va.scale);
        ev_add_int(ctx->c, va, (i64)Cd, vo);
        set_out(out, vo);
    });
}
int secpe_mul_const(secpe_ctx *ctx, const secpe_ct *a, double cval, double target_scale, int32_t target_level,
                    secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && out && out->data, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        CtView va = view_of(c, a);
        const int lv = target_level + 1;
        REQUIRE(target_level >= 0 && lv <= va.level, SECPE_ELEVEL, "not enough levels");
        va.level = lv;
        const double dc = (target_scale * (double)c.primes[lv]) / va.scale;
        const double Cd = round_half_away(cval * dc);
        REQUIRE(std::fabs(Cd) < 4611686018427387904.0, SECPE_EOVERFLOW, "constant exceeds 2^62");
        DevBuf tmp((size_t)c.ct_words(lv), c.st);
        CtView vt = compact_view(c, tmp.p, 1, lv, va.scale * dc);
        ev_mul_int(c, va, (i64)Cd, vt);
        CtView vo = compact_view(c, out->data, 1, target_level, target_scale);
        ev_rescale(c, vt, vo);
        set_out(out, vo);
    });
}
int secpe_mul_mask(secpe_ctx *ctx, const secpe_ct *a, const double *mask_slots, size_t n, double target_scale,
                   secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && out && out->data && mask_slots, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        CtView va = view_of(c, a);
        const int lv = va.level;
        REQUIRE(lv >= 1, SECPE_ELEVEL, "not enough levels");
        const double dm = (target_scale * (double)c.primes[lv]) / va.scale;
        std::vector<i64> M(c.N);
        encode_mask(c, mask_slots, n, dm, M.data());
        DevBuf mi(c.N, c.st), pt((size_t)(lv + 1) * c.N, c.st), tmp((size_t)c.ct_words(lv), c.st);
        CUDA_CHECK(cudaMemcpyAsync(mi.p, M.data(), c.N * 8, cudaMemcpyHostToDevice, c.st));
        k_int_to_rows(c.tab, c.logn, (const i64 *)mi.p, pt.p, LimbMap{lv + 1, lv + 1, 0, 0}, c.st);
        ev_ntt(c, RowsArg{pt.p, 2L * (lv + 1) * c.N, (long)(lv + 1) * c.N}, 1, LimbMap{lv + 1, lv + 1, 0, 0}, false);
        CtView vt = compact_view(c, tmp.p, 1, lv, va.scale * dm);
        ev_mul_plain_ntt(c, va, pt.p, vt);
        CtView vo = compact_view(c, out->data, 1, lv - 1, target_scale);
        ev_rescale(c, vt, vo);
        CUDA_CHECK(cudaStreamSynchronize(c.st));
        set_out(out, vo);
    });
}
int secpe_drop(secpe_ctx *ctx, const secpe_ct *a, int32_t level, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && out && out->data, SECPE_EINVAL, "null argument");
        CtView va = view_of(ctx->c, a);
        REQUIRE(level >= 0 && level <= va.level, SECPE_ELEVEL, "cannot raise the level");
        REQUIRE(out->data != a->data || level == va.level, SECPE_EINVAL, "drop cannot alias");
        CtView vo = compact_view(ctx->c, out->data, 1, level, va.scale);
        ev_copy(ctx->c, va, vo);
        set_out(out, vo);
    });
}
int secpe_mul_relin(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *a, const secpe_ct *b, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && out && out->data, SECPE_EINVAL, "null argument");
        CtView va = view_of(ctx->c, a), vb = view_of(ctx->c, b);
        REQUIRE(va.level == vb.level, SECPE_ELEVEL, "mul_relin needs equal levels");
        CtView vo = compact_view(ctx->c, out->data, 1, va.level, va.scale * vb.scale);
        ev_mul_relin(ctx->c, *keys->k, va, vb, vo);
        set_out(out, vo);
    });
}
int secpe_mul_relin_rescale(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *a, const secpe_ct *b, int32_t n,
                            secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && a && b && out && n >= 1, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        DevBuf sa, sb, so;
        CtView va = batch_in(c, a, n, sa), vb = batch_in(c, b, n, sb);
        REQUIRE(va.level == vb.level, SECPE_ELEVEL, "mul_relin_rescale needs equal levels");
        REQUIRE(va.level >= 1, SECPE_ELEVEL, "no level left to rescale");
        for (int i = 0; i < n; i++)
            REQUIRE(out[i].data != a[i].data && out[i].data != b[i].data, SECPE_EINVAL, "out must not alias");
        CtView vo = batch_out(c, out, n, va.level - 1, (va.scale * vb.scale) / (double)c.primes[va.level], so);
        ev_mul_relin_rescale(c, *keys->k, va, vb, nullptr, 0, vo);
        batch_out_finish(c, out, n, vo, so);
    });
}
int secpe_rotate_batch(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n, int32_t steps,
                       secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && in && out && n >= 1, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        DevBuf si, so;
        CtView vi = batch_in(c, in, n, si);
        for (int i = 0; i < n; i++) REQUIRE(out[i].data != in[i].data, SECPE_EINVAL, "out must not alias");
        CtView vo = batch_out(c, out, n, vi.level, vi.scale, so);
        ev_rotate(c, *keys->k, vi, steps, vo);
        batch_out_finish(c, out, n, vo, so);
    });
}
int secpe_rotate_hoisted(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n,
                         const int32_t *steps, int32_t n_steps, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && in && steps && out && n >= 1 && n_steps >= 1, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        DevBuf si;
        CtView vi = batch_in(c, in, n, si);
        const int lv = out[0].level;
        REQUIRE(lv >= 0 && lv <= vi.level, SECPE_ELEVEL, "output level above the input level");
        std::vector<DevBuf> so(n_steps);
        std::vector<CtView> vo(n_steps);
        for (int s = 0; s < n_steps; s++) {
            for (int i = 0; i < n; i++)
                for (int j = 0; j < n; j++)
                    REQUIRE(out[s * n + i].data != in[j].data, SECPE_EINVAL, "out must not alias in");
            vo[s] = batch_out(c, out + (long)s * n, n, lv, vi.scale, so[s]);
        }
        std::vector<int> st(steps, steps + n_steps);
        ev_rotate_hoisted(c, *keys->k, vi, st.data(), n_steps, vo.data());
        for (int s = 0; s < n_steps; s++) batch_out_finish(c, out + (long)s * n, n, vo[s], so[s]);
    });
}
int secpe_linear_transform(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const uint64_t *pts,
                           const int32_t *steps, int32_t n, double pt_scale, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && in && pts && steps && out && out->data && n >= 1, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        CtView vi = view_of(c, in);
        REQUIRE(vi.level >= 1, SECPE_ELEVEL, "no level left to rescale");
        REQUIRE(out->data != in->data, SECPE_EINVAL, "out must not alias in");
        const double osc = (vi.scale * pt_scale) / (double)c.primes[vi.level];
        CtView vo = compact_view(c, out->data, 1, vi.level - 1, osc);
        std::vector<int> st(steps, steps + n);
        ev_linear_transform(c, *keys->k, vi, pts, (long)(vi.level + 1) * c.N, st.data(), n, vo);
        vo.scale = osc;
        set_out(out, vo);
    });
}
int secpe_mod_raise(secpe_ctx *ctx, const secpe_ct *in, int32_t level, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && in && out && out->data, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        CtView vi = view_of(c, in);
        REQUIRE(vi.level == 0, SECPE_EINVAL, "mod_raise takes a level-0 ciphertext");
        REQUIRE(level >= 1 && level < c.nq, SECPE_EINVAL, "target level out of range");
        REQUIRE(out->data != in->data, SECPE_EINVAL, "out must not alias in");
        CtView vo = compact_view(c, out->data, 1, level, vi.scale);
        ev_mod_raise(c, vi, vo);
        set_out(out, vo);
    });
}
static BootCfg boot_cfg(const Ctx &c, const secpe_boot_cfg *cfg) {
    REQUIRE(cfg && cfg->poly && cfg->cts_re && cfg->cts_im && cfg->stc_re && cfg->stc_im, SECPE_EINVAL,
            "bad bootstrap config");
    REQUIRE(cfg->n1 >= 1 && cfg->n2 >= 1 && (long)cfg->n1 * cfg->n2 == c.N / 2, SECPE_EINVAL, "n1 n2 must be N/2");
    REQUIRE(cfg->r >= 0 && cfg->r <= 30 && cfg->K > 0, SECPE_EINVAL, "bad EvalMod range");
    BootCfg b{cfg->level, cfg->n1, cfg->n2, cfg->r, cfg->K, std::vector<double>(cfg->poly, cfg->poly + 16),
              cfg->cts_re, cfg->cts_im, cfg->stc_re, cfg->stc_im, cfg->cts_scale, cfg->stc_scale};
    REQUIRE(b.level < c.nq && b.level - boot_depth(b) >= 0, SECPE_ELEVEL, "not enough levels for a bootstrap");
    return b;
}
struct secpe_boot {
    std::unique_ptr<BootSetup> b;
};
int secpe_boot_create(secpe_ctx *ctx, int32_t level, double K, int32_t r, int32_t n1, int32_t n2, double in_scale,
                      secpe_boot **out) {
    return guard([&] {
        REQUIRE(ctx && out && in_scale > 0, SECPE_EINVAL, "null argument");
        auto h = std::make_unique<secpe_boot>();
        h->b.reset(boot_setup(ctx->c, level, K, r, n1, n2, in_scale));
        ctx->c.live_boots.insert(h->b.get());
        *out = h.release();
    });
}
int secpe_boot_get_cfg(const secpe_boot *boot, secpe_boot_cfg *cfg) {
    return guard([&] {
        REQUIRE(boot && boot->b && cfg, SECPE_EINVAL, "null argument");
        REQUIRE(!boot->b->fft, SECPE_EINVAL, "factorised material has no dense configuration");
        const BootCfg &b = boot->b->cfg;
        *cfg = secpe_boot_cfg{b.level, b.n1, b.n2, b.K, b.r, b.poly.data(), b.cts_re, b.cts_im, b.cts_scale,
                              b.stc_re, b.stc_im, b.stc_scale};
    });
}
// Synchronises the owning context's stream and drops every CUDA graph that reads this material.
void secpe_boot_destroy(secpe_boot *boot) {
    if (!boot) return;
    if (boot->b && boot->b->ctx) {
        Ctx &c = *boot->b->ctx;
        if (c.st) cudaStreamSynchronize(c.st);
        c.drop_graphs(boot->b.get());
        c.live_boots.erase(boot->b.get());
    }
    delete boot;
}
int secpe_boot_export(secpe_ctx *ctx, const secpe_boot *boot, int32_t which, uint64_t *host_out, size_t n_words) {
    return guard([&] {
        REQUIRE(ctx && boot && boot->b && host_out && which >= 0 && which < 4, SECPE_EINVAL, "bad argument");
        const BootSetup &b = *boot->b;
        const DevBuf *m[4] = {&b.cts_re, &b.cts_im, &b.stc_re, &b.stc_im};
        REQUIRE(n_words == m[which]->words, SECPE_EINVAL, "n_words does not match the matrix size");
        CUDA_CHECK(cudaMemcpyAsync(host_out, m[which]->p, n_words * 8, cudaMemcpyDeviceToHost, ctx->c.st));
        CUDA_CHECK(cudaStreamSynchronize(ctx->c.st));
    });
}
static LtStage lt_stage(const Ctx &c, const secpe_lt_stage &s) {
    LtStage t;
    if (s.n_giant > 0) {
        REQUIRE(s.n_baby >= 1 && s.baby && s.giant && s.pts, SECPE_EINVAL, "bad baby-step giant-step stage");
        t.baby.assign(s.baby, s.baby + s.n_baby);
        t.giant.assign(s.giant, s.giant + s.n_giant);
    } else {
        REQUIRE(s.n_diag >= 1 && s.steps && s.pts, SECPE_EINVAL, "bad transform stage");
        t.steps.assign(s.steps, s.steps + s.n_diag);
    }
    t.pts = s.pts;
    t.scale = s.pt_scale;
    (void)c;
    return t;
}
static void check_fft_keys(const Ctx &c, const secpe_keys *keys, const FftBootCfg &b) {
    auto chk = [&](const LtStage &s) {
        for (const auto *v : {&s.steps, &s.baby, &s.giant})
            for (int st : *v)
                REQUIRE(keys->k->gk.count(galois_elt(c, st)) || galois_elt(c, st) == 1, SECPE_ENOKEY,
                        "no Galois key for a transform step");
    };
    for (auto &s : b.cts) chk(s);
    for (auto &s : b.stc) chk(s);
    chk(b.cts_im);
    chk(b.stc_im);
    REQUIRE(keys->k->gk.count(galois_elt(c, kConjStep)), SECPE_ENOKEY, "no conjugation key");
}
static void bootstrap_fft_views(Ctx &c, const secpe_keys *keys, const secpe_ct *in, const FftBootCfg &b,
                                secpe_ct *out, const void *material = nullptr) {
    REQUIRE(b.level < c.nq && b.level - fft_boot_depth(b) >= 0, SECPE_ELEVEL, "not enough levels for a bootstrap");
    CtView vi = view_of(c, in);
    REQUIRE(vi.level == 0, SECPE_EINVAL, "bootstrap takes a level-0 ciphertext");
    REQUIRE(out->data != in->data, SECPE_EINVAL, "out must not alias in");
    check_fft_keys(c, keys, b);
    CtView vo = compact_view(c, out->data, 1, b.level - fft_boot_depth(b), 0.0);
    // library-built material (stable device memory): CUDA graph as secpe_enc_argmax
    char k[192];
    snprintf(k, sizeof k, "boot/%p/%p/%s/%p/%p", (void *)vi.data, (void *)vo.data, dkey(vi.scale).c_str(), material,
             (const void *)keys);
    graphed(c, material != nullptr, k, keys, material, vo, [&] { run_bootstrap_fft(c, *keys->k, vi, b, vo); });
    set_out(out, vo);
}
static FftBootCfg fft_cfg_of(const Ctx &c, const secpe_boot_fft_cfg *cfg) {
    REQUIRE(cfg && cfg->poly && cfg->cts && cfg->stc, SECPE_EINVAL, "null bootstrap configuration");
    REQUIRE(cfg->n_cts >= 1 && cfg->n_stc == cfg->n_cts, SECPE_EINVAL, "stage counts");
    REQUIRE(cfg->r >= 0 && cfg->r <= 30 && cfg->K > 0, SECPE_EINVAL, "bad EvalMod range");
    FftBootCfg b;
    b.level = cfg->level;
    b.r = cfg->r;
    b.K = cfg->K;
    b.poly.assign(cfg->poly, cfg->poly + 16);
    for (int i = 0; i < cfg->n_cts; i++) b.cts.push_back(lt_stage(c, cfg->cts[i]));
    for (int i = 0; i < cfg->n_stc; i++) b.stc.push_back(lt_stage(c, cfg->stc[i]));
    b.cts_im = lt_stage(c, cfg->cts_im);
    b.stc_im = lt_stage(c, cfg->stc_im);
    return b;
}
int secpe_bootstrap_fft(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const secpe_boot_fft_cfg *cfg,
                        secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && in && out && out->data, SECPE_EINVAL, "null argument");
        bootstrap_fft_views(ctx->c, keys, in, fft_cfg_of(ctx->c, cfg), out);
    });
}
// N4 (R38): argmax with bootstrapping, one ciphertext after another
static void argmax_boot_views(Ctx &c, const secpe_keys *keys, const secpe_ct *in, int n_in, const secpe_layout *layout,
                              const secpe_sign_cfg *scfg, const FftBootCfg &b, double boot_scale, int prompt_cts,
                              secpe_ct *out, const void *material = nullptr) {
    REQUIRE(keys && in && out && n_in >= 1 && boot_scale > 0, SECPE_EINVAL, "null argument");
    REQUIRE(prompt_cts >= 1 && n_in % prompt_cts == 0, SECPE_EINVAL, "n_in must be a multiple of prompt_cts");
    Layout lay = layout_of(c, layout);
    SignCfg sc = sign_cfg(scfg);
    check_fft_keys(c, keys, b);
    const int n_out = n_in / prompt_cts;
    DevBuf inb, outb;
    CtView vin = batch_in(c, in, n_in, inb);
    for (int i = 0; i < n_out; i++)
        for (int j = 0; j < n_in; j++) REQUIRE(out[i].data != in[j].data, SECPE_EINVAL, "out must not alias in");
    const int ol = argmax_boot_level(lay, sc, b, vin.level);
    CtView vout = batch_out(c, out, n_out, ol, c.scale, outb);
    char k[256];
    snprintf(k, sizeof k, "argmax_boot/%p/%p/%d/%d/%d/%s/%d/%d/%d/%d/%s/%p/%p/", (void *)vin.data, (void *)vout.data,
             n_in, prompt_cts, vin.level, dkey(vin.scale).c_str(), lay.queries, lay.prompts, lay.classes, lay.block,
             dkey(boot_scale).c_str(), material, (const void *)keys);
    std::string key = k;
    for (auto &stg : sc.stages)
        for (double x : stg) key += dkey(x) + ",";
    // graphable only on the caller's own (unstaged) buffers and library-built material
    graphed(c, material != nullptr && !inb.p && !outb.p, key, keys, material, vout,
            [&] { run_argmax_boot(c, *keys->k, vin, lay, sc, b, boot_scale, prompt_cts, vout); });
    batch_out_finish(c, out, n_out, vout, outb);
}
int secpe_argmax_boot_info(secpe_ctx *ctx, const secpe_layout *layout, const secpe_sign_cfg *cfg,
                           const secpe_boot *boot, int32_t in_level, int32_t *out_level) {
    return guard([&] {
        REQUIRE(ctx && boot && boot->b && boot->b->fft && out_level, SECPE_EINVAL, "null argument");
        *out_level = argmax_boot_level(layout_of(ctx->c, layout), sign_cfg(cfg), boot->b->fcfg, in_level);
    });
}
int secpe_enc_argmax_boot(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n_in,
                          int32_t prompt_cts, const secpe_layout *layout, const secpe_sign_cfg *cfg,
                          const secpe_boot *boot, double boot_scale, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && boot && boot->b && boot->b->fft, SECPE_EINVAL, "needs factorised bootstrap material");
        argmax_boot_views(ctx->c, keys, in, n_in, layout, cfg, boot->b->fcfg, boot_scale, prompt_cts, out,
                          boot->b.get());
    });
}
int secpe_enc_argmax_boot_cfg(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n_in,
                              int32_t prompt_cts, const secpe_layout *layout, const secpe_sign_cfg *cfg,
                              const secpe_boot_fft_cfg *bcfg, double boot_scale, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx, SECPE_EINVAL, "null argument");
        argmax_boot_views(ctx->c, keys, in, n_in, layout, cfg, fft_cfg_of(ctx->c, bcfg), boot_scale, prompt_cts, out);
    });
}
int secpe_boot_create_fft(secpe_ctx *ctx, int32_t level, double K, int32_t r, const int32_t *groups,
                          int32_t n_groups, double in_scale, int32_t bsgs, secpe_boot **out) {
    return guard([&] {
        REQUIRE(ctx && out && groups && n_groups >= 1 && in_scale > 0, SECPE_EINVAL, "null argument");
        auto h = std::make_unique<secpe_boot>();
        h->b.reset(boot_setup_fft(ctx->c, level, K, r, std::vector<int>(groups, groups + n_groups), in_scale,
                                  bsgs != 0));
        ctx->c.live_boots.insert(h->b.get());
        *out = h.release();
    });
}
int32_t secpe_boot_steps(const secpe_boot *boot, int32_t *steps, int32_t cap) {
    if (!boot || !boot->b) return -1;
    const BootSetup &b = *boot->b;
    std::set<int> st;
    if (b.fft) {
        auto add = [&](const LtStage &s) {
            for (const auto *v : {&s.steps, &s.baby, &s.giant})
                for (int x : *v)
                    if (galois_elt(*b.ctx, x) != 1) st.insert(x);
        };
        for (auto &s : b.fcfg.cts) add(s);
        for (auto &s : b.fcfg.stc) add(s);
        add(b.fcfg.cts_im);
        add(b.fcfg.stc_im);
    } else {
        for (int j = 1; j < b.cfg.n1; j++) st.insert(j);
        for (int g = 1; g < b.cfg.n2; g++) st.insert(g * b.cfg.n1);
    }
    std::vector<int> v(st.begin(), st.end());
    v.push_back(kConjStep);
    for (int i = 0; i < (int)v.size() && i < cap && steps; i++) steps[i] = v[i];
    return (int32_t)v.size();
}
int32_t secpe_boot_levels(const secpe_boot *boot, int32_t *raise_level) {
    if (!boot || !boot->b) return -1;
    const BootSetup &b = *boot->b;
    if (raise_level) *raise_level = b.fft ? b.fcfg.level : b.cfg.level;
    return b.fft ? fft_boot_depth(b.fcfg) : boot_depth(b.cfg);
}
int secpe_bootstrap_boot(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const secpe_boot *boot,
                         secpe_ct *out) {
    if (boot && boot->b && !boot->b->fft) {
        secpe_boot_cfg cfg;
        const int rc = secpe_boot_get_cfg(boot, &cfg);
        return rc ? rc : secpe_bootstrap(ctx, keys, in, &cfg, out);
    }
    return guard([&] {
        REQUIRE(ctx && keys && in && out && out->data && boot && boot->b, SECPE_EINVAL, "null argument");
        bootstrap_fft_views(ctx->c, keys, in, boot->b->fcfg, out, boot->b.get());
    });
}
int secpe_bootstrap_boot_batch(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n,
                               const secpe_boot *boot, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && in && out && n >= 1 && boot && boot->b && boot->b->fft, SECPE_EINVAL,
                "needs factorised bootstrap material");
        Ctx &c = ctx->c;
        const FftBootCfg &b = boot->b->fcfg;
        REQUIRE(b.level < c.nq && b.level - fft_boot_depth(b) >= 0, SECPE_ELEVEL, "not enough levels");
        DevBuf inb, outb;
        CtView vin = batch_in(c, in, n, inb);
        REQUIRE(vin.level == 0, SECPE_EINVAL, "bootstrap takes level-0 ciphertexts");
        no_overlap(in, n, c.ct_words(0), out, n, c.ct_words(b.level - fft_boot_depth(b)));
        check_fft_keys(c, keys, b);
        CtView vout = batch_out(c, out, n, b.level - fft_boot_depth(b), 0.0, outb);
        char k[192];
        snprintf(k, sizeof k, "bootb/%p/%p/%d/%s/%p/%p", (void *)vin.data, (void *)vout.data, n, dkey(vin.scale).c_str(),
                 (const void *)boot->b.get(), (const void *)keys);
        graphed(c, !inb.p && !outb.p, k, keys, boot->b.get(), vout,
                [&] { run_bootstrap_fft(c, *keys->k, vin, b, vout); });
        batch_out_finish(c, out, n, vout, outb);
    });
}
static const LtStage &boot_stage(const FftBootCfg &f, int kind, int idx, int &lv) {
    const int mc = (int)f.cts.size(), base = f.level - mc - 6 - f.r;
    REQUIRE(kind >= 0 && kind < 4, SECPE_EINVAL, "stage kind");
    if (kind == 0 || kind == 2)
        REQUIRE(idx >= 0 && idx < (kind == 0 ? (int)f.cts.size() : (int)f.stc.size()), SECPE_EINVAL, "stage index");
    lv = kind == 0 ? f.level - idx : kind == 1 ? f.level - (mc - 1) : kind == 2 ? base - idx : base;
    return kind == 0 ? f.cts[idx] : kind == 1 ? f.cts_im : kind == 2 ? f.stc[idx] : f.stc_im;
}
int secpe_boot_stage_export_bsgs(secpe_ctx *ctx, const secpe_boot *boot, int32_t kind, int32_t idx, int32_t *n_baby,
                                 int32_t *n_giant, int32_t *baby, int32_t *giant, uint64_t *host_out, size_t n_words) {
    return guard([&] {
        REQUIRE(ctx && boot && boot->b && boot->b->fft && n_baby && n_giant, SECPE_EINVAL, "bad argument");
        int lv = 0;
        const LtStage &s = boot_stage(boot->b->fcfg, kind, idx, lv);
        REQUIRE(!s.giant.empty(), SECPE_EINVAL, "not a baby-step giant-step stage");
        *n_baby = (int)s.baby.size();
        *n_giant = (int)s.giant.size();
        if (baby) std::copy(s.baby.begin(), s.baby.end(), baby);
        if (giant) std::copy(s.giant.begin(), s.giant.end(), giant);
        REQUIRE(!host_out || n_words == (size_t)*n_baby * *n_giant * (lv + 1) * ctx->c.N, SECPE_EINVAL,
                "n_words does not match the stage size");
        if (host_out) {
            CUDA_CHECK(cudaMemcpyAsync(host_out, s.pts, n_words * 8, cudaMemcpyDeviceToHost, ctx->c.st));
            CUDA_CHECK(cudaStreamSynchronize(ctx->c.st));
        }
    });
}
int secpe_boot_stage_export(secpe_ctx *ctx, const secpe_boot *boot, int32_t kind, int32_t idx, int32_t *n_diag,
                            int32_t *steps, uint64_t *host_out, size_t n_words) {
    return guard([&] {
        REQUIRE(ctx && boot && boot->b && boot->b->fft && n_diag && kind >= 0 && kind < 4, SECPE_EINVAL,
                "bad argument");
        const FftBootCfg &f = boot->b->fcfg;
        const LtStage *s = nullptr;
        if (kind == 1) s = &f.cts_im;
        if (kind == 3) s = &f.stc_im;
        if (kind == 0) {
            REQUIRE(idx >= 0 && idx < (int)f.cts.size(), SECPE_EINVAL, "stage index");
            s = &f.cts[idx];
        }
        if (kind == 2) {
            REQUIRE(idx >= 0 && idx < (int)f.stc.size(), SECPE_EINVAL, "stage index");
            s = &f.stc[idx];
        }
        *n_diag = (int)s->steps.size();
        if (steps) std::copy(s->steps.begin(), s->steps.end(), steps);
        const int mc = (int)f.cts.size(), base = f.level - mc - 6 - f.r;
        const int lv = kind == 0 ? f.level - idx : kind == 1 ? f.level - (mc - 1) : kind == 2 ? base - idx : base;
        REQUIRE(!host_out || n_words == (size_t)*n_diag * (lv + 1) * ctx->c.N, SECPE_EINVAL,
                "n_words does not match the stage size");
        if (host_out) {
            CUDA_CHECK(cudaMemcpyAsync(host_out, s->pts, n_words * 8, cudaMemcpyDeviceToHost, ctx->c.st));
            CUDA_CHECK(cudaStreamSynchronize(ctx->c.st));
        }
    });
}
int32_t secpe_boot_depth(const secpe_boot_cfg *cfg) { return cfg ? 8 + cfg->r : -1; }
int secpe_bootstrap(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const secpe_boot_cfg *cfg,
                    secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && in && out && out->data, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        BootCfg b = boot_cfg(c, cfg);
        CtView vi = view_of(c, in);
        REQUIRE(vi.level == 0, SECPE_EINVAL, "bootstrap takes a level-0 ciphertext");
        REQUIRE(out->data != in->data, SECPE_EINVAL, "out must not alias in");
        for (int j = 1; j < b.n1; j++)
            REQUIRE(keys->k->gk.count(galois_elt(c, j)), SECPE_ENOKEY, "no Galois key for a baby step");
        for (int g = 1; g < b.n2; g++)
            REQUIRE(keys->k->gk.count(galois_elt(c, g * b.n1)), SECPE_ENOKEY, "no Galois key for a giant step");
        REQUIRE(keys->k->gk.count(galois_elt(c, kConjStep)), SECPE_ENOKEY, "no conjugation key");
        CtView vo = compact_view(c, out->data, 1, b.level - boot_depth(b), 0.0);
        run_bootstrap(c, *keys->k, vi, b, vo);
        set_out(out, vo);
    });
}
int secpe_linear_transform_bsgs(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const uint64_t *pts,
                                int32_t n1, int32_t n2, double pt_scale, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && in && pts && out && out->data && n1 >= 1 && n2 >= 1, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        CtView vi = view_of(c, in);
        REQUIRE(vi.level >= 1, SECPE_ELEVEL, "no level left to rescale");
        REQUIRE(out->data != in->data, SECPE_EINVAL, "out must not alias in");
        for (int j = 1; j < n1; j++)
            REQUIRE(keys->k->gk.count(galois_elt(c, j)), SECPE_ENOKEY, "no Galois key for a baby step");
        for (int g = 1; g < n2; g++)
            REQUIRE(keys->k->gk.count(galois_elt(c, g * n1)), SECPE_ENOKEY, "no Galois key for a giant step");
        const double osc = (vi.scale * pt_scale) / (double)c.primes[vi.level];
        CtView vo = compact_view(c, out->data, 1, vi.level - 1, osc);
        ev_linear_transform_bsgs(c, *keys->k, vi, pts, (long)(vi.level + 1) * c.N, n1, n2, vo);
        vo.scale = osc;
        set_out(out, vo);
    });
}
int secpe_rescale(secpe_ctx *ctx, const secpe_ct *in, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && out && out->data, SECPE_EINVAL, "null argument");
        CtView vi = view_of(ctx->c, in);
        REQUIRE(vi.level >= 1, SECPE_ELEVEL, "no level left to rescale");
        CtView vo = compact_view(ctx->c, out->data, 1, vi.level - 1, vi.scale / (double)ctx->c.primes[vi.level]);
        ev_rescale(ctx->c, vi, vo);
        set_out(out, vo);
    });
}
int secpe_rotate(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t steps, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && out && out->data, SECPE_EINVAL, "null argument");
        CtView vi = view_of(ctx->c, in);
        CtView vo = compact_view(ctx->c, out->data, 1, vi.level, vi.scale);
        ev_rotate(ctx->c, *keys->k, vi, steps, vo);
        set_out(out, vo);
    });
}

int secpe_sign_poly(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, const secpe_sign_cfg *cfg,
                    double target_scale, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && out && out->data, SECPE_EINVAL, "null argument");
        SignCfg sc = sign_cfg(cfg);
        CtView vi = view_of(ctx->c, in);
        const int ol = vi.level - sign_depth(sc);
        REQUIRE(ol >= 0, SECPE_ELEVEL, "not enough levels for the sign polynomial");
        CtView vo = compact_view(ctx->c, out->data, 1, ol, target_scale);
        run_sign(ctx->c, *keys->k, vi, sc, target_scale, vo);
        set_out(out, vo);
    });
}
int32_t secpe_sign_depth(const secpe_sign_cfg *cfg) {
    int32_t d = -1;
    const int rc = guard([&] { d = sign_depth(sign_cfg(cfg)); });
    return rc == SECPE_OK ? d : rc;
}
int secpe_argmax_info(secpe_ctx *ctx, const secpe_layout *layout, const secpe_sign_cfg *cfg, int32_t in_level,
                      int32_t *out_level, double *out_scale) {
    return guard([&] {
        REQUIRE(ctx && out_level && out_scale, SECPE_EINVAL, "null argument");
        Layout lay = layout_of(ctx->c, layout);
        SignCfg sc = sign_cfg(cfg);
        const int ol = in_level - argmax_depth(lay, sc);
        REQUIRE(ol >= 0, SECPE_ELEVEL, "not enough levels for the argmax circuit");
        *out_level = ol;
        *out_scale = ctx->c.scale;
    });
}
// One batched argmax on device views.  CUDA graph: the circuit is data-independent, so a call on the
// same buffers replays the graph captured on the previous such call (the first call runs eagerly and
// fills the mask cache); the legacy / per-thread default streams cannot be captured: eager there.
static void argmax_views(Ctx &c, const secpe_keys *keys, const CtView &vin, const Layout &lay, const SignCfg &sc,
                         CtView &vout, bool buffers_fixed) {
    char b[256];
    snprintf(b, sizeof b, "%p/%p/%d/%d/%s/%d/%d/%d/%d/%p/", (void *)vin.data, (void *)vout.data, vin.n, vin.level,
             dkey(vin.scale).c_str(), lay.queries, lay.prompts, lay.classes, lay.block, (const void *)keys);
    std::string key = b;
    for (auto &stg : sc.stages)
        for (double x : stg) key += dkey(x) + ",";
    graphed(c, buffers_fixed, key, keys, nullptr, vout, [&] { run_argmax(c, *keys->k, vin, lay, sc, vout); });
}

int secpe_enc_argmax(secpe_ctx *ctx, const secpe_keys *keys, const secpe_ct *in, int32_t n_in,
                     const secpe_layout *layout, const secpe_sign_cfg *cfg, secpe_ct *out) {
    return guard([&] {
        REQUIRE(ctx && keys && in && out && n_in >= 1, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        Layout lay = layout_of(c, layout);
        SignCfg sc = sign_cfg(cfg);
        const int lv = in[0].level;
        for (int i = 0; i < n_in; i++) {
            REQUIRE(in[i].data && out[i].data, SECPE_EINVAL, "null ciphertext data");
            REQUIRE(in[i].level == lv && in[i].scale == in[0].scale, SECPE_EINVAL,
                    "batch inputs must share level and scale");
        }
        const int ol = lv - argmax_depth(lay, sc);
        REQUIRE(ol >= 0, SECPE_ELEVEL, "not enough levels for the argmax circuit");
        const long cw = c.ct_words(lv), ow = c.ct_words(ol);
        no_overlap(in, n_in, cw, out, n_in, ow);
        // batch view: reuse the caller's memory if the inputs are laid out contiguously
        bool contiguous = true;
        for (int i = 1; i < n_in; i++) contiguous &= in[i].data == in[0].data + (long)i * cw;
        DevBuf inb, outb;
        CtView vin = compact_view(c, in[0].data, n_in, lv, in[0].scale);
        if (!contiguous) {
            inb = DevBuf((size_t)n_in * cw, c.st);
            for (int i = 0; i < n_in; i++)
                CUDA_CHECK(cudaMemcpyAsync(inb.p + (long)i * cw, in[i].data, cw * 8, cudaMemcpyDeviceToDevice, c.st));
            vin.data = inb.p;
        }
        bool ocontig = true;
        for (int i = 1; i < n_in; i++) ocontig &= out[i].data == out[0].data + (long)i * ow;
        CtView vout = compact_view(c, out[0].data, n_in, ol, c.scale);
        if (!ocontig) {
            outb = DevBuf((size_t)n_in * ow, c.st);
            vout.data = outb.p;
        }
        argmax_views(c, keys, vin, lay, sc, vout, contiguous && ocontig);
        // result level/scale are those of the circuit (recomputed cheaply without running it)
        vout.level = ol;
        if (!ocontig)
            for (int i = 0; i < n_in; i++)
                CUDA_CHECK(
                    cudaMemcpyAsync(out[i].data, outb.p + (long)i * ow, ow * 8, cudaMemcpyDeviceToDevice, c.st));
        for (int i = 0; i < n_in; i++) set_out(&out[i], vout);
    });
}

int secpe_enc_argmax_host(secpe_ctx *ctx, const secpe_keys *keys, const uint64_t *h_in, int32_t n_in,
                          int32_t level, double scale, const secpe_layout *layout, const secpe_sign_cfg *cfg,
                          uint64_t *h_out, int32_t chunk, int32_t *out_level, double *out_scale) {
    return guard([&] {
        REQUIRE(ctx && keys && h_in && h_out && n_in >= 1, SECPE_EINVAL, "null argument");
        Ctx &c = ctx->c;
        REQUIRE(level >= 0 && level <= c.L(), SECPE_ELEVEL, "level out of range");
        REQUIRE(c.st != cudaStreamLegacy && c.st != cudaStreamPerThread, SECPE_EINVAL,
                "secpe_enc_argmax_host needs an explicit (non-default) context stream");
        Layout lay = layout_of(c, layout);
        SignCfg sc = sign_cfg(cfg);
        const int ol = level - argmax_depth(lay, sc);
        REQUIRE(ol >= 0, SECPE_ELEVEL, "not enough levels for the argmax circuit");
        if (chunk <= 0) chunk = 16;  // (16 ciphertexts per launch sequence: the measured sweet spot)
        chunk = std::min(chunk, n_in);
        const long cw = c.ct_words(level), ow = c.ct_words(ol);
        Ctx::HostPipe &hp = c.pipe;
        if (!hp.cp) {
            CUDA_CHECK(cudaStreamCreateWithFlags(&hp.cp, cudaStreamNonBlocking));
            for (int s = 0; s < 2; s++) {
                CUDA_CHECK(cudaEventCreateWithFlags(&hp.loaded[s], cudaEventDisableTiming));
                CUDA_CHECK(cudaEventCreateWithFlags(&hp.freed[s], cudaEventDisableTiming));
                CUDA_CHECK(cudaEventRecord(hp.freed[s], c.st));
            }
        }
        if (hp.in_words < (size_t)chunk * cw || hp.out_words < (size_t)chunk * ow) {
            // grow both slots (after every earlier use of them has finished on the context stream)
            CUDA_CHECK(cudaStreamWaitEvent(c.st, hp.freed[0], 0));
            CUDA_CHECK(cudaStreamWaitEvent(c.st, hp.freed[1], 0));
            hp.in_words = std::max(hp.in_words, (size_t)chunk * cw);
            hp.out_words = std::max(hp.out_words, (size_t)chunk * ow);
            for (int s = 0; s < 2; s++) {
                hp.in[s] = DevBuf(hp.in_words, c.st);
                hp.out[s] = DevBuf(hp.out_words, c.st);
                CUDA_CHECK(cudaEventRecord(hp.freed[s], c.st));
            }
        }
        double osc = c.scale;
        for (int i0 = 0; i0 < n_in; i0 += chunk) {
            const int n = std::min(chunk, n_in - i0);
            const int s = hp.next++ & 1;
            // copy stream: wait until slot s is free, then load this chunk (overlaps the other slot's compute)
            CUDA_CHECK(cudaStreamWaitEvent(hp.cp, hp.freed[s], 0));
            CUDA_CHECK(cudaMemcpyAsync(hp.in[s].p, h_in + (long)i0 * cw, (size_t)n * cw * 8, cudaMemcpyHostToDevice,
                                       hp.cp));
            CUDA_CHECK(cudaEventRecord(hp.loaded[s], hp.cp));
            // context stream: compute on slot s, copy the result back, release the slot
            CUDA_CHECK(cudaStreamWaitEvent(c.st, hp.loaded[s], 0));
            CtView vin = compact_view(c, hp.in[s].p, n, level, scale);
            CtView vout = compact_view(c, hp.out[s].p, n, ol, c.scale);
            argmax_views(c, keys, vin, lay, sc, vout, true);
            osc = vout.scale;
            CUDA_CHECK(cudaMemcpyAsync(h_out + (long)i0 * ow, hp.out[s].p, (size_t)n * ow * 8, cudaMemcpyDeviceToHost,
                                       c.st));
            CUDA_CHECK(cudaEventRecord(hp.freed[s], c.st));
        }
        if (out_level) *out_level = ol;
        if (out_scale) *out_scale = osc;
    });
}

int secpe_oplog_enable(secpe_ctx *ctx, int32_t on) {
    return guard([&] {
        REQUIRE(ctx, SECPE_EINVAL, "null ctx");
        ctx->c.log_on = on != 0;
    });
}
int64_t secpe_oplog_get(secpe_ctx *ctx, char *buf, size_t cap) {
    if (!ctx) return -1;
    const std::string &s = ctx->c.oplog;
    if (buf && cap) {
        const size_t n = std::min(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return (int64_t)s.size();
}
int secpe_oplog_clear(secpe_ctx *ctx) {
    return guard([&] {
        REQUIRE(ctx, SECPE_EINVAL, "null ctx");
        ctx->c.oplog.clear();
    });
}
int secpe_profile_begin(secpe_ctx *ctx) {
    return guard([&] {
        REQUIRE(ctx, SECPE_EINVAL, "null ctx");
        Prof &p = ctx->c.prof;
        CUDA_CHECK(cudaStreamSynchronize(ctx->c.st));
        p.used = 0;
        p.spans.clear();
        p.on = true;
    });
}
int secpe_profile_end(secpe_ctx *ctx, double *out, int32_t n_out) {
    return guard([&] {
        REQUIRE(ctx && out && n_out >= 12, SECPE_EINVAL, "need out[12]");
        Prof &p = ctx->c.prof;
        CUDA_CHECK(cudaStreamSynchronize(ctx->c.st));
        p.on = false;
        for (int i = 0; i < n_out; i++) out[i] = 0;
        // development: SECPE_PROF_DUMP=<file> appends every span (kind, units, bytes, ms)
        const char *dump = getenv("SECPE_PROF_DUMP");
        FILE *df = dump ? fopen(dump, "a") : nullptr;
        for (const auto &s : p.spans) {
            float ms = 0;
            CUDA_CHECK(cudaEventElapsedTime(&ms, p.pool[s.a], p.pool[s.b]));
            if (df) fprintf(df, "%d %.1f %.0f %.6f\n", s.kind, (double)s.units, s.bytes, ms);
            if (3 * s.kind + 2 >= n_out) continue;  // stage spans (kinds 4..8) only when asked for
            out[3 * s.kind + 0] += ms;
            out[3 * s.kind + 1] += s.bytes;
            out[3 * s.kind + 2] += (double)s.units;
        }
        if (df) fclose(df);
        p.spans.clear();
        p.used = 0;
    });
}
int32_t secpe_ntt_mode(int32_t mode) { return ntt_fused_mode(mode); }
int secpe_opcounts(secpe_ctx *ctx, int64_t *counts, int32_t reset) {
    return guard([&] {
        REQUIRE(ctx && counts, SECPE_EINVAL, "null argument");
        Counters &k = ctx->c.cnt;
        const long long v[8] = {k.ntt_limbs, k.keyswitch, k.rescale, k.rotate, k.mulct, k.mulconst, k.launches, k.sign};
        for (int i = 0; i < 8; i++) counts[i] = v[i];
        if (reset) k = Counters{};
    });
}

}  // extern "C"
