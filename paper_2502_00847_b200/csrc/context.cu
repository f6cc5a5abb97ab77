// context.cu -- parameters, precomputed tables and per-level constants (host side of the product).
//
// Everything here is computed by the library itself (independent of oracle/): prime chains
// (reading R1), psi = smallest primitive 2N-th root of unity (reading R4), twiddle tables with
// Shoup companions, Barrett constants, CRT / fast-base-conversion constants for hybrid key
// switching (R10, R11) and rescale (R12), and the Gaussian CDT in quad precision (R6).
#include <quadmath.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "context.h"

// ---------------------------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------------------------
DevBuf::DevBuf(size_t w, cudaStream_t s) : words(w), st(s) {
    if (w) CUDA_CHECK(cudaMallocAsync((void **)&p, w * sizeof(u64), s));
}
DevBuf::~DevBuf() {
    if (p) cudaFreeAsync(p, st);
}
DevBuf &DevBuf::operator=(DevBuf &&o) noexcept {
    if (this != &o) {
        if (p) cudaFreeAsync(p, st);
        p = o.p;
        words = o.words;
        st = o.st;
        o.p = nullptr;
        o.words = 0;
    }
    return *this;
}

// split-30 packed constant for the base-conversion MACs (ks.cu): (c >> 30) << 32 | (c mod 2^30)
static u64 pack30(u64 c) { return ((c >> 30) << 32) | (c & ((1ULL << 30) - 1)); }

static DevBuf upload(const std::vector<u64> &h, cudaStream_t st) {
    DevBuf b(std::max<size_t>(h.size(), 1), st);
    if (!h.empty()) CUDA_CHECK(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(u64), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaStreamSynchronize(st));  // h may be a temporary
    return b;
}

// ---------------------------------------------------------------------------------------------
// host modular arithmetic
// ---------------------------------------------------------------------------------------------
u64 h_mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
u64 h_powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    for (; e; e >>= 1) {
        if (e & 1) r = h_mulmod(r, a, q);
        a = h_mulmod(a, a, q);
    }
    return r;
}
u64 h_invmod(u64 a, u64 q) { return h_powmod(a % q, q - 2, q); }
u64 h_shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
u64 h_smod128(i128 v, u64 q) {
    const u128 a = (u128)(v < 0 ? -v : v);
    const u64 m = (u64)(a % q);
    return (v < 0 && m) ? q - m : m;
}
u64 h_smod(i64 v, u64 q) {
    if (v >= 0) return (u64)v % q;
    u64 m = (u64)(-(v + 1)) % q;  // (|v| - 1) mod q
    m = (m + 1) % q;
    return m ? q - m : 0;
}

bool h_is_prime(u64 n) {
    if (n < 2) return false;
    static const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (u64 p : small) {
        if (n == p) return true;
        if (n % p == 0) return false;
    }
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) d >>= 1, s++;
    for (u64 a : small) {
        u64 x = h_powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool witness = true;
        for (int r = 1; r < s && witness; r++) {
            x = h_mulmod(x, x, n);
            if (x == n - 1) witness = false;
        }
        if (witness) return false;
    }
    return true;
}

// mode 0: candidates 2^b + 1 + k 2N ordered by distance to 2^b (k = 0, -1, 1, -2, 2, ...);
// mode 1: largest below 2^b, descending.
int h_gen_primes(int bits, int count, int logn, int mode, const u64 *ex, int nex, u64 *out) {
    const u64 base = (u64)1 << bits, step = (u64)2 << logn;
    int got = 0;
    auto take = [&](u64 c) {
        if (got < count && h_is_prime(c) && std::find(ex, ex + nex, c) == ex + nex) out[got++] = c;
    };
    for (u64 k = 0; got < count && k < ((u64)1 << 40); k++) {
        if (mode == 0) {
            take(base + 1 + k * step);
            take(base + 1 - (k + 1) * step);
        } else {
            take(base + 1 - (k + 1) * step);
        }
    }
    return got;
}

// psi: generator g of Z_q^* from the factorisation of q-1, psi0 = g^((q-1)/2N), then the minimum
// over all primitive 2N-th roots psi0^(2j+1).
u64 h_find_psi(u64 q, int logn) {
    const u64 two_n = (u64)2 << logn;
    std::vector<u64> f;
    u64 m = q - 1;
    for (u64 p = 2; p * p <= m; p += (p == 2 ? 1 : 2)) {
        if (m % p == 0) {
            f.push_back(p);
            while (m % p == 0) m /= p;
        }
    }
    if (m > 1) f.push_back(m);
    u64 g = 2;
    for (;; g++) {
        bool gen = true;
        for (u64 p : f)
            if (h_powmod(g, (q - 1) / p, q) == 1) {
                gen = false;
                break;
            }
        if (gen) break;
    }
    const u64 psi0 = h_powmod(g, (q - 1) / two_n, q), psi2 = h_mulmod(psi0, psi0, q);
    u64 best = psi0, cur = psi0;
    for (u64 j = 0; j < two_n / 2; j++) {
        best = std::min(best, cur);
        cur = h_mulmod(cur, psi2, q);
    }
    return best;
}

// CDT over |e| <= 19, sigma = 3.2: T[m] = floor(2^63 F(m)), exp(-j^2 / (2 sigma^2)) = exp(-25 j^2 / 512)
void h_cdt(u64 *out, int n) {
    __float128 rho[32], tot = 0, acc = 0;
    for (int j = 0; j < n; j++) {
        rho[j] = expq(-(__float128)(25 * j * j) / 512);
        tot += j ? 2 * rho[j] : rho[j];
    }
    const __float128 two63 = ldexpq(1, 63);
    for (int m = 0; m < n; m++) {
        acc += m ? 2 * rho[m] : rho[m];
        out[m] = (u64)floorq(two63 * acc / tot);
    }
    out[n - 1] = (u64)1 << 63;
}

u64 galois_elt(const Ctx &c, int steps) {
    if (steps == kConjStep) return (u64)(2 * c.N - 1);  // conjugation (R32)
    const long half = c.N / 2;
    long s = ((steps % half) + half) % half;
    return h_powmod(5, (u64)s, (u64)(2 * c.N));
}

double round_half_away(double x) { return std::round(x); }

static unsigned brv(unsigned x, int bits) {
    unsigned r = 0;
    for (int i = 0; i < bits; i++) r = (r << 1) | ((x >> i) & 1);
    return r;
}

cudaEvent_t Prof::next() {
    if (used == pool.size()) {
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreate(&e));
        pool.push_back(e);
    }
    return pool[used++];
}
size_t Ctx::prof_begin(int) {
    if (!prof.on) return 0;
    const size_t a = prof.used;
    CUDA_CHECK(cudaEventRecord(prof.next(), st));
    return a;
}
void Ctx::prof_end(size_t a, int kind, double bytes, double units) {
    if (!prof.on) return;
    const size_t b = prof.used;
    CUDA_CHECK(cudaEventRecord(prof.next(), st));
    prof.spans.push_back(Prof::Span{a, b, kind, bytes, units});
}

void Ctx::log(const char *kind, int lin, int lout, double s, const std::string &extra) {
    if (!log_on) return;
    u64 bits;
    std::memcpy(&bits, &s, 8);
    char buf[96];
    snprintf(buf, sizeof buf, "%s %d %d %016llx ", kind, lin, lout, (unsigned long long)bits);
    oplog += buf;
    oplog += extra;  // unbounded (a transform's step list)
    oplog += '\n';
}

// ---------------------------------------------------------------------------------------------
// tensor-core base-conversion groups of a level (bconv_tc.cu): ModUp per digit, fused ModDown +
// rescale, plain ModDown.  Constants are exactly those of the integer kernels (R10, R11, R12).
// ---------------------------------------------------------------------------------------------
#ifndef SECPE_TC_PLANES6
#define SECPE_TC_PLANES6 1  // development switch: 0 = 8 byte planes and the integer epilogue everywhere
#endif
#ifndef SECPE_TC_RSLOT
#define SECPE_TC_RSLOT 1  // development switch: 0 = the fused ModDown + rescale adds r [P]_{q_i} per output
#endif
void Ctx::build_tc_groups(LevelConsts &lc, int l) {
    const int nl = l + 1, ne = nl + np, bt = beta(l);
    auto pid = [&](int e) { return e < nl ? e : nq + (e - nl); };
    std::vector<TcGroup> groups;
    std::vector<std::vector<uint8_t>> Bs;
    bool ok = np >= 1 && np + 1 <= 12;
    auto add = [&](TcGroup g, const std::vector<std::vector<u64>> &c, const std::vector<u64> &tp) {
        if (g.ns + 1 > 12 || (int)c.size() > 12 || g.nt > TC_TMAX) ok = false;
        if (!ok) return;
        // 6 byte planes suffice when every constant (< target prime) is < 2^48
        bool small = true;
        for (u64 t : tp) small &= t < (1ULL << 46);
        small = small && SECPE_TC_PLANES6;
        g.planes = small ? 6 : 8;
        const int ntp = (g.nt + 1) & ~1;
        g.ncols = small ? ((6 * g.nt + 15) / 16) * 16 : 8 * ntp;
        if (g.ncols < 16) g.ncols = 16;
        Bs.push_back(tc_bmatrix(c, tp, g.planes, g.ncols));
        groups.push_back(g);
    };
    // ModUp digits: sources y_i (i in I_j), targets every e outside the digit
    for (int j = 0; j < bt; j++) {
        const int i0 = j * alpha, i1 = std::min(i0 + alpha, nl), na = i1 - i0;
        TcGroup g{};
        g.ns = na;
        g.src_row0 = i0;
        std::vector<u64> tp;
        std::vector<std::vector<u64>> c(na);
        for (int e = 0; e < ne; e++) {
            if (e >= i0 && e < i1) continue;
            if (g.nt >= TC_TMAX) {
                ok = false;
                break;
            }
            const u64 t = primes[pid(e)];
            g.prime[g.nt] = pid(e);
            g.out_row[g.nt] = e;
            tp.push_back(t);
            for (int i = i0; i < i1; i++) {
                u64 h = 1;
                for (int i2 = i0; i2 < i1; i2++)
                    if (i2 != i) h = h_mulmod(h, primes[i2] % t, t);
                c[i - i0].push_back(h);
            }
            g.nt++;
        }
        add(g, c, tp);
    }
    // P, (P/p) and products with q_l
    auto Pmod = [&](u64 t) {
        u64 v = 1;
        for (int p2 = 0; p2 < np; p2++) v = h_mulmod(v, primes[nq + p2] % t, t);
        return v;
    };
    auto Phat = [&](int p, u64 t) {
        u64 v = 1;
        for (int p2 = 0; p2 < np; p2++)
            if (p2 != p) v = h_mulmod(v, primes[nq + p2] % t, t);
        return v;
    };
    // fused ModDown + rescale (l >= 1): sources y_p and the constant 1; target 0 = q_l (prelude), then q_i
    {
        TcGroup g{};
        g.ns = np;
        g.src_row0 = l + 1;
        std::vector<u64> tp;
        // with a free source slot, r [P]_{q_i} is a third source (slot np + 1) that a second MMA adds once r is
        // known (bconv_tc_kernel); else the epilogue adds it per output
        const bool rs = np + 2 <= 12 && SECPE_TC_RSLOT;
        std::vector<std::vector<u64>> c(np + (rs ? 2 : 1));
        g.rslot = rs ? np + 1 : -1;
        if (l >= 1 && l + 1 <= TC_TMAX) {
            const u64 ql = primes[l];
            g.prime[0] = l;
            g.out_row[0] = -1;
            tp.push_back(ql);
            for (int p = 0; p < np; p++) c[p].push_back(Phat(p, ql));
            c[np].push_back(0);
            if (rs) c[np + 1].push_back(0);
            for (int i = 0; i < l; i++) {
                const u64 qi = primes[i];
                g.prime[1 + i] = i;
                g.out_row[1 + i] = i;
                g.pmod[1 + i] = Pmod(qi);
                g.pmodsh[1 + i] = h_shoup(g.pmod[1 + i], qi);
                tp.push_back(qi);
                for (int p = 0; p < np; p++) c[p].push_back(Phat(p, qi));
                const u64 ph = h_mulmod(Pmod(qi), (ql >> 1) % qi, qi);
                c[np].push_back(ph ? qi - ph : 0);
                if (rs) c[np + 1].push_back(Pmod(qi));
            }
            g.nt = l + 1;
            add(g, c, tp);
        } else {
            add(g, std::vector<std::vector<u64>>(c.size()), tp);  // empty placeholder (never launched)
        }
    }
    // plain ModDown (rotations): sources y_p, targets q_0..q_l
    {
        TcGroup g{};
        g.ns = np;
        g.src_row0 = nl;
        std::vector<u64> tp;
        std::vector<std::vector<u64>> c(np);
        if (nl <= TC_TMAX) {
            for (int i = 0; i < nl; i++) {
                g.prime[i] = i;
                g.out_row[i] = i;
                tp.push_back(primes[i]);
                for (int p = 0; p < np; p++) c[p].push_back(Phat(p, primes[i]));
            }
            g.nt = nl;
        } else {
            ok = false;
        }
        add(g, c, tp);
    }
    lc.tc_ok = ok;
    if (!ok) return;
    for (auto &g : groups)
        for (int t = 0; t < g.nt; t++) g.qinv[t] = 1.0 / (double)primes[g.prime[t]];
    // one device buffer for every B matrix; TcGroup.B point into it
    std::vector<size_t> off;
    size_t total = 0;
    for (auto &b : Bs) {
        off.push_back(total);
        total += (b.size() + 255) / 256 * 256;
    }
    std::vector<u64> hb((total + 7) / 8, 0);
    for (size_t i = 0; i < Bs.size(); i++) std::memcpy(reinterpret_cast<uint8_t *>(hb.data()) + off[i], Bs[i].data(), Bs[i].size());
    lc.tc_B = upload(hb, st);
    for (size_t i = 0; i < groups.size(); i++)
        groups[i].B = reinterpret_cast<const uint8_t *>(lc.tc_B.p) + off[i];
    std::vector<u64> hg((groups.size() * sizeof(TcGroup) + 7) / 8, 0);
    std::memcpy(hg.data(), groups.data(), groups.size() * sizeof(TcGroup));
    lc.tc_groups = upload(hg, st);
}

// ---------------------------------------------------------------------------------------------
// context build
// ---------------------------------------------------------------------------------------------
void Ctx::drop_graphs(const void *keys) {
    for (auto it = graphs.begin(); it != graphs.end();) {
        if (it->second.keys == keys || it->second.aux == keys) {
            if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
            graph_order.erase(std::remove(graph_order.begin(), graph_order.end(), it->first), graph_order.end());
            it = graphs.erase(it);
        } else {
            ++it;
        }
    }
}

Ctx::~Ctx() {
    for (Keys *k : live_keys) k->owner = nullptr;  // keys may outlive the context
    for (BootSetup *b : live_boots) b->ctx = nullptr;
    if (st) cudaStreamSynchronize(st);
    for (auto &g : graphs)
        if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    pt_cache.clear();  // may have been allocated on an auxiliary stream: free before destroying it
    if (pipe.cp) {
        cudaStreamSynchronize(pipe.cp);
        cudaStreamDestroy(pipe.cp);
    }
    for (int s = 0; s < 2; s++) {
        if (pipe.loaded[s]) cudaEventDestroy(pipe.loaded[s]);
        if (pipe.freed[s]) cudaEventDestroy(pipe.freed[s]);
    }
    for (auto s : aux) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
}

void Ctx::build(const u64 *q, int nq_, const u64 *p, int np_, int alpha_, int logn_, double scale_) {
    {
        const char *e = getenv("SECPE_STREAMS");  // concurrent sub-batches in secpe_enc_argmax
        n_streams = e ? std::max(1, atoi(e)) : 2;
        const char *g = getenv("SECPE_GRAPH");
        use_graphs = !(g && atoi(g) == 0);
    }
    {
        const char *e = getenv("SECPE_NO_TC");  // development switch: integer base-conversion kernels
        use_tc = !(e && atoi(e) == 1);
        // development switch: single-pass cluster NTT (ntt.cu; measured slower on the FP64-bound rows, off)
        const char *c = getenv("SECPE_NTT_CLUSTER");
        ntt_cluster = c ? atoi(c) : 0;
    }
    // ~50-bit rows on the exact-FP64 NTT with reductions (FpB) for N >= 2^15: measured at N = 2^16 +14 %
    // batched bootstraps (53.9 -> 61.7 per s), +8 % K = 16 argmax with bootstrapping; at N = 2^12 (64-thread
    // CTAs, latency-bound) the integer path is faster.  SECPE_NO_FPB=1 keeps them on the integer Shoup NTT;
    // SECPE_FPB=1 takes FpB on every ring (the N = 2^12 parity tests of the FpB path), SECPE_FPB=0 on none
    const char *nofpb = getenv("SECPE_NO_FPB"), *fpb = getenv("SECPE_FPB");
    const bool use_fpb = fpb ? atoi(fpb) == 1 : !(nofpb && atoi(nofpb) == 1) && logn_ >= 15;
    constexpr u64 FPB_TABLE_LIMIT = 1286742750677284ULL;  // floor(2^52 / 3.5), ntt_core.cuh FPB_LIMIT
    logn = logn_;
    N = 1L << logn;
    nq = nq_;
    np = np_;
    alpha = alpha_;
    scale = scale_;
    primes.assign(q, q + nq);
    primes.insert(primes.end(), p, p + np);
    const int P = nprimes();
    psi.resize(P);
    std::vector<u64> hq(P), hr0(P), hr1(P), hni(P), hnish(P);
    std::vector<u64> tw(2 * (size_t)P * N), itw(2 * (size_t)P * N);  // interleaved {w, w'}
    for (int i = 0; i < P; i++) {
        const u64 qi = primes[i];
        psi[i] = h_find_psi(qi, logn);
        hq[i] = qi;
        const u128 r = (~(u128)0) / qi;  // floor((2^128 - 1)/q) = floor(2^128/q) for odd q
        hr0[i] = (u64)r;
        hr1[i] = (u64)(r >> 64);
        hni[i] = h_invmod((u64)N % qi, qi);
        hnish[i] = h_shoup(hni[i], qi);
        // powers psi^k and psi^-k, then bit-reversed tables
        std::vector<u64> pw(N), ipw(N);
        const u64 pinv = h_invmod(psi[i], qi);
        pw[0] = ipw[0] = 1;
        for (long k = 1; k < N; k++) {
            pw[k] = h_mulmod(pw[k - 1], psi[i], qi);
            ipw[k] = h_mulmod(ipw[k - 1], pinv, qi);
        }
        for (long k = 0; k < N; k++) {
            const unsigned b = brv((unsigned)k, logn);
            const size_t o = (size_t)i * N + k;
            if (qi < (1ULL << 46) || (use_fpb && i < 64 && qi < FPB_TABLE_LIMIT)) {
                // exact-FP64 butterflies (ntt_core.cuh FpA / FpB): dense doubles w in the first N words of the
                // prime's 2N-word region
                const double w = (double)pw[b], iw = (double)ipw[b];
                std::memcpy(&tw[2 * (size_t)i * N + k], &w, 8);
                std::memcpy(&itw[2 * (size_t)i * N + k], &iw, 8);
            } else {
                tw[2 * o] = pw[b];
                tw[2 * o + 1] = h_shoup(pw[b], qi);
                itw[2 * o] = ipw[b];
                itw[2 * o + 1] = h_shoup(ipw[b], qi);
            }
        }
    }
    h_br0 = hr0;
    h_br1 = hr1;
    d_q = upload(hq, st);
    d_br0 = upload(hr0, st);
    d_br1 = upload(hr1, st);
    d_ninv = upload(hni, st);
    d_ninvsh = upload(hnish, st);
    d_tw = upload(tw, st);
    d_itw = upload(itw, st);
    tab = Tab{d_q.p, d_br0.p, d_br1.p, reinterpret_cast<const ulonglong2 *>(d_tw.p),
              reinterpret_cast<const ulonglong2 *>(d_itw.p), d_ninv.p, d_ninvsh.p, 0, nullptr, nullptr, ntt_cluster};
    {
        std::vector<u64> a(P), b(P);
        for (int i = 0; i < P; i++) {
            const double qd = (double)primes[i], qi = 1.0 / qd;
            std::memcpy(&a[i], &qd, 8);
            std::memcpy(&b[i], &qi, 8);
        }
        d_qd = upload(a, st);
        d_qinv = upload(b, st);
        tab.qd = reinterpret_cast<const double *>(d_qd.p);
        tab.qinv = reinterpret_cast<const double *>(d_qinv.p);
    }
    for (int i = 0; i < P && i < 64; i++) {
        if (primes[i] < (1ULL << 46))
            tab.fp_mask |= 1ULL << i;
        else if (use_fpb && primes[i] < FPB_TABLE_LIMIT)
            tab.fpb_mask |= 1ULL << i;
    }
    // {w, w/q} pair tables of the exact-FP64 rows for the fused NTT (its row-tile stages read one 16-byte pair
    // per twiddle instead of forming w/q with a DMUL); integer rows keep their {w, w'} tables
    tab.twp = tab.tw2;
    tab.itwp = tab.itw2;
    if (tab.fp_mask) {
        std::vector<u64> tp(2 * (size_t)P * N), itp(2 * (size_t)P * N);
        for (int i = 0; i < P; i++) {
            const size_t o = 2 * (size_t)i * N;
            if (primes[i] < (1ULL << 46) || (i < 64 && ((tab.fpb_mask >> i) & 1))) {
                const double qinv = 1.0 / (double)primes[i];
                for (long k = 0; k < N; k++) {
                    double w, iw;
                    std::memcpy(&w, &tw[o + k], 8);
                    std::memcpy(&iw, &itw[o + k], 8);
                    const double wq = w * qinv, iwq = iw * qinv;
                    std::memcpy(&tp[o + 2 * k], &w, 8);
                    std::memcpy(&tp[o + 2 * k + 1], &wq, 8);
                    std::memcpy(&itp[o + 2 * k], &iw, 8);
                    std::memcpy(&itp[o + 2 * k + 1], &iwq, 8);
                }
            } else {
                std::copy(tw.begin() + o, tw.begin() + o + 2 * N, tp.begin() + o);
                std::copy(itw.begin() + o, itw.begin() + o + 2 * N, itp.begin() + o);
            }
        }
        d_twp = upload(tp, st);
        d_itwp = upload(itp, st);
        tab.twp = reinterpret_cast<const ulonglong2 *>(d_twp.p);
        tab.itwp = reinterpret_cast<const ulonglong2 *>(d_itwp.p);
    }

    // ModDown constants: P = prod p
    std::vector<u64> vihp(std::max(np, 1)), vihpsh(std::max(np, 1)), vhatp((size_t)std::max(np, 1) * nq),
        vpinv(nq), vpinvsh(nq);
    for (int a = 0; a < np; a++) {
        const u64 pa = primes[nq + a];
        u64 h = 1;
        for (int b = 0; b < np; b++)
            if (b != a) h = h_mulmod(h, primes[nq + b] % pa, pa);
        vihp[a] = h_invmod(h, pa);
        vihpsh[a] = h_shoup(vihp[a], pa);
        for (int i = 0; i < nq; i++) {
            u64 hq2 = 1;
            for (int b = 0; b < np; b++)
                if (b != a) hq2 = h_mulmod(hq2, primes[nq + b] % primes[i], primes[i]);
            vhatp[(size_t)a * nq + i] = pack30(hq2);
        }
    }
    for (int i = 0; i < nq; i++) {
        u64 pp = 1;
        for (int a = 0; a < np; a++) pp = h_mulmod(pp, primes[nq + a] % primes[i], primes[i]);
        vpinv[i] = h_invmod(pp, primes[i]);
        vpinvsh[i] = h_shoup(vpinv[i], primes[i]);
    }
    ihp = upload(vihp, st);
    ihp_sh = upload(vihpsh, st);
    {
        std::vector<u64> a(std::max(np, 1)), b(std::max(np, 1));
        for (int i = 0; i < np; i++) {
            const u64 pi = primes[nq + i];
            a[i] = h_mulmod(vihp[i], h_invmod((u64)N % pi, pi), pi);
            b[i] = h_shoup(a[i], pi);
        }
        ihp_ninv = upload(a, st);
        ihp_ninv_sh = upload(b, st);
    }
    hat_p = upload(vhatp, st);
    pinv = upload(vpinv, st);
    pinv_sh = upload(vpinvsh, st);
    h_pinv = vpinv;
    h_pinv_sh = vpinvsh;
    {
        std::vector<u64> pm(nq);
        for (int i = 0; i < nq; i++) pm[i] = h_invmod(vpinv[i], primes[i]);  // P mod q_i
        pmod = upload(pm, st);
    }

    // per-level constants
    lvl.clear();
    for (int l = 0; l < nq; l++) {
        auto lc = std::make_unique<LevelConsts>();
        const int nl = l + 1, ne = nl + np, bt = beta(l);
        lc->nl = nl;
        lc->beta = bt;
        std::vector<u64> ih(nl), ihs(nl), hat((size_t)bt * 16 * ne, 0);
        for (int j = 0; j < bt; j++) {
            const int i0 = j * alpha, i1 = std::min(i0 + alpha, nl);
            for (int i = i0; i < i1; i++) {
                u64 h = 1;
                for (int i2 = i0; i2 < i1; i2++)
                    if (i2 != i) h = h_mulmod(h, primes[i2] % primes[i], primes[i]);
                ih[i] = h_invmod(h, primes[i]);
                ihs[i] = h_shoup(ih[i], primes[i]);
                for (int e = 0; e < ne; e++) {
                    const u64 t = primes[e < nl ? e : nq + (e - nl)];
                    u64 ht = 1;
                    for (int i2 = i0; i2 < i1; i2++)
                        if (i2 != i) ht = h_mulmod(ht, primes[i2] % t, t);
                    hat[((size_t)j * 16 + (i - i0)) * ne + e] = pack30(ht);
                }
            }
        }
        lc->inv_hat = upload(ih, st);
        lc->inv_hat_sh = upload(ihs, st);
        {
            std::vector<u64> a(nl), b(nl);
            for (int i = 0; i < nl; i++) {
                a[i] = h_mulmod(ih[i], h_invmod((u64)N % primes[i], primes[i]), primes[i]);
                b[i] = h_shoup(a[i], primes[i]);
            }
            lc->inv_hat_ninv = upload(a, st);
            lc->inv_hat_ninv_sh = upload(b, st);
        }
        lc->hat = upload(hat, st);
        if (l >= 1) {
            std::vector<u64> hf(l), qi(l), qis(l);
            const u64 ql = primes[l];
            for (int i = 0; i < l; i++) {
                hf[i] = (ql >> 1) % primes[i];
                qi[i] = h_invmod(ql % primes[i], primes[i]);
                qis[i] = h_shoup(qi[i], primes[i]);
            }
            lc->half = upload(hf, st);
            lc->qlinv = upload(qi, st);
            lc->qlinv_sh = upload(qis, st);
            // fused relinearise-and-rescale (bit-identical to ModDown then rescale, eval.cu):
            //   rr_fold [np+1]: N^{-1} mod q_l, then N^{-1} (P/p)^{-1} mod p
            //   rr_hl   [np]  : (P/p) mod q_l (split-30 packed)
            //   rr_hat  [np+2][l]: (P/p) mod q_i, P mod q_i, -P floor(q_l/2) mod q_i (split-30 packed)
            //   rr_binv [l]   : (P q_l)^{-1} mod q_i
            std::vector<u64> fold(np + 1), foldsh(np + 1), hl(np), rhat((size_t)(np + 2) * l), binv(l), binvsh(l);
            fold[0] = h_invmod((u64)N % ql, ql);
            foldsh[0] = h_shoup(fold[0], ql);
            for (int p2 = 0; p2 < np; p2++) {
                const u64 pp = primes[nq + p2];
                fold[1 + p2] = h_mulmod(vihp[p2], h_invmod((u64)N % pp, pp), pp);
                foldsh[1 + p2] = h_shoup(fold[1 + p2], pp);
                u64 h = 1;
                for (int p3 = 0; p3 < np; p3++)
                    if (p3 != p2) h = h_mulmod(h, primes[nq + p3] % ql, ql);
                hl[p2] = pack30(h);
            }
            for (int i = 0; i < l; i++) {
                const u64 qi2 = primes[i];
                u64 Pm = 1;
                for (int p2 = 0; p2 < np; p2++) {
                    u64 h = 1;
                    for (int p3 = 0; p3 < np; p3++)
                        if (p3 != p2) h = h_mulmod(h, primes[nq + p3] % qi2, qi2);
                    rhat[(size_t)p2 * l + i] = pack30(h);
                    Pm = h_mulmod(Pm, primes[nq + p2] % qi2, qi2);
                }
                rhat[(size_t)np * l + i] = pack30(Pm);
                const u64 ph = h_mulmod(Pm, (ql >> 1) % qi2, qi2);
                rhat[(size_t)(np + 1) * l + i] = pack30(ph ? qi2 - ph : 0);
                binv[i] = h_invmod(h_mulmod(Pm, ql % qi2, qi2), qi2);
                binvsh[i] = h_shoup(binv[i], qi2);
            }
            lc->rr_hl = upload(hl, st);
            lc->rr_fold = upload(fold, st);
            lc->rr_fold_sh = upload(foldsh, st);
            lc->rr_hat = upload(rhat, st);
            lc->rr_binv = upload(binv, st);
            lc->rr_binv_sh = upload(binvsh, st);
        }
        build_tc_groups(*lc, l);
        lvl.push_back(std::move(lc));
    }
    u64 cdt[20];
    h_cdt(cdt, 20);
    set_cdt(cdt, 20);
    CUDA_CHECK(cudaStreamSynchronize(st));
}
