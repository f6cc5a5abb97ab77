// boot.cpp -- bootstrapping setup on the library side (readings R34, R35): the EvalMod
// polynomial and the four slot-domain matrices of CoeffToSlot / SlotToCoeff, encoded and NTT'd into
// device memory in the baby-step giant-step layout secpe_bootstrap reads.  Client/setup work, done once
// per (level, K, r, split, input scale); not on the hot path.
//
//   A[k][j] = zeta^{-5^j k} / n, U[j][k] = zeta^{5^j k}, n = N/2, zeta = e^{i pi / N} (the inverse of
//   encoding and decoding, R5); CoeffToSlot A/2, -i A/2; SlotToCoeff c U, i c U, c = R / (4 pi),
//   R = q_0 / S_in.  pts[g][j] = NTT(encode(RotR(d_{g n1 + j}, g n1), scale)), d_i[t] = M[t][(t + i) mod n].
//   poly: Taylor coefficients of 2 cos(a x + b), a = 2 pi K / 2^r, b = -pi / 2^(r+1), up to x^15.
#include <cmath>
#include <complex>
#include <algorithm>
#include <functional>
#include <map>
#include <numeric>

#include "context.h"

typedef std::complex<double> cd;

static void encode_matrix(Ctx &c, const std::function<cd(long, long)> &M, int n1, int n2, int level, double scale,
                          DevBuf &out) {
    const long N = c.N, n = N / 2;
    const int nl = level + 1;
    const long npt = (long)n1 * n2;
    out = DevBuf((size_t)npt * nl * N, c.st);
    std::vector<i64> coef((size_t)npt * N);
    std::vector<double> re(n), im(n);
    for (int g = 0; g < n2; g++)
        for (int j = 0; j < n1; j++) {
            const long i = (long)g * n1 + j, s = (long)g * n1;
            for (long t = 0; t < n; t++) {  // RotR(d_i, g n1)[t] = d_i[t - g n1]
                const long u = ((t - s) % n + n) % n;
                const cd v = M(u, (u + i) % n);
                re[t] = v.real();
                im[t] = v.imag();
            }
            encode_complex_int(c, re.data(), im.data(), n, scale, coef.data() + i * N);
        }
    DevBuf dc((size_t)npt * N, c.st);
    CUDA_CHECK(cudaMemcpyAsync(dc.p, coef.data(), (size_t)npt * N * 8, cudaMemcpyHostToDevice, c.st));
    for (long i = 0; i < npt; i++)
        k_int_to_rows(c.tab, c.logn, (const i64 *)dc.p + i * N, out.p + (size_t)i * nl * N, LimbMap{nl, nl, 0, 0},
                      c.st);
    ev_ntt(c, RowsArg{out.p, 2L * nl * N, (long)nl * N}, (int)npt, LimbMap{nl, nl, 0, 0}, false);
    CUDA_CHECK(cudaStreamSynchronize(c.st));  // coef is host memory of this frame
}

BootSetup *boot_setup(Ctx &c, int level, double K, int r, int n1, int n2, double in_scale) {
    const long N = c.N, n = N / 2;
    if (n1 < 1 || n2 < 1 || (long)n1 * n2 != n) throw SecpeError{-1, "boot: n1 n2 must be N/2"};
    if (!(K > 0) || r < 0 || r > 30) throw SecpeError{-1, "boot: bad EvalMod range"};
    const int l_stc = level - 7 - r;
    if (level >= c.nq || l_stc < 1) throw SecpeError{-2, "boot: not enough levels"};
    auto b = std::make_unique<BootSetup>();
    b->ctx = &c;
    const double a = 2.0 * M_PI * K / std::ldexp(1.0, r), ph = -M_PI / std::ldexp(1.0, r + 1);
    b->cfg.poly.resize(16);
    double fact = 1.0;
    for (int i = 0; i < 16; i++) {
        if (i) fact *= i;
        b->cfg.poly[i] = 2.0 * std::pow(a, i) * std::cos(ph + i * M_PI / 2) / fact;
    }
    const double R = (double)c.primes[0] / in_scale, cc = R / (4.0 * M_PI);
    // zeta^{+-e_j k} with the exponent reduced mod 2N first
    std::vector<long> e(n);
    for (long j = 0, v = 1; j < n; j++, v = (v * 5) % (2 * N)) e[j] = v;
    auto zpow = [&](long ej, long k, int sgn) {
        const long m = (ej * k) % (2 * N);
        const double ang = sgn * M_PI * (double)m / (double)N;
        return cd(std::cos(ang), std::sin(ang));
    };
    const double inv_n = 1.0 / (double)n;
    const double cts_scale = (double)c.primes[level], stc_scale = (double)c.primes[l_stc];
    encode_matrix(c, [&](long t, long col) { return zpow(e[col], t, -1) * inv_n * 0.5; }, n1, n2, level, cts_scale,
                  b->cts_re);
    encode_matrix(c, [&](long t, long col) { return zpow(e[col], t, -1) * inv_n * cd(0, -0.5); }, n1, n2, level,
                  cts_scale, b->cts_im);
    encode_matrix(c, [&](long t, long col) { return zpow(e[t], col, 1) * cc; }, n1, n2, l_stc, stc_scale, b->stc_re);
    encode_matrix(c, [&](long t, long col) { return zpow(e[t], col, 1) * cd(0, cc); }, n1, n2, l_stc, stc_scale,
                  b->stc_im);
    b->cfg.level = level;
    b->cfg.n1 = n1;
    b->cfg.n2 = n2;
    b->cfg.r = r;
    b->cfg.K = K;
    b->cfg.cts_re = b->cts_re.p;
    b->cfg.cts_im = b->cts_im.p;
    b->cfg.stc_re = b->stc_re.p;
    b->cfg.stc_im = b->stc_im.p;
    b->cfg.cts_scale = cts_scale;
    b->cfg.stc_scale = stc_scale;
    return b.release();
}

// ---- factorised CoeffToSlot / SlotToCoeff (R37) ------------------------------------------------------
// Special-FFT butterfly stage s (len = 2^s, h = len/2), block start i, j < h, w_j = zeta^m,
// m = (e_j mod 4 len) 2N / (4 len):  out[i+j] = v[i+j] + w_j v[i+j+h], out[i+j+h] = v[i+j] - w_j v[i+j+h];
// U w = S_log2n ... S_1 (bit-reversed w).  Diagonal form: offset (mod n) -> vector, out = sum d_o (.) RotL(v, o).
using Diag = std::map<long, std::vector<cd>>;

static std::vector<Diag> fft_stages(long N, bool inverse) {
    const long n = N / 2;
    std::vector<long> e(n);
    for (long j = 0, v = 1; j < n; j++, v = (v * 5) % (2 * N)) e[j] = v;
    std::vector<Diag> out;
    for (long ln = 2; ln <= n; ln *= 2) {
        const long h = ln / 2;
        std::vector<cd> d0(n), dp(n), dm(n);
        for (long i = 0; i < n; i += ln)
            for (long j = 0; j < h; j++) {
                const long m = (e[j] % (4 * ln)) * (2 * N / (4 * ln));
                const double ang = M_PI * (double)m / (double)N;
                if (!inverse) {
                    const cd w(std::cos(ang), std::sin(ang));
                    d0[i + j] = 1.0;
                    dp[i + j] = w;
                    dm[i + j + h] = 1.0;
                    d0[i + j + h] = -w;
                } else {
                    const cd wi(std::cos(ang), -std::sin(ang));
                    d0[i + j] = 0.5;
                    dp[i + j] = 0.5;
                    dm[i + j + h] = 0.5 * wi;
                    d0[i + j + h] = -0.5 * wi;
                }
            }
        Diag D;
        D[0] = d0;
        if (h == n - h) {
            for (long p = 0; p < n; p++) dp[p] += dm[p];
            D[h] = dp;
        } else {
            D[h] = dp;
            D[n - h] = dm;
        }
        out.push_back(std::move(D));
    }
    return out;
}

// A B (A applied after B): sum_{a,b} (alpha_a (.) RotL(beta_b, a)) (.) RotL(v, a + b)
static Diag diag_mul(const Diag &A, const Diag &B, long n) {
    Diag out;
    for (const auto &x : A)
        for (const auto &y : B) {
            auto &o = out[(x.first + y.first) % n];
            if (o.empty()) o.assign(n, cd(0, 0));
            for (long p = 0; p < n; p++) o[p] += x.second[p] * y.second[(p + x.first) % n];
        }
    return out;
}

// encode every diagonal of D (times `mul`) at `scale` on `level`; steps = signed offsets, ascending
static LtStage encode_stage(Ctx &c, const Diag &D, cd mul, int level, double scale, std::vector<DevBuf> &bufs) {
    const long N = c.N, n = N / 2;
    const int nl = level + 1;
    std::vector<std::pair<long, long>> order;  // (signed offset, key)
    for (const auto &x : D) order.push_back({x.first > n / 2 ? x.first - n : x.first, x.first});
    std::sort(order.begin(), order.end());
    const long nd = (long)order.size();
    LtStage st;
    std::vector<i64> coef((size_t)nd * N);
    std::vector<double> re(n), im(n);
    for (long i = 0; i < nd; i++) {
        const auto &d = D.at(order[i].second);
        for (long t = 0; t < n; t++) {
            const cd v = d[t] * mul;
            re[t] = v.real();
            im[t] = v.imag();
        }
        encode_complex_int(c, re.data(), im.data(), n, scale, coef.data() + i * N);
        st.steps.push_back((int)order[i].first);
    }
    DevBuf out((size_t)nd * nl * N, c.st), dc((size_t)nd * N, c.st);
    CUDA_CHECK(cudaMemcpyAsync(dc.p, coef.data(), (size_t)nd * N * 8, cudaMemcpyHostToDevice, c.st));
    for (long i = 0; i < nd; i++)
        k_int_to_rows(c.tab, c.logn, (const i64 *)dc.p + i * N, out.p + (size_t)i * nl * N, LimbMap{nl, nl, 0, 0},
                      c.st);
    ev_ntt(c, RowsArg{out.p, 2L * nl * N, (long)nl * N}, (int)nd, LimbMap{nl, nl, 0, 0}, false);
    CUDA_CHECK(cudaStreamSynchronize(c.st));
    st.pts = out.p;
    st.scale = scale;
    bufs.push_back(std::move(out));
    return st;
}

// baby-step giant-step form (R39): the signed offsets of a merged group are u k, k_min <= k <= k_max;
// n1 = the power of two >= sqrt(count), baby u j, giant u (k_min + n1 g), pts[g][j] = encode(RotR(d_k, giant_g))
// with k = k_min + n1 g + j (a zero polynomial past k_max)
static LtStage encode_stage_bsgs(Ctx &c, const Diag &D, cd mul, int level, double scale, std::vector<DevBuf> &bufs) {
    const long N = c.N, n = N / 2;
    const int nl = level + 1;
    std::vector<long> offs;
    for (const auto &x : D) offs.push_back(x.first > n / 2 ? x.first - n : x.first);
    std::sort(offs.begin(), offs.end());
    long u = 0;
    for (long o : offs) u = std::gcd(u, std::labs(o));
    if (u == 0) u = 1;
    const long kmin = offs.front() / u, kmax = offs.back() / u, cnt = kmax - kmin + 1;
    if (cnt != (long)offs.size()) throw SecpeError{-1, "boot: offsets are not a contiguous progression"};
    long n1 = 1;
    while (n1 * n1 < cnt) n1 *= 2;
    const long n2 = (cnt + n1 - 1) / n1;
    LtStage st;
    for (long j = 0; j < n1; j++) st.baby.push_back((int)(u * j));
    for (long g = 0; g < n2; g++) st.giant.push_back((int)(u * (kmin + n1 * g)));
    std::vector<i64> coef((size_t)n1 * n2 * N);
    std::vector<double> re(n), im(n);
    for (long g = 0; g < n2; g++)
        for (long j = 0; j < n1; j++) {
            const long kk = kmin + n1 * g + j, G = st.giant[g];
            const auto it = kk <= kmax ? D.find(((u * kk) % n + n) % n) : D.end();
            for (long t = 0; t < n; t++) {
                const cd v = it == D.end() ? cd(0, 0) : it->second[((t - G) % n + n) % n] * mul;
                re[t] = v.real();
                im[t] = v.imag();
            }
            encode_complex_int(c, re.data(), im.data(), n, scale, coef.data() + (g * n1 + j) * N);
        }
    const long npt = n1 * n2;
    DevBuf out((size_t)npt * nl * N, c.st), dc((size_t)npt * N, c.st);
    CUDA_CHECK(cudaMemcpyAsync(dc.p, coef.data(), (size_t)npt * N * 8, cudaMemcpyHostToDevice, c.st));
    for (long i = 0; i < npt; i++)
        k_int_to_rows(c.tab, c.logn, (const i64 *)dc.p + i * N, out.p + (size_t)i * nl * N, LimbMap{nl, nl, 0, 0},
                      c.st);
    ev_ntt(c, RowsArg{out.p, 2L * nl * N, (long)nl * N}, (int)npt, LimbMap{nl, nl, 0, 0}, false);
    CUDA_CHECK(cudaStreamSynchronize(c.st));
    st.pts = out.p;
    st.scale = scale;
    bufs.push_back(std::move(out));
    return st;
}

BootSetup *boot_setup_fft(Ctx &c, int level, double K, int r, const std::vector<int> &groups, double in_scale,
                          bool bsgs) {
    const long N = c.N, n = N / 2;
    int lg = 0;
    while ((1L << lg) < n) lg++;
    int sum = 0;
    for (int g : groups) {
        if (g < 1) throw SecpeError{-1, "boot: empty stage group"};
        sum += g;
    }
    if (sum != lg) throw SecpeError{-1, "boot: groups must cover log2(N/2) stages"};
    if (!(K > 0) || r < 0 || r > 30) throw SecpeError{-1, "boot: bad EvalMod range"};
    const int mg = (int)groups.size();
    if (level >= c.nq || level - (2 * mg + 6 + r) < 0) throw SecpeError{-2, "boot: not enough levels"};
    auto b = std::make_unique<BootSetup>();
    b->ctx = &c;
    b->fft = true;
    auto enc = [&](const Diag &D, cd mul, int lv, double sc) {
        return bsgs ? encode_stage_bsgs(c, D, mul, lv, sc, b->bufs) : encode_stage(c, D, mul, lv, sc, b->bufs);
    };
    FftBootCfg &f = b->fcfg;
    f.level = level;
    f.r = r;
    f.K = K;
    const double a = 2.0 * M_PI * K / std::ldexp(1.0, r), ph = -M_PI / std::ldexp(1.0, r + 1);
    f.poly.resize(16);
    double fact = 1.0;
    for (int i = 0; i < 16; i++) {
        if (i) fact *= i;
        f.poly[i] = 2.0 * std::pow(a, i) * std::cos(ph + i * M_PI / 2) / fact;
    }
    const auto st = fft_stages(N, false), si = fft_stages(N, true);
    std::vector<Diag> stc, cts;
    int pos = 0;
    for (int g : groups) {
        Diag D, Di;
        D[0].assign(n, cd(1, 0));
        Di[0].assign(n, cd(1, 0));
        for (int s = pos; s < pos + g; s++) {
            D = diag_mul(st[s], D, n);
            Di = diag_mul(Di, si[s], n);
        }
        stc.push_back(std::move(D));
        cts.push_back(std::move(Di));
        pos += g;
    }
    std::reverse(cts.begin(), cts.end());
    const double R = (double)c.primes[0] / in_scale, cc = R / (4.0 * M_PI);
    int lv = level;
    for (int i = 0; i < mg; i++, lv--) {
        const double sc = (double)c.primes[lv];
        if (i < mg - 1) {
            f.cts.push_back(enc(cts[i], cd(1, 0), lv, sc));
        } else {
            f.cts.push_back(enc(cts[i], cd(0.5, 0), lv, sc));
            f.cts_im = enc(cts[i], cd(0, -0.5), lv, sc);
        }
    }
    lv = level - mg - 6 - r;
    for (int i = 0; i < mg; i++, lv--) {
        const double sc = (double)c.primes[lv];
        if (i == 0) {
            f.stc.push_back(enc(stc[i], cd(cc, 0), lv, sc));
            f.stc_im = enc(stc[i], cd(0, cc), lv, sc);
        } else {
            f.stc.push_back(enc(stc[i], cd(1, 0), lv, sc));
        }
    }
    return b.release();
}
