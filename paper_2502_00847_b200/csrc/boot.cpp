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
#include <functional>

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
