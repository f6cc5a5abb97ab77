// encode.cpp -- CKKS canonical-embedding encode/decode (client side, host double precision).
//
// Reading R5: slot j <-> evaluation at zeta^{5^j mod 2N}, zeta = e^{i pi/N}.
//   encode: m_k = round_half_away((2 Delta / N) Re sum_j z_j zeta^{-5^j k})
//           = round_half_away(Delta Re(zeta^{-k} F[k]) / N),  F = DFT_N(W), W[t] = w[2t+1],
//           w[5^j] = z_j, w[-5^j] = conj(z_j)
//   decode: z_j = (1/Delta) sum_k m_k zeta^{5^j k} = (1/Delta) G[(5^j - 1)/2], G = IDFT_N(m_k zeta^k) * N
// Encoding is client work outside the server's hot path; the bit-exact contract starts at the
// integer plaintext (reading R16).  The argmax mask uses the quantised variant encode_mask.
#include <cmath>
#include <complex>
#include <vector>

#include "context.h"

typedef std::complex<double> cd;

// in-place radix-2 DFT: sign -1 -> sum x_t e^{-2 pi i t k / n}; sign +1 -> e^{+...} (no scaling)
static void fft(std::vector<cd> &a, int sign) {
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; i++) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t h = len / 2;
        std::vector<cd> w(h);
        for (size_t k = 0; k < h; k++) {
            const double ang = sign * 2.0 * M_PI * (double)k / (double)len;
            w[k] = cd(std::cos(ang), std::sin(ang));
        }
        for (size_t s = 0; s < n; s += len)
            for (size_t k = 0; k < h; k++) {
                const cd u = a[s + k], v = a[s + k + h] * w[k];
                a[s + k] = u + v;
                a[s + k + h] = u - v;
            }
    }
}

static std::vector<long> rot_group(long N) {
    std::vector<long> e(N / 2);
    long v = 1;
    for (long j = 0; j < N / 2; j++) {
        e[j] = v;
        v = (v * 5) % (2 * N);
    }
    return e;
}

void encode_real(const Ctx &c, const double *slots, size_t n, double scale, std::vector<double> &coef) {
    const long N = c.N;
    if ((long)n > N / 2) throw SecpeError{-1, "encode: more values than slots"};
    std::vector<cd> w(2 * N, cd(0, 0));
    const auto e = rot_group(N);
    for (size_t j = 0; j < n; j++) {
        w[e[j]] = cd(slots[j], 0);
        w[(2 * N - e[j]) % (2 * N)] = cd(slots[j], 0);
    }
    std::vector<cd> W(N);
    for (long t = 0; t < N; t++) W[t] = w[2 * t + 1];
    fft(W, -1);
    coef.resize(N);
    for (long k = 0; k < N; k++) {
        const double ang = -M_PI * (double)k / (double)N;
        const cd z = cd(std::cos(ang), std::sin(ang)) * W[k];
        coef[k] = z.real() / (double)N * scale;
    }
}

void encode_int(const Ctx &c, const double *slots, size_t n, double scale, i64 *out) {
    std::vector<double> coef;
    encode_real(c, slots, n, scale, coef);
    for (long k = 0; k < c.N; k++) {
        const double r = std::round(coef[k]);
        if (!(std::fabs(r) < 4611686018427387904.0)) throw SecpeError{-6, "encoded coefficient exceeds 2^62"};
        out[k] = (i64)r;
    }
}

// complex slots (bootstrapping's matrix diagonals, R34): w[5^j] = z_j, w[-5^j] = conj(z_j); for real z the
// same integers as encode_int
void encode_complex_int(const Ctx &c, const double *re, const double *im, size_t n, double scale, i64 *out) {
    const long N = c.N;
    if ((long)n > N / 2) throw SecpeError{-1, "encode: more values than slots"};
    std::vector<cd> w(2 * N, cd(0, 0));
    const auto e = rot_group(N);
    for (size_t j = 0; j < n; j++) {
        w[e[j]] = cd(re[j], im[j]);
        w[(2 * N - e[j]) % (2 * N)] = cd(re[j], -im[j]);
    }
    std::vector<cd> W(N);
    for (long t = 0; t < N; t++) W[t] = w[2 * t + 1];
    fft(W, -1);
    for (long k = 0; k < N; k++) {
        const double ang = -M_PI * (double)k / (double)N;
        const cd z = cd(std::cos(ang), std::sin(ang)) * W[k];
        const double r = std::round(z.real() / (double)N * scale);
        if (!(std::fabs(r) < 4611686018427387904.0)) throw SecpeError{-6, "encoded coefficient exceeds 2^62"};
        out[k] = (i64)r;
    }
}

// R16: M_k = rha(delta * rha(m_k 2^24) / 2^24), m_k the unit-scale real coefficients
void encode_mask(const Ctx &c, const double *slots, size_t n, double delta, i64 *out) {
    std::vector<double> coef;
    encode_real(c, slots, n, 1.0, coef);
    const double Q = 16777216.0;  // 2^24
    for (long k = 0; k < c.N; k++) {
        const double qk = std::round(coef[k] * Q) / Q;
        const double r = std::round(delta * qk);
        if (!(std::fabs(r) < 4611686018427387904.0)) throw SecpeError{-6, "mask coefficient exceeds 2^62"};
        out[k] = (i64)r;
    }
}

void decode_real(const Ctx &c, const std::vector<double> &coef, double scale, double *slots, size_t n) {
    const long N = c.N;
    std::vector<cd> a(N);
    for (long k = 0; k < N; k++) {
        const double ang = M_PI * (double)k / (double)N;
        a[k] = cd(std::cos(ang), std::sin(ang)) * coef[k];
    }
    fft(a, +1);
    const auto e = rot_group(N);
    for (size_t j = 0; j < n && (long)j < N / 2; j++) slots[j] = a[(e[j] - 1) / 2].real() / scale;
}
