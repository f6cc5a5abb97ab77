// context.h -- library context, keys, device buffers and the ciphertext evaluator.
#pragma once
#include <climits>
#include <map>
#include <set>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"

// RAII device buffer (stream-ordered allocation on the context stream)
struct BootSetup;

struct DevBuf {
    u64 *p = nullptr;
    size_t words = 0;
    cudaStream_t st = nullptr;
    DevBuf() = default;
    DevBuf(size_t w, cudaStream_t s);
    ~DevBuf();
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept { *this = std::move(o); }
    DevBuf &operator=(DevBuf &&o) noexcept;
};

// tensor-core base conversion (bconv_tc.cu): one conversion group = sources x targets + its B matrix
constexpr int TC_TMAX = 32;
struct TcGroup {
    int ns;                  // sources (rows of the source polynomial starting at src_row0)
    int nt;                  // targets (<= TC_TMAX)
    int src_row0;
    const uint8_t *B;        // device: canonical byte-sliced constant matrix, 8 * ntp rows x 96 bytes
    int prime[TC_TMAX];      // target prime (global index)
    int out_row[TC_TMAX];    // output row (limb) of the target in the destination polynomial
    u64 pmod[TC_TMAX];       // rescale variant: [P]_{q_t} and its Shoup companion
    u64 pmodsh[TC_TMAX];
    double qinv[TC_TMAX];    // RN(1 / q_t) for the FP64 quotient of the epilogue
    int planes;              // byte planes per target: 6 when every target prime is < 2^46, else 8
    int ncols;               // MMA N = TMEM columns used (multiple of 16, <= 256)
    int rslot = -1;          // fused ModDown + rescale: source slot of r (added by a second MMA), -1 = none
};
struct TcArgs {
    const u64 *src;
    long s_cs, s_ps;         // source polynomial p at src + (p / pdiv) s_cs + (p % pdiv) s_ps
    u64 *dst;
    long d_cs, d_ps;
    int pdiv, grouped;       // grouped: group = p % pdiv, else group 0 for every polynomial
    int rr, const1;          // rr: fused ModDown + rescale prelude on target 0; const1: extra source == 1
    u64 pinv_l, pinv_l_sh;
    const TcGroup *groups;   // device
    Tab tab;
    int logn;
};
std::vector<uint8_t> tc_bmatrix(const std::vector<std::vector<u64>> &c, const std::vector<u64> &tprimes, int planes,
                                int ncols);
void k_bconv_tc(const TcArgs &a, int n_polys, cudaStream_t st);

// per-level key-switching / rescale constants (device)
struct LevelConsts {
    int nl, beta;
    DevBuf inv_hat, inv_hat_sh;  // [nl]  (Q'_j / q_i)^{-1} mod q_i
    DevBuf inv_hat_ninv, inv_hat_ninv_sh;  // [nl]  N^{-1} (Q'_j / q_i)^{-1} mod q_i (folded into the INTT)
    DevBuf hat;                  // [beta][16][ne]  (Q'_j / q_i) mod t_e, split-30 packed
    DevBuf half, qlinv, qlinv_sh;  // rescale by q_{nl-1}: [nl-1]
    // fused relinearise-and-rescale (ev_mul_relin_rescale), l = nl - 1 >= 1; see context.cu
    DevBuf rr_fold, rr_fold_sh, rr_hl, rr_hat, rr_binv, rr_binv_sh;
    // tensor-core conversion groups: [0, beta) ModUp digits, beta: fused ModDown + rescale (l >= 1),
    // beta + 1: plain ModDown; tc_ok = every group fits (<= 12 sources, <= 32 targets)
    DevBuf tc_groups, tc_B;
    bool tc_ok = false;
};

// CUDA-event profiling of the dominant kernels inside a timed region (bench.py roofline)
struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    struct Span {
        size_t a, b;
        int kind;      // 0 NTT launch on FP64 rows, 1 key switch, 2 rescale, 3 NTT launch on integer rows,
                       // 4..8 argmax stages H1, H2, H3, H4, H6, 9 fused operand bytes of kind-0 launches (same
                       // events as their kind-0 span)
        double bytes;  // algorithmic bytes of the span
        double units;
    };
    std::vector<Span> spans;
    cudaEvent_t next();
};

struct Counters {
    long long ntt_limbs = 0, keyswitch = 0, rescale = 0, rotate = 0, mulct = 0, mulconst = 0, launches = 0,
              sign = 0;
};

// Ciphertext batch view: n cts; ct c polynomial b limb i at data + c * stride + b * ps + i * N.
// A view at a lower level than its storage is a zero-copy drop (limbs above `level` ignored).
struct CtView {
    u64 *data;
    long stride;  // elements between ciphertexts
    long ps;      // elements between c0 and c1 (= (storage level + 1) * N)
    int n;
    int level;
    double scale;
};

struct Keys;

struct Ctx {
    int logn = 0;
    long N = 0;
    int nq = 0, np = 0, alpha = 1;
    double scale = 0;
    std::vector<u64> primes, psi;  // q_0..q_L, p_0..p_{k-1}
    cudaStream_t st = nullptr;
    // tables
    DevBuf d_q, d_br0, d_br1, d_tw, d_itw, d_ninv, d_ninvsh, d_qd, d_qinv, d_twp, d_itwp;
    Tab tab{};
    // ModDown constants
    DevBuf ihp, ihp_sh, hat_p, pinv, pinv_sh;  // hat_p split-30 packed
    DevBuf ihp_ninv, ihp_ninv_sh;               // N^{-1} (P/p)^{-1} mod p (folded into the INTT)
    DevBuf pmod;                                // [nq] P mod q_i
    std::vector<std::unique_ptr<LevelConsts>> lvl;  // index = level
    // host copies used by planning
    std::vector<u64> h_br0, h_br1, h_pinv, h_pinv_sh;
    // instrumentation
    bool log_on = false;
    std::string oplog;
    Counters cnt;
    Prof prof;
    size_t prof_begin(int kind);
    void prof_end(size_t a, int kind, double bytes, double units);

    // encoded argmax masks (NTT form), keyed by layout / level / scale bits: encoded once per context
    std::map<std::string, std::shared_ptr<DevBuf>> pt_cache;
    // auxiliary streams for concurrent sub-batches (created on first use; SECPE_STREAMS, default 2)
    std::vector<cudaStream_t> aux;
    int n_streams = 2;
    // CUDA graphs of whole argmax calls (SECPE_GRAPH, default on), keyed by buffers / level / circuit;
    // replay adds the counters recorded at capture
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        Counters cnt;
        double out_scale = 0;
        const void *keys = nullptr;  // evaluation keys whose device memory the graph's kernels read
        const void *aux = nullptr;   // other library-owned device memory it reads (bootstrap material)
    };
    std::map<std::string, Graph> graphs;
    std::map<std::string, int> graph_seen;  // eager calls per key: capture on the second sighting only
    std::vector<std::string> graph_order;   // capture order (the oldest graph is evicted beyond kMaxGraphs)
    static constexpr int kMaxGraphs = 16;
    std::set<Keys *> live_keys;          // keys generated on this context (owner back-pointers)
    std::set<BootSetup *> live_boots;    // bootstrap material built on this context (likewise)
    void drop_graphs(const void *keys);  // destroy every graph that reads these keys
    bool use_graphs = true;
    // host-buffer argmax pipeline (secpe_enc_argmax_host): two device staging slots per direction and a
    // copy stream; loaded[s]: slot s's inputs are on the device, freed[s]: slot s's last use has finished
    struct HostPipe {
        DevBuf in[2], out[2];
        size_t in_words = 0, out_words = 0;
        cudaStream_t cp = nullptr;
        cudaEvent_t loaded[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
        int next = 0;
    } pipe;
    ~Ctx();

    int nprimes() const { return nq + np; }
    int L() const { return nq - 1; }
    int beta(int level) const { return (level + 1 + alpha - 1) / alpha; }
    long ct_words(int level) const { return 2L * (level + 1) * N; }
    void build(const u64 *q, int nq_, const u64 *p, int np_, int alpha_, int logn_, double scale_);
    const LevelConsts &level(int l) const { return *lvl[l]; }
    void build_tc_groups(LevelConsts &lc, int l);
    bool use_tc = true;  // tensor-core base conversion (SECPE_NO_TC=1 selects the integer kernels)
    int ntt_cluster = 0; // single-pass cluster NTT (SECPE_NTT_CLUSTER; copied into tab)
    void log(const char *kind, int lin, int lout, double s, const std::string &extra);
};

struct Keys {
    Ctx *owner = nullptr;  // context whose graph cache may reference this key material
    DevBuf s;      // [nq+np][N] NTT
    DevBuf pk;     // [2][nq][N]
    DevBuf rlk;    // [beta_top][2][nq+np][N]
    std::map<u64, DevBuf> gk;
    std::vector<i64> s_coeff;  // not kept (client secret stays on device); unused
};

// host modular helpers (context.cu)
u64 h_mulmod(u64 a, u64 b, u64 q);
u64 h_powmod(u64 a, u64 e, u64 q);
u64 h_invmod(u64 a, u64 q);
u64 h_shoup(u64 w, u64 q);
u64 h_smod(i64 v, u64 q);
u64 h_smod128(i128 v, u64 q);  // |v| < 2^127
bool h_is_prime(u64 n);
int h_gen_primes(int bits, int count, int logn, int mode, const u64 *ex, int nex, u64 *out);
u64 h_find_psi(u64 q, int logn);
void h_cdt(u64 *out, int n);  // 20-entry CDT (quad precision)
u64 galois_elt(const Ctx &c, int steps);
double round_half_away(double x);

// evaluator primitives (eval.cu) -- all operate on batches of n ciphertexts
// Outputs are compact views (stride = 2 (level+1) N, ps = (level+1) N) supplied by the caller.
CtView compact_view(const Ctx &c, u64 *data, int n, int level, double scale);
void ev_ntt(Ctx &c, RowsArg d, int n_polys, LimbMap lm, bool inverse, const NttFusion &f = NttFusion());
void ev_ntt_segs(Ctx &c, const std::vector<NttSeg> &segs, bool inverse);
void ev_ntt_segs_pass1(Ctx &c, const std::vector<NttSeg> &segs);
void ev_copy(Ctx &c, const CtView &a, const CtView &out);
void ev_addsub(Ctx &c, const CtView &a, const CtView &b, const CtView &out, bool sub);
void ev_mul_int(Ctx &c, const CtView &a, i128 C, const CtView &out);
void ev_add_int(Ctx &c, const CtView &a, i128 C, const CtView &out);
void ev_rescale(Ctx &c, const CtView &in, const CtView &out);
void ev_keyswitch(Ctx &c, const u64 *d, long d_stride, int n, int level, const u64 *key, const u64 *add,
                  long add_stride, int add_polys, u64 *out, long out_stride, const CRows *add3 = nullptr);
void ev_mul_relin(Ctx &c, const Keys &k, const CtView &a, const CtView &b, const CtView &out);
// a (x) b [+ a2 (x) b2] [+ C x] relinearised and rescaled by q_l in one pass (bit-identical to ev_mul_relin
// then ev_rescale); out at level a.level - 1.  lin_x: optional linear term (nullptr: none), C its constant;
// a2, b2: optional second product summed into the tensor before the relinearisation (R13b)
void ev_mul_relin_rescale(Ctx &c, const Keys &k, const CtView &a, const CtView &b, const CtView *lin_x, i128 C,
                          const CtView &out, const CtView *lin_x2 = nullptr, i128 C2 = 0, const CtView *a2 = nullptr,
                          const CtView *b2 = nullptr);
void ev_lincomb(Ctx &c, const CtView &a, i128 C1, const CtView *b, i128 C2, const CtView &out);
// rescale(C1 x1 + C2 x2) with the constant products fused into the rescale's transforms (x2 optional)
void ev_rescale_lin(Ctx &c, const CtView &x1, i128 C1, const CtView *x2, i128 C2, const CtView &out);
void ev_rotate(Ctx &c, const Keys &k, const CtView &in, int steps, const CtView &out,
               const CtView *add_after = nullptr);  // add_after: out = RotL(in) + add_after (fused)
void ev_rotate_hoisted(Ctx &c, const Keys &k, const CtView &in, const int *steps, int n_steps, const CtView *outs);
void ev_linear_transform(Ctx &c, const Keys &k, const CtView &in, const u64 *pts, long pt_stride, const int *steps,
                         int n, const CtView &out);
void ev_mod_raise(Ctx &c, const CtView &in, const CtView &out);
void ev_linear_transform_bsgs_gen(Ctx &c, const Keys &k, const CtView &in, const u64 *pts, long pt_stride,
                                  const int *baby, int n1, const int *giant, int n2, const CtView &out);
void ev_linear_transform_bsgs(Ctx &c, const Keys &k, const CtView &in, const u64 *pts, long pt_stride, int n1, int n2,
                              const CtView &out);
void ev_mul_plain_ntt(Ctx &c, const CtView &a, const u64 *pt, const CtView &out);
LimbConst limb_const(const Ctx &c, i128 C, int nl);

// host encode/decode (encode.cpp)
void encode_real(const Ctx &c, const double *slots, size_t n, double scale, std::vector<double> &coef);
void encode_int(const Ctx &c, const double *slots, size_t n, double scale, i64 *out);
void decode_real(const Ctx &c, const std::vector<double> &coef, double scale, double *slots, size_t n);
void encode_mask(const Ctx &c, const double *slots, size_t n, double delta, i64 *out);
void encode_complex_int(const Ctx &c, const double *re, const double *im, size_t n, double scale, i64 *out);

// circuits (plan.cu)
struct SignCfg {
    std::vector<std::vector<double>> stages;
};
// CKKS bootstrapping configuration (readings R32-R35; secpe_boot_cfg)
struct BootCfg {
    int level, n1, n2, r;
    double K;
    std::vector<double> poly;  // 16 power-basis coefficients
    const u64 *cts_re, *cts_im, *stc_re, *stc_im;
    double cts_scale, stc_scale;
};
constexpr int kConjStep = INT32_MIN;  // SECPE_CONJ: slot conjugation, Galois element 2N - 1 (R32)
int boot_depth(const BootCfg &b);
// factorised variant (R37): CoeffToSlot / SlotToCoeff as groups of special-FFT stages, each a hoisted
// diagonal transform (R30); pts dev [n_diag][stage level + 1][N]
struct LtStage {
    std::vector<int> steps;         // diagonal form (R30), or empty with:
    std::vector<int> baby, giant;   // baby-step giant-step form (R39), pts [giant][baby]
    const u64 *pts = nullptr;
    double scale = 0;
};
struct FftBootCfg {
    int level = 0, r = 0;
    double K = 0;
    std::vector<double> poly;
    std::vector<LtStage> cts, stc;  // cts.back(): Re variant of the last CoeffToSlot stage; stc[0]: Re variant
    LtStage cts_im, stc_im;
};
int fft_boot_depth(const FftBootCfg &b);
void run_bootstrap_fft(Ctx &c, const Keys &k, const CtView &in, const FftBootCfg &b, CtView &out);
struct SignCfg;
struct Layout;
int argmax_boot_level(const Layout &lay, const SignCfg &cfg, const FftBootCfg &b, int in_level);
void run_argmax_boot(Ctx &c, const Keys &k, const CtView &in, const Layout &lay, const SignCfg &cfg,
                     const FftBootCfg &b, double boot_scale, int prompt_cts, CtView &out);
// library-built bootstrapping material (secpe_boot_create): the EvalMod polynomial and the four encoded
// matrices, NTT form, [n2][n1][limbs][N] each
struct BootSetup {
    Ctx *ctx = nullptr;  // owner (graph cache); nulled when the context goes first
    bool fft = false;
    BootCfg cfg;
    DevBuf cts_re, cts_im, stc_re, stc_im;
    FftBootCfg fcfg;               // fft: the stages, pts in `bufs`
    std::vector<DevBuf> bufs;
};
BootSetup *boot_setup(Ctx &c, int level, double K, int r, int n1, int n2, double in_scale);
BootSetup *boot_setup_fft(Ctx &c, int level, double K, int r, const std::vector<int> &groups, double in_scale,
                          bool bsgs);
void run_bootstrap(Ctx &c, const Keys &k, const CtView &in, const BootCfg &b, CtView &out);
struct Layout {
    int queries, prompts, classes, block;
};
struct Ev;  // planned evaluator (plan.cu)
void run_sign(Ctx &c, const Keys &k, const CtView &in, const SignCfg &cfg, double target_scale, CtView &out);
void run_argmax(Ctx &c, const Keys &k, const CtView &in, const Layout &lay, const SignCfg &cfg, CtView &out);
int sign_depth(const SignCfg &cfg);
int argmax_depth(const Layout &lay, const SignCfg &cfg);
std::vector<int> argmax_rotations(const Layout &lay);
