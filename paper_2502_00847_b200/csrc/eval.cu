// eval.cu -- batched ciphertext primitives built from the kernels (server side).
//
//   add/sub, constant products, plaintext products, tensor + hybrid key switch
//   (relinearisation), rotation = NTT-domain automorphism + key switch,
//   rescale (leveled chain).  Readings R9-R12 of DESIGN.md fix the integers.
// Every primitive works on a batch of n ciphertexts in one set of launches, so the switching key
// is streamed once per op for the whole batch.
#include "context.h"

static inline RowsArg rows_of(const CtView &v) { return RowsArg{v.data, v.stride, v.ps}; }
static inline CRows crows_of(const CtView &v) { return CRows{v.data, v.stride, v.ps}; }
static inline LimbMap qmap(int nl) { return LimbMap{nl, nl, 0, 0}; }

CtView compact_view(const Ctx &c, u64 *data, int n, int level, double scale) {
    return CtView{data, 2L * (level + 1) * c.N, (long)(level + 1) * c.N, n, level, scale};
}

LimbConst limb_const(const Ctx &c, i128 C, int nl) {
    LimbConst lc{};
    for (int l = 0; l < nl; l++) {
        const u64 q = c.primes[l];
        lc.c[l] = h_smod128(C, q);
        lc.csh[l] = h_shoup(lc.c[l], q);
    }
    return lc;
}

namespace {
// profiling hook: one span per NTT launch, kind 0 (FP64 rows) or 3 (integer rows), algorithmic bytes
// (every limb read once and written once, split evenly over the passes)
struct NttSpans {
    Ctx *c;
    size_t open = 0;
};
void ntt_mark(void *p, int phase, bool fp, double bytes, double limbs, double opbytes) {
    NttSpans &s = *static_cast<NttSpans *>(p);
    if (phase == 0) {
        s.open = s.c->prof_begin(fp ? 0 : 3);
    } else {
        s.c->prof_end(s.open, fp ? 0 : 3, bytes, limbs);
        // the fused operands as a second span over the same two events (kind 9: FP64 rows)
        if (fp && opbytes > 0 && s.c->prof.on) {
            Prof::Span sp = s.c->prof.spans.back();
            sp.kind = 9;
            sp.bytes = opbytes;
            sp.units = 0;
            s.c->prof.spans.push_back(sp);
        }
    }
}
}  // namespace

void ev_ntt(Ctx &c, RowsArg d, int n_polys, LimbMap lm, bool inverse, const NttFusion &f) {
    NttSpans spans{&c};
    const NttProfHook hook{&spans, ntt_mark};
    if (c.prof.on) ntt_set_prof_hook(&hook);
    if (inverse)
        ntt_inverse(c.tab, c.logn, d, n_polys, lm, c.st, f);
    else
        ntt_forward(c.tab, c.logn, d, n_polys, lm, c.st, f);
    if (c.prof.on) ntt_set_prof_hook(nullptr);
    c.cnt.ntt_limbs += (long long)n_polys * lm.nl;
    c.cnt.launches += 2;
}

#ifndef SECPE_NTT_SEGS
#define SECPE_NTT_SEGS 1  // development switch: 0 = one launch pair per segment
#endif
void ev_ntt_segs(Ctx &c, const std::vector<NttSeg> &segs, bool inverse) {
    if (!SECPE_NTT_SEGS) {
        for (auto &g : segs) ev_ntt(c, g.d, g.n_polys, g.lm, inverse);
        return;
    }
    NttSpans spans{&c};
    const NttProfHook hook{&spans, ntt_mark};
    if (c.prof.on) ntt_set_prof_hook(&hook);
    ntt_segments(c.tab, c.logn, segs.data(), (int)segs.size(), inverse, c.st);
    if (c.prof.on) ntt_set_prof_hook(nullptr);
    for (auto &g : segs) c.cnt.ntt_limbs += (long long)g.n_polys * g.lm.nl;
    c.cnt.launches += 2;
}

// the first forward pass of the segments only (the fused ModUp pass 2 + key inner product completes them)
void ev_ntt_segs_pass1(Ctx &c, const std::vector<NttSeg> &segs) {
    NttSpans spans{&c};
    const NttProfHook hook{&spans, ntt_mark};
    if (c.prof.on) ntt_set_prof_hook(&hook);
    ntt_segments_pass1(c.tab, c.logn, segs.data(), (int)segs.size(), c.st);
    if (c.prof.on) ntt_set_prof_hook(nullptr);
    for (auto &g : segs) c.cnt.ntt_limbs += (long long)g.n_polys * g.lm.nl;
    c.cnt.launches += 1;
}

void ev_copy(Ctx &c, const CtView &a, const CtView &out) {
    k_copy_rows(c.logn, crows_of(a), rows_of(out), 2 * a.n, out.level + 1, c.st);
    c.cnt.launches++;
}

void ev_addsub(Ctx &c, const CtView &a, const CtView &b, const CtView &out, bool sub) {
    if (a.scale != b.scale) throw SecpeError{-3, "add/sub: scales are not bit-identical"};
    if (out.level > std::min(a.level, b.level)) throw SecpeError{-1, "add/sub: output level too high"};
    k_addsub(c.tab, c.logn, crows_of(a), crows_of(b), rows_of(out), 2 * a.n, qmap(out.level + 1), sub, c.st);
    c.cnt.launches++;
}

void ev_mul_int(Ctx &c, const CtView &a, i128 C, const CtView &out) {
    const int nl = out.level + 1;
    k_mul_const(c.tab, c.logn, crows_of(a), rows_of(out), 2 * a.n, qmap(nl), limb_const(c, C, nl), c.st);
    c.cnt.launches++;
}

void ev_add_int(Ctx &c, const CtView &a, i128 C, const CtView &out) {
    const int nl = out.level + 1;
    // c0 rows of every ct (poly P = ct: cs = 2 * stride, ps = stride), then copy c1 if out != a
    k_add_const(c.tab, c.logn, CRows{a.data, 2 * a.stride, a.stride}, RowsArg{out.data, 2 * out.stride, out.stride},
                a.n, qmap(nl), limb_const(c, C, nl), c.st);
    c.cnt.launches++;
    if (out.data != a.data) {
        k_copy_rows(c.logn, CRows{a.data + a.ps, 2 * a.stride, a.stride},
                    RowsArg{out.data + out.ps, 2 * out.stride, out.stride}, a.n, nl, c.st);
        c.cnt.launches++;
    }
}

// C1 a + C2 b (b may be null) at out's level (no rescale; the planner rescales the sum once)
void ev_lincomb(Ctx &c, const CtView &a, i128 C1, const CtView *b, i128 C2, const CtView &out) {
    const int nl = out.level + 1;
    k_lincomb2(c.tab, c.logn, crows_of(a), b ? crows_of(*b) : CRows{nullptr, 0, 0}, rows_of(out), 2 * a.n, qmap(nl),
               limb_const(c, C1, nl), b ? limb_const(c, C2, nl) : LimbConst{}, c.st);
    c.cnt.launches++;
}

void ev_mul_plain_ntt(Ctx &c, const CtView &a, const u64 *pt, const CtView &out) {
    const int nl = out.level + 1;
    k_mul_poly(c.tab, c.logn, crows_of(a), pt, rows_of(out), 2 * a.n, qmap(nl), c.st);
    c.cnt.launches++;
}

// Rescale (R12): per coefficient r = [c_l + floor(q_l/2)]_{q_l}; c'_i = (c_i + [floor(q_l/2)]_{q_i} - [r]_{q_i}) q_l^{-1}.
// Two fused transforms: INTT of the last limb (copy fused into its first pass), then a forward NTT
// whose first pass forms (half - r) under each q_i and whose last pass adds c_i and scales by q_l^{-1}.
void ev_rescale(Ctx &c, const CtView &in, const CtView &out) {
    const size_t pa = c.prof_begin(2);
    const int l = in.level;
    if (l < 1) throw SecpeError{-2, "rescale: no level left"};
    if (out.level != l - 1) throw SecpeError{-1, "rescale: bad output level"};
    const long N = c.N;
    const int n = in.n;
    DevBuf last(2L * n * N, c.st), T(2L * n * l * N, c.st);
    NttFusion fi;
    fi.in_mode = 1;
    fi.src = CRows{in.data + l * N, in.stride, in.ps};
    ev_ntt(c, RowsArg{last.p, 2 * N, N}, 2 * n, LimbMap{1, 1, l, 0}, true, fi);
    const LevelConsts &lc = c.level(l);
    NttFusion ff;
    ff.in_mode = 2;
    ff.src = CRows{last.p, 2 * N, N};
    ff.lp = l;
    ff.half = lc.half.p;
    ff.out_mode = 1;
    ff.e1 = crows_of(in);
    ff.out = rows_of(out);
    ff.k = lc.qlinv.p;
    ff.ksh = lc.qlinv_sh.p;
    ev_ntt(c, RowsArg{T.p, 2L * l * N, (long)l * N}, 2 * n, qmap(l), false, ff);
    c.cnt.rescale += n;
    // algorithmic bytes: read 2(l+1) limbs, write 2l limbs per ciphertext
    c.prof_end(pa, 2, 8.0 * (double)n * (2 * (l + 1) + 2 * l) * N, n);
}

// Rescale of C1 x1 (+ C2 x2) with the constant products fused in (no intermediate ciphertext): the INTT
// of the top limb forms C1 x1 + C2 x2 in its first pass, the rescale epilogue forms it per limb.  The
// same integers as ev_mul_int / ev_lincomb followed by ev_rescale.
void ev_rescale_lin(Ctx &c, const CtView &x1, i128 C1, const CtView *x2, i128 C2, const CtView &out) {
    const size_t pa = c.prof_begin(2);
    const int l = out.level + 1;
    if (l < 1) throw SecpeError{-2, "rescale: no level left"};
    if (x1.level < l || (x2 && x2->level < l)) throw SecpeError{-1, "rescale_lin: input level"};
    const long N = c.N;
    const int n = x1.n;
    DevBuf last(2L * n * N, c.st), T(2L * n * l * N, c.st);
    NttFusion fi;
    fi.in_mode = 5;
    fi.lin = x2 ? 2 : 1;
    fi.C1 = C1;
    fi.C2 = C2;
    fi.src = CRows{x1.data + l * N, x1.stride, x1.ps};
    if (x2) fi.src2 = CRows{x2->data + l * N, x2->stride, x2->ps};
    ev_ntt(c, RowsArg{last.p, 2 * N, N}, 2 * n, LimbMap{1, 1, l, 0}, true, fi);
    const LevelConsts &lc = c.level(l);
    NttFusion ff;
    ff.in_mode = 2;
    ff.src = CRows{last.p, 2 * N, N};
    ff.lp = l;
    ff.half = lc.half.p;
    ff.out_mode = 1;
    ff.e1 = crows_of(x1);
    ff.lin = fi.lin;
    ff.C1 = C1;
    ff.C2 = C2;
    if (x2) ff.e1b = crows_of(*x2);
    ff.out = rows_of(out);
    ff.k = lc.qlinv.p;
    ff.ksh = lc.qlinv_sh.p;
    ev_ntt(c, RowsArg{T.p, 2L * l * N, (long)l * N}, 2 * n, qmap(l), false, ff);
    c.cnt.rescale += n;
    c.prof_end(pa, 2, 8.0 * (double)n * ((x2 ? 4 : 2) * (l + 1) + 2 * l) * N, n);
}

// ModUp + key inner product (R10): acc[ct][b][ne][N] over Q_level u P (NTT form).  d01/d01s: optional
// tensor (d0, d1) rows whose [P] multiple is added on the Q limbs (the [P] d term lets the ModDown and the rescale share one conversion).
// ten != nullptr: relinearisation of the tensor of ten->a, ten->b formed on the fly (d unused): the
// INTT's first pass multiplies a1 b1, the inner product forms d0, d1 (+ C x) and adds [P] d_b.
// ModUp of d (or of the tensor's d2 = a1 b1): ext[c][j][e] in NTT form, exts = beta (nl + np) N per ct
static void ks_modup(Ctx &c, const u64 *d, long d_stride, int n, int level, DevBuf &ext,
                     const TensorSrc *ten = nullptr, bool pass1_only = false) {
    const long N = c.N;
    const int nl = level + 1, np = c.np, ne = nl + np, bt = c.beta(level);
    const LevelConsts &lc = c.level(level);
    // 1. y_i = [INTT(d)_i (Q'_j/q_i)^{-1}]_{q_i}: copy and the ModUp factor fused into the INTT
    DevBuf dc((size_t)n * nl * N, c.st);
    NttFusion f1;
    if (ten) {
        f1.in_mode = 3;  // d2 = a1 b1
        f1.src = CRows{ten->a.p + ten->a.ps, 2 * ten->a.cs, ten->a.cs};
        f1.src2 = CRows{ten->b.p + ten->b.ps, 2 * ten->b.cs, ten->b.cs};
        if (ten->a2.p) {  // d2 = a1 b1 + a2_1 b2_1 (R13b)
            f1.in_mode = 4;
            f1.src3 = CRows{ten->a2.p + ten->a2.ps, 2 * ten->a2.cs, ten->a2.cs};
            f1.src4 = CRows{ten->b2.p + ten->b2.ps, 2 * ten->b2.cs, ten->b2.cs};
        }
    } else {
        f1.in_mode = 1;
        f1.src = CRows{d, 2 * d_stride, d_stride};
    }
    f1.k = lc.inv_hat_ninv.p;
    f1.ksh = lc.inv_hat_ninv_sh.p;
    ev_ntt(c, RowsArg{dc.p, 2L * nl * N, (long)nl * N}, n, qmap(nl), true, f1);
    // 2. ModUp into every digit's complement, then NTT of the converted limbs
    const long exts = (long)bt * ne * N;
    ext = DevBuf((size_t)n * exts, c.st);
    if (c.use_tc && lc.tc_ok) {
        TcArgs t{};
        t.src = dc.p;
        t.s_cs = (long)nl * N;
        t.dst = ext.p;
        t.d_cs = exts;
        t.d_ps = (long)ne * N;
        t.pdiv = bt;
        t.grouped = 1;
        t.groups = reinterpret_cast<const TcGroup *>(lc.tc_groups.p);
        t.tab = c.tab;
        t.logn = c.logn;
        k_bconv_tc(t, n * bt, c.st);
    } else {
        k_modup(c.tab, c.logn, dc.p, (long)nl * N, ext.p, exts, n, nl, np, c.nq, c.alpha, lc.hat.p, c.st);
    }
    // NTT of the converted limbs: the Q limbs outside each digit per digit, then the special limbs of
    // every digit of every ciphertext in one launch (n beta polynomials of np rows, stride ne N)
    // (all of them batched into one launch pair per prime class: each alone is a small grid)
    std::vector<NttSeg> segs;
    for (int j = 0; j < bt; j++) {
        const int i0 = j * c.alpha, i1 = std::min(i0 + c.alpha, nl);
        if (i0 > 0) segs.push_back(NttSeg{RowsArg{ext.p + (long)j * ne * N, 2 * exts, exts}, n, LimbMap{i0, i0, 0, 0}});
        if (i1 < nl)
            segs.push_back(NttSeg{RowsArg{ext.p + ((long)j * ne + i1) * N, 2 * exts, exts}, n,
                                  LimbMap{nl - i1, nl - i1, i1, 0}});
    }
    segs.push_back(NttSeg{RowsArg{ext.p + (long)nl * N, 2L * ne * N, (long)ne * N}, n * bt, LimbMap{np, 0, 0, c.nq}});
    if (pass1_only) {
        ev_ntt_segs_pass1(c, segs);
    } else {
        ev_ntt_segs(c, segs, false);
    }
    c.cnt.launches += 1;
}

// Every row of Q_level u P on the exact-FP64 NTT (FpA, q < 2^46): a key switch's ModUp second forward pass and key
// inner product (relinearisation or plain) run as one kernel (ntt_ks_inner).  SECPE_KS_FUSE=0 keeps the separate
// kernels.
#ifndef SECPE_KS_FUSE_INTT
#define SECPE_KS_FUSE_INTT 1  // the fused kernel also runs the ModDown INTT's first pass on its rows
#endif
// SECPE_KS_FUSE: 2 (default) fused ModUp pass 2 + key inner product when every row of Q_level u P is an exact-FP64
// row (FpA or FpB); 1 on every level (integer rows too: bit-exact, measured slower -- configs[2] 4234 -> 3766 ops/s,
// single N = 2^16 bootstrap 28.2 -> 30.9 ms); 3 only when every row is FpA; 0 never
static bool ks_fuse_ok(const Ctx &c, int level) {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("SECPE_KS_FUSE");
        on = e ? atoi(e) : 2;
    }
    if (!on || c.beta(level) > 4) return false;
    if (on == 1) return true;
    const int nl = level + 1;
    const u64 mask = on == 3 ? c.tab.fp_mask : (c.tab.fp_mask | c.tab.fpb_mask);
    for (int i = 0; i < nl; i++)
        if (i >= 64 || !((mask >> i) & 1)) return false;
    for (int p = 0; p < c.np; p++)
        if (c.nq + p >= 64 || !((mask >> (c.nq + p)) & 1)) return false;
    return true;
}

// 3. inner product of the ModUp digits with the switching key (galois > 1: of sigma_g of the digits)
static void ks_inner(Ctx &c, const u64 *d, long d_stride, int n, int level, const u64 *key, const DevBuf &ext,
                     DevBuf &acc, const TensorSrc *ten = nullptr, u64 galois = 1) {
    const long N = c.N;
    const int nl = level + 1, np = c.np, ne = nl + np, bt = c.beta(level);
    const long exts = (long)bt * ne * N, accs = 2L * ne * N;
    acc = DevBuf((size_t)n * accs, c.st);
    k_ks_inner(c.tab, c.logn, d, d_stride, ext.p, exts, key, c.nq, np, acc.p, accs, n, nl, c.alpha, c.st, ten,
               c.pmod.p, galois);
    c.cnt.launches += 1;
}

// returns true when the fused kernel ran; then rows >= intt_row0 (if >= 0) of acc already hold the first pass of their
// inverse NTT (finish with ev_intt_last)
static bool ks_modup_inner(Ctx &c, const u64 *d, long d_stride, int n, int level, const u64 *key, DevBuf &acc,
                           const TensorSrc *ten = nullptr, int intt_row0 = -1) {
    DevBuf ext;
    if (ks_fuse_ok(c, level)) {
        ks_modup(c, d, d_stride, n, level, ext, ten, true);
        const long N = c.N;
        const int nl = level + 1, ne = nl + c.np, bt = c.beta(level);
        acc = DevBuf((size_t)n * 2L * ne * N, c.st);
        KsFuse f{ext.p, (long)bt * ne * N, key, acc.p, 2L * ne * N, n, nl, c.np, c.nq, c.alpha, bt,
                 ten ? *ten : TensorSrc{}, c.pmod.p, d, d_stride, SECPE_KS_FUSE_INTT ? intt_row0 : -1};
        NttSpans spans{&c};
        const NttProfHook hook{&spans, ntt_mark};
        if (c.prof.on) ntt_set_prof_hook(&hook);
        ntt_ks_inner(c.tab, c.logn, f, c.st);
        if (c.prof.on) ntt_set_prof_hook(nullptr);
        c.cnt.launches += 1;
        return SECPE_KS_FUSE_INTT && intt_row0 >= 0;
    }
    ks_modup(c, d, d_stride, n, level, ext, ten);
    ks_inner(c, d, d_stride, n, level, key, ext, acc, ten);
    return false;
}

// the inverse NTT's last pass only (the first ran inside the fused key-switch kernel)
static void ev_intt_last(Ctx &c, RowsArg d, int n_polys, LimbMap lm, const NttFusion &f) {
    NttSpans spans{&c};
    const NttProfHook hook{&spans, ntt_mark};
    if (c.prof.on) ntt_set_prof_hook(&hook);
    ntt_inverse_last_pass(c.tab, c.logn, d, n_polys, lm, c.st, f);
    if (c.prof.on) ntt_set_prof_hook(nullptr);
    c.cnt.ntt_limbs += (long long)n_polys * lm.nl;
    c.cnt.launches += 1;
}

// Hybrid key switching of d (NTT form; ct c at d + c * d_stride, level limbs), result added to
// `add` (add_polys of 2 polynomials; compact, ct stride add_stride) and written compact to out.
static void ks_moddown(Ctx &c, DevBuf &acc, int n, int level, const u64 *add, long add_stride, int add_polys,
                       u64 *out, long out_stride, const CRows *add3 = nullptr, bool intt_pre = false);

void ev_keyswitch(Ctx &c, const u64 *d, long d_stride, int n, int level, const u64 *key, const u64 *add,
                  long add_stride, int add_polys, u64 *out, long out_stride, const CRows *add3) {
    const long N = c.N;
    const int nl = level + 1, np = c.np, ne = nl + np, bt = c.beta(level);
    const size_t pa = c.prof_begin(1);
    DevBuf acc;
    const bool pre = ks_modup_inner(c, d, d_stride, n, level, key, acc, nullptr, level + 1);
    ks_moddown(c, acc, n, level, add, add_stride, add_polys, out, out_stride, add3, pre);
    c.cnt.keyswitch += n;
    // algorithmic bytes: input limbs + output limbs per ciphertext + the key once per batch
    c.prof_end(pa, 1, 8.0 * N * ((double)n * (nl + 2 * nl + add_polys * nl) + 2.0 * bt * ne), n);
}

// ModDown of acc (R11) with the addend fused into the final NTT's epilogue; result compact in out
static void ks_moddown(Ctx &c, DevBuf &acc, int n, int level, const u64 *add, long add_stride, int add_polys,
                       u64 *out, long out_stride, const CRows *add3, bool intt_pre) {
    const long N = c.N;
    const int nl = level + 1, np = c.np, ne = nl + np, bt = c.beta(level);
    const long accs = 2L * ne * N;
    // 4. ModDown: INTT of the special limbs (with (P/p)^{-1} folded in), conversion to Q, then an NTT
    //    whose last pass forms (acc - T) P^{-1} + addend
    NttFusion f4;
    f4.k = c.ihp_ninv.p;
    f4.ksh = c.ihp_ninv_sh.p;
    if (intt_pre)
        ev_intt_last(c, RowsArg{acc.p + (long)nl * N, accs, (long)ne * N}, 2 * n, LimbMap{np, 0, 0, c.nq}, f4);
    else
        ev_ntt(c, RowsArg{acc.p + (long)nl * N, accs, (long)ne * N}, 2 * n, LimbMap{np, 0, 0, c.nq}, true, f4);
    const long Ts = 2L * nl * N;
    DevBuf T((size_t)n * Ts, c.st);
    const LevelConsts &lc = c.level(level);
    if (c.use_tc && lc.tc_ok) {
        TcArgs t{};
        t.src = acc.p;
        t.s_cs = accs;
        t.s_ps = (long)ne * N;
        t.dst = T.p;
        t.d_cs = Ts;
        t.d_ps = (long)nl * N;
        t.pdiv = 2;
        t.groups = reinterpret_cast<const TcGroup *>(lc.tc_groups.p) + bt + 1;
        t.tab = c.tab;
        t.logn = c.logn;
        k_bconv_tc(t, 2 * n, c.st);
    } else {
        k_moddown_conv(c.tab, c.logn, acc.p, accs, ne, nl, np, T.p, Ts, nl, n, c.hat_p.p, c.nq, c.st);
    }
    NttFusion f6;
    f6.out_mode = 2;
    f6.e1 = CRows{acc.p, accs, (long)ne * N};
    f6.e2 = CRows{add, add_stride, (long)nl * N};
    f6.e2_polys = add ? add_polys : 0;
    if (add3) f6.e3 = *add3;
    f6.out = RowsArg{out, out_stride, (long)nl * N};
    f6.k = c.pinv.p;
    f6.ksh = c.pinv_sh.p;
    ev_ntt(c, RowsArg{T.p, Ts, (long)nl * N}, 2 * n, qmap(nl), false, f6);
    c.cnt.launches += 1;
}

// Relinearise and rescale in one pass, bit-identical to ev_mul_relin followed by ev_rescale (R10-R12):
// with x_b = acc_b + [P] d_b (formed inside the key inner product), the relinearised ciphertext is
// Y_b = (x_b - ModDownConv(x_b)) P^{-1} and its rescale is (Y_b + half - [r]) q_l^{-1}; both
// corrections are computed in the coefficient domain (k_rr_conv) and removed by ONE forward NTT whose
// epilogue forms (x_i - NTT(T_i)) (P q_l)^{-1}.  This saves the rescale's own INTT/NTT round trip.
void ev_mul_relin_rescale(Ctx &c, const Keys &k, const CtView &a, const CtView &b, const CtView *lin_x, i128 C,
                          const CtView &out, const CtView *lin_x2, i128 C2, const CtView *a2, const CtView *b2) {
    const int l = a.level, nl = l + 1;
    if (l < 1) throw SecpeError{-2, "mul_relin_rescale: no level left"};
    if (b.level != l || out.level != l - 1) throw SecpeError{-1, "mul_relin_rescale: levels"};
    const long N = c.N;
    const int n = a.n, np = c.np, ne = nl + np, bt = c.beta(l);
    const LevelConsts &lc = c.level(l);
    // the tensor (d0, d1, d2) is never materialised: d2 = a1 b1 is formed by the INTT's first pass and
    // d0, d1 (+ C x) inside the key inner product
    TensorSrc ten{};
    ten.a = crows_of(a);
    ten.b = crows_of(b);
    if (lin_x) {
        ten.x = crows_of(*lin_x);
        ten.C = limb_const(c, C, nl);
    }
    if (lin_x2) {
        ten.x2 = crows_of(*lin_x2);
        ten.C2 = limb_const(c, C2, nl);
    }
    if (a2) {
        if (!b2 || a2->level < l || b2->level < l || a2->n != n || b2->n != n)
            throw SecpeError{-1, "mul_relin_rescale: second product"};
        ten.a2 = crows_of(*a2);
        ten.b2 = crows_of(*b2);
    }
    const size_t pa = c.prof_begin(1);
    DevBuf acc;
    const bool pre = ks_modup_inner(c, nullptr, 0, n, l, k.rlk.p, acc, &ten, l);
    const long accs = 2L * ne * N;
    // INTT of the B rows (q_l row, then the special rows: contiguous rows l .. ne-1) with (B/s)^{-1} folded
    NttFusion f4;
    f4.k = lc.rr_fold.p;
    f4.ksh = lc.rr_fold_sh.p;
    if (pre)
        ev_intt_last(c, RowsArg{acc.p + (long)l * N, accs, (long)ne * N}, 2 * n, LimbMap{np + 1, 1, l, c.nq}, f4);
    else
        ev_ntt(c, RowsArg{acc.p + (long)l * N, accs, (long)ne * N}, 2 * n, LimbMap{np + 1, 1, l, c.nq}, true, f4);
    const long Ts = 2L * l * N;
    DevBuf T((size_t)n * Ts, c.st);
    if (c.use_tc && lc.tc_ok) {
        TcArgs t{};
        t.src = acc.p;
        t.s_cs = accs;
        t.s_ps = (long)ne * N;
        t.dst = T.p;
        t.d_cs = Ts;
        t.d_ps = (long)l * N;
        t.pdiv = 2;
        t.rr = 1;
        t.const1 = 1;
        t.pinv_l = c.h_pinv[l];
        t.pinv_l_sh = c.h_pinv_sh[l];
        t.groups = reinterpret_cast<const TcGroup *>(lc.tc_groups.p) + bt;
        t.tab = c.tab;
        t.logn = c.logn;
        k_bconv_tc(t, 2 * n, c.st);
    } else {
        k_rr_conv(c.tab, c.logn, acc.p, accs, ne, l, np, T.p, Ts, n, lc.rr_hat.p, lc.rr_hl.p, c.h_pinv[l],
                  c.h_pinv_sh[l], c.st);
    }
    NttFusion f6;
    f6.out_mode = 2;
    f6.e1 = CRows{acc.p, accs, (long)ne * N};
    f6.out = rows_of(out);
    f6.k = lc.rr_binv.p;
    f6.ksh = lc.rr_binv_sh.p;
    ev_ntt(c, RowsArg{T.p, Ts, (long)l * N}, 2 * n, qmap(l), false, f6);
    c.cnt.launches += 1;
    c.cnt.keyswitch += n;
    c.cnt.rescale += n;
    c.cnt.mulct += n;
    c.prof_end(pa, 1, 8.0 * N * ((double)n * ((a2 ? 5 : 3) * nl + 2 * l) + 2.0 * bt * ne), n);
}

void ev_mul_relin(Ctx &c, const Keys &k, const CtView &a, const CtView &b, const CtView &out) {
    const int l = out.level, nl = l + 1;
    if (a.level < l || b.level < l) throw SecpeError{-1, "mul_relin: level"};
    const long N = c.N, ds = 3L * nl * N;
    DevBuf d((size_t)a.n * ds, c.st);
    k_tensor(c.tab, c.logn, crows_of(a), crows_of(b), d.p, ds, a.n, nl, c.st);
    c.cnt.launches++;
    ev_keyswitch(c, d.p + 2L * nl * N, ds, a.n, l, k.rlk.p, d.p, ds, 2, out.data, out.stride);
    c.cnt.mulct += a.n;
}

void ev_rotate(Ctx &c, const Keys &k, const CtView &in, int steps, const CtView &out, const CtView *add_after) {
    const u64 g = galois_elt(c, steps);
    const int nl = out.level + 1;
    if (g == 1) {
        if (add_after) ev_addsub(c, in, *add_after, out, false);
        else ev_copy(c, in, out);
        return;
    }
    auto it = k.gk.find(g);
    if (it == k.gk.end()) throw SecpeError{-4, "no Galois key for rotation step " + std::to_string(steps)};
    const long N = c.N, ss = 2L * nl * N;
    DevBuf sig((size_t)in.n * ss, c.st);
    k_automorph(c.logn, crows_of(in), RowsArg{sig.p, ss, (long)nl * N}, 2 * in.n, nl, g, c.st);
    c.cnt.launches++;
    CRows a3{};
    if (add_after) {
        if (add_after->level < out.level || add_after->n != in.n) throw SecpeError{-1, "rotate: addend"};
        a3 = crows_of(*add_after);
    }
    ev_keyswitch(c, sig.p + (long)nl * N, ss, in.n, out.level, it->second.p, sig.p, ss, 1, out.data, out.stride,
                 add_after ? &a3 : nullptr);
    c.cnt.rotate += in.n;
}

// Hoisted diagonal-form linear transform (R30): out = Rescale(sum_i pt_i (.) RotL(in, steps[i])), one
// ModUp shared by all rotations (R29); pt_i dev [level+1][N] NTT-form rows at pts + i * pt_stride.
void ev_linear_transform(Ctx &c, const Keys &k, const CtView &in, const u64 *pts, long pt_stride, const int *steps,
                         int n, const CtView &out) {
    if (n < 1) throw SecpeError{-1, "linear_transform: no diagonals"};
    const int l = in.level, nl = l + 1, B = in.n;  // a batch of B ciphertexts, one transform
    if (l < 1) throw SecpeError{-2, "linear_transform: no level left to rescale"};
    if (out.level != l - 1 || out.n != B) throw SecpeError{-1, "linear_transform: output level"};
    const long N = c.N, cw = 2L * nl * N, bw = (long)B * cw;
    DevBuf rot((size_t)n * bw, c.st);
    std::vector<CtView> outs(n);
    for (int i = 0; i < n; i++) outs[i] = compact_view(c, rot.p + (long)i * bw, B, l, in.scale);
    ev_rotate_hoisted(c, k, in, steps, n, outs.data());
    DevBuf acc(bw, c.st);
    const CtView va = compact_view(c, acc.p, B, l, in.scale);
    k_mac_plain(c.tab, c.logn, CRows{rot.p, cw, (long)nl * N}, bw, pts, pt_stride, n, rows_of(va), 2 * B, qmap(nl),
                c.st);
    c.cnt.launches++;
    ev_rescale(c, va, out);
}

// ModRaise (R33, bootstrapping's first step): level-0 (c0, c1) -> INTT of limb 0 -> centred lift ->
// residues mod q_0..q_L -> NTT.  The result decrypts to t = m + q_0 I over the integers.
void ev_mod_raise(Ctx &c, const CtView &in, const CtView &out) {
    if (in.level != 0) throw SecpeError{-1, "mod_raise: input must be at level 0"};
    if (out.level < 1 || out.n != in.n) throw SecpeError{-1, "mod_raise: output level"};
    const long N = c.N;
    const int np = 2 * in.n;
    DevBuf coef((size_t)np * N, c.st);
    k_copy_rows(c.logn, crows_of(in), RowsArg{coef.p, 2 * N, N}, np, 1, c.st);
    ev_ntt(c, RowsArg{coef.p, 2 * N, N}, np, qmap(1), true);
    k_mod_raise(c.tab, c.logn, coef.p, rows_of(out), np, out.level + 1, c.st);
    ev_ntt(c, rows_of(out), np, qmap(out.level + 1), false);
    c.cnt.launches += 2;
}

// General baby-step giant-step transform (R39): out = Rescale( sum_g RotL( sum_j pt_{g,j} (.) RotL(in, baby_j),
// giant_g ) ); the baby rotations hoisted (R29), each giant rotation's addition fused into its key switch
// epilogue (a zero giant step is a plain copy / addition).  pt_{g,j}: dev [level+1][N] rows at
// pts + (g n1 + j) pt_stride.
void ev_linear_transform_bsgs_gen(Ctx &c, const Keys &k, const CtView &in, const u64 *pts, long pt_stride,
                                  const int *baby, int n1, const int *giant, int n2, const CtView &out) {
    if (n1 < 1 || n2 < 1) throw SecpeError{-1, "linear_transform_bsgs: empty"};
    const int l = in.level, nl = l + 1, B = in.n;  // a batch of B ciphertexts, one transform
    if (l < 1) throw SecpeError{-2, "linear_transform_bsgs: no level left to rescale"};
    if (out.level != l - 1 || out.n != B) throw SecpeError{-1, "linear_transform_bsgs: output level"};
    const long N = c.N, cw = 2L * nl * N, bw = (long)B * cw;
    DevBuf rot((size_t)n1 * bw, c.st);
    std::vector<CtView> outs(n1);
    for (int j = 0; j < n1; j++) outs[j] = compact_view(c, rot.p + (long)j * bw, B, l, in.scale);
    ev_rotate_hoisted(c, k, in, baby, n1, outs.data());
    DevBuf inner(bw, c.st), accb[2] = {DevBuf(bw, c.st), DevBuf(bw, c.st)};
    const CtView vin = compact_view(c, inner.p, B, l, in.scale);
    int cur = 0;
    for (int g = 0; g < n2; g++) {
        // the first term lands in the accumulator directly when it needs no rotation
        const bool direct = g == 0 && galois_elt(c, giant[0]) == 1;
        const CtView dst = compact_view(c, direct ? accb[0].p : inner.p, B, l, in.scale);
        k_mac_plain(c.tab, c.logn, CRows{rot.p, cw, (long)nl * N}, bw, pts + (long)g * n1 * pt_stride, pt_stride, n1,
                    rows_of(dst), 2 * B, qmap(nl), c.st);
        c.cnt.launches++;
        if (direct) continue;
        if (g == 0) {
            ev_rotate(c, k, vin, giant[0], compact_view(c, accb[0].p, B, l, in.scale));
        } else {
            const CtView acc = compact_view(c, accb[cur].p, B, l, in.scale);
            const CtView nxt = compact_view(c, accb[cur ^ 1].p, B, l, in.scale);
            ev_rotate(c, k, vin, giant[g], nxt, &acc);  // nxt = RotL(inner, giant_g) + acc
            cur ^= 1;
        }
    }
    ev_rescale(c, compact_view(c, accb[cur].p, B, l, in.scale), out);
}

// Baby-step giant-step linear transform (R31): baby steps 0..n1-1, giant steps g n1
void ev_linear_transform_bsgs(Ctx &c, const Keys &k, const CtView &in, const u64 *pts, long pt_stride, int n1, int n2,
                              const CtView &out) {
    if (n1 < 1 || n2 < 1) throw SecpeError{-1, "linear_transform_bsgs: empty"};
    std::vector<int> baby(n1), giant(n2);
    for (int j = 0; j < n1; j++) baby[j] = j;
    for (int g = 0; g < n2; g++) giant[g] = g * n1;
    ev_linear_transform_bsgs_gen(c, k, in, pts, pt_stride, baby.data(), n1, giant.data(), n2, out);
}

// Hoisted rotations (N2, reading R29): one ModUp of c1 shared by every step; per step the key inner
// product gathers sigma_g of the digits (k_ks_inner galois), ModDown adds sigma_g(c0) in its final NTT.
// Same integers as the oracle's rotate_hoisted_raw (not as ev_rotate: ModUp does not commute with sigma_g).
void ev_rotate_hoisted(Ctx &c, const Keys &k, const CtView &in, const int *steps, int n_steps, const CtView *outs) {
    if (n_steps <= 0) return;
    const int level = outs[0].level, nl = level + 1, n = in.n;
    for (int i = 0; i < n_steps; i++) {
        if (outs[i].level != level || outs[i].n != n) throw SecpeError{-1, "rotate_hoisted: output batches differ"};
        const u64 g = galois_elt(c, steps[i]);
        if (g != 1 && k.gk.find(g) == k.gk.end())
            throw SecpeError{-4, "no Galois key for rotation step " + std::to_string(steps[i])};
    }
    if (level > in.level) throw SecpeError{-1, "rotate_hoisted: output level above input"};
    const long N = c.N, np = c.np, ne = nl + np, bt = c.beta(level);
    const size_t pa = c.prof_begin(1);
    const u64 *c1 = in.data + in.ps;
    DevBuf ext;
    bool have_ext = false;
    int n_ks = 0;
    for (int i = 0; i < n_steps; i++) {
        const u64 g = galois_elt(c, steps[i]);
        if (g == 1) {
            ev_copy(c, in, outs[i]);
            continue;
        }
        if (!have_ext) {
            ks_modup(c, c1, in.stride, n, level, ext);
            have_ext = true;
        }
        const u64 *key = k.gk.find(g)->second.p;
        DevBuf sig0((size_t)n * nl * N, c.st);  // sigma_g(c0) of every ciphertext, compact
        k_automorph(c.logn, CRows{in.data, 2 * in.stride, in.stride}, RowsArg{sig0.p, 2L * nl * N, (long)nl * N}, n,
                    nl, g, c.st);
        c.cnt.launches++;
        DevBuf acc;
        ks_inner(c, c1, in.stride, n, level, key, ext, acc, nullptr, g);
        ks_moddown(c, acc, n, level, sig0.p, (long)nl * N, 1, outs[i].data, outs[i].stride);
        c.cnt.keyswitch += n;
        c.cnt.rotate += n;
        n_ks++;
    }
    // algorithmic bytes: c1 once + per rotation (c0 in, output, key once per batch)
    c.prof_end(pa, 1, 8.0 * N * ((double)n * nl + n_ks * ((double)n * 3 * nl + 2.0 * bt * ne)), (double)n * n_ks);
}
