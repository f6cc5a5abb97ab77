// plan.cu -- SecPE circuits on the GPU evaluator: composite Sign (Eq. 3-4 with
// BSGS), homomorphic Max (Eq. 6) and Algorithm 1 Argmax with
// prompt aggregation and Eq. 5 normalisation.
//
// Scale planning (R9): every sub-expression is requested at a target (scale, level);
// constant products absorb all scale drift (Delta_c = S_t q_l / S_x), ct x ct products are
// assigned their target scale after rescale, so every addition sees bit-identical scales.
// BSGS plans (R13) for odd degrees 3, 7, 15; emission order "first operand first".
#include <cmath>
#include <cstring>

#include "context.h"

namespace {

std::string dbits(double x) {
    u64 b;
    std::memcpy(&b, &x, 8);
    char buf[24];
    snprintf(buf, sizeof buf, "%016llx", (unsigned long long)b);
    return buf;
}

struct Val {
    std::shared_ptr<DevBuf> buf;
    CtView v;
    int level() const { return v.level; }
    double scale() const { return v.scale; }
};

}  // namespace

#ifndef SECPE_FUSE_LIN
#define SECPE_FUSE_LIN 1  // development switch: constant products fused into their rescale
#endif
#ifndef SECPE_FUSE_ROTADD
#define SECPE_FUSE_ROTADD 1  // development switch
#endif
struct Ev {
    Ctx &c;
    const Keys &k;
    int n;

    double q(int l) const { return (double)c.primes[l]; }

    Val fresh(int level, double scale) {
        auto b = std::make_shared<DevBuf>((size_t)n * c.ct_words(level), c.st);
        return Val{b, compact_view(c, b->p, n, level, scale)};
    }
    Val drop(const Val &x, int level) {
        if (level > x.level()) throw SecpeError{-2, "not enough levels"};
        Val y = x;
        y.v.level = level;
        return y;
    }
    Val add(const Val &a, const Val &b, bool sub = false) {
        const int lv = std::min(a.level(), b.level());
        Val out = fresh(lv, a.scale());
        ev_addsub(c, a.v, b.v, out.v, sub);
        c.log(sub ? "SUB" : "ADD", std::max(a.level(), b.level()), lv, out.scale(), "");
        return out;
    }
    Val sub(const Val &a, const Val &b) { return add(a, b, true); }
    Val rot(const Val &x, int steps) {
        Val out = fresh(x.level(), x.scale());
        ev_rotate(c, k, x.v, steps, out.v);
        c.log("ROT", x.level(), x.level(), x.scale(), std::to_string(galois_elt(c, steps)));
        return out;
    }
    // y + Rot(y, steps): the addition fused into the rotation's final NTT epilogue (same integers as
    // rot then add; the op log keeps both lines)
    Val rot_add(const Val &y, int steps) {
        if (!SECPE_FUSE_ROTADD || galois_elt(c, steps) == 1) return add(y, rot(y, steps));
        Val out = fresh(y.level(), y.scale());
        ev_rotate(c, k, y.v, steps, out.v, &y.v);
        c.log("ROT", y.level(), y.level(), y.scale(), std::to_string(galois_elt(c, steps)));
        c.log("ADD", y.level(), y.level(), y.scale(), "");
        return out;
    }
    Val mul_const(const Val &x, double cval, double St, int Lt) {
        const int lv = Lt + 1;
        if (lv < 1) throw SecpeError{-2, "mul_const: no level left"};
        Val xd = drop(x, lv);
        const double dc = (St * q(lv)) / x.scale();
        const i128 C = const_of(round_half_away(cval * dc));
        Val out = fresh(Lt, St);
        if (SECPE_FUSE_LIN) {
            ev_rescale_lin(c, xd.v, C, nullptr, 0, out.v);  // C x rescaled, the product fused in
        } else {
            Val tmp = fresh(lv, x.scale() * dc);
            ev_mul_int(c, xd.v, C, tmp.v);
            ev_rescale(c, tmp.v, out.v);
        }
        c.cnt.mulconst += n;
        c.log("MULC", lv, Lt, St, int_str(C));
        return out;
    }
    // integer constant C = rha(c Delta), Delta = (S_t q_l) / S_x (R9)
    i128 lin_const(double cval, double St, int lv, double Sx) {
        const double dc = (St * q(lv)) / Sx;
        return const_of(round_half_away(cval * dc));
    }
    // the integer value of an integer-valued double, |C| < 2^120 (with Delta_c ~ q ~ 2^49 the Sign coefficients,
    // up to 2^14.8, give C ~ 2^64; the conversion of an integer-valued double is exact)
    static i128 const_of(double Cd) {
        if (!(std::fabs(Cd) < 1329227995784915872903807060280344576.0)) throw SecpeError{-6, "constant exceeds 2^120"};
        return (i128)Cd;
    }
    static std::string int_str(i128 v) {
        if (v == 0) return "0";
        const bool neg = v < 0;
        u128 a = (u128)(neg ? -v : v);
        std::string r;
        while (a) {
            r.insert(r.begin(), char('0' + (int)(a % 10)));
            a /= 10;
        }
        return neg ? "-" + r : r;
    }
    using Lin = std::vector<std::pair<const Val *, double>>;
    static std::string join(const std::vector<i128> &v) {
        std::string r;
        for (size_t i = 0; i < v.size(); i++) r += (i ? "," : "") + int_str(v[i]);
        return r;
    }
    // a (x) b [+ sum c x] relinearised and rescaled in one pass; St = NAN: natural scale (S_a S_b) / q_l.
    // Up to two linear terms join the product before its rescale (R13).
    // a2, b2 (optional): a second product summed into the tensor, one relinearisation for both (R13b)
    Val mul_ct(const Val &a, const Val &b, double St, int Lt, const Lin &lin = {}, const Val *a2 = nullptr,
               const Val *b2 = nullptr) {
        const int lv = Lt + 1;
        if (lv < 1) throw SecpeError{-2, "mul_ct: no level left"};
        if (lin.size() > 2) throw SecpeError{-1, "mul_ct: at most two linear terms"};
        if (a2 && std::isnan(St)) throw SecpeError{-1, "mul_ct: a summed product needs a planned scale"};
        Val ad = drop(a, lv), bd = drop(b, lv);
        Val a2d = a2 ? drop(*a2, lv) : Val{}, b2d = a2 ? drop(*b2, lv) : Val{};
        const double s = std::isnan(St) ? (a.scale() * b.scale()) / q(lv) : St;
        Val out = fresh(Lt, s);
        std::vector<Val> xs;
        std::vector<i128> Cs;
        for (auto &t : lin) {
            xs.push_back(drop(*t.first, lv));
            Cs.push_back(lin_const(t.second, s, lv, t.first->scale()));
        }
        ev_mul_relin_rescale(c, k, ad.v, bd.v, xs.size() > 0 ? &xs[0].v : nullptr, xs.size() > 0 ? Cs[0] : 0, out.v,
                             xs.size() > 1 ? &xs[1].v : nullptr, xs.size() > 1 ? Cs[1] : 0, a2 ? &a2d.v : nullptr,
                             a2 ? &b2d.v : nullptr);
        c.log(a2 ? "MULCT2" : "MULCT", lv, Lt, s, join(Cs));
        return out;
    }
    // sum c_i x_i (one or two terms) at (St, Lt) with a single rescale (R13)
    Val lincomb(const Lin &terms, double St, int Lt) {
        const int lv = Lt + 1;
        if (lv < 1) throw SecpeError{-2, "lincomb: no level left"};
        if (terms.empty() || terms.size() > 2) throw SecpeError{-1, "lincomb: one or two terms"};
        std::vector<Val> xs;
        std::vector<i128> Cs;
        for (auto &t : terms) {
            xs.push_back(drop(*t.first, lv));
            Cs.push_back(lin_const(t.second, St, lv, t.first->scale()));
        }
        Val out = fresh(Lt, St);
        if (SECPE_FUSE_LIN) {
            ev_rescale_lin(c, xs[0].v, Cs[0], xs.size() > 1 ? &xs[1].v : nullptr, xs.size() > 1 ? Cs[1] : 0, out.v);
        } else {
            Val tmp = fresh(lv, St * q(lv));
            ev_lincomb(c, xs[0].v, Cs[0], xs.size() > 1 ? &xs[1].v : nullptr, xs.size() > 1 ? Cs[1] : 0, tmp.v);
            ev_rescale(c, tmp.v, out.v);
        }
        c.cnt.mulconst += n;
        c.log("LINC", lv, Lt, St, join(Cs));
        return out;
    }
    // cache_key: non-empty for masks that are a function of the key alone (the argmax mask of a layout):
    // the encoded plaintext is then kept in the context and reused (no host work or sync next time)
    Val mul_mask(const Val &x, const std::vector<double> &mask, double St, const std::string &cache_key = "") {
        const int lv = x.level();
        if (lv < 1) throw SecpeError{-2, "mul_mask: no level left"};
        const double dm = (St * q(lv)) / x.scale();
        const long N = c.N;
        const std::string key = cache_key.empty() ? "" : cache_key + "/" + std::to_string(lv) + "/" + dbits(dm);
        std::shared_ptr<DevBuf> pt;
        if (!key.empty()) {
            auto it = c.pt_cache.find(key);
            if (it != c.pt_cache.end()) pt = it->second;
        }
        if (!pt) {
            std::vector<i64> M(N);
            encode_mask(c, mask.data(), mask.size(), dm, M.data());
            DevBuf mi(N, c.st);
            pt = std::make_shared<DevBuf>((size_t)(lv + 1) * N, c.st);
            CUDA_CHECK(cudaMemcpyAsync(mi.p, M.data(), N * 8, cudaMemcpyHostToDevice, c.st));
            k_int_to_rows(c.tab, c.logn, (const i64 *)mi.p, pt->p, LimbMap{lv + 1, lv + 1, 0, 0}, c.st);
            ev_ntt(c, RowsArg{pt->p, 2L * (lv + 1) * N, (long)(lv + 1) * N}, 1, LimbMap{lv + 1, lv + 1, 0, 0},
                   false);
            CUDA_CHECK(cudaStreamSynchronize(c.st));  // M is host memory of this frame
            if (!key.empty()) c.pt_cache[key] = pt;
        }
        Val tmp = fresh(lv, x.scale() * dm);
        ev_mul_plain_ntt(c, x.v, pt->p, tmp.v);
        Val out = fresh(lv - 1, St);
        ev_rescale(c, tmp.v, out.v);
        c.log("MULP", lv, lv - 1, St, dbits(dm));
        return out;
    }
    Val add_const(const Val &x, double cval) {
        const i128 C = const_of(round_half_away(cval * x.scale()));
        Val out = fresh(x.level(), x.scale());
        ev_add_int(c, x.v, C, out.v);
        c.log("ADDC", x.level(), x.level(), x.scale(), int_str(C));
        return out;
    }

    // ---- bootstrapping (readings R32-R35) ---------------------------------------
    Val mod_raise(const Val &x, int level) {
        Val out = fresh(level, x.scale());
        ev_mod_raise(c, x.v, out.v);
        c.log("MODRAISE", 0, level, x.scale(), "");
        return out;
    }
    // Rescale(sum_g RotL(sum_j pt_{g,j} (.) RotL(x, j), g n1)) (R31); output scale (S_x pt_scale) / q_l
    Val lt_bsgs(const Val &x, const u64 *pts, int n1, int n2, double pt_scale) {
        const int l = x.level();
        const double s = (x.scale() * pt_scale) / q(l);
        Val out = fresh(l - 1, s);
        ev_linear_transform_bsgs(c, k, x.v, pts, (long)(l + 1) * c.N, n1, n2, out.v);
        c.log("LTB", l, l - 1, s, std::to_string(n1) + "x" + std::to_string(n2));
        return out;
    }
    // hoisted diagonal transform Rescale(sum_i pt_i (.) RotL(x, steps_i)) (R30); scale (S_x pt_scale) / q_l
    // or its baby-step giant-step form (R39) when the stage carries baby / giant steps
    Val lt(const Val &x, const LtStage &st) {
        const int l = x.level();
        const double s = (x.scale() * st.scale) / q(l);
        Val out = fresh(l - 1, s);
        auto join = [](const std::vector<int> &v) {
            std::string r;
            for (size_t i = 0; i < v.size(); i++) r += (i ? "," : "") + std::to_string(v[i]);
            return r;
        };
        if (!st.giant.empty()) {
            ev_linear_transform_bsgs_gen(c, k, x.v, st.pts, (long)(l + 1) * c.N, st.baby.data(), (int)st.baby.size(),
                                         st.giant.data(), (int)st.giant.size(), out.v);
            c.log("LTG", l, l - 1, s, join(st.baby) + ";" + join(st.giant));
        } else {
            ev_linear_transform(c, k, x.v, st.pts, (long)(l + 1) * c.N, st.steps.data(), (int)st.steps.size(),
                                out.v);
            c.log("LT", l, l - 1, s, join(st.steps));
        }
        return out;
    }
    // EvalMod on one CoeffToSlot output u (R35): x = u + conj(u), x / (K R), doubled cosine, r doublings
    Val evalmod(const Val &u, double K, int r, const std::vector<double> &poly, double S0) {
        const double inv = 1.0 / (K * ((double)c.primes[0] / S0));
        Val x = rot_add(u, kConjStep);
        Val xn = mul_const(x, inv, S0, x.level() - 1);  // EvalMod at the input's scale (R38)
        Val d = poly15(xn, poly, S0);
        for (int j = 0; j < r; j++) d = add_const(mul_ct(d, d, NAN, d.level() - 1), -2.0);
        return d;
    }
    // factorised bootstrap (R37): ModRaise; CoeffToSlot stages (the last in Re / Im variants); EvalMod on
    // both; SlotToCoeff's first stage on d_re and d_im, summed; the remaining SlotToCoeff stages
    Val bootstrap_fft(const Val &in, const FftBootCfg &b) {
        const double S0 = in.scale();
        Val v = mod_raise(in, b.level);
        for (size_t i = 0; i + 1 < b.cts.size(); i++) v = lt(v, b.cts[i]);
        Val us[2] = {lt(v, b.cts.back()), lt(v, b.cts_im)};
        Val ds[2] = {evalmod(us[0], b.K, b.r, b.poly, S0), evalmod(us[1], b.K, b.r, b.poly, S0)};
        Val o_re = lt(ds[0], b.stc[0]);
        Val o_im = lt(ds[1], b.stc_im);
        Val o = add(o_re, o_im);
        for (size_t i = 1; i < b.stc.size(); i++) o = lt(o, b.stc[i]);
        return o;
    }
    // general degree-15 p(x) = sum_i c_i x^i at (T, level(x) - 5) (R35): the odd plan's Paterson-Stockmeyer
    // shape with the even terms added, q_k = c_{4k} + c_{4k+1} x + c_{4k+2} x^2 + c_{4k+3} x^3,
    // p = (q_0 + q_1 x^4) + (q_2 + q_3 x^4) x^8
    Val poly15(const Val &x, const std::vector<double> &cf, double T) {
        const int l = x.level(), Lo = l - 5;
        Val x2 = mul_ct(x, x, NAN, l - 1);
        Val x3 = mul_ct(x, x2, NAN, l - 2);
        Val x4 = mul_ct(x2, x2, NAN, l - 2);
        Val x8 = mul_ct(x4, x4, NAN, l - 3);
        const double Sb1 = (T * q(l - 4)) / x8.scale();
        const double Sq3 = (Sb1 * q(l - 3)) / x4.scale();
        Val q3 = lincomb({{&x, cf[13]}, {&x3, cf[15]}}, Sq3, l - 3);
        Val q3e = lincomb({{&x2, cf[14]}}, Sq3, l - 3);
        q3 = add_const(add(q3, q3e), cf[12]);
        Val b1 = mul_ct(q3, x4, Sb1, l - 4, {{&x, cf[9]}, {&x3, cf[11]}});
        Val b1e = lincomb({{&x2, cf[10]}}, Sb1, l - 4);
        b1 = add_const(add(b1, b1e), cf[8]);
        const double Sq1 = (T * q(l - 4)) / x4.scale();
        Val q1 = lincomb({{&x, cf[5]}, {&x3, cf[7]}}, Sq1, l - 4);
        Val q1e = lincomb({{&x2, cf[6]}}, Sq1, l - 4);
        q1 = add_const(add(q1, q1e), cf[4]);
        Val p = mul_ct(q1, x4, T, Lo, {{&x, cf[1]}, {&x3, cf[3]}}, &b1, &x8);
        Val pe = lincomb({{&x2, cf[2]}}, T, Lo);
        return add_const(add(p, pe), cf[0]);
    }
    // ModRaise -> CoeffToSlot (two BSGS transforms) -> x = u + conj(u) -> x / (K R) -> doubled cosine ->
    // r steps d <- d^2 - 2 (natural scales) -> SlotToCoeff (two BSGS transforms, summed)
    Val bootstrap(const Val &in, const BootCfg &b) {
        const double S0 = in.scale();
        Val z = mod_raise(in, b.level);
        Val us[2] = {lt_bsgs(z, b.cts_re, b.n1, b.n2, b.cts_scale), lt_bsgs(z, b.cts_im, b.n1, b.n2, b.cts_scale)};
        Val ds[2] = {evalmod(us[0], b.K, b.r, b.poly, S0), evalmod(us[1], b.K, b.r, b.poly, S0)};
        Val o_re = lt_bsgs(ds[0], b.stc_re, b.n1, b.n2, b.stc_scale);
        Val o_im = lt_bsgs(ds[1], b.stc_im, b.n1, b.n2, b.stc_scale);
        return add(o_re, o_im);
    }

    // ---- composite sign --------------------------------------------------------------------
    Val odd_poly(const Val &x, const std::vector<double> &cf, double T) {
        const int deg = (int)cf.size() - 1;
        const int l = x.level();
        Val x2 = mul_ct(x, x, NAN, l - 1);
        Val x4 = deg >= 7 ? mul_ct(x2, x2, NAN, l - 2) : Val{};
        Val x8 = deg >= 15 ? mul_ct(x4, x4, NAN, l - 3) : Val{};
        auto A = [&](int i, double S, int L) {
            // (c_{4i+3} x) x^2 + c_{4i+1} x: the linear term joins the product before its rescale (R13)
            Val inner = mul_const(x, cf[4 * i + 3], (S * q(L + 1)) / x2.scale(), L + 1);
            return mul_ct(inner, x2, S, L, {{&x, cf[4 * i + 1]}});
        };
        auto B = [&](int i, double S, int L) {
            // x^4 A_{2i+1} + A_{2i}: A_{2i} = (c x) x^2 + c' x is a second product summed with the first,
            // one relinearisation and rescale for both (R13b)
            Val hi = A(2 * i + 1, (S * q(L + 1)) / x4.scale(), L + 1);
            Val inner = mul_const(x, cf[8 * i + 3], (S * q(L + 1)) / x2.scale(), L + 1);
            return mul_ct(hi, x4, S, L, {{&x, cf[8 * i + 1]}}, &inner, &x2);
        };
        if (deg == 3) return A(0, T, l - 2);
        if (deg == 7) return B(0, T, l - 3);
        // degree 15, Paterson-Stockmeyer (R13): x^3 shared, q_k = c_{4k+1} x + c_{4k+3} x^3 linear
        // combinations, p = (q_1 x^4 + q_0) + (q_3 x^4 + q_2) x^8 at depth 5 with 7 ct x ct products
        const int Lo = l - 5;
        Val x3 = mul_ct(x, x2, NAN, l - 2);
        const double Sb1 = (T * q(l - 4)) / x8.scale();
        Val q3 = lincomb({{&x, cf[13]}, {&x3, cf[15]}}, (Sb1 * q(l - 3)) / x4.scale(), l - 3);
        Val b1 = mul_ct(q3, x4, Sb1, l - 4, {{&x, cf[9]}, {&x3, cf[11]}});
        Val q1 = lincomb({{&x, cf[5]}, {&x3, cf[7]}}, (T * q(l - 4)) / x4.scale(), l - 4);
        // q_1 x^4 + q_0 + b_1 x^8: the two products share one relinearisation and rescale (R13b)
        return mul_ct(q1, x4, T, Lo, {{&x, cf[1]}, {&x3, cf[3]}}, &b1, &x8);
    }
    Val sign(Val x, const SignCfg &cfg, double T) {
        for (size_t i = 0; i < cfg.stages.size(); i++) {
            const double s = (i + 1 == cfg.stages.size()) ? T : c.scale;
            x = odd_poly(x, cfg.stages[i], s);
        }
        c.cnt.sign += n;
        return x;
    }
    // Eq. 6: Max(r, y) = (r + y)/2 + (r - y)/2 * Sign(r - y); output scale = scale(y)
    Val hom_max(const Val &r, const Val &y, const SignCfg &cfg) {
        const double Sy = y.scale();
        Val d = sub(r, y);
        Val s = sign(d, cfg, c.scale);
        const int Ls = s.level();
        Val g = mul_const(d, 0.5, (Sy * q(Ls)) / s.scale(), Ls);
        Val ry = add(r, y);
        // (r - y)/2 Sign(r - y) + (r + y)/2: the half-sum joins the product before its rescale
        return mul_ct(g, s, Sy, Ls - 1, {{&ry, 0.5}});
    }
    // N4 (R38): Algorithm 1 with a bootstrap (factorised, R37) before every Max / the final Sign that would
    // not fit: scale-up to level 0 at boot_scale, bootstrap, normalise back to the nominal scale
    Val refresh(const Val &x, const FftBootCfg &b, double boot_scale) {
        Val xs = mul_const(x, 1.0, boot_scale, 0);
        Val r = bootstrap_fft(xs, b);
        return mul_const(r, 1.0, c.scale, r.level() - 1);
    }
    // ins: the prompt groups (prompt_cts ciphertexts per query set, summed first: PAPER.md:141 y* = sum y_i);
    // the mask normalises by prompts x prompt_cts
    Val argmax_boot(const std::vector<Val> &ins, const Layout &lay, const SignCfg &cfg, const FftBootCfg &b,
                    double boot_scale) {
        const int P = lay.prompts, K = lay.classes, pc = (int)ins.size();
        Val y = ins[0];
        for (int i = 1; i < pc; i++) y = add(y, ins[i]);
        for (int t = 0; (1 << t) < P; t++) y = rot_add(y, K << t);
        std::vector<double> mask(c.N / 2, 0.0);
        for (int qi = 0; qi < lay.queries; qi++)
            for (int kk = 0; kk < K; kk++) mask[(size_t)qi * lay.block + kk] = (1.0 / P) / pc;
        y = mul_mask(y, mask, c.scale,
                     "argmax/" + std::to_string(lay.queries) + "/" + std::to_string(P) + "/" + std::to_string(K) + "/" +
                         std::to_string(lay.block) + "/" + std::to_string(pc));
        y = rot_add(y, -K);
        Val ydup = y;
        const int sd = sign_depth(cfg);
        for (int i = 0; (1 << i) < K; i++) {
            if (y.level() < sd + 2) y = refresh(y, b, boot_scale);
            y = hom_max(rot(y, 1 << i), y, cfg);
        }
        Val d = sub(ydup, y);
        if (d.level() < sd) d = refresh(d, b, boot_scale);
        Val z = sign(d, cfg, c.scale);
        return add_const(z, 1.0);
    }
    // Algorithm 1 with the H1..H6 steps of DESIGN.md section 2
    // profiler spans of the circuit stages (kinds 4..8: H1, H2, H3, H4, H6; only when profiling)
    Val argmax(const Val &in, const Layout &lay, const SignCfg &cfg) {
        const int P = lay.prompts, K = lay.classes;
        Val y = in;
        size_t sp = c.prof_begin(4);
        for (int t = 0; (1 << t) < P; t++) y = rot_add(y, K << t);
        c.prof_end(sp, 4, 0, n);
        std::vector<double> mask(c.N / 2, 0.0);
        for (int qi = 0; qi < lay.queries; qi++)
            for (int kk = 0; kk < K; kk++) mask[(size_t)qi * lay.block + kk] = 1.0 / P;
        sp = c.prof_begin(5);
        y = mul_mask(y, mask, c.scale,
                     "argmax/" + std::to_string(lay.queries) + "/" + std::to_string(P) + "/" + std::to_string(K) + "/" +
                         std::to_string(lay.block));
        c.prof_end(sp, 5, 0, n);
        sp = c.prof_begin(6);
        y = rot_add(y, -K);
        c.prof_end(sp, 6, 0, n);
        Val ydup = y;
        sp = c.prof_begin(7);
        for (int i = 0; (1 << i) < K; i++) y = hom_max(rot(y, 1 << i), y, cfg);
        c.prof_end(sp, 7, 0, n);
        sp = c.prof_begin(8);
        Val d = sub(ydup, y);
        Val z = sign(d, cfg, c.scale);
        Val r = add_const(z, 1.0);
        c.prof_end(sp, 8, 0, n);
        return r;
    }
};

static int ilog2(int v) {
    int r = 0;
    while ((1 << r) < v) r++;
    return r;
}
// BSGS depth ceil(log2(d+1)) for degrees 3 and 7; the degree-15 Paterson-Stockmeyer plan uses one more
static int poly_depth(int deg) { return deg == 15 ? 5 : ilog2(deg + 1); }

int sign_depth(const SignCfg &cfg) {
    int d = 0;
    for (auto &s : cfg.stages) d += poly_depth((int)s.size() - 1);
    return d;
}
int argmax_depth(const Layout &lay, const SignCfg &cfg) {
    return 1 + ilog2(lay.classes) * (sign_depth(cfg) + 1) + sign_depth(cfg);
}
std::vector<int> argmax_rotations(const Layout &lay) {
    std::vector<int> r;
    for (int t = 0; (1 << t) < lay.prompts; t++) r.push_back(lay.classes << t);
    r.push_back(-lay.classes);
    for (int i = 0; (1 << i) < lay.classes; i++) r.push_back(1 << i);
    return r;
}

int boot_depth(const BootCfg &b) { return 8 + b.r; }
int fft_boot_depth(const FftBootCfg &b) { return (int)b.cts.size() + (int)b.stc.size() + 6 + b.r; }

// output level of argmax_boot for an input at in_level (the plan's level walk, no arithmetic)
int argmax_boot_level(const Layout &lay, const SignCfg &cfg, const FftBootCfg &b, int in_level) {
    const int sd = sign_depth(cfg), bl = b.level - fft_boot_depth(b) - 1;  // level after refresh
    int y = in_level - 1;                                                   // mask
    if (y < 0) throw SecpeError{-2, "not enough levels for the mask"};
    for (int i = 0; (1 << i) < lay.classes; i++) {
        if (y < sd + 2) {
            if (y < 1) throw SecpeError{-2, "no level left for a refresh"};
            y = bl;
        }
        if (y < sd + 1) throw SecpeError{-2, "a refresh leaves too few levels for a Max"};
        y -= sd + 1;
    }
    int d = std::min(in_level - 1, y);
    if (d < sd) {
        if (d < 1) throw SecpeError{-2, "no level left for a refresh"};
        d = bl;
    }
    if (d < sd) throw SecpeError{-2, "a refresh leaves too few levels for the final Sign"};
    return d - sd;
}

// the whole batch through one plan: every key (and every transform plaintext) is read once per op for all
// in.n ciphertexts
void run_argmax_boot(Ctx &c, const Keys &k, const CtView &in, const Layout &lay, const SignCfg &cfg,
                     const FftBootCfg &b, double boot_scale, int prompt_cts, CtView &out) {
    if (prompt_cts < 1 || in.n % prompt_cts) throw SecpeError{-1, "argmax_boot: n_in must be a multiple of prompt_cts"};
    const int B = in.n / prompt_cts;
    Ev ev{c, k, B};
    std::vector<Val> ins;
    for (int i = 0; i < prompt_cts; i++) {  // member i of every group: ciphertexts i, i + pc, ...
        CtView v = in;
        v.data = in.data + (long)i * in.stride;
        v.stride = in.stride * prompt_cts;
        v.n = B;
        ins.push_back(Val{nullptr, v});
    }
    Val r = ev.argmax_boot(ins, lay, cfg, b, boot_scale);
    out.level = r.level();
    out.scale = r.scale();
    ev_copy(c, r.v, out);
}

void run_bootstrap_fft(Ctx &c, const Keys &k, const CtView &in, const FftBootCfg &b, CtView &out) {
    Ev ev{c, k, in.n};
    Val x{nullptr, in};
    Val r = ev.bootstrap_fft(x, b);
    out.level = r.level();
    out.scale = r.scale();
    ev_copy(c, r.v, out);
}

void run_bootstrap(Ctx &c, const Keys &k, const CtView &in, const BootCfg &b, CtView &out) {
    Ev ev{c, k, in.n};
    Val x{nullptr, in};
    Val r = ev.bootstrap(x, b);
    out.level = r.level();
    out.scale = r.scale();
    ev_copy(c, r.v, out);
}

static void copy_in(Ctx &c, const CtView &src, const Val &dst) { ev_copy(c, src, dst.v); }

void run_sign(Ctx &c, const Keys &k, const CtView &in, const SignCfg &cfg, double target_scale, CtView &out) {
    Ev ev{c, k, in.n};
    Val x{nullptr, in};
    Val r = ev.sign(x, cfg, target_scale);
    out.level = r.level();
    out.scale = r.scale();
    ev_copy(c, r.v, out);
}

// The batch runs as up to c.n_streams concurrent sub-batches, each planned on its own stream (forked
// from and joined back into the context stream): ciphertexts are independent, and kernels of one
// sub-batch (e.g. integer-pipe NTTs or tensor-core conversions) overlap those of another (FP64 NTTs).
// The planned op list of every sub-batch is the same; the op log is recorded with a single stream.
void run_argmax(Ctx &c, const Keys &k, const CtView &in, const Layout &lay, const SignCfg &cfg, CtView &out) {
    // (one stream while the op log or the CUDA-event profiler is on: the profiled spans must not overlap)
    const int S = (c.log_on || c.prof.on || in.n < 2) ? 1 : std::min(c.n_streams, in.n);
    if (S == 1) {
        Ev ev{c, k, in.n};
        Val x{nullptr, in};
        Val r = ev.argmax(x, lay, cfg);
        out.level = r.level();
        out.scale = r.scale();
        ev_copy(c, r.v, out);
        return;
    }
    while ((int)c.aux.size() < S) {
        cudaStream_t s;
        CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        c.aux.push_back(s);
    }
    cudaStream_t main = c.st;
    cudaEvent_t fork;
    CUDA_CHECK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventRecord(fork, main));
    std::vector<cudaEvent_t> done(S);
    try {
        for (int s = 0; s < S; s++) {
            const int b = (int)((long)in.n * s / S), e = (int)((long)in.n * (s + 1) / S);
            CUDA_CHECK(cudaStreamWaitEvent(c.aux[s], fork, 0));
            c.st = c.aux[s];
            {
                CtView vin = in, vout = out;
                vin.data += (long)b * in.stride;
                vin.n = e - b;
                vout.data += (long)b * out.stride;
                vout.n = e - b;
                Ev ev{c, k, vin.n};
                Val x{nullptr, vin};
                Val r = ev.argmax(x, lay, cfg);
                out.level = r.level();
                out.scale = r.scale();
                vout.level = r.level();
                ev_copy(c, r.v, vout);
            }  // temporaries are freed on their own stream here
            CUDA_CHECK(cudaEventCreateWithFlags(&done[s], cudaEventDisableTiming));
            CUDA_CHECK(cudaEventRecord(done[s], c.st));
            c.st = main;
        }
    } catch (...) {
        c.st = main;
        throw;
    }
    for (int s = 0; s < S; s++) {
        CUDA_CHECK(cudaStreamWaitEvent(main, done[s], 0));
        cudaEventDestroy(done[s]);
    }
    cudaEventDestroy(fork);
    (void)copy_in;
}
