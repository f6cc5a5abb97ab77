"""Thin ctypes binding of libsecpe.so (include/secpe.h).  Argument marshalling only: every
homomorphic step runs in the library's sm_100a kernels.  PyTorch provides device memory and the
stream.  There is no fallback: without the built library or a CUDA device, calls raise.
"""
import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsecpe.so")

u64p = ctypes.POINTER(ctypes.c_uint64)
i64p = ctypes.POINTER(ctypes.c_int64)
i32p = ctypes.POINTER(ctypes.c_int32)
f64p = ctypes.POINTER(ctypes.c_double)
vp = ctypes.c_void_p


class Params(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("n_q", ctypes.c_uint32), ("q", u64p), ("n_p", ctypes.c_uint32),
                ("p", u64p), ("alpha", ctypes.c_uint32), ("scale", ctypes.c_double)]


class CCt(ctypes.Structure):
    _fields_ = [("data", u64p), ("level", ctypes.c_int32), ("scale", ctypes.c_double)]


class SignCfg(ctypes.Structure):
    _fields_ = [("n_stages", ctypes.c_int32), ("degrees", i32p), ("coeffs", f64p)]


class CLtStage(ctypes.Structure):
    _fields_ = [("n_diag", ctypes.c_int32), ("steps", i32p), ("pts", u64p), ("pt_scale", ctypes.c_double),
                ("n_baby", ctypes.c_int32), ("baby", i32p), ("n_giant", ctypes.c_int32), ("giant", i32p)]


class CBootFftCfg(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("K", ctypes.c_double), ("r", ctypes.c_int32), ("poly", f64p),
                ("n_cts", ctypes.c_int32), ("cts", ctypes.POINTER(CLtStage)), ("cts_im", CLtStage),
                ("n_stc", ctypes.c_int32), ("stc", ctypes.POINTER(CLtStage)), ("stc_im", CLtStage)]


class CBootCfg(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("n1", ctypes.c_int32), ("n2", ctypes.c_int32), ("K", ctypes.c_double),
                ("r", ctypes.c_int32), ("poly", f64p), ("cts_re", u64p), ("cts_im", u64p), ("cts_scale", ctypes.c_double),
                ("stc_re", u64p), ("stc_im", u64p), ("stc_scale", ctypes.c_double)]


CONJ = -(2 ** 31)  # SECPE_CONJ: the rotation step meaning slot conjugation


class CSeed(ctypes.Structure):
    """secpe_seed: 256-bit master seed (reading R6)."""
    _fields_ = [("bytes", ctypes.c_uint8 * 32)]


def seed_arg(seed):
    """None -> NULL (the library draws 32 bytes of OS entropy: production mode); 32 bytes -> that seed; an
    integer -> secpe_seed_from_u64 (TEST-ONLY deterministic mode, what the parity tests and the bench use)."""
    if seed is None:
        return None
    s = CSeed()
    if isinstance(seed, (bytes, bytearray)):
        if len(seed) != 32:
            raise ValueError("a seed is 32 bytes")
        ctypes.memmove(s.bytes, bytes(seed), 32)
    else:
        lib().secpe_seed_from_u64(int(seed), ctypes.byref(s))
    return ctypes.byref(s)


class Layout(ctypes.Structure):
    _fields_ = [("queries", ctypes.c_int32), ("prompts", ctypes.c_int32), ("classes", ctypes.c_int32),
                ("block", ctypes.c_int32)]


_lib = None

SIGS = {
    "secpe_last_error": (ctypes.c_char_p, []),
    "secpe_version": (ctypes.c_char_p, []),
    "secpe_gen_primes": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int32, u64p,
                                        ctypes.c_uint32, u64p]),
    "secpe_ctx_create": (ctypes.c_int, [ctypes.POINTER(Params), vp, ctypes.POINTER(vp)]),
    "secpe_ctx_destroy": (None, [vp]),
    "secpe_set_stream": (ctypes.c_int, [vp, vp]),
    "secpe_sync": (ctypes.c_int, [vp]),
    "secpe_ctx_info": (ctypes.c_int, [vp, u64p, u64p]),
    "secpe_ct_bytes": (ctypes.c_size_t, [vp, ctypes.c_int32]),
    "secpe_seed_from_u64": (None, [ctypes.c_uint64, ctypes.POINTER(CSeed)]),
    "secpe_keygen": (ctypes.c_int, [vp, ctypes.POINTER(CSeed), i32p, ctypes.c_int32, ctypes.POINTER(vp)]),
    "secpe_keygen_sparse": (ctypes.c_int, [vp, ctypes.POINTER(CSeed), ctypes.c_int32, i32p, ctypes.c_int32,
                                           ctypes.POINTER(vp)]),
    "secpe_keys_destroy": (None, [vp]),
    "secpe_key_export": (ctypes.c_int, [vp, vp, ctypes.c_int32, ctypes.c_uint64, u64p, ctypes.c_size_t]),
    "secpe_encode": (ctypes.c_int, [vp, f64p, ctypes.c_size_t, ctypes.c_double, i64p]),
    "secpe_encrypt_coeffs": (ctypes.c_int, [vp, vp, i64p, ctypes.c_int32, ctypes.c_double, ctypes.POINTER(CSeed),
                                            ctypes.POINTER(CCt)]),
    "secpe_encrypt": (ctypes.c_int, [vp, vp, f64p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_double,
                                     ctypes.POINTER(CSeed), ctypes.POINTER(CCt)]),
    "secpe_decrypt_residues": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), u64p]),
    "secpe_decrypt": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), f64p, ctypes.c_size_t]),
    "secpe_ntt": (ctypes.c_int, [vp, u64p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "secpe_intt": (ctypes.c_int, [vp, u64p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "secpe_add": (ctypes.c_int, [vp, ctypes.POINTER(CCt), ctypes.POINTER(CCt), ctypes.POINTER(CCt)]),
    "secpe_sub": (ctypes.c_int, [vp, ctypes.POINTER(CCt), ctypes.POINTER(CCt), ctypes.POINTER(CCt)]),
    "secpe_add_const": (ctypes.c_int, [vp, ctypes.POINTER(CCt), ctypes.c_double, ctypes.POINTER(CCt)]),
    "secpe_mul_const": (ctypes.c_int, [vp, ctypes.POINTER(CCt), ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                       ctypes.POINTER(CCt)]),
    "secpe_mul_mask": (ctypes.c_int, [vp, ctypes.POINTER(CCt), f64p, ctypes.c_size_t, ctypes.c_double,
                                      ctypes.POINTER(CCt)]),
    "secpe_drop": (ctypes.c_int, [vp, ctypes.POINTER(CCt), ctypes.c_int32, ctypes.POINTER(CCt)]),
    "secpe_mul_relin": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.POINTER(CCt), ctypes.POINTER(CCt)]),
    "secpe_mul_relin_rescale": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.POINTER(CCt), ctypes.c_int32,
                                               ctypes.POINTER(CCt)]),
    "secpe_rotate_batch": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.c_int32, ctypes.c_int32,
                                          ctypes.POINTER(CCt)]),
    "secpe_rotate_hoisted": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.c_int32, i32p, ctypes.c_int32,
                                            ctypes.POINTER(CCt)]),
    "secpe_linear_transform": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), u64p, i32p, ctypes.c_int32,
                                              ctypes.c_double, ctypes.POINTER(CCt)]),
    "secpe_mod_raise": (ctypes.c_int, [vp, ctypes.POINTER(CCt), ctypes.c_int32, ctypes.POINTER(CCt)]),
    "secpe_boot_depth": (ctypes.c_int32, [ctypes.POINTER(CBootCfg)]),
    "secpe_boot_create": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_double, ctypes.POINTER(vp)]),
    "secpe_boot_get_cfg": (ctypes.c_int, [vp, ctypes.POINTER(CBootCfg)]),
    "secpe_boot_destroy": (None, [vp]),
    "secpe_boot_export": (ctypes.c_int, [vp, vp, ctypes.c_int32, u64p, ctypes.c_size_t]),
    "secpe_bootstrap_fft": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.POINTER(CBootFftCfg),
                                           ctypes.POINTER(CCt)]),
    "secpe_boot_create_fft": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, i32p,
                                             ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(vp)]),
    "secpe_boot_stage_export_bsgs": (ctypes.c_int, [vp, vp, ctypes.c_int32, ctypes.c_int32, i32p, i32p, i32p, i32p,
                                                    u64p, ctypes.c_size_t]),
    "secpe_bootstrap_boot": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), vp, ctypes.POINTER(CCt)]),
    "secpe_boot_levels": (ctypes.c_int32, [vp, i32p]),
    "secpe_boot_steps": (ctypes.c_int32, [vp, i32p, ctypes.c_int32]),
    "secpe_bootstrap_boot_batch": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.c_int32, vp,
                                                  ctypes.POINTER(CCt)]),
    "secpe_argmax_boot_info": (ctypes.c_int, [vp, ctypes.POINTER(Layout), ctypes.POINTER(SignCfg), vp,
                                              ctypes.c_int32, i32p]),
    "secpe_enc_argmax_boot": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.c_int32, ctypes.c_int32,
                                             ctypes.POINTER(Layout), ctypes.POINTER(SignCfg), vp, ctypes.c_double,
                                             ctypes.POINTER(CCt)]),
    "secpe_enc_argmax_boot_cfg": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.POINTER(Layout), ctypes.POINTER(SignCfg),
                                                 ctypes.POINTER(CBootFftCfg), ctypes.c_double, ctypes.POINTER(CCt)]),
    "secpe_boot_stage_export": (ctypes.c_int, [vp, vp, ctypes.c_int32, ctypes.c_int32, i32p, i32p, u64p,
                                               ctypes.c_size_t]),
    "secpe_bootstrap": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.POINTER(CBootCfg), ctypes.POINTER(CCt)]),
    "secpe_linear_transform_bsgs": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), u64p, ctypes.c_int32, ctypes.c_int32,
                                                   ctypes.c_double, ctypes.POINTER(CCt)]),
    "secpe_rescale": (ctypes.c_int, [vp, ctypes.POINTER(CCt), ctypes.POINTER(CCt)]),
    "secpe_rotate": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.c_int32, ctypes.POINTER(CCt)]),
    "secpe_sign_poly": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.POINTER(SignCfg), ctypes.c_double,
                                       ctypes.POINTER(CCt)]),
    "secpe_sign_depth": (ctypes.c_int32, [ctypes.POINTER(SignCfg)]),
    "secpe_argmax_info": (ctypes.c_int, [vp, ctypes.POINTER(Layout), ctypes.POINTER(SignCfg), ctypes.c_int32,
                                         i32p, f64p]),
    "secpe_enc_argmax": (ctypes.c_int, [vp, vp, ctypes.POINTER(CCt), ctypes.c_int32, ctypes.POINTER(Layout),
                                        ctypes.POINTER(SignCfg), ctypes.POINTER(CCt)]),
    "secpe_enc_argmax_host": (ctypes.c_int, [vp, vp, u64p, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                             ctypes.POINTER(Layout), ctypes.POINTER(SignCfg), u64p, ctypes.c_int32,
                                             i32p, f64p]),
    "secpe_oplog_enable": (ctypes.c_int, [vp, ctypes.c_int32]),
    "secpe_oplog_get": (ctypes.c_int64, [vp, ctypes.c_char_p, ctypes.c_size_t]),
    "secpe_oplog_clear": (ctypes.c_int, [vp]),
    "secpe_opcounts": (ctypes.c_int, [vp, i64p, ctypes.c_int32]),
    "secpe_ntt_mode": (ctypes.c_int32, [ctypes.c_int32]),
    "secpe_profile_begin": (ctypes.c_int, [vp]),
    "secpe_profile_end": (ctypes.c_int, [vp, f64p, ctypes.c_int32]),
}
EXPORTS = list(SIGS)


def lib():
    """Load libsecpe.so (built in-tree by paper_2502_00847_b200.build); raise if it is missing."""
    global _lib
    if _lib is None:
        path = os.environ.get("SECPE_LIB", LIB_PATH)  # development: alternative in-tree build variant
        if not os.path.exists(path):
            raise RuntimeError("libsecpe.so not built: run `python -m paper_2502_00847_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SecpeError(RuntimeError):
    pass


def ntt_mode(mode=-1):
    """secpe_ntt_mode: development switch of the N = 2^16 FP64-row NTT (0 two-pass, 1 fused, 2 auto)."""
    return lib().secpe_ntt_mode(mode)


def _chk(code):
    if code != 0:
        raise SecpeError("secpe error %d: %s" % (code, lib().secpe_last_error().decode()))


def _u64(a):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    return a, a.ctypes.data_as(u64p)


def gen_primes(bits, count, logn, mode, exclude=()):
    ex, exp_ = _u64(np.array(list(exclude) or [0], dtype=np.uint64))
    out = np.zeros(count, dtype=np.uint64)
    _chk(lib().secpe_gen_primes(bits, count, logn, 0 if mode == "nearest" else 1, exp_, len(exclude),
                                out.ctypes.data_as(u64p)))
    return [int(v) for v in out]


def primes_for(desc):
    """Prime chain of a parameter description (synth.PARAM_SETS entry), generated by the library."""
    q = []
    for mode, bits, cnt in desc["q"]:
        q += gen_primes(bits, cnt, desc["logn"], mode, q)
    p = []
    for mode, bits, cnt in desc["p"]:
        p += gen_primes(bits, cnt, desc["logn"], mode, q + p)
    return q, p


class Ct:
    """A ciphertext (or a batch): torch uint64 tensor [n, 2, level+1, N] on the GPU + level + scale."""

    def __init__(self, t, level, scale):
        self.t, self.level, self.scale = t, level, scale

    def c(self, i=0):
        return CCt(ctypes.cast(self.t[i].data_ptr(), u64p), self.level, self.scale)

    @property
    def n(self):
        return self.t.shape[0]


def sign_cfg(stages):
    deg = np.array([len(c) - 1 for c in stages], dtype=np.int32)
    co = np.ascontiguousarray(np.concatenate([np.asarray(c, dtype=np.float64) for c in stages]))
    cfg = SignCfg(len(stages), deg.ctypes.data_as(i32p), co.ctypes.data_as(f64p))
    cfg._keep = (deg, co)
    return cfg


def layout(d):
    return Layout(d["queries"], d["prompts"], d["classes"], d["block"])


class Keys:
    def __init__(self, ctx, handle):
        self.ctx, self.h = ctx, handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.secpe_keys_destroy(self.h)
            self.h = None

    def export(self, which, galois=0):
        cx = self.ctx
        N, P = cx.N, cx.nq + cx.np_
        beta = (cx.nq + cx.alpha - 1) // cx.alpha
        shape = {0: (P, N), 1: (2, cx.nq, N), 2: (beta, 2, P, N), 3: (beta, 2, P, N)}[which]
        out = np.zeros(shape, dtype=np.uint64)
        _chk(lib().secpe_key_export(cx.h, self.h, which, galois, out.ctypes.data_as(u64p), out.size))
        return out


class Boot:
    """secpe_boot handle: library-built bootstrapping material (device memory owned by the library)."""

    def __init__(self, ctx, handle, fft):
        self.ctx, self.h, self.fft = ctx, handle, fft

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.secpe_boot_destroy(self.h)
            self.h = None

    def export(self, which):
        """Matrix `which` (0 cts_re, 1 cts_im, 2 stc_re, 3 stc_im) as host uint64[n2][n1][limbs][N]."""
        c = self.cfg()
        lv = c["level"] if which < 2 else c["level"] - 7 - c["r"]
        out = np.zeros((c["n2"], c["n1"], lv + 1, self.ctx.N), dtype=np.uint64)
        _chk(lib().secpe_boot_export(self.ctx.h, self.h, which, out.ctypes.data_as(u64p), out.size))
        return out

    def steps(self):
        """Rotation steps whose keys this bootstrap needs (secpe_boot_steps; SECPE_CONJ last)."""
        n = lib().secpe_boot_steps(self.h, None, 0)
        out = np.zeros(max(n, 1), dtype=np.int32)
        lib().secpe_boot_steps(self.h, out.ctypes.data_as(i32p), n)
        return out[:n].tolist()

    def stage_bsgs(self, kind, idx, level):
        """Baby-step giant-step stage: (baby, giant, host pts [n_giant][n_baby][level+1][N])."""
        nb, ng = ctypes.c_int32(0), ctypes.c_int32(0)
        _chk(lib().secpe_boot_stage_export_bsgs(self.ctx.h, self.h, kind, idx, ctypes.byref(nb), ctypes.byref(ng),
                                                None, None, None, 0))
        b_ = np.zeros(nb.value, dtype=np.int32)
        g_ = np.zeros(ng.value, dtype=np.int32)
        pts = np.zeros((ng.value, nb.value, level + 1, self.ctx.N), dtype=np.uint64)
        _chk(lib().secpe_boot_stage_export_bsgs(self.ctx.h, self.h, kind, idx, ctypes.byref(nb), ctypes.byref(ng),
                                                b_.ctypes.data_as(i32p), g_.ctypes.data_as(i32p),
                                                pts.ctypes.data_as(u64p), pts.size))
        return b_.tolist(), g_.tolist(), pts

    def stage(self, kind, idx=0, level=None):
        """Factorised stage (kind 0 cts[idx], 1 cts_im, 2 stc[idx], 3 stc_im): (steps, host pts or None)."""
        nd = ctypes.c_int32(0)
        _chk(lib().secpe_boot_stage_export(self.ctx.h, self.h, kind, idx, ctypes.byref(nd), None, None, 0))
        steps = np.zeros(nd.value, dtype=np.int32)
        if level is None:
            _chk(lib().secpe_boot_stage_export(self.ctx.h, self.h, kind, idx, ctypes.byref(nd),
                                               steps.ctypes.data_as(i32p), None, 0))
            return steps.tolist(), None
        pts = np.zeros((nd.value, level + 1, self.ctx.N), dtype=np.uint64)
        _chk(lib().secpe_boot_stage_export(self.ctx.h, self.h, kind, idx, ctypes.byref(nd),
                                           steps.ctypes.data_as(i32p), pts.ctypes.data_as(u64p), pts.size))
        return steps.tolist(), pts

    def cfg(self):
        """(level, n1, n2, K, r, poly[16], cts_scale, stc_scale) of the configuration."""
        c = CBootCfg()
        _chk(lib().secpe_boot_get_cfg(self.h, ctypes.byref(c)))
        return dict(level=c.level, n1=c.n1, n2=c.n2, K=c.K, r=c.r, poly=[c.poly[i] for i in range(16)],
                    cts_scale=c.cts_scale, stc_scale=c.stc_scale, raw=c)


class Context:
    """Parameters + device tables on the current torch CUDA stream."""

    def __init__(self, desc=None, q=None, p=None, logn=None, alpha=None, scale=None, stream=None):
        if desc is not None:
            q, p = primes_for(desc)
            logn, alpha, scale = desc["logn"], desc["alpha"], float(2 ** desc["log_scale"])
        self.q, self.p = list(q), list(p)
        self.logn, self.N = logn, 1 << logn
        self.nq, self.np_, self.alpha, self.scale = len(q), len(p), alpha, scale
        self._qa, qp = _u64(q)
        self._pa, pp = _u64(p if p else [0])
        prm = Params(logn, len(q), qp, len(p), pp, alpha, scale)
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        h = vp()
        _chk(lib().secpe_ctx_create(ctypes.byref(prm), vp(stream), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.secpe_ctx_destroy(self.h)
            self.h = None

    @property
    def L(self):
        return self.nq - 1

    def info(self):
        P = self.nq + self.np_
        pr, ps = np.zeros(P, dtype=np.uint64), np.zeros(P, dtype=np.uint64)
        _chk(lib().secpe_ctx_info(self.h, pr.ctypes.data_as(u64p), ps.ctypes.data_as(u64p)))
        return [int(v) for v in pr], [int(v) for v in ps]

    def set_stream(self, stream):
        _chk(lib().secpe_set_stream(self.h, vp(stream)))

    def sync(self):
        _chk(lib().secpe_sync(self.h))

    # ---- memory -------------------------------------------------------------------------------
    def alloc(self, level, n=1):
        return torch.empty((n, 2, level + 1, self.N), dtype=torch.uint64, device="cuda")

    def new_ct(self, level, n=1):
        return Ct(self.alloc(level, n), level, 0.0)

    # ---- keys / client ----------------------------------------------------------------------------
    def keygen(self, seed, rot_steps=(), h=0):
        """secpe_keygen (h = 0) / secpe_keygen_sparse (Hamming weight h, reading R36)."""
        r = np.array(list(rot_steps) or [0], dtype=np.int32)
        kh = vp()
        _chk(lib().secpe_keygen_sparse(self.h, seed_arg(seed), h, r.ctypes.data_as(i32p), len(rot_steps),
                                       ctypes.byref(kh)))
        return Keys(self, kh)

    def encode(self, slots, scale):
        z = np.ascontiguousarray(slots, dtype=np.float64)
        out = np.zeros(self.N, dtype=np.int64)
        _chk(lib().secpe_encode(self.h, z.ctypes.data_as(f64p), len(z), scale, out.ctypes.data_as(i64p)))
        return out

    def encrypt_coeffs(self, keys, coeffs, level, scale, seed, out=None):
        m = np.ascontiguousarray(coeffs, dtype=np.int64)
        ct = out if out is not None else self.new_ct(level)
        cc = CCt(ctypes.cast(ct.t.data_ptr(), u64p), level, scale)
        _chk(lib().secpe_encrypt_coeffs(self.h, keys.h, m.ctypes.data_as(i64p), level, scale, seed_arg(seed),
                                        ctypes.byref(cc)))
        ct.level, ct.scale = level, scale
        return ct

    def encrypt(self, keys, slots, level, scale, seed):
        z = np.ascontiguousarray(slots, dtype=np.float64)
        ct = self.new_ct(level)
        cc = ct.c()
        _chk(lib().secpe_encrypt(self.h, keys.h, z.ctypes.data_as(f64p), len(z), level, scale, seed_arg(seed),
                                 ctypes.byref(cc)))
        ct.level, ct.scale = level, scale
        return ct

    def decrypt_residues(self, keys, ct, i=0):
        out = np.zeros((ct.level + 1, self.N), dtype=np.uint64)
        cc = ct.c(i)
        _chk(lib().secpe_decrypt_residues(self.h, keys.h, ctypes.byref(cc), out.ctypes.data_as(u64p)))
        return out

    def decrypt(self, keys, ct, i=0, n=None):
        n = self.N // 2 if n is None else n
        out = np.zeros(n, dtype=np.float64)
        cc = ct.c(i)
        _chk(lib().secpe_decrypt(self.h, keys.h, ctypes.byref(cc), out.ctypes.data_as(f64p), n))
        return out

    # ---- primitives -------------------------------------------------------------------------------
    def ntt(self, polys, first_prime, n_limbs, inverse=False):
        """In-place (I)NTT of a torch uint64 tensor [..., n_limbs, N] (contiguous)."""
        assert polys.is_contiguous() and polys.dtype == torch.uint64
        n_polys = polys.numel() // (n_limbs * self.N)
        f = lib().secpe_intt if inverse else lib().secpe_ntt
        _chk(f(self.h, ctypes.cast(polys.data_ptr(), u64p), n_polys, first_prime, n_limbs))
        return polys

    def _out(self, level):
        return self.new_ct(level)

    def _binary(self, fn, a, b):
        out = self._out(min(a.level, b.level))
        ca, cb, co = a.c(), b.c(), out.c()
        _chk(fn(self.h, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def add(self, a, b):
        return self._binary(lib().secpe_add, a, b)

    def sub(self, a, b):
        return self._binary(lib().secpe_sub, a, b)

    def add_const(self, a, c):
        out = self._out(a.level)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_add_const(self.h, ctypes.byref(ca), c, ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def mul_const(self, a, c, target_scale, target_level):
        out = self._out(target_level)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_mul_const(self.h, ctypes.byref(ca), c, target_scale, target_level, ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def mul_mask(self, a, mask, target_scale):
        m = np.ascontiguousarray(mask, dtype=np.float64)
        out = self._out(a.level - 1)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_mul_mask(self.h, ctypes.byref(ca), m.ctypes.data_as(f64p), len(m), target_scale,
                                  ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def drop(self, a, level):
        out = self._out(level)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_drop(self.h, ctypes.byref(ca), level, ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def mul_relin(self, keys, a, b):
        out = self._out(a.level)
        ca, cb, co = a.c(), b.c(), out.c()
        _chk(lib().secpe_mul_relin(self.h, keys.h, ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def _batch(self, ct):
        return (CCt * ct.n)(*[ct.c(i) for i in range(ct.n)])

    def mul_relin_rescale(self, keys, a, b, out=None):
        """Batched a (x) b relinearised and rescaled in one pass (bit-identical to mul_relin + rescale); a, b batch Cts."""
        if out is None:
            out = self.new_ct(a.level - 1, a.n)
        ca, cb = self._batch(a), self._batch(b)
        co = (CCt * a.n)(*[CCt(ctypes.cast(out.t[i].data_ptr(), u64p), a.level - 1, 0.0) for i in range(a.n)])
        _chk(lib().secpe_mul_relin_rescale(self.h, keys.h, ca, cb, a.n, co))
        out.level, out.scale = co[0].level, co[0].scale
        return out

    def rotate_batch(self, keys, a, steps, out=None):
        if out is None:
            out = self.new_ct(a.level, a.n)
        ca = self._batch(a)
        co = (CCt * a.n)(*[CCt(ctypes.cast(out.t[i].data_ptr(), u64p), a.level, 0.0) for i in range(a.n)])
        _chk(lib().secpe_rotate_batch(self.h, keys.h, ca, a.n, steps, co))
        out.level, out.scale = co[0].level, co[0].scale
        return out

    def rotate_hoisted(self, keys, a, steps, level=None):
        """secpe_rotate_hoisted: every ciphertext of batch `a` rotated by each step with one shared ModUp
        (N2, reading R29).  Returns one output batch per step."""
        lv = a.level if level is None else level
        outs = [self.new_ct(lv, a.n) for _ in steps]
        ca = self._batch(a)
        co = (CCt * (a.n * len(steps)))(*[CCt(ctypes.cast(o.t[i].data_ptr(), u64p), lv, 0.0)
                                         for o in outs for i in range(a.n)])
        st = np.asarray(steps, dtype=np.int32)
        _chk(lib().secpe_rotate_hoisted(self.h, keys.h, ca, a.n, st.ctypes.data_as(i32p), len(steps), co))
        for s, o in enumerate(outs):
            o.level, o.scale = co[s * a.n].level, co[s * a.n].scale
        return outs

    def linear_transform(self, keys, a, pts, steps, pt_scale):
        """secpe_linear_transform (reading R30): Rescale(sum_i pts[i] (.) RotL(a, steps[i])); pts a cuda
        uint64 tensor [n][a.level+1][N] of NTT-form plaintext residues."""
        assert pts.is_cuda and pts.dtype == torch.uint64 and pts.is_contiguous()
        assert pts.shape[0] == len(steps) and pts.shape[1] == a.level + 1
        out = self._out(a.level - 1)
        ca, co = a.c(), out.c()
        st = np.asarray(steps, dtype=np.int32)
        _chk(lib().secpe_linear_transform(self.h, keys.h, ctypes.byref(ca), ctypes.cast(pts.data_ptr(), u64p),
                                          st.ctypes.data_as(i32p), len(steps), pt_scale, ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def mod_raise(self, a, level):
        """secpe_mod_raise (reading R33)."""
        out = self._out(level)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_mod_raise(self.h, ctypes.byref(ca), level, ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def boot_create(self, level, K, r, n1, n2, in_scale):
        """secpe_boot_create: library-built bootstrapping material (readings R34, R35)."""
        h = vp()
        _chk(lib().secpe_boot_create(self.h, level, K, r, n1, n2, in_scale, ctypes.byref(h)))
        return Boot(self, h, fft=False)

    def boot_create_fft(self, level, K, r, groups, in_scale, bsgs=False):
        """secpe_boot_create_fft: library-built factorised material (reading R37; bsgs: R39 form)."""
        g = np.ascontiguousarray(groups, dtype=np.int32)
        h = vp()
        _chk(lib().secpe_boot_create_fft(self.h, level, K, r, g.ctypes.data_as(i32p), len(g), in_scale,
                                         1 if bsgs else 0, ctypes.byref(h)))
        return Boot(self, h, fft=True)

    def bootstrap_boot(self, keys, a, boot, out=None):
        """secpe_bootstrap_boot: bootstrap with library-built material of either kind (a CUDA graph is captured
        and replayed on a non-default stream when the same buffers come back)."""
        rl = ctypes.c_int32(0)
        depth = lib().secpe_boot_levels(boot.h, ctypes.byref(rl))
        if a.n > 1 and not boot.fft:  # dense material (secpe_boot_create): one ciphertext per call
            ol = max(rl.value - depth, 0)
            if out is None:
                out = self.new_ct(ol, a.n)
            for i in range(a.n):
                ca, co = a.c(i), CCt(ctypes.cast(out.t[i].data_ptr(), u64p), ol, 0.0)
                _chk(lib().secpe_bootstrap_boot(self.h, keys.h, ctypes.byref(ca), boot.h, ctypes.byref(co)))
            out.level, out.scale = co.level, co.scale
            return out
        if a.n > 1:  # secpe_bootstrap_boot_batch (factorised material): one plan for the batch
            ol = max(rl.value - depth, 0)
            if out is None:
                out = self.new_ct(ol, a.n)
            ins = (CCt * a.n)(*[a.c(i) for i in range(a.n)])
            outs = (CCt * a.n)(*[CCt(ctypes.cast(out.t[i].data_ptr(), u64p), ol, 0.0) for i in range(a.n)])
            _chk(lib().secpe_bootstrap_boot_batch(self.h, keys.h, ins, a.n, boot.h, outs))
            out.level, out.scale = outs[0].level, outs[0].scale
            return out
        if out is None:
            out = self._out(max(rl.value - depth, 0))
        ca, co = a.c(), out.c()
        _chk(lib().secpe_bootstrap_boot(self.h, keys.h, ctypes.byref(ca), boot.h, ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    @staticmethod
    def _fft_cfg(level, K, r, poly, cts, cts_im, stc, stc_im):
        """secpe_boot_fft_cfg from (steps, pts, pt_scale) stages; returns (cfg, keep-alive list)."""
        keep = []

        def stage(t):
            if len(t) == 4:  # (baby, giant, pts [n_giant][n_baby][limbs][N], scale): R39 form
                baby, giant, pts, sc = t
                assert pts.is_cuda and pts.dtype == torch.uint64 and pts.is_contiguous()
                assert tuple(pts.shape[:2]) == (len(giant), len(baby))
                b_ = np.ascontiguousarray(baby, dtype=np.int32)
                g_ = np.ascontiguousarray(giant, dtype=np.int32)
                keep.extend([b_, g_])
                return CLtStage(0, None, ctypes.cast(pts.data_ptr(), u64p), sc, len(baby), b_.ctypes.data_as(i32p),
                                len(giant), g_.ctypes.data_as(i32p))
            steps, pts, sc = t
            assert pts.is_cuda and pts.dtype == torch.uint64 and pts.is_contiguous() and pts.shape[0] == len(steps)
            st = np.ascontiguousarray(steps, dtype=np.int32)
            keep.append(st)
            return CLtStage(len(steps), st.ctypes.data_as(i32p), ctypes.cast(pts.data_ptr(), u64p), sc, 0, None, 0,
                            None)
        pc = np.ascontiguousarray(poly, dtype=np.float64)
        assert pc.shape == (16,)
        ca_ = (CLtStage * len(cts))(*[stage(t) for t in cts])
        cs_ = (CLtStage * len(stc))(*[stage(t) for t in stc])
        keep += [pc, ca_, cs_]
        cfg = CBootFftCfg(level, K, r, pc.ctypes.data_as(f64p), len(cts), ca_, stage(cts_im), len(stc), cs_,
                          stage(stc_im))
        return cfg, keep

    def enc_argmax_boot(self, keys, cts, lay, stages, boot, boot_scale, fft_cfg=None, prompt_cts=1):
        """secpe_enc_argmax_boot (N4, reading R38) with library-built material `boot`, or
        secpe_enc_argmax_boot_cfg when fft_cfg = (level, K, r, poly, cts, cts_im, stc, stc_im) is given.
        prompt_cts: consecutive groups of that many ciphertexts are one query set's prompt groups."""
        scfg, ly = sign_cfg(stages), layout(lay)
        assert cts.n % prompt_cts == 0
        n_out = cts.n // prompt_cts
        ol = ctypes.c_int32(0)
        if fft_cfg is None:
            _chk(lib().secpe_argmax_boot_info(self.h, ctypes.byref(ly), ctypes.byref(scfg), boot.h, cts.level,
                                              ctypes.byref(ol)))
        else:
            ol.value = 0
        out = self.new_ct(max(ol.value, 0) if fft_cfg is None else cts.level, n_out)
        ins = (CCt * cts.n)(*[cts.c(i) for i in range(cts.n)])
        outs = (CCt * n_out)(*[CCt(ctypes.cast(out.t[i].data_ptr(), u64p), 0, 0.0) for i in range(n_out)])
        if fft_cfg is None:
            _chk(lib().secpe_enc_argmax_boot(self.h, keys.h, ins, cts.n, prompt_cts, ctypes.byref(ly),
                                             ctypes.byref(scfg), boot.h, boot_scale, outs))
        else:
            bc, keep = self._fft_cfg(*fft_cfg)
            _chk(lib().secpe_enc_argmax_boot_cfg(self.h, keys.h, ins, cts.n, prompt_cts, ctypes.byref(ly),
                                                 ctypes.byref(scfg), ctypes.byref(bc), boot_scale, outs))
        out.level, out.scale = outs[0].level, outs[0].scale
        n, N = n_out, self.N
        # each output is written compactly ([2][level+1][N]) at the start of its slot
        out.t = out.t.reshape(n, -1)[:, : 2 * (out.level + 1) * N].reshape(n, 2, out.level + 1, N).contiguous()
        return out

    def bootstrap_fft(self, keys, a, level, K, r, poly, cts, cts_im, stc, stc_im):
        """secpe_bootstrap_fft (reading R37); every stage a (steps, pts, pt_scale) triple, pts a cuda
        uint64 tensor [n_diag][limbs][N]."""
        cfg, keep = self._fft_cfg(level, K, r, poly, cts, cts_im, stc, stc_im)
        out = self._out(max(level - (len(cts) + len(stc) + 6 + r), 0))
        ca, co = a.c(), out.c()
        _chk(lib().secpe_bootstrap_fft(self.h, keys.h, ctypes.byref(ca), ctypes.byref(cfg), ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def bootstrap_with(self, keys, a, boot):
        """secpe_bootstrap with the configuration of a Boot object (secpe_boot_get_cfg)."""
        cfg = CBootCfg()
        _chk(lib().secpe_boot_get_cfg(boot.h, ctypes.byref(cfg)))
        out = self._out(max(cfg.level - lib().secpe_boot_depth(ctypes.byref(cfg)), 0))
        ca, co = a.c(), out.c()
        _chk(lib().secpe_bootstrap(self.h, keys.h, ctypes.byref(ca), ctypes.byref(cfg), ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def bootstrap(self, keys, a, level, n1, n2, K, r, poly, cts_re, cts_im, cts_scale, stc_re, stc_im, stc_scale):
        """secpe_bootstrap (readings R32-R35); the four matrices as cuda uint64 tensors
        [n2][n1][limbs][N] (NTT-form encoded diagonals)."""
        for t in (cts_re, cts_im, stc_re, stc_im):
            assert t.is_cuda and t.dtype == torch.uint64 and t.is_contiguous()
        pc = np.ascontiguousarray(poly, dtype=np.float64)
        assert pc.shape == (16,)
        ptr = lambda t: ctypes.cast(t.data_ptr(), u64p)
        cfg = CBootCfg(level, n1, n2, K, r, pc.ctypes.data_as(f64p), ptr(cts_re), ptr(cts_im), cts_scale,
                       ptr(stc_re), ptr(stc_im), stc_scale)
        out = self._out(max(level - lib().secpe_boot_depth(ctypes.byref(cfg)), 0))
        ca, co = a.c(), out.c()
        _chk(lib().secpe_bootstrap(self.h, keys.h, ctypes.byref(ca), ctypes.byref(cfg), ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def linear_transform_bsgs(self, keys, a, pts, n1, n2, pt_scale):
        """secpe_linear_transform_bsgs (reading R31); pts a cuda uint64 tensor [n2][n1][a.level+1][N]."""
        assert pts.is_cuda and pts.dtype == torch.uint64 and pts.is_contiguous()
        assert tuple(pts.shape[:3]) == (n2, n1, a.level + 1)
        out = self._out(a.level - 1)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_linear_transform_bsgs(self.h, keys.h, ctypes.byref(ca), ctypes.cast(pts.data_ptr(), u64p),
                                               n1, n2, pt_scale, ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def rescale(self, a):
        out = self._out(a.level - 1)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_rescale(self.h, ctypes.byref(ca), ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def rotate(self, keys, a, steps):
        out = self._out(a.level)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_rotate(self.h, keys.h, ctypes.byref(ca), steps, ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    # ---- SecPE circuits ---------------------------------------------------------------------------
    def sign_poly(self, keys, a, stages, target_scale):
        cfg = sign_cfg(stages)
        depth = lib().secpe_sign_depth(ctypes.byref(cfg))
        _chk(depth if depth < 0 else 0)
        out = self._out(a.level - depth)
        ca, co = a.c(), out.c()
        _chk(lib().secpe_sign_poly(self.h, keys.h, ctypes.byref(ca), ctypes.byref(cfg), target_scale,
                                   ctypes.byref(co)))
        out.level, out.scale = co.level, co.scale
        return out

    def argmax_info(self, lay, stages, in_level):
        cfg, ly = sign_cfg(stages), layout(lay)
        ol, os_ = ctypes.c_int32(), ctypes.c_double()
        _chk(lib().secpe_argmax_info(self.h, ctypes.byref(ly), ctypes.byref(cfg), in_level, ctypes.byref(ol),
                                     ctypes.byref(os_)))
        return ol.value, os_.value

    def enc_argmax(self, keys, cts, lay, stages, out=None):
        """SecPE private voting on a batch Ct (n ciphertexts, contiguous) -> batch Ct."""
        cfg, ly = sign_cfg(stages), layout(lay)
        ol, _ = self.argmax_info(lay, stages, cts.level)
        if out is None:
            out = self.new_ct(ol, cts.n)
        ins = (CCt * cts.n)(*[cts.c(i) for i in range(cts.n)])
        outs = (CCt * cts.n)(*[CCt(ctypes.cast(out.t[i].data_ptr(), u64p), ol, 0.0) for i in range(cts.n)])
        _chk(lib().secpe_enc_argmax(self.h, keys.h, ins, cts.n, ctypes.byref(ly), ctypes.byref(cfg), outs))
        out.level, out.scale = outs[0].level, outs[0].scale
        return out

    def enc_argmax_host(self, keys, h_in, level, scale, lay, stages, h_out=None, chunk=0):
        """secpe_enc_argmax_host: h_in a host (CPU, ideally pinned) uint64 tensor [n][2][level+1][N];
        returns (h_out, out_level, out_scale).  Enqueue-only: h_out is complete after sync()."""
        cfg, ly = sign_cfg(stages), layout(lay)
        assert h_in.device.type == "cpu" and h_in.dtype == torch.uint64 and h_in.is_contiguous()
        n = h_in.shape[0]
        ol, _ = self.argmax_info(lay, stages, level)
        if h_out is None:
            h_out = torch.empty((n, 2, ol + 1, self.N), dtype=torch.uint64, pin_memory=h_in.is_pinned())
        assert h_out.device.type == "cpu" and h_out.is_contiguous() and h_out.numel() >= n * 2 * (ol + 1) * self.N
        olv, osc = ctypes.c_int32(0), ctypes.c_double(0.0)
        _chk(lib().secpe_enc_argmax_host(self.h, keys.h, ctypes.cast(h_in.data_ptr(), u64p), n, level, scale,
                                         ctypes.byref(ly), ctypes.byref(cfg), ctypes.cast(h_out.data_ptr(), u64p),
                                         chunk, ctypes.byref(olv), ctypes.byref(osc)))
        return h_out, olv.value, osc.value

    # ---- instrumentation --------------------------------------------------------------------------
    def oplog(self, enable=None, clear=False):
        if enable is not None:
            _chk(lib().secpe_oplog_enable(self.h, 1 if enable else 0))
        n = lib().secpe_oplog_get(self.h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        lib().secpe_oplog_get(self.h, buf, n + 1)
        if clear:
            _chk(lib().secpe_oplog_clear(self.h))
        return [l for l in buf.value.decode().split("\n") if l]

    def profile_begin(self):
        _chk(lib().secpe_profile_begin(self.h))

    def profile_end(self):
        o = np.zeros(30, dtype=np.float64)
        _chk(lib().secpe_profile_end(self.h, o.ctypes.data_as(f64p), 30))
        r = {}
        for k, name in enumerate(("ntt_fp", "keyswitch", "rescale", "ntt_int", "stage_H1_aggregate", "stage_H2_mask",
                                  "stage_H3_duplicate", "stage_H4_quickmax", "stage_H6_final_sign",
                                  "ntt_fp_operands")):
            r[name] = dict(ms=float(o[3 * k]), bytes=float(o[3 * k + 1]), units=float(o[3 * k + 2]))
        r["ntt"] = {f: r["ntt_fp"][f] + r["ntt_int"][f] for f in ("ms", "bytes", "units")}
        return r

    def opcounts(self, reset=False):
        c = np.zeros(8, dtype=np.int64)
        _chk(lib().secpe_opcounts(self.h, c.ctypes.data_as(i64p), 1 if reset else 0))
        keys = ["ntt_limbs", "keyswitch", "rescale", "rotate", "mulct", "mulconst", "launches", "sign"]
        return dict(zip(keys, (int(v) for v in c)))


def pack(scores, lay, n_slots):
    """H0 client packing: score[q, p, k] -> slot q*block + p*K + k."""
    P, K, b = lay["prompts"], lay["classes"], lay["block"]
    z = np.zeros(n_slots)
    q = scores.shape[0]
    idx = (np.arange(q)[:, None, None] * b + np.arange(P)[None, :, None] * K + np.arange(K)[None, None, :])
    z[idx.ravel()] = scores.ravel()
    return z


def argmax_rotations(lay):
    """Rotation steps the argmax circuit uses (Galois keys to request from the client)."""
    P, K = lay["prompts"], lay["classes"]
    r = [K << t for t in range(P.bit_length() - 1)] + [-K] + [1 << i for i in range(K.bit_length() - 1)]
    return sorted(set(r))


def labels(z, lay):
    """Client decode: argmax over each query's K window slots (first index on ties)."""
    K, b, q = lay["classes"], lay["block"], lay["queries"]
    w = np.asarray(z)[: q * b].reshape(q, b)[:, :K]
    return np.argmax(w, axis=1)
