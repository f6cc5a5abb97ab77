"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Integer ciphertext arithmetic must be bit-exact (north_star); decrypted values within 2^-10 of
the plaintext mirror; labels exact.  Inputs are seeded (synth) and shared as data; the oracle
never consumes anything the CUDA path produced.
"""
import json
import os

import numpy as np
import pytest
import torch

import synth
from oracle import ckks, plan

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def load_sign(name):
    d = json.load(open(os.path.join(HERE, "..", "data", name)))
    return [list(map(float, c)) for c in d["coeffs"]]


@pytest.fixture(scope="module")
def S():
    from paper_2502_00847_b200 import build, secpe
    build.build()
    return secpe


class Pair:
    """Oracle params + GPU context for the same parameter description."""

    def __init__(self, secpe, name):
        self.desc = synth.PARAM_SETS[name]
        self.prm = ckks.Params(self.desc)
        self.gpu = secpe.Context(self.desc)
        self.secpe = secpe

    def up(self, ct):
        """oracle Ct -> GPU Ct (upload of oracle data as an input)."""
        t = torch.from_numpy(ct.data[None].copy()).cuda()
        return self.secpe.Ct(t, ct.level, ct.scale)

    @staticmethod
    def down(ct, i=0):
        torch.cuda.synchronize()
        return ct.t[i].cpu().numpy()


_pairs = {}


def pair(S, name):
    if name not in _pairs:
        _pairs[name] = Pair(S, name)
    return _pairs[name]


# ---------------------------------------------------------------------------------------------
def test_context_tables(S):
    for name in ("toy", "argmax"):
        P = pair(S, name)
        primes, psi = P.gpu.info()
        assert primes == P.prm.primes and psi == P.prm.psi


@pytest.mark.parametrize("name,n_polys,first,n_limbs", [
    ("toy", 1, 0, 8), ("toy", 3, 2, 5), ("toy", 2, 8, 1),       # ragged batch, offset limbs, special prime
    ("ntt", 2, 0, 24), ("ntt", 1, 13, 11),                       # configs[1] primes at N = 2^16
    ("argmax", 1, 25, 13),                                       # q tail + special primes
    ("boot16", 3, 0, 30),                                        # 60-bit + 50-bit (FpB) + 60-bit rows
])
def test_ntt_bit_exact(S, name, n_polys, first, n_limbs):
    P = pair(S, name)
    prm = P.prm
    primes = prm.primes[first:first + n_limbs]
    x = synth.uniform_residues(100 + first, primes, n_polys, prm.logn)
    t = torch.from_numpy(x.copy()).cuda()
    P.gpu.ntt(t, first, n_limbs)
    got = t.cpu().numpy()
    # compare sampled limbs (oracle NTT is ~6 ms per 2^16 limb)
    rng = np.random.default_rng(1)
    for pi in range(n_polys):
        for l in sorted(set(rng.integers(0, n_limbs, 3).tolist())):
            want = ckks.ntt(x[pi, l], primes[l], prm.psi[first + l], prm.logn)
            assert np.array_equal(got[pi, l], want), (pi, l)
    P.gpu.ntt(t, first, n_limbs, inverse=True)
    assert np.array_equal(t.cpu().numpy(), x)


@pytest.mark.parametrize("name,first,n_limbs", [
    ("toy", 0, 9),        # 40-bit chain + 50-bit special (integer rows)
    ("argmax", 0, 40),    # configs[4]: 45-bit chain + 46-bit special primes (exact-FP64 rows, |v| <= 13 q < 2^51)
    ("ntt", 0, 24),       # configs[1]: 60-bit primes (integer rows, Harvey bounds near 2^62)
    ("boot16", 0, 30),    # bootstrap chain at N = 2^16: 60-bit q0 + 22 x 50-bit (exact-FP64 rows with reductions,
                          # FpB, |v| <= 3.24 q ~ 2^51.9) + 7 x 60-bit special primes
])
def test_ntt_edge_inputs(S, name, first, n_limbs):
    """Worst-case magnitudes for the lazy butterflies: all-(q-1), all-zero, alternating q-1 / 0 and
    (q-1)/2 inputs, forward against the oracle's NTT on sampled limbs (incl. the first and last), and the
    inverse of an all-(q-1) NTT-domain input against the oracle's INTT."""
    P = pair(S, name)
    prm = P.prm
    primes = prm.primes[first:first + n_limbs]
    qv = np.array(primes, dtype=np.uint64)[None, :, None]
    check = sorted({0, n_limbs - 1, n_limbs // 2, 1 % n_limbs})
    for fill in ("zero", "max", "alt", "half"):
        x = np.zeros((1, n_limbs, prm.N), dtype=np.uint64)
        if fill == "max":
            x[:] = qv - np.uint64(1)
        elif fill == "alt":
            x[:, :, ::2] = (qv - np.uint64(1))[:, :, :1]
        elif fill == "half":
            x[:] = (qv - np.uint64(1)) // np.uint64(2)
        t = torch.from_numpy(x.copy()).cuda()
        P.gpu.ntt(t, first, n_limbs)
        got = t.cpu().numpy()
        for l in check:
            assert np.array_equal(got[0, l], ckks.ntt(x[0, l], primes[l], prm.psi[first + l], prm.logn)), (fill, l)
    x = np.zeros((1, n_limbs, prm.N), dtype=np.uint64)
    x[:] = qv - np.uint64(1)
    t = torch.from_numpy(x.copy()).cuda()
    P.gpu.ntt(t, first, n_limbs, inverse=True)
    got = t.cpu().numpy()
    for l in check:
        assert np.array_equal(got[0, l], ckks.intt(x[0, l], primes[l], prm.psi[first + l], prm.logn)), ("inv", l)


def test_keys_bit_exact(S):
    P = pair(S, "toy")
    ev = ckks.Oracle(P.prm)
    seed = synth.KEY_SEED_BASE + 1
    ko = ev.keygen(seed, [1, -1, 4])
    kg = P.gpu.keygen(seed, [1, -1, 4])
    assert np.array_equal(kg.export(0), ko.s_ntt)
    assert np.array_equal(kg.export(1), ko.pk)
    assert np.array_equal(kg.export(2), ko.rlk)
    for g, swk in ko.gk.items():
        assert np.array_equal(kg.export(3, g), swk)


@pytest.fixture(scope="module")
def toy_env(S):
    P = pair(S, "toy")
    ev = ckks.Oracle(P.prm)
    seed = synth.KEY_SEED_BASE + 1
    steps = [1, -1, 3, 64]
    return P, ev, ev.keygen(seed, steps), P.gpu.keygen(seed, steps)


def test_encrypt_decrypt_bit_exact(toy_env):
    P, ev, ko, kg = toy_env
    prm = P.prm
    z = synth.uniform_slots(7, prm.N // 2)
    m = ckks.encode(prm, z, prm.scale)                      # oracle encoding = shared integer input
    for level in (prm.L, 3, 0):
        co = ev.encrypt_int(ko, m, level, prm.scale, 99)
        cg = P.gpu.encrypt_coeffs(kg, m, level, prm.scale, 99)
        assert np.array_equal(P.down(cg), co.data)
        res = np.zeros((level + 1, prm.N), dtype=np.uint64)
        ckks.lib().o_decrypt_residues(prm.cptr, ckks.P(ko.s_ntt), ckks.P(co.data), level, ckks.P(res))
        assert np.array_equal(P.gpu.decrypt_residues(kg, cg), res)
    # client encoders agree within +-1 per coefficient (reading R16) and decrypt is accurate
    assert np.abs(P.gpu.encode(z, prm.scale) - m).max() <= 1
    cg = P.gpu.encrypt(kg, z, prm.L, prm.scale, 5)
    assert np.abs(P.gpu.decrypt(kg, cg) - z).max() < 2 ** -20


def test_ops_bit_exact_toy(toy_env):
    P, ev, ko, kg = toy_env
    prm, g = P.prm, P.gpu
    z1, z2 = synth.uniform_slots(1, prm.N // 2), synth.uniform_slots(2, prm.N // 2)
    a = ev.encrypt(ko, z1, prm.scale, 1)
    b = ev.encrypt(ko, z2, prm.scale, 2)
    ga, gb = P.up(a), P.up(b)
    b5 = ev.drop(b, 5)
    chk = lambda gct, oct_: np.array_equal(P.down(gct), oct_.data)
    assert chk(g.add(ga, gb), ev.add_raw(a, b))
    assert chk(g.sub(ga, P.up(b5)), ev.sub_raw(a, b5))               # level alignment by drop
    assert chk(g.add_const(ga, -0.3125), ckks.Ct(ev.add_int_raw(a, ckks.round_half_away(-0.3125 * a.scale)), 0))
    assert chk(g.drop(ga, 2), ev.drop(a, 2))
    r = g.rescale(ga)
    ro = ev.rescale(a)
    assert chk(r, ro) and r.scale == ro.scale
    mr = g.mul_relin(kg, ga, gb)
    assert chk(mr, ev.mul_relin(ko, a, b))
    mc = g.mul_const(ga, 0.7, prm.scale, 4)
    assert chk(mc, ev.mul_const(a, 0.7, prm.scale, 4))
    # fused relinearise-and-rescale (bit-identical to mul_relin then rescale), batched: (a, b), (b, a)
    ab = P.secpe.Ct(torch.cat([ga.t, gb.t]), ga.level, ga.scale)
    ba = P.secpe.Ct(torch.cat([gb.t, ga.t]), ga.level, ga.scale)
    rr = g.mul_relin_rescale(kg, ab, ba)
    want = ev.rescale(ev.mul_relin(ko, a, b))
    assert rr.level == a.level - 1 and rr.scale == want.scale
    assert np.array_equal(P.down(rr, 0), want.data) and np.array_equal(P.down(rr, 1), want.data)
    assert np.abs(g.decrypt(kg, rr, 1) - z1 * z2).max() < 2 ** -10
    for s in (1, -1, 3, 64):
        assert chk(g.rotate(kg, ga, s), ev.rotate_raw(ko, a, s))
    lay = dict(synth.LAYOUTS["toy"], queries=16)
    mask = plan.mask_slots(lay, prm.N // 2)
    assert chk(g.mul_mask(ga, mask, prm.scale), ev.mul_mask(a, mask, prm.scale))
    with pytest.raises(P.secpe.SecpeError, match="scales"):
        g.add(ga, g.rescale(gb))


def test_ops_bit_exact_ks_config(S):
    """configs[2]/[3] parameters (N = 2^16, 24 x 60-bit, dnum 3, 8 special primes)."""
    P = pair(S, "ks")
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 3
    ko, kg = ev.keygen(seed, [1]), g.keygen(seed, [1])
    z1, z2 = synth.uniform_slots(31, prm.N // 2), synth.uniform_slots(32, prm.N // 2)
    a = ev.encrypt(ko, z1, prm.scale, 1)
    b = ev.encrypt(ko, z2, prm.scale, 2)
    ga, gb = P.up(a), P.up(b)
    mo = ev.rescale(ev.mul_relin(ko, a, b))
    mg = g.rescale(g.mul_relin(kg, ga, gb))
    assert np.array_equal(P.down(mg), mo.data)
    assert np.abs(P.gpu.decrypt(kg, mg) - z1 * z2).max() < 2 ** -10
    ro = ev.rotate_raw(ko, a, 1)
    assert np.array_equal(P.down(g.rotate(kg, ga, 1)), ro.data)
    # batched rotation and relinearise-and-rescale at full size (N = 2^16, 24 limbs)
    rb = g.rotate_batch(kg, P.secpe.Ct(torch.cat([ga.t, ga.t]), ga.level, ga.scale), 1)
    assert np.array_equal(P.down(rb, 1), ro.data)
    rr = g.mul_relin_rescale(kg, ga, gb)
    assert np.array_equal(P.down(rr), mo.data)
    assert np.abs(g.decrypt(kg, rr) - z1 * z2).max() < 2 ** -10


def test_sign_poly_bit_exact(toy_env):
    P, ev, ko, kg = toy_env
    prm = P.prm
    st = load_sign("sign_f1_f1.json")
    x = synth.uniform_slots(9, prm.N // 2, -1, 1)
    a = ev.encrypt(ko, x, prm.scale, 3)
    so = plan.sign(ev, ko, a, st, prm.scale)
    sg = P.gpu.sign_poly(kg, P.up(a), st, prm.scale)
    assert np.array_equal(P.down(sg), so.data) and sg.scale == so.scale and sg.level == so.level


def run_argmax_pair(S, pname, lname, sname, seed_in, n_ct=1, oracle_cts=1):
    P = pair(S, pname)
    prm, g = P.prm, P.gpu
    st = load_sign(sname)
    lay = synth.LAYOUTS[lname] if isinstance(lname, str) else lname
    steps = plan.argmax_rotations(lay)
    seed = synth.KEY_SEED_BASE + 7
    ev = ckks.Oracle(prm)
    ko, kg = ev.keygen(seed, steps), g.keygen(seed, steps)
    gen = synth.toy_scores if pname.startswith("toy") else synth.softmax_scores
    scores = [gen(seed_in + i, lay["queries"], lay["prompts"], lay["classes"]) for i in range(n_ct)]
    cts = [ev.encrypt(ko, plan.pack(s, lay, prm.N // 2), prm.scale, 500 + i) for i, s in enumerate(scores)]
    batch = S.Ct(torch.from_numpy(np.stack([c.data for c in cts])).cuda(), prm.L, prm.scale)
    g.oplog(enable=True, clear=True)
    out = g.enc_argmax(kg, batch, lay, st)
    glog = g.oplog(enable=False, clear=True)
    got = out.t.cpu().numpy()
    # the unlogged call runs the batch as concurrent sub-batches on auxiliary streams: same integers
    out2 = g.enc_argmax(kg, batch, lay, st)
    assert np.array_equal(out2.t.cpu().numpy(), got) and out2.level == out.level and out2.scale == out.scale
    mir = ckks.Mirror(prm)
    for i in range(n_ct):
        z = plan.pack(scores[i], lay, prm.N // 2)
        ref = plan.argmax(ckks.Mirror(prm), None, ckks.MirrorCt(z, prm.L, prm.scale), lay, st)
        dec = g.decrypt(kg, out, i)
        assert np.abs(dec - ref.v).max() < 2 ** -10
        mean = scores[i].mean(axis=1)
        srt = np.sort(mean, axis=1)
        ok = srt[:, -1] - srt[:, -2] >= 2.0 ** -7
        assert (S.labels(dec, lay)[ok] == plan.true_labels(scores[i])[ok]).all()
        if i < oracle_cts:
            oo = plan.argmax(ev, ko, cts[i], lay, st)
            assert np.array_equal(got[i], oo.data), "ciphertext %d differs from the oracle" % i
            assert out.level == oo.level and out.scale == oo.scale
    plan.argmax(mir, None, ckks.MirrorCt(np.zeros(prm.N // 2), prm.L, prm.scale), lay, st)
    assert glog == mir.log  # identical planned op lists (reading R13)
    return out


def test_argmax_graph_replay(S):
    """secpe_enc_argmax on a non-default stream with the same buffers: the first call runs eagerly and
    captures a CUDA graph, later calls replay it -- every result equals the eager one word for word."""
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        desc = synth.PARAM_SETS["toy_argmax"]
        g = S.Context(desc, stream=stream.cuda_stream)
        lay = dict(synth.LAYOUTS["toy"], queries=64)
        st = load_sign("sign_f1_f1.json")
        kg = g.keygen(synth.KEY_SEED_BASE + 7, plan.argmax_rotations(lay))
        batch = g.new_ct(g.L, 2)
        for i in range(2):
            z = plan.pack(synth.toy_scores(1001 + i, lay["queries"], lay["prompts"], lay["classes"]), lay, g.N // 2)
            g.encrypt_coeffs(kg, g.encode(z, g.scale), g.L, g.scale, 500 + i,
                             out=S.Ct(batch.t[i:i + 1], g.L, g.scale))
        batch.level, batch.scale = g.L, g.scale
        ol, _ = g.argmax_info(lay, st, g.L)
        out = g.new_ct(ol, 2)
        g.enc_argmax(kg, batch, lay, st, out=out)
        stream.synchronize()
        first = out.t.cpu().numpy().copy()
        for _ in range(3):
            out.t.zero_()
            g.enc_argmax(kg, batch, lay, st, out=out)
            stream.synchronize()
            assert np.array_equal(out.t.cpu().numpy(), first)
    assert g.opcounts()["keyswitch"] > 0


def test_argmax_host_pipeline(S):
    """secpe_enc_argmax_host (host buffers, two staging slots, copy stream) on a ragged chunking
    (5 ciphertexts in chunks of 2) and twice in a row (slot reuse across calls), pinned and pageable:
    every result equals the device-buffer secpe_enc_argmax word for word."""
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        desc = synth.PARAM_SETS["toy_argmax"]
        g = S.Context(desc, stream=stream.cuda_stream)
        lay = dict(synth.LAYOUTS["toy"], queries=64)
        st = load_sign("sign_f1_f1.json")
        kg = g.keygen(synth.KEY_SEED_BASE + 7, plan.argmax_rotations(lay))
        n = 5
        batch = g.new_ct(g.L, n)
        for i in range(n):
            z = plan.pack(synth.toy_scores(2001 + i, lay["queries"], lay["prompts"], lay["classes"]), lay, g.N // 2)
            g.encrypt_coeffs(kg, g.encode(z, g.scale), g.L, g.scale, 600 + i,
                             out=S.Ct(batch.t[i:i + 1], g.L, g.scale))
        batch.level, batch.scale = g.L, g.scale
        ol, osc = g.argmax_info(lay, st, g.L)
        ref = g.enc_argmax(kg, batch, lay, st)
        stream.synchronize()
        want = ref.t.cpu().numpy()
        for pinned in (True, False):
            h_in = batch.t.cpu()
            if pinned:
                h_in = h_in.pin_memory()
            outs = []
            for _ in range(2):
                h_out, lv, sc = g.enc_argmax_host(kg, h_in, g.L, g.scale, lay, st, chunk=2)
                outs.append(h_out)
                assert lv == ol and sc == ref.scale
            g.sync()
            for h_out in outs:
                assert np.array_equal(h_out.numpy(), want)


def test_integer_base_conversion_fallback(S, monkeypatch):
    """SECPE_NO_TC=1 selects the integer split-30 base-conversion kernels (ModUp, ModDown, fused ModDown +
    rescale) instead of the tensor-core ones: the same integers (configs[2]/[3] parameters)."""
    monkeypatch.setenv("SECPE_NO_TC", "1")
    P = Pair(S, "ks")
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 3
    ko, kg = ev.keygen(seed, [1]), g.keygen(seed, [1])
    z1, z2 = synth.uniform_slots(41, prm.N // 2), synth.uniform_slots(42, prm.N // 2)
    a = ev.encrypt(ko, z1, prm.scale, 1)
    b = ev.encrypt(ko, z2, prm.scale, 2)
    ga, gb = P.up(a), P.up(b)
    assert np.array_equal(P.down(g.mul_relin_rescale(kg, ga, gb)), ev.rescale(ev.mul_relin(ko, a, b)).data)
    assert np.array_equal(P.down(g.rotate(kg, ga, 1)), ev.rotate_raw(ko, a, 1).data)


def test_argmax_toy_bit_exact(S):
    lay = dict(synth.LAYOUTS["toy"], queries=64)
    run_argmax_pair(S, "toy_argmax", lay, "sign_f1_f1.json", 1001, n_ct=3, oracle_cts=3)


def test_argmax_small_ring_bit_exact(S):
    run_argmax_pair(S, "argmax_small", "argmax_small_k2", "sign_7_15_15.json", 5001, n_ct=2, oracle_cts=2)


@pytest.mark.parametrize("fpb", ["0", "1"])
def test_argmax_small49_bit_exact(S, monkeypatch, fpb):
    """configs[4]'s circuit on 49-bit primes at scale 2^49 (reading R41, the paper's prime size): plan constants
    pass 2^63 (wide constants); with SECPE_FPB=1 every row of Q u P takes the FP64 NTT with reductions (FpB) that
    N >= 2^15 uses by default, with 0 the integer NTT -- both word for word against the oracle, identical op
    logs."""
    monkeypatch.setenv("SECPE_FPB", fpb)
    _pairs.pop("argmax_small49", None)
    try:
        run_argmax_pair(S, "argmax_small49", "argmax_small_k2", "sign_7_15_15.json", 5101, n_ct=2, oracle_cts=1)
        P = pair(S, "argmax_small49")
        assert max(P.prm.q + P.prm.p) >= 2 ** 46  # FpB-class rows
    finally:
        _pairs.pop("argmax_small49", None)


@pytest.mark.slow
def test_argmax49_full(S):
    """configs[4] at 49-bit primes (R41) at full size (N = 2^16, FpB rows by default), batch of 2: ciphertext 0
    bit-exact against the oracle, every label exact above the margin."""
    run_argmax_pair(S, "argmax49", "argmax_k2", "sign_7_15_15.json", 1000 * 5 + 11, n_ct=2, oracle_cts=1)


@pytest.mark.slow
def test_argmax_config5_full(S):
    """BASELINE configs[4] at full size (N = 2^16, 30 limbs, 2048 queries x P=8 x K=2), batch of 2 as bench:
    ciphertext 0 bit-exact against the oracle, every query's label exact above the margin."""
    run_argmax_pair(S, "argmax", "argmax_k2", "sign_7_15_15.json", 1000 * 5 + 1, n_ct=2, oracle_cts=1)


@pytest.mark.parametrize("mode", [1, 2])
def test_cluster_ntt_path(S, monkeypatch, mode):
    """SECPE_NTT_CLUSTER=1 (FP rows) / 2 (all rows): the single-pass thread-block-cluster NTT (ntt.cu
    ntt_cluster, DSMEM transpose) gives the same integers as the oracle -- plain forward/inverse on the
    configs[4] 45-bit chain + special primes and on the configs[1] 60-bit primes, and the fused
    prologue/epilogue modes through mul_relin_rescale and rotate (configs[2]/[3] parameters)."""
    monkeypatch.setenv("SECPE_NTT_CLUSTER", str(mode))
    for name, first, n_limbs in (("argmax", 20, 18), ("ntt", 3, 5)):
        prm = ckks.Params(synth.PARAM_SETS[name])
        g = S.Context(synth.PARAM_SETS[name])
        primes = prm.primes[first:first + n_limbs]
        x = synth.uniform_residues(300 + first, primes, 2, prm.logn)
        t = torch.from_numpy(x.copy()).cuda()
        g.ntt(t, first, n_limbs)
        got = t.cpu().numpy()
        for pi, l in ((0, 0), (1, n_limbs - 1), (1, n_limbs // 2)):
            assert np.array_equal(got[pi, l], ckks.ntt(x[pi, l], primes[l], prm.psi[first + l], prm.logn)), (name, pi, l)
        g.ntt(t, first, n_limbs, inverse=True)
        assert np.array_equal(t.cpu().numpy(), x)
    P = Pair(S, "argmax" if mode == 1 else "ks")  # 45-bit FP rows / 60-bit integer rows
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 3
    ko, kg = ev.keygen(seed, [1]), g.keygen(seed, [1])
    z1, z2 = synth.uniform_slots(51, prm.N // 2), synth.uniform_slots(52, prm.N // 2)
    a = ev.encrypt(ko, z1, prm.scale, 1)
    b = ev.encrypt(ko, z2, prm.scale, 2)
    ga, gb = P.up(a), P.up(b)
    assert np.array_equal(P.down(g.mul_relin_rescale(kg, ga, gb)), ev.rescale(ev.mul_relin(ko, a, b)).data)
    assert np.array_equal(P.down(g.rotate(kg, ga, 1)), ev.rotate_raw(ko, a, 1).data)


@pytest.mark.parametrize("name,steps,n_ct,level_drop", [
    ("toy", [1, 2, -1, 0, 3], 2, 0),          # ragged step set incl. identity, batch of 2
    ("toy", [1, -1], 1, 2),                   # outputs below the input level
    ("ks", [1, 4, 16384], 1, 0),              # configs[3] primes (60-bit integer rows), N = 2^16
    ("argmax", [2, -2], 1, 10),               # configs[4] 45-bit FP rows, mid-chain level
])
def test_rotate_hoisted_bit_exact(S, name, steps, n_ct, level_drop):
    """N2 hoisted rotations (secpe_rotate_hoisted, reading R29): every (step, ciphertext) output equal
    word for word to the oracle's rotate_hoisted_raw; decrypts to RotL(z, step) within 2^-10."""
    P = pair(S, name)
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 7
    rot = sorted({s for s in steps if s % (prm.N // 2)})
    ko, kg = ev.keygen(seed, rot), g.keygen(seed, rot)
    level = prm.L - level_drop
    cts = [ev.encrypt(ko, synth.uniform_slots(60 + i, prm.N // 2), prm.scale, 20 + i) for i in range(n_ct)]
    cts = [ev.drop(c, level) if level < c.level else c for c in cts]
    batch = S.Ct(torch.from_numpy(np.stack([c.data for c in cts])).cuda(), level, prm.scale)
    outs = g.rotate_hoisted(kg, batch, steps)
    torch.cuda.synchronize()
    for i, c in enumerate(cts):
        want = ev.rotate_hoisted_raw(ko, c, steps)
        for s, (st, o) in enumerate(zip(steps, outs)):
            assert o.level == level and o.scale == prm.scale
            assert np.array_equal(o.t[i].cpu().numpy(), want[s].data), (name, st, i)
    z0 = synth.uniform_slots(60, prm.N // 2)
    for st, o in zip(steps, outs):
        got = ev.decrypt(ko, ckks.Ct(o.t[0].cpu().numpy(), o.scale))
        assert np.abs(got.real - np.roll(z0, -st)).max() < 2 ** -10


def test_rotate_hoisted_errors(S):
    P = pair(S, "toy")
    prm, g = P.prm, P.gpu
    kg = g.keygen(synth.KEY_SEED_BASE + 7, [1])
    z = synth.uniform_slots(1, prm.N // 2)
    a = g.encrypt(kg, z, prm.L, prm.scale, 1)
    with pytest.raises(Exception, match="Galois"):
        g.rotate_hoisted(kg, a, [1, 5])


@pytest.mark.slow
def test_argmax_config5_bench_launch(S):
    """BASELINE configs[4] in bench.py's launch configuration: 16 ciphertexts on a non-default stream
    (two concurrent sub-batch streams, CUDA graph captured on the first call and replayed), full size.
    The last ciphertext (second sub-batch) is compared word for word with the oracle; every query of
    every ciphertext decodes to the plaintext argmax wherever the top-1 gap is above the Sign margin."""
    stream = torch.cuda.Stream()
    desc = synth.PARAM_SETS["argmax"]
    prm = ckks.Params(desc)
    lay = synth.LAYOUTS["argmax_k2"]
    st = load_sign("sign_7_15_15.json")
    steps = plan.argmax_rotations(lay)
    seed = synth.KEY_SEED_BASE + 5
    B = 16
    with torch.cuda.stream(stream):
        g = S.Context(desc, stream=stream.cuda_stream)
        kg = g.keygen(seed, steps)
        scores = [synth.softmax_scores(9000 + i, lay["queries"], lay["prompts"], lay["classes"]) for i in range(B)]
        batch = g.new_ct(g.L, B)
        for i in range(B - 1):  # library-encrypted (checked through decryption + labels)
            z = S.pack(scores[i], lay, g.N // 2)
            g.encrypt_coeffs(kg, g.encode(z, g.scale), g.L, g.scale, 900 + i, out=S.Ct(batch.t[i:i + 1], g.L, g.scale))
        ev = ckks.Oracle(prm)
        ko = ev.keygen(seed, steps)
        last = ev.encrypt(ko, plan.pack(scores[-1], lay, prm.N // 2), prm.scale, 777)
        batch.t[B - 1].copy_(torch.from_numpy(last.data))
        batch.level, batch.scale = g.L, g.scale
        ol, _ = g.argmax_info(lay, st, g.L)
        out = g.new_ct(ol, B)
        g.enc_argmax(kg, batch, lay, st, out=out)  # eager + capture
        stream.synchronize()
        first = out.t.cpu().numpy().copy()
        out.t.zero_()
        g.enc_argmax(kg, batch, lay, st, out=out)  # graph replay
        stream.synchronize()
        got = out.t.cpu().numpy()
    assert np.array_equal(got, first)
    want = plan.argmax(ev, ko, last, lay, st)
    assert np.array_equal(got[B - 1], want.data) and out.level == want.level and out.scale == want.scale
    for i in range(B):
        dec = g.decrypt(kg, out, i)
        srt = np.sort(scores[i].mean(axis=1), axis=1)
        ok = srt[:, -1] - srt[:, -2] >= 2.0 ** -7
        assert ok.mean() > 0.9
        assert (S.labels(dec, lay)[ok] == plan.true_labels(scores[i])[ok]).all(), i


def test_argmax_errors(S):
    """Depth exhausted (K = 16 needs 60 levels > 29 without bootstrapping, reading R18), empty batch,
    no level left to rescale: error codes, never a crash or a wrong result."""
    P = pair(S, "argmax")
    g = P.gpu
    st = load_sign("sign_7_15_15.json")
    with pytest.raises(S.SecpeError):
        g.argmax_info(synth.LAYOUTS["argmax_k16"], st, P.prm.L)
    P = pair(S, "toy")
    g, prm = P.gpu, P.prm
    kg = g.keygen(synth.KEY_SEED_BASE + 7, [1])
    a = g.encrypt(kg, synth.uniform_slots(1, prm.N // 2), 0, prm.scale, 1)  # level 0
    with pytest.raises(S.SecpeError):
        g.rescale(a)
    with pytest.raises(S.SecpeError):
        g.mul_relin_rescale(kg, a, a)


def test_keys_destroy_drops_captured_graphs(S):
    """A captured argmax graph reads its keys' device memory: destroying the keys must drop it, so a new
    keys object (possibly at the same address) on the same buffers computes with the NEW keys."""
    stream = torch.cuda.Stream()
    desc = synth.PARAM_SETS["toy_argmax"]
    lay = dict(synth.LAYOUTS["toy"], queries=64)
    st = load_sign("sign_f1_f1.json")
    rot = plan.argmax_rotations(lay)
    with torch.cuda.stream(stream):
        g = S.Context(desc, stream=stream.cuda_stream)
        ref = S.Context(desc, stream=stream.cuda_stream)
        batch = g.new_ct(g.L, 2)
        batch.t.copy_(torch.from_numpy(np.random.default_rng(5).integers(0, 2 ** 20, batch.t.shape,
                                                                            dtype=np.uint64)))
        batch.level, batch.scale = g.L, g.scale
        ol, _ = g.argmax_info(lay, st, g.L)
        out = g.new_ct(ol, 2)
        k1 = g.keygen(synth.KEY_SEED_BASE + 1, rot)
        for _ in range(2):  # eager + capture, then replay
            g.enc_argmax(k1, batch, lay, st, out=out)
        del k1
        k2 = g.keygen(synth.KEY_SEED_BASE + 2, rot)
        g.enc_argmax(k2, batch, lay, st, out=out)
        stream.synchronize()
        got = out.t.cpu().numpy().copy()
        r2 = ref.keygen(synth.KEY_SEED_BASE + 2, rot)
        want = ref.enc_argmax(r2, batch, lay, st)
        stream.synchronize()
        assert np.array_equal(got, want.t.cpu().numpy())
        del r2, ref  # keys and context destroyed in either order
        k3 = g.keygen(synth.KEY_SEED_BASE + 3, rot)
        del g
        del k3


def test_argmax_degenerate_scores_bit_exact(S):
    """Degenerate inputs of the method on the configs[4] circuit (2^12 ring): exact ties (Sign(0) = 0,
    every tied slot ~1, PAPER.md:184 / reading R28), all-zero and all-one prompts, extreme one-hot
    scores.  Ciphertext bit-exact vs the oracle; decrypted window within 2^-10 of the plaintext mirror."""
    P = pair(S, "argmax_small")
    prm, g = P.prm, P.gpu
    lay = synth.LAYOUTS["argmax_small_k2"]
    st = load_sign("sign_7_15_15.json")
    nq, Pp, K = lay["queries"], lay["prompts"], lay["classes"]
    rng = np.random.default_rng(77)
    scores = rng.uniform(0, 1, (nq, Pp, K))
    scores[0] = 0.5                      # exact tie
    scores[1] = 0.0                      # all zero
    scores[2] = 1.0                      # all one
    scores[3, :, 0], scores[3, :, 1] = 1.0, 0.0
    scores[4, :, 0], scores[4, :, 1] = 0.0, 1.0
    scores[5, :4, :] = [0.9, 0.1]        # half the prompts vote each way: aggregated tie
    scores[5, 4:, :] = [0.1, 0.9]
    seed = synth.KEY_SEED_BASE + 7
    steps = plan.argmax_rotations(lay)
    ev = ckks.Oracle(prm)
    ko, kg = ev.keygen(seed, steps), g.keygen(seed, steps)
    ct = ev.encrypt(ko, plan.pack(scores, lay, prm.N // 2), prm.scale, 41)
    out = g.enc_argmax(kg, P.up(ct), lay, st)
    want = plan.argmax(ev, ko, ct, lay, st)
    assert np.array_equal(P.down(out), want.data)
    ref = plan.argmax(ckks.Mirror(prm), None, ckks.MirrorCt(plan.pack(scores, lay, prm.N // 2), prm.L, prm.scale),
                      lay, st)
    dec = g.decrypt(kg, out)
    b = lay["block"]
    for qi in range(nq):
        assert np.abs(dec[qi * b: qi * b + K] - ref.v[qi * b: qi * b + K]).max() < 2 ** -10
    for qi in (0, 1, 2, 5):              # ties: both window slots ~1
        assert np.all(np.abs(dec[qi * b: qi * b + K] - 1.0) < 0.05)
    assert S.labels(dec, lay)[3] == 0 and S.labels(dec, lay)[4] == 1


def test_argmax_k16_shape_bit_exact(S):
    """BASELINE configs[4]'s K = 16 variant shape (P = 8 prompts x K = 16 classes in 128-slot blocks; QuickMax
    with four iterations, rotations 1..8, aggregation steps 16..64) on a 30-prime 2^12 ring.  The (7,15,15)
    Sign needs 60 levels here (reading R18), so the depth-4 toy Sign f1 o f1 stands in: ciphertext bit-exact
    vs the oracle, decrypted within 2^-10 of the plaintext mirror, labels exact (top-1 gap >= 0.1)."""
    P = pair(S, "argmax_small")
    prm, g = P.prm, P.gpu
    lay = dict(queries=16, prompts=8, classes=16, block=128)
    st = load_sign("sign_f1_f1.json")
    steps = plan.argmax_rotations(lay)
    seed = synth.KEY_SEED_BASE + 9
    ev = ckks.Oracle(prm)
    ko, kg = ev.keygen(seed, steps), g.keygen(seed, steps)
    scores = synth.toy_scores(4242, lay["queries"], lay["prompts"], lay["classes"])
    z = plan.pack(scores, lay, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 17)
    out = g.enc_argmax(kg, P.up(ct), lay, st)
    want = plan.argmax(ev, ko, ct, lay, st)
    assert np.array_equal(P.down(out), want.data) and out.level == want.level
    ref = plan.argmax(ckks.Mirror(prm), None, ckks.MirrorCt(z, prm.L, prm.scale), lay, st)
    dec = g.decrypt(kg, out)
    b, K = lay["block"], lay["classes"]
    for qi in range(lay["queries"]):
        assert np.abs(dec[qi * b: qi * b + K] - ref.v[qi * b: qi * b + K]).max() < 2 ** -10
    assert (S.labels(dec, lay) == plan.true_labels(scores)).all()


def test_empty_inputs(S):
    """Empty batches: a zero-polynomial NTT is a no-op; an empty argmax batch or step list is SECPE_EINVAL."""
    import ctypes
    P = pair(S, "toy")
    g, prm = P.gpu, P.prm
    t = torch.zeros((0, 8, prm.N), dtype=torch.uint64, device="cuda")
    g.ntt(t, 0, 8)
    lay = dict(synth.LAYOUTS["toy"], queries=1)
    st = load_sign("sign_f1_f1.json")
    kg = g.keygen(synth.KEY_SEED_BASE + 7, plan.argmax_rotations(lay))
    cfg, ly = S.sign_cfg(st), S.layout(lay)
    rc = S.lib().secpe_enc_argmax(g.h, kg.h, None, 0, ctypes.byref(ly), ctypes.byref(cfg), None)
    assert rc == -1
    a = g.encrypt(kg, synth.uniform_slots(1, prm.N // 2), prm.L, prm.scale, 1)
    with pytest.raises(S.SecpeError):
        g.rotate_hoisted(kg, a, [])


@pytest.mark.parametrize("logn", [13, 14, 15])
def test_other_ring_dimensions(S, logn):
    """The NTT and key-switching templates for N = 2^13..2^15 (the configs use 2^12 and 2^16): forward /
    inverse NTT, relinearise-and-rescale and a rotation, bit-exact vs the oracle on a small chain."""
    desc = dict(logn=logn, q=[("nearest", 40, 6)], p=[("below", 50, 2)], alpha=3, log_scale=40)
    prm = ckks.Params(desc)
    g = S.Context(desc)
    x = synth.uniform_residues(70 + logn, prm.primes[:8], 2, logn)
    t = torch.from_numpy(x.copy()).cuda()
    g.ntt(t, 0, 8)
    got = t.cpu().numpy()
    for pi, l in ((0, 0), (1, 7), (1, 3)):
        assert np.array_equal(got[pi, l], ckks.ntt(x[pi, l], prm.primes[l], prm.psi[l], logn)), (pi, l)
    g.ntt(t, 0, 8, inverse=True)
    assert np.array_equal(t.cpu().numpy(), x)
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 11
    ko, kg = ev.keygen(seed, [1]), g.keygen(seed, [1])
    a = ev.encrypt(ko, synth.uniform_slots(5, prm.N // 2), prm.scale, 1)
    b = ev.encrypt(ko, synth.uniform_slots(6, prm.N // 2), prm.scale, 2)
    ga = S.Ct(torch.from_numpy(a.data[None].copy()).cuda(), a.level, a.scale)
    gb = S.Ct(torch.from_numpy(b.data[None].copy()).cuda(), b.level, b.scale)
    out = g.mul_relin_rescale(kg, ga, gb)
    torch.cuda.synchronize()
    assert np.array_equal(out.t[0].cpu().numpy(), ev.rescale(ev.mul_relin(ko, a, b)).data)
    r = g.rotate(kg, ga, 1)
    torch.cuda.synchronize()
    assert np.array_equal(r.t[0].cpu().numpy(), ev.rotate_raw(ko, a, 1).data)


@pytest.mark.parametrize("alpha", [2, 4, 8])
def test_key_switching_digit_counts(S, alpha):
    """dnum = 4, 2, 1 at the top level (alpha = 2, 4, 8 over 8 primes): the key inner-product template
    instances for beta = 4 / 2 / 1 (both kernels) and the conversion groups, bit-exact vs the oracle."""
    desc = dict(logn=12, q=[("nearest", 40, 8)], p=[("below", 50, max(2, alpha // 2))], alpha=alpha, log_scale=40)
    prm = ckks.Params(desc)
    g = S.Context(desc)
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 13
    ko, kg = ev.keygen(seed, [3]), g.keygen(seed, [3])
    a = ev.encrypt(ko, synth.uniform_slots(7, prm.N // 2), prm.scale, 1)
    b = ev.encrypt(ko, synth.uniform_slots(8, prm.N // 2), prm.scale, 2)
    ga = S.Ct(torch.from_numpy(a.data[None].copy()).cuda(), a.level, a.scale)
    gb = S.Ct(torch.from_numpy(b.data[None].copy()).cuda(), b.level, b.scale)
    out = g.mul_relin_rescale(kg, ga, gb)
    torch.cuda.synchronize()
    assert np.array_equal(out.t[0].cpu().numpy(), ev.rescale(ev.mul_relin(ko, a, b)).data)
    r = g.rotate(kg, ga, 3)
    torch.cuda.synchronize()
    assert np.array_equal(r.t[0].cpu().numpy(), ev.rotate_raw(ko, a, 3).data)


@pytest.mark.parametrize("alpha", [2, 4, 8])
def test_fused_keyswitch_digit_counts(S, alpha):
    """The fused ModUp second pass + relinearisation key inner product (ntt_ks_inner_kernel: every row of Q u P an
    exact-FP64 row, 45-bit chain + 46-bit special primes) at dnum = 4, 2, 1 and at two levels (full and a ragged last
    digit), word for word against the oracle; the rotation path (separate kernels) on the same keys."""
    desc = dict(logn=12, q=[("nearest", 45, 8)], p=[("below", 46, max(2, alpha // 2))], alpha=alpha, log_scale=45)
    prm = ckks.Params(desc)
    assert all(q < (1 << 46) for q in list(prm.q) + list(prm.p))
    g = S.Context(desc)
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 14
    ko, kg = ev.keygen(seed, [3]), g.keygen(seed, [3])
    a = ev.encrypt(ko, synth.uniform_slots(9, prm.N // 2), prm.scale, 1)
    b = ev.encrypt(ko, synth.uniform_slots(10, prm.N // 2), prm.scale, 2)
    for drop in (0, 3):
        ao, bo = (a, b) if drop == 0 else (ev.drop(a, a.level - drop), ev.drop(b, b.level - drop))
        ga = S.Ct(torch.from_numpy(ao.data[None].copy()).cuda(), ao.level, ao.scale)
        gb = S.Ct(torch.from_numpy(bo.data[None].copy()).cuda(), bo.level, bo.scale)
        out = g.mul_relin_rescale(kg, ga, gb)
        torch.cuda.synchronize()
        assert np.array_equal(out.t[0].cpu().numpy(), ev.rescale(ev.mul_relin(ko, ao, bo)).data), drop
    r = g.rotate(kg, S.Ct(torch.from_numpy(a.data[None].copy()).cuda(), a.level, a.scale), 3)
    torch.cuda.synchronize()
    assert np.array_equal(r.t[0].cpu().numpy(), ev.rotate_raw(ko, a, 3).data)


@pytest.mark.parametrize("name,steps,level_drop", [
    ("toy", [0, 1, 2, 5, -3], 0),
    ("argmax", [0, 1, 3, 2048, -7, 16], 12),
])
def test_linear_transform_bit_exact(S, name, steps, level_drop):
    """secpe_linear_transform (reading R30, a building block of bootstrapping's CoeffToSlot / SlotToCoeff):
    word for word equal to the oracle's linear_transform; decrypts to the plaintext matrix-vector product."""
    P = pair(S, name)
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 17
    rot = sorted({s for s in steps if s})
    ko, kg = ev.keygen(seed, rot), g.keygen(seed, rot)
    n = prm.N // 2
    rng = np.random.default_rng(31)
    z = rng.uniform(-1, 1, n)
    diags = [rng.uniform(-1, 1, n) for _ in steps]
    ct = ev.encrypt(ko, z, prm.scale, 9)
    level = prm.L - level_drop
    if level < ct.level:
        ct = ev.drop(ct, level)
    pt_scale = float(prm.primes[level])
    pts = [ev.plain_ntt(ckks.encode(prm, d, pt_scale), level) for d in diags]
    want = ev.linear_transform(ko, ct, pts, steps, pt_scale)
    got = g.linear_transform(kg, P.up(ct), torch.from_numpy(np.stack(pts)).cuda(), steps, pt_scale)
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    ref = sum(d * np.roll(z, -s) for d, s in zip(diags, steps))
    assert np.abs(ev.decrypt(ko, want).real - ref).max() < 2 ** -10


@pytest.mark.gpu
@pytest.mark.parametrize("name,n1,n2,level_drop", [
    ("toy", 4, 3, 0),
    ("toy", 1, 3, 0),   # giant steps only
    ("toy", 3, 1, 0),   # baby steps only (= R30 with steps 0..n1-1)
    ("argmax", 4, 3, 12),
])
def test_linear_transform_bsgs_bit_exact(S, name, n1, n2, level_drop):
    """secpe_linear_transform_bsgs (reading R31): word for word equal to the oracle's
    linear_transform_bsgs; decrypts to sum_i d_i (.) RotL(z, i) over n1 n2 diagonals."""
    P = pair(S, name)
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    seed = synth.KEY_SEED_BASE + 19
    rot = list(range(1, n1)) + [j * n1 for j in range(1, n2)]
    ko, kg = ev.keygen(seed, rot), g.keygen(seed, rot)
    n = prm.N // 2
    rng = np.random.default_rng(37)
    z = rng.uniform(-1, 1, n)
    d = [rng.uniform(-1, 1, n) for _ in range(n1 * n2)]
    ct = ev.encrypt(ko, z, prm.scale, 11)
    level = prm.L - level_drop
    if level < ct.level:
        ct = ev.drop(ct, level)
    pt_scale = float(prm.primes[level])
    pts = [[ev.plain_ntt(ckks.encode(prm, np.roll(d[j * n1 + i], j * n1), pt_scale), level) for i in range(n1)]
           for j in range(n2)]
    want = ev.linear_transform_bsgs(ko, ct, pts, n1, n2, pt_scale)
    got = g.linear_transform_bsgs(kg, P.up(ct), torch.from_numpy(np.stack([np.stack(r) for r in pts])).cuda(),
                                  n1, n2, pt_scale)
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    ref = sum(d[i] * np.roll(z, -i) for i in range(n1 * n2))
    assert np.abs(ev.decrypt(ko, want).real - ref).max() < 2 ** -10


@pytest.mark.gpu
def test_linear_transform_bsgs_errors(S):
    """R31 argument checks: a missing giant-step key, n1 or n2 < 1 are rejected, nothing written."""
    P = pair(S, "toy")
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    ko, kg = ev.keygen(5, [1]), g.keygen(5, [1])
    ct = P.up(ev.encrypt(ko, np.zeros(prm.N // 2), prm.scale, 1))
    pts = torch.zeros((2, 2, ct.level + 1, prm.N), dtype=torch.uint64, device="cuda")
    with pytest.raises(S.SecpeError):
        g.linear_transform_bsgs(kg, ct, pts, 2, 2, 1.0)   # needs the key for step 2
    with pytest.raises(S.SecpeError):
        g.linear_transform_bsgs(kg, ct, pts[:, :0].contiguous(), 0, 2, 1.0)


# ---------------------------------------------------------------------------------------------
# Bootstrapping (readings R32-R36) on the "boot" parameters (N = 2^12, 2048 slots)
# ---------------------------------------------------------------------------------------------
BOOT = dict(n1=64, n2=32, K=16, r=7, h=64)


@pytest.fixture(scope="module")
def boot(S):
    P = pair(S, "boot")
    ev = ckks.Oracle(P.prm)
    rot = plan.boot_rotations(BOOT["n1"], BOOT["n2"])
    seed = synth.KEY_SEED_BASE + 23
    return P, ev, ev.keygen(seed, rot, h=BOOT["h"]), P.gpu.keygen(seed, rot, h=BOOT["h"])


@pytest.mark.gpu
def test_sparse_keys_and_conjugation_bit_exact(boot):
    """R36 sparse secret and every key built on it word for word; R32 conjugation (SECPE_CONJ) word for
    word equal to the oracle's sigma_{2N-1} + key switch."""
    P, ev, ko, kg = boot
    prm = P.prm
    assert np.array_equal(kg.export(0), ko.s_ntt)
    assert np.array_equal(kg.export(2), ko.rlk)
    gc = ckks.galois_elt(prm, ckks.CONJ)
    assert np.array_equal(kg.export(3, gc), ko.gk[gc])
    rng = np.random.default_rng(4)
    z = rng.uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 21, level=6)
    want = ev.rotate_raw(ko, ct, ckks.CONJ)
    got = P.gpu.rotate(kg, P.up(ct), P.secpe.CONJ)
    assert np.array_equal(P.down(got), want.data)


@pytest.mark.gpu
def test_mod_raise_bit_exact(boot):
    """R33 ModRaise word for word, to the top and to a middle level; level-0 input required."""
    P, ev, ko, kg = boot
    prm = P.prm
    ct = ev.encrypt(ko, np.linspace(-1, 1, prm.N // 2), prm.scale, 22, level=0)
    for lv in (prm.L, 7):
        want = ev.mod_raise(ct, lv)
        got = P.gpu.mod_raise(P.up(ct), lv)
        assert got.level == lv and got.scale == ct.scale
        assert np.array_equal(P.down(got), want.data)
    with pytest.raises(P.secpe.SecpeError):
        P.gpu.mod_raise(P.up(ev.encrypt(ko, np.zeros(4), prm.scale, 1, level=2)), prm.L)


@pytest.fixture(scope="module")
def boot_cfg(boot):
    P, ev = boot[0], boot[1]
    return plan.boot_config(ev, P.prm.scale, P.prm.L, BOOT["K"], BOOT["r"], BOOT["n1"], BOOT["n2"])


@pytest.mark.gpu
@pytest.mark.slow
def test_bootstrap_bit_exact(boot, boot_cfg):
    """N3 end to end: secpe_bootstrap of a level-0 ciphertext is word for word the oracle's bootstrap plan
    (same op list), lands at level L - (8 + r) and decrypts to the input slots within 2^-12."""
    P, ev, ko, kg = boot
    prm, g = P.prm, P.gpu
    rng = np.random.default_rng(5)
    z = rng.uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 23, level=0)
    cfg = boot_cfg
    ev.log.clear()
    want = plan.bootstrap(ev, ko, ct, cfg)
    olog = list(ev.log)
    dev = {nm: torch.from_numpy(np.stack([np.stack(row) for row in cfg[nm]])).cuda()
           for nm in ("cts_re", "cts_im", "stc_re", "stc_im")}
    g.oplog(enable=True, clear=True)
    got = g.bootstrap(kg, P.up(ct), cfg["level"], BOOT["n1"], BOOT["n2"], cfg["K"], cfg["r"], cfg["poly"],
                      dev["cts_re"], dev["cts_im"], cfg["cts_scale"], dev["stc_re"], dev["stc_im"], cfg["stc_scale"])
    glog = g.oplog(enable=False, clear=True)
    assert glog == olog
    assert got.level == want.level == prm.L - plan.boot_depth(BOOT["r"]) and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    assert np.abs(g.decrypt(kg, got) - z).max() < 2 ** -12
    # errors: a level-0 input is required; a missing key is reported
    with pytest.raises(P.secpe.SecpeError):
        g.bootstrap(kg, P.up(ev.encrypt(ko, z, prm.scale, 2, level=1)), cfg["level"], BOOT["n1"], BOOT["n2"],
                    cfg["K"], cfg["r"], cfg["poly"], dev["cts_re"], dev["cts_im"], cfg["cts_scale"], dev["stc_re"],
                    dev["stc_im"], cfg["stc_scale"])
    k2 = g.keygen(5, [1])
    with pytest.raises(P.secpe.SecpeError):
        g.bootstrap(k2, P.up(ct), cfg["level"], BOOT["n1"], BOOT["n2"], cfg["K"], cfg["r"], cfg["poly"],
                    dev["cts_re"], dev["cts_im"], cfg["cts_scale"], dev["stc_re"], dev["stc_im"], cfg["stc_scale"])


@pytest.mark.gpu
@pytest.mark.slow
def test_boot_setup_matches_oracle_encoding(boot, boot_cfg):
    """secpe_boot_create (library-built material): the same polynomial (to a double's rounding), scales, and
    encoded matrices whose integer coefficients equal the oracle's except for +-1 at rare rounding ties of
    two double-precision FFTs; bootstrapping with it decrypts like the oracle-encoded one."""
    P, ev, ko, kg = boot
    prm, g, cfg = P.prm, P.gpu, boot_cfg
    b = g.boot_create(prm.L, BOOT["K"], BOOT["r"], BOOT["n1"], BOOT["n2"], prm.scale)
    c = b.cfg()
    assert c["level"] == cfg["level"] and c["cts_scale"] == cfg["cts_scale"] and c["stc_scale"] == cfg["stc_scale"]
    assert np.allclose(c["poly"], cfg["poly"], rtol=1e-13, atol=1e-300)
    q0 = prm.primes[0]
    for w, nm in enumerate(("cts_re", "cts_im", "stc_re", "stc_im")):
        got = b.export(w)
        want = np.stack([np.stack(row) for row in cfg[nm]])
        assert got.shape == want.shape
        same = (got == want).all(axis=(2, 3))
        if same.all():
            continue
        gi = ckks.ntt_limbs(got[~same][:, :1], prm, [0], inverse=True)[:, 0].astype(object)
        wi = ckks.ntt_limbs(want[~same][:, :1], prm, [0], inverse=True)[:, 0].astype(object)
        d = (gi - wi) % q0
        d = np.where(d > q0 // 2, d - q0, d)
        wc = np.where(wi > q0 // 2, wi - q0, wi)
        # two double-precision FFTs of values up to max|w| agree to about 2^-46 max|w| (N = 2^12)
        tol = 1 + int(float(np.abs(wc).max()) * 2.0 ** -46)
        assert np.abs(d).max() <= tol, (nm, int(np.abs(d).max()), tol)
        if tol == 1:  # small coefficients: the two roundings differ only at rare near-ties
            assert np.count_nonzero(d) <= 5e-3 * got.shape[0] * got.shape[1] * prm.N, nm
    rng = np.random.default_rng(6)
    z = rng.uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 24, level=0)
    out = g.bootstrap_with(kg, P.up(ct), b)
    assert out.level == prm.L - plan.boot_depth(BOOT["r"])
    assert np.abs(g.decrypt(kg, out) - z).max() < 2 ** -12


FFT_GROUPS = [4, 4, 3]


@pytest.fixture(scope="module")
def boot_fft(S):
    P = pair(S, "boot")
    ev = ckks.Oracle(P.prm)
    rot = plan.fft_boot_rotations(P.prm.N, FFT_GROUPS)
    seed = synth.KEY_SEED_BASE + 29
    ko, kg = ev.keygen(seed, rot, h=BOOT["h"]), P.gpu.keygen(seed, rot, h=BOOT["h"])
    cfg = plan.fft_boot_config(ev, P.prm.scale, P.prm.L, BOOT["K"], BOOT["r"], FFT_GROUPS)
    return P, ev, ko, kg, cfg


@pytest.mark.gpu
@pytest.mark.slow
def test_bootstrap_fft_bit_exact(boot_fft):
    """R37: secpe_bootstrap_fft (special-FFT CoeffToSlot / SlotToCoeff in 3 + 3 hoisted diagonal transforms)
    is word for word the oracle's bootstrap_fft with the same op list; decrypts within 2^-12."""
    P, ev, ko, kg, cfg = boot_fft
    prm, g = P.prm, P.gpu
    z = np.random.default_rng(7).uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 25, level=0)
    ev.log.clear()
    want = plan.bootstrap_fft(ev, ko, ct, cfg)
    olog = list(ev.log)
    dev = lambda t: (t[0], torch.from_numpy(np.stack(t[1])).cuda(), t[2])
    g.oplog(enable=True, clear=True)
    got = g.bootstrap_fft(kg, P.up(ct), cfg["level"], cfg["K"], cfg["r"], cfg["poly"], [dev(t) for t in cfg["cts"]],
                          dev(cfg["cts_im"]), [dev(t) for t in cfg["stc"]], dev(cfg["stc_im"]))
    glog = g.oplog(enable=False, clear=True)
    assert glog == olog
    assert got.level == want.level == prm.L - plan.fft_boot_depth(FFT_GROUPS, BOOT["r"])
    assert got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    assert np.abs(g.decrypt(kg, got) - z).max() < 2 ** -12


@pytest.mark.gpu
@pytest.mark.slow
def test_boot_fft_setup_matches_oracle(boot_fft):
    """secpe_boot_create_fft: the library's own special-FFT factorisation has the oracle's steps per stage,
    pts equal up to FFT rounding (coefficients within 1 + 2^-46 max|c|), and bootstraps within 2^-12."""
    P, ev, ko, kg, cfg = boot_fft
    prm, g = P.prm, P.gpu
    b = g.boot_create_fft(prm.L, BOOT["K"], BOOT["r"], FFT_GROUPS, prm.scale)
    mc = len(FFT_GROUPS)
    base = prm.L - mc - 6 - BOOT["r"]
    cases = [(0, i, cfg["cts"][i], prm.L - i) for i in range(mc)] + [(1, 0, cfg["cts_im"], prm.L - mc + 1)]
    cases += [(2, i, cfg["stc"][i], base - i) for i in range(mc)] + [(3, 0, cfg["stc_im"], base)]
    q0 = prm.primes[0]
    for kind, idx, (steps, pts, sc), lv in cases:
        gs, gp = b.stage(kind, idx, lv)
        assert gs == list(steps), (kind, idx)
        want = np.stack(pts)
        same = (gp == want).all(axis=(1, 2))
        if same.all():
            continue
        gi = ckks.ntt_limbs(gp[~same][:, :1], prm, [0], inverse=True)[:, 0].astype(object)
        wi = ckks.ntt_limbs(want[~same][:, :1], prm, [0], inverse=True)[:, 0].astype(object)
        d = (gi - wi) % q0
        d = np.where(d > q0 // 2, d - q0, d)
        wc = np.where(wi > q0 // 2, wi - q0, wi)
        tol = 1 + int(float(np.abs(wc).max()) * 2.0 ** -46)
        assert np.abs(d).max() <= tol, (kind, idx, int(np.abs(d).max()), tol)
    z = np.random.default_rng(8).uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 26, level=0)
    out = g.bootstrap_boot(kg, P.up(ct), b)
    assert out.level == prm.L - plan.fft_boot_depth(FFT_GROUPS, BOOT["r"])
    assert np.abs(g.decrypt(kg, out) - z).max() < 2 ** -12


@pytest.mark.gpu
@pytest.mark.slow
def test_bootstrap_n16_refreshes(S):
    """N3 at the paper's ring, N = 2^16 (32768 slots): library-built factorised material (groups 5/5/5, baby-step
    giant-step form), sparse
    secret h = 64; the refreshed ciphertext decrypts to the input slots within 2^-11 (the oracle is too slow at
    this size for a word-for-word run; the N = 2^12 tests pin the same code path word for word)."""
    from paper_2502_00847_b200 import secpe
    g = secpe.Context(synth.PARAM_SETS["boot16"])
    groups, K, r = [5, 5, 5], 16, 7
    n = g.N // 2
    b = g.boot_create_fft(g.L, K, r, groups, g.scale, bsgs=True)
    kg = g.keygen(synth.KEY_SEED_BASE + 31, b.steps(), h=64)
    z = np.random.default_rng(9).uniform(-1, 1, n)
    ct = g.encrypt(kg, z, 0, g.scale, 27)
    out = g.bootstrap_boot(kg, ct, b)
    assert out.level == g.L - (2 * len(groups) + 6 + r)
    assert np.abs(g.decrypt(kg, out) - z).max() < 2 ** -11



@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("pname,groups", [("boot_argmax", [4, 4, 3]), ("boot_argmax_g4", [2, 3, 3, 3])])
def test_argmax_boot_k16_bit_exact(S, pname, groups):
    """N4 (reading R38): secpe_enc_argmax_boot_cfg with K = 16 (16 queries per ciphertext at N = 2^12, four
    bootstraps) is word for word the oracle's argmax_boot with the same op list, and every label is exact
    above the Sign margin.  Three stage groups, and four groups on a chain built like bench.py's
    boot_argmax16_g4 (two more bootstrap levels)."""
    P = pair(S, pname)
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    lay = synth.LAYOUTS["boot_k16"]
    st = load_sign("sign_7_15_15.json")
    rot = plan.argmax_rotations(lay) + plan.fft_boot_rotations(prm.N, groups)
    seed = synth.KEY_SEED_BASE + 37
    ko, kg = ev.keygen(seed, rot, h=64), g.keygen(seed, rot, h=64)
    bs = 2.0 ** 50
    cfg = plan.fft_boot_config(ev, bs, prm.L, 16, 7, groups)
    scores = synth.softmax_scores(41, lay["queries"], lay["prompts"], lay["classes"])
    ct = ev.encrypt(ko, plan.pack(scores, lay, prm.N // 2), prm.scale, 43, level=16)
    ev.log.clear()
    want = plan.argmax_boot(ev, ko, ct, lay, st, lambda c: plan.bootstrap_fft(ev, ko, c, cfg), bs)
    olog = list(ev.log)
    dev = lambda t: (t[0], torch.from_numpy(np.stack(t[1])).cuda(), t[2])
    fc = (cfg["level"], cfg["K"], cfg["r"], cfg["poly"], [dev(t) for t in cfg["cts"]], dev(cfg["cts_im"]),
          [dev(t) for t in cfg["stc"]], dev(cfg["stc_im"]))
    g.oplog(enable=True, clear=True)
    got = g.enc_argmax_boot(kg, P.up(ct), lay, st, None, bs, fft_cfg=fc)
    glog = g.oplog(enable=False, clear=True)
    assert glog == olog
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    dec = g.decrypt(kg, got)
    mean = scores.mean(axis=1)
    srt = np.sort(mean, axis=1)
    ok = srt[:, -1] - srt[:, -2] >= 2.0 ** -7
    assert ok.sum() >= 8
    assert (S.labels(dec, lay)[ok] == plan.true_labels(scores)[ok]).all()


@pytest.mark.gpu
@pytest.mark.slow
def test_argmax_boot_k16_n16(S):
    """N4 at the paper's ring: K = 16, 256 queries per ciphertext at N = 2^16 with library-built factorised
    bootstrap material (secpe_enc_argmax_boot); every label above the Sign margin is exact (property check:
    the oracle cannot run this size word for word; the N = 2^12 test pins the same plan)."""
    from paper_2502_00847_b200 import secpe
    g = secpe.Context(synth.PARAM_SETS["boot_argmax16"])
    lay = synth.LAYOUTS["argmax_k16"]
    st = load_sign("sign_7_15_15.json")
    bs = 2.0 ** 50
    b = g.boot_create_fft(g.L, 16, 7, [5, 5, 5], bs, bsgs=True)
    kg = g.keygen(synth.KEY_SEED_BASE + 39, sorted(set(plan.argmax_rotations(lay))) + b.steps(), h=64)
    sc2 = [synth.softmax_scores(47 + i, lay["queries"], lay["prompts"], lay["classes"]) for i in range(2)]
    cts = [g.encrypt(kg, plan.pack(sc, lay, g.N // 2), 16, g.scale, 49 + i) for i, sc in enumerate(sc2)]
    batch = S.Ct(torch.cat([c.t for c in cts]), 16, g.scale)
    out = g.enc_argmax_boot(kg, batch, lay, st, b, bs)
    # the batched plan (keys and transform plaintexts read once per op for both) gives the single-ciphertext words
    one = g.enc_argmax_boot(kg, cts[1], lay, st, b, bs)
    assert one.level == out.level and one.scale == out.scale
    assert torch.equal(one.t[0], out.t[1])
    for i, scores in enumerate(sc2):
        dec = g.decrypt(kg, out, i)
        mean = scores.mean(axis=1)
        srt = np.sort(mean, axis=1)
        ok = srt[:, -1] - srt[:, -2] >= 2.0 ** -7
        assert ok.sum() >= 200
        assert (S.labels(dec, lay)[ok] == plan.true_labels(scores)[ok]).all()


@pytest.fixture(scope="module")
def boot_fft_bsgs(S):
    P = pair(S, "boot")
    ev = ckks.Oracle(P.prm)
    rot = plan.fft_boot_rotations(P.prm.N, FFT_GROUPS, bsgs=True)
    seed = synth.KEY_SEED_BASE + 33
    ko, kg = ev.keygen(seed, rot, h=BOOT["h"]), P.gpu.keygen(seed, rot, h=BOOT["h"])
    cfg = plan.fft_boot_config(ev, P.prm.scale, P.prm.L, BOOT["K"], BOOT["r"], FFT_GROUPS, bsgs=True)
    return P, ev, ko, kg, cfg


def _dev_stage(t):
    if len(t) == 3:
        return (t[0], torch.from_numpy(np.stack(t[1])).cuda(), t[2])
    return (t[0], t[1], torch.from_numpy(np.stack([np.stack(r) for r in t[2]])).cuda(), t[3])


@pytest.mark.gpu
@pytest.mark.slow
def test_bootstrap_fft_bsgs_bit_exact(boot_fft_bsgs):
    """R39: the factorised bootstrap with every group in baby-step giant-step form (secpe_lt_stage with baby /
    giant steps; general giant steps incl. negative and zero) is word for word the oracle's, same op list."""
    P, ev, ko, kg, cfg = boot_fft_bsgs
    prm, g = P.prm, P.gpu
    z = np.random.default_rng(17).uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 35, level=0)
    ev.log.clear()
    want = plan.bootstrap_fft(ev, ko, ct, cfg)
    olog = list(ev.log)
    g.oplog(enable=True, clear=True)
    got = g.bootstrap_fft(kg, P.up(ct), cfg["level"], cfg["K"], cfg["r"], cfg["poly"],
                          [_dev_stage(t) for t in cfg["cts"]], _dev_stage(cfg["cts_im"]),
                          [_dev_stage(t) for t in cfg["stc"]], _dev_stage(cfg["stc_im"]))
    glog = g.oplog(enable=False, clear=True)
    assert glog == olog and any(l.startswith("LTG") for l in glog)
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    assert np.abs(g.decrypt(kg, got) - z).max() < 2 ** -12


@pytest.mark.gpu
@pytest.mark.slow
def test_boot_fft_bsgs_setup_matches_oracle(boot_fft_bsgs):
    """secpe_boot_create_fft(bsgs): the library's baby / giant steps equal the oracle's split, pts equal up to FFT
    rounding, secpe_boot_steps lists exactly the oracle's keys, and it bootstraps within 2^-12."""
    P, ev, ko, kg, cfg = boot_fft_bsgs
    prm, g = P.prm, P.gpu
    b = g.boot_create_fft(prm.L, BOOT["K"], BOOT["r"], FFT_GROUPS, prm.scale, bsgs=True)
    assert b.steps() == plan.fft_boot_rotations(prm.N, FFT_GROUPS, bsgs=True)
    mc = len(FFT_GROUPS)
    base = prm.L - mc - 6 - BOOT["r"]
    cases = [(0, i, cfg["cts"][i], prm.L - i) for i in range(mc)] + [(1, 0, cfg["cts_im"], prm.L - mc + 1)]
    cases += [(2, i, cfg["stc"][i], base - i) for i in range(mc)] + [(3, 0, cfg["stc_im"], base)]
    q0 = prm.primes[0]
    for kind, idx, (baby, giant, pts, sc), lv in cases:
        gb, gg, gp = b.stage_bsgs(kind, idx, lv)
        assert gb == list(baby) and gg == list(giant), (kind, idx)
        want = np.stack([np.stack(r) for r in pts]).reshape(-1, lv + 1, prm.N)
        gp = gp.reshape(-1, lv + 1, prm.N)
        same = (gp == want).all(axis=(1, 2))
        if same.all():
            continue
        gi = ckks.ntt_limbs(gp[~same][:, :1], prm, [0], inverse=True)[:, 0].astype(object)
        wi = ckks.ntt_limbs(want[~same][:, :1], prm, [0], inverse=True)[:, 0].astype(object)
        d = (gi - wi) % q0
        d = np.where(d > q0 // 2, d - q0, d)
        wc = np.where(wi > q0 // 2, wi - q0, wi)
        tol = 1 + int(float(np.abs(wc).max()) * 2.0 ** -46)
        assert np.abs(d).max() <= tol, (kind, idx, int(np.abs(d).max()), tol)
    z = np.random.default_rng(18).uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 36, level=0)
    out = g.bootstrap_boot(kg, P.up(ct), b)
    assert np.abs(g.decrypt(kg, out) - z).max() < 2 ** -12


@pytest.mark.gpu
@pytest.mark.slow
def test_argmax_boot_n256_bit_exact(S):
    """N4 large n (SURVEY 8(f) N4 "n = 256 with 64 per ciphertext"): 256 classes, eight Max steps
    and eight bootstraps per ciphertext; at N = 2^12 (4 queries per ciphertext) word for word the oracle's plan,
    labels exact above the margin."""
    P = pair(S, "boot_argmax")
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    lay = synth.LAYOUTS["boot_n256"]
    st = load_sign("sign_7_15_15.json")
    groups = [4, 4, 3]
    rot = plan.argmax_rotations(lay) + plan.fft_boot_rotations(prm.N, groups, bsgs=True)
    seed = synth.KEY_SEED_BASE + 41
    ko, kg = ev.keygen(seed, rot, h=64), g.keygen(seed, rot, h=64)
    bs = 2.0 ** 50
    cfg = plan.fft_boot_config(ev, bs, prm.L, 16, 7, groups, bsgs=True)
    scores = synth.softmax_scores(51, lay["queries"], lay["prompts"], lay["classes"], sigma=6.0)
    ct = ev.encrypt(ko, plan.pack(scores, lay, prm.N // 2), prm.scale, 53, level=16)
    nb = [0]

    def boot(c):
        nb[0] += 1
        return plan.bootstrap_fft(ev, ko, c, cfg)
    want = plan.argmax_boot(ev, ko, ct, lay, st, boot, bs)
    assert nb[0] == 8
    fc = (cfg["level"], cfg["K"], cfg["r"], cfg["poly"], [_dev_stage(t) for t in cfg["cts"]],
          _dev_stage(cfg["cts_im"]), [_dev_stage(t) for t in cfg["stc"]], _dev_stage(cfg["stc_im"]))
    got = g.enc_argmax_boot(kg, P.up(ct), lay, st, None, bs, fft_cfg=fc)
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    mean = scores.mean(axis=1)
    srt = np.sort(mean, axis=1)
    ok = srt[:, -1] - srt[:, -2] >= 2.0 ** -7
    assert ok.sum() >= 2
    assert (S.labels(g.decrypt(kg, got), lay)[ok] == plan.true_labels(scores)[ok]).all()


def _pack_groups(scores, lay, n_slots, pc):
    """Prompt groups: member i holds prompts i * P .. i * P + P - 1 of every query (same layout)."""
    P = lay["prompts"]
    return [plan.pack(scores[:, i * P:(i + 1) * P], lay, n_slots) for i in range(pc)]


@pytest.mark.gpu
@pytest.mark.slow
def test_argmax_boot_clip_prompt_groups_bit_exact(S):
    """N4 CLIP scale: 1024 classes, 6 prompts spread over 3 ciphertexts (prompt_cts = 3)
    summed first, ten bootstraps per query set; at N = 2^12 word for word the oracle's plan, label exact."""
    P = pair(S, "boot_argmax")
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    lay = synth.LAYOUTS["boot_clip"]
    pc = 3
    st = load_sign("sign_7_15_15.json")
    groups = [4, 4, 3]
    rot = plan.argmax_rotations(lay) + plan.fft_boot_rotations(prm.N, groups, bsgs=True)
    seed = synth.KEY_SEED_BASE + 43
    ko, kg = ev.keygen(seed, rot, h=64), g.keygen(seed, rot, h=64)
    bs = 2.0 ** 50
    cfg = plan.fft_boot_config(ev, bs, prm.L, 16, 7, groups, bsgs=True)
    scores = synth.softmax_scores(55, lay["queries"], lay["prompts"] * pc, lay["classes"], sigma=6.0)
    cts = [ev.encrypt(ko, z, prm.scale, 60 + i, level=16) for i, z in enumerate(_pack_groups(scores, lay, prm.N // 2, pc))]
    nb = [0]

    def boot(c):
        nb[0] += 1
        return plan.bootstrap_fft(ev, ko, c, cfg)
    ev.log.clear()
    want = plan.argmax_boot(ev, ko, cts, lay, st, boot, bs, prompt_cts=pc)
    olog = list(ev.log)
    assert nb[0] == 10
    fc = (cfg["level"], cfg["K"], cfg["r"], cfg["poly"], [_dev_stage(t) for t in cfg["cts"]],
          _dev_stage(cfg["cts_im"]), [_dev_stage(t) for t in cfg["stc"]], _dev_stage(cfg["stc_im"]))
    batch = S.Ct(torch.from_numpy(np.stack([c.data for c in cts])).cuda(), 16, prm.scale)
    g.oplog(enable=True, clear=True)
    got = g.enc_argmax_boot(kg, batch, lay, st, None, bs, fft_cfg=fc, prompt_cts=pc)
    glog = g.oplog(enable=False, clear=True)
    assert glog == olog
    assert got.n == 1 and got.level == want.level and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    mean = scores.mean(axis=1)
    srt = np.sort(mean, axis=1)
    assert srt[0, -1] - srt[0, -2] >= 2.0 ** -7
    assert S.labels(g.decrypt(kg, got), lay)[0] == plan.true_labels(scores)[0]


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("groups", [[5, 5, 5], [4, 5, 6]])
def test_bootstrap_n16_bit_exact(S, groups):
    """N3 at full size (N = 2^16, 32768 slots, groups 5/5/5 and bench.py's 4/5/6, in baby-step giant-step form):
    the GPU bootstrap with the oracle's encoded material is word for word the oracle's (about two minutes of
    oracle time each), same op list, refresh within 2^-11."""
    P = pair(S, "boot16")
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    rot = plan.fft_boot_rotations(prm.N, groups, bsgs=True)
    seed = synth.KEY_SEED_BASE + 47
    ko, kg = ev.keygen(seed, rot, h=64), g.keygen(seed, rot, h=64)
    z = np.random.default_rng(21).uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 71, level=0)
    cfg = plan.fft_boot_config(ev, prm.scale, prm.L, 16, 7, groups, bsgs=True)
    ev.log.clear()
    want = plan.bootstrap_fft(ev, ko, ct, cfg)
    olog = list(ev.log)
    g.oplog(enable=True, clear=True)
    got = g.bootstrap_fft(kg, P.up(ct), cfg["level"], cfg["K"], cfg["r"], cfg["poly"],
                          [_dev_stage(t) for t in cfg["cts"]], _dev_stage(cfg["cts_im"]),
                          [_dev_stage(t) for t in cfg["stc"]], _dev_stage(cfg["stc_im"]))
    glog = g.oplog(enable=False, clear=True)
    assert glog == olog
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    assert np.abs(g.decrypt(kg, got) - z).max() < 2 ** -11


@pytest.mark.gpu
def test_bootstrap_api_errors(S):
    """Argument checks of the bootstrapping entry points: stage groups that do not cover log2(N/2), a
    non-level-0 input, a missing Galois key, prompt groups that do not divide the batch, too few levels."""
    P = pair(S, "boot")
    g = P.gpu
    with pytest.raises(S.SecpeError):
        g.boot_create_fft(g.L, 16, 7, [4, 4], g.scale, bsgs=True)      # 8 of 11 stages
    with pytest.raises(S.SecpeError):
        g.boot_create_fft(g.L, 16, 7, [4, 4, 3, 0], g.scale)           # empty group
    with pytest.raises(S.SecpeError):
        g.boot_create_fft(10, 16, 7, [4, 4, 3], g.scale)               # depth 19 > level 10
    with pytest.raises(S.SecpeError):
        g.boot_create(g.L, 16, 7, 64, 16, g.scale)                      # n1 n2 != N/2
    b = g.boot_create_fft(g.L, 16, 7, [4, 4, 3], g.scale, bsgs=True)
    steps = b.steps()
    assert steps[-1] == S.CONJ and len(set(steps)) == len(steps)
    kg = g.keygen(3, steps, h=64)
    z = np.zeros(g.N // 2)
    with pytest.raises(S.SecpeError):
        g.bootstrap_boot(kg, g.encrypt(kg, z, 1, g.scale, 1), b)        # level 1, not 0
    with pytest.raises(S.SecpeError):
        g.bootstrap_boot(g.keygen(3, steps[:-1], h=64), g.encrypt(kg, z, 0, g.scale, 2), b)  # no conj key
    out = g.bootstrap_boot(kg, g.encrypt(kg, z, 0, g.scale, 3), b)
    assert out.level == g.L - (2 * 3 + 6 + 7)
    lay = synth.LAYOUTS["boot_k16"]
    st = load_sign("sign_7_15_15.json")
    two = S.Ct(torch.cat([g.encrypt(kg, z, 16, g.scale, 4).t] * 3), 16, g.scale)
    with pytest.raises((S.SecpeError, AssertionError)):
        g.enc_argmax_boot(kg, two, lay, st, b, 2.0 ** 50, prompt_cts=2)   # 3 ciphertexts, groups of 2


def test_bsgs_split_rejects_gaps():
    """R39's split needs a contiguous progression of offsets (every merged special-FFT group has one)."""
    n = 64
    D = {0: np.ones(n), 2: np.ones(n), 6: np.ones(n)}
    with pytest.raises(ValueError):
        plan.bsgs_split(D, n)


@pytest.mark.gpu
def test_bootstrap_graph_replay_and_material_destroy(S):
    """secpe_bootstrap_boot on a non-default stream with the same buffers: eager first, captured CUDA graph
    replayed afterwards -- word for word the eager result; destroying the material drops the graph, so new
    material (possibly at the same address) is used, not the old graph."""
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        g = S.Context(synth.PARAM_SETS["boot"], stream=stream.cuda_stream)
        b = g.boot_create_fft(g.L, 16, 7, [4, 4, 3], g.scale, bsgs=True)
        kg = g.keygen(9, b.steps(), h=64)
        z = np.random.default_rng(2).uniform(-1, 1, g.N // 2)
        c0 = g.new_ct(0)
        g.encrypt_coeffs(kg, g.encode(z, g.scale), 0, g.scale, 3, out=c0)
        c0.level, c0.scale = 0, g.scale
        out = g.new_ct(g.L - (2 * 3 + 6 + 7))
        g.bootstrap_boot(kg, c0, b, out=out)
        stream.synchronize()
        first = out.t.cpu().numpy().copy()
        for _ in range(3):
            out.t.zero_()
            g.bootstrap_boot(kg, c0, b, out=out)
            stream.synchronize()
            assert np.array_equal(out.t.cpu().numpy(), first)
        assert np.abs(g.decrypt(kg, out) - z).max() < 2 ** -12
        del b
        b2 = g.boot_create_fft(g.L, 16, 7, [4, 4, 3], g.scale, bsgs=True)   # same shapes, fresh material
        for _ in range(3):
            g.bootstrap_boot(kg, c0, b2, out=out)
            stream.synchronize()
        assert np.abs(g.decrypt(kg, out) - z).max() < 2 ** -12


@pytest.mark.gpu
def test_bootstrap_batch_equals_single(S):
    """secpe_bootstrap_boot_batch: three ciphertexts through one plan give, word for word, the three
    single-ciphertext bootstraps."""
    P = pair(S, "boot")
    g = P.gpu
    b = g.boot_create_fft(g.L, 16, 7, [4, 4, 3], g.scale, bsgs=True)
    kg = g.keygen(11, b.steps(), h=64)
    zs = [np.random.default_rng(30 + i).uniform(-1, 1, g.N // 2) for i in range(3)]
    cts = [g.encrypt(kg, z, 0, g.scale, 40 + i) for i, z in enumerate(zs)]
    batch = S.Ct(torch.cat([c.t for c in cts]), 0, g.scale)
    out = g.bootstrap_boot(kg, batch, b)
    for i, c in enumerate(cts):
        one = g.bootstrap_boot(kg, c, b)
        assert one.level == out.level and one.scale == out.scale
        assert torch.equal(one.t[0], out.t[i])
        assert np.abs(g.decrypt(kg, out, i) - zs[i]).max() < 2 ** -12


@pytest.mark.gpu
@pytest.mark.slow
def test_bootstrap_fft_bsgs_four_groups_bit_exact(S):
    """R37 + R39 with four stage groups (2/3/3/3 at N = 2^12, the shape of bench.py's 3/4/4/4 at N = 2^16):
    word for word the oracle's bootstrap with the same op list; the library-built material bootstraps within
    2^-12 and its rotation steps are the oracle's."""
    P = pair(S, "boot_g4")
    prm, g = P.prm, P.gpu
    ev = ckks.Oracle(prm)
    groups = [2, 3, 3, 3]
    rot = plan.fft_boot_rotations(prm.N, groups, bsgs=True)
    seed = synth.KEY_SEED_BASE + 53
    ko, kg = ev.keygen(seed, rot, h=64), g.keygen(seed, rot, h=64)
    cfg = plan.fft_boot_config(ev, prm.scale, prm.L, 16, 7, groups, bsgs=True)
    z = np.random.default_rng(23).uniform(-1, 1, prm.N // 2)
    ct = ev.encrypt(ko, z, prm.scale, 37, level=0)
    ev.log.clear()
    want = plan.bootstrap_fft(ev, ko, ct, cfg)
    olog = list(ev.log)
    g.oplog(enable=True, clear=True)
    got = g.bootstrap_fft(kg, P.up(ct), cfg["level"], cfg["K"], cfg["r"], cfg["poly"],
                          [_dev_stage(t) for t in cfg["cts"]], _dev_stage(cfg["cts_im"]),
                          [_dev_stage(t) for t in cfg["stc"]], _dev_stage(cfg["stc_im"]))
    glog = g.oplog(enable=False, clear=True)
    assert glog == olog
    assert got.level == want.level == prm.L - plan.fft_boot_depth(groups, 7) and got.scale == want.scale
    assert np.array_equal(P.down(got), want.data)
    assert np.abs(g.decrypt(kg, got) - z).max() < 2 ** -12
    b = g.boot_create_fft(prm.L, 16, 7, groups, prm.scale, bsgs=True)
    assert b.steps() == rot
    out = g.bootstrap_boot(kg, P.up(ct), b)
    assert np.abs(g.decrypt(kg, out) - z).max() < 2 ** -12


@pytest.mark.gpu
def test_bootstrap_batch_stream_capture_replay(S):
    """secpe_bootstrap_boot_batch on a non-default stream with the same buffers called four times (eager,
    capture, replay, replay) on three DISTINCT ciphertexts: every output, every time, equals the
    single-ciphertext bootstrap of its own input word for word (a per-ciphertext stride or graph-replay bug
    would show up here)."""
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        g = S.Context(synth.PARAM_SETS["boot"], stream=stream.cuda_stream)
        groups = [4, 4, 3]
        b = g.boot_create_fft(g.L, 16, 7, groups, g.scale, bsgs=True)
        kg = g.keygen(13, b.steps(), h=64)
        n = 3
        zs = [np.random.default_rng(60 + i).uniform(-1, 1, g.N // 2) for i in range(n)]
        cb = g.new_ct(0, n)
        for i, z in enumerate(zs):
            g.encrypt_coeffs(kg, g.encode(z, g.scale), 0, g.scale, 50 + i, out=S.Ct(cb.t[i:i + 1], 0, g.scale))
        cb.level, cb.scale = 0, g.scale
        ol = g.L - plan.fft_boot_depth(groups, 7)
        singles = []
        for i in range(n):
            o1 = g.bootstrap_boot(kg, S.Ct(cb.t[i:i + 1].clone(), 0, g.scale), b)
            stream.synchronize()
            singles.append(o1.t[0].cpu().numpy().copy())
        out = g.new_ct(ol, n)
        for rep in range(4):
            out.t.zero_()
            g.bootstrap_boot(kg, cb, b, out=out)
            stream.synchronize()
            got = out.t.cpu().numpy()
            for i in range(n):
                assert np.array_equal(got[i], singles[i]), (rep, i)
        for i in range(n):
            assert np.abs(g.decrypt(kg, out, i) - zs[i]).max() < 2 ** -12


@pytest.mark.gpu
def test_batch_overlap_rejected(S):
    """An output batch that overlaps the input batch without sharing a start pointer is rejected (byte-range
    check) by secpe_bootstrap_boot_batch and secpe_enc_argmax."""
    g = S.Context(synth.PARAM_SETS["boot"])
    b = g.boot_create_fft(g.L, 16, 7, [4, 4, 3], g.scale, bsgs=True)
    kg = g.keygen(15, b.steps(), h=64)
    cb = g.new_ct(0, 2)
    cb.level, cb.scale = 0, g.scale
    ol = g.L - plan.fft_boot_depth([4, 4, 3], 7)
    words0 = cb.t[0].numel()
    big = torch.zeros(2 * g.new_ct(ol, 1).t[0].numel() + 2 * words0, dtype=torch.uint64, device="cuda")
    ins = big[words0: 3 * words0].view(2, *cb.t.shape[1:])      # inputs start one ciphertext into the buffer
    outs = big[:2 * g.new_ct(ol, 1).t[0].numel()].view(2, *g.new_ct(ol, 1).t.shape[1:])
    with pytest.raises(S.SecpeError):
        g.bootstrap_boot(kg, S.Ct(ins, 0, g.scale), b, out=S.Ct(outs, ol, g.scale))
    P = pair(S, "toy_argmax")
    gp = P.gpu
    lay = synth.LAYOUTS["toy"]
    st = load_sign("sign_f1_f1.json")
    kk = gp.keygen(17, plan.argmax_rotations(lay))
    x = gp.new_ct(gp.L, 2)
    x.level, x.scale = gp.L, gp.scale
    ol2, _ = gp.argmax_info(lay, st, gp.L)
    o = S.Ct(x.t.view(-1)[x.t[0].numel() // 2:][: 2 * gp.new_ct(ol2, 1).t[0].numel()].view(
        2, *gp.new_ct(ol2, 1).t.shape[1:]), ol2, gp.scale)
    with pytest.raises(S.SecpeError):
        gp.enc_argmax(kk, x, lay, st, out=o)


@pytest.mark.gpu
@pytest.mark.slow
def test_argmax_boot_bench_config_n16(S):
    """bench.py's N4 row exactly: boot_argmax16_g4 chain, four stage groups 3/4/4/4, K = 16, 8 distinct
    ciphertexts per call (256 queries each).  Every label above the Sign margin is exact for every
    ciphertext, and ciphertext 5 of the batch equals its single-ciphertext run word for word (property check:
    the oracle cannot run this size; test_argmax_boot_k16_bit_exact pins the four-group plan at N = 2^12)."""
    g = S.Context(synth.PARAM_SETS["boot_argmax16_g4"])
    lay = synth.LAYOUTS["argmax_k16"]
    st = load_sign("sign_7_15_15.json")
    bs = 2.0 ** 50
    groups = [3, 4, 4, 4]
    b = g.boot_create_fft(g.L, 16, 7, groups, bs, bsgs=True)
    assert g.L - plan.fft_boot_depth(groups, 7) == 16
    kg = g.keygen(synth.KEY_SEED_BASE + 39, sorted(set(plan.argmax_rotations(lay))) + b.steps(), h=64)
    B = 8
    scs = [synth.softmax_scores(47 + i, lay["queries"], lay["prompts"], lay["classes"]) for i in range(B)]
    cts = [g.encrypt(kg, plan.pack(sc, lay, g.N // 2), 16, g.scale, 49 + i) for i, sc in enumerate(scs)]
    batch = S.Ct(torch.cat([c.t for c in cts]), 16, g.scale)
    out = g.enc_argmax_boot(kg, batch, lay, st, b, bs)
    one = g.enc_argmax_boot(kg, cts[5], lay, st, b, bs)
    assert one.level == out.level and one.scale == out.scale
    assert torch.equal(one.t[0], out.t[5])
    for i, scores in enumerate(scs):
        dec = g.decrypt(kg, out, i)
        mean = scores.mean(axis=1)
        srt = np.sort(mean, axis=1)
        ok = srt[:, -1] - srt[:, -2] >= 2.0 ** -7
        assert ok.sum() >= 180
        assert (S.labels(dec, lay)[ok] == plan.true_labels(scores)[ok]).all(), i


@pytest.mark.gpu
def test_keygen_os_entropy_and_seed_modes(S):
    """Reading R6: seed=None draws the 256-bit master seed from OS entropy (two unseeded keygens differ and
    still decrypt); an explicit 32-byte seed is deterministic and equals the oracle's keys; the integer
    (test-only) mode is the 32-byte seed LE64(s) || 0^24."""
    P = pair(S, "toy")
    g, ev = P.gpu, ckks.Oracle(P.prm)
    k1, k2 = g.keygen(None), g.keygen(None)
    assert not np.array_equal(k1.export(0), k2.export(0))
    z = np.random.default_rng(4).uniform(-1, 1, g.N // 2)
    for k in (k1, k2):
        assert np.abs(g.decrypt(k, g.encrypt(k, z, g.L, g.scale, None)) - z).max() < 2 ** -20
    raw = bytes(range(7, 39))
    kb, ko = g.keygen(raw), ev.keygen(raw)
    assert np.array_equal(kb.export(0), ko.s_ntt) and np.array_equal(kb.export(1), ko.pk)
    s = 0x0123456789ABCDEF
    assert np.array_equal(g.keygen(s).export(0), g.keygen(s.to_bytes(8, "little") + bytes(24)).export(0))


@pytest.mark.gpu
def test_fused_ntt_matches_two_pass_and_oracle(S):
    """The persistent TMA-pipelined NTT (ntt_fused.cu, secpe_ntt_mode 1) against the two-pass kernels (mode 0) on
    the configs[4] exact-FP64 rows: plain forward / inverse transforms of ragged shapes (1 .. 1856 limb rows,
    offset limbs, special primes, worst-case all-(q-1) input) give identical words and equal the oracle on
    sampled limbs; the fused prologues / epilogues (relinearise-and-rescale, rescale, rotation, whole argmax)
    give identical ciphertexts."""
    P = pair(S, "argmax")
    prm, g = P.prm, P.gpu
    prev = S.ntt_mode(-1)
    try:
        for n_polys, first, n_limbs in ((1, 3, 1), (3, 0, 7), (2, 25, 15), (64, 1, 29)):
            primes = prm.primes[first:first + n_limbs]
            x = synth.uniform_residues(300 + n_polys, primes, n_polys, prm.logn)
            if n_polys == 3:
                x[1] = np.array(primes, dtype=np.uint64)[:, None] - np.uint64(1)
            outs = {}
            for mode in (0, 1):
                S.ntt_mode(mode)
                t = torch.from_numpy(x.copy()).cuda()
                g.ntt(t, first, n_limbs)
                f = t.cpu().numpy()
                g.ntt(t, first, n_limbs, inverse=True)
                outs[mode] = (f, t.cpu().numpy())
            assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
            assert np.array_equal(outs[1][1], x)
            pi, l = n_polys - 1, n_limbs - 1
            assert np.array_equal(outs[1][0][pi, l], ckks.ntt(x[pi, l], primes[l], prm.psi[first + l], prm.logn))
        # fused prologue / epilogue modes inside the evaluator: word-for-word equal under both implementations
        lay = synth.LAYOUTS["argmax_k2"]
        st = load_sign("sign_7_15_15.json")
        kg = g.keygen(synth.KEY_SEED_BASE + 61, plan.argmax_rotations(lay))
        cts = []
        for i in range(2):
            sc = synth.softmax_scores(600 + i, lay["queries"], lay["prompts"], lay["classes"])
            cts.append(g.encrypt(kg, plan.pack(sc, lay, g.N // 2), g.L, g.scale, 610 + i))
        res = {}
        for mode in (0, 1):
            S.ntt_mode(mode)
            a, b = cts
            m = g.mul_relin_rescale(kg, a, b)
            r = g.rotate(kg, a, 2)
            rs = g.rescale(a)
            batch = S.Ct(torch.cat([c.t for c in cts]), g.L, g.scale)
            am = g.enc_argmax(kg, batch, lay, st)
            torch.cuda.synchronize()
            res[mode] = [x.t.cpu().numpy() for x in (m, r, rs, am)]
        for u, v in zip(res[0], res[1]):
            assert np.array_equal(u, v)
    finally:
        S.ntt_mode(prev)
