"""Host-side checks of the C-ABI library that need no GPU: the shared object loads, exports every
symbol include/secpe.h declares, its host prime generator agrees with the oracle's, and compute
entry points fail loudly (no CPU fallback) when no CUDA device is present."""
import ctypes
import os
import re

import pytest
import torch

import synth
from oracle import ckks
from paper_2502_00847_b200 import secpe

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    from paper_2502_00847_b200 import build
    build.build()
    return secpe.lib()


def header_symbols():
    h = open(os.path.join(ROOT, "include", "secpe.h")).read()
    return sorted(set(re.findall(r"\b(secpe_[a-z_0-9]+)\s*\(", h)))


def test_exports_every_header_symbol(built):
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(built, s), s
    assert set(syms) == set(secpe.EXPORTS)


def test_north_star_entry_points_declared():
    syms = header_symbols()
    for name in ["secpe_keygen", "secpe_encrypt", "secpe_decrypt", "secpe_ntt", "secpe_intt", "secpe_mul_relin",
                 "secpe_rescale", "secpe_rotate", "secpe_sign_poly", "secpe_enc_argmax"]:
        assert name in syms


@pytest.mark.parametrize("name", ["toy", "toy_argmax", "ks", "argmax", "ntt"])
def test_library_primes_equal_oracle(built, name):
    d = synth.PARAM_SETS[name]
    q, p = secpe.primes_for(d)
    assert q + p == ckks.Params(d).primes


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device error path")
def test_no_device_fails_loudly(built):
    q, p = secpe.primes_for(synth.PARAM_SETS["toy"])
    with pytest.raises(secpe.SecpeError, match="no CUDA device"):
        secpe.Context(q=q, p=p, logn=12, alpha=1, scale=2.0 ** 40, stream=0)


def test_errors_are_codes_not_crashes(built):
    out = (ctypes.c_uint64 * 1)()
    assert built.secpe_gen_primes(5, 1, 12, 0, None, 0, out) == -1
    assert b"bad prime" in built.secpe_last_error()
