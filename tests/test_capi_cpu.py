"""C ABI checks that need no GPU: both shared libraries build and load, every symbol the
header declares is exported, host-only entry points agree with the oracle, and the compute
entry points fail loudly (no CPU fallback) when no device is present."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "benelux_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"BNX_API\s+[\w\s\*]+?\b(bnx_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2506_01099_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    return _native.load()


def test_header_declares_the_documented_entry_points():
    syms = declared_symbols()
    for name in ("bnx_search", "bnx_search_domain", "bnx_sieve_radicals", "bnx_primes_up_to",
                 "bnx_radicals_trial_division", "bnx_slot_of", "bnx_ctx_create"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2506_01099_b200 import _native

    syms = declared_symbols()
    assert set(syms) == set(_native.EXPORTED_SYMBOLS)
    for name in syms:
        assert hasattr(lib, name), name


def test_no_torch_or_cuda_types_in_the_abi():
    text = open(HEADER).read()
    assert "torch" not in text.split("*/", 1)[1]
    assert "cudaStream_t" not in text.split("*/", 1)[1]


def test_version_and_host_hash(lib, golden):
    assert lib.bnx_version() == 10000
    from oracle import oracle as orc

    for lo, hi, size, slot in golden["commutative_hash"][:60]:
        assert lib.bnx_slot_of(lo, hi, size - 1, *orc.HASH_CONSTANTS) == slot


def test_compute_entry_points_fail_loudly_without_a_gpu(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2506_01099_b200 as bp
    from paper_2506_01099_b200 import _native

    n = ctypes.c_int(-1)
    assert lib.bnx_device_count(ctypes.byref(n)) != 0 and n.value == 0
    h = ctypes.c_void_p()
    assert lib.bnx_ctx_create(0, ctypes.byref(h)) == _native.BNX_ERR_CUDA
    with pytest.raises(_native.CudaError):
        bp.find_pairs_sorted(100)
    with pytest.raises(_native.CudaError):
        bp.sieve_radicals(bp.Interval(1, 10))


def test_oracle_library_builds_and_loads(orc):
    assert orc.lib().orc_num_chunks(2**32, 2**27) == 33
