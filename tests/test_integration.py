"""The reference-side binding (integration/benelux_pairs_b200.py) on CPU: it imports with the
reference's own result types (the real `benelux_pairs` when /root/reference is present, else
the stand-in) and binds every C-ABI entry point it calls; no device work."""
import pytest

import integration_support as sup


def test_binding_loads_and_binds(tmp_path):
    mod, sig, _real = sup.load(str(tmp_path))
    assert mod.BeneluxPair is sig.BeneluxPair and mod.Kind is sig.Kind
    lib = mod.library()
    for name, (args, res) in mod.SIGNATURES.items():
        fn = getattr(lib, name)
        assert fn.argtypes == args and fn.restype == res


def test_binding_argument_checks(tmp_path):
    mod, _, _ = sup.load(str(tmp_path))
    with pytest.raises(ValueError):
        list(mod.run_full_chunked(2, 100))
    with pytest.raises(ValueError):
        list(mod.run_full_chunked(100, 2))
    with pytest.raises(ValueError):
        mod.search_chunk(0, 2)
    assert mod._chunk_domain(0, 1300) == (1, 1299) and mod._chunk_domain(3, 100) == (298, 396)
