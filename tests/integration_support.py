"""Load integration/benelux_pairs_b200.py (the reference-side binding) the way the reference
would: with the reference's own `benelux_pairs.signatures` types.  Where /root/reference is
absent (the GPU box), a minimal stand-in package with the reference's result types
(signatures.py:14-64: Kind, BeneluxPair) is written to a temporary directory instead."""
import importlib.util
import os
import sys
from dataclasses import dataclass

from conftest import ROOT

REF_SRC = "/root/reference/pkg/src"

STANDIN_SIGNATURES = '''
from dataclasses import dataclass
from enum import IntEnum


class Kind(IntEnum):
    FIRST = 1
    SECOND = 2


@dataclass(frozen=True)
class BeneluxPair:
    m: int
    n: int
    kind: Kind
    rad_m: int
    rad_m_plus_1: int

    def __post_init__(self):
        if not 0 < self.m < self.n:
            raise ValueError("need 0 < m < n")
'''


@dataclass(frozen=True)
class PrimeListStandIn:
    """The two attributes of the reference's PrimeList (primes.py:10-21) the binding reads."""
    primes: object
    limit: int


def load(tmp_dir: str):
    """(binding module, the `benelux_pairs.signatures` module it returns types of, is_real_reference)."""
    real = os.path.isdir(os.path.join(REF_SRC, "benelux_pairs"))
    if "benelux_pairs" not in sys.modules:
        if real:
            sys.path.insert(0, REF_SRC)
        else:
            pkg = os.path.join(tmp_dir, "benelux_pairs")
            os.makedirs(pkg, exist_ok=True)
            open(os.path.join(pkg, "__init__.py"), "w").close()
            with open(os.path.join(pkg, "signatures.py"), "w") as f:
                f.write(STANDIN_SIGNATURES)
            sys.path.insert(0, tmp_dir)
    import benelux_pairs.signatures as sig

    path = os.path.join(ROOT, "integration", "benelux_pairs_b200.py")
    spec = importlib.util.spec_from_file_location("benelux_pairs_b200", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod, sig, real and sig.__file__.startswith(REF_SRC)
