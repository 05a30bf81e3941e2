"""CPU checks of the C-ABI library: it loads, exports every symbol include/crksr.h
declares, and validates parameters before touching the device."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2310_16122_b200 import build as b

    return b.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "crksr.h")).read()
    return sorted(set(re.findall(r"\b(crk_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (crk_\w+)", out))
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    from paper_2310_16122_b200 import EXPORTS

    assert sorted(EXPORTS) == declared


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_parameter_validation_without_gpu(libpath):
    from gen.configs import make_params
    from paper_2310_16122_b200.binding import lib, params_struct

    good = make_params([16.0, 16.0, 16.0])
    bad_cases = [
        dict(good, box=[12.0, 16.0, 16.0]),   # not a power of two
        dict(good, rcut2=25.0),               # rcut >= box/4
        dict(good, eps2=0.0),                 # softening must be positive
        dict(good, leaf_max_i=48),            # not a compiled leaf size
        dict(good, leaf_max_j=16),
        dict(good, cell_side=8.0),            # > box/4
        dict(good, leaf_max_gas_i=128),
    ]
    for p in bad_cases:
        h = C.c_void_p()
        st = lib().crk_create(C.byref(params_struct(p)), 0, C.byref(h))
        assert st == -1, p
    assert lib().crk_status_string(-4) == b"call order violated"


def test_exchange_calls_reject_bad_arguments_without_gpu(libpath):
    """The weak-scaling exchange calls validate their arguments before touching the device
    (CRK_EINVAL = -1): no context, no masks or counts, peer / set numbers out of range."""
    from paper_2310_16122_b200.binding import CrkParticles, lib

    L = lib()
    vp = C.c_void_p
    p = CrkParticles()
    assert L.crk_select_peers_dev(None, vp(), vp(), vp(), vp(), 10, vp(), 2, vp(), 10, vp(), None) == -1
    assert L.crk_select_gas_multi_dev(None, vp(), 2, vp(), 10, vp(), None) == -1
    assert L.crk_compact_own(None, C.byref(p), 0, C.byref(p), None) == -1
