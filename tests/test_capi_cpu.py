"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only entry points (probes, seed mixing) match
the oracle bitwise.  No device compute here."""
import ctypes as C

import numpy as np
import pytest

from paper_2107_00243_b200 import capi, gpkrylov


def test_library_exports_every_header_symbol():
    lib = capi.lib()
    names = capi.header_functions()
    assert len(names) >= 24
    for name in names:
        assert hasattr(lib, name), name
        assert name in capi.SIGNATURES, f"{name} has no ctypes signature"


def test_version_string():
    assert b"sm_100a" in capi.lib().gpk_version()


def test_make_probes_bitwise_vs_oracle(orc):
    for n, l, seed in [(1, 1, 0), (37, 3, 17), (2048, 8, orc.mix_seed(17, 1))]:
        z = gpkrylov.make_probes(n, l, seed).probes
        assert np.array_equal(z, orc.make_probes(n, l, seed))


def test_mix_seed_matches_oracle(orc):
    for s, t in [(17, 1), (0, 0), (12345, 0xB2D), (2**64 - 1, 7)]:
        assert gpkrylov.mix_seed(s, t) == orc.mix_seed(s, t)


def test_probe_input_errors():
    with pytest.raises(gpkrylov.InputError):
        gpkrylov.make_probes(0, 3, 1)
    with pytest.raises(gpkrylov.InputError):
        gpkrylov.make_probes(5, 0, 1)


def test_status_codes_match_exception_types():
    # common.hpp:19-35 mapping
    assert gpkrylov.InputError.status == 1
    assert gpkrylov.NumericalError.status == 2
    assert gpkrylov.SolverError.status == 3 and issubclass(gpkrylov.SolverError, gpkrylov.NumericalError)


def test_struct_layouts_match_header():
    # gpk_mll_result: 19 fields; pointers and doubles aligned to 8
    r = capi.gpk_mll_result()
    assert C.sizeof(r) % 8 == 0
    assert C.sizeof(capi.gpk_cg_cfg) == 32
    assert C.sizeof(capi.gpk_mll_cfg) == 48
