"""The C-ABI library loads and exports every symbol include/parsmc_b200.h
declares (no GPU needed; no compute calls)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "parsmc_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for must in ("pf_engine_create", "pf_engine_run", "pf_engine_destroy", "pf_tree_cdf",
                 "pf_cut_table", "pf_cutpoint_lookup", "pf_resample_cutpoint",
                 "pf_uniforms_at", "pf_weighted_quantiles"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_ctypes_signatures_cover_header(lib):
    from paper_1212_1639_b200 import _lib

    assert set(header_symbols()) == set(_lib.SIGNATURES)


def test_version_and_device_count_without_compute(lib):
    assert b"sm_100a" in lib.pf_version()
    assert lib.pf_device_count() >= 0
    assert lib.pf_launch_count() >= 0


def test_struct_layouts_match_header(lib):
    """pf_config / pf_outputs / pf_feed: the ctypes mirrors have the sizes the
    compiled library reports (pf_abi_sizes), and the expected field count."""
    from paper_1212_1639_b200 import _lib

    sizes = (_lib.C.c_int64 * 3)()
    assert lib.pf_abi_sizes(sizes) == 0
    assert list(sizes) == [_lib.C.sizeof(_lib.PfConfig), _lib.C.sizeof(_lib.PfOutputs),
                           _lib.C.sizeof(_lib.PfFeed)]
    assert _lib.C.sizeof(_lib.PfConfig) == 8 + 8 + 4 * 4 + 8 * 11 + 4 * 8
    assert _lib.C.sizeof(_lib.PfOutputs) == 8 * 23 + 8 * 7 + 8 + 8
    assert _lib.C.sizeof(_lib.PfFeed) == 32


def test_no_device_means_loud_failure(lib):
    import paper_1212_1639_b200 as P

    if lib.pf_device_count() > 0:
        pytest.skip("device present")
    with pytest.raises(P.DeviceError):
        P.run_particle_learning(P.Priors(), [1.0, 2.0], 16)
    with pytest.raises(P.DeviceError):
        P.parallel_cdf(np.ones(4))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1212_1639_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), fn
