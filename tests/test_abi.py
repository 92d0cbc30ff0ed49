"""CPU: the C-ABI library builds, loads and exports every symbol the header
declares; without a GPU every compute entry point fails loudly (no CPU
fallback)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vecchia_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vgp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "vgp_loglik" in syms and "vgp_knn_predecessors" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2403_07412_b200 import _native as N

    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(vgp_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(N.EXPORTS) == set(declared_symbols())
    lib = ctypes.CDLL(N.LIB_PATH)
    for s in declared_symbols():
        getattr(lib, s)


def test_library_is_sm100a_code():
    from paper_2403_07412_b200 import _native as N

    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_and_device_count():
    from paper_2403_07412_b200 import _native as N

    assert "sm_100a" in N.version()
    assert N.device_count() >= 0


@pytest.mark.skipif(bool(int(os.environ.get("VGP_HAVE_GPU", "0"))), reason="GPU present")
def test_no_cpu_fallback_without_gpu():
    import paper_2403_07412_b200 as vg
    from paper_2403_07412_b200 import _native as N

    if N.device_count() > 0:
        pytest.skip("a GPU is visible")
    locs = np.random.default_rng(0).random((50, 2))
    with pytest.raises(N.NativeError, match="no CPU fallback"):
        vg.nearest_neighbors(vg.Dataset(locs, np.zeros(50)), 5)
    with pytest.raises(N.NativeError):
        vg.matern_cov(np.array([0.1, 0.2]), vg.KernelParams(1.0, 0.1, 0.5))


def test_argument_errors_reported_before_device_use():
    from paper_2403_07412_b200 import _native as N

    out = np.zeros((1, 1), dtype=np.int64)
    locs = np.zeros((2, 2))
    rc = N.lib.vgp_knn_predecessors(0, N.dptr(locs), 2, 5, N.iptr(out))
    assert rc == N.VGP_E_INVALID
    assert "m < n" in N.last_error()
    rc = N.lib.vgp_cov(0, 0, -1.0, 0.1, 0.5, N.dptr(locs), 0, N.dptr(locs))
    assert rc == N.VGP_E_INVALID


def test_status_mapping_to_reference_exceptions():
    import paper_2403_07412_b200 as vg
    from paper_2403_07412_b200 import _native as N

    with pytest.raises(vg.LikelihoodEvaluationError) as e:
        N.raise_for_status(N.VGP_NOT_POSITIVE_DEFINITE, 7)
    assert e.value.block_index == 7
    assert isinstance(e.value.__cause__, vg.NonPositiveDefiniteError)
    with pytest.raises(vg.LikelihoodEvaluationError) as e:
        N.raise_for_status(N.VGP_BAD_CONDITIONAL_VARIANCE, 3)
    assert e.value.block_index == 3
    with pytest.raises(vg.SingularTriangularError):
        N.raise_for_status(N.VGP_SINGULAR_TRIANGULAR, 1)
    N.raise_for_status(N.VGP_OK, -1)
