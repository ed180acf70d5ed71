"""CPU-side checks of the C ABI: the library loads, exports every function
include/dippm_b200.h declares with the ctypes signature table in _lib.py, and
the host instance of the MIG rule reproduces the reference sweep."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2303_11733_b200 import _lib, mig

HEADER = Path(__file__).resolve().parents[1] / "include" / "dippm_b200.h"
HOST_HEADER = Path(__file__).resolve().parents[1] / "include" / "dippm_host.h"


def declared_functions(header=HEADER):
    text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(dippm_[a-z0-9_]+)\s*\(", text)))


def test_host_library_exports_every_declared_symbol():
    from paper_2303_11733_b200 import featurize
    lib = featurize._host()
    names = declared_functions(HOST_HEADER)
    assert len(names) >= 8
    for name in names:
        assert hasattr(lib, name), name
    text = re.sub(r"/\*.*?\*/", "", HOST_HEADER.read_text(), flags=re.S)
    assert 'extern "C"' in text and "std::" not in text and "torch" not in text


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.dippm_abi_version() == _lib.ABI_VERSION


def test_header_is_plain_c():
    assert 'extern "C"' in HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    for banned in ("torch", "at::", "std::", "template"):
        assert banned not in text


def test_host_mig_rule_matches_reference_sweep(golden):
    codes = []
    for a in golden["mig_alpha"]:
        c = ctypes.c_int32()
        assert _lib.load().dippm_mig_code(float(a), ctypes.byref(c)) == 0
        codes.append(c.value)
    assert codes == golden["mig_code"].tolist()


@pytest.mark.parametrize("alpha,label", [(2865, "1g.5gb"), (5952, "2g.10gb"), (2873, "1g.5gb"), (6736, "2g.10gb"),
                                         (4771, "1g.5gb"), (26439, "7g.40gb")])
def test_mig_table5_replay(alpha, label):
    # T/test_mig.py:11-23, Table 5
    assert mig.mig_profile(alpha).label == label


def test_mig_boundaries_and_nonfinite():
    # T/test_mig.py:26-47
    assert mig.mig_profile(0) is None
    assert mig.mig_profile(-5.0) is None
    assert mig.mig_profile(5120) is mig.MigProfile.MIG_1G_5GB
    assert mig.mig_profile(5120.000001) is mig.MigProfile.MIG_2G_10GB
    assert mig.mig_profile(10240) is mig.MigProfile.MIG_2G_10GB
    assert mig.mig_profile(20480) is mig.MigProfile.MIG_3G_20GB
    assert mig.mig_profile(40960) is mig.MigProfile.MIG_7G_40GB
    assert mig.mig_profile(45000) is None
    assert [p.max_memory_mb for p in mig.MigProfile] == [5120, 10240, 20480, 40960]
    from paper_2303_11733_b200.errors import NonFinite
    for bad in (float("nan"), float("inf"), -float("inf")):
        with pytest.raises(NonFinite):
            mig.mig_profile(bad)


def test_mig_monotone_total():
    hyp = pytest.importorskip("hypothesis")
    st = hyp.strategies

    @hyp.given(st.floats(allow_nan=False, allow_infinity=False), st.floats(allow_nan=False, allow_infinity=False))
    @hyp.settings(max_examples=300, deadline=None)
    def check(a, b):
        pa, pb = mig.mig_profile(a), mig.mig_profile(b)
        for alpha, p in ((a, pa), (b, pb)):
            if not (0 < alpha <= 40960):
                assert p is None
            else:
                assert p is not None and p.max_memory_mb >= alpha
        if 0 < a <= b <= 40960:
            assert pa.max_memory_mb <= pb.max_memory_mb

    check()


def test_cpu_has_no_compute_fallback():
    """Compute entry points need a GPU; without one they raise, never fall back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2303_11733_b200 import gnn
    from paper_2303_11733_b200.types import GraphEncoding
    model = gnn.create_model(hidden=8)
    with pytest.raises(_lib.DeviceUnavailable):
        gnn.forward(GraphEncoding(2, [(0, 1)], np.zeros((2, 32))), np.zeros(5), model)
