"""CPU checks of the C-ABI library: it loads, exports every symbol
include/qsb200.h declares, and fails loudly (no CPU fallback) without a GPU."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_1805_00988_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "qsb200.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qs_[a-z_0-9]+)\s*\(", text)))


def test_header_matches_binding_table():
    assert declared_symbols() == sorted(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(qs_[a-z_0-9]+)\b", out))
    assert set(declared_symbols()) <= exported


def test_abi_version():
    assert N.lib().qs_abi_version() == 2


def test_sm100a_cubin_embedded():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_fused_kernel_uses_tma_tensor_copies():
    """The fused pass stages tiles through the TMA engine (tensor copies in SASS)."""
    sass = subprocess.run(["cuobjdump", "-sass", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTMALDG.5D" in sass  # global -> shared tensor load
    assert "UTMASTG.5D" in sass  # shared -> global tensor store
    assert "SYNCS.ARRIVE.TRANS64" in sass  # mbarrier expect_tx


def test_null_handle_errors_without_device():
    L = N.lib()
    assert L.qs_synchronize(None) == N.QS_ERR_NULL
    assert "null" in N.last_error()
    assert L.qs_destroy(None) == N.QS_OK


def test_no_cpu_fallback_when_no_device():
    if N.device_count() > 0:
        pytest.skip("a CUDA device is visible")
    h = ctypes.c_void_p()
    rc = N.lib().qs_create(4, 0, 0, ctypes.byref(h))
    assert rc != N.QS_OK and not h.value
    from paper_1805_00988_b200 import State

    with pytest.raises(Exception):
        State(4)


def test_status_codes_map_to_reference_exceptions():
    from paper_1805_00988_b200.errors import CapacityError, DegenerateStateError, DeviceError

    for rc, exc in [(N.QS_ERR_INDEX, IndexError), (N.QS_ERR_VALUE, ValueError),
                    (N.QS_ERR_CAPACITY, CapacityError), (N.QS_ERR_DEGENERATE, DegenerateStateError),
                    (N.QS_ERR_CUDA, DeviceError)]:
        with pytest.raises(exc):
            N.check(rc)
