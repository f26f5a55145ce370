"""CPU: the C-ABI library builds for sm_100a, loads, and exports the header's API."""
import os
import re
import subprocess

import pytest

from paper_2412_03451_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "psplat_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_api():
    fns = header_functions()
    assert "psg_render_view" in fns and "psg_backward" in fns and "psg_step" in fns
    assert len(fns) >= 30


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    missing = [f for f in header_functions() if not hasattr(L, f)]
    assert missing == []


def test_binding_table_covers_header():
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_library_is_sm100a_device_code():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cuda_device_fails_loudly_without_fallback():
    import ctypes
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    st = _lib.lib().psg_create(0, 0, ctypes.byref(h))
    assert st == _lib.PSG_ECUDA and "CUDA" in _lib.last_error()


def test_host_lambda_schedule_matches_reference_literal():
    # acceptance_main.cpp:268-292 (criterion 4); pure host arithmetic
    assert abs(_lib.lib().psg_lambda_schedule(0, 20.0, 0.001, 300.0) - 7.357588823428847) < 1e-9
    assert _lib.lib().psg_lambda_schedule(3709, 20.0, 0.001, 300.0) == 300.0


def test_host_view_for_slot_matches_oracle(orc):
    # Optimizer::view_for_slot (optimizer.cpp:49-59) is host code in the library
    import ctypes
    orc.lib.orc_view_for_slot.restype = ctypes.c_int64
    orc.lib.orc_view_for_slot.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64]
    L = _lib.lib()
    for seed in (0, 7, 2**63 + 5):
        for n in (1, 3, 1024):
            for slot in list(range(0, 40)) + [5 * n + 1, 17 * n - 1]:
                assert L.psg_view_for_slot(seed, n, slot) == orc.lib.orc_view_for_slot(seed, n, slot)


def test_host_lambda_schedule_bitwise_vs_reference(ref):
    L = _lib.lib()
    for ite in range(0, 4000, 37):
        assert L.psg_lambda_schedule(ite, 20.0, 0.001, 300.0) == ref.lambda_schedule(ite)
