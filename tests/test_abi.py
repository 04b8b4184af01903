"""CPU checks of the C-ABI library: it loads without a GPU, exports every symbol
include/sv.h declares, and refuses to compute without an sm_100 device (no CPU
fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2505_21594_b200 import sv
from workload import tiny

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "sv.h")).read()
    return sorted(set(re.findall(r"SV_API\s+[\w\s\*]+?\b(sv_\w+)\s*\(", txt)))


def test_header_declares_api():
    names = _declared()
    for must in ("sv_engine_create", "sv_verify_submit", "sv_wait_early", "sv_wait_final", "sv_verify",
                 "sv_session_open", "sv_debug_accept", "sv_weights_generate"):
        assert must in names


def test_library_exports_every_declared_symbol(svlib):
    for name in _declared():
        assert hasattr(svlib, name), name
    assert set(_declared()) == set(sv.EXPORTS), "binding and header disagree"


def test_status_strings(svlib):
    assert sv.status_name(sv.SV_E_PROTOCOL) == "SV_E_PROTOCOL"
    assert svlib.sv_abi_version() == 4


def test_pure_host_calls(svlib):
    cfg = sv.make_cfg(tiny())
    assert svlib.sv_kv_block_bytes(C.byref(cfg)) == 2 * 2 * 128 * 64 * 2
    sz = [C.c_size_t() for _ in range(7)]
    assert svlib.sv_weight_sizes(C.byref(cfg), *[C.byref(s) for s in sz]) == sv.SV_OK
    assert sz[3].value == 3 * 128 * 128 * 2
    bad = sv.make_cfg(tiny())
    bad.vocab = 500
    assert svlib.sv_weight_sizes(C.byref(bad), *[None] * 7) == sv.SV_E_INVALID


def test_no_cpu_fallback(svlib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    o = (C.c_uint32 * 4)()
    s = svlib.sv_debug_philox((C.c_uint32 * 4)(0, 0, 0, 0), (C.c_uint32 * 2)(0, 0), o)
    assert s == sv.SV_E_DEVICE
    cfg = sv.make_cfg(tiny())
    h = C.c_void_p()
    w = sv.sv_weights()
    opts = sv.sv_engine_opts(1, 4, 1, 0)
    s = svlib.sv_engine_create(C.byref(cfg), C.byref(w), C.byref(opts), 0, C.c_void_p(1), 1 << 20, C.byref(h))
    assert s == sv.SV_E_DEVICE
