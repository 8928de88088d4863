"""The C-ABI library: loads without a GPU, exports every symbol
include/pse_b200.h declares, and reports errors as negative codes (no
compute calls here)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2101_10881_b200 as pe
from paper_2101_10881_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pse_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pse_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (pse_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    assert sorted(_lib.EXPORTS) == names


def test_library_is_built_for_sm_100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_codes():
    L = _lib.lib()
    assert b"sm_100a" in L.pse_version()
    h = C.c_void_p()
    bad = np.array([2, 1], np.int32)
    rc = L.pse_graph_build(3, 2, 1, np.array([2], np.int32).ctypes.data, bad.ctypes.data, None, C.byref(h))
    assert rc == -1
    assert b"strictly increasing" in L.pse_last_error()
    out = np.zeros(4, np.int64)
    assert L.pse_cost(6, out.ctypes.data) == -1
    assert L.pse_cost(10, out.ctypes.data) == 0 and out.tolist() == [279, 1944, 397, 3089]


def test_describe_roundtrip_and_validate_through_abi():
    g = pe.build_jobgraph_shape(6, 3, [3, 4, 3], [1, 3, 6, 1, 2, 5, 6, 2, 3, 4])
    d = g.desc(10, "real")
    assert (d.n, d.N, d.d, d.m, d.mode, d.total_slots) == (6, 3, 3, 10, 0, 28)
    msg = C.create_string_buffer(256)
    assert _lib.lib().pse_graph_validate(C.byref(d), msg, 256) == 1


def test_plan_create_rejects_invalid_graph_before_touching_the_device():
    g = pe.build_jobgraph_shape(16, 2, *(lambda p: (p.nvars, p.indices))(pe.gen_benchmark("p1", 1, 1, with_static=False)))
    off = g.conv_layer_off.copy()
    off[1] += 1
    bad = pe.GraphArrays(g.n, g.N, g.d, g.total_slots, g.value_slot, g.gradient_slots, g.multipliers, off,
                         g.conv_in1, g.conv_in2, g.conv_out, g.conv_copy, g.add_layer_off, g.add_src, g.add_dst)
    with pytest.raises(pe.InvalidArgument, match="invalid job graph"):
        pe.DevicePlan(bad, 2)
    with pytest.raises(pe.InvalidArgument):
        pe.DevicePlan(g, 6)
