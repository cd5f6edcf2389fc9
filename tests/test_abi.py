"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/parpa.h declares, and
its host-side DFA compiler validates tables (no device work is issued here)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1905_13415_b200 import _lib, dialects
import paper_1905_13415_b200 as parpa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "parpa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(parpa_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for must in ["parpa_create_dfa", "parpa_parse", "parpa_parse_into", "parpa_summarize", "parpa_count",
                 "parpa_parse_range", "parpa_debug_trace"]:
        assert must in fns


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    for f in header_functions():
        assert hasattr(lib, f)
    assert set(_lib.EXPORTS) == set(header_functions())


def test_library_built_for_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", _lib.LIB_PATH], text=True)
    assert "sm_100a" in out


def _create(S, start, inv, gob, trans, emit, eoi):
    lib = _lib.load()
    G = len(trans)
    h = ctypes.c_void_p()
    rc = lib.parpa_create_dfa(S, start, inv, G, (ctypes.c_uint8 * 256)(*gob),
                              (ctypes.c_uint8 * (G * S))(*[v for r in trans for v in r]),
                              (ctypes.c_uint8 * (G * S))(*[v for r in emit for v in r]),
                              (ctypes.c_uint8 * S)(*eoi), ctypes.byref(h))
    if rc == 0:
        lib.parpa_destroy_dfa(h)
    return rc


@pytest.mark.parametrize("name", ["csv", "csv_comment", "clf"])
def test_create_dialects(name):
    t = dialects.get(name)
    assert _create(t.S, t.start, t.invalid, t.group_of_byte, t.transition, t.emit, t.eoi) == parpa.OK


def test_create_dfa_validation():
    t = dialects.rfc4180()
    base = (t.S, t.start, t.invalid, t.group_of_byte, t.transition, t.emit, t.eoi)
    bad_target = [r[:] for r in t.transition]
    bad_target[0][0] = 9                                   # target outside [0, S)
    assert _create(t.S, 0, 5, t.group_of_byte, bad_target, t.emit, t.eoi) == parpa.EINVAL
    not_absorbing = [r[:] for r in t.transition]
    not_absorbing[3][5] = 0                                # INV must be absorbing
    assert _create(t.S, 0, 5, t.group_of_byte, not_absorbing, t.emit, t.eoi) == parpa.EINVAL
    bad_emit = [r[:] for r in t.emit]
    bad_emit[0][5] = 0                                     # emission inside INV must be CTRL
    assert _create(t.S, 0, 5, t.group_of_byte, t.transition, bad_emit, t.eoi) == parpa.EINVAL
    gob = list(t.group_of_byte)
    gob[7] = 4                                             # group id >= G
    assert _create(t.S, 0, 5, gob, t.transition, t.emit, t.eoi) == parpa.EINVAL
    assert _create(t.S, 6, 5, *base[3:]) == parpa.EINVAL   # start out of range
    big = 11                                               # 10 live states + INV > 8 + INV
    tr = [[(s + 1) % (big - 1) for s in range(big - 1)] + [big - 1]]
    em = [[0] * (big - 1) + [1]]
    assert _create(big, 0, big - 1, [0] * 256, tr, em, [0] * big) == parpa.EUNSUPPORTED


def test_status_strings():
    lib = _lib.load()
    for code in range(-7, 1):
        assert lib.parpa_status_string(code)
