"""The C-ABI library loads and exports every entry point include/*.h declares
(no compute, CPU only)."""
import ctypes
import glob
import os
import re

import paper_1310_4218_b200 as od

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(od_\w+)\s*\(", text, re.M):
            names.add(m.group(1))
    return names


def test_every_declared_symbol_is_exported():
    names = declared_symbols()
    assert len(names) >= 40, names
    lib = ctypes.CDLL(od.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_every_declared_symbol_has_a_python_prototype():
    from paper_1310_4218_b200._lib import PROTOTYPES
    assert declared_symbols() <= set(PROTOTYPES), declared_symbols() - set(PROTOTYPES)


def test_abi_version_and_error_codes():
    assert od.lib.od_abi_version() == 1
    # ValidationError -> 2 with a message; nothing thrown across the ABI
    rc = od.lib.od_initial_block_mapping(3, 4, (ctypes.c_int32 * 3)())
    assert rc == 2
    assert b"vp count" in od.lib.od_last_error()


def test_library_has_sm100a_code():
    # the shared object carries sm_100a cubins (cross-compiled here)
    data = open(od.LIB_PATH, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data
