"""The C-ABI library loads on CPU and exports every symbol include/dlx.h declares.  No
compute calls (there is no GPU here)."""
import glob
import os
import re
import subprocess

import pytest

from paper_1109_0778_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        with open(h) as f:
            text = f.read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(dlx_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_header_matches_bindings():
    assert declared_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (dlx_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_errors_are_reported_without_gpu():
    L = _lib.load()
    assert L.dlx_version().startswith(b"dlx")
    # argument validation happens before any device work
    rc = L.dlx_groupby_count(None, -1, 4, None, None, 0, None)
    assert rc == _lib.DLX_ERR_ARG
    assert b"groupby" in L.dlx_last_error()
    with pytest.raises(_lib.DlxError):
        _lib.check(rc)
