"""Run a staged reference program (the "dlx-program/1" descriptor of a scheduled, fused
stagekit graph, produced by integration/stagekit_dlx.cpp) on the B200 executor.

This is the Python face of ``dlx_program_run`` (include/dlx_program.h), the drop-in for the
reference's missing ``interpret`` / ``executeDEG`` (interp.hpp:10).
"""
from __future__ import annotations

import ctypes
import json

from . import _lib


def run_program(program: str | dict, seed: int = 1, device: int = 0) -> tuple[str, list]:
    """Returns (printed output text, per-loop lowering report)."""
    if isinstance(program, dict):
        program = json.dumps(program)
    L = _lib.load()
    out = ctypes.c_void_p()
    rep = ctypes.c_void_p()
    _lib.check(L.dlx_program_run(program.encode(), seed, device, ctypes.byref(out), ctypes.byref(rep)))
    try:
        text = ctypes.string_at(out).decode()
        report = json.loads(ctypes.string_at(rep).decode())
    finally:
        L.dlx_string_free(out)
        L.dlx_string_free(rep)
    return text, report
