"""Run a staged reference program (the "dlx-program/1" descriptor of a scheduled, fused stagekit
graph, produced by integration/stagekit_dlx.cpp, or built directly by ``descriptors``) on the
B200 executor.

This is the Python face of ``include/dlx_program.h``, the drop-in for the reference's missing
``interpret`` / ``executeDEG`` (interp.hpp:10) and its
``RunResult {output, result}`` (runtime.hpp:100-103).

    prog = Program(descriptor)          # parse + static analysis once (dlx_program_create)
    r = prog.run(seed=1)                # r.output, r.report, r.result (lowerings cached)
    r = prog.run(inputs={sym: array})   # caller data for a VectorRand / VectorRandInt statement
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _lib


@dataclass
class RunResult:
    output: str
    report: list = field(default_factory=list)
    result: Any = None          # int / float / bool / str / numpy array (vector) / None (Unit)


def _input_struct(sym: int, data) -> tuple[_lib.ProgramInput, Any]:
    """(struct, keep-alive) for one input: a numpy array (host) or a torch tensor (host or device)."""
    inp = _lib.ProgramInput()
    inp.sym = int(sym)
    keep = data
    if hasattr(data, "data_ptr"):   # torch tensor
        import torch
        if data.dtype not in (torch.float64, torch.int64) or not data.is_contiguous():
            raise ValueError("program inputs are contiguous float64 / int64 tensors")
        inp.elem = _lib.VAL_DOUBLE if data.dtype == torch.float64 else _lib.VAL_INT
        inp.n = data.numel()
        if data.is_cuda:
            inp.d_data = data.data_ptr()
        else:
            inp.h_data = data.data_ptr()
    else:
        arr = np.ascontiguousarray(data)
        if arr.dtype not in (np.float64, np.int64):
            raise ValueError("program inputs are float64 / int64 arrays")
        inp.elem = _lib.VAL_DOUBLE if arr.dtype == np.float64 else _lib.VAL_INT
        inp.n = arr.size
        inp.h_data = arr.ctypes.data
        keep = arr
    return inp, keep


class Program:
    """A parsed, analysed program (``dlx_program_create``); ``run`` executes it."""

    def __init__(self, program: str | dict | bytes):
        if isinstance(program, dict):
            program = json.dumps(program)
        if isinstance(program, str):
            program = program.encode()
        L = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(L.dlx_program_create(program, len(program), ctypes.byref(h)))
        self._h = h
        self._L = L

    def close(self):
        if self._h:
            self._L.dlx_program_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, seed: int = 1, device: int = 0, devices=None, inputs: dict | None = None,
            serial: bool = False, dry_run: bool = False, no_cache: bool = False) -> RunResult:
        o = _lib.ExecOptions()
        o.seed = seed
        devs = list(devices) if devices is not None else [device]
        dev_arr = (ctypes.c_int32 * len(devs))(*devs)
        o.ndevices = len(devs)
        o.devices = ctypes.cast(dev_arr, ctypes.POINTER(ctypes.c_int32))
        keep = []
        if inputs:
            arr = (_lib.ProgramInput * len(inputs))()
            for q, (sym, data) in enumerate(inputs.items()):
                arr[q], k = _input_struct(sym, data)
                keep.append(k)
            o.ninputs = len(inputs)
            o.inputs = ctypes.cast(arr, ctypes.POINTER(_lib.ProgramInput))
        o.flags = (_lib.EXEC_SERIAL if serial else 0) | (_lib.EXEC_DRYRUN if dry_run else 0) | \
            (_lib.EXEC_NOCACHE if no_cache else 0)
        r = _lib.RunResult()
        _lib.check(self._L.dlx_program_execute(self._h, ctypes.byref(o), ctypes.byref(r)))
        try:
            text = ctypes.string_at(r.text).decode()
            report = json.loads(ctypes.string_at(r.report).decode())
            if r.kind == _lib.VAL_INT:
                res = int(r.i)
            elif r.kind == _lib.VAL_DOUBLE:
                res = float(r.d)
            elif r.kind == _lib.VAL_BOOL:
                res = bool(r.i)
            elif r.kind == _lib.VAL_STR:
                res = ctypes.string_at(r.s).decode()
            elif r.kind == _lib.VAL_VECTOR:
                dt = {_lib.VAL_INT: np.int64, _lib.VAL_DOUBLE: np.float64, _lib.VAL_BOOL: np.bool_}[r.vec_elem]
                nbytes = r.vec_len * np.dtype(dt).itemsize
                res = np.frombuffer(ctypes.string_at(r.vec_data, nbytes), dtype=dt).copy() if nbytes else np.zeros(0, dt)
            else:
                res = None
        finally:
            self._L.dlx_run_result_free(ctypes.byref(r))
        return RunResult(text, report, res)


def run_program(program: str | dict, seed: int = 1, device: int = 0) -> tuple[str, list]:
    """One-shot ``dlx_program_run``: returns (printed output text, per-loop lowering report)."""
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
