"""ctypes binding of tests/engine_host.cpp: the PRODUCT engine (policy.cuh)
compiled for the CPU, width 1 (HostWarp) or an emulated 32-lane warp
(SimWarp). Test infrastructure: lets the non-GPU suite check the engine's
lane-parallel logic against the oracle without a GPU."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

import oracle_lib as O

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "engine_host.cpp"
DEPS = [SRC, ROOT / "paper_2401_08156_b200" / "csrc" / "policy.cuh", ROOT / "include" / "gml.h"]
LIB = ROOT / "build" / "libgml_engine_host.so"
CUDA_INC = os.environ.get("CUDA_HOME", "/usr/local/cuda") + "/include"


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < max(d.stat().st_mtime for d in DEPS):
        LIB.parent.mkdir(parents=True, exist_ok=True)
        tmp = LIB.with_suffix(f".{os.getpid()}.tmp")
        subprocess.check_call(["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-pthread",
                               f"-I{ROOT / 'include'}", f"-I{CUDA_INC}", str(SRC), "-o", str(tmp)])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(str(build()))
        L.eng_replay.restype = C.c_int
        L.eng_replay.argtypes = [C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(O.Policy), C.c_int,
                                 C.POINTER(C.c_uint64), C.POINTER(O.Stats), C.POINTER(C.c_uint32)]
        _lib = L
    return _lib


def replay(events: np.ndarray, pol: dict, width: int = 1, hw: list | None = None):
    """-> (assignments u64[n], stats dict, overflow bits); hw (optional list)
    receives the table high-water marks [pBlocks, sBlocks, intervals, BFC rows, index nodes]."""
    ev = np.ascontiguousarray(events, dtype=np.uint64)
    n = len(ev)
    asg = np.zeros(max(n, 1), dtype=np.uint64)
    st = O.Stats()
    p = O.to_policy(pol)
    hwa = (C.c_uint32 * 5)()
    rc = lib().eng_replay(ev.ctypes.data_as(C.POINTER(C.c_uint64)), n, C.byref(p), width,
                          asg.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(st), hwa)
    assert rc == 0
    if hw is not None:
        hw[:] = list(hwa)
    ovf = st._p
    st._p = 0
    return asg[:n], st.to_dict(), ovf
