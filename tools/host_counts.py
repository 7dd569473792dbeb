"""Operation counts of the product engine per policy on a bench workload, on
the CPU (width 1): where the per-event work goes, without a GPU.
Usage: python tools/host_counts.py [c2|c3] [policy indices]"""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import oracle_lib as O  # noqa: E402

NAMES = ["s1s_rounds", "s1s_cands_in_group", "s1s_unowned_witness", "proofs", "proof_intervals",
         "s_own_calls", "s_own_intervals", "s_own_members", "s1s_calls", "bfc_mallocs", "bfc_freelist_len",
         "shift_entries", "iv_compactions", "iv_compaction_rows", "s_lru_calls", "shifts",
         "seq_words", "seq_calls", "par_words", "par_calls"] + [f"seq_w{i + 1}" for i in range(8)] + ["seq_w9+"]


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    lib = ROOT / "build" / "libgml_host_counts.so"
    lib.parent.mkdir(exist_ok=True)
    cuda_inc = os.environ.get("CUDA_HOME", "/usr/local/cuda") + "/include"
    subprocess.check_call(["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-pthread", f"-I{ROOT / 'include'}",
                           f"-I{cuda_inc}", str(ROOT / "tools" / "host_counts.cpp"), "-o", str(lib)])
    L = C.CDLL(str(lib))
    L.eng_replay.restype = C.c_int
    L.eng_replay.argtypes = [C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(O.Policy), C.c_int,
                             C.POINTER(C.c_uint64), C.POINTER(O.Stats), C.POINTER(C.c_uint32)]
    W = bench.Workload(wl, 1)
    traces, pols, desc = W.load(list(range(W.n))), W.pols, W.desc
    ev = np.ascontiguousarray(traces[0], dtype=np.uint64)
    idx = [int(x) for x in sys.argv[2:]] or range(len(pols))
    print(desc)
    for v in idx:
        asg = np.zeros(len(ev), dtype=np.uint64)
        st = O.Stats()
        hw = (C.c_uint32 * 5)()
        L.eng_replay(ev.ctypes.data_as(C.POINTER(C.c_uint64)), len(ev), C.byref(O.to_policy(pols[v])), 1,
                     asg.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(st), hw)
        o = (C.c_ulonglong * 32)()
        L.hc_get(o)
        print(f"V{v} " + " ".join(f"{n}={o[i]}" for i, n in enumerate(NAMES)))


if __name__ == "__main__":
    main()
