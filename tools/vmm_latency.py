"""f2: Table 1 / fig:virtual of the paper re-measured on
this device through libgml's gml_vmm_profile: per-API latency of building one
allocation from physical chunks, normalised by cudaMalloc of the same size.

    python tools/vmm_latency.py [--reps 5] > profiles/<round>/vmm_latency.json
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

MiB = 1 << 20
NAMES = ["cudaMalloc", "cudaFree", "cuMemAddressReserve", "cuMemCreate", "cuMemMap", "cuMemSetAccess_per_chunk",
         "cuMemSetAccess_one_call", "teardown", "vmm_total_table1", "vmm_total_gml_alloc"]
PAPER_TABLE1 = {  # normalised to cuMalloc, 2 GB allocation, A100
    2: {"cuMemAddressReserve": 0.003, "cuMemCreate": 18.1, "cuMemMap": 0.70, "cuMemSetAccess": 96.8, "total": 115.4},
    128: {"cuMemAddressReserve": 0.003, "cuMemCreate": 0.89, "cuMemMap": 0.01, "cuMemSetAccess": 8.2, "total": 9.1},
    1024: {"cuMemAddressReserve": 0.002, "cuMemCreate": 0.79, "cuMemMap": 0.002, "cuMemSetAccess": 0.7, "total": 1.5},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--device", type=int, default=0)
    args = ap.parse_args()
    import __graft_entry__ as ge
    ge.build()
    from paper_2401_08156_b200 import gml
    L = gml.lib()
    rows = []
    cases = [(2048, c) for c in (2, 4, 8, 16, 32, 64, 128, 256, 512, 1024)] + \
            [(b, c) for b in (512, 1024) for c in (2, 128, 512)]
    for block, chunk in cases:
        out = (C.c_double * 10)()
        rc = L.gml_vmm_profile(args.device, block * MiB, chunk * MiB, args.reps, out)
        if rc != 0:
            rows.append({"block_mib": block, "chunk_mib": chunk, "error": gml.status_string(rc)})
            continue
        us = dict(zip(NAMES, list(out)))
        base = us["cudaMalloc"]
        norm = {k: us[k] / base for k in NAMES}
        row = {"block_mib": block, "chunk_mib": chunk, "us": us, "normalised_to_cudaMalloc": norm}
        if block == 2048 and chunk in PAPER_TABLE1:
            row["paper_a100_normalised"] = PAPER_TABLE1[chunk]
        rows.append(row)
    print(json.dumps({"device": args.device, "reps": args.reps, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
