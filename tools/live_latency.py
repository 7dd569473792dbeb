"""C5: per-call host latency of the live allocator (gml_malloc / gml_free) vs
cudaMalloc / cudaFree vs PyTorch's caching allocator on the same
PyTorch-shaped malloc/free stream (C2 prefix), plus stitched-buffer
bandwidth (K2). Prints one JSON object.

    python tools/live_latency.py [--iters 4]
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pct(xs):
    a = np.asarray(xs) * 1e6
    return {"p50_us": float(np.percentile(a, 50)), "p99_us": float(np.percentile(a, 99)),
            "mean_us": float(a.mean()), "n": int(a.size)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=4)
    args = ap.parse_args()
    import torch
    import __graft_entry__ as ge
    ge.build()
    from paper_2401_08156_b200 import gml
    from tracegen import decode, synth, policies as P

    torch.cuda.init()
    ev, starts = synth.config_c2(iters=args.iters)
    ops = [decode(e) for e in ev]
    out = {"trace": f"C2 OPT-1.3B + R b16, {args.iters} iterations, {len(ev)} events"}

    # --- GMLake live allocator
    pol = P.policy(P.GMLAKE, capacity=60 << 30)
    a = gml.Allocator(0, pol)
    ptr, tm, tf = {}, [], []
    per_iter = []
    for k, (f, slot, size) in enumerate(ops):
        t = time.perf_counter()
        if f:
            a.free(ptr.pop(slot))
            tf.append(time.perf_counter() - t)
        else:
            ptr[slot] = a.malloc(size)
            tm.append(time.perf_counter() - t)
    st = a.stats()
    calls = a.driver_calls()
    for p in ptr.values():
        a.free(p)
    a.destroy()
    # steady state: mallocs of the last iteration only (after convergence)
    last = starts[-1]
    n_m_last = sum(1 for f, _, _ in ops[last:] if not f)
    out["gmlake"] = {"malloc": pct(tm), "free": pct(tf), "malloc_last_iter": pct(tm[-n_m_last:]),
                     "states": st["state_count"], "driver_calls": calls}

    # --- cudaMalloc / cudaFree
    rt = C.CDLL("libcudart.so.12")
    rt.cudaMalloc.argtypes = [C.POINTER(C.c_void_p), C.c_size_t]
    rt.cudaFree.argtypes = [C.c_void_p]
    ptr, tm, tf = {}, [], []
    for f, slot, size in ops:
        t = time.perf_counter()
        if f:
            rt.cudaFree(ptr.pop(slot))
            tf.append(time.perf_counter() - t)
        else:
            p = C.c_void_p()
            rt.cudaMalloc(C.byref(p), size)
            ptr[slot] = p.value
            tm.append(time.perf_counter() - t)
    for p in ptr.values():
        rt.cudaFree(p)
    out["cudaMalloc"] = {"malloc": pct(tm), "free": pct(tf)}

    # --- PyTorch caching allocator
    torch.cuda.empty_cache()
    ptr, tm, tf = {}, [], []
    for f, slot, size in ops:
        t = time.perf_counter()
        if f:
            torch.cuda.caching_allocator_delete(ptr.pop(slot))
            tf.append(time.perf_counter() - t)
        else:
            ptr[slot] = torch.cuda.caching_allocator_alloc(size)
            tm.append(time.perf_counter() - t)
    for p in ptr.values():
        torch.cuda.caching_allocator_delete(p)
    out["torch_caching"] = {"malloc": pct(tm), "free": pct(tf)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
