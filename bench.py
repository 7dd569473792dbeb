"""Benchmark: allocation-trace replay through the GMLake engine on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4]
                    [--impl ours|reference] [--no-secondary] [--no-cpu-baseline]

A step is one gml_replay of the workload batch -- every row of SURVEY §8(a):
ingest, classify, small path, S1..S5, free, stats -- for all 8 policy
variants V0..V7, inputs resident in HBM, L2 flushed between steps. Default
workload (N=1): BASELINE.json configs[1], the synthetic OPT-1.3B fine-tune
trace with recomputation, batch 16 (C2). With N ranks the global batch is N
such traces (weak scaling), LPT-sharded by event count over the ranks
(`shard.shard_plan`); the per-(trace, policy) stats are gathered with one
all_gather (`shard.gather_all`) and the device time is the max over ranks. A
secondary line measures the throughput configuration C4 (512 Llama-13B
traces x 8 policies per GPU: N x 512 traces of the 4096-trace sweep, LPT-
sharded; 8 ranks replay the whole C4 set).

`--impl reference` times the CPU oracle (the reference arm for this tier; the
paper ships no code) on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "alloc events/sec replayed @1/2/4/8 B200; utilization & frag % vs BFC"
UNIT = "event-replays/s"
GiB = 1 << 30


def _c4_trace(i):
    from tracegen import synth
    return synth.config_c4(i)[0]


def _c4_len(i):
    return len(_c4_trace(i))


class Workload:
    """A GLOBAL batch of traces (all ranks together) x the 8 policy variants;
    each rank generates only the traces its LPT shard gives it (SURVEY
    §8(e)). `lengths` are the event counts the shard plan balances."""

    def __init__(self, name: str, world: int):
        from tracegen import synth
        from tracegen import policies as P
        self.name = name
        self._cache = {}
        if name == "c2":
            # weak scaling: one C2 trace per rank, seed = trace_seed(2, i)
            self.n = world
            self.pols = P.variants(80 * GiB)
            self.desc = "C2: OPT-1.3B full fine-tune + recompute, b16 s512, 30 iters, 80 GiB"

            def gen(i):
                spec = synth.FinetuneSpec(synth.OPT_1_3B, batch=16, seq=512, iters=30, recompute=True,
                                          seed=synth.trace_seed(2, i))
                return synth.finetune_trace(spec)[0]
            self._gen = gen
            self.lengths = [len(self.get(i)) for i in range(self.n)]
        elif name == "c3":
            # one GPT-NeoX-20B ZeRO-3 rank trace per GPU (trace k of the 8-rank job)
            self.n = world
            self.pols = P.variants(80 * GiB)
            self.desc = "C3: GPT-NeoX-20B ZeRO-3(8) + recompute, b8 s1024, one rank trace per GPU"
            self._gen = lambda i: synth.config_c3(i % 8)[0]
            self.lengths = [len(self.get(i)) for i in range(self.n)]
        elif name == "c4":
            per = int(os.environ.get("GML_C4_PER_GPU", "512"))
            # the global set for N ranks: every 8th trace of the 4096-trace
            # sweep from offsets 0..N-1 (8 ranks: the whole sweep)
            self.idx = [(i * 8 + r) % 4096 for r in range(world) for i in range(per)]
            self.n = len(self.idx)
            self.pols = P.variants(180 * GiB)
            self.desc = f"C4: Llama-13B LoRA+offload sweep, {per} traces/GPU x {world} GPU(s), LPT-sharded, 180 GiB"
            # a trace's length depends on its {b, s, R, r} combo only (the
            # jitter swaps frees): one representative per combo
            combos = sorted({i // 16 for i in self.idx})
            from concurrent.futures import ProcessPoolExecutor
            with ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
                cl = dict(zip(combos, ex.map(_c4_len, [16 * c for c in combos], chunksize=4)))
            self.lengths = [cl[i // 16] for i in self.idx]
            self._gen = lambda j: _c4_trace(self.idx[j])
        else:
            raise SystemExit(f"unknown workload {name}")

    def get(self, i):
        if i not in self._cache:
            self._cache[i] = self._gen(i)
        return self._cache[i]

    def load(self, ids):
        """the traces `ids` (process pool for the C4 sweep)"""
        if self.name == "c4" and len(ids) > 8:
            from concurrent.futures import ProcessPoolExecutor
            with ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
                return list(ex.map(_c4_trace, [self.idx[j] for j in ids], chunksize=8))
        return [self.get(i) for i in ids]


class Clocks:
    """nvidia-smi sampling during the timed region (profiling recipe)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = [r.split(",") for r in self.out.strip().splitlines() if r.count(",") >= 6]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def oracle_time(traces, pols, budget_s: float = 20.0, which: int = 0):
    """Single-core oracle replay timing over a bounded sample (whole traces,
    every policy of a trace before the next trace) -> (event-replays/s,
    event-replays, seconds, sample). `which` picks the host core (the
    which-th of this process's allowed cores: one per rank at N > 1)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    O.lib()
    n_ev, t_tot, done = 0, 0.0, 0
    with _one_core(which) as core:
        t0 = time.perf_counter()
        for tr in traces:
            for pol in pols:
                a = time.perf_counter()
                O.replay(tr, pol)
                t_tot += time.perf_counter() - a
                n_ev += len(tr)
                done += 1
            if time.perf_counter() - t0 > budget_s:
                break
    return (n_ev / t_tot, n_ev, t_tot,
            f"{done} whole-trace (trace, policy) replays, {n_ev} event-replays, pinned to core {core}")


class _one_core:
    """Pin this process to one host core for the oracle timing (the SURVEY's
    `taskset -c 0`; rank k takes the k-th allowed core); restores the
    affinity afterwards."""

    def __init__(self, which: int = 0):
        self.which = which

    @staticmethod
    def physical(allowed):
        """one logical CPU per physical core (the first of its SMT siblings),
        so that concurrent ranks never share a core"""
        out = []
        for c in sorted(allowed):
            try:
                sib = open(f"/sys/devices/system/cpu/cpu{c}/topology/thread_siblings_list").read().strip()
                first = int(sib.replace("-", ",").split(",")[0])
            except (OSError, ValueError):
                first = c
            if first == c or first not in allowed:
                out.append(c)
        return out or sorted(allowed)

    def __enter__(self):
        self.old = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
        cores = self.physical(self.old) if self.old else None
        core = cores[self.which % len(cores)] if cores else None
        if core is not None:
            os.sched_setaffinity(0, {core})
        return core

    def __exit__(self, *a):
        if self.old:
            os.sched_setaffinity(0, self.old)


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" (nproc {os.cpu_count()})"
    except OSError:
        pass
    return f"nproc {os.cpu_count()}"


def measure(name, steps, warmup, rank, world, local, dev, with_cpu, cold_steps=0, cpu_budget_s=25.0):
    """Time `steps` replays of workload `name` on this rank (its LPT shard of
    the global batch); returns the fields of a bench line (rank 0
    meaningful). Table-size hints: the warm-up replays size each unit's
    tables (D30) and the timed steps reuse them (`hinted`); `cold_steps`
    more steps are timed from no hint at all (middle size class, overflow
    re-runs inside the call) and reported as `cold`."""
    import torch
    import torch.distributed as dist
    from paper_2401_08156_b200 import gml
    from paper_2401_08156_b200 import replay as R
    from paper_2401_08156_b200.shard import gather_all, shard_plan

    W = Workload(name, world)
    plan = shard_plan(W.lengths, world, rank)
    assert plan.mine, f"rank {rank} has no trace of {name}"
    traces = W.load(plan.mine)
    pols, desc = W.pols, W.desc
    n_events = int(sum(len(t) for t in traces))
    V = len(pols)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(stream):
        batch = R.upload(traces, dev)
        asg = torch.empty((V, max(batch.total, 1)), dtype=torch.int64, device=dev)
        st = torch.empty((len(traces) * V * 272,), dtype=torch.uint8, device=dev)
    stream.synchronize()
    caps = np.zeros((len(traces) * V, 4), dtype=np.uint32)

    def step():
        R.run(batch, pols, stream=stream, caps=caps, assignments=asg, stats=st)

    # warm-up; gml_replay writes back into `caps` the size class each unit
    # ended in, which the hinted steps reuse (no overflow re-runs)
    for _ in range(max(warmup, 1)):
        with torch.cuda.stream(stream):
            flush.zero_()
        step()
    stream.synchronize()
    hint = caps.copy()

    def timed(k, cold):
        """device time (ms, max over ranks) of k steps and the K0/K1 launches"""
        ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        kern, launches = [], 0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(k):
            caps[:] = 0 if cold else hint
            with torch.cuda.stream(stream):
                flush.zero_()
            ev_a[i].record(stream)
            step()
            ev_b[i].record(stream)
            kern.append(gml.gml_last_kernel_ms())
            launches += gml.gml_last_launch_count()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t = torch.tensor([float(sum(a.elapsed_time(b) for a, b in zip(ev_a, ev_b)))], dtype=torch.float64,
                         device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), kern, launches

    # ---- timed region: device time of K replays, L2 flushed between steps ----
    with Clocks(local) as clk:
        max_ms, kern_ms, launches = timed(steps, cold=False)
    n_split, n_rerun = gml.gml_last_split_count()
    cold = None
    if cold_steps:
        c_ms, c_kern, _ = timed(cold_steps, cold=True)
    caps[:] = hint
    # one all_gather of the per-(trace, policy) statistics
    all_arr = gather_all(plan, st, V)
    all_stats = [[gml.stats_dict(x) for x in row] for row in all_arr]
    replays = sum(s["n_events_done"] for per_t in all_stats for s in per_t)
    value = replays * steps / (max_ms / 1e3)
    if cold_steps:
        cold = {"value": replays * cold_steps / (c_ms / 1e3), "ms_per_step": c_ms / cold_steps,
                "steps": cold_steps, "kernel_ms": float(np.mean(c_kern)),
                "note": "no table-size hint: every unit starts in its family's middle size class, "
                        "overflowing units re-run in the next class inside the same gml_replay call"}

    # ---- e2e: host buffers through the C ABI, copies inside the timed region ----
    host_ev = torch.from_numpy(np.concatenate(traces).view(np.int64)).pin_memory()
    offs = np.zeros(len(traces) + 1, np.int64)
    offs[1:] = np.cumsum([len(x) for x in traces])
    host_off = torch.from_numpy(offs).pin_memory()
    host_asg = torch.empty((V, max(batch.total, 1)), dtype=torch.int64).pin_memory()
    host_st = torch.empty((len(traces) * V * 272,), dtype=torch.uint8).pin_memory()
    e_ms = []
    for _ in range(max(2, steps // 2)):
        with torch.cuda.stream(stream):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            batch.events.copy_(host_ev, non_blocking=True)
            batch.offsets.copy_(host_off, non_blocking=True)
        step()
        with torch.cuda.stream(stream):
            host_asg.copy_(asg, non_blocking=True)
            host_st.copy_(st, non_blocking=True)
            b.record(stream)
        stream.synchronize()
        e_ms.append(a.elapsed_time(b))
    et = torch.tensor([float(np.sum(e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e = {"value": replays * len(e_ms) / (float(et.item()) / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(host_ev.numel() * 8 + host_off.numel() * 8),
           "d2h_bytes_per_step": int(host_asg.numel() * 8 + host_st.numel())}

    # ---- roofline of K1: algorithmic DRAM bytes = each event read once for
    # all V policies (8 B) + one 8-byte record per event-replay ----
    pk = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(pk.read_text()) if pk.exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    local_replays = sum(int(all_arr[t, p]["n_events_done"]) for t in plan.mine for p in range(V))
    algo_bytes = 8 * n_events + 8 * local_replays
    k_ms = float(np.mean(kern_ms))
    achieved = algo_bytes / (k_ms / 1e3) / 1e9
    tf = ROOT / "profiles" / f"ncu_{name}_traffic.json"
    tj = json.loads(tf.read_text()) if tf.exists() else {}
    traffic = tj.get("dram_bytes_per_launch")
    if traffic is not None and (not np.isfinite(traffic) or tj.get("kernels_without_dram_counters")):
        traffic = None   # a partial ncu capture is only a lower bound
    roof = {"bound": "hbm", "achieved": round(achieved, 4), "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else
            "fallback 6650 GB/s (B200_PROFILING.md)",
            "algorithmic_bytes_per_launch": algo_bytes, "bytes_per_event_replay": algo_bytes / local_replays,
            "kernel_ms": k_ms,
            "kernel": "every kernel of one gml_replay (K0; K1 single-warp units, K1s split units or K1p path units "
                      "of every size class; K1l ledger, K1m merge), concurrent on side streams"}
    # the binding resource is instruction latency along each unit's chain:
    # warp instructions of one replay step (ncu, profiles/) over the chip's
    # issue rate = 148 SMs x 4 schedulers x 1 warp-instruction/cycle x SM clock
    clk = clk.summary()
    inst = tj.get("warp_instructions_per_launch")
    if inst is not None and not np.isfinite(inst):
        inst = None
    sm_hz = (clk.get("sm_mhz") or 1965.0) * 1e6
    issue = None
    if inst:
        a_ = inst / (k_ms / 1e3)
        pk_ = 148 * 4 * sm_hz
        issue = {"bound": "issue", "achieved": a_, "peak": pk_, "unit": "warp-inst/s", "frac": a_ / pk_,
                 "warp_instructions_per_step": inst, "warp_instructions_per_event_replay": inst / local_replays,
                 "source": "smsp__inst_executed.sum of the K1 launches of one replay (ncu, profiles/)"}
    # the C2 step is the slowest unit's chain (one warp per unit): its
    # cycles per warp instruction against the 4-cycle dependent-issue floor
    # (ncu, each policy replayed alone: profiles/ncu_c2_units.json)
    chain = None
    uf = ROOT / "profiles" / f"ncu_{name}_units.json"
    if uf.exists():
        uj = json.loads(uf.read_text())
        cu = uj["units"][uj["critical_unit"]]
        chain = {"bound": "latency", "unit": "cycles per warp instruction", "critical_unit": uj["critical_unit"],
                 "achieved": cu["cycles_per_inst"], "floor": uj["floor_cycles_per_inst"],
                 "frac": uj["floor_cycles_per_inst"] / cu["cycles_per_inst"],
                 "warp_instructions_per_event_replay": cu["warp_instructions"] / n_events,
                 "stall_share": cu["stall_share"],
                 "source": "profiles/" + uf.name + " (" + uj["floor_note"] + ")"}
    cpu = None
    if with_cpu:
        # the oracle on host cores: rank k on its own core over its own shard
        v1, n1, t1, sample = oracle_time(traces, pols, budget_s=cpu_budget_s, which=local)
        tot = torch.tensor([float(n1), v1], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tot)
        cpu = {"value": float(tot[1].item()), "unit": UNIT, "cores": world, "kind": "oracle",
               "single_core_value": v1 if world == 1 else float(tot[1].item()) / world,
               "sample": (sample if world == 1 else
                          f"{world} ranks, each its own host core over whole traces of its own shard "
                          f"({int(tot[0].item())} event-replays in total); value = sum of the per-core rates; "
                          f"rank 0: {sample}"),
               "cpu": _cpu_model()}
    from paper_2401_08156_b200 import analysis as An
    util = An.policy_report(all_stats)
    return {"value": value, "ms_per_step": max_ms / steps, "steps": steps, "warmup": warmup,
            "config": {"workload": desc, "traces_per_gpu": len(traces), "traces_total": plan.n_traces,
                       "policies": V, "events_per_gpu": n_events, "event_replays_per_step": replays,
                       "l2": "flushed between steps (256 MiB write)",
                       "sharding": "LPT by event count (shard.lpt_shard), one stats all_gather",
                       "table_hints": "the size classes the warm-up replays ended in (see `cold` for none)",
                       "two_path_units": {"completed": n_split, "single_warp_reruns": n_rerun,
                                          "note": "GMLake units whose VMM path and small path replayed concurrently "
                                                  "(split units in the latency placement, path units in the "
                                                  "throughput placement; DESIGN.md 6a)"},
                       "parallelism": f"trace-parallel x{world}"},
            "roofline": roof, "roofline_issue": issue, "roofline_chain": chain, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "cold": cold, "clocks": clk, "policies": util}


def _pct(ns):
    a = np.asarray(ns, dtype=np.float64) / 1e3
    if not a.size:
        return None
    return {"p50_us": float(np.percentile(a, 50)), "p99_us": float(np.percentile(a, 99)),
            "mean_us": float(a.mean()), "n": int(a.size)}


def measure_c5(dev_idx: int, cudamalloc_iters: int = 3):
    """C5 (BASELINE configs[4]): the live VMM allocator on this
    GPU. Per-call host latency of gml_malloc / gml_free over the whole C2
    stream (C-side steady_clock, gml_live_trace) vs cudaMalloc / cudaFree
    (C-side, a prefix of `cudamalloc_iters` iterations: ~300 us per call) vs
    PyTorch's caching allocator (timed from Python, as is gml through its
    Python binding for a like-for-like pair); then K2 stream copy over an
    8 GiB S3-stitched buffer (64 non-adjacent 128 MiB pBlocks) vs a
    cudaMalloc'd one (Table 1)."""
    import torch
    from paper_2401_08156_b200 import gml
    from tracegen import synth, decode
    from tracegen import policies as P
    ev, starts = synth.config_c2()
    is_free = (ev >> np.uint64(63)).astype(bool)
    pol = P.variants(80 * GiB)[2]
    a = gml.Allocator(dev_idx, pol)
    a.set_stream(torch.cuda.current_stream(dev_idx))
    rc, done, rec, ns = a.trace(ev)
    st, calls = a.stats(), a.driver_calls()
    a.destroy()
    last = np.zeros(len(ev), bool)
    last[starts[-1]:] = True
    out = {"trace": f"C2 OPT-1.3B + R b16, {len(starts)} iterations, {len(ev)} events", "policy": "V2",
           "gml_c": {"status": rc, "malloc": _pct(ns[~is_free]), "free": _pct(ns[is_free]),
                     "malloc_steady_state": _pct(ns[~is_free & last]), "states": st["state_count"],
                     "driver_calls": calls}}
    n_pre = starts[min(cudamalloc_iters, len(starts) - 1)]
    rc2, done2, ns2 = gml.gml_cudamalloc_trace(dev_idx, ev[:n_pre])
    f2 = is_free[:n_pre]
    out["cudaMalloc_c"] = {"status": rc2, "events": int(n_pre), "malloc": _pct(ns2[~f2]), "free": _pct(ns2[f2])}
    ops = [decode(e) for e in ev]

    def py_loop(alloc, free):
        ptr, tm = {}, np.zeros(len(ops), np.int64)
        pc = time.perf_counter_ns
        for i, (f, slot, size) in enumerate(ops):
            t = pc()
            if f:
                free(ptr.pop(slot))
            else:
                ptr[slot] = alloc(size)
            tm[i] = pc() - t
        for p_ in ptr.values():
            free(p_)
        return tm
    torch.cuda.empty_cache()
    tm = py_loop(torch.cuda.caching_allocator_alloc, torch.cuda.caching_allocator_delete)
    out["torch_caching_py"] = {"malloc": _pct(tm[~is_free]), "free": _pct(tm[is_free]),
                               "malloc_steady_state": _pct(tm[~is_free & last])}
    torch.cuda.empty_cache()
    a = gml.Allocator(dev_idx, pol)
    tm = py_loop(a.malloc, a.free)
    a.destroy()
    out["gml_py"] = {"malloc": _pct(tm[~is_free]), "free": _pct(tm[is_free]),
                     "malloc_steady_state": _pct(tm[~is_free & last])}
    # stitched vs native bandwidth (K2)
    a = gml.Allocator(dev_idx, P.policy(P.GMLAKE, capacity=40 * GiB))
    blocks = [a.malloc(128 << 20) for _ in range(128)]
    for p_ in blocks[::2]:
        a.free(p_)
    stitched = a.malloc(8 * GiB)
    n = 8 * GiB
    src = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev_idx}")
    dst = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev_idx}")
    gml.gml_stream_copy(src.data_ptr(), dst.data_ptr(), n, 2)
    t_nat = min(gml.gml_stream_copy(src.data_ptr(), dst.data_ptr(), n, 5) for _ in range(3))
    gml.gml_stream_copy(stitched, dst.data_ptr(), n, 2)
    t_st = min(gml.gml_stream_copy(stitched, dst.data_ptr(), n, 5) for _ in range(3))
    del src, dst
    a.free(stitched)
    for p_ in blocks[1::2]:
        a.free(p_)
    a.destroy()
    torch.cuda.empty_cache()
    bw_n, bw_s = 2 * n / (t_nat / 1e3) / 1e9, 2 * n / (t_st / 1e3) / 1e9   # gml_stream_copy: ms per pass
    out["stream_copy_gbs"] = {"native": bw_n, "stitched": bw_s, "ratio": bw_s / bw_n,
                              "buffer": "8 GiB stitched from 64 non-adjacent 128 MiB pBlocks (S3)",
                              "pass_within_2pct": abs(bw_s / bw_n - 1) < 0.02}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=os.environ.get("GML_WORKLOAD", "c2"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the live-allocator (C5) object")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    import __graft_entry__ as ge
    from paper_2401_08156_b200 import gml

    # (test plumbing: GML_SAME_DEVICE=1 puts every rank on cuda:0 and
    # GML_DIST_BACKEND=gloo lets N ranks share one GPU to exercise the N>1
    # path; the driver's runs use one GPU per rank and NCCL)
    dev_idx = 0 if os.environ.get("GML_SAME_DEVICE") == "1" else local
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    if world > 1:
        backend = os.environ.get("GML_DIST_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    if rank == 0:
        ge.build()
    if world > 1:
        dist.barrier()
    gml.lib()

    main_res = measure(args.workload, args.steps, args.warmup, rank, world, dev_idx, dev,
                       with_cpu=not args.no_cpu_baseline, cold_steps=3)
    secondary = None
    if not args.no_secondary and args.workload != "c4":
        s = measure("c4", 3, 3, rank, world, dev_idx, dev, with_cpu=not args.no_cpu_baseline, cold_steps=2)
        secondary = {k: s[k] for k in ("value", "ms_per_step", "steps", "warmup", "config", "roofline", "roofline_issue",
                                       "cpu_baseline", "e2e", "gpu_launches", "cold", "clocks", "policies")}
        secondary["unit"] = UNIT
    tertiary = None
    if not args.no_secondary and args.workload != "c3":
        # C3 (BASELINE configs[2]): one GPT-NeoX-20B ZeRO-3 rank trace per GPU
        s = measure("c3", 5, 3, rank, world, dev_idx, dev, with_cpu=not args.no_cpu_baseline, cold_steps=2,
                    cpu_budget_s=10.0)
        tertiary = {k: s[k] for k in ("value", "ms_per_step", "steps", "warmup", "config", "roofline",
                                      "cpu_baseline", "e2e", "gpu_launches", "cold", "clocks", "policies")}
        tertiary["unit"] = UNIT
    c5 = None
    if not args.no_c5:
        # C5 runs per GPU (one process each, no communication); rank 0 reports its own
        c5 = measure_c5(dev_idx)
    if rank == 0:
        line = {"metric": METRIC, "value": main_res["value"], "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": main_res["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic", "config": main_res["config"], "roofline": main_res["roofline"],
                "roofline_issue": main_res["roofline_issue"], "roofline_chain": main_res["roofline_chain"],
                "cpu_baseline": main_res["cpu_baseline"], "e2e": main_res["e2e"],
                "gpu_launches": main_res["gpu_launches"], "cold": main_res["cold"], "clocks": main_res["clocks"],
                "policies": main_res["policies"], "secondary_c4": secondary, "secondary_c3": tertiary,
                "c5_live": c5}
        print(json.dumps(line, allow_nan=False))
    if world > 1:
        dist.destroy_process_group()


def reference_arm(args, rank, world):
    """The CPU oracle as the reference arm, rank 0 only (other ranks exit 0)."""
    if rank != 0:
        return
    W = Workload(args.workload, 1)
    traces, pols, desc = W.load(list(range(W.n))), W.pols, W.desc
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    O.lib()
    per_step = float(os.environ.get("GML_REF_STEP_S", "3.0"))   # bounded sample per step
    for _ in range(args.warmup):
        O.replay(traces[0][:2000], pols[2])
    n_tot, t_tot, k = 0, 0.0, 0
    pin = _one_core()
    core = pin.__enter__()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < per_step:
            tr = traces[k % len(traces)]
            pol = pols[(k // len(traces)) % len(pols)]
            a = time.perf_counter()
            O.replay(tr, pol)
            t_tot += time.perf_counter() - a
            n_tot += len(tr)
            k += 1
    pin.__exit__()
    v = n_tot / t_tot
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": desc, "policies": len(pols)}, "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{k} whole-trace (trace, policy) replays over {args.steps} steps, "
                                       f"pinned to core {core}",
                             "cpu": _cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
