"""A small PyTorch training run (test workload, not product code): an MLP
language-model-like stack trained with Adam for a few steps, with activation
sizes that span the small path (< 2 MiB) and the VMM path. Prints one JSON
line: per-step losses, torch memory statistics and, with --gml, the GMLake
allocator's statistics. Used by tests/test_torch_backend_gpu.py in a fresh
process (the allocator can only be switched before CUDA memory is used)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gml", action="store_true")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--limit-mib", type=int, default=128)
    ap.add_argument("--snapshot", default="")
    args = ap.parse_args()
    import torch
    if args.gml:
        from paper_2401_08156_b200 import torch_backend
        torch_backend.enable({"kind": 2, "flags": 0, "capacity_bytes": 64 << 30, "chunk_bytes": 2 << 20,
                              "small_threshold_bytes": 2 << 20, "frag_limit_bytes": args.limit_mib << 20,
                              "spool_max_entries": 4096, "_pad": 0, "spool_max_inactive_bytes": 64 << 30})
    if args.snapshot:
        torch.cuda.memory._record_memory_history(max_entries=1_000_000)
    torch.manual_seed(0)
    dev = torch.device("cuda", 0)
    d, f, layers, vocab = 1024, 4096, 6, 8192
    blocks = []
    for _ in range(layers):
        blocks += [torch.nn.LayerNorm(d), torch.nn.Linear(d, f), torch.nn.GELU(), torch.nn.Linear(f, d)]
    model = torch.nn.Sequential(torch.nn.Embedding(vocab, d), *blocks, torch.nn.Linear(d, vocab)).to(dev)
    opt = torch.optim.Adam(model.parameters(), lr=1e-4)
    g = torch.Generator(device="cpu").manual_seed(1)
    losses, per_step, step_ms = [], [], []
    prev = [0] * 7
    import time
    for step in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bsz = 8 + 4 * (step % 3)                      # varying batch: irregular sizes across steps
        x = torch.randint(0, vocab, (bsz, 256), generator=g).to(dev)
        y = torch.randint(0, vocab, (bsz, 256), generator=g).to(dev)
        logits = model(x)
        loss = torch.nn.functional.cross_entropy(logits.float().view(-1, vocab), y.view(-1))
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        losses.append(float(loss.item()))
        step_ms.append(1e3 * (time.perf_counter() - t0))
        if args.gml:
            from paper_2401_08156_b200 import torch_backend
            sc = torch_backend.stats(0)["state_count"]
            per_step.append([a - b for a, b in zip(sc, prev)])
            prev = sc
    torch.cuda.synchronize()
    out = {"losses": losses, "per_step": per_step, "step_ms": step_ms}
    if args.snapshot:
        snap = torch.cuda.memory._snapshot()
        torch.cuda.memory._record_memory_history(enabled=None)
        import pickle
        with open(args.snapshot, "wb") as fh:
            pickle.dump(snap, fh)
    if args.gml:
        from paper_2401_08156_b200 import torch_backend
        out["gml"] = torch_backend.stats(0)
    else:
        ms = torch.cuda.memory_stats(0)
        out["torch"] = {k: ms.get(k) for k in ("allocated_bytes.all.peak", "reserved_bytes.all.peak",
                                               "requested_bytes.all.peak", "num_alloc_retries")}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
