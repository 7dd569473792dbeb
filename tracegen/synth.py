"""Seeded synthetic allocation traces shaped like the paper's workloads.

INPUT infrastructure only (no allocator arithmetic). Recipes are documented in
DESIGN.md §"Input recipe"; the paper gives only the workload names
(Table 2: OPT-1.3b / GPT-NeoX-20b / ... with L/R/O under
DeepSpeed ZeRO-3) and the footprint statistics of fig:irregularity
(46k allocations of 93 MB mean without strategies vs 76k of
85 MB mean with LoRA+Recompute). Model dimensions are the public configs of
those models, not paper content.

Every trace is a deterministic function of its arguments; the only randomness
is (i) parameter sweeps and (ii) a jitter that swaps adjacent independent frees
with probability `jitter` (allocator-visible asynchrony),
drawn from splitmix64 seeded per trace.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np

from .events import SlotAssigner, pack

MiB = 1 << 20
GiB = 1 << 30
KiB = 1 << 10

_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Rng:
    """Counter-based splitmix64 stream (deterministic, language-independent)."""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / (1 << 53))

    def randint(self, lo: int, hi: int) -> int:
        """uniform integer in [lo, hi]"""
        return lo + self.next() % (hi - lo + 1)

    def normal(self) -> float:
        u1 = max(self.uniform(), 1e-300)
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2 * math.pi * u2)


def trace_seed(config: int, index: int) -> int:
    """seed of trace i of config c = splitmix64((c << 32) | i)."""
    return splitmix64(((config & 0xFFFFFFFF) << 32) | (index & 0xFFFFFFFF))


# ---------------------------------------------------------------------------
# C1: fig:intro worked example
# ---------------------------------------------------------------------------

def fig_intro() -> np.ndarray:
    """Three 8 MiB 'lines' filled, freed, then Blocks 1..6 of fig:intro.
    Block 6 (6 MiB) is larger than every free hole (Block 2 = 4 MiB hole,
    Block 5 = 2 MiB hole) but not than their sum."""
    ops = [
        ("m", 0, 8 * MiB), ("m", 1, 8 * MiB), ("m", 2, 8 * MiB),   # e0-e2 lines
        ("f", 0, 0), ("f", 1, 0), ("f", 2, 0),                      # e3-e5
        ("m", 3, 4 * MiB),   # e6  Block 1
        ("m", 4, 4 * MiB),   # e7  Block 2
        ("m", 5, 8 * MiB),   # e8  Block 3
        ("m", 6, 6 * MiB),   # e9  Block 4 (splits the third line)
        ("m", 7, 2 * MiB),   # e10 Block 5
        ("f", 4, 0),         # e11 free Block 2
        ("f", 7, 0),         # e12 free Block 5
        ("m", 8, 6 * MiB),   # e13 Block 6
        ("f", 3, 0), ("f", 5, 0), ("f", 6, 0), ("f", 8, 0),  # e14-e17
    ]
    return pack(ops)


def periodic(iteration: list[tuple[str, str, int]], iters: int) -> np.ndarray:
    """Repeat one iteration [('m'|'f', name, bytes)] `iters` times."""
    sa = SlotAssigner()
    for it in range(iters):
        for op, name, size in iteration:
            if op == "m":
                sa.malloc((it, name), size)
            else:
                sa.free((it, name))
    return sa.array()


# ---------------------------------------------------------------------------
# SPEC-style irregular corpus (parity only)
# ---------------------------------------------------------------------------

def lognormal_trace(seed: int, iters: int, allocs_per_iter: int, mean_bytes: float,
                    sigma: float = 0.5, lo: int = 2 * MiB, hi: int = 2 * GiB,
                    extra_frac: float = 0.0, interleave_frac: float = 0.0,
                    small_frac: float = 0.0) -> np.ndarray:
    """Per iteration: a forward phase of mallocs with log-normal sizes (fixed
    per position across iterations), then LIFO frees, with optional
    irregularity: short-lived extra mallocs (recompute proxy), re-mallocs at
    shifted sizes (offload proxy), partially shuffled frees, and a fraction of
    sub-2-MiB requests (small path)."""
    rng = Rng(seed)
    mu = math.log(mean_bytes) - sigma * sigma / 2
    base = []
    for _ in range(allocs_per_iter):
        if small_frac and rng.uniform() < small_frac:
            base.append(rng.randint(1, 2 * MiB - 1))
        else:
            v = int(math.exp(mu + sigma * rng.normal()))
            base.append(min(max(v, lo), hi))
    sa = SlotAssigner()
    uid = itertools.count()
    for it in range(iters):
        live = []
        for k, sz in enumerate(base):
            t = next(uid)
            sa.malloc(t, sz)
            live.append((t, sz))
            if extra_frac and rng.uniform() < extra_frac:
                e = next(uid)
                esz = min(max(int(sz * (0.25 + rng.uniform())), 1), hi)
                sa.malloc(e, esz)
                sa.free(e)
            if interleave_frac and rng.uniform() < interleave_frac and len(live) > 1:
                j = rng.randint(0, len(live) - 1)
                t2, s2 = live[j]
                sa.free(t2)
                n2 = next(uid)
                s2b = min(max(int(s2 * (0.5 + rng.uniform())), 1), hi)
                sa.malloc(n2, s2b)
                live[j] = (n2, s2b)
        order = list(reversed(live))
        if interleave_frac:
            for i in range(len(order) - 1):
                if rng.uniform() < interleave_frac:
                    order[i], order[i + 1] = order[i + 1], order[i]
        for t, _ in order:
            sa.free(t)
    return sa.array()


def random_trace(seed: int, n_events: int, max_live: int, sizes: list[int] | None = None,
                 p_malloc: float = 0.55, size_lo: int = 1, size_hi: int = 8 * MiB,
                 balanced: bool = True) -> np.ndarray:
    """Unstructured fuzz trace: random interleaving of mallocs and frees."""
    rng = Rng(seed)
    sa = SlotAssigner()
    live: list[int] = []
    uid = 0
    while len(sa.events) < n_events:
        if live and (len(live) >= max_live or rng.uniform() >= p_malloc):
            j = rng.randint(0, len(live) - 1)
            live[j], live[-1] = live[-1], live[j]
            sa.free(live.pop())
        else:
            sz = sizes[rng.randint(0, len(sizes) - 1)] if sizes else rng.randint(size_lo, size_hi)
            sa.malloc(uid, sz)
            live.append(uid)
            uid += 1
    if balanced:
        while live:
            sa.free(live.pop())
    return sa.array()


def tiny_corpus(m: int, sizes: list[int]):
    """Exhaustive tiny traces (SURVEY §4 layer 3): m mallocs with every size
    choice from `sizes` and every valid interleaving of frees in which the
    mallocs happen in id order; every tensor is freed by the end."""
    # interleavings: sequences over {M_i, F_i} with M_i before F_i and M in order
    def orders(n_m, live, seq):
        if n_m == m and not live:
            yield list(seq)
            return
        if n_m < m:
            seq.append(("m", n_m))
            yield from orders(n_m + 1, live | {n_m}, seq)
            seq.pop()
        for t in sorted(live):
            seq.append(("f", t))
            yield from orders(n_m, live - {t}, seq)
            seq.pop()
    all_orders = list(orders(0, frozenset(), []))
    for choice in itertools.product(sizes, repeat=m):
        for o in all_orders:
            sa = SlotAssigner()
            for op, t in o:
                if op == "m":
                    sa.malloc(t, choice[t])
                else:
                    sa.free(t)
            yield sa.array()


# ---------------------------------------------------------------------------
# Transformer fine-tuning step traces (C2-C4)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Model:
    name: str
    d: int
    layers: int
    ffn: int
    heads: int
    vocab: int
    style: str            # "opt" | "neox" | "llama"
    max_pos: int = 2048

    def layer_params(self) -> list[tuple[str, int]]:
        d, f = self.d, self.ffn
        if self.style == "opt":
            return [("ln1_w", d), ("ln1_b", d), ("q_w", d * d), ("q_b", d), ("k_w", d * d), ("k_b", d),
                    ("v_w", d * d), ("v_b", d), ("o_w", d * d), ("o_b", d), ("ln2_w", d), ("ln2_b", d),
                    ("fc1_w", d * f), ("fc1_b", f), ("fc2_w", f * d), ("fc2_b", d)]
        if self.style == "neox":
            return [("ln1_w", d), ("ln1_b", d), ("qkv_w", 3 * d * d), ("qkv_b", 3 * d),
                    ("o_w", d * d), ("o_b", d), ("ln2_w", d), ("ln2_b", d),
                    ("fc1_w", d * f), ("fc1_b", f), ("fc2_w", f * d), ("fc2_b", d)]
        return [("ln1_w", d), ("q_w", d * d), ("k_w", d * d), ("v_w", d * d), ("o_w", d * d),
                ("ln2_w", d), ("gate_w", d * f), ("up_w", d * f), ("down_w", f * d)]

    def lora_targets(self) -> list[str]:
        return ["qkv_w"] if self.style == "neox" else ["q_w", "v_w"]


OPT_1_3B = Model("opt-1.3b", 2048, 24, 8192, 32, 50272, "opt")
GPT_NEOX_20B = Model("gpt-neox-20b", 6144, 44, 24576, 64, 50432, "neox")
LLAMA_13B = Model("llama-13b", 5120, 40, 13824, 40, 32000, "llama")
OPT_13B = Model("opt-13b", 5120, 40, 20480, 40, 50272, "opt")

FP16, FP32 = 2, 4


@dataclass
class FinetuneSpec:
    model: Model
    batch: int
    seq: int
    iters: int
    recompute: bool = False      # R
    lora: bool = False           # L
    offload: bool = False        # O
    world: int = 1               # ZeRO-3 data-parallel degree (1 = plain DDP/single GPU)
    rank: int = 0
    lora_r: int = 16
    jitter: float = 0.1
    seed: int = 0
    flash: bool = False          # attention without materialised b*h*s*s scores


class _Gen:
    def __init__(self, spec: FinetuneSpec):
        self.s = spec
        self.sa = SlotAssigner()
        self.rng = Rng(spec.seed)
        self.uid = itertools.count()
        self.size = {}
        self.masks = set()

    # -- primitives --------------------------------------------------------
    def m(self, size: int, mask: bool = False):
        t = next(self.uid)
        self.sa.malloc(t, max(int(size), 1))
        self.size[t] = max(int(size), 1)
        if mask:
            self.masks.add(t)
        return t

    def f(self, t):
        self.sa.free(t)
        self.size.pop(t, None)
        self.masks.discard(t)

    def free_all(self, ts):
        """Free a group of independent tensors, adjacent pairs swapped with
        probability `jitter`."""
        ts = [t for t in ts if t is not None]
        j = self.s.jitter
        if j:
            for i in range(len(ts) - 1):
                if self.rng.uniform() < j:
                    ts[i], ts[i + 1] = ts[i + 1], ts[i]
        for t in ts:
            self.f(t)

    # -- sizes ---------------------------------------------------------------
    def part(self, numel: int) -> int:
        """ZeRO-3 partition of `numel` on this rank: ceil(numel / W), the
        remainder on the last rank."""
        W, r = self.s.world, self.s.rank
        if W == 1:
            return numel
        p = -(-numel // W)
        if r == W - 1:
            return max(numel - p * (W - 1), 1)
        return p


def finetune_trace(spec: FinetuneSpec) -> tuple[np.ndarray, list[int]]:
    """One fine-tuning run: setup, then `iters` iterations of forward, head,
    backward and optimizer step. Returns (events, iteration_start_indices)."""
    g = _Gen(spec)
    M = spec.model
    b, s, d, h, f, V = spec.batch, spec.seq, M.d, M.heads, M.ffn, M.vocab
    A = b * s * d * FP16               # one hidden-state activation
    AF = b * s * f * FP16              # MLP intermediate
    SC = b * h * s * s * FP16          # attention scores / probs
    MK = b * h * s * s                 # dropout mask (1 B)
    MKd = b * s * d                    # hidden dropout mask (1 B)
    zero = spec.world > 1
    lora = spec.lora
    R = spec.lora_r
    lp = M.layer_params()
    targets = set(M.lora_targets()) if lora else set()
    use_dropout = M.style == "opt"

    # ---- persistent state: parameters -----------------------------------
    params = {}          # (layer, name) -> tensor id (fp16 weight or partition)
    trainable = []       # [(key, numel)]
    embed = [("embed", V * d), ("pos", M.max_pos * d if M.style == "opt" else 0), ("lnf_w", d)]
    if M.style != "opt":
        embed.append(("lm_head", V * d))
    for name, n in embed:
        if n:
            params[(-1, name)] = g.m(g.part(n) * FP16)
            if not lora:
                trainable.append(((-1, name), n))
    for l in range(M.layers):
        for name, n in lp:
            params[(l, name)] = g.m(g.part(n) * FP16)
            if not lora:
                trainable.append(((l, name), n))
        if lora:
            for tname in M.lora_targets():
                out = 3 * d if tname == "qkv_w" else d
                for nm, n in ((tname + ".A", d * R), (tname + ".B", R * out)):
                    params[(l, nm)] = g.m(g.part(n) * FP16)
                    trainable.append(((l, nm), n))
    opt_state = {}       # key -> (master, m, v) allocated at first step
    grads = {}           # key -> grad tensor (partition when zero)
    gathered = {}

    def gather(l):
        """ZeRO-3 all-gather (and, with offload, swap-in) of layer l's
        weights into full-size buffers (partitioned weights)."""
        if not zero and not spec.offload:
            return
        bufs = []
        for name, n in lp:
            if spec.offload:
                sw = g.m(g.part(n) * FP16)          # swap-in staging of the partition
            else:
                sw = None
            bufs.append(g.m(n * FP16))
            if sw is not None:
                g.f(sw)
        gathered[l] = bufs

    def release(l):
        if l in gathered:
            g.free_all(gathered.pop(l))

    def param_grad(key, numel):
        if key in grads:
            return
        if zero:
            # ZeRO-3: autograd allocates the full gradient, which is copied
            # into the (pre-allocated) reduce-scatter bucket and freed; the
            # partition lives in a flat buffer allocated at setup.
            full = g.m(numel * FP16)
            g.f(full)
        else:
            gt = g.m(numel * FP16)
            if spec.offload:
                g.f(gt)
            else:
                grads[key] = gt

    def attn_fwd(l, keep):
        """Allocations of one attention block forward. Returns the tensors
        that backward consumes (or, with keep=False, frees them)."""
        saved = []
        ln1 = g.m(A)
        saved.append(ln1)
        if M.style == "neox":
            qkv = g.m(3 * A)
            saved.append(qkv)
        else:
            q, k, v = g.m(A), g.m(A), g.m(A)
            saved += [q, k, v]
        if lora:
            # PEFT-style LoRA branch per target projection: dropout(x) -> x@A
            # -> @B -> scale -> add into the base projection output.
            for tname in M.lora_targets():
                out = (3 * A) if tname == "qkv_w" else A
                drop = g.m(A)
                xa = g.m(b * s * R * FP16)
                xb = g.m(out)
                sc = g.m(out)
                g.f(xb)
                summ = g.m(out)
                g.f(sc)
                g.f(summ)
                saved += [drop, xa]
        if spec.flash:
            lse = g.m(b * h * s * FP32)
            saved.append(lse)
        else:
            sc = g.m(SC)
            pr = g.m(SC)
            g.f(sc)
            saved.append(pr)
            if use_dropout:
                mk = g.m(MK, mask=True)
                dp = g.m(SC)
                saved += [mk, dp]
        ctx = g.m(A)
        saved.append(ctx)
        o = g.m(A)
        if use_dropout:
            mk2 = g.m(MKd, mask=True)
            do = g.m(A)
            g.f(o)
            saved.append(mk2)
            o = do
        h1 = g.m(A)
        g.f(o)
        saved.append(h1)
        return saved

    def mlp_fwd(l):
        saved = []
        ln2 = g.m(A)
        saved.append(ln2)
        if M.style == "llama":
            gt, up = g.m(AF), g.m(AF)
            act = g.m(AF)
            prod = g.m(AF)
            saved += [gt, up, act, prod]
        else:
            fc1 = g.m(AF)
            act = g.m(AF)
            saved += [fc1, act]
        o = g.m(A)
        if use_dropout:
            mk = g.m(MKd, mask=True)
            do = g.m(A)
            g.f(o)
            saved.append(mk)
            o = do
        out = g.m(A)
        g.f(o)
        return saved, out

    iter_starts = []
    x = None
    for it in range(spec.iters):
        iter_starts.append(len(g.sa.events))
        # ---------------- forward ----------------
        ids = g.m(b * s * 8)                       # int64 input ids (small path)
        lbl = g.m(b * s * 8)
        x = g.m(A)                                 # embeddings output
        if zero:
            gather(-1)
        layer_in = [x]
        saved_by_layer = {}
        for l in range(M.layers):
            if zero or spec.offload:
                gather(l)
                if l > 0:
                    release(l - 1)                 # 1-layer prefetch overlap
            sa_ = attn_fwd(l, True)
            sm_, out = mlp_fwd(l)
            if spec.recompute:
                g.free_all(list(reversed(sa_ + sm_)))
                saved_by_layer[l] = None
            else:
                saved_by_layer[l] = sa_ + sm_
            layer_in.append(out)
        release(M.layers - 1)
        # ---------------- head ----------------
        lnf = g.m(A)
        logits = g.m(b * s * V * FP16)
        logits32 = g.m(b * s * V * FP32)           # fp32 upcast for the loss
        loss = g.m(4)
        g.f(logits)
        glog32 = g.m(b * s * V * FP32)
        g.f(logits32)
        glog = g.m(b * s * V * FP16)
        g.f(glog32)
        gx = g.m(A)
        g.free_all([glog, lnf, loss])
        if not lora:
            param_grad((-1, "lm_head" if M.style != "opt" else "embed"), V * d)
            param_grad((-1, "lnf_w"), d)
        # ---------------- backward ----------------
        for l in reversed(range(M.layers)):
            if zero or spec.offload:
                gather(l)
            if spec.recompute:
                sa_ = attn_fwd(l, True)
                sm_, out = mlp_fwd(l)
                g.f(out)
                saved = sa_ + sm_
                if zero or spec.offload:
                    # ZeRO-3 releases the weights after the recompute forward
                    # (post-forward hook) and re-gathers them for backward.
                    release(l)
                    gather(l)
            else:
                saved = saved_by_layer[l]
            # backward through the block: each saved tensor is consumed in
            # reverse order; the gradient w.r.t. the op input has the size of
            # the saved input (masks are consumed without a new gradient).
            cur = gx
            for t in reversed(saved):
                if t in g.masks:
                    g.f(t)
                    continue
                gn = g.m(g.size[t])
                g.f(t)
                g.f(cur)
                cur = gn
            for name, n in lp:
                if not lora:
                    param_grad((l, name), n)
            if lora:
                # autograd through each LoRA branch: grad of the scale, of
                # x@A (small), of dropout(x), and the accumulation into dx.
                for tname in M.lora_targets():
                    out_dim = 3 * d if tname == "qkv_w" else d
                    gsc = g.m(b * s * out_dim * FP16)
                    gxa = g.m(b * s * R * FP16)
                    g.f(gsc)
                    param_grad((l, tname + ".B"), R * out_dim)
                    gdr = g.m(A)
                    g.f(gxa)
                    param_grad((l, tname + ".A"), d * R)
                    gx2 = g.m(A)
                    g.f(gdr)
                    acc = g.m(A)
                    g.f(gx2)
                    g.f(cur)
                    cur = acc
            release(l)
            g.f(layer_in.pop())                     # layer output consumed
            gx = cur
        g.free_all([gx] + layer_in)
        layer_in = []
        if not lora:
            param_grad((-1, "embed"), V * d)
        if zero:
            release(-1)
        g.free_all([ids, lbl])
        # ---------------- optimizer step ----------------
        if zero and not spec.offload:
            if "flat" not in opt_state:
                tot = sum(g.part(n) for _, n in trainable)
                # flat fp32 master / exp_avg / exp_avg_sq / grad partitions
                opt_state["flat"] = tuple(g.m(tot * FP32) for _ in range(4))
        elif not spec.offload:
            for key, n in trainable:
                pn = g.part(n)
                if key not in opt_state:
                    opt_state[key] = (g.m(pn * FP32), g.m(pn * FP32), g.m(pn * FP32))
                tmp = g.m(pn * FP32)                # unscaled fp32 grad
                g.f(tmp)
        g.free_all([grads.pop(k) for k, _ in trainable if k in grads])
    return g.sa.array(), iter_starts


# ---------------------------------------------------------------------------
# Benchmark configurations (BASELINE.json configs)
# ---------------------------------------------------------------------------

CAP_80G = 80 * GiB
CAP_180G = 180 * GiB


def config_c2(iters: int = 30):
    """C2: OPT-1.3B full fine-tune with recomputation, batch 16, seq 512."""
    spec = FinetuneSpec(OPT_1_3B, batch=16, seq=512, iters=iters, recompute=True,
                        seed=trace_seed(2, 0))
    return finetune_trace(spec)


def config_c3(rank: int, world: int = 8, iters: int = 6):
    """C3: GPT-NeoX-20B ZeRO-3 + recomputation, per-rank b=8, s=1024."""
    spec = FinetuneSpec(GPT_NEOX_20B, batch=8, seq=1024, iters=iters, recompute=True,
                        world=world, rank=rank, seed=trace_seed(3, rank))
    return finetune_trace(spec)


C4_BATCH = [1, 2, 3, 4, 6, 8, 12, 16]
C4_SEQ = [256, 512, 1024, 2048]
C4_RANK = [8, 16, 32, 64]


def config_c4_spec(index: int, iters: int = 6) -> FinetuneSpec:
    """C4 trace `index` in [0, 4096): 256 combos {b, s, R, r} x 16 jitter seeds
    of Llama-13B LoRA + offload."""
    combo, rep = divmod(index, 16)
    bi, rest = divmod(combo, 32)
    si, rest = divmod(rest, 8)
    ri, li = divmod(rest, 4)
    return FinetuneSpec(LLAMA_13B, batch=C4_BATCH[bi], seq=C4_SEQ[si], iters=iters,
                        recompute=bool(ri), lora=True, offload=True, lora_r=C4_RANK[li],
                        seed=trace_seed(4, index), flash=True)


def config_c4(index: int, iters: int = 6):
    return finetune_trace(config_c4_spec(index, iters))
