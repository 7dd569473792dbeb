"""NEXT rows f3 and f1 on a real PyTorch workload (tests/workloads/torch_train.py,
run in fresh processes):

f3  GMLake as PyTorch's allocator (CUDAPluggableAllocator over the live VMM
    allocator, the paper's deployment mode): the
    training run is unchanged (same losses) and the allocator's statistics
    are consistent; after the first batch-size cycle the VMM path serves
    requests by exact matches (S1), the convergence of PAPER.md L558-561.
f1  A PyTorch memory snapshot of the same run, converted by
    tracegen.snapshot, replays on the GPU bit-exact against the oracle for
    all 8 policy variants; BFC-torch (V0) reproduces the caching allocator's
    own peaks (SURVEY §8(c) pin I13: requested and allocated bytes).
"""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from tracegen import snapshot
from tracegen import policies as P

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
WORKLOAD = ROOT / "tests" / "workloads" / "torch_train.py"
GiB = 1 << 30


def _run(*args):
    r = subprocess.run([sys.executable, str(WORKLOAD), *args], capture_output=True, text=True, timeout=900,
                       cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()


def test_training_under_gmlake_allocator(built):
    base = _run("--steps", "9")
    g = _run("--steps", "9", "--gml")
    print(json.dumps({"default": base, "gmlake": g}))
    np.testing.assert_allclose(g["losses"], base["losses"], rtol=1e-6, atol=0)
    s = g["gml"]
    assert s["status"] == 0 and s["oom_event"] == -1
    assert 0 < s["peak_active_bytes"] <= s["peak_reserved_bytes"]
    assert s["state_count"][0] > 0                       # S1 exact matches happen
    steps = g["per_step"]
    vmm = [sum(c[:5]) for c in steps]
    s234 = [sum(c[1:4]) for c in steps]
    # after the first cycle of batch sizes (3 steps) the VMM path is all S1
    assert sum(vmm[6:]) > 0 and sum(s234[6:]) == 0, steps


def test_snapshot_replay_parity_and_torch_peaks(built, tmp_path):
    import torch
    from paper_2401_08156_b200 import replay as R
    snap = tmp_path / "snap.pkl"
    base = _run("--steps", "6", "--snapshot", str(snap))
    ev = snapshot.load(str(snap))
    assert len(ev) > 1000
    pols = P.variants(capacity=80 * GiB)
    batch = R.upload([ev])
    asg, st = R.run(batch, pols)
    torch.cuda.synchronize()
    stats = R.decode_stats(st, 1, len(pols))[0]
    a = asg.cpu().numpy().view(np.uint64)
    for p, pol in enumerate(pols):
        ao, so = O.replay(ev, pol)
        assert np.array_equal(a[p], ao), p
        assert stats[p] == so, p
    t = base["torch"]
    v0 = stats[0]
    print(json.dumps({"torch": t, "bfc_torch": {k: v0[k] for k in ("peak_requested_bytes", "peak_active_bytes",
                                                                    "peak_reserved_bytes")},
                      "events": int(len(ev))}))
    assert v0["peak_requested_bytes"] == t["requested_bytes.all.peak"]
    assert v0["peak_active_bytes"] == t["allocated_bytes.all.peak"]
    # segment sizes and release rules (D21) decide the reserved peak
    assert v0["peak_reserved_bytes"] == t["reserved_bytes.all.peak"]
