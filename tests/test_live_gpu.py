"""Live allocator over the CUDA VMM driver API:
same decisions as the oracle / replay, real memory that does not alias,
stitched buffers that stream at cudaMalloc bandwidth (north star)."""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
from tracegen import decode, synth
from tracegen import policies as P

pytestmark = pytest.mark.gpu

MiB = 1 << 20
GiB = 1 << 30


@pytest.fixture(scope="module")
def gml():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()
    from paper_2401_08156_b200 import gml as g
    torch.cuda.init()
    return g


@pytest.fixture(scope="module")
def cudart():
    L = C.CDLL("libcudart.so.12")
    L.cudaMemset.argtypes = [C.c_void_p, C.c_int, C.c_size_t]
    L.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    L.cudaMalloc.argtypes = [C.POINTER(C.c_void_p), C.c_size_t]
    L.cudaFree.argtypes = [C.c_void_p]
    L.cudaDeviceSynchronize.argtypes = []
    return L


def _drive(gml, pol, events):
    a = gml.Allocator(0, pol)
    ptr = {}
    for ev in events:
        f, slot, size = decode(ev)
        if f:
            a.free(ptr.pop(slot))
        else:
            ptr[slot] = a.malloc(size)
    return a, ptr


def _cmp_stats(live, oracle):
    skip = {"n_events", "n_events_done", "oom_event", "status"}
    diff = {k: (live[k], oracle[k]) for k in oracle if k not in skip and live[k] != oracle[k]}
    assert not diff, diff


def test_live_matches_oracle(gml):
    """The live allocator takes the oracle's decisions (identical policy code
    as the replay kernel): every statistic matches on a C2 prefix and on an
    irregular trace, for the default policy and the limit = 1 chunk variant."""
    ev, starts = synth.config_c2(iters=3)
    irr = synth.lognormal_trace(4, 3, 40, 60e6, extra_frac=0.3, interleave_frac=0.3, small_frac=0.2)
    for trace in (ev, irr):
        for pol in (P.policy(P.GMLAKE, capacity=40 * GiB), P.policy(P.GMLAKE, capacity=40 * GiB, frag_limit=2 * MiB)):
            a, ptr = _drive(gml, pol, trace)
            _, so = O.replay(trace, pol)
            _cmp_stats(a.stats(), so)
            for p in list(ptr.values()):
                a.free(p)
            a.destroy()


def test_live_memory_is_exclusive(gml, cudart):
    """Each live allocation owns its bytes (I2): fill every
    live block with its own byte after a churn that forces splits and
    stitches, then read back the first and last byte of each."""
    pol = P.policy(P.GMLAKE, capacity=8 * GiB, frag_limit=2 * MiB)
    trace = synth.random_trace(21, 600, 40, sizes=[1 * MiB, 2 * MiB, 6 * MiB, 10 * MiB, 34 * MiB, 70 * MiB],
                               balanced=False)
    a, ptr = _drive(gml, pol, trace)
    st = a.stats()
    assert st["n_stitch"] > 0 and st["n_split"] > 0
    sizes = {}
    for ev in trace:
        f, slot, size = decode(ev)
        if not f:
            sizes[slot] = size
    for i, (slot, p) in enumerate(ptr.items()):
        assert cudart.cudaMemset(p, (i % 250) + 1, sizes[slot]) == 0
    assert cudart.cudaDeviceSynchronize() == 0
    b = C.c_ubyte()
    for i, (slot, p) in enumerate(ptr.items()):
        for off in (0, sizes[slot] - 1):
            assert cudart.cudaMemcpy(C.byref(b), p + off, 1, 2) == 0
            assert b.value == (i % 250) + 1, (slot, off)
    for p in list(ptr.values()):
        a.free(p)
    a.destroy()


def test_live_errors_and_oom(gml):
    pol = P.policy(P.GMLAKE, capacity=64 * MiB, frag_limit=2 * MiB)
    a = gml.Allocator(0, pol)
    p1 = a.malloc(32 * MiB)
    p2 = a.malloc(30 * MiB)
    with pytest.raises(gml.GmlError) as e:
        a.malloc(16 * MiB)                      # S5
    assert e.value.code == gml.GML_ERR_OOM
    a.free(p2)
    p3 = a.malloc(16 * MiB)                     # usable after the OOM
    with pytest.raises(gml.GmlError):
        a.free(p3 + 4096)                       # unknown pointer
    a.free(p3)
    with pytest.raises(gml.GmlError):
        a.free(p3)                              # double free
    with pytest.raises(gml.GmlError):
        a.destroy()                             # p1 still live
    a.free(p1)
    a.destroy()


def test_stitched_buffer_streams_at_native_bandwidth(gml, cudart):
    """K2 over an 8 GiB S3-stitched buffer made of 64 non-adjacent 128 MiB
    pBlocks vs a cudaMalloc'd buffer: same HBM bandwidth (north star)."""
    pol = P.policy(P.GMLAKE, capacity=40 * GiB)
    a = gml.Allocator(0, pol)
    blocks = [a.malloc(128 * MiB) for _ in range(128)]
    for p in blocks[::2]:
        a.free(p)
    stitched = a.malloc(8 * GiB)
    st = a.stats()
    assert st["state_count"][2] == 1            # S3: stitched from the 64 holes
    assert a.driver_calls()[1] == 128 * 64      # one cuMemCreate per 2 MiB chunk, none for the stitch
    n = 8 * GiB
    dst = C.c_void_p()
    src = C.c_void_p()
    assert cudart.cudaMalloc(C.byref(dst), n) == 0
    assert cudart.cudaMalloc(C.byref(src), n) == 0
    gml.gml_stream_copy(src.value, dst.value, n, 2)          # warm
    t_native = min(gml.gml_stream_copy(src.value, dst.value, n, 5) for _ in range(3))
    gml.gml_stream_copy(stitched, dst.value, n, 2)
    t_stitch = min(gml.gml_stream_copy(stitched, dst.value, n, 5) for _ in range(3))
    bw_native = 2 * n / t_native / 1e6
    bw_stitch = 2 * n / t_stitch / 1e6
    print(f"stream copy GB/s: native {bw_native:.1f} stitched {bw_stitch:.1f}")
    assert abs(bw_stitch / bw_native - 1) < 0.02          # C5 pass criterion
    cudart.cudaFree(dst)
    cudart.cudaFree(src)
    a.free(stitched)
    for p in blocks[1::2]:
        a.free(p)
    a.destroy()


def test_vmm_profile_probe(gml):
    """f2: gml_vmm_profile measures each VMM API for one allocation built from
    chunks (Table 1 / fig:virtual method); totals add up,
    a 2 MiB-chunk build costs more than a 128 MiB-chunk one, and one
    cuMemSetAccess over the range is cheaper than one per chunk."""
    L = gml.lib()
    out2 = (C.c_double * 10)()
    out128 = (C.c_double * 10)()
    assert L.gml_vmm_profile(0, 256 * MiB, 2 * MiB, 3, out2) == 0
    assert L.gml_vmm_profile(0, 256 * MiB, 128 * MiB, 3, out128) == 0
    a, b = list(out2), list(out128)
    assert all(x > 0 for x in a[:8]) and all(x > 0 for x in b[:8])
    assert a[8] == pytest.approx(a[2] + a[3] + a[4] + a[5]) and a[9] == pytest.approx(a[2] + a[3] + a[4] + a[6])
    assert a[3] > b[3] and a[8] > b[8]          # 128 chunks cost more than 2
    assert a[6] < a[5]                          # one set-access over the range < one per chunk
    bad = (C.c_double * 10)()
    assert L.gml_vmm_profile(0, 3 * MiB, 2 * MiB, 1, bad) == gml.GML_ERR_INVALID


def test_live_replay_oracle_agree_per_event_c2(gml):
    """Three-way decision check on the whole C2 trace (BASELINE configs[1],
    121,968 events): the live allocator (real VMM calls), K1 on the GPU and
    the CPU oracle give the same assignment record for every event, under
    the default policy V2 and the literal-D8 policy V7 (PAPER.md L306-327,
    L381-387: the live path is the same policy as the replay)."""
    import torch
    from paper_2401_08156_b200 import replay as R
    ev, _ = synth.config_c2()
    pols = [P.variants(80 * GiB)[2], P.variants(80 * GiB)[7]]
    asg, _ = R.run(R.upload([ev]), pols)
    torch.cuda.synchronize()
    k1 = asg.cpu().numpy().view(np.uint64)
    for p, pol in enumerate(pols):
        ao, so = O.replay(ev, pol)
        a = gml.Allocator(0, pol)
        rc, done, rec, ns = a.trace(ev)
        assert rc == 0 and done == len(ev)
        bad = np.nonzero(rec != ao)[0]
        assert len(bad) == 0, [(int(i), O.rec_fields(rec[i]), O.rec_fields(ao[i])) for i in bad[:3]]
        assert np.array_equal(k1[p], ao), p
        # gml_live_trace frees the blocks still live at the end (include/gml.h):
        # every other statistic is the oracle's, and nothing stays active
        st = a.stats()
        assert st["final_active_bytes"] == 0
        st["final_active_bytes"] = so["final_active_bytes"]
        _cmp_stats(st, so)
        a.destroy()


def test_live_driver_oom_is_recoverable(gml):
    """A request the device cannot back (cuMemCreate fails part-way) is the
    paper's S5 ('If the Alloc function call fails, GMLake immediately
    reports an OOM'): the chunks already created are rolled
    back and the allocator keeps working."""
    import torch
    free_b, total_b = torch.cuda.mem_get_info(0)
    pol = P.policy(P.GMLAKE, capacity=250 * GiB, frag_limit=2 * MiB)
    a = gml.Allocator(0, pol)
    p1 = a.malloc(64 * MiB)
    with pytest.raises(gml.GmlError) as e:
        a.malloc(free_b + 8 * GiB)
    assert e.value.code == gml.GML_ERR_OOM
    st = a.stats()
    assert st["state_count"][4] == 1 and st["final_reserved_bytes"] == 64 * MiB
    assert torch.cuda.mem_get_info(0)[0] > free_b - 1 * GiB      # nothing leaked
    p2 = a.malloc(1 * GiB)
    a.free(p1)
    a.free(p2)
    a.destroy()


def test_live_stitchfree_defers_unmap(gml, cudart):
    """StitchFree of an sBlock whose VA a queued copy is
    still reading: the unmap waits behind an event on the allocator's stream,
    so the copy completes correctly and the evicting gml_malloc does not
    stall the host for the GPU's queued work."""
    import time
    import torch
    pol = P.policy(P.GMLAKE, capacity=40 * GiB, frag_limit=2 * MiB, spool_max_inactive_bytes=0)
    a = gml.Allocator(0, pol)
    s = torch.cuda.Stream()
    a.set_stream(s)
    blocks = [a.malloc(64 * MiB) for _ in range(64)]
    for p in blocks[::2]:
        a.free(p)
    stitched = a.malloc(2 * GiB)                        # S3 over the 32 holes
    assert a.stats()["state_count"][2] == 1
    n = 2 * GiB
    src = torch.arange(n // 8, dtype=torch.int64, device="cuda")
    dst = torch.empty(n // 8, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    rt = cudart
    rt.cudaMemcpyAsync.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
    with torch.cuda.stream(s):
        assert rt.cudaMemcpyAsync(stitched, src.data_ptr(), n, 3, C.c_void_p(s.cuda_stream)) == 0
        for _ in range(20):                              # ~20 x 2 GiB of queued reads through the stitched VA
            assert rt.cudaMemcpyAsync(dst.data_ptr(), stitched, n, 3, C.c_void_p(s.cuda_stream)) == 0
    unmaps0 = a.driver_calls()[4]
    a.free(stitched)
    t0 = time.perf_counter()
    q = a.malloc(4 * MiB)                               # byte cap 0: evicts the inactive stitched sBlock
    host_s = time.perf_counter() - t0
    assert a.stats()["n_evict"] >= 1
    assert a.driver_calls()[4] == unmaps0               # unmap deferred: the copies are still queued
    s.synchronize()
    assert torch.equal(dst, src)                        # the queued reads saw the mapped data
    r = a.malloc(4 * MiB)                               # drains the deferred unmap
    assert a.driver_calls()[4] > unmaps0
    assert host_s < 0.005, host_s                       # no device-wide wait in the malloc
    for p in (q, r, *blocks[1::2]):
        a.free(p)
    a.destroy()
