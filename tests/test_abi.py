"""The C ABI library loads on a CPU box and exports every entry point that
include/gml.h declares; host-only helpers behave (no GPU compute here)."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def gml():
    import __graft_entry__ as ge
    ge.build()
    from paper_2401_08156_b200 import gml as g
    g.lib()
    return g


def _declared():
    hdr = (ROOT / "include" / "gml.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:gml_status|double|uint32_t|float|const char\*|void\s*\*|void)\s*(gml_\w+)\s*\(", hdr, re.M)))


def test_exports_every_declared_symbol(gml):
    names = _declared()
    assert len(names) == 23, names
    out = subprocess.run(["nm", "-D", "--defined-only", str(gml.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gml_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    bound = {s[0] for s in gml.SIGNATURES}
    assert set(names) <= bound, set(names) - bound


def test_struct_sizes_match_header(gml):
    import ctypes as C
    assert C.sizeof(gml.gml_policy) == 56
    assert C.sizeof(gml.gml_stats_t) == 272


def test_validate_host(gml):
    from tracegen import pack, synth
    assert gml.gml_trace_validate(synth.fig_intro()) == 9
    with pytest.raises(gml.GmlError):
        gml.gml_trace_validate(pack([("f", 3, 0)]))
    with pytest.raises(gml.GmlError):
        gml.gml_trace_validate(pack([("m", 0, 1), ("m", 0, 1)]))


def test_metrics_host(gml):
    """PAPER.md L629-635 via the C ABI's host functions, against the oracle's
    transcription of the formulas."""
    from oracle import metrics as M
    for a, r in [(72, 80), (0, 0), (5, 5), (1, 3)]:
        s = dict(peak_active_bytes=a, peak_reserved_bytes=r)
        assert gml.gml_utilization(s) == pytest.approx(M.utilization(a, r))
        assert gml.gml_utilization(s) + gml.gml_fragmentation(s) == pytest.approx(1.0)


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle or falls back to CPU."""
    for p in (ROOT / "paper_2401_08156_b200").rglob("*.py"):
        src = p.read_text()
        assert "oracle" not in src.replace("oracle/", ""), p
    for p in (ROOT / "paper_2401_08156_b200" / "csrc").rglob("*"):
        if p.suffix in (".cu", ".cuh", ".cpp", ".h"):
            assert "gml_oracle" not in p.read_text(), p
