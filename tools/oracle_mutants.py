"""Mutation check of the oracle's pins (test infrastructure).

Each mutant is a one-line change of oracle/gml_oracle.cpp that a plausible
slip would make. The tool builds every mutant in a scratch directory, runs
the non-GPU oracle pins against it (GML_ORACLE_LIB) and reports whether the
pins kill it. Every mutant must die:

    python tools/oracle_mutants.py [-k name] [--tests tests/test_oracle_pins.py ...]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "oracle" / "gml_oracle.cpp"
TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_properties.py"]

# name -> (exact text in the oracle, replacement, what the slip means)
MUTANTS = {
    "bfc_no_release_retry": ("        release_free_segments(st);\n        if (other_reserved",
                             "        if (other_reserved",
                             "BFC OOM without PyTorch's release-and-retry (D21)"),
    "lru_most_recent": ("      if (!v || s->last_use < v->last_use) v = s;\n    }\n    return v;",
                        "      if (!v || s->last_use > v->last_use) v = s;\n    }\n    return v;",
                        "count-cap StitchFree evicts the MOST recently used sBlock (P:L487)"),
    "lru_no_born_exclusion": ("      if (s->born == malloc_serial) continue;\n", "",
                              "count-cap victim may be an sBlock created during this malloc (D17)"),
    "invalidate_nothing": ("      for (SBlock* s : dead_s) evict(s);\n", "",
                           "SPLIT_INVALIDATES keeps the sBlocks over the split parent (S:L324)"),
    "large_split_ge": ("    return rem > BFC_SMALL_SIZE;", "    return rem >= BFC_SMALL_SIZE;",
                       "large-pool split when the remainder is exactly 1 MiB (D21)"),
    "large_buffer_40": ("constexpr uint64_t BFC_LARGE_BUFFER = 20ull << 20;",
                        "constexpr uint64_t BFC_LARGE_BUFFER = 40ull << 20;",
                        "kLargeBuffer 40 MiB instead of 20 MiB (D21)"),
    "s5_ge": ("    if (reserved() + (uint64_t)shortfall * G() > pol.capacity_bytes) {\n      // ---- S5",
              "    if (reserved() + (uint64_t)shortfall * G() >= pol.capacity_bytes) {\n      // ---- S5",
              "S5 when the shortfall exactly fills capacity (P:L528)"),
    # further slips of the same kind
    "s2_tie_lowest": ("      if (p->n >= b) {\n        CB.assign(1, p);",
                      "      if (p->n >= b) {\n        if (!CB.empty() && CB[0]->n == p->n) continue;\n        CB.assign(1, p);",
                      "S2 tie -> lowest ordinal instead of the replace-loop's last (D6)"),
    "s1_pblock_before_sblock": ("      bool spool = (pass == 0) != pfirst;", "      bool spool = (pass == 0) == pfirst;",
                                "S1 searches the pPool before the sPool (D5)"),
    "d14_split_whole_last": ("        uint32_t n = (uint32_t)(b - (CBsize - last->n));                          // D14",
                             "        uint32_t n = (uint32_t)(b - CBsize + last->n + 1);",
                             "S3 split of the last candidate off by one (D14)"),
    "small_path_le": ("    if (raw < pol.small_threshold_bytes) return malloc_bfc(slot, raw, out);",
                      "    if (raw <= pol.small_threshold_bytes) return malloc_bfc(slot, raw, out);",
                      "a 2 MiB request takes the small path (D1)"),
    "bfc_tie_highest_addr": ("    return a->off < b->off;\n  }\n};", "    return a->off > b->off;\n  }\n};",
                             "BFC ties go to the highest address (D22)"),
    "companion_not_lru_fresh": ("    SBlock* s = new SBlock{next_s++, {}, 0, ++T, malloc_serial};",
                                "    SBlock* s = new SBlock{next_s++, {}, 0, 0, malloc_serial};",
                                "a new sBlock's LRU key is not a fresh touch (S:L328)"),
    "s1_no_touch": ("            s->last_use = ++T;\n            st.state_count[ST_S1 - 1]++;",
                    "            st.state_count[ST_S1 - 1]++;",
                    "S1 reuse does not refresh the sBlock's LRU key (S:L328)"),
    "frag_limit_gt": ("  bool eligible(const PBlock* p) const { return (uint64_t)p->n * G() >= pol.frag_limit_bytes; }",
                      "  bool eligible(const PBlock* p) const { return (uint64_t)p->n * G() > pol.frag_limit_bytes; }",
                      "a block exactly at the fragmentation limit is not eligible (D8, P:L571)"),
    "bytecap_mru": ("        if (s_inactive(s) && (!v || s->last_use < v->last_use)) v = s;",
                    "        if (s_inactive(s) && (!v || s->last_use > v->last_use)) v = s;",
                    "byte-cap StitchFree releases the most recently used sBlock first (P:L487)"),
    "split_map_calls": ("    st.vmm_calls[V_MAP] += pn;", "    st.vmm_calls[V_MAP] += 1;",
                        "Split remaps one chunk instead of all of them (D26, P:L378)"),
    "companion_order": ("      if (!(pol.flags & F_NO_COMPANION)) stitch({fr.first, fr.second}, true);\n      bind_p",
                        "      if (!(pol.flags & F_NO_COMPANION)) stitch({fr.second, fr.first}, true);\n      bind_p",
                        "S2 companion members in the order [R, F] (D11, D13)"),
    "s4_never_stitch": ("    if (CB.empty()) {\n      bind_p(slot, p, raw);", "    if (true) {\n      bind_p(slot, p, raw);",
                        "S4 ignores the candidates and assigns the fresh pBlock alone (P:L525-527)"),
    "free_keeps_requested": ("    requested -= x.raw;\n", "", "a free does not return its requested bytes (D20)"),
    "no_reserved_peak": ("    st.peak_reserved_bytes = std::max(st.peak_reserved_bytes, reserved());\n", "",
                         "peak reserved bytes never sampled (P:L630)"),
    "s5_no_small_release": ("      bfc.release_free_segments(st);\n    }\n", "    }\n",
                            "S5 without the small path's release of its free segments (D16)"),
    "gate_le": ("&& raw < pol.frag_limit_bytes) return malloc_bfc", "&& raw <= pol.frag_limit_bytes) return malloc_bfc",
                "a request exactly at the fragmentation limit takes the small path (D8')"),
    "gate_ignored": ("    if ((pol.flags & F_LIMIT_GATES_REQUEST) && raw", "    if (false && raw",
                     "LIMIT_GATES_REQUEST has no effect (D8')"),
}


def build(text: str, out: Path) -> None:
    src = out.with_suffix(".cpp")
    src.write_text(text)
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", str(src), "-o", str(out)])


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default=None, help="only mutants whose name contains this")
    ap.add_argument("--tests", nargs="*", default=TESTS)
    ap.add_argument("-j", type=int, default=min(8, os.cpu_count() or 2))
    a = ap.parse_args()
    base = SRC.read_text()
    todo = {k: v for k, v in MUTANTS.items() if a.k is None or a.k in k}
    survived = []
    with tempfile.TemporaryDirectory() as td:
        from concurrent.futures import ThreadPoolExecutor

        def run(item):
            name, (old, new, why) = item
            if base.count(old) != 1:
                return name, why, "stale", ""
            lib = Path(td) / f"mut_{name}.so"
            build(base.replace(old, new), lib)
            env = dict(os.environ, GML_ORACLE_LIB=str(lib))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                                *a.tests], cwd=ROOT, env=env, capture_output=True, text=True)
            fail = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            return name, why, "killed" if r.returncode != 0 else "SURVIVED", fail[0] if fail else ""

        with ThreadPoolExecutor(a.j) as ex:
            for name, why, verdict, by in ex.map(run, todo.items()):
                print(f"{verdict:8s} {name:26s} {why}\n{'':9s}{by}", flush=True)
                if verdict != "killed":
                    survived.append(name)
    print(f"{len(todo) - len(survived)}/{len(todo)} mutants killed")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
