"""Build library variants build/libgml_<name>.so with extra -D flags (for
tools/gpu_variants.sh). Usage: python tools/build_variants.py name=FLAG,FLAG ..."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import __graft_entry__ as g  # noqa: E402

for spec in sys.argv[1:]:
    name, _, flags = spec.partition("=")
    fl = tuple(f if f.startswith("-") else f"-D{f}" for f in flags.split(",") if f)   # raw nvcc flags or -D
    g.build(extra_flags=fl, lib=g.ROOT / "build" / f"libgml_{name}.so")
    print("built", name, fl)
