"""Every one-line oracle mutant of tools/oracle_mutants.py (plausible slips
in Alg. 1, StitchFree, BFC/D21 and the accounting) must fail the non-GPU pins:
the pins constrain the oracle, not just agree with it."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_every_oracle_mutant_is_killed():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "oracle_mutants.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "SURVIVED" not in r.stdout and "stale" not in r.stdout
