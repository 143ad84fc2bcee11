"""CPU: the reference arm of bench.py (the reference algorithm on every host
core, shared-memory arrays, row-range FFTs in the workers) runs, prints the
contract's JSON line, and its transform round-trips (small N)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--n", "16", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "transforms/s"
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["value"] == line["value"]
    rt = float(line["cpu_baseline"]["sample"].split("round trip ")[1])
    assert rt < 1e-12
