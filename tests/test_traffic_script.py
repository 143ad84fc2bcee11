"""The evidence pipeline behind bench.py's roofline.traffic: the committed
ncu launch list -> scripts/traffic_from_launches.py -> the committed traffic
JSON, and bench.measured_traffic reads that JSON for the same workload only."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_traffic_json_reproduces_from_launch_list():
    csv = os.path.join("profiles", "r02_launches_bench_n1024.csv")
    out = subprocess.run([sys.executable, os.path.join("scripts", "traffic_from_launches.py"), csv],
                         cwd=ROOT, check=True, capture_output=True, text=True).stdout
    got = json.loads(out)
    with open(os.path.join(ROOT, "profiles", "r02_traffic_n1024.json")) as fh:
        want = json.load(fh)
    assert got == want
    assert got["n"] == 1024
    # one direction = the chain-kernel stages plus the stage-kernel final (and combine) stages
    for d in ("fwd", "inv"):
        assert got[d]["chain_kernel_launches"] >= 1
        assert got[d]["launches"] > got[d]["chain_kernel_launches"]
        assert 13.0e9 < got[d]["traffic_bytes"] < 16.0e9
    share = got["step"]["share_pct"]
    assert abs(sum(share.values()) - 100.0) < 0.5


def test_bench_reads_traffic_for_the_same_workload_only():
    sys.path.insert(0, ROOT)
    import bench
    t = bench.measured_traffic(1024, 1, 0.0)
    assert t is not None and 13.0e9 < t < 16.0e9
    assert bench.measured_traffic(512, 1, 0.0) is None
    assert bench.measured_traffic(1024, 2, 0.0) is None
    assert bench.measured_traffic(1024, 1, 0.5) is None
