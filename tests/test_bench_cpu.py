"""bench.py on the CPU: the reference arm runs the reference's CPU path (the
pinned oracle port) without importing the product package or mapping
liblch.so, on the GPU arm's exact config, and prints one contract line."""

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

PROBE = r"""
import json, runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3", "--no-cpu"]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit as e:
    assert not e.code, e.code
maps = open("/proc/self/maps").read()
print(json.dumps({"pkg": any(m.startswith("paper_1404_3458_b200") for m in sys.modules),
                  "liblch": "liblch.so" in maps}))
"""


def test_reference_arm_does_not_load_the_product():
    res = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=600,
                         env={k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE")})
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    line = json.loads(lines[0])
    probe = json.loads(lines[-1])
    assert probe == {"pkg": False, "liblch": False}
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    args = argparse.Namespace(batch=bench.BATCH, rate="1/2", groups=0)
    assert line["config"] == json.loads(json.dumps(bench.workload_config("codec", args, 1)))
