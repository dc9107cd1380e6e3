"""CPU: bench.py's reference arm (the oracle port on the host) prints one valid JSON line."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-sample-n", "192"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, check=True).stdout.strip().splitlines()
    line = json.loads(out[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "TFLOP/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    # the line reports the size actually run (a bounded sample of config 4), never the
    # config's nominal size (the ratio was void because of that)
    assert line["config"]["n"] == 192 and line["config"]["m"] == 192 and line["config"]["q"] == 2
    assert line["config"]["sample_of"] == "config4" and "192x192" in line["cpu_baseline"]["sample"]
    assert line["source"]["sources_sha256"]
