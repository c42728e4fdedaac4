"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line (the reference CPU engine from oracle/_ref), and the string-gate counts
bench.py uses, pinned against the reference engine's own count."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "oracle", "_ref", "libppref.so")


@pytest.mark.skipif(not os.path.exists(REF), reason="reference library not built")
def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "config1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "string_gates_per_s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    import bench
    assert line["config"] == bench.config_dict(type("A", (), {"workload": "config1"})(), bench.WORKLOADS["config1"], 1)
    assert line["cpu_baseline"]["sample_string_gates_per_step"] == bench.COUNTS["config1"][0]


@pytest.mark.skipif(not os.path.exists(REF), reason="reference library not built")
def test_string_gate_counts_match_reference():
    import bench
    for wl in ("config1", "config0_t8"):
        _, sg = bench.cpu_reference_time(bench.WORKLOADS[wl], 1, 0, os.cpu_count() or 1)
        assert int(sg) == bench.COUNTS[wl][0], wl
