"""The bench.py contract on CPU: the reference arm (the oracle on a bounded sample) prints one JSON
line with the keys the driver reads, for an assembly config, a discrete-operator config and the
post-assembly configs; the CPU baseline helper reports its sample and core count."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cfg", ["C2", "C4-G"])
def test_reference_arm_json_line(cfg):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", cfg,
                        "--steps", "1", "--warmup", "0", "--ref-n", "3"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "impl",
              "cpu_baseline", "e2e", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.parametrize("cfg", ["C2-A4", "C2-X", "C2-V"])
def test_cpu_baseline_helper(cfg):
    sys.path.insert(0, ROOT)
    import bench
    c = bench.cpu_baseline(cfg, 4)
    assert c["value"] and c["value"] > 0, c
    assert c["cores"] == 1 and c["kind"] == "oracle" and "sample" in c
