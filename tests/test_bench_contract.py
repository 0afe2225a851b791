"""bench.py contract on CPU: the reference arm runs here (compiled reference in
oracle/_ref), so its JSON line is checked end to end; the B200 arm's line
shape is checked on the GPU box by the driver."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_available():
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    return O.ref_available()


@pytest.mark.skipif(not _ref_available(), reason="compiled reference (oracle/_ref) not available")
def test_reference_arm_json_line():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
           "--warmup", "1", "--batch", "256", "--vocab", "100000", "--slots", "4", "--dim", "8",
           "--hidden", "16,8"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "cpu_baseline"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
    # the arm is the reference alone: none of this repo's CUDA libraries mapped
    assert d["repo_so_loaded"] and all(p.startswith("oracle/_ref/") for p in d["repo_so_loaded"])
    assert d["config"]["mlp"] == "[8->16->8->1]"
    assert d["cpu_baseline_1core_full_batch"]["cores"] == 1
