"""bench.py end to end on one GPU at a small configuration: the JSON line
carries the contract's keys and plausible values (guards the harness the
driver runs at round end)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line_small():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "bench.py", "--shape", "mixtral-8x7b", "--b-a", "64", "--micro-batches", "1",
           "--layers", "1", "--steps", "3", "--warmup", "3", "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "roofline", "e2e", "gpu_launches", "clocks", "m2n"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3
    assert d["roofline"]["achieved"] > 0 and d["roofline"]["bound"] == "tensor"
    assert d["e2e"]["results_checked"] and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["m2n"]["p50_us"] > 0 and d["m2n"]["steady_state"]["per_trip_p50_us"] > 0
