"""bench.py's driver contract, run end to end on the GPU (short runs):

* N = 1: one JSON line with the required keys (metric, value, e2e with
  h2d/d2h bytes, roofline, cpu_baseline, clocks, gpu_launches) and a
  consistent ms_per_step;
* N = 2 without torchrun: bench.py re-launches itself under
  torch.distributed.run; with BENCH_BACKEND=gloo both ranks share the one
  GPU (host-staged collectives: a functional check of the slab path, not a
  timing);
* --impl reference: the CPU arm's line.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _run(args, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, cwd=ROOT, env=e, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert lines, out.stdout[-2000:]
    return json.loads(lines[-1])


def test_single_gpu_line():
    d = _run(["--config", "2", "--steps", "4", "--warmup", "3", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "gpu_launches", "e2e", "roofline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert "e2e_sync" in d and d["roofline"]["bound"] == "hbm"


def test_two_ranks_slab_functional():
    d = _run(["--gpus", "2", "--config", "2", "--steps", "4", "--warmup", "3", "--no-cpu-baseline"],
             env={"BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["config"]["parallelism"].startswith("slab") or "slab" in json.dumps(d["config"])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "2", "--steps", "2", "--warmup", "1"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0
