"""bench.py end to end on the GPU (short runs): the JSON line's contract, the e2e host-buffer
check against the device path, and the phase canaries (the fused finisher's counters stay
consistent across every bench section)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
        "gpu_launches", "clocks"}


@pytest.mark.parametrize("mode", ["train", "infer"])
def test_bench_short_run(dfx, mode):
    env = dict(os.environ, DFX_BENCH_CANARY="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--mode", mode,
                        "--steps", "8", "--warmup", "3", "--no-cpu-baseline", "--no-cpu-full-module", "--e2e-steps", "2",
                        "--lora-steps", "2", "--variant-steps", "8", "--prof-steps", "4"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert KEYS <= set(line), KEYS - set(line)
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    st = line["roofline_step"]
    assert st["bytes_per_step"] > 0 and 0 < st["frac_of_floor"] <= 1.0, st
    canaries = [l for l in (r.stdout + r.stderr).splitlines() if "canary after" in l]
    assert canaries and all(l.rstrip().endswith("ok") for l in canaries), canaries
