"""bench.py's CPU-side contract: the reference arm (the reference's own C++ compiled in
oracle/_ref) prints one JSON line with the fields the driver reads; the algorithmic
byte / flop model matches SURVEY sec. 8(d)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_algorithmic_model_c2():
    import bench
    a = bench.algorithmic(bench.CONFIGS["c2"])
    assert a["u_rowdot_tc"][1] == 2.0 * 8192 * 8192 * 384                 # 51.5 GFLOP
    assert a["compose_fwd"][2] == 3 * 2 * 4096 * 8192 + 4 * 8192          # 201.4 MB
    assert a["compose_fwd_dual"][2] == 4 * 2 * 4096 * 8192 + 4 * 8192
    assert a["norm_total"][2] == 2 * (8192 * 8192 + 384 * 8192 + 8192 * 384) + 4 * 8192


def test_reference_arm_json(reference):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "0",
                          "--no-cpu-full-module"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "modules/s" and line["value"] > 0
    assert line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["mode"] == "train"


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` without torchrun re-execs itself under torch.distributed.run: two
    ranks rendezvous on 127.0.0.1, reduce their timings (max) and rank 0 reports n_gpus 2.
    --stub swaps the GPU work for a CPU loop on gloo (this box has no GPU)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--stub",
                          "--steps", "5"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["ranks_reporting"] == 2 and line["stub"] is True


def test_reference_arm_nonzero_rank_exits_quietly():
    """Under torchrun (N > 1) only rank 0 runs the reference arm; the others exit 0 with no line."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2"], capture_output=True, text=True, timeout=120, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip() == ""
