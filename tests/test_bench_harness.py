"""bench.py's contract: one JSON line with the driver's keys, and the N>1
path (torchrun, one rank per GPU) exercised on a one-GPU box through the
VMT_BENCH_SHARED_GPU test hook (gloo collectives, every rank on cuda:0): the
per-rank ranges of a weak N=2 run and of a strong N=2 run fold to the same
checksum as N=1 over the same words."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "clocks", "e2e"}


def run(args, env=None, nproc=1, port=29561):
    e = dict(os.environ, **(env or {}))
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", "bench.py", *args]
    else:
        cmd = [sys.executable, "bench.py", *args]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_single_and_multi_rank_paths():
    words = str(1 << 29)
    one = run(["--words", str(1 << 30), "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-extras"])
    assert KEYS <= set(one) and one["n_gpus"] == 1 and one["value"] > 0
    r = one["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.2 and r["peak"] > 0
    assert one["gpu_launches"] >= 3 and one["e2e"]["d2h_bytes_per_step"] == 4 << 30
    shared = {"VMT_BENCH_SHARED_GPU": "1"}
    weak = run(["--gpus", "2", "--words", words, "--steps", "3", "--warmup", "3", "--no-extras"], shared, 2, 29562)
    strong = run(["--gpus", "2", "--words", str(1 << 30), "--scaling", "strong", "--steps", "3", "--warmup", "3",
                  "--no-e2e"], shared, 2, 29563)
    assert weak["n_gpus"] == strong["n_gpus"] == 2
    # N > 1 end to end: every rank fills its own pinned host buffer
    assert weak["e2e"]["d2h_bytes_per_step"] == 2 * 4 * (1 << 29) and weak["e2e"]["value"] > 0
    assert weak["checksum_xor"] == strong["checksum_xor"] == one["checksum_xor"]


@pytest.mark.gpu
def test_reference_arm_under_torchrun():
    d = run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"],
            {"VMT_BENCH_SHARED_GPU": "1"}, 2, 29564)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["cores"] >= 1 and d["e2e"]["h2d_bytes_per_step"] == 0
