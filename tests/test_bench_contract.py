"""bench.py's output contract, checked on CPU (no GPU needed):
the reference arm (the oracle, --impl reference) prints one JSON line with the
required keys, only rank 0 prints under a multi-rank launch, and the product
arm fails loudly instead of falling back to the CPU when CUDA is absent."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env_extra=None, timeout=300):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                          env=env, capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = _bench(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "tok/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 1
    assert d["warmup"] >= 3                      # the contract's minimum is enforced
    assert d["vs_baseline"] is None               # BASELINE.md has no number for this metric
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    r = _bench(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1",
                "--gpus", "2"], {"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_arm_fails_loudly_without_cuda():
    r = _bench(["--config", "c1", "--steps", "1", "--warmup", "1"])
    assert r.returncode != 0
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]


def test_gpus_mismatch_with_world_size_fails():
    r = _bench(["--impl", "reference", "--config", "c1", "--steps", "1", "--gpus", "4"],
               {"RANK": "0", "LOCAL_RANK": "0", "WORLD_SIZE": "2"})
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


def test_gpus_n_spawns_n_rendezvousing_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-executes itself
    under torch.distributed.run: 2 ranks rendezvous (gloo dry run on CPU), the
    max over ranks reaches rank 0, and only rank 0 prints (n_gpus = 2)."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dry-run"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["dry_run"] and d["n_gpus"] == 2 and d["world_size"] == 2
    assert d["max_over_ranks"] == 2.0
