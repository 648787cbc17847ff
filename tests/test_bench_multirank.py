"""bench.py's multi-rank path end to end (the driver's N = 2, 4, 8 runs):
two torchrun ranks sharing the one test GPU through the
AIDW_BENCH_SHARED_DEVICE hook (gloo instead of NCCL, same code otherwise):
data broadcast, global-bbox all-reduce, per-rank shards, max-over-ranks
timing, one JSON line from rank 0 — and the reference arm run by rank 0 only."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def torchrun(port, *args):
    env = dict(os.environ, AIDW_BENCH_SHARED_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", *args]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_two_rank_bench_line():
    b = torchrun(29531, "--config", "100k", "--steps", "2", "--warmup", "3",
                 "--no-cpu-baseline", "--no-fp64", "--verify")
    # the two shards, gathered, are the one-device run of all 100K queries
    assert b["verify"] == {"shards_bit_identical": True, "n": 100_000}
    # configs as written: the 100K queries sharded over the 2 ranks (strong)
    assert b["n_gpus"] == 2 and b["scaling"] == "strong"
    assert b["config"]["n"] == 100_000 and b["hardware"]["per_rank_queries"] == 50_000
    assert b["value"] > 0 and b["e2e"]["value"] > 0
    assert abs(b["value"] - 100_000 / (b["ms_per_step"] / 1e3)) <= 1e-6 * b["value"]
    assert b["gpu_launches"] > 0
    # the weak-scaling figure beside it: 100K queries per rank
    w = b["weak_scaling"]
    assert w["n"] == 200_000 and w["per_rank"] == 100_000 and w["value"] > 0


@pytest.mark.gpu
def test_two_rank_reference_arm():
    b = torchrun(29532, "--impl", "reference", "--config", "100k", "--steps", "1",
                 "--warmup", "1")
    assert b["impl"] == "reference" and b["value"] > 0
    # the reference arm never maps the repo's library
    assert b["config"]["n"] == 100_000 and b["scaling"] == "strong"
    assert b["repo_library_mapped"] is False
