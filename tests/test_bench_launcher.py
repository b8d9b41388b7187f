"""bench.py's own multi-rank launch path on CPU (gloo; no GPU): `python bench.py --gpus 2` re-execs itself
under torch.distributed.run with two ranks, and the JSON line reports both ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=e, capture_output=True,
                          text=True, timeout=300)


def test_self_launch_two_ranks_reports_n_gpus_2():
    r = _run(["--plumbing", "--gpus", "2", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["comm"]["world_size"] == 2
    assert line["config"]["per_gpu_batch"] == 128 and line["config"]["parallelism"] == "batch-shard x2"
    assert line["choices_from_rank0"] is True


def test_single_rank_plumbing_unchanged():
    r = _run(["--plumbing", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["config"]["per_gpu_batch"] == 256


def test_world_size_mismatch_is_an_error():
    r = _run(["--plumbing", "--gpus", "4"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
