"""bench.py's multi-GPU plumbing on CPU: --gpus N re-launches itself as N torchrun ranks,
refuses a box with fewer GPUs, and refuses a WORLD_SIZE that disagrees with --gpus."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

STUB = '''
import json, os, sys
out = sys.argv[sys.argv.index("--out") + 1]
with open(os.path.join(out, "rank%s.json" % os.environ["RANK"]), "w") as f:
    json.dump({k: os.environ.get(k) for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "NCCL_DEBUG")} |
              {"argv": sys.argv[1:]}, f)
'''


def test_launcher_starts_one_rank_per_gpu(tmp_path, monkeypatch):
    stub = tmp_path / "stub.py"
    stub.write_text(STUB)
    monkeypatch.setattr(bench, "gpu_count", lambda: 2)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    argv = ["--gpus", "2", "--steps", "3", "--out", str(tmp_path)]
    args = bench.parse(["--gpus", "2", "--steps", "3"])
    args.master_port = 29000 + os.getpid() % 1000
    assert bench.launch_ranks(args, argv, script=str(stub)) == 0
    seen = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(2)]
    assert sorted(s["RANK"] for s in seen) == ["0", "1"]
    assert all(s["WORLD_SIZE"] == "2" and s["MASTER_ADDR"] == "127.0.0.1" for s in seen)
    assert all(s["NCCL_DEBUG"] == "INFO" for s in seen)
    assert all(s["argv"][:4] == ["--gpus", "2", "--steps", "3"] for s in seen)


def test_bench_refuses_more_gpus_than_the_box_has():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["PATH"] = "/nonexistent"  # no nvidia-smi: zero GPUs visible
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True,
                       text=True, env=env, timeout=120)
    assert r.returncode == 2
    assert "needs 2 GPUs" in r.stderr and "this box has 0" in r.stderr


@pytest.mark.parametrize("impl", ["ours", "reference"])
def test_bench_refuses_a_world_size_mismatch(impl):
    env = dict(os.environ, WORLD_SIZE="4", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", impl],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=4 but --gpus 2" in r.stderr
