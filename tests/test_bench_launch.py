"""CPU: `bench.py --gpus N` without a launcher re-runs itself as N ranks under
torch.distributed.run (the driver may call it that way); checked with a gloo
rendezvous instead of GPU work."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_bench_self_launch_two_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert lines == [{"launch_check": True, "world": 2, "rank_sum": 3}], res.stdout
