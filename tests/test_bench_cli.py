"""bench.py's launcher contract on CPU: `--gpus N` without a launcher re-runs itself under
torch.distributed.run with N ranks (127.0.0.1 rendezvous, gloo control plane), and exactly
one JSON line comes out (rank 0) with n_gpus = N and the shared workload config. The
reference arm runs on the host, so this needs no GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libfdref.so")),
                    reason="oracle/_ref not built")
def test_bench_spawns_ranks_and_prints_one_line():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "products", "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                       timeout=900, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["unit"] == "batches/s" and d["value"] > 0
    assert d["config"]["global_batch"] == 2000 and d["config"]["parallelism"].startswith("dp2")
    assert d["cpu_baseline"]["cores"] == os.cpu_count() and d["execution"]["batches_timed"] % os.cpu_count() == 0
