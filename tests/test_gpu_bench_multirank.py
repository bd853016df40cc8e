"""bench.py's N > 1 path (torchrun, sharded fit with all_reduce, winner gather, the pipelined e2e)
run end to end with two ranks sharing one GPU over gloo (RP_BENCH_SHARED_GPU=1): guards the
multi-rank control flow (a collective reached by one rank only deadlocks the driver's scaling run),
not the numbers."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc", [2, 3])
def test_bench_multirank_shared_gpu(nproc):
    env = dict(os.environ, RP_BENCH_SHARED_GPU="1", RP_BENCH_HANG_S="150")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29540 + nproc), "bench.py", "--gpus", str(nproc),
           "--steps", "2", "--warmup", "3", "--nD", "20011", "--K", "20003", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == nproc and d["value"] > 0
    assert d["selfcheck"]["device_step_equals_host_api_step"]
    assert d["e2e"]["winners_match_device_step"]
