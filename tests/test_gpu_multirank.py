"""Multi-rank runs on one GPU (world > visible GPUs): bench.py under torchrun with 2, 3 and 4 ranks
sharing cuda:0 -- gloo for the host exchange, the fused ZeRO-1 kernel over CUDA IPC peer memory as
the data plane (SURVEY 8(e)/(f) row 1, P:110 block independence, reading Z1).  Each run prints the
N-rank JSON line, whose zero1.fused.check is the bit-exact comparison of the sharded result (every
rank's parameter replica, every rank's codes and absmax) with the unsharded single-GPU step on the
rank-order reduced gradient (bench.zero_fused_check)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,workload", [(2, "cfg1_1m"), (3, "cfg1_1m"), (4, "cfg1_1m"),
                                            (2, "cfg2_gpt2_medium")])
def test_bench_multirank_shared_gpu(world, workload):
    port = 29700 + (os.getpid() % 200) + 10 * world
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "4", "--warmup", "3", "--workload", workload, "--no-e2e",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == world and out["value"] > 0 and out["steps"] == 4
    assert out["zero1"]["fused"]["check"].startswith("bit-exact"), out["zero1"]
    assert out["gpu_launches"] == 4
