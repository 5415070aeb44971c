"""Multi-process (replicas) harness on CPU with the gloo backend, world size 2:
the max-over-ranks timing and whole-job rate bench.py uses under torchrun,
and the reference arm's rank-0-only rule. The decomposition itself does not
shard, so this is the only N > 1 logic."""

import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import torch.distributed as dist
dist.init_process_group("gloo", init_method="env://")
import bench
rank = dist.get_rank()
world = dist.get_world_size()
ms = 100.0 + 50.0 * rank          # rank 1 is the slowest
mx = bench.max_over_ranks(ms)
rate = bench.whole_job_rate(world, 1000, 4, mx)
print(json.dumps({{"rank": rank, "max": mx, "rate": rate}}), flush=True)
dist.barrier()
dist.destroy_process_group()
"""


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_max_over_ranks_gloo_world2(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER.format(root=ROOT))
    port = free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                   WORLD_SIZE="2", LOCAL_RANK=str(rank))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        out, err = p.communicate(timeout=120)
        assert p.returncode == 0, err
        outs.append(out)
    import json

    recs = [json.loads(o.strip().splitlines()[-1]) for o in outs]
    assert all(r["max"] == 150.0 for r in recs)
    # 2 ranks x 1000 units x 4 steps over the slowest rank's 150 ms
    assert all(abs(r["rate"] - 2 * 1000 * 4 / 0.150) < 1e-6 for r in recs)


def test_reference_arm_nonzero_ranks_exit_clean():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0
    assert r.stdout.strip() == ""


@pytest.mark.slow
def test_reference_arm_json_line():
    """rank 0 prints one JSON line with the contract keys (oracle on host)."""
    import json

    env = dict(os.environ, RANK="0", WORLD_SIZE="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--config", "1"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "cpu_baseline", "e2e", "config"):
        assert key in line
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
