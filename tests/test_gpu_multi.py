"""Multi-rank parity of the W > 1 device path through torchrun.

* test_multi_gpu_parity: one GPU per rank, NCCL bootstrap (gear_comm_create);
  runs where at least n GPUs are visible (gpurun --gpus 2|4).
* test_shared_device_parity: n rank processes on the ONE visible GPU,
  bootstrapped through a gloo group (gear_comm_create_host).  CUDA-IPC
  mappings and POSIX shared memory work between processes on one device, so
  the per-step mailbox exchanges (shard totals, update records, FIFO / TopK
  candidates), the search of the owner's CDF through its IPC mapping, the
  peer-HBM collect rows and the shared host shards all run the same code as
  on n GPUs (kernels of different processes are time-sliced, so this is a
  correctness run, not a performance one).  Both compare every rank's slice
  with the unsharded CPU oracle.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _run(n, port, env_extra, script="dist_gpu_parity.py", done="all multi-GPU parity cases ok"):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", script)]
    env = dict(os.environ, **env_extra)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert r.stdout.count(done) == n


@pytest.mark.parametrize("n", [2, 4])
def test_multi_gpu_parity(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    _run(n, 29533 + n, {"GEAR_SHARED_DEVICE": "0"})


@pytest.mark.parametrize("n", [2, 4, 8])
def test_shared_device_parity(n):
    if _ngpus() < 1:
        pytest.skip("needs a GPU")
    _run(n, 29543 + n, {"GEAR_SHARED_DEVICE": "1", "CUDA_VISIBLE_DEVICES": os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]})


@pytest.mark.parametrize("n", [2, 4])
def test_shared_device_fullsize_c2(n):
    """c2 at full size (84.7 GB) sharded over W=2 / 4 rank processes on the
    one visible GPU: every id, weight and collected row vs the oracle, both
    assignments, collective updates (tests/dist_gpu_fullsize.py)."""
    if _ngpus() < 1:
        pytest.skip("needs a GPU")
    _run(n, 29561 + n, {"GEAR_SHARED_DEVICE": "1",
                    "CUDA_VISIBLE_DEVICES": os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]},
         script="dist_gpu_fullsize.py", done="full-size multi-rank parity ok")


@pytest.mark.parametrize("n", [2, 4])
def test_multi_gpu_fullsize_c2(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    _run(n, 29571 + n, {"GEAR_SHARED_DEVICE": "0"}, script="dist_gpu_fullsize.py",
         done="full-size multi-rank parity ok")
