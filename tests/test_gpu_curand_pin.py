"""Pins the GPU draw (reading Q4: Philox4x32-10, counter (j, 0, 0, 0), key =
seed; u = floor(r * T / 2^64)) to a library routine: curand's Philox4_32_10
(SURVEY.md §8 c.3).  On a full table under UNIFORM every bin has width 1, so
the sampled global id of draw j is exactly u_j = floor(r_j * N / 2^64)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def curand_lib(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    out = str(tmp_path_factory.mktemp("curand") / "libcurand_philox.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O2", "-shared", "-Xcompiler", "-fPIC",
                           "-gencode", "arch=compute_100a,code=sm_100a",
                           os.path.join(HERE, "helpers", "curand_philox.cu"), "-o", out])
    lib = ctypes.CDLL(out)
    lib.curand_philox_draws.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32,
                                        ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("N,seed", [(1 << 16, 0x5EED0000), (100_003, 0x0123456789ABCDEF),
                                    (3 * 4096 + 7, 1)])
def test_gpu_draws_match_curand(curand_lib, N, seed):
    import torch
    from gpu_harness import Pair
    G = __import__("paper_2310_05205_b200")
    P = Pair(capacity=N, seq_len=1, colspecs=[synth.ColSpec("x", "u8", ())], R=1, mirror=False)
    P.fill(np.ones(N))
    B = 4096
    idx = torch.empty(B, dtype=torch.int64, device="cuda")
    G.gear_sample(P.t.handle, G.GEAR_UNIFORM, B, seed, 0.0, idx)
    torch.cuda.synchronize()
    got = idx.cpu().numpy().view(np.uint64)
    j = np.arange(B, dtype=np.uint64)
    r = np.zeros(B, dtype=np.uint64)
    assert curand_lib.curand_philox_draws(seed, j.ctypes.data, B, r.ctypes.data) == 0
    want = np.array([(int(x) * N) >> 64 for x in r], dtype=np.uint64)
    assert np.array_equal(got, want)
    P.close()
