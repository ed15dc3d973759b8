"""The tcgen05 (kind::i8) tile used for exact u8 verification: u8 x u8 -> s32
is exact, so the tile must equal the integer matrix product bit for bit."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,K", [(256, 128), (32, 32), (128, 256), (64, 96)])
def test_tc_gemm_u8_exact(gpu, N, K):
    g = np.random.Generator(np.random.PCG64(N * 1000 + K))
    A = g.integers(0, 256, (128, K), dtype=np.uint8)
    B = g.integers(0, 256, (N, K), dtype=np.uint8)
    Cm = np.zeros((128, N), np.int32)
    rc = gpu.load().detlsh_test_tc_gemm_u8(C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data), N, K,
                                           C.c_void_p(Cm.ctypes.data))
    assert rc == 0, gpu.load().detlsh_gpu_last_error()
    want = A.astype(np.int64) @ B.astype(np.int64).T
    assert np.array_equal(Cm.astype(np.int64), want)
