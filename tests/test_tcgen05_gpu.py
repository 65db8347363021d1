"""GPU unit tests of the sm_100a building blocks under the tensor path:
TMA (SWIZZLE_128B) -> smem descriptors -> tcgen05.mma kind::f16 -> TMEM ->
tcgen05.ld 32x32b, checked against a float64 matmul of the same fp16 data."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K", [16, 32, 64, 96, 112, 128, 144, 256])
def test_mma_probe_matches_fp64_matmul(knn, K):
    import torch
    lib = knn.library()
    fn = lib.knn_b200_debug_mma_probe
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
    g = torch.Generator().manual_seed(K)
    A = (torch.rand((128, K), generator=g) * 4 - 2).half()
    B = (torch.rand((128, K), generator=g) * 4 - 2).half()
    dA, dB = A.cuda(), B.cuda()
    dD = torch.empty((128, 128), dtype=torch.float32, device="cuda")
    assert fn(dA.data_ptr(), dB.data_ptr(), K, dD.data_ptr()) == 0
    ref = A.double() @ B.double().T
    got = dD.cpu().double()
    # fp16 products are exact in fp32; only the fp32 accumulation rounds
    bound = (K + 4) * 2.0 ** -23 * (A.double().abs() @ B.double().abs().T)
    assert ((got - ref).abs() <= bound + 1e-30).all(), float((got - ref).abs().max())
