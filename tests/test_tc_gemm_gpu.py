"""The batched solvers' fp32 product on the tensor pipe (csrc/tc_gemm.cu, 3xTF32
tcgen05 kernel) through the C ABI `ell1_gemm_f32`, against an fp64 product.

The bar is fp32-level accuracy (the batched DALM certificate needs it): the
error relative to sum_k |a_ik b_kj| is at most 1.5x that of cuBLAS's fp32
SIMT SGEMM on the same operands (floor 4e-7), including nonnegative
operands, where every rounding has the same sign and the tensor core's
truncating accumulation is biased (only the per-k-block fp32 sums keep it in
check: a single TMEM accumulation over K = 1216 is ~10x worse).  Shapes cover every tile / K-split variant the launcher
picks at the BASELINE config-3/5 sizes plus ragged edges."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gemm(torch, A, B, trans):
    from paper_1007_3753_b200 import _lib
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    # column-major device copies with 4-aligned leading dimensions
    def colmajor(X):
        r, c = X.shape
        ld = (r + 3) // 4 * 4
        t = torch.zeros((c, ld), dtype=torch.float32, device=dev)
        t[:, :r] = torch.from_numpy(np.ascontiguousarray(X.T, dtype=np.float32)).to(dev)
        return t, ld
    Ad, lda = colmajor(A)
    Bd, ldb = colmajor(B)
    M = A.shape[1] if trans else A.shape[0]
    K = A.shape[0] if trans else A.shape[1]
    N = B.shape[1]
    ldc = M + 3
    Cd = torch.full((N, ldc), float("nan"), dtype=torch.float32, device=dev)
    wsb = L.ell1_gemm_f32_workspace(int(trans), M, K)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    rc = L.ell1_gemm_f32(int(trans), M, N, K, ctypes.c_void_p(Ad.data_ptr()), lda,
                         ctypes.c_void_p(Bd.data_ptr()), ldb, ctypes.c_void_p(Cd.data_ptr()), ldc,
                         ctypes.c_void_p(ws.data_ptr()), wsb, stream)
    assert rc == 0, rc
    torch.cuda.synchronize()
    return Cd[:, :M].cpu().numpy().T.astype(np.float64)


@pytest.mark.parametrize("trans", [0, 1])
@pytest.mark.parametrize("M,N,K,nonneg", [
    (100, 37, 50, False),          # ragged, one k-block
    (128, 64, 32, False),
    (1024, 1024, 1216, False),     # config 3: A X
    (1024, 1024, 1216, True),      # config 3 CAB dictionary is nonnegative
    (1216, 1024, 1024, True),      # config 3: A^T Y
    (1024, 2048, 1216, True),      # config 3: A [U | x]
    (1024, 700, 2240, True),       # config 3: [M | Ginv] V after compaction
    (512, 1024, 2048, False),      # config 5
    (2048, 300, 512, False),
    (300, 1, 1001, False),         # single instance left after compaction, odd K
    (517, 5, 1001, True),          # ragged M, tiny N, odd K
])
def test_tc_gemm_matches_fp64(trans, M, N, K, nonneg):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    rng = np.random.default_rng(M * 31 + N * 7 + K + trans)
    lo = 0.0 if nonneg else -0.5
    A = rng.uniform(lo, 1.0, size=(K, M) if trans else (M, K)).astype(np.float32)
    B = rng.uniform(lo, 1.0, size=(K, N)).astype(np.float32)
    C = _gemm(torch, A, B, trans)
    A64 = A.astype(np.float64).T if trans else A.astype(np.float64)
    ref = A64 @ B.astype(np.float64)
    scale = np.abs(A64) @ np.abs(B.astype(np.float64))
    err = float(np.max(np.abs(C - ref) / scale))
    # fp32 SIMT SGEMM on the same operands (TF32 off) as the accuracy yardstick
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        dev = torch.device("cuda", 0)
        At = torch.from_numpy(np.ascontiguousarray(A.T if trans else A)).to(dev)
        S = (At @ torch.from_numpy(B).to(dev)).cpu().numpy().astype(np.float64)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    err_sgemm = float(np.max(np.abs(S - ref) / scale))
    assert np.all(np.isfinite(C))
    assert err <= max(4e-7, 1.5 * err_sgemm), (err, err_sgemm)


def test_tc_gemm_is_the_active_fp32_path():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1007_3753_b200 import _lib
    A = np.ones((64, 32), np.float32)
    B = np.ones((32, 8), np.float32)
    C = _gemm(torch, A, B, 0)
    assert np.all(C == 32.0)
    assert not hasattr(_lib.lib(), "ell1_blas_fp32_mode")      # no alternative fp32 backend
