"""GPU: the hand-written GEMMs (tcgen05 bf16 and SIMT fp32) against a plain torch fp32
reference of the same contraction, through the C ABI (adpsgd_gemm)."""
import itertools

import pytest

torch = pytest.importorskip("torch")

from paper_2110_11199_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


def _operand(rows_mn, K, mn, dtype, gen):
    # logical (rows_mn x K); stored K-major [rows_mn x K] or MN-major [K x rows_mn]
    x = torch.randn(rows_mn, K, generator=gen, device="cuda", dtype=torch.float32)
    if dtype == torch.bfloat16:
        x = x.to(torch.bfloat16).float()
    store = (x.t().contiguous() if mn else x.contiguous()).to(dtype)
    return x, store


def _run(bf16, M, N, K, amn, bmn, c_bf16=False, accumulate=False, bias=False, alpha=1.0, seed=0):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    dt = torch.bfloat16 if bf16 else torch.float32
    a, A = _operand(M, K, amn, dt, gen)
    b, Bm = _operand(N, K, bmn, dt, gen)
    cdt = torch.bfloat16 if c_bf16 else torch.float32
    C0 = torch.randn(M, N, generator=gen, device="cuda").to(cdt)
    Cout = C0.clone()
    bvec = torch.randn(N, generator=gen, device="cuda") if bias else None
    rc = _lib.lib().adpsgd_gemm(int(bf16), M, N, K, A.data_ptr(), A.stride(0), int(amn), Bm.data_ptr(), Bm.stride(0),
                                int(bmn), Cout.data_ptr(), Cout.stride(0), int(c_bf16), alpha, int(accumulate),
                                bvec.data_ptr() if bias else None, torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    torch.cuda.synchronize()
    ref = alpha * (a.double() @ b.double().t())
    if accumulate:
        ref = ref + C0.double()
    if bias:
        ref = ref + bvec.double()
    return Cout.double(), ref


@pytest.mark.parametrize("amn,bmn", list(itertools.product([0, 1], [0, 1])))
@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 320), (300, 200, 136), (1024, 4096, 1024),
                                   (64, 1000, 264), (4096, 264, 2048),
                                   # MN-major operands through the 3-D tensor-map views (extent % 64 == 0) with a
                                   # partial last n-tile and a ragged K (zero-filled blocks / rows)
                                   (512, 320, 1000), (768, 576, 4160)])
def test_tc_gemm_majorness_and_shapes(amn, bmn, shape):
    M, N, K = shape
    if (amn and M % 8) or (bmn and N % 8):
        pytest.skip("MN-major TMA pitch needs a multiple of 8 elements")
    got, ref = _run(True, M, N, K, amn, bmn)
    err = (got - ref).abs().max().item()
    # bf16 operands are exact in fp32; accumulation order differs only
    assert err <= 1e-3 * (K ** 0.5), (shape, amn, bmn, err)


@pytest.mark.parametrize("c_bf16", [0, 1])
def test_tc_gemm_epilogue_options(c_bf16):
    got, ref = _run(True, 384, 768, 192, 0, 1, c_bf16=c_bf16, accumulate=True, bias=True, alpha=0.5)
    tol = 2e-2 * ref.abs().max().item() if c_bf16 else 1e-3
    assert (got - ref).abs().max().item() <= tol


def test_tc_gemm_large_k_wgrad_shape():
    # dW = dZ^T X shape of the LSTM weight gradients: both operands MN-major, K = T*B
    got, ref = _run(True, 512, 640, 21 * 128, 1, 1)
    assert (got - ref).abs().max().item() <= 1e-3 * (21 * 128) ** 0.5


@pytest.mark.parametrize("amn,bmn", list(itertools.product([0, 1], [0, 1])))
def test_simt_gemm(amn, bmn):
    got, ref = _run(False, 150, 77, 45, amn, bmn, accumulate=True, bias=True, alpha=0.7)
    assert (got - ref).abs().max().item() <= 1e-4


def test_mix_update_kernel():
    n = 1000003
    g = torch.Generator(device="cuda").manual_seed(3)
    w, wl, wr, gr = (torch.randn(n, generator=g, device="cuda") for _ in range(4))
    out = torch.empty_like(w)
    sh = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.lib().adpsgd_mix_update(n, w.data_ptr(), wl.data_ptr(), wr.data_ptr(), gr.data_ptr(), 0.25,
                                            out.data_ptr(), sh.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ref = (w.double() + wl.double() + wr.double()) / 3.0 - 0.25 * gr.double()
    assert (out.double() - ref).abs().max().item() <= 2e-6
    assert (sh.float() - out).abs().max().item() <= 2e-2
