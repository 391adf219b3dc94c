"""GPU numerics of the library's GEMM kernels (tcgen05 and SIMT) against a
plain PyTorch fp32 reference of the same op, through the C ABI test hook."""
import pytest
import torch

pytestmark = pytest.mark.gpu
hsd = pytest.importorskip("paper_2602_21224_b200.hsd")

SHAPES = [(1, 64, 64), (16, 128, 64), (7, 4096, 8192), (65, 12288, 4096), (65, 4096, 11008),
          (300, 200, 136), (257, 384, 192), (1, 32000, 4096), (24, 22016, 4096), (61, 130, 4104)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("accumulate", [False, True])
def test_tcgen05_gemm_matches_fp32_reference(M, N, K, accumulate):
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    C0 = torch.randn(M, N, device="cuda", generator=g)
    C = C0.clone()
    hsd.debug_gemm(A, W, C, accumulate=accumulate, use_tc=True)
    torch.cuda.synchronize()
    ref = A.float() @ W.float().T + (C0 if accumulate else 0)
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-5, err


@pytest.mark.parametrize("M,N,K", [(5, 70, 33), (65, 300, 256)])
def test_simt_gemm_matches_fp32_reference(M, N, K):
    torch.backends.cuda.matmul.allow_tf32 = False
    A = torch.randn(M, K, device="cuda")
    W = torch.randn(N, K, device="cuda")
    C = torch.zeros(M, N, device="cuda")
    hsd.debug_gemm(A, W, C)
    torch.cuda.synchronize()
    ref = A @ W.T
    assert ((C - ref).abs().max() / ref.abs().max()).item() < 1e-5


@pytest.mark.parametrize("M,N,K", [(1024, 28672, 512), (2080, 36864, 256), (700, 128256, 128)])
@pytest.mark.parametrize("accumulate", [False, True])
def test_tcgen05_data_parallel_gemm(M, N, K, accumulate):
    """Shapes with >= 4 output tiles per SM run data-parallel (plain store /
    residual add epilogues instead of red.add partial sums)."""
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    C0 = torch.randn(M, N, device="cuda", generator=g)
    C = C0.clone()
    hsd.debug_gemm(A, W, C, accumulate=accumulate, use_tc=True)
    torch.cuda.synchronize()
    ref = A.float() @ W.float().T + (C0 if accumulate else 0)
    assert ((C - ref).abs().max() / ref.abs().max()).item() < 1e-5


@pytest.mark.parametrize("M,f,K", [(1024, 14336, 512), (2080, 11008, 256)])
def test_tcgen05_fused_swiglu(M, f, K):
    """Gate/up rows interleaved in 64-row groups; h = silu(gate) * up in bf16."""
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(M + f)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    Wg = (torch.randn(f, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    Wu = (torch.randn(f, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    W = torch.stack([Wg.view(f // 64, 64, K), Wu.view(f // 64, 64, K)], dim=1).reshape(2 * f, K).contiguous()
    H = torch.zeros(M, f, device="cuda", dtype=torch.bfloat16)
    hsd.debug_gemm(A, W, H, use_tc="swiglu")
    torch.cuda.synchronize()
    gt, ut = A.float() @ Wg.float().T, A.float() @ Wu.float().T
    ref = torch.nn.functional.silu(gt) * ut
    assert ((H.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2
