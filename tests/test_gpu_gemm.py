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
    """Gate/up rows interleaved in 16-row groups (GU_GROUP); h = silu(gate) * up in bf16."""
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(M + f)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    Wg = (torch.randn(f, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    Wu = (torch.randn(f, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    W = torch.stack([Wg.view(f // 16, 16, K), Wu.view(f // 16, 16, K)], dim=1).reshape(2 * f, K).contiguous()
    H = torch.zeros(M, f, device="cuda", dtype=torch.bfloat16)
    hsd.debug_gemm(A, W, H, use_tc="swiglu")
    torch.cuda.synchronize()
    gt, ut = A.float() @ Wg.float().T, A.float() @ Wu.float().T
    ref = torch.nn.functional.silu(gt) * ut
    assert ((H.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2


@pytest.mark.parametrize("M,N,K,accumulate", [
    (2080, 6144, 4096, False),     # c3 QKV (GQA 32/8, hd 128): CTA-pair, plain store
    (2080, 4096, 4096, True),      # c3 O projection: CTA-pair, residual add
    (2080, 4096, 14336, True),     # c3 down projection, K = 14336
    (8512, 5120, 13824, True),     # c4 down projection
    (4160, 4096, 11008, True),     # Llama-2-7B down at K = 11008
])
def test_tcgen05_pair_gemm_production_k(M, N, K, accumulate):
    """The CTA-pair (cta_group::2) data-parallel kernel at the verify shapes of
    c3 / c4 with their real reduction depths (K = 4096 .. 14336): many k-blocks
    through the TMA ring, both SMs of the pair staging half the operands."""
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    C0 = torch.randn(M, N, device="cuda", generator=g)
    C = C0.clone()
    hsd.debug_gemm(A, W, C, accumulate=accumulate, use_tc=True)
    torch.cuda.synchronize()
    ref = (A.double() @ W.double().T + (C0.double() if accumulate else 0))
    err = ((C.double() - ref).abs().max() / ref.abs().max()).item()
    # fp32 accumulation: rounding error grows like sqrt(K) (random-sign partial
    # sums); the 1e-5 bar of the K <= 4096 tests, scaled by sqrt(K / 4096)
    assert err < 1e-5 * max(1.0, (K / 4096) ** 0.5), err


@pytest.mark.parametrize("M,f,K", [(2080, 14336, 4096), (8512, 13824, 5120)])
def test_tcgen05_fused_swiglu_production_k(M, f, K):
    """c3 / c4 gate/up with the SwiGLU epilogue at the real K."""
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(M + f + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    Wg = (torch.randn(f, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    Wu = (torch.randn(f, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    W = torch.stack([Wg.view(f // 16, 16, K), Wu.view(f // 16, 16, K)], dim=1).reshape(2 * f, K).contiguous()
    H = torch.zeros(M, f, device="cuda", dtype=torch.bfloat16)
    hsd.debug_gemm(A, W, H, use_tc="swiglu")
    torch.cuda.synchronize()
    gt, ut = A.float() @ Wg.float().T, A.float() @ Wu.float().T
    ref = torch.nn.functional.silu(gt) * ut
    assert ((H.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2
