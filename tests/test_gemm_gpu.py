"""tcgen05 GEMM vs a plain PyTorch fp32 reference of the same contraction."""
import pytest
import torch

from paper_2102_03161_b200 import ops

pytestmark = pytest.mark.gpu

RTOL = 1e-2  # bf16 operands, fp32 accumulation (BASELINE.json north_star)


def _ref(a, b, a_mn, b_mn):
    A = (a.t() if a_mn else a).float()
    B = (b.t() if b_mn else b).float()
    return A @ B.t()


def _close(out, ref, rtol=RTOL):
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= rtol * scale + 1e-3, f"max err {err} vs scale {scale}"


# (4100, 512), (4500, 2304), (5000, 768): CTA-pair (256-row, cta_group::2)
# tiles, including pairs whose second CTA is partly / wholly past M.
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (3546, 2304, 768), (300, 768, 3072),
                                   (1000, 1000, 768), (77, 768, 768), (400, 1000, 777),
                                   (4100, 512, 192), (4500, 2304, 768), (5000, 768, 3072)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False),
                                       (True, True)])
def test_gemm_store(cuda, M, N, K, a_mn, b_mn):
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N + K)
    pad = lambda n: (n + 7) // 8 * 8  # noqa: E731  (TMA needs 16B row pitch)
    a = torch.randn((K, pad(M)) if a_mn else (M, pad(K)), device=cuda, generator=g).bfloat16()
    a = a[:, :M] if a_mn else a[:, :K]
    b = torch.randn((K, N) if b_mn else (N, pad(K)), device=cuda, generator=g).bfloat16()
    b = b if b_mn else b[:, :K]
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    ops.gemm(a, b, out, a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    _close(out, _ref(a, b, a_mn, b_mn))


def test_gemm_epilogues(cuda):
    M, N, K = 1000, 3072, 768
    g = torch.Generator(device=cuda).manual_seed(3)
    a = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    b = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g)
    ref = _ref(a, b, False, False) + bias
    pre = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    out = torch.empty_like(pre)
    ops.gemm(a, b, out, epilogue=ops.EPI_BIAS_GELU_BF16, bias=bias, aux=pre)
    torch.cuda.synchronize()
    _close(pre, ref)
    _close(out, torch.nn.functional.gelu(ref))
    res = torch.randn(M, N, device=cuda, generator=g).bfloat16()
    out2 = res.clone()
    ops.gemm(a, b, out2, epilogue=ops.EPI_BIAS_RESID_BF16, bias=bias, aux=out2)
    torch.cuda.synchronize()
    _close(out2, ref + res.float())
    # dgelu + column sum (bias grad)
    u = torch.randn(M, N, device=cuda, generator=g).bfloat16()
    colsum = torch.zeros(N, device=cuda)
    d = torch.empty_like(pre)
    ops.gemm(a, b, d, epilogue=ops.EPI_DGELU_BF16, aux=u, colsum=colsum)
    torch.cuda.synchronize()
    uf = u.float()
    gprime = 0.5 * (1 + torch.erf(uf / 2 ** 0.5)) + uf * torch.exp(-0.5 * uf * uf) / (2 * torch.pi) ** 0.5
    refd = _ref(a, b, False, False) * gprime
    _close(d, refd)
    _close(colsum, refd.sum(0), rtol=2e-2)


@pytest.mark.parametrize("M,N", [(1000, 3072), (77, 200), (4096, 1000)])
def test_gemm_gelu2_mul(cuda, M, N):
    """FC1 forward stores gelu(u) and gelu'(u); the FC2 dgrad multiplies by gelu'
    and sums columns (bias gradient; N = 200 / 1000 end in partial 32-column
    chunks of the vector reduction)."""
    K = 768
    g = torch.Generator(device=cuda).manual_seed(9)
    a = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    b = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g)
    u = _ref(a, b, False, False) + bias
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    gp = torch.empty_like(out)
    ops.gemm(a, b, out, epilogue=ops.EPI_BIAS_GELU2_BF16, bias=bias, aux=gp)
    torch.cuda.synchronize()
    _close(out, torch.nn.functional.gelu(u))
    want_gp = 0.5 * (1 + torch.erf(u / 2 ** 0.5)) + u * torch.exp(-0.5 * u * u) / (2 * torch.pi) ** 0.5
    _close(gp, want_gp)
    colsum = torch.zeros(N, device=cuda)
    d = torch.empty_like(out)
    ops.gemm(a, b, d, epilogue=ops.EPI_MUL_BF16, aux=gp, colsum=colsum)
    torch.cuda.synchronize()
    refd = _ref(a, b, False, False) * gp.float()
    _close(d, refd)
    _close(colsum, refd.sum(0), rtol=2e-2)


@pytest.mark.parametrize("M,N", [(1000, 768), (77, 128), (4000, 1024)])
def test_gemm_rowdot(cuda, M, N):
    """C = acc; D[m, g] = sum over 64-column group g of bf16(acc) * aux (attention D)."""
    K = 768
    g = torch.Generator(device=cuda).manual_seed(M + N)
    a = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    b = (torch.randn(N, K, device=cuda, generator=g) * 0.05).bfloat16()
    aux = torch.randn(M, N, device=cuda, generator=g).bfloat16()
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    drow = torch.zeros(M, N // 64, device=cuda)
    ops.gemm(a, b, out, epilogue=ops.EPI_ROWDOT_BF16, aux=aux, colsum=drow)
    torch.cuda.synchronize()
    ref = _ref(a, b, False, False)
    _close(out, ref)
    want = (out.float() * aux.float()).reshape(M, N // 64, 64).sum(-1)
    assert (drow - want).abs().max().item() <= 1e-3 * want.abs().max().item() + 1e-3


@pytest.mark.parametrize("split", [1, 4, 9])
def test_gemm_wgrad_f32(cuda, split):
    R, out_f, in_f = 7880, 768, 2304  # dW[out,in] = dY^T X over R token rows
    g = torch.Generator(device=cuda).manual_seed(split)
    dy = torch.randn(R, out_f, device=cuda, generator=g).bfloat16()
    x = torch.randn(R, in_f, device=cuda, generator=g).bfloat16()
    dw = torch.full((out_f, in_f), 0.5, device=cuda)
    ops.gemm(dy, x, dw, a_mn=True, b_mn=True, epilogue=ops.EPI_ACCUM_F32, split_k=split)
    torch.cuda.synchronize()
    ref = dy.float().t() @ x.float() + 0.5
    _close(dw, ref, rtol=1e-3)
