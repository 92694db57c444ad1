"""tcgen05 / SIMT GEMM primitive vs a float64 CPU matmul of the same inputs."""
import pytest
import torch

from paper_2504_19232_b200 import _lib as L
from paper_2504_19232_b200 import ops

pytestmark = pytest.mark.gpu


def _ref(A, B, a_mn, b_mn):
    A64 = A.double().cpu()
    B64 = B.double().cpu()
    Am = A64.t() if a_mn else A64
    Bm = B64.t() if b_mn else B64
    return Am @ Bm.t()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(256, 384, 192), (200, 2304, 320), (128, 128, 64), (384, 4096, 1024)])
def test_gemm_layouts(dtype, a_mn, b_mn, M, N, K):
    torch.manual_seed(0)
    dev = "cuda"
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(dev, dtype)
    B = (torch.randn(K, N) if b_mn else torch.randn(N, K)).to(dev, dtype)
    Cm = torch.zeros(M, N, device=dev, dtype=dtype)
    ops.gemm(A, B, Cm, M=M, N=N, K=K, a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    ref = _ref(A, B, a_mn, b_mn)
    err = (Cm.double().cpu() - ref).abs().max() / ref.abs().max()
    assert err < (1e-2 if dtype == torch.bfloat16 else 1e-5), float(err)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_gemm_epilogues(dtype):
    torch.manual_seed(1)
    dev = "cuda"
    M, N, K = 256, 512, 256
    A = torch.randn(M, K, device=dev).to(dtype)
    B = (torch.randn(N, K, device=dev) / 16).to(dtype)
    bias = torch.randn(N, device=dev)
    ref = _ref(A, B, 0, 0)
    # GELU: aux = acc + bias; C = gelu(aux)
    Cm = torch.zeros(M, N, device=dev, dtype=dtype)
    aux = torch.zeros(M, N, device=dev, dtype=dtype)
    ops.gemm(A, B, Cm, M=M, N=N, K=K, epi=L.EPI_GELU, bias=bias, aux=aux)
    a_ref = ref + bias.double().cpu()
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    assert ((aux.double().cpu() - a_ref).abs().max() / a_ref.abs().max()) < tol
    g_ref = torch.nn.functional.gelu(aux.double().cpu(), approximate="tanh")
    assert ((Cm.double().cpu() - g_ref).abs().max() / g_ref.abs().max()) < tol
    # RESID
    R = torch.randn(M, N, device=dev).to(dtype)
    ops.gemm(A, B, Cm, M=M, N=N, K=K, epi=L.EPI_RESID, bias=bias, R=R)
    r_ref = a_ref + R.double().cpu()
    assert ((Cm.double().cpu() - r_ref).abs().max() / r_ref.abs().max()) < tol
    # ACC_F32 twice
    Cf = torch.zeros(M, N, device=dev)
    ops.gemm(A, B, Cf, M=M, N=N, K=K, epi=L.EPI_ACC_F32)
    ops.gemm(A, B, Cf, M=M, N=N, K=K, epi=L.EPI_ACC_F32)
    assert ((Cf.double().cpu() - 2 * ref).abs().max() / (2 * ref).abs().max()) < (1e-3 if dtype == torch.bfloat16 else 1e-5)
    # DGELU
    ops.gemm(A, B, Cm, M=M, N=N, K=K, epi=L.EPI_DGELU, aux=aux)
    x = aux.double().cpu().requires_grad_(True)
    gg = torch.autograd.grad(torch.nn.functional.gelu(x, approximate="tanh").sum(), x)[0]
    d_ref = ref * gg
    assert ((Cm.double().cpu() - d_ref).abs().max() / d_ref.abs().max()) < tol


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_gemm_batched_causal_heads(dtype):
    """QK^T per (sequence, head) from a packed qkv [b*T, 3d] with causal tile skip,
    and P V with the K-range limit, as the attention path uses them."""
    torch.manual_seed(2)
    dev = "cuda"
    b, T, H, dh = 2, 256, 2, 128
    d = H * dh
    qkv = torch.randn(b * T, 3 * d, device=dev).to(dtype)
    S = torch.full((b * H, T, T), float("nan"), device=dev)
    ops.gemm(qkv[:, :d], qkv[:, d:2 * d], S, M=T, N=T, K=dh, Z=b * H, zdiv=H,
             a_off=(T, 0, 0, dh), b_off=(T, 0, 0, dh), c_off=(H * T * T, T * T),
             epi=L.EPI_STORE_F32, alpha=0.5, causal=L.CAUSAL_TILE, ldc=T)
    torch.cuda.synchronize()
    q = qkv[:, :d].double().cpu().reshape(b, T, H, dh).transpose(1, 2)
    k = qkv[:, d:2 * d].double().cpu().reshape(b, T, H, dh).transpose(1, 2)
    ref = 0.5 * q @ k.transpose(-1, -2)
    got = S.double().cpu().reshape(b, H, T, T)
    tri = torch.tril(torch.ones(T, T, dtype=torch.bool))
    err = (got - ref).abs()[..., tri].max() / ref.abs().max()
    assert err < (1e-2 if dtype == torch.bfloat16 else 1e-5)
    # P V with KEND, P lower triangular
    P = torch.tril(torch.rand(b * H, T, T, device=dev)).to(dtype)
    O = torch.zeros(b * T, d, device=dev, dtype=dtype)
    P2 = P.reshape(b * H * T, T)
    ops.gemm(P2, qkv[:, 2 * d:], O, M=T, N=dh, K=T, Z=b * H, zdiv=H, b_mn=1,
             a_off=(H * T, T, 0, 0), b_off=(T, 0, 0, dh), c_off=(T * d, dh),
             causal=L.CAUSAL_KEND, ldc=d)
    torch.cuda.synchronize()
    v = qkv[:, 2 * d:].double().cpu().reshape(b, T, H, dh).transpose(1, 2)
    oref = (P.double().cpu().reshape(b, H, T, T) @ v).transpose(1, 2).reshape(b * T, d)
    err = (O.double().cpu() - oref).abs().max() / oref.abs().max()
    assert err < (1e-2 if dtype == torch.bfloat16 else 1e-5)
