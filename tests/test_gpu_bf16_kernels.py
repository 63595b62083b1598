"""bf16 tier kernels on the B200 through the C ABI: tcgen05 GEMM (+ fused LoRA), attention, shrink.

Reference for every floating-point kernel: the same bf16 input values in fp64
(torch), tolerance written per test. Integer/selection properties (row select
of the LoRA delta, row independence) are bitwise.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_2512_17910_b200")
from paper_2512_17910_b200 import _native  # noqa: E402

lib = _native.lib


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _bf(shape, gen, scale=1.0):
    return (torch.randn(shape, generator=gen, device="cuda") * scale).to(torch.bfloat16)


_WS = {}


def gemm(epi, A, Bt, C, M, N, K, split=False):
    ws = None
    if split:
        if "ws" not in _WS:
            _WS["ws"] = torch.zeros(lib.alora_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
        ws = _WS["ws"]
    rc = lib.alora_gemm_bf16(epi, A.data_ptr(), A.shape[1], Bt.data_ptr(), Bt.shape[1], C.data_ptr(), C.shape[1],
                             M, N, K, None if ws is None else ws.data_ptr(), 0 if ws is None else ws.numel(),
                             _stream())
    _native.check(rc, "alora_gemm_bf16")
    torch.cuda.synchronize()


@pytest.mark.parametrize("M,N,K", [(1, 2048, 8192), (48, 3072, 2048), (240, 2048, 2048), (130, 1024, 4096)])
def test_gemm_split_k_deterministic_and_correct(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A, Bt = _bf((M, K), g), _bf((N, K), g, 0.05)
    ref = A.double() @ Bt.double().T
    mag = A.double().abs() @ Bt.double().abs().T
    outs = []
    for _ in range(2):
        C = torch.full((M, N), float("nan"), device="cuda")
        gemm(16, A, Bt, C, M, N, K, split=True)
        outs.append(C)
    assert torch.equal(outs[0], outs[1])  # fixed split order: bitwise repeatable
    assert ((outs[0].double() - ref).abs() / (mag + 1e-6)).max().item() < 1e-5
    X = torch.randn((M, N), generator=g, device="cuda")
    X0 = X.clone()
    gemm(1, A, Bt, X, M, N, K, split=True)  # residual add epilogue through the split reduction
    assert ((X.double() - X0.double() - ref).abs() / (mag + 1.0)).max().item() < 1e-5
    if N % 128 == 0:
        Sg = torch.empty((M, N // 2), device="cuda", dtype=torch.bfloat16)
        gemm(3, A, Bt, Sg, M, N, K, split=True)
        r = ref.view(M, N // 128, 2, 64)
        gate, up = r[:, :, 0, :].reshape(M, N // 2), r[:, :, 1, :].reshape(M, N // 2)
        np.testing.assert_allclose(Sg.float().cpu().numpy(), (gate * torch.sigmoid(gate) * up).float().cpu().numpy(),
                                   rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (5, 128, 256), (128, 256, 512), (200, 384, 1000), (1000, 512, 2048),
                                   (77, 3072, 2048),
                                   (2100, 2048, 1024), (4100, 640, 512)])  # > 148 tiles: persistent kernel
def test_gemm_store_and_fp32(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A, Bt = _bf((M, K), g), _bf((N, K), g)
    ref = A.double() @ Bt.double().T
    C32 = torch.full((M, N), float("nan"), device="cuda")
    gemm(16, A, Bt, C32, M, N, K)
    mag = A.double().abs() @ Bt.double().abs().T
    err = ((C32.double() - ref).abs() / (mag + 1e-6)).max().item()
    assert err < 1e-5, err  # fp32 accumulation of exact bf16 products: error relative to sum |a||b|
    C16 = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    gemm(0, A, Bt, C16, M, N, K)
    np.testing.assert_array_equal(C16.float().cpu().numpy(), C32.to(torch.bfloat16).float().cpu().numpy())


@pytest.mark.parametrize("M,N,K", [(300, 512, 640), (3000, 2048, 640)])  # the second: persistent, SwiGLU BN=256
def test_gemm_add_relu_swiglu(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(1)
    A, Bt = _bf((M, K), g), _bf((N, K), g, 0.05)
    ref = A.double() @ Bt.double().T
    X = torch.randn((M, N), generator=g, device="cuda")
    X0 = X.clone()
    gemm(1, A, Bt, X, M, N, K)
    assert ((X.double() - X0.double() - ref).abs().max().item()) < 1e-4
    R = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    gemm(2, A, Bt, R, M, N, K)
    np.testing.assert_allclose(R.float().cpu().numpy(), ref.clamp_min(0).to(torch.bfloat16).float().cpu().numpy(),
                               rtol=1e-2, atol=1e-2)
    Sg = torch.empty((M, N // 2), device="cuda", dtype=torch.bfloat16)
    gemm(3, A, Bt, Sg, M, N, K)
    r = ref.view(M, N // 128, 2, 64)
    gate, up = r[:, :, 0, :].reshape(M, N // 2), r[:, :, 1, :].reshape(M, N // 2)
    want = (gate * torch.sigmoid(gate) * up)
    np.testing.assert_allclose(Sg.float().cpu().numpy(), want.float().cpu().numpy(), rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("M", [333, 2500])  # 2500 rows: the persistent kernel (160 tiles)
def test_gemm_rows_independent_of_batch_bitwise(M):
    K, N = 2048, 1024
    g = torch.Generator(device="cuda").manual_seed(2)
    A, Bt = _bf((M, K), g), _bf((N, K), g)
    big = torch.empty((M, N), device="cuda")
    gemm(16, A, Bt, big, M, N, K)
    for r in (0, 127, 128, M - 1):
        one = torch.empty((1, N), device="cuda")
        gemm(16, A[r:r + 1].contiguous(), Bt, one, 1, N, K)
        assert torch.equal(one[0], big[r]), r


def _qkv(x, w_t, nq, nkv, row_slot, row_apply, down, up_t, n_slots, rank, targets):
    M, K = x.shape
    out = torch.empty((M, nq + 2 * nkv), device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(3 * M * n_slots * rank + 4096, device="cuda", dtype=torch.bfloat16)
    rc = lib.alora_qkv_proj(_native.ALORA_BF16, x.data_ptr(), M, K, w_t.data_ptr(), nq, nkv,
                            row_slot.data_ptr(), row_apply.data_ptr(), down.data_ptr(), up_t.data_ptr(),
                            n_slots, rank, targets.data_ptr(), ws.data_ptr(), out.data_ptr(), out.shape[1], _stream())
    _native.check(rc, "alora_qkv_proj")
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("M", [3, 130, 700, 4000])  # 4000: persistent kernel with the LoRA extra K
def test_qkv_proj_fused_lora_bf16(M):
    K, nq, nkv, n_slots, rank = 512, 512, 128, 3, 32
    g = torch.Generator(device="cuda").manual_seed(M)
    x = _bf((M, K), g)
    w_t = _bf((nq + 2 * nkv, K), g, 0.05)
    down = _bf((3, n_slots, rank, K), g, 0.05)
    up_t = _bf((nq + 2 * nkv, n_slots * rank), g, 0.05)
    targets = torch.tensor([0b111, 0b101, 0b010], dtype=torch.uint8, device="cuda")
    row_slot = torch.randint(-1, n_slots, (M,), generator=g, device="cuda", dtype=torch.int32)
    row_apply = (torch.rand(M, generator=g, device="cuda") < 0.6).to(torch.uint8)
    out = _qkv(x, w_t, nq, nkv, row_slot, row_apply, down, up_t, n_slots, rank, targets)
    base = _qkv(x, w_t, nq, nkv, torch.full_like(row_slot, -1), torch.zeros_like(row_apply), down, up_t, n_slots,
                rank, targets)
    # reference: base + bf16(x @ down_t[slot]) @ up_t[slot cols] where the row takes the delta and t is targeted
    ref = x.double() @ w_t.double().T
    offs = [(0, nq), (nq, nq + nkv), (nq + nkv, nq + 2 * nkv)]
    rs, ra = row_slot.cpu().numpy(), row_apply.cpu().numpy()
    tg = targets.cpu().numpy()
    takes = np.zeros((M, 3), bool)
    for m in range(M):
        s = rs[m]
        if s < 0 or not ra[m]:
            continue
        for t, (a, b) in enumerate(offs):
            if not (tg[s] >> t) & 1:
                continue
            takes[m, t] = True
            sh = (x[m].double() @ down[t, s].double().T).float().to(torch.bfloat16).double()
            ref[m, a:b] += sh @ up_t[a:b, s * rank:(s + 1) * rank].double().T
    got = out.double()
    err = ((got - ref).abs() / (ref.abs() + 1.0)).max().item()
    assert err < 2e-2, err
    # row select: untouched (row, projection) blocks are bit-identical to the base-only GEMM
    for t, (a, b) in enumerate(offs):
        keep = torch.as_tensor(~takes[:, t], device="cuda")
        assert torch.equal(out[keep, a:b], base[keep, a:b]), t
        if takes[:, t].any():
            chg = torch.as_tensor(takes[:, t], device="cuda")
            assert not torch.equal(out[chg, a:b], base[chg, a:b])
