"""Device-kernel parity: every CUDA kernel (through the C-ABI) against the CPU
oracle on identical inputs.  Integer / index outputs are bit-exact; floating
outputs carry the tolerance stated in each test."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
from oracle_lib import (O, REF, bf16_bits_to_f32, f32_to_bf16_bits, fill_bf16, fill_f32, ptr,
                        i32a, f64a)

pytestmark = pytest.mark.gpu

# Output tolerance of the expert FFN vs the fp64 oracle (bf16 storage of H and
# y, fp32 tensor-core accumulation):  |y - y_ref| <= ATOL + RTOL * |y_ref|.
BF16_ATOL, BF16_RTOL = 3e-2, 2e-2
# tf32 path (kind::tf32, 10-bit mantissa inputs, fp32 H): looser relative error
TF32_ATOL, TF32_RTOL = 2e-2, 2e-2


def _bf16_tensor(bits: np.ndarray, shape, dev):
    return torch.from_numpy(bits.view(np.int16).reshape(shape)).to(dev).view(torch.bfloat16)


def _to_np_f32(t):
    return t.float().cpu().numpy()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_fill_matches_oracle(cuda, dtype):
    n, seed, scale = 100003, 1234567, 0.37
    if dtype == "bf16":
        t = torch.empty(n, dtype=torch.bfloat16, device=cuda)
        dv.fill_uniform(t, seed, scale)
        got = t.view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, fill_bf16(seed, n, scale))
    else:
        t = torch.empty(n, dtype=torch.float32, device=cuda)
        dv.fill_uniform(t, seed, scale)
        assert np.array_equal(t.cpu().numpy().view(np.uint32),
                              fill_f32(seed, n, scale).view(np.uint32))


def _oracle_softmax(xf, wg, bias, E, k):
    N, d = xf.shape
    idx = np.zeros((N, k), np.int32)
    w = np.zeros((N, k), np.float32)
    cnt = np.zeros(E, np.int32)
    O.or_gate_softmax(ptr(np.ascontiguousarray(xf)), N, d, ptr(np.ascontiguousarray(wg)),
                      None if bias is None else ptr(bias), E, k, ptr(idx), ptr(w), ptr(cnt))
    return idx, w, cnt


@pytest.mark.parametrize("N,d,E,k,dtype,use_bias", [
    (512, 768, 8, 1, "f32", False),      # config 1 (C1)
    (1000, 4096, 32, 1, "bf16", False),  # C2 shape, ragged N
    (777, 1024, 64, 2, "bf16", True),    # C5-style top-2 with Zipf bias
    (37, 200, 5, 2, "bf16", True),       # d not a multiple of the chunk, E < 32
    (64, 256, 128, 3, "f32", False),
    (300, 512, 100, 8, "bf16", True),    # > 64 experts (16 per warp), k = 8
    (5, 8, 3, 3, "bf16", False),         # d = 8: one partial chunk, k = E
])
@pytest.mark.parametrize("inputs", ["uniform", "gaussian"])
def test_gate_softmax_topk_bitexact(cuda, N, d, E, k, dtype, use_bias, inputs):
    seed = 99 + N
    if inputs == "gaussian":  # gaussian_tokens x, W_g = GaussianStream x d^-1/2
        xb = im.gaussian_bf16(im.derive_seed(seed, 0), N * d)
        xf32 = np.empty(N * d, np.float32)
        im.gaussian_fill_typed("f32", [im.derive_seed(seed, 0)], [1.0], N * d, [xf32])
        xf = bf16_bits_to_f32(xb).reshape(N, d) if dtype == "bf16" else xf32.reshape(N, d)
        wg = np.ascontiguousarray((im.gaussian_stream(im.derive_seed(seed, 1), d * E) /
                                   np.sqrt(d)).astype(np.float32).reshape(d, E).T)
    else:
        xb = fill_bf16(seed, N * d, 1.7320508)
        xf = bf16_bits_to_f32(xb).reshape(N, d) if dtype == "bf16" else \
            fill_f32(seed, N * d, 1.7320508).reshape(N, d)
        wg = fill_f32(seed + 1, E * d, 1.7320508 / np.sqrt(d)).reshape(E, d)
    bias = (-0.8 * np.log(np.arange(1, E + 1))).astype(np.float32) if use_bias else None
    x = _bf16_tensor(xb, (N, d), cuda) if dtype == "bf16" else torch.from_numpy(xf).to(cuda)
    idx, w, cnt = dv.gate_softmax_topk(x, torch.from_numpy(wg).to(cuda), k,
                                       None if bias is None else torch.from_numpy(bias).to(cuda))
    ridx, rw, rcnt = _oracle_softmax(xf, wg, bias, E, k)
    assert np.array_equal(idx.cpu().numpy(), ridx)
    assert np.array_equal(cnt.cpu().numpy(), rcnt)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=1e-5, atol=1e-6)


def test_gate_softmax_ties_and_nan(cuda):
    # all-zero gate weights -> every logit ties -> experts 0..k-1 in order
    N, d, E, k = 40, 64, 6, 2
    x = torch.ones((N, d), dtype=torch.float32, device=cuda)
    wg = torch.zeros((E, d), dtype=torch.float32, device=cuda)
    idx, w, cnt = dv.gate_softmax_topk(x, wg, k)
    assert (idx[:, 0] == 0).all() and (idx[:, 1] == 1).all()
    assert torch.allclose(w, torch.full_like(w, 0.5))
    # NaN in one token: NaN logits never win over finite ones
    wg = torch.zeros((E, d), dtype=torch.float32, device=cuda)
    wg[3, 0] = 1.0
    x = torch.zeros((N, d), dtype=torch.float32, device=cuda)
    x[5, 0] = float("nan")
    idx, _, _ = dv.gate_softmax_topk(x, wg, 1)
    assert idx[5, 0].item() == 0  # expert 3 is NaN, the rest tie at 0 -> lowest index
    xf = x.cpu().numpy()
    ridx, _, _ = _oracle_softmax(xf, wg.cpu().numpy(), None, E, 1)
    assert np.array_equal(idx.cpu().numpy(), ridx)


@pytest.mark.parametrize("N,d,E,bits", [(512, 768, 8, 3), (4096, 4096, 32, 5),
                                        (3001, 1000, 64, 6), (100, 64, 3, 2)])
@pytest.mark.parametrize("inputs", ["uniform", "gaussian"])
def test_gate_lsh_matches_reference(cuda, N, d, E, bits, inputs):
    seed = 7 + N
    xb = im.gaussian_bf16(im.derive_seed(seed, 0), N * d) if inputs == "gaussian" else \
        fill_bf16(seed, N * d, 1.7320508)
    xf = bf16_bits_to_f32(xb).reshape(N, d)
    proj = im.gating_projection(im.derive_seed(seed, 2), bits, d)
    codes, idx, w, cnt = dv.gate_lsh(_bf16_tensor(xb, (N, d), cuda),
                                     torch.from_numpy(proj).to(cuda), E)
    # reference lsh_codes on the fp64 promotion of the same bf16 hidden states
    x64 = np.ascontiguousarray(xf.astype(np.float64))
    ref_codes = np.zeros(N, np.uint32)
    lib = REF if REF is not None else O
    fn = lib.ref_lsh_codes if REF is not None else lib.or_lsh_codes
    assert fn(im.derive_seed(seed, 2), bits, d, ptr(x64), N, ptr(ref_codes)) == 0
    assert np.array_equal(codes.cpu().numpy().view(np.uint32), ref_codes)
    assert np.array_equal(idx.cpu().numpy()[:, 0], (ref_codes % E).astype(np.int32))
    assert np.array_equal(cnt.cpu().numpy(), np.bincount(ref_codes % E, minlength=E))
    assert (w == 1.0).all()


@pytest.mark.parametrize("N,k,E,skew", [(4096, 1, 32, 0.0), (16384, 2, 64, 1.0), (5, 2, 7, 0.0),
                                        (3000, 1, 16, 3.0), (1, 1, 1, 0.0),
                                        (20000, 2, 64, 1.0),    # > 32768: multi-CTA path
                                        (4096, 1, 300, 0.5)])  # > 128 experts: multi-CTA
def test_dispatch_bitexact(cuda, N, k, E, skew):
    rng = np.random.default_rng(N + E)
    p = np.arange(1, E + 1, dtype=np.float64) ** (-skew)
    p /= p.sum()
    idx = rng.choice(E, size=(N, k), p=p).astype(np.int32)
    off, perm, inv = dv.dispatch(torch.from_numpy(idx).to(cuda), E)
    roff = np.zeros(E + 1, np.int32)
    rperm = np.zeros(N * k, np.int32)
    rinv = np.zeros(N * k, np.int32)
    O.or_dispatch(ptr(idx), N, k, E, ptr(roff), ptr(rperm), ptr(rinv))
    assert np.array_equal(off.cpu().numpy(), roff)
    assert np.array_equal(perm.cpu().numpy(), rperm)
    assert np.array_equal(inv.cpu().numpy(), rinv)


def _ffn_case(cuda, dtype, d, f, counts, seed=5):
    E = len(counts)
    R = int(sum(counts))
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    if dtype == "bf16":
        xb = fill_bf16(seed, R * d, 1.7320508)
        wib = fill_bf16(seed + 1, E * f * d, 1.7320508 / np.sqrt(d))
        wob = fill_bf16(seed + 2, E * d * f, 1.5340 * 1.7320508 / np.sqrt(f))
        xf, wif, wof = (bf16_bits_to_f32(a) for a in (xb, wib, wob))
        x = _bf16_tensor(xb, (R, d), cuda)
        wi = _bf16_tensor(wib, (E, f, d), cuda)
        wo = _bf16_tensor(wob, (E, d, f), cuda)
    else:
        xf = fill_f32(seed, R * d, 1.7320508)
        wif = fill_f32(seed + 1, E * f * d, 1.7320508 / np.sqrt(d))
        wof = fill_f32(seed + 2, E * d * f, 1.5340 * 1.7320508 / np.sqrt(f))
        x = torch.from_numpy(xf.reshape(R, d)).to(cuda)
        wi = torch.from_numpy(wif.reshape(E, f, d)).to(cuda)
        wo = torch.from_numpy(wof.reshape(E, d, f)).to(cuda)
    h, y = dv.expert_ffn(x, torch.from_numpy(offsets).to(cuda), wi, wo)
    torch.cuda.synchronize()
    ref = np.zeros((R, d), np.float32)
    xf = xf.reshape(R, d)
    for e in range(E):
        a, b = offsets[e], offsets[e + 1]
        if b > a:
            O.or_expert_ffn(ptr(np.ascontiguousarray(xf[a:b])), b - a, d, f,
                            ptr(np.ascontiguousarray(wif[e * f * d:(e + 1) * f * d])),
                            ptr(np.ascontiguousarray(wof[e * d * f:(e + 1) * d * f])),
                            1 if dtype == "bf16" else 0, ptr(ref[a:b]))
    return _to_np_f32(y), ref


@pytest.mark.parametrize("counts", [
    [128, 0, 1, 300, 127, 129, 256, 513],  # empty expert, tails, >2 sub-tiles
    [40] * 4,
])
def test_expert_ffn_bf16_vs_oracle(cuda, counts):
    y, ref = _ffn_case(cuda, "bf16", 256, 512, counts)
    err = np.abs(y - ref)
    assert np.all(err <= BF16_ATOL + BF16_RTOL * np.abs(ref)), (err.max(), np.abs(ref).max())
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert rel < 5e-3, rel


def test_expert_ffn_tf32_vs_oracle(cuda):
    y, ref = _ffn_case(cuda, "f32", 768, 384, [64, 100, 0, 200])
    err = np.abs(y - ref)
    assert np.all(err <= TF32_ATOL + TF32_RTOL * np.abs(ref)), err.max()


def test_expert_ffn_vs_torch_fp32(cuda):
    """fp32 torch reference of the same op (bf16 inputs, fp32 math)."""
    d, f, counts = 512, 1024, [130, 70, 0, 255]
    E, R = len(counts), sum(counts)
    g = torch.Generator(device="cpu").manual_seed(0)
    x = (torch.randn(R, d, generator=g)).to(torch.bfloat16).to(cuda)
    wi = (torch.randn(E, f, d, generator=g) / d ** 0.5).to(torch.bfloat16).to(cuda)
    wo = (torch.randn(E, d, f, generator=g) / f ** 0.5).to(torch.bfloat16).to(cuda)
    offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int32, device=cuda)
    h, y = dv.expert_ffn(x, offs, wi, wo)
    ref = torch.empty(R, d, device=cuda)
    for e in range(E):
        a, b = int(offs[e]), int(offs[e + 1])
        hh = torch.nn.functional.gelu(x[a:b].float() @ wi[e].float().t())
        ref[a:b] = hh.to(torch.bfloat16).float() @ wo[e].float().t()
    err = (y.float() - ref).abs()
    assert (err <= BF16_ATOL + BF16_RTOL * ref.abs()).all(), err.max().item()


@pytest.mark.parametrize("d", [256, 1160])
@pytest.mark.parametrize("k,dtype", [(1, "bf16"), (2, "bf16"), (2, "f32")])
def test_combine_bitexact(cuda, k, dtype, d):
    N, E = 300, 9
    rng = np.random.default_rng(k)
    idx = np.stack([rng.permutation(E)[:k] for _ in range(N)]).astype(np.int32)
    w = rng.random((N, k)).astype(np.float32)
    roff = np.zeros(E + 1, np.int32)
    perm = np.zeros(N * k, np.int32)
    inv = np.zeros(N * k, np.int32)
    O.or_dispatch(ptr(idx), N, k, E, ptr(roff), ptr(perm), ptr(inv))
    yp = rng.standard_normal((N * k, d)).astype(np.float32)
    if dtype == "bf16":
        yb = f32_to_bf16_bits(yp)
        yp = bf16_bits_to_f32(yb).reshape(N * k, d)
        ypt = _bf16_tensor(yb, (N * k, d), cuda)
    else:
        ypt = torch.from_numpy(yp).to(cuda)
    y = dv.combine(ypt, torch.from_numpy(inv).to(cuda), torch.from_numpy(w).to(cuda), N, k)
    ref = np.zeros((N, d), np.float32)
    O.or_combine(ptr(np.ascontiguousarray(yp)), ptr(inv), ptr(w), N, k, d, ptr(ref))
    if dtype == "bf16":
        assert np.array_equal(y.view(torch.int16).cpu().numpy().view(np.uint16),
                              f32_to_bf16_bits(ref))
    else:
        assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("counts", [[128, 0, 1, 300, 127, 129, 256, 513], [150] * 32])
def test_fused_ffn_equals_two_launch_path(cuda, counts):
    """The one-launch FFN (phase-2 tiles gated on per-expert completion
    counters) is bit-identical to the two-launch path, and its fused top-1
    combine is bit-identical to the separate combine kernel."""
    E, d, f = len(counts), 256, 512
    R = int(sum(counts))
    offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int32, device=cuda)
    g = torch.Generator(device="cpu").manual_seed(3)
    x = torch.randn(R, d, generator=g).to(torch.bfloat16).to(cuda)
    wi = (torch.randn(E, f, d, generator=g) / d ** 0.5).to(torch.bfloat16).to(cuda)
    wo = (torch.randn(E, d, f, generator=g) / f ** 0.5).to(torch.bfloat16).to(cuda)
    h2, y2 = dv.expert_ffn(x, offs, wi, wo)
    h1, y1 = dv.expert_ffn_fused(x, offs, wi, wo)
    torch.cuda.synchronize()
    assert torch.equal(h1.view(torch.int16), h2.view(torch.int16))
    assert torch.equal(y1.view(torch.int16), y2.view(torch.int16))
    # fused combine: rows are a permutation of R tokens (top-1)
    perm = torch.randperm(R, generator=g).to(torch.int32).to(cuda)
    inv = torch.empty_like(perm)
    inv[perm.long()] = torch.arange(R, dtype=torch.int32, device=cuda)
    w = torch.rand(R, generator=g).to(cuda)
    _, yc = dv.expert_ffn_fused(x, offs, wi, wo, perm=perm, topk_w=w, n_tokens=R)
    ref = dv.combine(y2, inv, w, R, 1)
    torch.cuda.synchronize()
    assert torch.equal(yc.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("d", [256, 1160, 4096])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_gather_rows_both_forms(cuda, k, d):
    """x_perm[p] = x[perm[p] / k]: the perm-driven and the token-major
    (inv-driven, one read per token row) gathers are bit-identical to numpy."""
    N, E = 777, 13
    rng = np.random.default_rng(100 + k)
    idx = np.stack([rng.permutation(E)[:k] for _ in range(N)]).astype(np.int32)
    off, perm, inv = dv.dispatch(torch.from_numpy(idx).to(cuda), E)
    xb = fill_bf16(7 + k, N * d, 1.0)
    x = _bf16_tensor(xb, (N, d), cuda)
    a = dv.gather_rows(x, perm, k)
    b = dv.gather_rows_by_token(x, inv, k)
    ref = xb.reshape(N, d)[perm.cpu().numpy() // k]
    assert np.array_equal(a.view(torch.int16).cpu().numpy().view(np.uint16), ref)
    assert np.array_equal(b.view(torch.int16).cpu().numpy().view(np.uint16), ref)
