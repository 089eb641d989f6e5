"""N1a softmax gate on tensor cores (gate.cu, "N1a on tensor cores"): the
tcgen05 logits only pre-select candidates; every pick comes from the exact
fmaf chain, so indices and counts must equal the CUDA-core gate's (and the
oracle's, oracle.c or_gate_softmax) bit for bit, weights within rtol 1e-5.
These tests drive the path through the C-ABI test hook
infmoe_gate_softmax_debug, which also returns the approximate logits and the
candidate counters, so each test states which path it exercised."""
import os

import numpy as np
import pytest
import torch

import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
from oracle_lib import O, bf16_bits_to_f32, ptr

pytestmark = pytest.mark.gpu

W_RTOL, W_ATOL = 1e-5, 1e-6


def _inputs(seed, N, d, E, bias_c):
    xb = im.gaussian_bf16(im.derive_seed(seed, 0), N * d)
    xf = bf16_bits_to_f32(xb).reshape(N, d)
    wg = np.ascontiguousarray((im.gaussian_stream(im.derive_seed(seed, 1), d * E) /
                               np.sqrt(d)).astype(np.float32).reshape(d, E).T)
    bias = (-bias_c * np.log(np.arange(1, E + 1))).astype(np.float32) if bias_c else None
    return xb, xf, wg, bias


def _oracle(xf, wg, bias, k):
    N, d = xf.shape
    E = wg.shape[0]
    idx = np.zeros((N, k), np.int32)
    w = np.zeros((N, k), np.float32)
    cnt = np.zeros(E, np.int32)
    O.or_gate_softmax(ptr(np.ascontiguousarray(xf)), N, d, ptr(np.ascontiguousarray(wg)),
                      None if bias is None else ptr(bias), E, k, ptr(idx), ptr(w), ptr(cnt))
    return idx, w, cnt


def _run(cuda, xb, wg, bias, k):
    d = wg.shape[1]
    x = torch.from_numpy(xb.view(np.int16).reshape(xb.size // d, d)).to(cuda).view(torch.bfloat16)
    return dv.gate_softmax_topk(x, torch.from_numpy(wg).to(cuda), k,
                                None if bias is None else torch.from_numpy(bias).to(cuda),
                                debug=True)


def _check(got, ref):
    idx, w, cnt = got[:3]
    ridx, rw, rcnt = ref
    assert np.array_equal(idx.cpu().numpy(), ridx)
    assert np.array_equal(cnt.cpu().numpy(), rcnt)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=W_RTOL, atol=W_ATOL)


@pytest.mark.parametrize("N,d,E,k,bias_c", [
    (16384, 4096, 64, 2, 0.6258),  # C5: the bench's calibrated Zipf bias
    (1000, 4096, 32, 2, 0.0),
    (129, 1024, 5, 2, 1.0),        # E = 5 (Ep = 32), one token past a 128-row tile
    (300, 512, 100, 8, 0.8),       # E = 100 (Ep = 128), k = 8
    (513, 768, 80, 3, 0.5),        # E = 80 (Ep = 96: 4 hi segments of 96 TMEM columns)
    (1, 64, 8, 3, 0.0),            # one token, one K-block
])
def test_tc_gate_matches_oracle(cuda, N, d, E, k, bias_c):
    xb, xf, wg, bias = _inputs(7 + N + E, N, d, E, bias_c)
    got = _run(cuda, xb, wg, bias, k)
    assert got[3] is not None, "expected the tensor-core path"
    _check(got, _oracle(xf, wg, bias, k))
    stats = got[4]
    assert stats["certified"] + stats["fallback"] == N
    assert stats["full_exact"] == 0
    # most tokens are decided by the tensor-core logits; the rest need few chains
    if N >= 1000:
        assert stats["fallback"] <= 0.25 * N, stats
    assert stats["candidates"] <= stats["fallback"] * min(E, k + 6)


def test_tc_gate_error_within_model(cuda):
    """|L~ - x.w| against the bound's tensor-core term gamma_tc ||x|| ||w||: the
    model must hold with room to spare on the C5 inputs."""
    N, d, E = 4096, 4096, 64
    xb, xf, wg, _ = _inputs(311, N, d, E, 0.0)
    got = _run(cuda, xb, wg, None, 2)
    approx = got[3].cpu().numpy().astype(np.float64)
    exact = xf.astype(np.float64) @ wg.astype(np.float64).T
    scale = np.linalg.norm(xf.astype(np.float64), axis=1)[:, None] * \
        np.linalg.norm(wg.astype(np.float64), axis=1)[None, :]
    ratio = np.abs(approx - exact) / scale
    # the bound's hi term: 17 2^-23 (m + 1), m = 4 MMAs x 10 K-blocks per hi
    # accumulator (d = 4096, Ep = 64: 7 hi segments + the mid/lo accumulator)
    gamma_tc = 17 * 2.0 ** -23 * (4 * 10 + 1)
    print(f"max |L~ - x.w| / (||x|| ||w||) = {ratio.max():.3e}  (gamma_tc {gamma_tc:.3e})")
    assert ratio.max() < gamma_tc / 8, (ratio.max(), gamma_tc)


def test_tc_gate_planted_near_ties(cuda):
    """Experts whose gate rows are equal or one ulp apart: the approximate
    logits cannot order them, the exact chain must (lower index on ties)."""
    N, d, E, k = 2048, 1024, 16, 2
    xb, xf, wg, _ = _inputs(5, N, d, E, 0.0)
    wg[1] = wg[0]                                        # exact ties
    wg[3] = wg[2]
    wg[3, 17] = np.nextafter(wg[3, 17], np.float32(np.inf))  # one ulp apart
    wg[5] = wg[4] * np.float32(1 + 2 ** -20)
    wg = np.ascontiguousarray(wg)
    got = _run(cuda, xb, wg, None, k)
    assert got[3] is not None
    ref = _oracle(xf, wg, None, k)
    _check(got, ref)
    # pairs that tie on the approximate logits really did go through the chain
    assert got[4]["fallback"] > 0 and got[4]["candidates"] > k * got[4]["fallback"]
    picks = ref[0]
    assert ((picks[:, 0] == 0) & (picks[:, 1] == 1)).sum() > 0  # the tie resolved to 0, 1


def test_tc_gate_nonfinite_rows_take_exact_path(cuda):
    N, d, E, k = 256, 512, 32, 2
    xb, xf, wg, bias = _inputs(19, N, d, E, 0.5)
    for t, v in ((3, 0x7FC0), (40, 0x7F80), (41, 0xFF80)):  # NaN, +inf, -inf
        xb[t * d + 11] = v
    xf = bf16_bits_to_f32(xb).reshape(N, d)
    got = _run(cuda, xb, wg, bias, k)
    ref = _oracle(xf, wg, bias, k)
    idx, w = got[0].cpu().numpy(), got[1].cpu().numpy()
    assert np.array_equal(idx, ref[0])
    assert np.array_equal(got[2].cpu().numpy(), ref[2])
    finite = np.isfinite(ref[1]).all(axis=1)
    np.testing.assert_allclose(w[finite], ref[1][finite], rtol=W_RTOL, atol=W_ATOL)
    assert got[4]["full_exact"] >= 3


def test_tc_gate_force_exact_and_cuda_core_path_agree(cuda):
    N, d, E, k = 3000, 2048, 64, 2
    xb, xf, wg, bias = _inputs(23, N, d, E, 0.6)
    ref = _oracle(xf, wg, bias, k)
    tc = _run(cuda, xb, wg, bias, k)
    _check(tc, ref)
    try:
        os.environ["INFMOE_GATE_TC_FORCE_EXACT"] = "1"
        fe = _run(cuda, xb, wg, bias, k)
    finally:
        del os.environ["INFMOE_GATE_TC_FORCE_EXACT"]
    assert fe[4]["certified"] == 0 and fe[4]["full_exact"] == N
    assert fe[4]["candidates"] == N * E
    _check(fe, ref)
    try:
        os.environ["INFMOE_GATE_TC"] = "0"
        cc = _run(cuda, xb, wg, bias, k)
    finally:
        del os.environ["INFMOE_GATE_TC"]
    assert cc[3] is None  # the CUDA-core kernel ran
    _check(cc, ref)
    assert np.array_equal(cc[0].cpu().numpy(), tc[0].cpu().numpy())


def test_tc_gate_workspace_api(cuda):
    """infmoe_gate_softmax_ws_bytes / _prepare / _topk_ws: W_g split once, same
    results as the one-shot call; 0 bytes (CUDA-core path) for top-1."""
    N, d, E, k = 700, 1024, 48, 2
    xb, xf, wg, bias = _inputs(31, N, d, E, 0.7)
    x = torch.from_numpy(xb.view(np.int16).reshape(N, d)).to(cuda).view(torch.bfloat16)
    g, b = torch.from_numpy(wg).to(cuda), torch.from_numpy(bias).to(cuda)
    ws = dv.GateWorkspace(g, N, k)
    assert ws.nbytes > 0
    ref = _oracle(xf, wg, bias, k)
    for n in (N, 300):  # fewer tokens than the workspace was sized for
        got = dv.gate_softmax_topk(x[:n], g, k, b, workspace=ws)
        r = _oracle(xf[:n], wg, bias, k)
        _check(got, r)
    assert dv.GateWorkspace(g, N, 1).nbytes == 0
    got1 = dv.gate_softmax_topk(x, g, 1, b, workspace=dv.GateWorkspace(g, N, 1))
    _check(got1, _oracle(xf, wg, bias, 1))
    del ref


def test_tc_gate_faster_than_cuda_core_at_c5(cuda):
    N, d, E, k = 16384, 4096, 64, 2
    xb, _, wg, bias = _inputs(29, N, d, E, 0.6258)
    x = torch.from_numpy(xb.view(np.int16).reshape(N, d)).to(cuda).view(torch.bfloat16)
    g, b = torch.from_numpy(wg).to(cuda), torch.from_numpy(bias).to(cuda)
    ws = dv.GateWorkspace(g, N, k)

    def timed(**kw):
        for _ in range(3):
            dv.gate_softmax_topk(x, g, k, b, **kw)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            dv.gate_softmax_topk(x, g, k, b, **kw)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / 10

    t_ws = timed(workspace=ws)
    t_tc = timed()
    try:
        os.environ["INFMOE_GATE_TC"] = "0"
        t_cc = timed()
    finally:
        del os.environ["INFMOE_GATE_TC"]
    print(f"C5 gate: tensor-core {t_ws * 1e3:.1f} us with a prepared workspace, "
          f"{t_tc * 1e3:.1f} us one-shot, CUDA-core {t_cc * 1e3:.1f} us")
    assert t_ws < 0.3 * t_cc and t_tc < 0.5 * t_cc
