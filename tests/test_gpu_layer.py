"""End-to-end MoE layer (the C-ABI handle) on the GPU against the oracle
chain, resident and offloaded; the offloaded order against the reference
scheduler; the measured timeline against replay_check's rules."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
from oracle_lib import (O, REF, EventRec, bf16_bits_to_f32, f32_to_bf16_bits, fill_bf16, ptr,
                        f64a, i32a, schedule)

pytestmark = pytest.mark.gpu

ATOL, RTOL = 3e-2, 2e-2  # bf16 layer output vs fp64 oracle chain


def _setup(cuda, N, d, f, E, seed=11):
    xb = fill_bf16(im.derive_seed(seed, 0), N * d, 1.7320508)
    wib = fill_bf16(im.derive_seed(seed, 1000), E * f * d, 1.7320508 / np.sqrt(d))
    wob = fill_bf16(im.derive_seed(seed, 1001), E * d * f, 1.5340 * 1.7320508 / np.sqrt(f))
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    return (xb, wib, wob), (t(xb, (N, d)).to(cuda), t(wib, (E, f, d)), t(wob, (E, d, f)))


def _oracle_layer(xb, wib, wob, N, d, f, E, k, idx, w):
    xf = bf16_bits_to_f32(xb).reshape(N, d)
    wif, wof = bf16_bits_to_f32(wib), bf16_bits_to_f32(wob)
    off = np.zeros(E + 1, np.int32)
    perm = np.zeros(N * k, np.int32)
    inv = np.zeros(N * k, np.int32)
    O.or_dispatch(ptr(idx), N, k, E, ptr(off), ptr(perm), ptr(inv))
    xp = np.ascontiguousarray(xf[perm // k])
    yp = np.zeros((N * k, d), np.float32)
    for e in range(E):
        a, b = off[e], off[e + 1]
        if b > a:
            O.or_expert_ffn(ptr(np.ascontiguousarray(xp[a:b])), b - a, d, f,
                            ptr(np.ascontiguousarray(wif[e * f * d:(e + 1) * f * d])),
                            ptr(np.ascontiguousarray(wof[e * d * f:(e + 1) * d * f])), 1,
                            ptr(yp[a:b]))
    yp = bf16_bits_to_f32(f32_to_bf16_bits(yp)).reshape(N * k, d)  # device stores y_perm bf16
    y = np.zeros((N, d), np.float32)
    O.or_combine(ptr(yp), ptr(inv), ptr(np.ascontiguousarray(w)), N, k, d, ptr(y))
    return y


@pytest.mark.parametrize("gate", ["lsh", "softmax"])
def test_resident_layer_vs_oracle(cuda, gate):
    N, d, f, E = 600, 256, 512, 8
    k = 1 if gate == "lsh" else 2
    (xb, wib, wob), (x, wi, wo) = _setup(cuda, N, d, f, E)
    gw = (np.random.default_rng(0).standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
    layer = dv.MoELayer(d, f, E, k, wi.to(cuda), wo.to(cuda), gate=gate, gate_weight=gw,
                        lsh_seed=77, lsh_bits=3, max_tokens=N)
    y, info = layer.forward(x)
    torch.cuda.synchronize()
    xf = bf16_bits_to_f32(xb).reshape(N, d)
    idx = np.zeros((N, k), np.int32)
    w = np.zeros((N, k), np.float32)
    cnt = np.zeros(E, np.int32)
    if gate == "lsh":
        proj = im.gating_projection(77, 3, d)
        O.or_gate_lsh(ptr(xf), N, d, ptr(np.ascontiguousarray(proj)), 3, E, ptr(idx), ptr(w),
                      ptr(cnt))
    else:
        O.or_gate_softmax(ptr(xf), N, d, ptr(gw), None, E, k, ptr(idx), ptr(w), ptr(cnt))
    assert np.array_equal(info["counts"], cnt)
    ref = _oracle_layer(xb, wib, wob, N, d, f, E, k, idx, w)
    got = y.float().cpu().numpy()
    err = np.abs(got - ref)
    assert np.all(err <= ATOL + RTOL * np.abs(ref)), err.max()
    layer.close()


@pytest.mark.parametrize("K,policy", [(1, im.POLICY_AUTO), (3, im.POLICY_AUTO),
                                      (2, im.POLICY_NAIVE)])
def test_offloaded_layer_equals_resident_and_reference_order(cuda, K, policy):
    N, d, f, E = 1000, 256, 384, 12
    (xb, wib, wob), (x, wi, wo) = _setup(cuda, N, d, f, E, seed=3)
    res = dv.MoELayer(d, f, E, 1, wi.to(cuda), wo.to(cuda), gate="lsh", lsh_seed=5, lsh_bits=4,
                      max_tokens=N)
    y_res, info_r = res.forward(x)
    hw = im.Hardware(1e12, 2e10, 80 << 30, 8 << 30)
    off = dv.MoELayer(d, f, E, 1, wi.pin_memory(), wo.pin_memory(), gate="lsh", lsh_seed=5,
                      lsh_bits=4, offloaded=True, K=K, policy=policy, max_tokens=N, hw=hw)
    y_off, info = off.forward(x, want_timeline=True)
    torch.cuda.synchronize()
    # same kernels, same tiles -> bit-identical output whatever the expert order
    assert torch.equal(y_res.view(torch.int16), y_off.view(torch.int16))
    assert np.array_equal(info["counts"], info_r["counts"])
    # the executed order is the reference scheduler's order for these counts
    g = im.make_geometry(d, f, E, 2)
    cv = im.compute_costs(info["counts"].astype(np.uint64), g, hw)
    if policy == im.POLICY_AUTO:
        want = schedule("ref" if REF is not None else "or", cv.alphas, cv.beta, K, "auto")[1]
    else:
        want = list(range(E))
    assert info["order"].tolist() == want
    # measured timeline: one lane each, causality, <= K completed residents
    # (simulator.hpp:147-155: load j completes after compute j-K ends; the copy
    # in flight uses the (K+1)-th slot, D6)
    ev = info["events"]
    loads = sorted([e for e in ev if e[0] == 0], key=lambda e: e[3])
    comps = sorted([e for e in ev if e[0] == 1], key=lambda e: e[3])
    for lane in (loads, comps):
        for a, b in zip(lane, lane[1:]):
            assert a[4] <= b[3] + 1e-6
    le = {e[2]: e[4] for e in loads}
    for c in comps:
        assert c[3] >= le[c[2]] - 1e-6
    marks = sorted([(le[c[2]], 1) for c in comps] + [(c[4] - 1e-6, -1) for c in comps])
    cur = peak = 0
    for _, dlt in sorted(marks, key=lambda m: (m[0], m[1])):
        cur += dlt
        peak = max(peak, cur)
    assert peak <= K
    assert info["exposed_copy_s"] > 0
    off.close()
    res.close()


def test_offloaded_layer_host_weight_swap(cuda):
    N, d, f, E = 256, 128, 256, 4
    (_, _, _), (x, wi, wo) = _setup(cuda, N, d, f, E, seed=8)
    (_, _, _), (_, wi2, wo2) = _setup(cuda, N, d, f, E, seed=9)
    off = dv.MoELayer(d, f, E, 1, wi.pin_memory(), wo.pin_memory(), gate="lsh", lsh_seed=1,
                      lsh_bits=2, offloaded=True, K=1, max_tokens=N)
    res2 = dv.MoELayer(d, f, E, 1, wi2.to(cuda), wo2.to(cuda), gate="lsh", lsh_seed=1,
                       lsh_bits=2, max_tokens=N)
    off.set_host_weights(wi2.clone(), wo2.clone())  # pageable: registered by the handle
    y1, _ = off.forward(x)
    y2, _ = res2.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.int16), y2.view(torch.int16))
    off.close()
    res2.close()


def test_layer_rejects_bad_config(cuda):
    wi = torch.zeros(2, 128, 128, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ValueError):
        dv.MoELayer(128, 128, 2, 2, wi, wi, gate="lsh", lsh_bits=1)  # LSH is top-1
    with pytest.raises(ValueError):
        dv.MoELayer(128, 100, 2, 1, wi, wi, gate="lsh", lsh_bits=1).forward(
            torch.zeros(4, 128, dtype=torch.bfloat16, device=cuda))  # d_ff % 128


def test_offloaded_skip_empty_experts_and_measured_timeline(cuda):
    """skip_empty_experts: with few tokens most experts get no
    rows; they are neither scheduled nor loaded, the output is unchanged, and
    the MEASURED timeline passes the replay_check rules (one lane per stream,
    causality, <= K residents)."""
    from paper_2106_10715_b200 import trace
    N, d, f, E, K = 24, 256, 384, 16, 2
    (_, _, _), (x, wi, wo) = _setup(cuda, N, d, f, E, seed=21)
    res = dv.MoELayer(d, f, E, 1, wi.to(cuda), wo.to(cuda), gate="lsh", lsh_seed=2, lsh_bits=4,
                      max_tokens=N)
    y_res, info_r = res.forward(x)
    full = dv.MoELayer(d, f, E, 1, wi.pin_memory(), wo.pin_memory(), gate="lsh", lsh_seed=2,
                       lsh_bits=4, offloaded=True, K=K, max_tokens=N)
    skip = dv.MoELayer(d, f, E, 1, wi.pin_memory(), wo.pin_memory(), gate="lsh", lsh_seed=2,
                       lsh_bits=4, offloaded=True, K=K, max_tokens=N, skip_empty_experts=True)
    y_full, info_f = full.forward(x, want_timeline=True)
    y_skip, info_s = skip.forward(x, want_timeline=True)
    torch.cuda.synchronize()
    assert torch.equal(y_res.view(torch.int16), y_full.view(torch.int16))
    assert torch.equal(y_res.view(torch.int16), y_skip.view(torch.int16))
    nonempty = int((info_r["counts"] > 0).sum())
    assert nonempty < E
    loaded = [e for e in info_s["order"].tolist() if e >= 0]
    assert sorted(loaded) == sorted(np.nonzero(info_r["counts"])[0].tolist())
    assert len(info_s["events"]) == 2 * nonempty and len(info_f["events"]) == 2 * E
    g = im.make_geometry(d, f, E, 2)
    cv = im.compute_costs(info_r["counts"].astype(np.uint64), g,
                          im.Hardware(1643.6e12, 55.5e9, 180 << 30, 8 << 30))
    for info in (info_f, info_s):
        assert im.replay_check(info["events"], [cv], K, check_durations=False,
                               tol_s=2e-6) == {}
    trace.write(info_f["events"], "/tmp/infmoe_layer_timeline")
    for lay in (res, full, skip):
        lay.close()


def test_resident_stack_cuda_graph_replay_matches_eager(cuda):
    """A resident layer never synchronises with the host, so a multi-layer
    stack is capturable as one CUDA graph; replay must equal eager bit for bit."""
    N, d, f, E, L = 512, 256, 384, 8, 3
    (_, _, _), (x, wi, wo) = _setup(cuda, N, d, f, E, seed=31)
    wi, wo = wi.to(cuda), wo.to(cuda)
    layers = [dv.MoELayer(d, f, E, 1, wi, wo, gate="lsh", lsh_seed=40 + l, lsh_bits=3,
                          max_tokens=N) for l in range(L)]
    bufs = [torch.empty_like(x) for _ in range(2)]

    def run():
        cur = x
        for i, lay in enumerate(layers):
            lay.forward(cur, bufs[i % 2], want_info=False)
            cur = bufs[i % 2]
        return cur

    eager = run().clone()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = run()
    bufs[0].zero_()
    bufs[1].zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), eager.view(torch.int16))
    for lay in layers:
        lay.close()


def test_offloaded_stack_shares_one_slot_pool(cuda):
    """Offloaded layers of a stack sharing ONE pool of K+1 slots (the InfMoE
    memory model: K experts on the GPU in total) give the same bits as layers
    with private slots and as the resident stack; every layer's measured
    timeline passes replay_check with <= K residents; a pool of another K or
    expert size is rejected."""
    N, d, f, E, K, L = 700, 256, 384, 8, 2, 3
    sets = [_setup(cuda, N, d, f, E, seed=50 + l)[1] for l in range(L)]
    x = sets[0][0]
    pool = dv.SlotPool(K, d, f)
    kw = dict(gate="lsh", lsh_bits=3, max_tokens=N)
    shared = [dv.MoELayer(d, f, E, 1, s[1].pin_memory(), s[2].pin_memory(), lsh_seed=60 + l,
                          offloaded=True, K=K, slot_pool=pool, **kw) for l, s in enumerate(sets)]
    private = [dv.MoELayer(d, f, E, 1, s[1].pin_memory(), s[2].pin_memory(), lsh_seed=60 + l,
                           offloaded=True, K=K, **kw) for l, s in enumerate(sets)]
    resident = [dv.MoELayer(d, f, E, 1, s[1].to(cuda), s[2].to(cuda), lsh_seed=60 + l, **kw)
                for l, s in enumerate(sets)]
    outs, infos = [], []
    for stack in (shared, private, resident):
        cur = x
        for lay in stack:
            cur, info = lay.forward(cur, want_timeline=stack is shared)
            if stack is shared:
                infos.append(info)
        outs.append(cur)
    torch.cuda.synchronize()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    assert torch.equal(outs[0].view(torch.int16), outs[2].view(torch.int16))
    g = im.make_geometry(d, f, E, 2)
    hw = im.Hardware(1643.6e12, 55.5e9, 180 << 30, 8 << 30)
    for info in infos:
        cv = im.compute_costs(info["counts"].astype(np.uint64), g, hw)
        assert im.replay_check(info["events"], [cv], K, check_durations=False,
                               tol_s=2e-6) == {}
    with pytest.raises(ValueError):
        dv.MoELayer(d, f, E, 1, sets[0][1].pin_memory(), sets[0][2].pin_memory(), lsh_seed=1,
                    offloaded=True, K=K + 1, slot_pool=pool, **kw)
    with pytest.raises(ValueError):
        dv.MoELayer(d, 2 * f, E, 1, torch.zeros(E, 2 * f, d, dtype=torch.bfloat16).pin_memory(),
                    torch.zeros(E, d, 2 * f, dtype=torch.bfloat16).pin_memory(), lsh_seed=1,
                    offloaded=True, K=K, slot_pool=pool, **kw)
    for lay in shared + private + resident:
        lay.close()
    pool.close()


@pytest.mark.parametrize("gate,k", [("lsh", 1), ("softmax", 2)])
@pytest.mark.parametrize("offloaded", [False, True])
def test_layer_edge_token_counts(cuda, gate, k, offloaded):
    """N = 0 (nothing routed: every expert empty) and N = 1 through the layer
    handle, resident and offloaded; N = 1 matches the oracle chain."""
    N, d, f, E = 64, 256, 384, 6
    (xb, wib, wob), (x, wi, wo) = _setup(cuda, N, d, f, E, seed=71)
    gw = (np.random.default_rng(1).standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
    wts = (wi.pin_memory(), wo.pin_memory()) if offloaded else (wi.to(cuda), wo.to(cuda))
    layer = dv.MoELayer(d, f, E, k, *wts, gate=gate, gate_weight=gw, lsh_seed=9, lsh_bits=3,
                        offloaded=offloaded, K=2, max_tokens=N)
    y0, info0 = layer.forward(x[:0])
    torch.cuda.synchronize()
    assert y0.shape == (0, d) and int(info0["counts"].sum()) == 0
    y1, info1 = layer.forward(x[:1])
    torch.cuda.synchronize()
    xf = bf16_bits_to_f32(xb).reshape(N, d)[:1].copy()
    idx = np.zeros((1, k), np.int32)
    w = np.zeros((1, k), np.float32)
    cnt = np.zeros(E, np.int32)
    if gate == "lsh":
        proj = np.ascontiguousarray(im.gating_projection(9, 3, d))
        O.or_gate_lsh(ptr(xf), 1, d, ptr(proj), 3, E, ptr(idx), ptr(w), ptr(cnt))
    else:
        O.or_gate_softmax(ptr(xf), 1, d, ptr(gw), None, E, k, ptr(idx), ptr(w), ptr(cnt))
    assert np.array_equal(info1["counts"], cnt)
    ref = _oracle_layer(xb[:d], wib, wob, 1, d, f, E, k, idx, w)
    err = np.abs(y1.float().cpu().numpy() - ref)
    assert np.all(err <= ATOL + RTOL * np.abs(ref)), err.max()
    layer.close()


def test_layer_error_paths(cuda):
    """Misuse is reported through the status codes (Python exceptions here),
    never a crash: too many tokens, device weights for an offloaded layer,
    K < 1, an unknown EP transport, N = 0 with NULL buffers allowed."""
    d, f, E = 128, 256, 4
    wi = torch.zeros(E, f, d, dtype=torch.bfloat16, device=cuda)
    wo = torch.zeros(E, d, f, dtype=torch.bfloat16, device=cuda)
    lay = dv.MoELayer(d, f, E, 1, wi, wo, gate="lsh", lsh_bits=2, max_tokens=8)
    with pytest.raises(ValueError):
        lay.forward(torch.zeros(9, d, dtype=torch.bfloat16, device=cuda))  # > max_tokens
    lay.close()
    with pytest.raises(ValueError):  # offloaded weights must be host memory
        dv.MoELayer(d, f, E, 1, wi, wo, gate="lsh", lsh_bits=2, offloaded=True, K=2)
    with pytest.raises(ValueError):
        dv.MoELayer(d, f, E, 1, wi.cpu().pin_memory(), wo.cpu().pin_memory(), gate="lsh",
                    lsh_bits=2, offloaded=True, K=0)
    comm = im.ep_comm_init(im.ep_unique_id(), 1, 0)
    try:
        lay = dv.MoELayer(d, f, E, 1, wi, wo, gate="lsh", lsh_bits=2, ep_size=1, ep_rank=0,
                          ep_comm=comm)
        lay.desc.ep_transport = 7  # the struct is copied at create: rebuild through the C-ABI
        h = C.c_void_p()
        assert im._lib.infmoe_layer_create(C.byref(lay.desc), C.byref(h)) == 6
        assert b"ep_transport" in im._lib.infmoe_last_error()
        lay.close()
    finally:
        im.ep_comm_destroy(comm)


@pytest.mark.parametrize("gate,k,offloaded", [("lsh", 1, False), ("softmax", 2, True)])
def test_forward_routing_outputs(cuda, gate, k, offloaded):
    """infmoe_forward_out's per-token routing (topk_idx, topk_w, perm, offsets;
    device pointers filled in stream order) equals the standalone gate and
    dispatch kernels on the same input."""
    N, d, f, E = 300, 256, 384, 8
    (_, _, _), (x, wi, wo) = _setup(cuda, N, d, f, E, seed=71)
    gw = (np.random.default_rng(3).standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
    w_in, w_out = (wi.pin_memory(), wo.pin_memory()) if offloaded else (wi.to(cuda), wo.to(cuda))
    lay = dv.MoELayer(d, f, E, k, w_in, w_out, gate=gate, gate_weight=gw, lsh_seed=9,
                      lsh_bits=3, max_tokens=N, offloaded=offloaded, K=2)
    _, info = lay.forward(x, want_routing=True)
    if gate == "lsh":
        proj = torch.from_numpy(im.gating_projection(9, 3, d)).to(cuda)
        _, idx, w, cnt = dv.gate_lsh(x, proj, E)
    else:
        idx, w, cnt = dv.gate_softmax_topk(x, torch.from_numpy(gw).to(cuda), k)
    offs, perm, _ = dv.dispatch(idx, E)
    torch.cuda.synchronize()
    assert torch.equal(info["topk_idx"].view(-1), idx.view(-1))
    assert torch.equal(info["topk_w"].view(-1), w.view(-1))
    assert torch.equal(info["perm"], perm.view(-1))
    assert torch.equal(info["offsets"], offs.view(-1))
    assert np.array_equal(info["counts"], cnt.cpu().numpy())
    lay.close()


def test_layer_fuzz_vs_oracle(cuda):
    """30 random small layers (d, f, E, top-k, gate, token count, residency, K,
    host-link codec): counts equal the oracle gate's, the output is within the
    bf16 tolerance of the fp64 oracle chain, and an offloaded layer equals the
    resident one bit for bit."""
    rng = np.random.default_rng(20261019)
    for case in range(30):
        d = int(rng.choice([128, 256, 384, 512]))
        f = int(rng.choice([256, 384, 512, 768]))
        E = int(rng.integers(2, 17))
        gate = str(rng.choice(["lsh", "softmax"]))
        k = 1 if gate == "lsh" else int(rng.integers(1, min(4, E) + 1))
        bits = max(1, int(np.ceil(np.log2(E))))
        N = int(rng.integers(1, 401))
        seed = 1000 + case
        (xb, wib, wob), (x, wi, wo) = _setup(cuda, N, d, f, E, seed=seed)
        gw = (rng.standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
        kw = dict(gate=gate, gate_weight=gw, lsh_seed=seed, lsh_bits=bits, max_tokens=N)
        res = dv.MoELayer(d, f, E, k, wi.to(cuda), wo.to(cuda), **kw)
        y, info = res.forward(x)
        K = int(rng.integers(1, E + 1))
        codec = str(rng.choice(["raw", "exph"]))
        off = dv.MoELayer(d, f, E, k, wi.pin_memory(), wo.pin_memory(), offloaded=True, K=K,
                          h2d_codec=codec, **kw)
        y_off, _ = off.forward(x)
        torch.cuda.synchronize()
        what = (case, d, f, E, k, gate, N, K, codec)
        assert torch.equal(y.view(torch.int16), y_off.view(torch.int16)), what
        xf = bf16_bits_to_f32(xb).reshape(N, d)
        idx = np.zeros((N, k), np.int32)
        w = np.zeros((N, k), np.float32)
        cnt = np.zeros(E, np.int32)
        if gate == "lsh":
            proj = im.gating_projection(seed, bits, d)
            O.or_gate_lsh(ptr(xf), N, d, ptr(np.ascontiguousarray(proj)), bits, E, ptr(idx),
                          ptr(w), ptr(cnt))
        else:
            O.or_gate_softmax(ptr(xf), N, d, ptr(gw), None, E, k, ptr(idx), ptr(w), ptr(cnt))
        assert np.array_equal(info["counts"], cnt), what
        ref = _oracle_layer(xb, wib, wob, N, d, f, E, k, idx, w)
        err = np.abs(y.float().cpu().numpy() - ref)
        assert np.all(err <= ATOL + RTOL * np.abs(ref)), (what, float(err.max()))
        res.close()
        off.close()
