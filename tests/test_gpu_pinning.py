"""Hot-expert pinning (not in the reference, whose eviction is
immediate): pinned experts are computed from device copies with
no load, the rest stream in the InfMoE order over their own costs, and the
layer output is bit-identical to the unpinned / resident layer."""
import numpy as np
import pytest
import torch

import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
from oracle_lib import fill_bf16, schedule

pytestmark = pytest.mark.gpu


def _weights(N, d, f, E, seed):
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    xb = fill_bf16(im.derive_seed(seed, 0), N * d, 1.7320508)
    wib = fill_bf16(im.derive_seed(seed, 1), E * f * d, 1.7320508 / np.sqrt(d))
    wob = fill_bf16(im.derive_seed(seed, 2), E * d * f, 1.5340 * 1.7320508 / np.sqrt(f))
    return t(xb, (N, d)), t(wib, (E, f, d)).pin_memory(), t(wob, (E, d, f)).pin_memory()


def _bits(y):
    return y.view(torch.int16).cpu()


@pytest.mark.parametrize("gate,k,skip", [("lsh", 1, False), ("softmax", 2, False),
                                         ("softmax", 2, True)])
def test_pinned_layer_bit_identical(cuda, gate, k, skip):
    N, d, f, E, K = 512, 256, 512, 8, 2
    x, wi, wo = _weights(N, d, f, E, 5)
    x = x.to(cuda)
    gw = (np.random.default_rng(1).standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
    bias = (-1.0 * np.log(np.arange(1, E + 1))).astype(np.float32)
    kw = dict(gate=gate, gate_weight=gw, gate_bias=bias, lsh_seed=9, lsh_bits=3, max_tokens=N,
              skip_empty_experts=skip)
    res = dv.MoELayer(d, f, E, k, wi.to(cuda), wo.to(cuda), **kw)
    off = dv.MoELayer(d, f, E, k, wi, wo, offloaded=True, K=K, **kw)
    y_res, _ = res.forward(x)
    y0, info0 = off.forward(x, want_timeline=True)
    counts = info0["counts"]
    hot = [int(e) for e in np.argsort(-counts, kind="stable")[:3]]
    for pins in (hot, list(range(E)), [E - 1], []):
        off.pin_experts(pins)
        y, info = off.forward(x, want_timeline=True)
        torch.cuda.synchronize()
        assert torch.equal(_bits(y), _bits(y_res)), pins
        loads = [ev for ev in info["events"] if ev[0] == 0]
        comps = [ev for ev in info["events"] if ev[0] == 1]
        streamed = [e for e in range(E) if e not in pins and (not skip or counts[e] > 0)]
        assert sorted(ev[2] for ev in loads) == streamed
        assert not any(ev[2] in pins for ev in loads)
        # pinned experts with rows appear as compute-only events
        assert sorted(ev[2] for ev in comps if ev[2] in pins) == \
            sorted(e for e in pins if counts[e] > 0)
        # the streamed experts follow the InfMoE order over their own costs
        if streamed:
            g = im.make_geometry(d, f, len(streamed), 2)
            cv = im.compute_costs(counts[streamed].astype(np.uint64), g,
                                  im.Hardware(1643.6e12, 55.5e9, 180 << 30, 8 << 30))
            want = [streamed[i] for i in schedule("or", cv.alphas, cv.beta, K, "auto")[1]]
            assert list(info["order"][:len(streamed)]) == want
        assert all(o == -1 for o in info["order"][len(streamed):])
    res.close()
    off.close()


def test_pinned_follow_new_host_weights(cuda):
    N, d, f, E = 256, 256, 512, 4
    x, wi, wo = _weights(N, d, f, E, 6)
    _, wi2, wo2 = _weights(N, d, f, E, 7)
    x = x.to(cuda)
    off = dv.MoELayer(d, f, E, 1, wi, wo, offloaded=True, K=1, lsh_seed=3, lsh_bits=2,
                      max_tokens=N)
    off.pin_experts([0, 2])
    off.set_host_weights(wi2, wo2)
    y, _ = off.forward(x)
    ref = dv.MoELayer(d, f, E, 1, wi2.to(cuda), wo2.to(cuda), lsh_seed=3, lsh_bits=2,
                      max_tokens=N)
    y_ref, _ = ref.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(_bits(y), _bits(y_ref))
    off.close()
    ref.close()


def test_pin_errors(cuda):
    N, d, f, E = 64, 256, 512, 4
    x, wi, wo = _weights(N, d, f, E, 8)
    res = dv.MoELayer(d, f, E, 1, wi.to(cuda), wo.to(cuda), lsh_bits=2, max_tokens=N)
    with pytest.raises(im.InvalidArgument):
        res.pin_experts([0])
    off = dv.MoELayer(d, f, E, 1, wi, wo, offloaded=True, K=1, lsh_bits=2, max_tokens=N)
    for bad in ([E], [-1], [1, 1], list(range(E + 1))):
        with pytest.raises(im.InvalidArgument):
            off.pin_experts(bad)
    off.pin_experts([1])
    off.pin_experts([])  # unpin
    y, info = off.forward(x.to(cuda), want_timeline=True)
    assert len([ev for ev in info["events"] if ev[0] == 0]) == E
    res.close()
    off.close()


def test_pin_hottest_cache_policy(cuda):
    """pin_hottest picks the top-n experts by the EMA (decay 0.5) of routed rows
    over the layer's offloaded forwards; re-pinning re-uses device copies; the
    output stays bit-identical throughout."""
    N, d, f, E, k = 512, 256, 512, 8, 2
    x, wi, wo = _weights(N, d, f, E, 12)
    x = x.to(cuda)
    gw = (np.random.default_rng(3).standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
    bias = (-0.7 * np.log(np.arange(1, E + 1))).astype(np.float32)
    kw = dict(gate="softmax", gate_weight=gw, gate_bias=bias, max_tokens=N)
    res = dv.MoELayer(d, f, E, k, wi.to(cuda), wo.to(cuda), **kw)
    off = dv.MoELayer(d, f, E, k, wi, wo, offloaded=True, K=2, **kw)
    ema = None
    for xb in (x, -x, x.roll(1, dims=1)):  # three batches, three routings
        _, info = off.forward(xb.contiguous())
        c = info["counts"].astype(np.float64)
        ema = c if ema is None else 0.5 * ema + 0.5 * c
    want = sorted(int(e) for e in np.argsort(-ema, kind="stable")[:3])
    assert off.pin_hottest(3) == want
    y_res, _ = res.forward(x)
    y, info = off.forward(x, want_timeline=True)
    torch.cuda.synchronize()
    assert torch.equal(_bits(y), _bits(y_res))
    assert not any(ev[2] in want for ev in info["events"] if ev[0] == 0)
    got5 = off.pin_hottest(5)  # grows the pinned set, re-using the kept device copies
    assert len(got5) == 5 and len(set(got5)) == 5
    y, _ = off.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(_bits(y), _bits(y_res))
    assert off.pin_hottest(0) == []
    res.close()
    off.close()
