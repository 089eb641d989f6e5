"""continuous_load_stream in the executor (simulator.hpp:99-101, :131-133):
once a layer's last load is issued, the load lane flows into the next layer's
predicted first experts (prefetched into that layer's own slot set), and the
next forward reuses the positions that match its real InfMoE order.  Outputs
are bit-identical to the drain mode whether the prediction hits or misses;
with a repeated batch every layer's prediction hits; every measured timeline
passes replay_check's rules per layer with <= K residents."""
import numpy as np
import pytest
import torch

import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
from oracle_lib import fill_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("codec,depth", [("raw", 1), ("exph", 2)])
def test_continuous_stack_bit_identical_and_prefetch_hits(cuda, codec, depth):
    N, d, f, E, K, L = 512, 256, 512, 8, 2, 4
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    sets = [(t(fill_bf16(100 + 2 * s, E * f * d, 1.7320508 / 16), (E, f, d)).pin_memory(),
             t(fill_bf16(101 + 2 * s, E * d * f, 0.03), (E, d, f)).pin_memory())
            for s in range(2)]
    x1 = t(fill_bf16(7, N * d, 1.7320508), (N, d)).to(cuda)
    x2 = t(fill_bf16(8, N * d, 1.7320508), (N, d)).to(cuda)
    pool1, pool2 = dv.SlotPool(K, d, f), dv.SlotPool(K, d, f, sets=2)
    kw = dict(gate="lsh", lsh_bits=3, max_tokens=N, offloaded=True, K=K, h2d_codec=codec)
    drain = [dv.MoELayer(d, f, E, 1, *sets[l % 2], lsh_seed=40 + l, slot_pool=pool1, **kw)
             for l in range(L)]
    cont = [dv.MoELayer(d, f, E, 1, *sets[l % 2], lsh_seed=40 + l, slot_pool=pool2,
                        continuous_load_stream=True, prefetch_depth=depth, **kw)
            for l in range(L)]
    for l in range(L):
        cont[l].set_next(cont[(l + 1) % L])  # an even cycle: alternate slot sets

    def run(stack, x, timeline=False):
        cur, infos = x, []
        for lay in stack:
            cur, info = lay.forward(cur, want_timeline=timeline)
            infos.append(info)
        return cur, infos

    hw = im.Hardware(1643.6e12, 55.5e9, 180 << 30, 8 << 30)
    g = im.make_geometry(d, f, E, 2)
    for p, x in enumerate([x1, x1, x1, x2, x2]):
        y_d, _ = run(drain, x)
        y_c, infos = run(cont, x, timeline=True)
        torch.cuda.synchronize()
        assert torch.equal(y_d.view(torch.int16), y_c.view(torch.int16)), p
        if p in (2, 4):  # the same batch again: every layer's prediction hits
            assert all(i["prefetched"] == depth for i in infos), [i["prefetched"] for i in infos]
        for info in infos:
            cv = im.compute_costs(info["counts"].astype(np.uint64), g, hw)
            assert im.replay_check(info["events"], [cv], K, check_durations=False,
                                   tol_s=2e-6) == {}
    with pytest.raises(im.InvalidArgument):  # continuous on a one-set pool
        dv.MoELayer(d, f, E, 1, *sets[0], lsh_seed=1, slot_pool=pool1,
                    continuous_load_stream=True, **kw)
    odd = cont[:3]
    with pytest.raises(im.InvalidArgument):  # odd cycle on one pool: sets would collide
        odd[2].set_next(odd[0])
    for lay in drain + cont:
        lay.close()
    pool1.close()
    pool2.close()


def test_continuous_links_survive_destroy(cuda):
    """Destroying a layer unlinks it from the layer that would prefetch into it."""
    N, d, f, E, K = 128, 256, 512, 4, 1
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    wi = t(fill_bf16(1, E * f * d, 0.1), (E, f, d)).pin_memory()
    wo = t(fill_bf16(2, E * d * f, 0.03), (E, d, f)).pin_memory()
    x = t(fill_bf16(3, N * d, 1.0), (N, d)).to(cuda)
    kw = dict(gate="lsh", lsh_bits=2, max_tokens=N, offloaded=True, K=K,
              continuous_load_stream=True)
    a = dv.MoELayer(d, f, E, 1, wi, wo, lsh_seed=1, **kw)
    b = dv.MoELayer(d, f, E, 1, wi, wo, lsh_seed=2, **kw)
    a.set_next(b)
    a.forward(x)
    b.forward(x)
    b.close()            # a's link to b must go with it
    y, info = a.forward(x)   # would prefetch into freed memory if still linked
    torch.cuda.synchronize()
    a.close()
