"""exp4 lossless host-link codec (codec.cuh): packs decode bit for bit on the
GPU for every bf16 pattern (zeros, subnormals, Inf, NaN, wide exponent
ranges), and an offloaded layer streaming exp4 packs gives exactly the raw
layer's output with ~25% fewer bytes per load."""
import numpy as np
import pytest
import torch

import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
from oracle_lib import fill_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("codec", ["exp4", "exph"])
@pytest.mark.parametrize("case", ["all_patterns", "weights", "zeros", "wide", "tail_block",
                                  "one_symbol", "long_codes"])
def test_roundtrip_bit_exact(cuda, case, codec):
    rng = np.random.default_rng(1)
    if case == "all_patterns":
        a = np.tile(np.arange(1 << 16, dtype=np.uint16), 3)
        rng.shuffle(a)
    elif case == "weights":
        a = fill_bf16(5, 1 << 20, 1.7320508 / 64)
    elif case == "zeros":
        a = np.zeros(4096, np.uint16)
        a[::7] = 0x8000  # -0.0
    elif case == "wide":  # exponents spread over the whole range: mostly escapes
        a = rng.integers(0, 1 << 16, size=200_000, dtype=np.uint16)
    elif case == "tail_block":  # a last block shorter than 32768 values
        a = fill_bf16(9, 32768 * 3 + 128, 2.0)
    elif case == "one_symbol":  # one exponent everywhere: a 1-bit code
        a = (np.full(8192, 0x3F80, np.uint16) | rng.integers(0, 128, 8192, dtype=np.uint16))
    else:  # a skewed exponent histogram: Huffman lengths hit the 12-bit limit
        e = np.minimum(rng.geometric(0.75, size=300_000) - 1, 40)
        a = (((127 - e) & 0xFF) << 7).astype(np.uint16) | rng.integers(0, 128, 300_000,
                                                                        dtype=np.uint16)
    n = (a.size // 256) * 256
    a = np.ascontiguousarray(a[:n])
    out, nbytes = dv.codec_roundtrip(a, codec)
    assert np.array_equal(out, a)
    if case == "weights":  # exp4: 12 bits per value; exph: ~10.3 (exponent entropy 2.14)
        assert nbytes < (0.76 if codec == "exp4" else 0.66) * 2 * n


@pytest.mark.parametrize("codec", ["exp4", "exph"])
@pytest.mark.parametrize("gate,k,pins", [("lsh", 1, []), ("softmax", 2, [1])])
def test_codec_layer_bit_identical(cuda, gate, k, pins, codec):
    N, d, f, E, K = 512, 256, 512, 8, 2
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    x = t(fill_bf16(1, N * d, 1.7320508), (N, d)).to(cuda)
    wi = t(fill_bf16(2, E * f * d, 1.7320508 / 16), (E, f, d)).pin_memory()
    wo = t(fill_bf16(3, E * d * f, 1.534 * 1.7320508 / np.sqrt(f)), (E, d, f)).pin_memory()
    wi[2].zero_()  # an all-zero expert matrix: every value escapes
    gw = (np.random.default_rng(4).standard_normal((E, d)) / np.sqrt(d)).astype(np.float32)
    kw = dict(gate=gate, gate_weight=gw, lsh_seed=5, lsh_bits=3, max_tokens=N, offloaded=True,
              K=K)
    raw = dv.MoELayer(d, f, E, k, wi, wo, **kw)
    pool = dv.SlotPool(K, d, f)
    ex1 = dv.MoELayer(d, f, E, k, wi, wo, h2d_codec=codec, slot_pool=pool, **kw)
    ex2 = dv.MoELayer(d, f, E, k, wi, wo, h2d_codec=codec, slot_pool=pool, **kw)  # shared pack
    if pins:
        ex1.pin_experts(pins)
    y0, info0 = raw.forward(x, want_timeline=True)
    y1, info1 = ex1.forward(x, want_timeline=True)
    y2, _ = ex2.forward(y1)
    y2r, _ = raw.forward(y0)
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.int16), y0.view(torch.int16))
    assert torch.equal(y2.view(torch.int16), y2r.view(torch.int16))
    assert list(info1["order"][:E - len(pins)]) == [e for e in info0["order"] if e not in pins]
    assert raw.packed_bytes() == E * 2 * d * f * 2  # raw stream: expert_param_bytes per expert
    assert ex1.packed_bytes() == ex2.packed_bytes() < raw.packed_bytes()
    assert len([ev for ev in info1["events"] if ev[0] == 0]) == E - len(pins)
    for lay in (raw, ex1, ex2):
        lay.close()
    pool.close()


def test_exp4_needs_bf16(cuda):
    N, d, f, E = 64, 256, 512, 4
    wi = torch.zeros((E, f, d), dtype=torch.float32).pin_memory()
    wo = torch.zeros((E, d, f), dtype=torch.float32).pin_memory()
    with pytest.raises(im.InvalidArgument):
        dv.MoELayer(d, f, E, 1, wi, wo, dtype="f32", offloaded=True, K=1, lsh_bits=2,
                    max_tokens=N, h2d_codec="exp4")


def test_codec_packs_are_snapshots_that_follow_set_host_weights(cuda):
    """exph packs are snapshots of the host weights (include/infmoe.h): after
    the host buffers are refilled IN PLACE, a new codec layer created on them
    while an old one is alive re-packs (content digest mismatch) and matches the
    raw stream, the old layer keeps its snapshot until set_host_weights, which
    always re-packs -- after which it matches the raw stream again."""
    N, d, f, E, K = 256, 256, 512, 4, 1
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    x = t(fill_bf16(31, N * d, 1.7320508), (N, d)).to(cuda)
    wi = t(fill_bf16(32, E * f * d, 1.7320508 / 16), (E, f, d)).pin_memory()
    wo = t(fill_bf16(33, E * d * f, 1.534 * 1.7320508 / np.sqrt(f)), (E, d, f)).pin_memory()
    kw = dict(gate="lsh", lsh_seed=7, lsh_bits=2, max_tokens=N, offloaded=True, K=K)
    raw = dv.MoELayer(d, f, E, 1, wi, wo, **kw)
    old = dv.MoELayer(d, f, E, 1, wi, wo, h2d_codec="exph", **kw)
    y_raw0, _ = raw.forward(x)
    y_old0, _ = old.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y_old0.view(torch.int16), y_raw0.view(torch.int16))
    # refill the host weights in place (same pointers)
    wi.copy_(t(fill_bf16(34, E * f * d, 1.7320508 / 16), (E, f, d)))
    wo.copy_(t(fill_bf16(35, E * d * f, 1.534 * 1.7320508 / np.sqrt(f)), (E, d, f)))
    new = dv.MoELayer(d, f, E, 1, wi, wo, h2d_codec="exph", **kw)  # old is alive: cache hit?
    y_raw1, _ = raw.forward(x)   # the raw stream reads the host buffers live
    y_new1, _ = new.forward(x)
    y_old1, _ = old.forward(x)   # still the snapshot taken at create
    torch.cuda.synchronize()
    assert not torch.equal(y_raw1.view(torch.int16), y_raw0.view(torch.int16))
    assert torch.equal(y_new1.view(torch.int16), y_raw1.view(torch.int16))
    assert torch.equal(y_old1.view(torch.int16), y_raw0.view(torch.int16))
    old.set_host_weights(wi, wo)  # re-packs
    y_old2, _ = old.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y_old2.view(torch.int16), y_raw1.view(torch.int16))
    for lay in (raw, old, new):
        lay.close()


def test_codec_layer_from_pageable_weights(cuda):
    """A packed-codec layer streams its pinned packs only, so pageable raw host
    weights stay pageable (not registered); output equals the raw stream."""
    N, d, f, E, K = 256, 256, 512, 4, 1
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    x = t(fill_bf16(41, N * d, 1.7320508), (N, d)).to(cuda)
    wi = t(fill_bf16(42, E * f * d, 1.7320508 / 16), (E, f, d))        # pageable
    wo = t(fill_bf16(43, E * d * f, 1.534 * 1.7320508 / np.sqrt(f)), (E, d, f))
    assert not wi.is_pinned()
    kw = dict(gate="lsh", lsh_seed=3, lsh_bits=2, max_tokens=N, offloaded=True, K=K)
    raw = dv.MoELayer(d, f, E, 1, wi.pin_memory(), wo.pin_memory(), **kw)
    ex = dv.MoELayer(d, f, E, 1, wi, wo, h2d_codec="exph", **kw)
    ex.pin_experts([1])  # the one-time device copy reads the pageable weights
    y0, _ = raw.forward(x)
    y1, _ = ex.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(y0.view(torch.int16), y1.view(torch.int16))
    assert not wi.is_pinned()
    raw.close()
    ex.close()


@pytest.mark.parametrize("codec", ["exp4", "exph"])
def test_pack_cache_dir(cuda, tmp_path, codec):
    """set_pack_cache_dir: the first codec layer encodes and writes one file per
    host-weight content; a later layer on the same content reads it back (no
    encode) with output bit-identical to the raw stream; a damaged file or new
    content is never used -- it is re-encoded (and the file replaced)."""
    N, d, f, E, K = 256, 256, 512, 4, 1
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    x = t(fill_bf16(51, N * d, 1.7320508), (N, d)).to(cuda)
    wi = t(fill_bf16(52, E * f * d, 1.7320508 / 16), (E, f, d)).pin_memory()
    wo = t(fill_bf16(53, E * d * f, 1.534 * 1.7320508 / np.sqrt(f)), (E, d, f)).pin_memory()
    kw = dict(gate="lsh", lsh_seed=5, lsh_bits=2, max_tokens=N, offloaded=True, K=K)
    raw = dv.MoELayer(d, f, E, 1, wi, wo, **kw)
    y_raw, _ = raw.forward(x)
    im.set_pack_cache_dir(tmp_path)
    try:
        a = dv.MoELayer(d, f, E, 1, wi, wo, h2d_codec=codec, **kw)
        assert a.pack_source() == "encoded"
        files = sorted(tmp_path.glob("*.infmoe-pack"))
        assert len(files) == 1 and not list(tmp_path.glob("*.tmp.*"))
        a.close()
        b = dv.MoELayer(d, f, E, 1, wi, wo, h2d_codec=codec, **kw)
        assert b.pack_source() == "cache"
        y_b, _ = b.forward(x)
        torch.cuda.synchronize()
        assert torch.equal(y_b.view(torch.int16), y_raw.view(torch.int16))
        assert b.packed_bytes() < 2 * E * d * f * 2
        b.close()
        # flip one byte of the pack area: the checksum rejects the file
        blob = bytearray(files[0].read_bytes())
        blob[-100] ^= 0x5A
        files[0].write_bytes(bytes(blob))
        c = dv.MoELayer(d, f, E, 1, wi, wo, h2d_codec=codec, **kw)
        assert c.pack_source() == "encoded"
        y_c, _ = c.forward(x)
        torch.cuda.synchronize()
        assert torch.equal(y_c.view(torch.int16), y_raw.view(torch.int16))
        c.close()
        assert files[0].read_bytes() != bytes(blob)  # replaced by the fresh encode
        # a damaged table (expert 0's size, right after the 72-byte header) too
        blob = bytearray(files[0].read_bytes())
        blob[72 + 8] ^= 0x01
        files[0].write_bytes(bytes(blob))
        c2 = dv.MoELayer(d, f, E, 1, wi, wo, h2d_codec=codec, **kw)
        assert c2.pack_source() == "encoded"
        y_c2, _ = c2.forward(x)
        torch.cuda.synchronize()
        assert torch.equal(y_c2.view(torch.int16), y_raw.view(torch.int16))
        c2.close()
        # new content -> a second file, encoded
        wi.copy_(t(fill_bf16(54, E * f * d, 1.7320508 / 16), (E, f, d)))
        e2 = dv.MoELayer(d, f, E, 1, wi, wo, h2d_codec=codec, **kw)
        assert e2.pack_source() == "encoded"
        assert len(list(tmp_path.glob("*.infmoe-pack"))) == 2
        e2.close()
    finally:
        im.set_pack_cache_dir(None)
    assert raw.pack_source() == "none"
    raw.close()


def _fuzz_case(rng):
    n = 256 * int(rng.integers(1, 2400))
    kind = rng.choice(["gauss", "laplace", "uniform", "outliers", "drift", "special", "runs"])
    sig = float(10.0 ** rng.uniform(-5, 1))
    if kind == "gauss":
        x = rng.normal(0, sig, n)
    elif kind == "laplace":
        x = rng.laplace(0, sig, n)
    elif kind == "uniform":
        x = rng.uniform(-sig, sig, n)
    elif kind == "outliers":
        x = rng.normal(0, sig, n)
        m = rng.random(n) < 0.02
        x[m] *= 10.0 ** rng.uniform(1, 6, m.sum())
    elif kind == "drift":  # magnitude drifting along the matrix: block bases differ
        x = rng.normal(0, 1, n) * np.exp(np.linspace(-12, 12, n))
    elif kind == "special":  # subnormals, zeros, +-inf, NaN sprinkled into normal data
        x = rng.normal(0, sig, n)
        idx = rng.integers(0, n, max(1, n // 50))
        x[idx] = rng.choice([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-39, -3e-40, 1e38], idx.size)
    else:  # long runs of one value
        x = np.repeat(rng.normal(0, sig, n // 256 + 1), 256)[:n]
    u = x.astype(np.float32).view(np.uint32)
    return kind, ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def test_roundtrip_fuzz(cuda):
    """40 random inputs (distribution, scale, size, NaN / Inf / subnormals, drift
    of the block maxima, constant runs): the GPU decoders and the host reference
    decoder restore every bit pattern."""
    rng = np.random.default_rng(20261019)
    for _ in range(40):
        kind, a = _fuzz_case(rng)
        for codec in ("exph", "exp4"):
            out, _ = dv.codec_roundtrip(a, codec)
            assert np.array_equal(out, a), (kind, codec, a.size)
        out, _ = im.codec_roundtrip_host(a, "exph")
        assert np.array_equal(out, a), (kind, "host", a.size)
