"""The exp4 / exph pack formats round-trip bit for bit through the host
packer and the host reference decoder (CPU; the GPU decoders are checked
against the same inputs in tests/test_gpu_codec.py)."""
import numpy as np
import pytest

import paper_2106_10715_b200 as im


@pytest.mark.parametrize("codec", ["exp4", "exph"])
def test_host_roundtrip_all_patterns_and_weights(codec):
    rng = np.random.default_rng(3)
    a = np.tile(np.arange(1 << 16, dtype=np.uint16), 2)
    rng.shuffle(a)
    out, nb = im.codec_roundtrip_host(a, codec)
    assert np.array_equal(out, a)
    # uniform weights (the bench's distribution): 12 / ~10.3 bits per value
    w = (rng.uniform(-0.027, 0.027, 1 << 21).astype(np.float32).view(np.uint32) >> 16
         ).astype(np.uint16)
    out, nb = im.codec_roundtrip_host(w, codec)
    assert np.array_equal(out, w)
    bits = 8.0 * nb / w.size
    assert (11.9 < bits < 12.1) if codec == "exp4" else (10.0 < bits < 10.6), bits


def test_host_roundtrip_rejects_bad_sizes():
    with pytest.raises(im.InvalidArgument):
        im.codec_roundtrip_host(np.zeros(100, np.uint16), "exph")


def test_exph_length_limit_fibonacci_histogram():
    """Exponent distances with Fibonacci counts (each spread over the four top
    mantissa pairs) give a Huffman tree far deeper than 12 bits; the encoder's
    length-limited code (package-merge) must stay prefix-free and complete, so
    the round trip is exact."""
    rng = np.random.default_rng(5)
    fib = [1, 1]
    while len(fib) < 31:
        fib.append(fib[-1] + fib[-2])
    deltas = np.concatenate([np.full(c, i) for i, c in enumerate(fib[::-1][:26])])
    rng.shuffle(deltas)
    n = (deltas.size // 256) * 256
    exps = (200 - deltas[:n]).astype(np.uint16)
    a = (exps << 7) | rng.integers(0, 128, n, dtype=np.uint16) | \
        (rng.integers(0, 2, n, dtype=np.uint16) << 15)
    out, nb = im.codec_roundtrip_host(a, "exph")
    assert np.array_equal(out, a)


def test_exph_gaussian_weights_bits():
    """SURVEY 8(d) weights (GaussianStream x d^-1/2, bf16): the (dist, m2) code
    with package-merge lengths takes 10.61 bits per value (the exponent-only
    code: 10.67; i.i.d. entropy of the bf16 values: 10.46)."""
    n = 10240 * 4096  # one expert matrix (the per-matrix tables amortised as in use)
    w = im.gaussian_bf16(im.derive_seed(20261018, 1000), n, 4096 ** -0.5)
    out, nb = im.codec_roundtrip_host(w, "exph")
    assert np.array_equal(out, w)
    bits = 8.0 * nb / n
    assert 10.5 < bits < 10.62, bits
