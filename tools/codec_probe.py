"""Dev probe: pack one expert matrix (d_ff x d_model = 10240 x 4096 bf16, the
bench's weight distribution: GaussianStream x d^-1/2) with exp4
and exph, decode on the GPU through the round-trip hook, and print sizes; run under ncu for the decode kernels' times."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402

n = 10240 * 4096
bits = im.gaussian_bf16(im.derive_seed(int(sys.argv[1]) if len(sys.argv) > 1 else 20261018, 1000),
                        n, 4096 ** -0.5)
out = {}
for codec in ("exp4", "exph"):
    dec, nbytes = dv.codec_roundtrip(bits, codec)
    assert np.array_equal(dec, bits), codec
    out[codec] = {"pack_bytes": nbytes, "bits_per_value": 8.0 * nbytes / n}
print(json.dumps(out))
