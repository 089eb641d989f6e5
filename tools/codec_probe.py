"""Dev probe: pack one expert matrix (d_ff x d_model = 10240 x 4096 bf16, the
bench's weight distribution) with exp4 and exph, decode on the GPU through the
round-trip hook, and print sizes; run under ncu for the decode kernels' times."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2106_10715_b200 import device as dv  # noqa: E402

n = 10240 * 4096
w = torch.empty(n, dtype=torch.bfloat16, device="cuda")
dv.fill_uniform(w, 123, 3 ** 0.5 / 4096 ** 0.5)
bits = w.view(torch.int16).cpu().numpy().view(np.uint16)
out = {}
for codec in ("exp4", "exph"):
    dec, nbytes = dv.codec_roundtrip(bits, codec)
    assert np.array_equal(dec, bits), codec
    out[codec] = {"pack_bytes": nbytes, "bits_per_value": 8.0 * nbytes / n}
print(json.dumps(out))
