"""The host-side gating / workload entry points of the drop-in boundary
(include/infmoe.h: infmoe_lsh_codes, infmoe_route_tokens,
infmoe_explicit_workload, infmoe_workload_from_csv) against the reference
itself (oracle/_ref: the moesim headers compiled in place): bit-exact codes and
counts on fp64 rows (including signed zeros, exact cancellations, NaN and Inf),
identical counts and error class for well-formed and malformed CSV files."""
import ctypes as C

import numpy as np
import pytest

import paper_2106_10715_b200 as im
from oracle_lib import REF, ptr

pytestmark = pytest.mark.skipif(REF is None, reason="reference build (oracle/_ref) not present")

if REF is not None:
    REF.ref_workload_from_csv.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_void_p,
                                          C.c_void_p]
    REF.ref_explicit_workload.argtypes = [C.c_void_p, C.c_int, C.c_void_p]


@pytest.mark.parametrize("n,hidden,bits,E", [(700, 256, 5, 24), (33, 768, 3, 8),
                                             (5000, 64, 6, 64), (1, 4096, 5, 32)])
def test_lsh_codes_and_route_tokens_bit_exact(n, hidden, bits, E):
    seed = im.derive_seed(n, hidden)
    x = im.gaussian_stream(im.derive_seed(seed, 0), n * hidden)
    x[: hidden] = 0.0                       # an all-zero row: every bit set (+0 >= 0)
    if n > 3:
        x[hidden: 2 * hidden] = -0.0
        x[2 * hidden + 5] = np.nan          # NaN row: dot is NaN, bits clear
        x[3 * hidden + 1] = np.inf
    codes = im.lsh_codes(seed, bits, hidden, x)
    ref = np.zeros(n, np.uint32)
    assert REF.ref_lsh_codes(seed, bits, hidden, ptr(x), n, ptr(ref)) == 0
    assert np.array_equal(codes, ref)
    counts = im.route_tokens(seed, bits, hidden, x, E)
    rc = np.zeros(E, np.uint64)
    assert REF.ref_route_tokens(seed, bits, hidden, ptr(x), n, E, ptr(rc)) == 0
    assert np.array_equal(counts, rc)


def test_gating_errors_match_reference():
    x = np.zeros(64, np.float64)
    with pytest.raises(im.ConfigError):
        im.route_tokens(1, 3, 8, x, 9)      # 2^3 < 9 experts
    with pytest.raises(im.InvalidArgument):
        im.route_tokens(1, 3, 8, x, 0)
    with pytest.raises(im.ConfigError):
        im.lsh_codes(1, 32, 8, x)
    with pytest.raises(im.InvalidArgument):
        im.lsh_codes(1, 3, 7, x)            # 64 values are not whole rows of 7


CSV_CASES = {
    "header_crlf_gaps": "expert_id,token_count\r\n3,10\n\n0,4\n1,2,9\n",
    "no_header": "0,5\n2,7\n1,0\n",
    "spaces": " 1, 3\n0 ,2\n",
    "duplicate": "0,1\n0,2\n",
    "missing_count": "0,\n",
    "no_comma": "5\n",
    "bad_number": "x,1\n1,y\n",
    "header_only": "expert,count\n",
    "empty": "",
    "leading_comma": ",7\n",
    "header_not_first": "0,1\nid,count\n",
    "big_id": "7,1\n",
}


@pytest.mark.parametrize("name", sorted(CSV_CASES))
def test_workload_from_csv_matches_reference(tmp_path, name):
    path = tmp_path / f"{name}.csv"
    path.write_bytes(CSV_CASES[name].encode())
    n = C.c_int(0)
    total = C.c_uint64(0)
    buf = np.zeros(64, np.uint64)
    rc = REF.ref_workload_from_csv(str(path).encode(), ptr(buf), 64, C.byref(n), C.byref(total))
    if rc == 0:
        counts, tot = im.workload_from_csv(path)
        assert np.array_equal(counts, buf[: n.value]) and tot == total.value
    else:
        assert rc == 2
        with pytest.raises(im.ConfigError):
            im.workload_from_csv(path)


def test_explicit_workload_matches_reference():
    for counts in ([5, 0, 7], [0], [2 ** 40, 3]):
        c = np.asarray(counts, np.uint64)
        t = C.c_uint64(0)
        assert REF.ref_explicit_workload(ptr(c), c.size, C.byref(t)) == 0
        got, tot = im.explicit_workload(counts)
        assert np.array_equal(got, c) and tot == t.value
    t = C.c_uint64(0)
    assert REF.ref_explicit_workload(None, 0, C.byref(t)) == 2
    with pytest.raises(im.ConfigError):
        im.explicit_workload([])
