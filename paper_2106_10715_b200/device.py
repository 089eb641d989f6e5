"""Device-path wrappers: call the C-ABI kernels on torch-allocated device memory.

torch is plumbing here (allocation, streams); every computation runs in
libinfmoe.so.  Functions take/return torch tensors and launch on the current
torch CUDA stream.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import (DTYPE_BF16, DTYPE_F32, GATE_LSH, GATE_SOFTMAX, OFFLOADED, POLICY_AUTO, RESIDENT,
               Event, ForwardOut, Hardware, LayerDesc, _check, _lib)


def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    if t.dtype == torch.float32:
        return DTYPE_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream_ptr():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("device-path call needs CUDA tensors")


def fill_uniform(t, seed: int, scale: float) -> None:
    """Counter-hash uniform fill (same bits as oracle or_fill_uniform_*)."""
    _need_cuda(t)
    _check(_lib.infmoe_fill_uniform(_p(t), _dtype_code(t), t.numel(), seed, scale,
                                    _stream_ptr()))


def occupy_sms(n_ctas: int, release, timed_out, smem_bytes: int = 200 * 1024,
               timeout_s: float = 20.0, stream=None) -> None:
    """Test hook: n_ctas spinning CTAs (one per SM at ~200 KB of shared memory)
    until release[0] != 0 or the timeout; timed_out[0] = 1 if any gave up."""
    torch = _torch()
    _need_cuda(release, timed_out)
    s = C.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    _check(_lib.infmoe_debug_occupy_sms(n_ctas, smem_bytes, _p(release), int(timeout_s * 1e9),
                                        _p(timed_out), s))


def set_flag(flag, stream=None) -> None:
    torch = _torch()
    _need_cuda(flag)
    s = C.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    _check(_lib.infmoe_debug_set_flag(_p(flag), s))


class GateWorkspace:
    """Device workspace of the softmax gate for fixed gate weights wg [E, d]
    (infmoe_gate_softmax_ws_bytes / _prepare): W_g's bf16 split is made once;
    None-sized (nbytes == 0) when the calls take the CUDA-core path."""

    def __init__(self, wg, max_tokens: int, k: int, dtype=None):
        torch = _torch()
        _need_cuda(wg)
        E, d = wg.shape
        code = _dtype_code(torch.empty(0, dtype=dtype or torch.bfloat16))
        self.nbytes = int(_lib.infmoe_gate_softmax_ws_bytes(code, max_tokens, d, E, k))
        self.buf = torch.empty(max(self.nbytes, 1), dtype=torch.uint8, device=wg.device)
        self.wg = wg
        if self.nbytes:
            _check(_lib.infmoe_gate_softmax_prepare(_p(wg), d, E, _p(self.buf), self.nbytes,
                                                    _stream_ptr()))


def gate_softmax_topk(x, wg, k: int, bias=None, debug: bool = False, workspace=None):
    """N1a gate.  debug=True also returns the tensor-core path's approximate
    logits [N, E] and its counters {certified, fallback, candidates, full_exact}
    (None on the CUDA-core path)."""
    torch = _torch()
    _need_cuda(x, wg, bias)
    N, d = x.shape
    E = wg.shape[0]
    idx = torch.empty((N, k), dtype=torch.int32, device=x.device)
    w = torch.empty((N, k), dtype=torch.float32, device=x.device)
    counts = torch.empty(E, dtype=torch.int32, device=x.device)
    if workspace is not None and not debug:
        _check(_lib.infmoe_gate_softmax_topk_ws(_p(x), _dtype_code(x), N, d, _p(wg), _p(bias),
                                                E, k, _p(idx), _p(w), _p(counts),
                                                _p(workspace.buf), workspace.nbytes,
                                                _stream_ptr()))
        return idx, w, counts
    if not debug:
        _check(_lib.infmoe_gate_softmax_topk(_p(x), _dtype_code(x), N, d, _p(wg), _p(bias), E,
                                             k, _p(idx), _p(w), _p(counts), _stream_ptr()))
        return idx, w, counts
    approx = torch.empty((N, E), dtype=torch.float32, device=x.device)
    stats = torch.zeros(4, dtype=torch.int64, device=x.device)
    _check(_lib.infmoe_gate_softmax_debug(_p(x), _dtype_code(x), N, d, _p(wg), _p(bias), E, k,
                                          _p(idx), _p(w), _p(counts), _p(approx), _p(stats),
                                          _stream_ptr()))
    st = stats.cpu().tolist()
    if st[0] == -1:
        return idx, w, counts, None, None
    return idx, w, counts, approx, {"certified": st[0], "fallback": st[1],
                                    "candidates": st[2], "full_exact": st[3]}


def gate_lsh(x, proj, n_experts: int):
    torch = _torch()
    _need_cuda(x, proj)
    N, d = x.shape
    bits = proj.shape[0]
    codes = torch.empty(N, dtype=torch.int32, device=x.device)
    idx = torch.empty((N, 1), dtype=torch.int32, device=x.device)
    w = torch.empty((N, 1), dtype=torch.float32, device=x.device)
    counts = torch.empty(n_experts, dtype=torch.int32, device=x.device)
    _check(_lib.infmoe_gate_lsh(_p(x), _dtype_code(x), N, d, _p(proj), bits, n_experts,
                                _p(codes), _p(idx), _p(w), _p(counts), _stream_ptr()))
    return codes, idx, w, counts


def dispatch(topk_idx, n_experts: int):
    torch = _torch()
    _need_cuda(topk_idx)
    N, k = topk_idx.shape
    A = N * k
    offsets = torch.empty(n_experts + 1, dtype=torch.int32, device=topk_idx.device)
    perm = torch.empty(max(A, 1), dtype=torch.int32, device=topk_idx.device)
    inv = torch.empty(max(A, 1), dtype=torch.int32, device=topk_idx.device)
    ws = torch.empty(int(_lib.infmoe_dispatch_workspace_bytes(A, n_experts)), dtype=torch.uint8,
                     device=topk_idx.device)
    _check(_lib.infmoe_dispatch(_p(topk_idx), N, k, n_experts, _p(offsets), _p(perm), _p(inv),
                                _p(ws), _stream_ptr()))
    return offsets, perm[:A], inv[:A]


def gather_rows(x, perm, k: int):
    torch = _torch()
    N, d = x.shape
    xp = torch.empty((N * k, d), dtype=x.dtype, device=x.device)
    _check(_lib.infmoe_gather_rows(_p(x), _dtype_code(x), N, d, k, _p(perm), _p(xp),
                                   _stream_ptr()))
    return xp


def gather_rows_by_token(x, inv, k: int):
    """x_perm[inv[t*k+j]] = x[t]: gather_rows' output, each token row read once."""
    torch = _torch()
    N, d = x.shape
    xp = torch.empty((N * k, d), dtype=x.dtype, device=x.device)
    _check(_lib.infmoe_gather_rows_by_token(_p(x), _dtype_code(x), N, d, k, _p(inv), _p(xp),
                                            _stream_ptr()))
    return xp


def expert_ffn(x_perm, offsets, w_in, w_out, experts: Optional[Sequence[int]] = None,
               slots: Optional[Sequence[int]] = None, h=None, y_perm=None):
    """h = GeLU(x_perm . w_in[slot]^T), y = h . w_out[slot]^T per expert segment.

    w_in: [n_slots, d_ff, d_model], w_out: [n_slots, d_model, d_ff]."""
    torch = _torch()
    _need_cuda(x_perm, offsets, w_in, w_out)
    R, d = x_perm.shape
    n_slots, f, _ = w_in.shape
    E = offsets.numel() - 1
    if h is None:
        h = torch.empty((R, f), dtype=x_perm.dtype, device=x_perm.device)
    if y_perm is None:
        y_perm = torch.empty((R, d), dtype=x_perm.dtype, device=x_perm.device)
    if experts is None:
        ex = sl = None
        n = E
    else:
        ex = np.ascontiguousarray(np.asarray(experts, dtype=np.int32))
        sl = np.ascontiguousarray(np.asarray(slots if slots is not None else experts,
                                             dtype=np.int32))
        n = len(ex)
    _check(_lib.infmoe_expert_ffn(_p(x_perm), R, d, f, _dtype_code(x_perm), _p(offsets), E,
                                  _p(w_in), _p(w_out), n_slots,
                                  None if ex is None else ex.ctypes.data_as(C.c_void_p),
                                  None if sl is None else sl.ctypes.data_as(C.c_void_p), n,
                                  _p(h), _p(y_perm), _stream_ptr()))
    return h, y_perm


def expert_ffn_fused(x_perm, offsets, w_in, w_out, experts=None, slots=None, perm=None,
                     topk_w=None, n_tokens: Optional[int] = None):
    """Both projections in one persistent launch.  With perm/topk_w (top-1) the
    combine is fused and the result is y [n_tokens, d]; else y_perm [rows, d]."""
    torch = _torch()
    _need_cuda(x_perm, offsets, w_in, w_out)
    R, d = x_perm.shape
    n_slots, f, _ = w_in.shape
    E = offsets.numel() - 1
    h = torch.empty((R, f), dtype=x_perm.dtype, device=x_perm.device)
    rows_out = n_tokens if perm is not None else R
    y = torch.empty((rows_out, d), dtype=x_perm.dtype, device=x_perm.device)
    done = torch.empty(max(E, 1) + 1, dtype=torch.int32, device=x_perm.device)
    if experts is None:
        ex = sl = None
        n = E
    else:
        ex = np.ascontiguousarray(np.asarray(experts, dtype=np.int32))
        sl = np.ascontiguousarray(np.asarray(slots if slots is not None else experts,
                                             dtype=np.int32))
        n = len(ex)
    _check(_lib.infmoe_expert_ffn_fused(
        _p(x_perm), R, d, f, _p(offsets), E, _p(w_in), _p(w_out), n_slots,
        None if ex is None else ex.ctypes.data_as(C.c_void_p),
        None if sl is None else sl.ctypes.data_as(C.c_void_p), n, _p(h), _p(y), _p(perm),
        _p(topk_w), _p(done), _stream_ptr()))
    return h, y


def scatter_rows(src, index, n_out: int, out=None):
    """out[index[p]] = src[p]."""
    torch = _torch()
    R, d = src.shape
    if out is None:
        out = torch.empty((n_out, d), dtype=src.dtype, device=src.device)
    _check(_lib.infmoe_scatter_rows(_p(src), _dtype_code(src), R, d, _p(index), _p(out),
                                    _stream_ptr()))
    return out


def combine(y_perm, inv, topk_w, N: int, k: int):
    torch = _torch()
    d = y_perm.shape[1]
    y = torch.empty((N, d), dtype=y_perm.dtype, device=y_perm.device)
    _check(_lib.infmoe_combine(_p(y_perm), _dtype_code(y_perm), _p(inv), _p(topk_w), N, k, d,
                               _p(y), _stream_ptr()))
    return y


CODECS = {"raw": 0, "exp4": 1, "exph": 2}


def codec_roundtrip(bits: np.ndarray, codec: str = "exp4", device: int = 0):
    """Pack bf16 bit patterns on the host with codec, decode on the GPU:
    (decoded, pack bytes)."""
    a = np.ascontiguousarray(bits, dtype=np.uint16)
    out = np.empty_like(a)
    nb = C.c_uint64(0)
    _check(_lib.infmoe_codec_roundtrip(CODECS[codec], a.ctypes.data_as(C.c_void_p), a.size,
                                       out.ctypes.data_as(C.c_void_p), C.byref(nb), device))
    return out, nb.value


class SlotPool:
    """K+1 device expert slots shared by the offloaded layers of a stack
    (infmoe_slot_pool: K experts resident on the GPU in total + one in flight)."""

    def __init__(self, K: int, d_model: int, d_ff: int, dtype: str = "bf16", device: int = 0,
                 sets: int = 1):
        """sets=2: two slot sets, for stacks of continuous_load_stream layers."""
        esz = 2 if dtype == "bf16" else 4
        self.K = K
        self._h = C.c_void_p()
        _check(_lib.infmoe_slot_pool_create_ex(device, K, d_model * d_ff * esz, sets,
                                               C.byref(self._h)))

    @property
    def handle(self):
        return self._h.value

    def close(self) -> None:
        if self._h:
            _lib.infmoe_slot_pool_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class MoELayer:
    """Owning wrapper of an infmoe_layer handle (the paper's MoE plugin)."""

    def __init__(self, d_model: int, d_ff: int, n_experts: int, top_k: int, w_in, w_out, *,
                 dtype: str = "bf16", gate: str = "lsh", gate_weight=None, gate_bias=None,
                 lsh_seed: int = 0, lsh_bits: int = 5, offloaded: bool = False, K: int = 4,
                 policy: int = POLICY_AUTO, max_tokens: int = 4096, device: int = 0,
                 hw: Optional[Hardware] = None, ep_size: int = 1, ep_rank: int = 0,
                 ep_comm: Optional[int] = None, skip_empty_experts: bool = False,
                 slot_pool: Optional["SlotPool"] = None, ep_transport: str = "nccl",
                 h2d_codec: str = "raw", continuous_load_stream: bool = False,
                 prefetch_depth: int = 0):
        d = LayerDesc()
        d.d_model, d.d_ff, d.n_experts, d.top_k = d_model, d_ff, n_experts, top_k
        d.dtype = DTYPE_BF16 if dtype == "bf16" else DTYPE_F32
        d.gate_kind = GATE_LSH if gate == "lsh" else GATE_SOFTMAX
        d.residency = OFFLOADED if offloaded else RESIDENT
        d.K, d.policy, d.max_tokens, d.device = K, policy, max_tokens, device
        self._keep = []
        if gate_weight is not None:
            gw = np.ascontiguousarray(np.asarray(gate_weight, dtype=np.float32))
            self._keep.append(gw)
            d.gate_weight = gw.ctypes.data
        if gate_bias is not None:
            gb = np.ascontiguousarray(np.asarray(gate_bias, dtype=np.float32))
            self._keep.append(gb)
            d.gate_bias = gb.ctypes.data
        d.lsh_seed, d.lsh_bits = lsh_seed, lsh_bits
        d.w_in, d.w_out = w_in.data_ptr(), w_out.data_ptr()
        self._keep += [w_in, w_out]
        d.hw = hw if hw is not None else Hardware(1643.6e12, 55.5e9, 180 << 30, 8 << 30)
        d.ep_size, d.ep_rank, d.ep_comm = ep_size, ep_rank, ep_comm
        d.skip_empty_experts = int(skip_empty_experts)
        d.ep_transport = {"nccl": 0, "peer": 1}[ep_transport]
        d.h2d_codec = CODECS[h2d_codec]
        d.continuous_load_stream = int(continuous_load_stream)
        d.prefetch_depth = prefetch_depth
        if slot_pool is not None:
            d.slot_pool = slot_pool.handle
            self._keep.append(slot_pool)  # the pool outlives the layer
        self.desc = d
        self.n_experts = n_experts
        self.top_k = top_k
        self.n_local = n_experts // max(ep_size, 1)
        self._h = C.c_void_p()
        _check(_lib.infmoe_layer_create(C.byref(d), C.byref(self._h)))

    def set_next(self, nxt: Optional["MoELayer"]) -> None:
        """continuous_load_stream: the layer forwarded after this one."""
        _check(_lib.infmoe_layer_set_next(self._h, None if nxt is None else nxt._h))

    def set_host_weights(self, w_in, w_out) -> None:
        self._keep += [w_in, w_out]
        _check(_lib.infmoe_layer_set_host_weights(self._h, C.c_void_p(w_in.data_ptr()),
                                                  C.c_void_p(w_out.data_ptr())))

    def pin_experts(self, experts) -> None:
        """Hot-expert pinning (not in the reference): keep these
        local experts on the device across forwards.  [] unpins."""
        ex = np.ascontiguousarray(np.asarray(list(experts), dtype=np.int32))
        _check(_lib.infmoe_layer_pin_experts(self._h, ex.ctypes.data_as(C.c_void_p) if len(ex)
                                             else None, len(ex)))
        self.pinned = [int(e) for e in ex]

    def packed_bytes(self) -> int:
        """Bytes one pass moves over the host link for this layer's experts (its codec)."""
        pk, raw = C.c_uint64(0), C.c_uint64(0)
        _check(_lib.infmoe_layer_h2d_bytes(self._h, C.byref(pk), C.byref(raw)))
        return pk.value

    def pack_source(self) -> str:
        """Where the h2d-codec pack came from: "none" (raw stream), "encoded" or
        "cache" (read from the pack cache directory, set_pack_cache_dir)."""
        v = C.c_int32(0)
        _check(_lib.infmoe_layer_pack_source(self._h, C.byref(v)))
        return {0: "none", 1: "encoded", 2: "cache"}[v.value]

    def pin_hottest(self, n: int) -> list:
        """Cross-batch cache policy: pin the n local experts with the highest
        running load estimate (EMA of routed rows, decay 0.5).  Returns them."""
        out = np.zeros(max(n, 1), dtype=np.int32)
        _check(_lib.infmoe_layer_pin_hottest(self._h, n, out.ctypes.data_as(C.c_void_p)))
        self.pinned = [int(e) for e in out[:n]]
        return self.pinned

    def forward(self, x, y=None, *, want_timeline: bool = False, want_info: bool = True,
                want_routing: bool = False, routing=None, time_origin=None):
        """Run the layer on x [N, d_model] (device).  want_info=False passes no
        output struct: a resident layer then never synchronises with the host
        (and can be captured in a CUDA graph).  want_routing adds the per-token
        routing as device tensors: topk_idx / topk_w [N, k], perm [N*k], offsets [E+1].
        routing=(topk_idx, topk_w) (device int32 / f32 [N, k]) replaces the gate
        (infmoe_layer_forward_routed); time_origin (a torch.cuda.Event recorded
        earlier) puts the measured timeline on that event's time axis."""
        torch = _torch()
        N = x.shape[0]
        if y is None:
            y = torch.empty_like(x)
        def call(out):
            if routing is None:
                return _lib.infmoe_layer_forward(self._h, _p(x), N, _p(y), out, _stream_ptr())
            ti, tw = routing
            _need_cuda(ti, tw)
            return _lib.infmoe_layer_forward_routed(self._h, _p(x), N, _p(ti), _p(tw), _p(y), out,
                                                    _stream_ptr())
        if not want_info and not want_timeline:
            _check(call(None))
            return y, None
        E, El = self.n_experts, self.n_local
        counts = np.zeros(E, dtype=np.int32)
        order = np.zeros(El, dtype=np.int32)
        feas = C.c_int32(0)
        exposed = C.c_double(0.0)
        events = (Event * (2 * El))()
        local_rows = np.zeros(El, dtype=np.int32)
        prefetched = C.c_int32(0)
        rt = None
        if want_routing:
            k = self.top_k
            rt = {"topk_idx": torch.empty((N, k), dtype=torch.int32, device=x.device),
                  "topk_w": torch.empty((N, k), dtype=torch.float32, device=x.device),
                  "perm": torch.empty(N * k, dtype=torch.int32, device=x.device),
                  "offsets": torch.empty(E + 1, dtype=torch.int32, device=x.device)}
        out = ForwardOut(counts.ctypes.data, order.ctypes.data, C.addressof(feas),
                         C.addressof(events) if want_timeline else None,
                         C.addressof(exposed) if want_timeline else None,
                         local_rows.ctypes.data,
                         *([rt[n].data_ptr() for n in ("topk_idx", "topk_w", "perm", "offsets")]
                           if rt else [None] * 4),
                         None if time_origin is None else time_origin.cuda_event,
                         C.addressof(prefetched))
        _check(call(C.byref(out)))
        info = {"counts": counts, "order": order, "feasible": bool(feas.value),
                "local_rows": local_rows, "pinned": list(getattr(self, "pinned", [])),
                "prefetched": int(prefetched.value)}
        if rt:
            info.update(rt)
        if want_timeline:
            info["events"] = [(e.stream, e.layer_id, e.expert_id, e.start, e.end)
                              for e in events if e.stream >= 0]
            info["exposed_copy_s"] = exposed.value
        return y, info

    def close(self) -> None:
        if self._h:
            _lib.infmoe_layer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
