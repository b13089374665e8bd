"""paper_2408_00008_b200 -- B200-native Mixtral-8x7B sparse-MoE block (ScaleLLM's
engine hot path, arXiv 2408.00008 Sec. 4.1) behind the C ABI of include/moe.h.

This module is argument marshalling only (ctypes over libmoe.so): every step of
the forward runs in libmoe's CUDA kernels. torch is used for device memory and
streams. There is no CPU fallback: if libmoe.so is missing, importing this
package raises; if no sm_100 device is present, moe_init fails loudly.

Names follow the C ABI: moe_init, moe_packed_sizes, moe_pack_weights,
moe_forward, moe_forward_routed, moe_forward_host, moe_destroy, plus the
instrumentation and NCCL helpers. `MoEBlock` is a small convenience owner of a
context and its packed weights.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# MOE_LIB selects an experiment build of the same sources (scripts/ab_*.sh); default in-tree
LIB_PATH = os.environ.get("MOE_LIB") or os.path.join(_PKG, "libmoe.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libmoe.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = ctypes.CDLL(LIB_PATH)

MOE_OK, MOE_ERR_INVALID, MOE_ERR_UNSUPPORTED, MOE_ERR_OOM, MOE_ERR_CUDA, MOE_ERR_NCCL, MOE_ERR_STATE = range(7)
MOE_PAR_NONE, MOE_PAR_EP, MOE_PAR_TP, MOE_PAR_HYBRID = 0, 1, 2, 3
MOE_FLAG_RESIDUAL, MOE_FLAG_FORCE_SWAP, MOE_FLAG_FORCE_TILED, MOE_FLAG_NO_PDL, MOE_FLAG_NO_PAIR = 0x1, 0x2, 0x4, 0x8, 0x10
MOE_FLAG_EP_EXACT = 0x20
MOE_FLAG_FP8_WEIGHTS = 0x40
MOE_FLAG_GATHER = 0x80
MOE_FLAG_P2P = 0x100
MOE_FLAG_NVLS = 0x200
P2P_HANDLE_BYTES = 128
NUM_KERNEL_SLOTS = 8
KERNEL_SLOTS = ("router", "permute", "gemm1_w13_swiglu", "gemm2_w2", "combine", "dispatch", "exchange", "pack")

# every symbol include/moe.h declares (tests check the .so exports all of them)
EXPORTED = ("moe_init", "moe_packed_sizes", "moe_pack_weights", "moe_forward", "moe_forward_routed",
            "moe_forward_host", "moe_destroy", "moe_last_error", "moe_status_string", "moe_set_profiling",
            "moe_reset_profile", "moe_kernel_times", "moe_launch_count", "moe_nccl_unique_id",
            "moe_nccl_comm_init", "moe_nccl_comm_destroy", "moe_loopback_comm_create", "moe_loopback_comm_rank",
            "moe_loopback_comm_destroy", "moe_packed_sizes_fp8", "moe_pack_weights_fp8", "moe_p2p_handle",
            "moe_p2p_connect")


TUNING_FIELDS = ("g1_swap_rows", "g2_swap_rows", "g1_grid", "g2_grid", "spec_l2", "swap_nb_cap", "pair_nblk",
                 "pair_order", "router_cc_max_T", "weight_hint", "host_stage", "g1_nb", "g2_nb",
                 "pair_hints", "swap_pair", "fused", "fused_splits", "fused_stages", "fused_uniform", "fused_combine", "fused_chain", "fused_half", "combine_vec", "ep_fold")


class moe_tuning(ctypes.Structure):
    """include/moe.h moe_tuning: kernel-variant / grid overrides (0 = default)."""
    _fields_ = [(n, ctypes.c_int32) for n in TUNING_FIELDS] + [("reserved", ctypes.c_int32 * 8)]


class moe_config(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("ffn", ctypes.c_int32), ("num_experts", ctypes.c_int32),
                ("top_k", ctypes.c_int32), ("max_tokens", ctypes.c_int32), ("par", ctypes.c_int32),
                ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32), ("nccl_comm", ctypes.c_void_p),
                ("flags", ctypes.c_uint32), ("split_k", ctypes.c_int32), ("device", ctypes.c_int32),
                ("tp_size", ctypes.c_int32), ("tp_comm", ctypes.c_void_p),
                ("tuning", ctypes.POINTER(moe_tuning)), ("reserved", ctypes.c_int32 * 2)]


class moe_expert_weights(ctypes.Structure):
    _fields_ = [("w13", ctypes.c_void_p), ("w2", ctypes.c_void_p), ("w13_scale", ctypes.c_void_p),
                ("w2_scale", ctypes.c_void_p)]


class moe_aux(ctypes.Structure):
    _fields_ = [("logits", ctypes.c_void_p), ("topk_idx", ctypes.c_void_p), ("topk_w", ctypes.c_void_p),
                ("expert_counts", ctypes.c_void_p), ("expert_offsets", ctypes.c_void_p), ("pos", ctypes.c_void_p),
                ("out_f32", ctypes.c_void_p)]


_P, _I32, _I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_sig = {
    "moe_init": ([ctypes.POINTER(moe_config), ctypes.POINTER(_P)], _I32),
    "moe_packed_sizes": ([ctypes.POINTER(moe_config), ctypes.POINTER(ctypes.c_size_t),
                          ctypes.POINTER(ctypes.c_size_t)], _I32),
    "moe_pack_weights": ([_P, _P, _P, _P, _P, _P, _P], _I32),
    "moe_forward": ([_P, _P, _I32, _P, ctypes.POINTER(moe_expert_weights), _P, ctypes.POINTER(moe_aux), _P], _I32),
    "moe_forward_routed": ([_P, _P, _I32, _P, _P, ctypes.POINTER(moe_expert_weights), _P,
                            ctypes.POINTER(moe_aux), _P], _I32),
    "moe_forward_host": ([_P, _P, _I32, _P, ctypes.POINTER(moe_expert_weights), _P, _P], _I32),
    "moe_destroy": ([_P], _I32),
    "moe_last_error": ([_P], ctypes.c_char_p),
    "moe_status_string": ([_I32], ctypes.c_char_p),
    "moe_set_profiling": ([_P, ctypes.c_int], _I32),
    "moe_reset_profile": ([_P], _I32),
    "moe_kernel_times": ([_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)], _I32),
    "moe_launch_count": ([_P], _I64),
    "moe_nccl_unique_id": ([_P], _I32),
    "moe_nccl_comm_init": ([_P, _I32, _I32, _I32, ctypes.POINTER(_P)], _I32),
    "moe_nccl_comm_destroy": ([_P], _I32),
    "moe_loopback_comm_create": ([_I32, ctypes.POINTER(_P)], _I32),
    "moe_packed_sizes_fp8": ([ctypes.POINTER(moe_config)] + [ctypes.POINTER(ctypes.c_size_t)] * 4, _I32),
    "moe_pack_weights_fp8": ([_P] * 12, _I32),
    "moe_loopback_comm_rank": ([_P, _I32, ctypes.POINTER(_P)], _I32),
    "moe_loopback_comm_destroy": ([_P], _I32),
    "moe_p2p_handle": ([_P, _P], _I32),
    "moe_p2p_connect": ([_P, _P, _I32], _I32),
}
for _name, (_args, _res) in _sig.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


class MoEError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{_lib.moe_status_string(status).decode()}: {msg}")


def _check(status, ctx=None):
    if status != MOE_OK:
        raise MoEError(status, (_lib.moe_last_error(ctx) or b"").decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def make_tuning(tuning=None):
    """dict of moe_tuning fields (unknown names raise) -> moe_tuning, or None."""
    if not tuning:
        return None
    t = moe_tuning()
    for k, v in tuning.items():
        if k not in TUNING_FIELDS:
            raise KeyError(f"unknown tuning field {k!r} (fields: {TUNING_FIELDS})")
        setattr(t, k, int(v))
    return t


def make_config(hidden, ffn, num_experts, top_k, max_tokens, par=MOE_PAR_NONE, world_size=1, rank=0,
                nccl_comm=None, flags=0, split_k=0, device=-1, tp_size=0, tp_comm=None, tuning=None) -> moe_config:
    c = moe_config()
    c.hidden, c.ffn, c.num_experts, c.top_k, c.max_tokens = hidden, ffn, num_experts, top_k, max_tokens
    c.par, c.world_size, c.rank, c.nccl_comm = par, world_size, rank, nccl_comm
    c.flags, c.split_k, c.device = flags, split_k, device
    c.tp_size, c.tp_comm = tp_size, tp_comm
    t = make_tuning(tuning) if not isinstance(tuning, moe_tuning) else tuning
    if t is not None:
        c._tuning_ref = t  # keep the struct alive as long as the config (moe_init copies it)
        c.tuning = ctypes.pointer(t)
    return c


# ------------------------------------------------------------------ C-ABI mirrors
def moe_init(cfg: moe_config):
    ctx = _P()
    _check(_lib.moe_init(ctypes.byref(cfg), ctypes.byref(ctx)))
    return ctx.value


def moe_packed_sizes(cfg: moe_config):
    a, b = ctypes.c_size_t(), ctypes.c_size_t()
    _check(_lib.moe_packed_sizes(ctypes.byref(cfg), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def moe_pack_weights(ctx, w1, w3, w2, w13_out, w2_out, stream=None):
    _check(_lib.moe_pack_weights(ctx, _ptr(w1), _ptr(w3), _ptr(w2), _ptr(w13_out), _ptr(w2_out),
                                 _stream(stream)), ctx)


def _aux(aux):
    if aux is None:
        return None
    a = moe_aux()
    for k in ("logits", "topk_idx", "topk_w", "expert_counts", "expert_offsets", "pos", "out_f32"):
        setattr(a, k, _ptr(aux.get(k)))
    return ctypes.byref(a)


def _weights(w13, w2, w13_scale=None, w2_scale=None):
    return ctypes.byref(moe_expert_weights(_ptr(w13), _ptr(w2), _ptr(w13_scale), _ptr(w2_scale)))


def moe_forward(ctx, tokens, T, router_w, w13, w2, out, aux=None, stream=None, w13_scale=None, w2_scale=None):
    _check(_lib.moe_forward(ctx, _ptr(tokens), int(T), _ptr(router_w), _weights(w13, w2, w13_scale, w2_scale),
                            _ptr(out), _aux(aux), _stream(stream)), ctx)


def moe_packed_sizes_fp8(cfg: moe_config):
    v = [ctypes.c_size_t() for _ in range(4)]
    _check(_lib.moe_packed_sizes_fp8(ctypes.byref(cfg), *[ctypes.byref(x) for x in v]))
    return tuple(x.value for x in v)


def moe_pack_weights_fp8(ctx, q1, q3, q2, s1, s3, s2, w13_out, w2_out, s13_out, s2_out, stream=None):
    _check(_lib.moe_pack_weights_fp8(ctx, *[_ptr(t) for t in (q1, q3, q2, s1, s3, s2, w13_out, w2_out, s13_out,
                                                               s2_out)], _stream(stream)), ctx)


def moe_forward_routed(ctx, tokens, T, topk_idx, topk_w, w13, w2, out, aux=None, stream=None):
    _check(_lib.moe_forward_routed(ctx, _ptr(tokens), int(T), _ptr(topk_idx), _ptr(topk_w), _weights(w13, w2),
                                   _ptr(out), _aux(aux), _stream(stream)), ctx)


def moe_forward_host(ctx, tokens_host, T, router_w, w13, w2, out_host, stream=None, w13_scale=None, w2_scale=None):
    _check(_lib.moe_forward_host(ctx, _ptr(tokens_host), int(T), _ptr(router_w),
                                 _weights(w13, w2, w13_scale, w2_scale), _ptr(out_host), _stream(stream)), ctx)


def moe_destroy(ctx):
    _check(_lib.moe_destroy(ctx))


def moe_last_error(ctx=None) -> str:
    return (_lib.moe_last_error(ctx) or b"").decode()


def moe_set_profiling(ctx, enable: bool):
    _check(_lib.moe_set_profiling(ctx, int(bool(enable))), ctx)


def moe_reset_profile(ctx):
    _check(_lib.moe_reset_profile(ctx), ctx)


def moe_kernel_times(ctx):
    ms = (ctypes.c_double * NUM_KERNEL_SLOTS)()
    n = (_I64 * NUM_KERNEL_SLOTS)()
    _check(_lib.moe_kernel_times(ctx, ms, n), ctx)
    return {KERNEL_SLOTS[i]: (ms[i], n[i]) for i in range(NUM_KERNEL_SLOTS)}


def moe_launch_count(ctx) -> int:
    return int(_lib.moe_launch_count(ctx))


def moe_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.moe_nccl_unique_id(buf))
    return buf.raw


def moe_nccl_comm_init(uid: bytes, world: int, rank: int, device: int):
    comm = _P()
    buf = ctypes.create_string_buffer(uid, 128)
    _check(_lib.moe_nccl_comm_init(buf, world, rank, device, ctypes.byref(comm)))
    return comm.value


def moe_nccl_comm_destroy(comm):
    _check(_lib.moe_nccl_comm_destroy(comm))


def moe_loopback_comm_create(world: int):
    g = _P()
    _check(_lib.moe_loopback_comm_create(world, ctypes.byref(g)))
    return g.value


def moe_loopback_comm_rank(group, rank: int):
    c = _P()
    _check(_lib.moe_loopback_comm_rank(group, rank, ctypes.byref(c)))
    return c.value


def moe_loopback_comm_destroy(handle):
    _check(_lib.moe_loopback_comm_destroy(handle))


def moe_p2p_handle(ctx) -> bytes:
    """This rank's symmetric-region handle (MOE_P2P_HANDLE_BYTES opaque bytes)."""
    buf = ctypes.create_string_buffer(P2P_HANDLE_BYTES)
    _check(_lib.moe_p2p_handle(ctx, buf), ctx)
    return buf.raw


def moe_p2p_connect(ctx, handles):
    """handles: the group's handles in rank order (list of bytes, or their concatenation)."""
    blob = b"".join(handles) if isinstance(handles, (list, tuple)) else bytes(handles)
    if len(blob) % P2P_HANDLE_BYTES:
        raise ValueError("handle blob size is not a multiple of P2P_HANDLE_BYTES")
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(_lib.moe_p2p_connect(ctx, buf, len(blob) // P2P_HANDLE_BYTES), ctx)


def p2p_connect_process_group(ctx, group=None):
    """MOE_FLAG_P2P over torch.distributed: all-gather the handles on the host
    process group (any backend), then connect. Call on every rank of the group."""
    import torch.distributed as dist
    mine = moe_p2p_handle(ctx)
    allh = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    moe_p2p_connect(ctx, allh)


def nccl_comm_from_process_group(world: int, rank: int, device: int):
    """Create libmoe's NCCL communicator for the current torch.distributed group:
    rank 0 draws the ncclUniqueId, the host process group broadcasts it."""
    import torch.distributed as dist
    obj = [moe_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return moe_nccl_comm_init(obj[0], world, rank, device)


def nccl_hybrid_comms(world: int, rank: int, tp: int, device: int):
    """EP x TP communicators for MOE_PAR_HYBRID: rank = ep_rank * tp + tp_rank.
    Returns (ep_comm over the ranks sharing my tp_rank, tp_comm over my EP group).
    Rank 0 draws every group's ncclUniqueId; the host process group broadcasts them."""
    ep = world // tp
    obj = [[moe_nccl_unique_id() for _ in range(tp + ep)] if rank == 0 else None]
    if world > 1:
        import torch.distributed as dist
        dist.broadcast_object_list(obj, src=0)
    ids = obj[0]
    e, t = rank // tp, rank % tp
    ep_comm = moe_nccl_comm_init(ids[t], ep, e, device)
    tp_comm = moe_nccl_comm_init(ids[tp + e], tp, t, device)
    return ep_comm, tp_comm


# ------------------------------------------------------------------ convenience owner
class MoEBlock:
    """Owns a libmoe context and this rank's packed weights (torch device memory).

    w1, w3: [E, f, d], w2: [E, d, f], router_w: [E, d] -- bf16 HF layout (device).
    """

    def __init__(self, router_w, w1, w3, w2, top_k=2, max_tokens=64, par=MOE_PAR_NONE, world_size=1, rank=0,
                 nccl_comm=None, flags=0, split_k=0, device=None, tp_size=0, tp_comm=None, tuning=None):
        """FP8 weights: pass flags |= MOE_FLAG_FP8_WEIGHTS and w1/w3/w2 as (q, scale) pairs
        (synth.quantize_fp8_rows). tuning: dict of moe_tuning overrides (include/moe.h)."""
        dev = router_w.device if device is None else torch.device(device)
        w1_fp8 = (w1, w3, w2) if flags & MOE_FLAG_FP8_WEIGHTS else None
        E, f, d = (w1[0] if w1_fp8 else w1).shape
        self.cfg = make_config(d, f, E, top_k, max_tokens, par, world_size, rank, nccl_comm, flags, split_k,
                               dev.index if dev.index is not None else torch.cuda.current_device(), tp_size, tp_comm,
                               tuning)
        self.ctx = moe_init(self.cfg)
        self.d, self.f, self.E, self.k = d, f, E, top_k
        self.router_w = router_w.contiguous()
        self.s13 = self.s2 = None
        if flags & MOE_FLAG_FP8_WEIGHTS:
            # w1, w3, w2 are (q uint8 E4M3 bytes, s fp32 per-row power-of-two scale) pairs
            (q1, s1), (q3, s3), (q2, s2) = w1_fp8
            b13, b2, bs13, bs2 = moe_packed_sizes_fp8(self.cfg)
            self.w13 = torch.empty(b13, dtype=torch.uint8, device=dev)
            self.w2 = torch.empty(b2, dtype=torch.uint8, device=dev)
            self.s13 = torch.empty(bs13 // 4, dtype=torch.float32, device=dev)
            self.s2 = torch.empty(bs2 // 4, dtype=torch.float32, device=dev)
            moe_pack_weights_fp8(self.ctx, q1.contiguous(), q3.contiguous(), q2.contiguous(), s1.contiguous(),
                                 s3.contiguous(), s2.contiguous(), self.w13, self.w2, self.s13, self.s2)
        else:
            b13, b2 = moe_packed_sizes(self.cfg)
            self.w13 = torch.empty(b13 // 2, dtype=torch.bfloat16, device=dev)
            self.w2 = torch.empty(b2 // 2, dtype=torch.bfloat16, device=dev)
            moe_pack_weights(self.ctx, w1.contiguous(), w3.contiguous(), w2.contiguous(), self.w13, self.w2)

    def forward(self, x, out=None, aux=None, stream=None):
        T = x.shape[0]
        if out is None:
            out = torch.empty_like(x)
        moe_forward(self.ctx, x, T, self.router_w, self.w13, self.w2, out, aux, stream, self.s13, self.s2)
        return out

    def p2p_handle(self) -> bytes:
        return moe_p2p_handle(self.ctx)

    def p2p_connect(self, handles):
        moe_p2p_connect(self.ctx, handles)

    def forward_routed(self, x, topk_idx, topk_w, out=None, aux=None, stream=None):
        if out is None:
            out = torch.empty_like(x)
        _check(_lib.moe_forward_routed(self.ctx, _ptr(x), int(x.shape[0]), _ptr(topk_idx), _ptr(topk_w),
                                       _weights(self.w13, self.w2, self.s13, self.s2), _ptr(out), _aux(aux),
                                       _stream(stream)), self.ctx)
        return out

    def close(self):
        if getattr(self, "ctx", None):
            moe_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MoEStack:
    """A stack of L MoE layers, x_{l+1} = x_l + MoE_l(x_l) (reading R12; the
    residual add is fused into the combine kernel via MOE_FLAG_RESIDUAL). All layers
    share one libmoe context (one workspace, cached per-layer TMA descriptors).

    layers: list of dicts with HF-layout bf16 device tensors wg, w1, w3, w2 (each
    layer's tensors may be freed by the caller after construction: they are packed).
    """

    def __init__(self, layers, top_k=2, max_tokens=64, par=MOE_PAR_NONE, world_size=1, rank=0, nccl_comm=None,
                 flags=0, split_k=0, device=None, tuning=None):
        first = layers[0]
        dev = first["wg"].device if device is None else torch.device(device)
        E, f, d = first["w1"].shape
        self.cfg = make_config(d, f, E, top_k, max_tokens, par, world_size, rank, nccl_comm,
                               flags | MOE_FLAG_RESIDUAL, split_k,
                               dev.index if dev.index is not None else torch.cuda.current_device(), tuning=tuning)
        self.ctx = moe_init(self.cfg)
        self.d, self.T_max = d, max_tokens
        b13, b2 = moe_packed_sizes(self.cfg)
        self.w13, self.w2, self.router_w = [], [], []
        for lw in layers:
            self.add_layer(lw, b13, b2, dev)
        self._buf = [torch.empty(max_tokens, d, dtype=torch.bfloat16, device=dev) for _ in range(2)]

    def add_layer(self, lw, b13=None, b2=None, dev=None):
        if b13 is None:
            b13, b2 = moe_packed_sizes(self.cfg)
        dev = dev or lw["wg"].device
        w13 = torch.empty(b13 // 2, dtype=torch.bfloat16, device=dev)
        w2 = torch.empty(b2 // 2, dtype=torch.bfloat16, device=dev)
        moe_pack_weights(self.ctx, lw["w1"].contiguous(), lw["w3"].contiguous(), lw["w2"].contiguous(), w13, w2)
        self.w13.append(w13)
        self.w2.append(w2)
        self.router_w.append(lw["wg"].contiguous())

    @property
    def num_layers(self):
        return len(self.w13)

    def forward(self, x, out=None, stream=None, layer_outputs=None, layer_aux=None):
        """x [T, d] bf16 -> out [T, d] bf16 after all layers. layer_outputs: optional
        list that receives each layer's output tensor (views of internal buffers are
        cloned); layer_aux: optional list of per-layer moe_aux dicts (or None) filled by
        the layer's forward (routing, out_f32 before the rounding) -- both used by the
        per-layer parity tests."""
        T = x.shape[0]
        cur = x
        for l in range(self.num_layers):
            dst = out if (l == self.num_layers - 1 and out is not None) else self._buf[l % 2][:T]
            aux = layer_aux[l] if layer_aux is not None else None
            moe_forward(self.ctx, cur, T, self.router_w[l], self.w13[l], self.w2[l], dst, aux, stream)
            if layer_outputs is not None:
                layer_outputs.append(dst.clone())
            cur = dst
        return cur

    def close(self):
        if getattr(self, "ctx", None):
            moe_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
