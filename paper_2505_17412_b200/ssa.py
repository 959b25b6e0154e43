"""Thin ctypes binding of libssa_b200.so (include/ssa.h). Argument marshalling only.

Every step of SSA runs in the library's CUDA kernels; PyTorch supplies device memory (torch.empty on
the tensors' device) and the current CUDA stream. There is NO CPU fallback: if the shared library is
missing or a tensor is not on a CUDA device, these functions raise.

Entry points (same names as the C ABI):
    ssa_build_blocks(coords, grid, batch, m_cmp, m_slc, m_win, m_q)  -> Plan
    ssa_forward(plan, cfg, q, k, v, gates)                          -> (out, Saved)
    ssa_backward(plan, cfg, saved, q, k, v, gates, dout)            -> (dq, dk, dv, dgates)
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSA_LIB", os.path.join(_HERE, "libssa_b200.so"))   # SSA_LIB: debug builds only

SSA_F32, SSA_BF16 = 0, 1
SSA_INPUT_SORTED, SSA_FORCE_SIMT, SSA_SAVE_SCORES, SSA_KV_GRAD_FP32, SSA_WINDOW_ONLY, SSA_LOCAL_ROWS = 1, 2, 4, 8, 16, 32
SSA_NO_WINDOW, SSA_ACCUMULATE = 64, 128
LEVEL_CMP, LEVEL_SLC, LEVEL_WIN, LEVEL_Q = 0, 1, 2, 3
STATUS = ["SSA_OK", "SSA_ERR_ARG", "SSA_ERR_DUP_COORD", "SSA_ERR_COORD_RANGE", "SSA_ERR_HIERARCHY",
          "SSA_ERR_BAD_STATE", "SSA_ERR_WORKSPACE", "SSA_ERR_UNSUPPORTED", "SSA_ERR_CUDA"]


class SSAError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.code = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{where}: {self.code}: {detail}")


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("batch", ctypes.c_int32), ("grid", ctypes.c_int32 * 3),
                ("m", ctypes.c_int32 * 4), ("n_blocks", ctypes.c_int32 * 4), ("max_fill", ctypes.c_int32 * 4),
                ("max_blocks_per_batch", ctypes.c_int32 * 4), ("perm", ctypes.c_void_p),
                ("inv_perm", ctypes.c_void_p), ("sorted_coords", ctypes.c_void_p),
                ("offsets", ctypes.c_void_p * 4), ("block_coords", ctypes.c_void_p * 4),
                ("batch_blocks", ctypes.c_void_p * 4), ("batch_tokens", ctypes.c_void_p),
                ("cmp_to_slc", ctypes.c_void_p)]


class LearnedC(ctypes.Structure):
    _fields_ = [("conv_k_w", ctypes.c_void_p), ("conv_k_b", ctypes.c_void_p), ("conv_v_w", ctypes.c_void_p),
                ("conv_v_b", ctypes.c_void_p), ("x", ctypes.c_void_p), ("c", ctypes.c_int32),
                ("gate_w", ctypes.c_void_p), ("gate_b", ctypes.c_void_p), ("d_conv_k_w", ctypes.c_void_p),
                ("d_conv_k_b", ctypes.c_void_p), ("d_conv_v_w", ctypes.c_void_p), ("d_conv_v_b", ctypes.c_void_p),
                ("dx", ctypes.c_void_p), ("d_gate_w", ctypes.c_void_p), ("d_gate_b", ctypes.c_void_p)]


class AttnCfgC(ctypes.Structure):
    _fields_ = [("h_q", ctypes.c_int32), ("h_kv", ctypes.c_int32), ("d", ctypes.c_int32),
                ("top_k", ctypes.c_int32), ("scale", ctypes.c_float), ("dtype", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("pe_k", ctypes.c_void_p), ("pe_v", ctypes.c_void_p),
                ("q_begin", ctypes.c_int32), ("q_end", ctypes.c_int32), ("kc_in", ctypes.c_void_p),
                ("vc_in", ctypes.c_void_p), ("kv_event", ctypes.c_void_p), ("learned", ctypes.POINTER(LearnedC)),
                ("n_peer", ctypes.c_int32), ("my_rank", ctypes.c_int32), ("peer_k", ctypes.c_void_p * 16),
                ("peer_v", ctypes.c_void_p * 16), ("peer_tok", ctypes.c_int32 * 17)]


class SavedView(ctypes.Structure):
    _fields_ = [("idx", ctypes.c_void_p), ("scores", ctypes.c_void_p), ("o_branch", ctypes.c_void_p * 3),
                ("lse_branch", ctypes.c_void_p * 3), ("k_cmp", ctypes.c_void_p), ("v_cmp", ctypes.c_void_p),
                ("used_tcgen05", ctypes.c_int32), ("d_internal", ctypes.c_int32)]


_lib = None

# symbol -> (restype, argtypes)
_P = ctypes.c_void_p
_SZ = ctypes.POINTER(ctypes.c_size_t)
SIGNATURES = {
    "ssa_build_blocks_size": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                             ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _SZ, _SZ]),
    "ssa_build_blocks": (ctypes.c_int, [_P, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                        ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P,
                                        ctypes.c_size_t, _P, ctypes.c_size_t, _P, ctypes.POINTER(_P)]),
    "ssa_plan_destroy": (None, [_P]),
    "ssa_get_plan_info": (ctypes.c_int, [_P, ctypes.POINTER(PlanInfo)]),
    "ssa_forward_size": (ctypes.c_int, [_P, ctypes.POINTER(AttnCfgC), _SZ, _SZ]),
    "ssa_forward": (ctypes.c_int, [_P, ctypes.POINTER(AttnCfgC), _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P,
                                   ctypes.c_size_t, _P]),
    "ssa_backward_size": (ctypes.c_int, [_P, ctypes.POINTER(AttnCfgC), _SZ]),
    "ssa_backward": (ctypes.c_int, [_P, ctypes.POINTER(AttnCfgC), _P, _P, _P, _P, _P, ctypes.c_size_t, _P, _P, _P,
                                    _P, _P, _P, ctypes.c_size_t, _P]),
    "ssa_pool": (ctypes.c_int, [_P, ctypes.POINTER(AttnCfgC), _P, _P, _P, _P, _P]),
    "ssa_ipc_handle": (ctypes.c_int, [_P, _P]),
    "ssa_ipc_open": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "ssa_ipc_close": (ctypes.c_int, [_P]),
    "ssa_saved_state": (ctypes.c_int, [_P, ctypes.POINTER(AttnCfgC), _P, ctypes.c_size_t,
                                       ctypes.POINTER(SavedView)]),
    "ssa_status_str": (ctypes.c_char_p, [ctypes.c_int]),
    "ssa_last_error": (ctypes.c_char_p, []),
    "ssa_launch_count": (ctypes.c_int64, []),
    "ssa_reset_launch_count": (None, []),
    "ssa_build_info": (ctypes.c_char_p, []),
    "ssa_profile_enable": (None, [ctypes.c_int]),
    "ssa_profile_reset": (None, []),
    "ssa_profile_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_int64)]),
}


def lib():
    """Load libssa_b200.so (raises if it has not been built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2505_17412_b200.build` "
                              "(the SSA path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, where: str):
    if status != 0:
        raise SSAError(status, where, lib().ssa_last_error().decode())


def _stream(device: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev(t: torch.Tensor, name: str, optional: bool = False):
    if t is None and optional:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return SSA_F32
    if dt == torch.bfloat16:
        return SSA_BF16
    raise ValueError(f"unsupported dtype {dt} (float32 or bfloat16)")


class Plan:
    """Owns the device plan buffer and the host handle of one block partition."""

    def __init__(self, handle, plan_buf: torch.Tensor, coords: torch.Tensor):
        self._handle = handle
        self.buf = plan_buf
        self.device = plan_buf.device
        info = PlanInfo()
        _check(lib().ssa_get_plan_info(handle, ctypes.byref(info)), "ssa_get_plan_info")
        self.info = info
        self.n = int(info.n)
        self.batch = int(info.batch)
        self.m = tuple(info.m)
        self.n_blocks = tuple(info.n_blocks)
        self.max_fill = tuple(info.max_fill)
        self.max_blocks_per_batch = tuple(info.max_blocks_per_batch)

    @property
    def handle(self):
        return self._handle

    def _i32(self, ptr: int, count: int) -> torch.Tensor:
        """Copy `count` int32 from a device pointer inside the plan buffer (parity hooks)."""
        base = self.buf.data_ptr()
        off = (ptr - base) // 4
        return self.buf.view(torch.int32)[off:off + count].clone()

    def perm(self):
        return self._i32(self.info.perm, self.n)

    def offsets(self, level: int):
        return self._i32(self.info.offsets[level], self.n_blocks[level] + 1)

    def q_offsets_host(self):
        """Query-block token offsets on the host (cached; one device read)."""
        if getattr(self, "_q_off", None) is None:
            self._q_off = self.offsets(LEVEL_Q).cpu().numpy()
        return self._q_off

    def block_coords(self, level: int):
        return self._i32(self.info.block_coords[level], 4 * self.n_blocks[level]).view(-1, 4)

    def batch_blocks(self, level: int):
        return self._i32(self.info.batch_blocks[level], self.batch + 1)

    def cmp_to_slc(self):
        return self._i32(self.info.cmp_to_slc, self.n_blocks[LEVEL_CMP])

    def __del__(self):
        if getattr(self, "_handle", None) is not None and _lib is not None:
            _lib.ssa_plan_destroy(self._handle)
            self._handle = None


def ssa_build_blocks(coords: torch.Tensor, grid, batch: int, m_cmp: int, m_slc: int, m_win: int,
                     m_q: int) -> Plan:
    """C: ssa_build_blocks. coords: CUDA int32 [N,4] (b,x,y,z)."""
    L = lib()
    if coords.dtype != torch.int32 or coords.dim() != 2 or coords.shape[1] != 4:
        raise ValueError("coords must be int32 [N,4]")
    cp = _dev(coords, "coords")
    n = coords.shape[0]
    g = (ctypes.c_int32 * 3)(*[int(x) for x in grid])
    pb, wb = ctypes.c_size_t(), ctypes.c_size_t()
    _check(L.ssa_build_blocks_size(n, batch, g, m_cmp, m_slc, m_win, m_q, ctypes.byref(pb), ctypes.byref(wb)),
           "ssa_build_blocks_size")
    plan_buf = torch.empty(pb.value, dtype=torch.uint8, device=coords.device)
    ws = torch.empty(wb.value, dtype=torch.uint8, device=coords.device)
    h = ctypes.c_void_p()
    _check(L.ssa_build_blocks(cp, n, batch, g, m_cmp, m_slc, m_win, m_q, ctypes.c_void_p(plan_buf.data_ptr()),
                              pb.value, ctypes.c_void_p(ws.data_ptr()), wb.value, _stream(coords.device),
                              ctypes.byref(h)), "ssa_build_blocks")
    return Plan(h, plan_buf, coords)


@dataclass
class Learned:
    """Learned compression delta (Eq. 7, reading R17) and gate projection (Eq. 6 / P:153, reading R18):
    conv_*_w fp32 [m_cmp^3, h_kv, d, d], conv_*_b fp32 [h_kv, d]; x [N, C] (dtype, caller order),
    gate_w fp32 [C, 3 h_q], gate_b fp32 [3 h_q]. ssa_backward fills `grads` (same names with a d_ prefix;
    dx in x's dtype)."""
    conv_k_w: torch.Tensor | None = None
    conv_k_b: torch.Tensor | None = None
    conv_v_w: torch.Tensor | None = None
    conv_v_b: torch.Tensor | None = None
    x: torch.Tensor | None = None
    gate_w: torch.Tensor | None = None
    gate_b: torch.Tensor | None = None
    grads: dict | None = None

    def c(self, grads: dict | None = None) -> LearnedC:
        def ptr(t):
            return t.data_ptr() if t is not None else None
        g = grads or {}
        return LearnedC(ptr(self.conv_k_w), ptr(self.conv_k_b), ptr(self.conv_v_w), ptr(self.conv_v_b), ptr(self.x),
                        int(self.x.shape[1]) if self.x is not None else 0, ptr(self.gate_w), ptr(self.gate_b),
                        ptr(g.get("d_conv_k_w")), ptr(g.get("d_conv_k_b")), ptr(g.get("d_conv_v_w")),
                        ptr(g.get("d_conv_v_b")), ptr(g.get("dx")), ptr(g.get("d_gate_w")), ptr(g.get("d_gate_b")))

    def alloc_grads(self) -> dict:
        g = {}
        for name in ("conv_k_w", "conv_k_b", "conv_v_w", "conv_v_b", "gate_w", "gate_b"):
            t = getattr(self, name)
            if t is not None:
                g["d_" + name] = torch.zeros_like(t, dtype=torch.float32)
        if self.x is not None:
            g["dx"] = torch.empty_like(self.x)
        return g


@dataclass
class AttnCfg:
    h_q: int
    h_kv: int
    d: int
    top_k: int
    dtype: torch.dtype = torch.bfloat16
    scale: float = 0.0
    flags: int = 0
    pe_k: torch.Tensor | None = None
    pe_v: torch.Tensor | None = None
    q_begin: int = 0            # query-block shard [q_begin, q_end) in plan order; q_end <= 0: all
    q_end: int = 0
    kc_in: torch.Tensor | None = None    # caller-supplied pooled keys / values, fp32 [h_kv, n_cmp, d]
    vc_in: torch.Tensor | None = None
    kv_event: torch.cuda.Event | None = None   # raw k / v ready (recorded after a K/V all-gather)
    learned: Learned | None = None
    # one-sided fetch of the selected K/V blocks: (peer_k ptrs, peer_v ptrs, token offsets [world + 1], my rank)
    peers: tuple | None = None

    def c(self, learned_grads: dict | None = None) -> AttnCfgC:
        def ptr(t):
            return t.data_ptr() if t is not None else None
        ev = self.kv_event.cuda_event if self.kv_event is not None else None
        lc = self.learned.c(learned_grads) if self.learned is not None else None
        cc = AttnCfgC(self.h_q, self.h_kv, self.d, self.top_k, float(self.scale), _dtype_code(self.dtype),
                      int(self.flags), ptr(self.pe_k), ptr(self.pe_v), int(self.q_begin), int(self.q_end),
                      ptr(self.kc_in), ptr(self.vc_in), ev, ctypes.pointer(lc) if lc is not None else None)
        cc._keep = lc          # the struct the pointer refers to lives as long as cc
        if self.peers is not None:
            pk, pv, tok, me = self.peers
            cc.n_peer, cc.my_rank = len(pk), int(me)
            for r in range(len(pk)):
                cc.peer_k[r], cc.peer_v[r] = int(pk[r]), int(pv[r])
            for r, t in enumerate(tok):
                cc.peer_tok[r] = int(t)
        return cc


class Saved:
    """Saved forward state (device buffer) + parity views into it."""

    def __init__(self, plan: Plan, cfg: AttnCfg, buf: torch.Tensor):
        self.plan, self.cfg, self.buf = plan, cfg, buf
        v = SavedView()
        cc = cfg.c()
        _check(lib().ssa_saved_state(plan.handle, ctypes.byref(cc), ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                     ctypes.byref(v)), "ssa_saved_state")
        self.view = v
        self.used_tcgen05 = bool(v.used_tcgen05)
        self.d_internal = int(v.d_internal)     # 64 when a d = 32 problem ran the tcgen05 kernels padded

    def _slice(self, ptr, count, dtype):
        es = torch.tensor([], dtype=dtype).element_size()
        off = ptr - self.buf.data_ptr()
        assert off % es == 0
        return self.buf[off:off + count * es].view(dtype)

    def indices(self) -> torch.Tensor:
        nq = self.plan.n_blocks[LEVEL_Q]
        return self._slice(self.view.idx, nq * self.cfg.h_kv * self.cfg.top_k, torch.int32).view(
            nq, self.cfg.h_kv, self.cfg.top_k)

    def scores(self) -> torch.Tensor | None:
        if not self.view.scores:
            return None
        nq = self.plan.n_blocks[LEVEL_Q]
        ms = max(self.plan.max_blocks_per_batch[LEVEL_SLC], 1)
        return self._slice(self.view.scores, nq * self.cfg.h_kv * ms, torch.float32).view(nq, self.cfg.h_kv, ms)

    def branch(self, b: int):
        """(o, lse) of branch b (0 cmp, 1 slc, 2 win), internal layout [h_kv][N][h_s][d], sorted order."""
        n, hk, hs, d = self.plan.n, self.cfg.h_kv, self.cfg.h_q // self.cfg.h_kv, self.d_internal
        o = self._slice(self.view.o_branch[b], n * self.cfg.h_q * d, torch.float32).view(hk, n, hs, d)
        lse = self._slice(self.view.lse_branch[b], n * self.cfg.h_q, torch.float32).view(hk, n, hs)
        return o, lse

    def k_cmp(self):
        nc = self.plan.n_blocks[LEVEL_CMP]
        d = self.d_internal
        return (self._slice(self.view.k_cmp, self.cfg.h_kv * nc * d, torch.float32).view(self.cfg.h_kv, nc, d),
                self._slice(self.view.v_cmp, self.cfg.h_kv * nc * d, torch.float32).view(self.cfg.h_kv, nc, d))


def owned_rows(plan: Plan, cfg: AttnCfg):
    """(first, end) plan-order rows of cfg's query-block range (all rows without a range)."""
    if cfg.q_end <= 0:
        return 0, plan.n
    off = plan.q_offsets_host()
    return int(off[cfg.q_begin]), int(off[cfg.q_end])


def _check_inputs(plan: Plan, cfg: AttnCfg, q, k, v, gates):
    n = plan.n
    a, b = owned_rows(plan, cfg) if cfg.flags & SSA_LOCAL_ROWS else (0, n)
    nr = b - a
    lg = cfg.learned is not None and cfg.learned.x is not None
    if gates is None and not lg:
        raise ValueError("gates are required unless cfg.learned.x supplies the gate projection input")
    if tuple(q.shape) != (nr, cfg.h_q, cfg.d) or tuple(k.shape) != (n, cfg.h_kv, cfg.d) or \
            tuple(v.shape) != (n, cfg.h_kv, cfg.d) or (gates is not None and tuple(gates.shape) != (nr, cfg.h_q, 3)):
        raise ValueError("shape mismatch: q [N,h_q,d], k/v [N,h_kv,d], gates [N,h_q,3] "
                         "(q, gates: owned rows only with SSA_LOCAL_ROWS)")
    for t in (q, k, v, gates, cfg.learned.x if lg else None):
        if t is not None and t.dtype != cfg.dtype:
            raise ValueError(f"tensor dtype {t.dtype} != cfg.dtype {cfg.dtype}")


class Workspace:
    """Reusable device scratch (grown on demand) so steady-state calls allocate nothing."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        return self.buf


_default_ws = {}


def _ws(device, key):
    """Per (device, stream) scratch: calls on different streams never share (or free) each other's
    buffer, and a buffer replaced on growth was only ever used on its own stream, so the caching
    allocator's stream-ordered reuse is safe."""
    sid = torch.cuda.current_stream(device).cuda_stream
    return _default_ws.setdefault((str(device), sid, key), Workspace())


def ssa_forward(plan: Plan, cfg: AttnCfg, q, k, v, gates, out=None, saved: Saved | None = None,
                ws: Workspace | None = None):
    """C: ssa_forward. Returns (out [N,h_q,d], Saved)."""
    L = lib()
    _check_inputs(plan, cfg, q, k, v, gates)
    cc = cfg.c()
    wsb, svb = ctypes.c_size_t(), ctypes.c_size_t()
    _check(L.ssa_forward_size(plan.handle, ctypes.byref(cc), ctypes.byref(wsb), ctypes.byref(svb)), "ssa_forward_size")
    dev = q.device
    if out is None:
        out = torch.empty_like(q)
    if saved is None:
        saved = Saved(plan, cfg, torch.empty(svb.value, dtype=torch.uint8, device=dev))
    w = (ws or _ws(dev, "fwd")).get(wsb.value, dev)
    _check(L.ssa_forward(plan.handle, ctypes.byref(cc), _dev(q, "q"), _dev(k, "k"), _dev(v, "v"),
                         _dev(gates, "gates", optional=True), _dev(out, "out"), ctypes.c_void_p(saved.buf.data_ptr()),
                         saved.buf.numel(), ctypes.c_void_p(w.data_ptr()), w.numel(), _stream(dev)), "ssa_forward")
    return out, saved


def ssa_pool(plan: Plan, cfg: AttnCfg, k, v, kc=None, vc=None):
    """C: ssa_pool. Pooled keys / values (Eq. 7) fp32 [h_kv, n_cmp, d] of the compression blocks inside
    the owned rows (all blocks without a query-block range); other blocks are 0. k, v in plan order
    (SSA_INPUT_SORTED), the owned rows only with SSA_LOCAL_ROWS."""
    nc = plan.n_blocks[LEVEL_CMP]
    if kc is None:
        kc = torch.empty(cfg.h_kv, nc, cfg.d, dtype=torch.float32, device=k.device)
        vc = torch.empty_like(kc)
    cc = cfg.c()
    _check(lib().ssa_pool(plan.handle, ctypes.byref(cc), _dev(k, "k"), _dev(v, "v"), _dev(kc, "kc"), _dev(vc, "vc"),
                          _stream(k.device)), "ssa_pool")
    return kc, vc


def ssa_backward(plan: Plan, cfg: AttnCfg, saved: Saved, q, k, v, gates, dout, grads=None,
                 ws: Workspace | None = None):
    """C: ssa_backward. Returns (dq, dk, dv, dgates)."""
    L = lib()
    _check_inputs(plan, cfg, q, k, v, gates)
    if tuple(dout.shape) != tuple(q.shape) or dout.dtype != cfg.dtype:
        raise ValueError("dout must match q")
    lgrads = cfg.learned.alloc_grads() if cfg.learned is not None else None
    cc = cfg.c(lgrads)
    wsb = ctypes.c_size_t()
    _check(L.ssa_backward_size(plan.handle, ctypes.byref(cc), ctypes.byref(wsb)), "ssa_backward_size")
    dev = q.device
    if grads is None:
        kvd = torch.float32 if cfg.flags & SSA_KV_GRAD_FP32 else k.dtype
        grads = (torch.empty_like(q), torch.empty_like(k, dtype=kvd), torch.empty_like(v, dtype=kvd),
                 torch.empty(q.shape[0], cfg.h_q, 3, dtype=q.dtype, device=q.device))
    dq, dk, dv, dg = grads
    w = (ws or _ws(dev, "bwd")).get(wsb.value, dev)
    _check(L.ssa_backward(plan.handle, ctypes.byref(cc), _dev(q, "q"), _dev(k, "k"), _dev(v, "v"),
                          _dev(gates, "gates", optional=True), ctypes.c_void_p(saved.buf.data_ptr()), saved.buf.numel(),
                          _dev(dout, "dout"), _dev(dq, "dq"), _dev(dk, "dk"), _dev(dv, "dv"), _dev(dg, "dgates"),
                          ctypes.c_void_p(w.data_ptr()), w.numel(), _stream(dev)), "ssa_backward")
    if lgrads is not None:
        cfg.learned.grads = lgrads
    return dq, dk, dv, dg


def window_attention(coords: torch.Tensor, grid, batch: int, m_win: int, q, k, v, *, h_kv: int, shift: int = 0,
                     dtype: torch.dtype = torch.bfloat16, window_only: bool = True):
    """Sparse 3D (shifted-)window attention, the SS-VAE's attention layer and SSA's window
    branch on its own: every active token attends the active tokens of its own aligned
    m_win^3 window; with shift = s the windows are those of coords + s (Swin-style shifted windows).

    Composition over the C ABI only (no arithmetic here): the plan is built on the shifted coordinates
    (grid + s) and ssa_forward runs with gates (0, 0, 1), which makes Eq. 6 return the window branch
    exactly. window_only=True sets SSA_WINDOW_ONLY (the compression and selection branches are skipped
    in the kernels); False runs the full SSA step with those gates (the reference composition).
    Returns (out, ctx) with ctx = (plan, cfg, saved, gates) for window_attention_backward."""
    if shift:
        coords = coords.clone()
        coords[:, 1:] += int(shift)
        grid = tuple(int(g) + int(shift) for g in grid)
    m_cmp = 4 if m_win % 4 == 0 else m_win
    plan = ssa_build_blocks(coords, grid, batch, m_cmp, m_win, m_win, m_win)
    cfg = AttnCfg(h_q=q.shape[1], h_kv=h_kv, d=q.shape[2], top_k=1, dtype=dtype,
                  flags=SSA_WINDOW_ONLY if window_only else 0)
    gates = torch.zeros(q.shape[0], q.shape[1], 3, dtype=q.dtype, device=q.device)
    gates[..., 2] = 1
    out, saved = ssa_forward(plan, cfg, q, k, v, gates)
    return out, (plan, cfg, saved, gates)


def shifted_window_ssa(coords: torch.Tensor, grid, batch: int, m_cmp: int, m_slc: int, shift: int, cfg: AttnCfg,
                       q, k, v, gates):
    """SSA with SHIFTED sparse 3D windows (the SS-VAE's Swin-style alternation, P:87-88,
    applied to SSA's window branch): compression and selection on the blocks of `coords`, the
    window branch on the aligned m_slc^3 windows of coords + shift. Composition over the C ABI (no
    arithmetic here): ssa_forward with SSA_NO_WINDOW on the plan of coords, then ssa_forward with
    SSA_WINDOW_ONLY | SSA_ACCUMULATE on the plan of the shifted coordinates (grid + shift), which adds
    omega_win * O_win(shifted) into the same `out`. Returns (out, ctx) for shifted_window_ssa_backward."""
    import dataclasses
    plan0 = ssa_build_blocks(coords, grid, batch, m_cmp, m_slc, m_slc, m_slc)
    cs = coords.clone()
    cs[:, 1:] += int(shift)
    plan1 = ssa_build_blocks(cs, tuple(int(x) + int(shift) for x in grid), batch, m_cmp, m_slc, m_slc, m_slc)
    c0 = dataclasses.replace(cfg, flags=cfg.flags | SSA_NO_WINDOW)
    c1 = dataclasses.replace(cfg, flags=cfg.flags | SSA_WINDOW_ONLY | SSA_ACCUMULATE)
    out, s0 = ssa_forward(plan0, c0, q, k, v, gates)
    out, s1 = ssa_forward(plan1, c1, q, k, v, gates, out=out)
    return out, (plan0, plan1, c0, c1, s0, s1)


def shifted_window_ssa_backward(ctx, q, k, v, gates, dout):
    """(dq, dk, dv, dgates) of shifted_window_ssa: the SSA_NO_WINDOW backward, then the shifted
    window-only backward accumulated into the same buffers (SSA_ACCUMULATE)."""
    plan0, plan1, c0, c1, s0, s1 = ctx
    grads = ssa_backward(plan0, c0, s0, q, k, v, gates, dout)
    return ssa_backward(plan1, c1, s1, q, k, v, gates, dout, grads=grads)


def window_attention_backward(ctx, q, k, v, dout):
    """Gradients (dq, dk, dv) of window_attention (the gate gradients are dropped)."""
    plan, cfg, saved, gates = ctx
    dq, dk, dv, _ = ssa_backward(plan, cfg, saved, q, k, v, gates, dout)
    return dq, dk, dv


def ipc_export(t: torch.Tensor):
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t's data in it) — for ipc_open in
    another process (the caching allocator sub-allocates, so the offset is carried separately)."""
    st = t.untyped_storage()
    info = st._share_cuda_()
    handle, off = bytes(info[1]), int(info[3])
    # torch's shareable handle: [format version byte][allocation kind byte][cudaIpcMemHandle_t, 64 B]
    # (a plain cudaMalloc'ed block; expandable segments are not IPC-exportable this way)
    if len(handle) > 64:
        handle = handle[-64:]
    return handle, off + (t.data_ptr() - st.data_ptr())


def ipc_open(handle: bytes, offset: int) -> tuple:
    """Open a peer's exported allocation: returns (mapped base, data pointer = base + offset)."""
    p = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(handle, 64)
    _check(lib().ssa_ipc_open(buf, ctypes.byref(p)), "ssa_ipc_open")
    return p.value, p.value + offset


def ipc_close(base: int):
    _check(lib().ssa_ipc_close(ctypes.c_void_p(base)), "ssa_ipc_close")


def launch_count() -> int:
    return int(lib().ssa_launch_count())


def reset_launch_count():
    lib().ssa_reset_launch_count()


def profile_enable(on: bool = True):
    lib().ssa_profile_enable(1 if on else 0)


def profile_reset():
    lib().ssa_profile_reset()


def profile_read(kernel: str):
    """(total device ms, launches) of `kernel` since the last profile_reset (synchronises)."""
    t, n = ctypes.c_double(), ctypes.c_int64()
    _check(lib().ssa_profile_read(kernel.encode(), ctypes.byref(t), ctypes.byref(n)), "ssa_profile_read")
    return t.value, n.value


def build_info() -> str:
    return lib().ssa_build_info().decode()


class SSAFunction(torch.autograd.Function):
    """Autograd wrapper: out = SSA(q, k, v, gates) for a fixed plan (block structure) and cfg."""

    @staticmethod
    def forward(ctx, q, k, v, gates, plan, cfg):
        out, saved = ssa_forward(plan, cfg, q.contiguous(), k.contiguous(), v.contiguous(), gates.contiguous())
        ctx.plan, ctx.cfg, ctx.saved = plan, cfg, saved
        ctx.save_for_backward(q, k, v, gates)
        return out

    @staticmethod
    def backward(ctx, dout):
        q, k, v, gates = ctx.saved_tensors
        dq, dk, dv, dg = ssa_backward(ctx.plan, ctx.cfg, ctx.saved, q.contiguous(), k.contiguous(), v.contiguous(),
                                      gates.contiguous(), dout.contiguous())
        return dq, dk, dv, dg, None, None


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)


def nsa1d_coords(lengths, m_cmp: int, m_slc: int):
    """The NSA-1D blocking arm ("treating latent tokens as a 1D sequence and partitioning it into
    fixed-length blocks based on token indices, analogous to NSA"; the paper's ablation baseline):
    coordinates whose spatial blocks ARE runs of consecutive token indices, so ssa_build_blocks + the
    unchanged SSA kernels compute NSA-style 1D block attention. Token i of a batch item gets
    x = 8 * (i // m_slc^3) ... such that compression blocks = l_cmp = m_cmp^3 consecutive tokens,
    selection blocks (and windows, query blocks with m_win = m_q = m_slc) = l_slc = m_slc^3 consecutive
    tokens, and the plan order is the index order. Index arithmetic only (no method arithmetic).
    lengths: tokens per batch item. Returns (coords int32 [N, 4] on the host, grid (3,))."""
    import numpy as np
    if m_slc % m_cmp:
        raise ValueError("m_slc must be a multiple of m_cmp")
    r = m_slc // m_cmp
    l_cmp, l_slc = m_cmp ** 3, m_slc ** 3
    out = []
    for b, n in enumerate(int(x) for x in lengths):
        i = np.arange(n, dtype=np.int64)
        B, rem = i // l_slc, i % l_slc
        c, v = rem // l_cmp, rem % l_cmp                       # cmp sub-block in the slc block, voxel
        cx, cy, cz = c // (r * r), (c // r) % r, c % r
        vx, vy, vz = v // (m_cmp * m_cmp), (v // m_cmp) % m_cmp, v % m_cmp
        out.append(np.stack([np.full(n, b), B * m_slc + cx * m_cmp + vx, cy * m_cmp + vy, cz * m_cmp + vz], 1))
    coords = np.concatenate(out).astype(np.int32) if out else np.zeros((0, 4), np.int32)
    n_max = max([int(x) for x in lengths] + [1])
    grid = (-(-n_max // l_slc) * m_slc, m_slc, m_slc)
    return coords, grid
