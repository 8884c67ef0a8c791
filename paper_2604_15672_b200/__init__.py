"""paper_2604_15672_b200 -- B200-native verification hot path of SMC-SD (arxiv 2604.15672).

Thin Python binding of ``libsmcsd.so`` (C ABI in ``include/smcsd.h``).  Every function here
only marshals ``torch.Tensor`` arguments into pointers and sizes and calls the entry point of
the same name; every step of the path runs in the library's sm_100a kernels.  PyTorch is used
for device memory, streams and process groups only.  There is no CPU fallback: importing
the package without the built library raises, and CPU tensors are rejected.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

__all__ = [
    "SMCSD_F32", "SMCSD_BF16", "SMCSD_SYSTEMATIC", "SMCSD_MULTINOMIAL", "SEGMENT",
    "ST_DEGENERATE", "ST_NOT_ABSCONT", "ST_BAD_TOKEN", "ST_NONFINITE",
    "SmcsdError", "Workspace", "StepPlan", "lib_path",
    "smcsd_workspace_bytes", "smcsd_workspace_init", "smcsd_weights", "smcsd_step",
    "smcsd_resample", "smcsd_weights_partial", "smcsd_weights_combine", "smcsd_kv_reindex",
    "smcsd_kv_reindex_multi", "kv_tensor", "smcsd_partials_rescale",
    "smcsd_version", "kv_geometry", "smcsd_select", "smcsd_kv_reindex_paged", "ST_BAD_PAGE",
    "smcsd_powersmc_weights", "smcsd_tp_exchange_bytes", "smcsd_tp_exchange_init",
    "smcsd_ipc_handle_bytes", "smcsd_ipc_export", "smcsd_ipc_open", "smcsd_ipc_close", "smcsd_tp_step",
    "ST_EXCHANGE", "ST_BAD_INDEX", "ST_OUT_OF_PAGES", "smcsd_kv_append_paged", "kv_pool",
    "paged_pool_geometry", "AppendOutputs", "smcsd_kv_append_workspace_bytes",
    "smcsd_set_poll_tail", "smcsd_set_small_tail",
]

SMCSD_F32, SMCSD_BF16 = 0, 1
SMCSD_SYSTEMATIC, SMCSD_MULTINOMIAL = 0, 1
SEGMENT = 8192
ST_DEGENERATE, ST_NOT_ABSCONT, ST_BAD_TOKEN, ST_NONFINITE, ST_BAD_PAGE = 1, 2, 4, 8, 16
ST_EXCHANGE, ST_BAD_INDEX, ST_OUT_OF_PAGES = 32, 64, 128
_RC = {0: "ok", 1: "invalid argument", 2: "CUDA launch or runtime error", 3: "not implemented"}

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("SMCSD_LIB_OVERRIDE") or os.path.join(_HERE, "libsmcsd.so")  # debug builds only


class SmcsdError(RuntimeError):
    def __init__(self, name, rc):
        super().__init__(f"{name} failed: rc={rc} ({_RC.get(rc, 'unknown')})")
        self.rc = rc


class _KvTensor(ctypes.Structure):
    """include/smcsd.h smcsd_kv_tensor (byte geometry of one state tensor)."""
    _fields_ = [("dst", ctypes.c_void_p), ("src", ctypes.c_void_p), ("n_outer", ctypes.c_int64),
                ("outer_stride", ctypes.c_int64), ("prompt_stride", ctypes.c_int64),
                ("particle_stride", ctypes.c_int64), ("seg_count", ctypes.c_int64),
                ("seg_bytes", ctypes.c_int64), ("seg_stride", ctypes.c_int64)]


class _KvPool(ctypes.Structure):
    """include/smcsd.h smcsd_kv_pool (byte geometry of one paged KV pool)."""
    _fields_ = [("base", ctypes.c_void_p), ("n_planes", ctypes.c_int64), ("plane_stride", ctypes.c_int64),
                ("page_stride", ctypes.c_int64), ("token_bytes", ctypes.c_int64)]


def _load():
    if not os.path.exists(lib_path):
        raise ImportError(f"{lib_path} is missing: run `python paper_2604_15672_b200/build.py` "
                          "(or __graft_entry__.build()) -- there is no fallback path")
    L = ctypes.CDLL(lib_path)
    vp, i32, i64, f32, u64, sz = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float,
                                  ctypes.c_uint64, ctypes.c_size_t)
    L.smcsd_workspace_bytes.argtypes = [i32, i32, i32, i64]
    L.smcsd_workspace_bytes.restype = sz
    L.smcsd_workspace_init.argtypes = [vp, sz, vp]
    L.smcsd_weights.argtypes = [vp, i64, i32, vp, i64, i32, i32, vp, vp, vp, i32, i32, i32, i64,
                                f32, f32, f32, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.smcsd_resample.argtypes = [vp, i32, i32, i64, f32, i32, u64, u64, vp, vp, vp, vp, vp, vp,
                                 vp, vp, vp, vp, vp, vp]
    L.smcsd_step.argtypes = [vp, i64, i32, vp, i64, i32, i32, vp, vp, vp, i32, i32, i32, i64,
                             f32, f32, f32, f32, i32, u64, u64, i64, vp,
                             vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.smcsd_weights_partial.argtypes = [vp, i64, i32, vp, i64, i32, i32, vp, vp, i32, i32, i32,
                                        i64, i64, f32, f32, vp, vp, sz, vp]
    L.smcsd_weights_combine.argtypes = [vp, i32, vp, vp, vp, i32, i32, i32, i64, f32, vp, vp, vp,
                                        vp, vp, vp, vp, vp, sz, vp]
    L.smcsd_kv_reindex.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, i32, i32, vp, vp]
    L.smcsd_kv_reindex_multi.argtypes = [ctypes.POINTER(_KvTensor), i32, vp, i32, i32, vp, vp]
    L.smcsd_partials_rescale.argtypes = [vp, vp, vp, i64, vp]
    L.smcsd_select.argtypes = [vp, i32, i32, i64, u64, u64, vp, vp, vp, vp, sz, vp]
    L.smcsd_kv_reindex_paged.argtypes = [vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, vp, vp]
    L.smcsd_powersmc_weights.argtypes = [vp, i64, i32, i32, vp, i32, i32, i64, f32, f32, vp, vp,
                                         vp, vp, vp, vp, vp, sz, vp]
    u32 = ctypes.c_uint32
    L.smcsd_tp_exchange_bytes.argtypes = [i32, i32, i32, i32, i32]
    L.smcsd_tp_exchange_bytes.restype = sz
    L.smcsd_tp_exchange_init.argtypes = [vp, sz, vp]
    L.smcsd_ipc_handle_bytes.argtypes = []
    L.smcsd_ipc_handle_bytes.restype = sz
    L.smcsd_ipc_export.argtypes = [vp, vp]
    L.smcsd_ipc_open.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p)]
    L.smcsd_ipc_close.argtypes = [vp, vp]
    L.smcsd_tp_step.argtypes = [vp, i64, i32, vp, i64, i32, i32, vp, vp, vp, i32, i32, i32, i64,
                                i64, i64, f32, f32, f32, f32, i32, u64, u64, i64, vp,
                                i32, i32, i32, u32, vp, vp,
                                vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.smcsd_kv_append_workspace_bytes.argtypes = [i32, i32, i32, i32]
    L.smcsd_kv_append_workspace_bytes.restype = sz
    L.smcsd_kv_append_paged.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp, vp, vp,
                                        vp, vp, vp, ctypes.POINTER(_KvPool), i32, vp, sz, vp]
    for name in ("smcsd_kv_append_paged", "smcsd_workspace_init", "smcsd_weights", "smcsd_resample", "smcsd_step",
                 "smcsd_weights_partial", "smcsd_weights_combine", "smcsd_kv_reindex",
                 "smcsd_kv_reindex_multi", "smcsd_partials_rescale", "smcsd_select", "smcsd_kv_reindex_paged", "smcsd_powersmc_weights",
                 "smcsd_tp_exchange_init", "smcsd_ipc_export", "smcsd_ipc_open", "smcsd_ipc_close",
                 "smcsd_tp_step"):
        getattr(L, name).restype = i32
    L.smcsd_set_small_tail.argtypes = [i32]
    L.smcsd_set_small_tail.restype = i32
    L.smcsd_set_poll_tail.argtypes = [i32]
    L.smcsd_set_poll_tail.restype = i32
    L.smcsd_version.restype = ctypes.c_char_p
    L.smcsd_strerror.restype = ctypes.c_char_p
    L.smcsd_strerror.argtypes = [i32]
    return L


_lib = _load()


def _check(name, rc):
    if rc != 0:
        raise SmcsdError(name, rc)


def _p(t):
    """Device pointer of a CUDA tensor (None -> NULL).  CPU tensors are rejected."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libsmcsd takes device tensors only (no CPU fallback)")
    return t.data_ptr()


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _dtype_code(t):
    if t.dtype == torch.bfloat16:
        return SMCSD_BF16
    if t.dtype == torch.float32:
        return SMCSD_F32
    raise TypeError(f"logits must be bfloat16 or float32, got {t.dtype}")


def _logits_geom(t, name):
    if t.dim() != 4:
        raise ValueError(f"{name} must be [P][N][rows_per_particle][ld]")
    if t.stride(3) != 1 or t.stride(2) != t.shape[3] or t.stride(1) != t.shape[2] * t.shape[3] \
            or t.stride(0) != t.shape[1] * t.shape[2] * t.shape[3]:
        raise ValueError(f"{name} must be contiguous (row pitch = last dim)")
    return t.shape[3], t.shape[2]


def _chk(t, name, dtypes, shape, device, *, optional=True):
    """Argument validation (marshalling only): dtype, shape, device and contiguity of a tensor
    whose data_ptr() goes to the C ABI.  Raises ValueError; None passes when optional."""
    if t is None:
        if optional:
            return
        raise ValueError(f"{name} is required")
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype not in dtypes:
        raise ValueError(f"{name} must be {' or '.join(str(d) for d in dtypes)}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_cuda or t.device != device:
        raise ValueError(f"{name} must be on {device} (no CPU fallback), got {t.device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


_I32 = (torch.int32,)
_U32 = (torch.int32, torch.uint32) if hasattr(torch, "uint32") else (torch.int32,)
_F32 = (torch.float32,)


def _check_inputs(dev, P, N, K, *, tokens=None, n_drafted=None, logw_prev=None, uniforms=None,
                  scheme=SMCSD_SYSTEMATIC):
    _chk(tokens, "tokens", _I32, (P, N, K), dev, optional=False)
    _chk(n_drafted, "n_drafted", _I32, (P, N), dev)
    _chk(logw_prev, "logw_prev", _F32, (P, N), dev)
    _chk(uniforms, "uniforms", _U32, (P,) if scheme == SMCSD_SYSTEMATIC else (P, N), dev)


def _resolve_eta(eta, N):
    """eta = None selects the reference threshold ESS < N/2 (reading G2)."""
    return N / 2.0 if eta is None else eta


def _empty(shape, dtype, device):
    return torch.empty(shape, dtype=dtype, device=device)


def smcsd_version() -> str:
    return _lib.smcsd_version().decode()


def smcsd_set_small_tail(enable: bool) -> bool:
    """Process-wide switch for the small (K1-resident) polling tail (include/smcsd.h); returns
    the previous setting."""
    return bool(_lib.smcsd_set_small_tail(1 if enable else 0))


def smcsd_set_poll_tail(enable: bool) -> bool:
    """Process-wide switch for the polling tail (include/smcsd.h); returns the previous setting."""
    return bool(_lib.smcsd_set_poll_tail(1 if enable else 0))


def smcsd_workspace_bytes(P: int, N: int, K: int, v_len: int) -> int:
    return int(_lib.smcsd_workspace_bytes(P, N, K, v_len))


def smcsd_workspace_init(ws: torch.Tensor, stream=None):
    _check("smcsd_workspace_init", _lib.smcsd_workspace_init(_p(ws), ws.numel(), _stream(stream)))


class Workspace:
    """A zero-initialised device workspace that grows on demand (plumbing only)."""

    def __init__(self, device=None):
        self.device = torch.device("cuda" if device is None else device)
        self.buf = None
        self.shape = None

    def get(self, P, N, K, v_len, stream=None):
        need = smcsd_workspace_bytes(P, N, K, v_len)
        if self.buf is None or self.buf.numel() < need:
            self.buf = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
            self.shape = None
        if self.shape != (P, N, K, v_len):
            # counters sit at shape-dependent offsets: re-zero on every shape change (smcsd.h)
            smcsd_workspace_init(self.buf, stream)
            self.shape = (P, N, K, v_len)
        return self.buf


_default_ws = {}


def _ws(ws, device, P, N, K, v_len, stream):
    if ws is None:
        # one default workspace per (device, stream): concurrent calls on different streams
        # must not share one (include/smcsd.h), calls on one stream are ordered by it
        key = (device.type, device.index, _stream(stream))
        ws = _default_ws.setdefault(key, Workspace(device))
    if isinstance(ws, Workspace):
        return ws.get(P, N, K, v_len, stream)
    return ws


@dataclass
class Outputs:
    logw: torch.Tensor = None
    logw_pre: torch.Tensor = None
    logp_tok: torch.Tensor = None
    logq_tok: torch.Tensor = None
    lse: torch.Tensor = None
    ess: torch.Tensor = None
    wnorm: torch.Tensor = None
    status: torch.Tensor = None
    ancestors: torch.Tensor = None
    offspring: torch.Tensor = None
    slot_src: torch.Tensor = None
    resampled: torch.Tensor = None
    n_ties: torch.Tensor = None
    partials: torch.Tensor = None
    bonus: torch.Tensor = None


def _alloc(out: Outputs, dev, P, N, K, fields):
    shapes = dict(logw=((P, N), torch.float32), logw_pre=((P, N), torch.float32),
                  logp_tok=((P, N, K), torch.float32), logq_tok=((P, N, K), torch.float32),
                  lse=((P,), torch.float64), ess=((P,), torch.float64),
                  wnorm=((P, N), torch.float32), status=((P,), torch.int32),
                  ancestors=((P, N), torch.int32), offspring=((P, N), torch.int32),
                  slot_src=((P, N), torch.int32), resampled=((P,), torch.uint8),
                  n_ties=((P,), torch.int32), bonus=((P, N), torch.int32))
    for f in fields:
        shp, dt = shapes[f]
        if getattr(out, f) is None:
            setattr(out, f, _empty(shp, dt, dev))
        else:
            _chk(getattr(out, f), f"out.{f}", (dt,), shp, dev)
    return out


_ALL_W = ("logw", "logp_tok", "logq_tok", "lse", "ess", "wnorm", "status")
_ALL_S = _ALL_W + ("logw_pre", "ancestors", "offspring", "slot_src", "resampled", "n_ties")


def smcsd_weights(logits_p, logits_q, tokens, *, V=None, n_drafted=None, logw_prev=None,
                  alpha=1.0, inv_temp_p=1.0, inv_temp_q=1.0, out: Outputs | None = None,
                  fields=_ALL_W, workspace=None, stream=None) -> Outputs:
    """S1-S4.  logits_*: [P][N][rows][ld] bf16/fp32 CUDA tensors; tokens [P][N][K] int32."""
    ld_p, rpp_p = _logits_geom(logits_p, "logits_p")
    ld_q, rpp_q = _logits_geom(logits_q, "logits_q")
    if logits_p.dtype != logits_q.dtype:
        raise TypeError("logits_p and logits_q must share a dtype")
    P, N, K = tokens.shape
    V = ld_p if V is None else V
    dev = logits_p.device
    _check_inputs(dev, P, N, K, tokens=tokens, n_drafted=n_drafted, logw_prev=logw_prev)
    if logits_q.device != dev:
        raise ValueError("logits_p and logits_q must be on one device")
    out = _alloc(out or Outputs(), dev, P, N, K, ("logw", "status") + tuple(fields))
    ws = _ws(workspace, dev, P, N, K, V, stream)
    rc = _lib.smcsd_weights(_p(logits_p), ld_p, rpp_p, _p(logits_q), ld_q, rpp_q,
                            _dtype_code(logits_p), _p(tokens), _p(n_drafted), _p(logw_prev),
                            P, N, K, V, alpha, inv_temp_p, inv_temp_q, _p(out.logw),
                            _p(out.logp_tok), _p(out.logq_tok), _p(out.lse), _p(out.ess),
                            _p(out.wnorm), _p(out.status), _p(ws), ws.numel(), _stream(stream))
    _check("smcsd_weights", rc)
    return out


def _step_args(logits_p, logits_q, tokens, *, V=None, n_drafted=None, logw_prev=None,
               alpha=1.0, inv_temp_p=1.0, inv_temp_q=1.0, eta=None,
               scheme=SMCSD_SYSTEMATIC, seed=0x5EED5EED, step=0, prompt_base=0, uniforms=None,
               out: Outputs | None = None, fields=_ALL_S, workspace=None, stream=None, bonus=False):
    """Validated smcsd_step argument list (in ABI order) and the Outputs it writes."""
    ld_p, rpp_p = _logits_geom(logits_p, "logits_p")
    ld_q, rpp_q = _logits_geom(logits_q, "logits_q")
    if logits_p.dtype != logits_q.dtype:
        raise TypeError("logits_p and logits_q must share a dtype")
    P, N, K = tokens.shape
    V = ld_p if V is None else V
    dev = logits_p.device
    _check_inputs(dev, P, N, K, tokens=tokens, n_drafted=n_drafted, logw_prev=logw_prev,
                  uniforms=uniforms, scheme=scheme)
    if logits_q.device != dev:
        raise ValueError("logits_p and logits_q must be on one device")
    eta = _resolve_eta(eta, N)
    out = _alloc(out or Outputs(), dev, P, N, K,
                 ("logw", "status", "ancestors", "resampled") + tuple(fields)
                 + (("bonus",) if bonus else ()))
    ws = _ws(workspace, dev, P, N, K, V, stream)
    args = [_p(logits_p), ld_p, rpp_p, _p(logits_q), ld_q, rpp_q,
            _dtype_code(logits_p), _p(tokens), _p(n_drafted), _p(logw_prev),
            P, N, K, V, alpha, inv_temp_p, inv_temp_q, eta, scheme,
            seed & (2 ** 64 - 1), step & (2 ** 64 - 1), prompt_base, _p(uniforms),
            _p(out.logw), _p(out.logw_pre), _p(out.logp_tok), _p(out.logq_tok),
            _p(out.lse), _p(out.ess), _p(out.wnorm), _p(out.status),
            _p(out.ancestors), _p(out.offspring), _p(out.slot_src),
            _p(out.resampled), _p(out.n_ties), _p(out.bonus) if bonus else None,
            _p(ws), ws.numel(), _stream(stream)]
    return args, out, ws


def smcsd_step(logits_p, logits_q, tokens, *, V=None, n_drafted=None, logw_prev=None,
               alpha=1.0, inv_temp_p=1.0, inv_temp_q=1.0, eta=None,
               scheme=SMCSD_SYSTEMATIC, seed=0x5EED5EED, step=0, prompt_base=0, uniforms=None,
               out: Outputs | None = None, fields=_ALL_S, workspace=None,
               stream=None, bonus=False) -> Outputs:
    """Fused S1-S7 (one launch).  bonus=True also draws the bonus token x+ of every particle
    from target row k_n (NEXT #2; logits_p needs K+1 rows) into out.bonus [P][N].
    eta: resample iff ESS < eta; None = N/2 (reading G2), math.inf forces a resample."""
    args, out, _ = _step_args(logits_p, logits_q, tokens, V=V, n_drafted=n_drafted,
                           logw_prev=logw_prev, alpha=alpha, inv_temp_p=inv_temp_p,
                           inv_temp_q=inv_temp_q, eta=eta, scheme=scheme, seed=seed, step=step,
                           prompt_base=prompt_base, uniforms=uniforms, out=out, fields=fields,
                           workspace=workspace, stream=stream, bonus=bonus)
    _check("smcsd_step", _lib.smcsd_step(*args))
    return out


class StepPlan:
    """smcsd_step with its argument list prepared once (plumbing for tight decode loops: the
    binding's per-call validation and marshalling cost ~25 us of host time, more than a cfg2
    step on the GPU).  run() swaps in new logits / tokens of the SAME shape, dtype and device
    and the step counter, then makes the one C call.  Outputs land in plan.out.  Everything
    else -- output buffers, workspace, scalars and the CUDA stream (the current one at
    construction unless stream= is given) -- is fixed at construction."""
    _I_LP, _I_LQ, _I_TOK, _I_STEP = 0, 3, 7, 20

    def __init__(self, logits_p, logits_q, tokens, **kw):
        # The plan keeps a private workspace (a raw tensor passed as workspace= is used as is
        # and must be exclusive to the plan): run() skips Workspace's shape bookkeeping, so a
        # shared Workspace could be regrown (freeing the buffer the plan writes) or re-zeroed /
        # overwritten by another shape's call between runs.
        ws = kw.get("workspace")
        if ws is None or isinstance(ws, Workspace):
            kw["workspace"] = Workspace(logits_p.device)
        self._args, self.out, self._ws = _step_args(logits_p, logits_q, tokens, **kw)
        self._ws_owner = kw["workspace"]           # keeps the buffer alive as long as the plan
        self._sig = (tuple(logits_p.shape), tuple(logits_q.shape), tuple(tokens.shape),
                     logits_p.dtype, logits_p.device)
        ctypes_types = _lib.smcsd_step.argtypes
        # pre-convert every argument to its ctypes type once
        self._c = [t(a) if a is not None else None for t, a in zip(ctypes_types, self._args)]
        self._fn = _lib.smcsd_step

    def run(self, logits_p=None, logits_q=None, tokens=None, *, step=None):
        c = self._c
        if logits_p is not None:
            if (tuple(logits_p.shape), tuple(logits_q.shape), tuple(tokens.shape),
                    logits_p.dtype, logits_p.device) != self._sig or logits_q.dtype != logits_p.dtype:
                raise ValueError("StepPlan.run: inputs differ in shape/dtype/device from the plan")
            if not (logits_p.is_contiguous() and logits_q.is_contiguous() and tokens.is_contiguous()):
                raise ValueError("StepPlan.run: inputs must be contiguous")
            c[self._I_LP] = ctypes.c_void_p(logits_p.data_ptr())
            c[self._I_LQ] = ctypes.c_void_p(logits_q.data_ptr())
            c[self._I_TOK] = ctypes.c_void_p(tokens.data_ptr())
        if step is not None:
            c[self._I_STEP] = ctypes.c_uint64(step & (2 ** 64 - 1))
        _check("smcsd_step", self._fn(*c))
        return self.out


def smcsd_resample(logw, *, eta=None, scheme=SMCSD_SYSTEMATIC, seed=0x5EED5EED, step=0,
                   prompt_base=0, uniforms=None, out: Outputs | None = None,
                   fields=("offspring", "slot_src", "ess", "lse", "wnorm", "n_ties"),
                   stream=None) -> Outputs:
    """S4-S7 from fp32 log-weights [P][N].  eta: None = N/2 (reading G2), math.inf forces."""
    if logw.dim() != 2:
        raise ValueError("logw must be [P][N]")
    P, N = logw.shape
    _chk(logw, "logw", _F32, (P, N), logw.device, optional=False)
    _chk(uniforms, "uniforms", _U32, (P,) if scheme == SMCSD_SYSTEMATIC else (P, N), logw.device)
    eta = _resolve_eta(eta, N)
    out = _alloc(out or Outputs(), logw.device, P, N, 1,
                 ("ancestors", "logw", "resampled", "status") + tuple(fields))
    rc = _lib.smcsd_resample(_p(logw), P, N, prompt_base, eta, scheme, seed & (2 ** 64 - 1),
                             step & (2 ** 64 - 1), _p(uniforms), _p(out.ancestors),
                             _p(out.offspring), _p(out.slot_src), _p(out.logw), _p(out.resampled),
                             _p(out.ess), _p(out.lse), _p(out.wnorm), _p(out.n_ties),
                             _p(out.status), _stream(stream))
    _check("smcsd_resample", rc)
    return out


def smcsd_weights_partial(logits_p, logits_q, tokens, *, v_begin, v_len=None, n_drafted=None,
                          inv_temp_p=1.0, inv_temp_q=1.0, partials=None, workspace=None,
                          stream=None) -> torch.Tensor:
    """S1 on a vocab shard: rows of logits_* hold columns [v_begin, v_begin + v_len)
    (v_len defaults to the row pitch).  Returns partials [P][2][N][K][4] (log2 domain)."""
    ld_p, rpp_p = _logits_geom(logits_p, "logits_p")
    ld_q, rpp_q = _logits_geom(logits_q, "logits_q")
    P, N, K = tokens.shape
    v_len = ld_p if v_len is None else v_len
    dev = logits_p.device
    _check_inputs(dev, P, N, K, tokens=tokens, n_drafted=n_drafted)
    if partials is None:
        partials = _empty((P, 2, N, K, 4), torch.float32, dev)
    ws = _ws(workspace, dev, P, N, K, v_len, stream)
    rc = _lib.smcsd_weights_partial(_p(logits_p), ld_p, rpp_p, _p(logits_q), ld_q, rpp_q,
                                    _dtype_code(logits_p), _p(tokens), _p(n_drafted), P, N, K,
                                    v_begin, v_len, inv_temp_p, inv_temp_q, _p(partials), _p(ws),
                                    ws.numel(), _stream(stream))
    _check("smcsd_weights_partial", rc)
    return partials


def smcsd_weights_combine(gathered, tokens, *, V, n_drafted=None, logw_prev=None, alpha=1.0,
                          out: Outputs | None = None, fields=_ALL_W, workspace=None,
                          stream=None) -> Outputs:
    """S2-S4 from G gathered shard partials [G][P][2][N][K][4] (rank order)."""
    G = gathered.shape[0]
    P, N, K = tokens.shape
    dev = gathered.device
    _check_inputs(dev, P, N, K, tokens=tokens, n_drafted=n_drafted, logw_prev=logw_prev)
    _chk(gathered, "gathered", _F32, (G, P, 2, N, K, 4), dev, optional=False)
    out = _alloc(out or Outputs(), dev, P, N, K, ("logw", "status") + tuple(fields))
    ws = _ws(workspace, dev, P, N, K, 1, stream)
    rc = _lib.smcsd_weights_combine(_p(gathered), G, _p(tokens), _p(n_drafted), _p(logw_prev),
                                    P, N, K, V, alpha, _p(out.logw), _p(out.logp_tok),
                                    _p(out.logq_tok), _p(out.lse), _p(out.ess), _p(out.wnorm),
                                    _p(out.status), _p(ws), ws.numel(), _stream(stream))
    _check("smcsd_weights_combine", rc)
    return out


def smcsd_select(logw, *, seed=0x5EED5EED, step=0, prompt_base=0, uniforms=None, selected=None,
                 status=None, workspace=None, stream=None):
    """Terminal selection: one particle index per prompt (-1 if degenerate)."""
    P, N = logw.shape
    dev = logw.device
    _chk(logw, "logw", _F32, (P, N), dev, optional=False)
    _chk(uniforms, "uniforms", _U32, (P,), dev)
    selected = _empty((P,), torch.int32, dev) if selected is None else selected
    status = _empty((P,), torch.int32, dev) if status is None else status
    ws = _ws(workspace, dev, P, N, 1, 1, stream)
    rc = _lib.smcsd_select(_p(logw), P, N, prompt_base, seed & (2 ** 64 - 1), step & (2 ** 64 - 1),
                           _p(uniforms), _p(selected), _p(status), _p(ws), ws.numel(), _stream(stream))
    _check("smcsd_select", rc)
    return selected, status


def smcsd_powersmc_weights(logits, *, V=None, logw_prev=None, alpha=1.0, inv_temp=1.0,
                           out: Outputs | None = None, workspace=None, stream=None) -> Outputs:
    """PowerSMC S1-S4 (App. F): log w = ln sum_v p_v^alpha of each particle's row 0.
    Outputs: logw, logp_tok (= per-particle log w, [P][N]), lse, ess, wnorm, status."""
    ld, rpp = _logits_geom(logits, "logits")
    P, N = logits.shape[0], logits.shape[1]
    V = ld if V is None else V
    dev = logits.device
    _chk(logw_prev, "logw_prev", _F32, (P, N), dev)
    out = out or Outputs()
    if out.logp_tok is None:
        out.logp_tok = _empty((P, N), torch.float32, dev)
    out = _alloc(out, dev, P, N, 1, ("logw", "status", "lse", "ess", "wnorm"))
    ws = _ws(workspace, dev, P, N, 1, V, stream)
    rc = _lib.smcsd_powersmc_weights(_p(logits), ld, rpp, _dtype_code(logits), _p(logw_prev), P, N, V,
                                     alpha, inv_temp, _p(out.logw), _p(out.logp_tok), _p(out.lse),
                                     _p(out.ess), _p(out.wnorm), _p(out.status), _p(ws), ws.numel(),
                                     _stream(stream))
    _check("smcsd_powersmc_weights", rc)
    return out


def smcsd_tp_exchange_bytes(P: int, N: int, K: int, G: int, xnseg: int) -> int:
    return int(_lib.smcsd_tp_exchange_bytes(P, N, K, G, xnseg))


def smcsd_tp_exchange_init(xbuf: torch.Tensor, stream=None):
    _check("smcsd_tp_exchange_init", _lib.smcsd_tp_exchange_init(_p(xbuf), xbuf.numel(), _stream(stream)))


def smcsd_ipc_handle_bytes() -> int:
    return int(_lib.smcsd_ipc_handle_bytes())


def smcsd_ipc_export(t: torch.Tensor) -> bytes:
    """Opaque bytes naming t's device address for another process (IPC handle + offset)."""
    buf = ctypes.create_string_buffer(smcsd_ipc_handle_bytes())
    _check("smcsd_ipc_export", _lib.smcsd_ipc_export(_p(t), buf))
    return buf.raw


def smcsd_ipc_open(handle: bytes) -> int:
    ptr = ctypes.c_void_p()
    _check("smcsd_ipc_open", _lib.smcsd_ipc_open(handle, ctypes.byref(ptr)))
    return int(ptr.value)


def smcsd_ipc_close(ptr: int, handle: bytes):
    _check("smcsd_ipc_close", _lib.smcsd_ipc_close(ptr, handle))


def smcsd_tp_step(logits_p, logits_q, tokens, *, V, v_begin, rank, G, xnseg, epoch, xpeer, xlocal,
                  v_len=None, n_drafted=None, logw_prev=None, alpha=1.0, inv_temp_p=1.0, inv_temp_q=1.0,
                  eta=None, scheme=SMCSD_SYSTEMATIC, seed=0x5EED5EED, step=0, prompt_base=0,
                  uniforms=None, out: Outputs | None = None, fields=_ALL_S, workspace=None,
                  stream=None) -> Outputs:
    """S1 + fused peer-memory exchange (S10) + S2-S7 on this rank's vocabulary shard.
    logits_* rows hold columns [v_begin, v_begin + v_len); xpeer: int64 device tensor [G] of
    every rank's exchange buffer address in this process; xlocal: this rank's buffer."""
    ld_p, rpp_p = _logits_geom(logits_p, "logits_p")
    ld_q, rpp_q = _logits_geom(logits_q, "logits_q")
    if logits_p.dtype != logits_q.dtype:
        raise TypeError("logits_p and logits_q must share a dtype")
    if xpeer.dtype != torch.int64 or xpeer.numel() != G or not xpeer.is_cuda:
        raise ValueError("xpeer must be an int64 CUDA tensor of G buffer addresses")
    P, N, K = tokens.shape
    v_len = min(ld_p, V - v_begin) if v_len is None else v_len
    dev = logits_p.device
    _check_inputs(dev, P, N, K, tokens=tokens, n_drafted=n_drafted, logw_prev=logw_prev,
                  uniforms=uniforms, scheme=scheme)
    if logits_q.device != dev or xlocal.device != dev or xpeer.device != dev:
        raise ValueError("logits, xlocal and xpeer must be on one device")
    eta = _resolve_eta(eta, N)
    out = _alloc(out or Outputs(), dev, P, N, K,
                 ("logw", "status", "ancestors", "resampled") + tuple(fields))
    ws = _ws(workspace, dev, P, N, K, v_len, stream)
    rc = _lib.smcsd_tp_step(_p(logits_p), ld_p, rpp_p, _p(logits_q), ld_q, rpp_q,
                            _dtype_code(logits_p), _p(tokens), _p(n_drafted), _p(logw_prev),
                            P, N, K, V, v_begin, v_len, alpha, inv_temp_p, inv_temp_q, eta, scheme,
                            seed & (2 ** 64 - 1), step & (2 ** 64 - 1), prompt_base, _p(uniforms),
                            rank, G, xnseg, epoch & 0xFFFFFFFF, _p(xpeer), _p(xlocal),
                            _p(out.logw), _p(out.logw_pre), _p(out.logp_tok), _p(out.logq_tok),
                            _p(out.lse), _p(out.ess), _p(out.wnorm), _p(out.status),
                            _p(out.ancestors), _p(out.offspring), _p(out.slot_src),
                            _p(out.resampled), _p(out.n_ties), _p(ws), ws.numel(), _stream(stream))
    _check("smcsd_tp_step", rc)
    return out


def smcsd_kv_reindex_paged(table_src, n_pages_src, refcount, src_index, *, table_dst=None,
                           n_pages_dst=None, freed=None, status=None, stream=None):
    """Paged (pointer) reindex: block-table rows + refcounts, no KV bytes."""
    P, N, MP = table_src.shape
    dev = table_src.device
    _chk(table_src, "table_src", _I32, (P, N, MP), dev, optional=False)
    _chk(n_pages_src, "n_pages_src", _I32, (P, N), dev, optional=False)
    _chk(src_index, "src_index", _I32, (P, N), dev, optional=False)
    if refcount.dtype != torch.int32 or refcount.device != dev or not refcount.is_contiguous():
        raise ValueError("refcount must be a contiguous int32 tensor on the tables' device")
    table_dst = torch.empty_like(table_src) if table_dst is None else table_dst
    n_pages_dst = torch.empty_like(n_pages_src) if n_pages_dst is None else n_pages_dst
    status = _empty((P,), torch.int32, dev) if status is None else status
    rc = _lib.smcsd_kv_reindex_paged(_p(table_src), _p(n_pages_src), _p(table_dst), _p(n_pages_dst),
                                     _p(refcount), _p(freed), _p(src_index), P, N, MP,
                                     refcount.numel(), _p(status), _stream(stream))
    _check("smcsd_kv_reindex_paged", rc)
    return table_dst, n_pages_dst, status


def kv_geometry(kv: torch.Tensor, seq_len: int | None = None) -> dict:
    """Strides for a dense KV cache laid out [L][2][P][N][H][S][d] (any element type)."""
    if kv.dim() != 7 or not kv.is_contiguous():
        raise ValueError("kv must be a contiguous [L][2][P][N][H][S][d] tensor")
    L, C, P, N, H, S, d = kv.shape
    e = kv.element_size()
    seq_len = S if seq_len is None else seq_len
    return dict(n_outer=L * C, outer_stride=P * N * H * S * d * e, prompt_stride=N * H * S * d * e,
                particle_stride=H * S * d * e, seg_count=H, seg_bytes=seq_len * d * e,
                seg_stride=S * d * e)


def smcsd_partials_rescale(partials, max_partials, out=None, *, stream=None):
    """S10 all-reduce form, step 3: {M, s 2^(m - M), X, 0} per row from this rank's partials
    [..., 4] and their all_reduce(MAX) (see include/smcsd.h)."""
    out = torch.empty_like(partials) if out is None else out
    rows = partials.numel() // 4
    _check("smcsd_partials_rescale", _lib.smcsd_partials_rescale(_p(partials), _p(max_partials), _p(out),
                                                                 rows, _stream(stream)))
    return out


def kv_tensor(dst, src, *, n_outer, outer_stride, prompt_stride, particle_stride, seg_count,
              seg_bytes, seg_stride):
    """One entry of smcsd_kv_reindex_multi: (dst, src) device tensors and their byte geometry
    (as kv_geometry returns it); dst is src for the in-place slot plan."""
    return (dst, src, dict(n_outer=n_outer, outer_stride=outer_stride, prompt_stride=prompt_stride,
                           particle_stride=particle_stride, seg_count=seg_count, seg_bytes=seg_bytes,
                           seg_stride=seg_stride))


def smcsd_kv_reindex_multi(tensors, src_index, *, status=None, stream=None):
    """S8/S9 over several state tensors in one launch (per-layer K/V tensors, token history):
    tensors is a list of kv_tensor(...) entries sharing src_index [P][N].  status (optional,
    int32 [P]) receives ST_BAD_INDEX for a prompt with an out-of-range or hazardous index."""
    P, N = src_index.shape
    _chk(src_index, "src_index", _I32, (P, N), src_index.device, optional=False)
    _chk(status, "status", _I32, (P,), src_index.device)
    arr = (_KvTensor * len(tensors))()
    for k, (dst, src, g) in enumerate(tensors):
        if dst.device != src_index.device or src.device != src_index.device:
            raise ValueError("state tensors and src_index must be on one device")
        arr[k] = _KvTensor(_p(dst), _p(src), g["n_outer"], g["outer_stride"], g["prompt_stride"],
                           g["particle_stride"], g["seg_count"], g["seg_bytes"], g["seg_stride"])
    rc = _lib.smcsd_kv_reindex_multi(arr, len(tensors), _p(src_index), P, N, _p(status),
                                     _stream(stream))
    _check("smcsd_kv_reindex_multi", rc)
    return status


def smcsd_kv_reindex(dst, src, src_index, *, n_outer, outer_stride, prompt_stride,
                     particle_stride, seg_count, seg_bytes, seg_stride, status=None, stream=None):
    """S8/S9 block gather; pass dst is src for the in-place slot plan.  status: see
    smcsd_kv_reindex_multi."""
    P, N = src_index.shape
    _chk(src_index, "src_index", _I32, (P, N), src_index.device, optional=False)
    _chk(status, "status", _I32, (P,), src_index.device)
    if dst.device != src_index.device or src.device != src_index.device:
        raise ValueError("dst, src and src_index must be on one device")
    rc = _lib.smcsd_kv_reindex(_p(dst), _p(src), n_outer, outer_stride, prompt_stride,
                               particle_stride, seg_count, seg_bytes, seg_stride, _p(src_index),
                               P, N, _p(status), _stream(stream))
    _check("smcsd_kv_reindex", rc)
    return status


# ------------------------------------------------------------------------------------------
# Paged append with copy-on-write (NEXT #1; include/smcsd.h)
# ------------------------------------------------------------------------------------------
def kv_pool(pool: torch.Tensor, *, n_planes, plane_stride, page_stride, token_bytes):
    """One KV pool descriptor: (device tensor, byte geometry) -- see paged_pool_geometry."""
    return (pool, dict(n_planes=n_planes, plane_stride=plane_stride, page_stride=page_stride,
                       token_bytes=token_bytes))


def paged_pool_geometry(pool: torch.Tensor) -> dict:
    """Byte geometry of a contiguous paged KV pool laid out [planes][num_pages][page_size][H][d]
    (planes = L x {K, V}; the per-layer [2][num_blocks][block][H][d] tensors of a serving
    engine are one pool each with 2 planes)."""
    if pool.dim() != 5 or not pool.is_contiguous():
        raise ValueError("pool must be a contiguous [planes][num_pages][page_size][H][d] tensor")
    Lp, G, S, H, d = pool.shape
    e = pool.element_size()
    return dict(n_planes=Lp, plane_stride=G * S * H * d * e, page_stride=S * H * d * e,
                token_bytes=H * d * e)


@dataclass
class AppendOutputs:
    slot_mapping: torch.Tensor = None
    cow_src: torch.Tensor = None
    cow_dst: torch.Tensor = None
    cow_tokens: torch.Tensor = None
    status: torch.Tensor = None
    result: torch.Tensor = None


_append_ws = {}


def smcsd_kv_append_workspace_bytes(P: int, N: int, num_pages: int, max_pages: int) -> int:
    return int(_lib.smcsd_kv_append_workspace_bytes(P, N, num_pages, max_pages))


def _append_workspace(dev, stream, P, N, num_pages, max_pages):
    need = smcsd_kv_append_workspace_bytes(P, N, num_pages, max_pages)
    key = (dev.type, dev.index, _stream(stream))
    ent = _append_ws.get(key)
    shape = (P, N, num_pages, max_pages)
    if ent is None or ent[0].numel() < need or ent[1] != shape:
        buf = ent[0] if ent is not None and ent[0].numel() >= need else \
            torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        smcsd_workspace_init(buf, stream)           # zero once per layout; the call keeps it zero
        ent = (buf, shape)
        _append_ws[key] = ent
    return ent[0]


def smcsd_kv_append_paged(table, n_pages, seq_len, refcount, n_new, *, page_size, max_new=None,
                          pools=(), out: AppendOutputs | None = None, stream=None) -> AppendOutputs:
    """Append n_new[p][n] tokens to every particle's page list, copying a shared partial tail
    page first (copy-on-write).  table / n_pages / seq_len / refcount are updated in place;
    pools: kv_pool(...) entries whose copy-on-write content the call copies.  out.result[0] = 1
    means the call changed nothing (see out.status)."""
    if table.dim() != 3:
        raise ValueError("table must be [P][N][max_pages]")
    P, N, MP = table.shape
    dev = table.device
    _chk(table, "table", _I32, (P, N, MP), dev, optional=False)
    for name, t in (("n_pages", n_pages), ("seq_len", seq_len), ("n_new", n_new)):
        _chk(t, name, _I32, (P, N), dev, optional=False)
    if refcount.dim() != 1:
        raise ValueError("refcount must be [num_pages]")
    _chk(refcount, "refcount", _I32, (refcount.numel(),), dev, optional=False)
    if max_new is None:
        max_new = max(1, int(n_new.max().item()))
    out = out or AppendOutputs()
    shapes = dict(slot_mapping=(P, N, max_new), cow_src=(P, N), cow_dst=(P, N), cow_tokens=(P, N),
                  status=(P,), result=(1,))
    for f, shp in shapes.items():
        if getattr(out, f) is None:
            setattr(out, f, torch.empty(shp, dtype=torch.int32, device=dev))
        else:
            _chk(getattr(out, f), f"out.{f}", _I32, shp, dev)
    arr = (_KvPool * max(1, len(pools)))()
    for k, (t, g) in enumerate(pools):
        if t.device != dev:
            raise ValueError("pools must be on the tables' device")
        arr[k] = _KvPool(_p(t), g["n_planes"], g["plane_stride"], g["page_stride"], g["token_bytes"])
    ws = _append_workspace(dev, stream, P, N, refcount.numel(), MP)
    rc = _lib.smcsd_kv_append_paged(_p(table), _p(n_pages), _p(seq_len), _p(refcount), _p(n_new),
                                    P, N, MP, refcount.numel(), page_size, max_new,
                                    _p(out.slot_mapping), _p(out.cow_src), _p(out.cow_dst),
                                    _p(out.cow_tokens), _p(out.status), _p(out.result), arr,
                                    len(pools), _p(ws), ws.numel(), _stream(stream))
    _check("smcsd_kv_append_paged", rc)
    return out
