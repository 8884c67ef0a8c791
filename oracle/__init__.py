"""CPU oracle for the SMC-SD verification hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2604_15672_b200`` never imports it, and the C source here shares no code with
``paper_2604_15672_b200/csrc``.

The arithmetic lives in ``smcsd_oracle.c`` (plain fp64 loops, built with
``-ffp-contract=off``); this module only builds it and marshals numpy arrays.
Every function cites the PAPER.md passage it follows (see the C file).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smcsd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")     # timing-only build (-fopenmp)
_libs = {}
_threads = 1

ST_DEGENERATE = 1
ST_NOT_ABSCONT = 2
ST_BAD_TOKEN = 4
ST_NONFINITE = 8
ST_BAD_PAGE = 16
ST_BAD_INDEX = 64
ST_OUT_OF_PAGES = 128


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FMA contraction): liboracle.so (plain,
    single-threaded) and liboracle_omp.so (the same source with -fopenmp, timing only)."""
    for out, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
            cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                   *extra, "-shared", "-o", out + ".tmp", _SRC, "-lm"]
            subprocess.run(cmd, check=True)
            os.replace(out + ".tmp", out)
    return _LIB


def set_threads(n: int) -> int:
    """Select the plain build (n = 1) or the OpenMP timing build with n threads (n > 1) for
    the following calls.  Returns the threads the selected build will use."""
    global _threads
    _threads = max(1, int(n))
    L = lib()
    return int(L.orc_set_threads(_threads)) if _threads > 1 else 1


def lib():
    key = "omp" if _threads > 1 else "plain"
    if key not in _libs:
        build()
        L = ctypes.CDLL(_LIB_OMP if key == "omp" else _LIB)
        vp, i64, i32, dbl, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
        L.orc_philox4x32_10.argtypes = [vp, vp, vp]
        L.orc_row_logprob.argtypes = [vp, i32, i64, dbl, i64, vp]
        L.orc_row_logprob.restype = dbl
        L.orc_row_partial.argtypes = [vp, i32, i64, i64, dbl, i64, vp]
        L.orc_row_partial.restype = i32
        L.orc_combine_partials.argtypes = [vp, i32, i64, vp]
        L.orc_combine_partials.restype = dbl
        L.orc_weights.argtypes = [vp, i64, i32, vp, i64, i32, i32, vp, vp, vp, i32, i32, i32, i64,
                                  dbl, dbl, dbl, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_resample.argtypes = [vp, i32, i32, i64, dbl, i32, u64, u64, vp, vp, vp, vp, vp, vp,
                                   vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_select.argtypes = [vp, i32, i32, i64, u64, u64, vp, vp, vp, vp]
        L.orc_powersmc_weights.argtypes = [vp, i64, i32, i32, vp, i32, i32, i64, dbl, dbl, vp, vp,
                                           vp, vp, vp, vp, vp]
        L.orc_bonus.argtypes = [vp, i64, i32, i32, vp, i32, i32, i32, i64, dbl, u64, u64, i64, i64,
                                vp, vp, vp, vp, vp, vp]
        L.orc_kv_reindex.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, i32, i32, vp]
        L.orc_kv_reindex_paged.argtypes = [vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, vp]
        L.orc_kv_append_paged.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp, vp,
                                          vp, vp, vp, vp]
        L.orc_paged_cow_copy.argtypes = [vp, i64, i64, i64, i64, vp, vp, vp, i64]
        L.orc_set_threads.argtypes = [i32]
        L.orc_set_threads.restype = i32
        _libs[key] = L
    return _libs[key]


def _ptr(a):
    return None if a is None else a.ctypes.data


def _dtype_code(arr: np.ndarray) -> int:
    if arr.dtype == np.float32:
        return 0
    if arr.dtype == np.uint16:   # bf16 bit patterns
        return 1
    raise TypeError(f"logits must be float32 or uint16 (bf16 bits), got {arr.dtype}")


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def row_logprob(row: np.ndarray, d: int, tau: float = 1.0):
    """ell = log-softmax(tau*z)[d] in fp64.  Returns (ell, flag)."""
    row = np.ascontiguousarray(row)
    flag = np.zeros(1, dtype=np.uint32)
    ell = lib().orc_row_logprob(_ptr(row), _dtype_code(row), row.shape[-1], float(tau), int(d), _ptr(flag))
    return ell, int(flag[0])


def row_partial(row_shard: np.ndarray, v_begin: int, d: int, tau: float = 1.0):
    """(m, s, x) of one vocab shard, natural-log domain; returns (array[3], has_nan_or_posinf)."""
    row_shard = np.ascontiguousarray(row_shard)
    out = np.zeros(3, dtype=np.float64)
    bad = lib().orc_row_partial(_ptr(row_shard), _dtype_code(row_shard), int(v_begin),
                                row_shard.shape[-1], float(tau), int(d), _ptr(out))
    return out, bool(bad)


def combine_partials(parts: np.ndarray):
    """Merge [G][3] shard partials in rank order -> (ell, flag)."""
    parts = np.ascontiguousarray(parts, dtype=np.float64)
    flag = np.zeros(1, dtype=np.uint32)
    ell = lib().orc_combine_partials(_ptr(parts), parts.shape[0], 3, _ptr(flag))
    return ell, int(flag[0])


def weights(logits_p, logits_q, tokens, *, V=None, n_drafted=None, logw_prev=None,
            alpha=1.0, tau_p=1.0, tau_q=1.0):
    """S1-S4 oracle.  logits_p: [P][N][rpp_p][ld], logits_q: [P][N][rpp_q][ld] (float32 or
    uint16 bf16 bits), tokens: [P][N][K] int32.  Returns a dict of numpy outputs."""
    lp = np.ascontiguousarray(logits_p)
    lq = np.ascontiguousarray(logits_q)
    assert lp.dtype == lq.dtype
    tok = np.ascontiguousarray(tokens, dtype=np.int32)
    P, N, K = tok.shape
    ld_p, rpp_p = lp.shape[-1], lp.shape[-2]
    ld_q, rpp_q = lq.shape[-1], lq.shape[-2]
    V = ld_p if V is None else V
    nd = None if n_drafted is None else np.ascontiguousarray(n_drafted, dtype=np.int32)
    lw = None if logw_prev is None else np.ascontiguousarray(logw_prev, dtype=np.float32)
    out = dict(logw=np.zeros((P, N), np.float32), logp_tok=np.zeros((P, N, K)),
               logq_tok=np.zeros((P, N, K)), lse=np.zeros(P), ess=np.zeros(P),
               wnorm=np.zeros((P, N)), status=np.zeros(P, np.uint32))
    scratch = np.zeros(2 * N)
    lib().orc_weights(_ptr(lp), ld_p, rpp_p, _ptr(lq), ld_q, rpp_q, _dtype_code(lp), _ptr(tok),
                      _ptr(nd), _ptr(lw), P, N, K, V, float(alpha), float(tau_p), float(tau_q),
                      _ptr(out["logw"]), _ptr(out["logp_tok"]), _ptr(out["logq_tok"]),
                      _ptr(out["lse"]), _ptr(out["ess"]), _ptr(out["wnorm"]), _ptr(out["status"]),
                      _ptr(scratch))
    return out


def resample(logw, *, eta=float("inf"), seed=0x5EED5EED, step=0, prompt_base=0, uniforms=None,
             scheme=0):
    """S4-S7 oracle from fp32 log-weights [P][N]; scheme 0 systematic, 1 multinomial
    (uniforms override: [P] words for systematic, [P][N] for multinomial)."""
    lw = np.ascontiguousarray(logw, dtype=np.float32)
    P, N = lw.shape
    un = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.uint32)
    out = dict(ancestors=np.zeros((P, N), np.int32), offspring=np.zeros((P, N), np.int32),
               slot_src=np.zeros((P, N), np.int32), logw=np.zeros((P, N), np.float32),
               resampled=np.zeros(P, np.uint8), ess=np.zeros(P), lse=np.zeros(P),
               n_ties=np.zeros(P, np.int32), status=np.zeros(P, np.uint32),
               wnorm=np.zeros((P, N)), cdf=np.zeros((P, N)))
    scratch = np.zeros(4 * N)
    iscratch = np.zeros(3 * N, np.int32)
    lib().orc_resample(_ptr(lw), P, N, int(prompt_base), float(eta), int(scheme), int(seed) & (2**64 - 1),
                       int(step) & (2**64 - 1), _ptr(un), _ptr(out["ancestors"]),
                       _ptr(out["offspring"]), _ptr(out["slot_src"]), _ptr(out["logw"]),
                       _ptr(out["resampled"]), _ptr(out["ess"]), _ptr(out["lse"]),
                       _ptr(out["n_ties"]), _ptr(out["status"]), _ptr(out["wnorm"]),
                       _ptr(out["cdf"]), _ptr(scratch), _ptr(iscratch))
    return out


def powersmc_weights(logits, *, V=None, logw_prev=None, alpha=1.0, tau=1.0):
    """PowerSMC oracle (App. F): log w = ln sum_x p(x)^alpha of row j = 0."""
    lg = np.ascontiguousarray(logits)
    P, N, rpp, ld = lg.shape
    V = ld if V is None else V
    lw = None if logw_prev is None else np.ascontiguousarray(logw_prev, dtype=np.float32)
    out = dict(logw=np.zeros((P, N), np.float32), inc=np.zeros((P, N)), lse=np.zeros(P),
               ess=np.zeros(P), wnorm=np.zeros((P, N)), status=np.zeros(P, np.uint32))
    scratch = np.zeros(2 * N)
    lib().orc_powersmc_weights(_ptr(lg), ld, rpp, _dtype_code(lg), _ptr(lw), P, N, V, float(alpha),
                               float(tau), _ptr(out["logw"]), _ptr(out["inc"]), _ptr(out["lse"]),
                               _ptr(out["ess"]), _ptr(out["wnorm"]), _ptr(out["status"]), _ptr(scratch))
    return out


def bonus(logits_p, *, K, V=None, n_drafted=None, tau=1.0, seed=0x5EED5EED, step=0, prompt_base=0,
          seg=8192):
    """Bonus-token oracle (NEXT #2; reading G22): one exact draw from
    softmax(tau z) of target row k_n per particle, with segment width `seg` (a parameter of the
    reading).  Returns bonus, seg_margin, key_margin, second (runner-up column of the chosen
    segment), alt (the draw of the segment across the nearest CDF boundary) and status."""
    lg = np.ascontiguousarray(logits_p)
    P, N, rpp, ld = lg.shape
    V = ld if V is None else V
    nd = None if n_drafted is None else np.ascontiguousarray(n_drafted, dtype=np.int32)
    out = dict(bonus=np.zeros((P, N), np.int32), seg_margin=np.zeros((P, N)),
               key_margin=np.zeros((P, N)), second=np.zeros((P, N), np.int32),
               alt=np.zeros((P, N), np.int32), status=np.zeros(P, np.uint32))
    lib().orc_bonus(_ptr(lg), ld, rpp, _dtype_code(lg), _ptr(nd), P, N, K, V, float(tau),
                    int(seed) & (2**64 - 1), int(step) & (2**64 - 1), int(prompt_base), int(seg),
                    _ptr(out["bonus"]), _ptr(out["seg_margin"]), _ptr(out["key_margin"]),
                    _ptr(out["second"]), _ptr(out["alt"]), _ptr(out["status"]))
    return out


def select(logw, *, seed=0x5EED5EED, step=0, prompt_base=0, uniforms=None):
    """Terminal selection oracle: one index per prompt, -1 if degenerate."""
    lw = np.ascontiguousarray(logw, dtype=np.float32)
    P, N = lw.shape
    un = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.uint32)
    sel = np.zeros(P, np.int32)
    st = np.zeros(P, np.uint32)
    scratch = np.zeros(2 * N)
    lib().orc_select(_ptr(lw), P, N, int(prompt_base), int(seed) & (2**64 - 1),
                     int(step) & (2**64 - 1), _ptr(un), _ptr(sel), _ptr(st), _ptr(scratch))
    return dict(selected=sel, status=st)


def kv_reindex(dst: np.ndarray, src: np.ndarray, src_index: np.ndarray, *, n_outer, outer_stride,
               prompt_stride, particle_stride, seg_count, seg_bytes, seg_stride):
    """S8/S9 oracle: byte copies (strides in bytes).  dst is src for in-place.  Returns the
    per-prompt status (ST_BAD_INDEX for an out-of-range or, in place, hazardous index)."""
    idx = np.ascontiguousarray(src_index, dtype=np.int32)
    P, N = idx.shape
    st = np.zeros(P, np.uint32)
    lib().orc_kv_reindex(_ptr(dst), _ptr(src), n_outer, outer_stride, prompt_stride,
                         particle_stride, seg_count, seg_bytes, seg_stride, _ptr(idx), P, N, _ptr(st))
    return st


def kv_reindex_paged(table, n_pages, refcount, src_index, *, num_pages=None):
    """Paged reindex oracle.  table [P][N][max_pages] int32, n_pages [P][N],
    refcount [num_pages] (updated copy returned).  Returns dict of new arrays."""
    t = np.ascontiguousarray(table, dtype=np.int32)
    P, N, MP = t.shape
    npg = np.ascontiguousarray(n_pages, dtype=np.int32)
    rc = np.ascontiguousarray(refcount, dtype=np.int32).copy()
    idx = np.ascontiguousarray(src_index, dtype=np.int32)
    num_pages = rc.size if num_pages is None else num_pages
    out = dict(table=np.zeros_like(t), n_pages=np.zeros_like(npg), refcount=rc,
               freed=np.zeros(num_pages, np.uint8), status=np.zeros(P, np.uint32))
    lib().orc_kv_reindex_paged(_ptr(t), _ptr(npg), _ptr(out["table"]), _ptr(out["n_pages"]),
                               _ptr(rc), _ptr(out["freed"]), _ptr(idx), P, N, MP, num_pages,
                               _ptr(out["status"]))
    return out


def kv_append_paged(table, n_pages, seq_len, refcount, n_new, *, page_size, max_new=None,
                    pools=()):
    """Paged append with copy-on-write oracle (NEXT #1; PAPER.md:488-490, SPEC.md:466-470,
    reading G24).  Arrays are copied, never modified in place: returns a dict with the new
    table / n_pages / seq_len / refcount, slot_mapping [P][N][max_new], cow_src / cow_dst /
    cow_tokens [P][N], status [P] and result (0 ok, 1 nothing changed).  pools: iterable of
    (uint8 array, n_planes, plane_stride, page_stride, token_bytes) KV pools whose copy-on-write
    content is copied in place."""
    t = np.ascontiguousarray(table, dtype=np.int32).copy()
    P, N, MP = t.shape
    npg = np.ascontiguousarray(n_pages, dtype=np.int32).copy()
    sl = np.ascontiguousarray(seq_len, dtype=np.int32).copy()
    rc = np.ascontiguousarray(refcount, dtype=np.int32).copy()
    nn = np.ascontiguousarray(n_new, dtype=np.int32)
    max_new = int(nn.max()) if max_new is None else int(max_new)
    max_new = max(max_new, 1)
    out = dict(table=t, n_pages=npg, seq_len=sl, refcount=rc,
               slot_mapping=np.zeros((P, N, max_new), np.int32), cow_src=np.zeros((P, N), np.int32),
               cow_dst=np.zeros((P, N), np.int32), cow_tokens=np.zeros((P, N), np.int32),
               status=np.zeros(P, np.uint32), result=np.zeros(1, np.int32))
    lib().orc_kv_append_paged(_ptr(t), _ptr(npg), _ptr(sl), _ptr(rc), _ptr(nn), P, N, MP, rc.size,
                              int(page_size), max_new, _ptr(out["slot_mapping"]), _ptr(out["cow_src"]),
                              _ptr(out["cow_dst"]), _ptr(out["cow_tokens"]), _ptr(out["status"]),
                              _ptr(out["result"]))
    out["result"] = int(out["result"][0])
    if out["result"] == 0:
        for pool, n_planes, plane_stride, page_stride, token_bytes in pools:
            lib().orc_paged_cow_copy(_ptr(pool), n_planes, plane_stride, page_stride, token_bytes,
                                     _ptr(out["cow_src"]), _ptr(out["cow_dst"]),
                                     _ptr(out["cow_tokens"]), P * N)
    return out


def neg_log_n(N: int) -> np.float32:
    """The S7 reset value fl32(-ln N) as the oracle computes it (via one resample call)."""
    out = resample(np.zeros((1, N), np.float32), eta=float("inf"))
    return out["logw"][0, 0]
