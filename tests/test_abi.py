"""CPU-side checks of the C ABI: the library loads, exports every symbol include/smcsd.h
declares, and rejects invalid arguments synchronously (EINVAL before any CUDA call).
No compute call is made here (no GPU in the CPU suite)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = []
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            src = open(os.path.join(inc, f)).read()
            names += re.findall(r"SMCSD_API\s+[\w\s\*]+?\b(smcsd_\w+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_smcsd_build", os.path.join(ROOT, "paper_2604_15672_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)  # by path: the package __init__ needs the library to exist
    b.build()
    return ctypes.CDLL(b.LIB)


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) == 26, names
    for n in names:
        assert hasattr(lib, n), n


def test_binding_names_match_abi():
    import paper_2604_15672_b200 as m
    for n in _declared():
        if n in ("smcsd_strerror",):
            continue
        assert callable(getattr(m, n)), n


def test_strerror_and_version(lib):
    lib.smcsd_strerror.restype = ctypes.c_char_p
    lib.smcsd_version.restype = ctypes.c_char_p
    assert lib.smcsd_strerror(0) == b"ok"
    assert lib.smcsd_strerror(1) == b"invalid argument"
    assert b"sm_100a" in lib.smcsd_version()


def test_workspace_bytes(lib):
    lib.smcsd_workspace_bytes.restype = ctypes.c_size_t
    lib.smcsd_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64]
    b1 = lib.smcsd_workspace_bytes(1, 16, 8, 128256)
    b2 = lib.smcsd_workspace_bytes(64, 32, 8, 128256)
    assert b1 >= 2 * 16 * 8 * 16 * 16 and b2 > b1
    assert lib.smcsd_workspace_bytes(0, 16, 8, 128256) == 0


def _weights(lib, lp=0x1000, ld=128256, P=1, N=16, K=8, V=128256, dtype=1, alpha=1.0, tp=1.0,
             ws_bytes=1 << 30, rpp=9):
    vp, i64, i32, f32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_size_t
    lib.smcsd_weights.argtypes = [vp, i64, i32, vp, i64, i32, i32, vp, vp, vp, i32, i32, i32, i64,
                                  f32, f32, f32, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.smcsd_weights.restype = i32
    return lib.smcsd_weights(lp, ld, rpp, 0x2000, ld, K, dtype, 0x3000, None, None, P, N, K, V,
                             alpha, tp, 1.0, 0x4000, None, None, None, None, None, 0x5000, 0x6000,
                             ws_bytes, None)


def test_einval_paths(lib):
    assert _weights(lib, lp=0x1001) == 1                 # misaligned base
    assert _weights(lib, ld=128255) == 1                 # ld not a multiple of 16 bytes
    assert _weights(lib, ld=1000, V=1001) == 1           # ld < V
    assert _weights(lib, rpp=7) == 1                     # rows per particle < K
    assert _weights(lib, P=0) == 1
    assert _weights(lib, dtype=5) == 1
    assert _weights(lib, alpha=0.0) == 1
    assert _weights(lib, alpha=float("nan")) == 1
    assert _weights(lib, tp=-1.0) == 1
    assert _weights(lib, ws_bytes=100) == 1              # workspace too small


def test_resample_and_kv_einval(lib):
    vp, i64, i32, f32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_uint64
    lib.smcsd_resample.argtypes = [vp, i32, i32, i64, f32, i32, u64, u64, vp, vp, vp, vp, vp, vp,
                                   vp, vp, vp, vp, vp, vp]
    lib.smcsd_resample.restype = i32
    args = lambda N, eta, scheme: (0x1000, 1, N, 0, eta, scheme, 1, 2, None, 0x2000, None, None,
                                   0x3000, 0x4000, None, None, None, None, 0x5000, None)
    assert lib.smcsd_resample(*args(1025, 1.0, 0)) == 1          # N > 1024
    assert lib.smcsd_resample(*args(16, float("nan"), 0)) == 1   # NaN eta
    assert lib.smcsd_resample(*args(1025, 1.0, 1)) == 1          # multinomial, N > 1024
    assert lib.smcsd_resample(*args(16, 1.0, 7)) == 1            # unknown scheme
    lib.smcsd_kv_reindex.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, i32, i32, vp, vp]
    lib.smcsd_kv_reindex.restype = i32
    ok = dict(dst=0x10000, src=0x20000, n_outer=4, outer=4096, prompt=2048, particle=512,
              segc=2, segb=256, segs=256)
    def kv(**kw):
        a = {**ok, **kw}
        return lib.smcsd_kv_reindex(a["dst"], a["src"], a["n_outer"], a["outer"], a["prompt"],
                                    a["particle"], a["segc"], a["segb"], a["segs"], 0x30000, 1, 4,
                                    None, None)
    assert kv(segb=100) == 1            # not a multiple of 16
    assert kv(dst=0x10008) == 1         # misaligned
    assert kv(particle=520) == 1
    assert kv(n_outer=0) == 1


def test_kv_reindex_multi_rejects_bad_arguments(lib):
    """smcsd_kv_reindex_multi validates synchronously (EINVAL, nothing enqueued)."""
    import ctypes as c

    class T(c.Structure):
        _fields_ = [("dst", c.c_void_p), ("src", c.c_void_p)] + [
            (n, c.c_int64) for n in ("n_outer", "outer_stride", "prompt_stride", "particle_stride",
                                     "seg_count", "seg_bytes", "seg_stride")]
    lib.smcsd_kv_reindex_multi.argtypes = [c.POINTER(T), c.c_int, c.c_void_p, c.c_int, c.c_int, c.c_void_p,
                                           c.c_void_p]
    lib.smcsd_kv_reindex_multi.restype = c.c_int
    good = T(0x10000, 0x20000, 4, 4096, 2048, 512, 2, 256, 256)
    arr = (T * 2)(good, good)
    assert lib.smcsd_kv_reindex_multi(arr, 0, 0x30000, 1, 4, None, None) == 1      # no tensors
    assert lib.smcsd_kv_reindex_multi(arr, 257, 0x30000, 1, 4, None, None) == 1    # > 256 tensors
    assert lib.smcsd_kv_reindex_multi(None, 1, 0x30000, 1, 4, None, None) == 1     # null list
    assert lib.smcsd_kv_reindex_multi(arr, 2, None, 1, 4, None, None) == 1         # null src_index
    arr[1] = T(0x10000, 0x20008, 4, 4096, 2048, 512, 2, 256, 256)            # misaligned 2nd
    assert lib.smcsd_kv_reindex_multi(arr, 2, 0x30000, 1, 4, None, None) == 1
    arr[1] = T(0x10000, 0x20000, 4, 4096, 2048, 512, 2, 100, 256)            # seg_bytes % 16
    assert lib.smcsd_kv_reindex_multi(arr, 2, 0x30000, 1, 4, None, None) == 1



def test_kv_append_paged_rejects_bad_arguments(lib):
    """smcsd_kv_append_paged validates synchronously (EINVAL, nothing enqueued)."""
    import ctypes as c

    class Pool(c.Structure):
        _fields_ = [("base", c.c_void_p)] + [(n, c.c_int64) for n in
                                              ("n_planes", "plane_stride", "page_stride", "token_bytes")]
    vp, i32, sz = c.c_void_p, c.c_int, c.c_size_t
    lib.smcsd_kv_append_workspace_bytes.argtypes = [i32, i32, i32, i32]
    lib.smcsd_kv_append_workspace_bytes.restype = sz
    wsb = lib.smcsd_kv_append_workspace_bytes(2, 4, 100, 8)
    assert wsb > 0 and lib.smcsd_kv_append_workspace_bytes(0, 4, 100, 8) == 0
    lib.smcsd_kv_append_paged.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp, vp, vp,
                                          vp, vp, vp, c.POINTER(Pool), i32, vp, sz, vp]
    lib.smcsd_kv_append_paged.restype = i32
    good = Pool(0x100000, 2, 1 << 20, 16 * 256, 256)
    arr = (Pool * 1)(good)
    A = [0x1000, 0x2000, 0x3000, 0x4000, 0x5000]
    O = [0x6000, 0x7000, 0x8000, 0x9000, 0xa000, 0xb000]

    def call(P=2, N=4, MP=8, NP=100, page=16, mx=9, pools=arr, npool=1, ws=0x200000, wb=wsb):
        return lib.smcsd_kv_append_paged(*A, P, N, MP, NP, page, mx, *O, pools, npool, ws, wb, None)
    assert call(page=0) == 1
    assert call(NP=1 << 28, page=16) == 1                   # num_pages * page_size >= 2^31
    assert call(wb=wsb - 1) == 1                            # short workspace
    assert call(npool=65) == 1
    arr[0] = Pool(0x100008, 2, 1 << 20, 16 * 256, 256)      # misaligned pool
    assert call() == 1
    arr[0] = Pool(0x100000, 2, 1 << 20, 16 * 256, 100)      # token bytes not a multiple of 16
    assert call() == 1
    arr[0] = Pool(0x100000, 2, 1 << 20, 256, 256)           # page stride < page_size x token
    assert call() == 1
    assert lib.smcsd_kv_append_paged(None, *A[1:], 2, 4, 8, 100, 16, 9, *O, arr, 0, 0x200000, wsb,
                                     None) == 1
