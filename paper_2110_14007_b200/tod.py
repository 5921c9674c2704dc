"""Thin ctypes binding over libtod.so (include/tod.h).  Argument marshalling
only: every step of the hot path runs in the library's CUDA kernels.  There is
no CPU fallback — if libtod.so is missing or no sm_100 GPU is present, calls
raise.

Accepts torch tensors (CUDA on the context's device, or CPU) and numpy arrays
(host).  Outputs are allocated like the input: CUDA tensors for CUDA input,
numpy arrays for host input (then the library stages the copies inside the
call, which is what bench.py's e2e leg measures).
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtod.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "tod.h")

TOD_OK = 0
STATUS = {0: "TOD_OK", -1: "TOD_E_ARG", -2: "TOD_E_NONFINITE", -3: "TOD_E_RANGE",
          -4: "TOD_E_NOMEM", -5: "TOD_E_CUDA", -6: "TOD_E_NCCL", -7: "TOD_E_UNSUPPORTED",
          -8: "TOD_E_INTERNAL"}
MAX_K = 128  # include/tod.h TOD_MAX_K
FORMATS = {"auto": 0, "fp16": 1, "bf16": 2, "fp32": 3}
F_NO_CERTIFY = 0x1
F_TIMING = 0x2
F_PASS1_V1 = 0x10   # force the single-query-tile tensor-core schedule (knn_tc.cu)
F_MAIN_1SM = 0x20   # run the two-pass main pass on single SMs (knn_tc3.cu), not CTA pairs


class TodError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS.get(status, str(status)), msg))
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("format", ctypes.c_int32), ("kprime", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("stream", ctypes.c_void_p), ("chunks", ctypes.c_int32),
                ("epilogue_split", ctypes.c_int32), ("workspace_bytes", ctypes.c_size_t)]


class Stats(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("certified", ctypes.c_int64),
                ("fallback_rows", ctypes.c_int64), ("kprime", ctypes.c_int32),
                ("format", ctypes.c_int32), ("chunks", ctypes.c_int32), ("dpad", ctypes.c_int32),
                ("scale", ctypes.c_double), ("max_abs_err", ctypes.c_double),
                ("ms_stage", ctypes.c_float), ("ms_prep", ctypes.c_float),
                ("ms_main", ctypes.c_float), ("ms_certify", ctypes.c_float),
                ("ms_fallback", ctypes.c_float), ("ms_lof", ctypes.c_float),
                ("ms_total", ctypes.c_float), ("kernel_launches", ctypes.c_int64),
                ("cand_groups", ctypes.c_int64), ("visited_groups", ctypes.c_int64),
                ("cand_columns", ctypes.c_int64), ("ms_main_kernel", ctypes.c_float),
                ("main_kernel", ctypes.c_int32), ("sample_pass", ctypes.c_int32),
                ("query_chunks", ctypes.c_int32), ("prebound_skipped", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class KnnOut(ctypes.Structure):
    _fields_ = [("idx", ctypes.c_void_p), ("dist", ctypes.c_void_p), ("dist64", ctypes.c_void_p),
                ("score_kth", ctypes.c_void_p), ("score_mean", ctypes.c_void_p),
                ("kdist64", ctypes.c_void_p), ("row_tier", ctypes.c_void_p)]


_lib = None


ABI_VERSION = 4  # include/tod.h TOD_ABI_VERSION


def load_library(path: str = LIB_PATH):
    """Load libtod.so; raise (loudly) if it is missing.  Never falls back."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libtod.so not built (%s); run __graft_entry__.build()" % path)
    lib = ctypes.CDLL(path)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "tod_create": ([ctypes.POINTER(Config), ctypes.POINTER(P)], ctypes.c_int),
        "tod_destroy": ([P], ctypes.c_int),
        "tod_status_str": ([ctypes.c_int], ctypes.c_char_p),
        "tod_last_message": ([P], ctypes.c_char_p),
        "tod_abi_version": ([], I32),
        "tod_build_info": ([], ctypes.c_char_p),
        "tod_knn": ([P, P, I64, I32, I32, I64, I64, ctypes.POINTER(KnnOut), ctypes.POINTER(Stats)],
                    ctypes.c_int),
        "tod_knn_query": ([P, P, I64, P, I64, I32, I32, ctypes.POINTER(KnnOut),
                           ctypes.POINTER(Stats)], ctypes.c_int),
        "tod_lof": ([P, P, I64, I32, I32, P, P, ctypes.POINTER(KnnOut), ctypes.POINTER(Stats)],
                    ctypes.c_int),
        "tod_lof_lrd": ([P, I64, I32, I64, P, P, P, P], ctypes.c_int),
        "tod_abod": ([P, P, I64, I32, I32, I64, I64, P, ctypes.POINTER(KnnOut),
                      ctypes.POINTER(Stats)], ctypes.c_int),
        "tod_knn_classify": ([P, P, I64, P, I64, I32, I32, P, P, ctypes.POINTER(Stats)],
                             ctypes.c_int),
        "tod_nwr": ([P, P, I64, I32, ctypes.c_double, I64, I64, P, P, P, I64,
                     ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(Stats)], ctypes.c_int),
        "tod_lof_finish": ([P, I64, I32, I64, I64, P, P, P, P], ctypes.c_int),
        "tod_debug_mainpass": ([P, P, I64, I32, P, P, P, ctypes.POINTER(ctypes.c_int32),
                                ctypes.POINTER(ctypes.c_int32)], ctypes.c_int),
        "tod_comm_id_create": ([P], ctypes.c_int),
        "tod_comm_init": ([P, P, I32, I32], ctypes.c_int),
        "tod_comm_init_loopback": ([P, I32], ctypes.c_int),
        "tod_shard_rows": ([I64, I32, I32, ctypes.POINTER(ctypes.c_int64),
                            ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
        "tod_knn_sharded": ([P, P, I64, I64, I64, I32, I32, ctypes.POINTER(KnnOut), P, P,
                             ctypes.POINTER(Stats)], ctypes.c_int),
        "tod_lof_sharded": ([P, P, I64, I64, I64, I32, I32, P, P, ctypes.POINTER(KnnOut),
                             ctypes.POINTER(Stats)], ctypes.c_int),
        "tod_workspace_size": ([I64, I32, I32, I64, ctypes.POINTER(Config)], ctypes.c_size_t),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.tod_abi_version() != ABI_VERSION:  # a stale build: struct layouts would disagree
        raise ImportError("libtod.so ABI %d, binding expects %d; rebuild (__graft_entry__.build())"
                          % (lib.tod_abi_version(), ABI_VERSION))
    _lib = lib
    return lib


def comm_id_create() -> bytes:
    """tod_comm_id_create: a fresh 128-byte communicator id (rank 0 of a job)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.tod_comm_id_create(buf)
    if st != TOD_OK:
        raise TodError(st, "tod_comm_id_create failed (libnccl.so.2 not loadable?)")
    return buf.raw


def shard_rows(n: int, world: int, rank: int):
    """tod_shard_rows: the library's balanced 256-row-aligned split (row_offset, n_local)."""
    lib = load_library()
    b, c = ctypes.c_int64(), ctypes.c_int64()
    st = lib.tod_shard_rows(n, world, rank, ctypes.byref(b), ctypes.byref(c))
    if st != TOD_OK:
        raise TodError(st, "tod_shard_rows(n=%d, world=%d, rank=%d)" % (n, world, rank))
    return b.value, c.value


def workspace_size(n: int, d: int, k: int, q_count: int, fmt: str = "auto", kprime: int = 0) -> int:
    """tod_workspace_size: estimated device bytes of one tod_knn call."""
    lib = load_library()
    cfg = Config(device=0, format=FORMATS[fmt], kprime=kprime)
    return int(lib.tod_workspace_size(n, d, k, q_count, ctypes.byref(cfg)))


def header_symbols(header: str = HEADER):
    """Function names declared in include/tod.h."""
    with open(header) as f:
        txt = f.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tod_[a-z_0-9]+)\s*\(", txt)))


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        return x.data_ptr()
    return x.ctypes.data


def _as_f32_2d(x):
    if _is_torch(x):
        import torch
        if x.dtype != torch.float32 or x.dim() != 2:
            raise ValueError("X must be a 2-D float32 tensor")
        return x.contiguous()
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError("X must be 2-D")
    return x


def _empty_like_host_or_dev(ref, shape, dtype_np):
    if _is_torch(ref):
        import torch
        tmap = {np.int64: torch.int64, np.int32: torch.int32, np.float32: torch.float32,
                np.float64: torch.float64}
        # host outputs of a pinned host input are pinned too (torch's caching host
        # allocator), so the library's device->host copies run at DMA speed
        pin = ref.device.type == "cpu" and ref.is_pinned()
        return torch.empty(shape, dtype=tmap[dtype_np], device=ref.device, pin_memory=pin)
    return np.empty(shape, dtype=dtype_np)


@dataclass
class KnnResult:
    idx: object
    dist: object
    dist64: object
    score_kth: object
    score_mean: object
    kdist64: object
    stats: dict
    row_tier: object = None


class Context:
    """Owns a tod_ctx (device workspace + stream binding)."""

    def __init__(self, device: int = 0, fmt: str = "auto", kprime: int = 0, chunks: int = 0,
                 flags: int = 0, stream=None, split: int = 0, workspace_bytes: int = 0):
        self.lib = load_library()
        if stream is None:
            # default to torch's current stream on this device, so kernels queued
            # there (producing X) are ordered before the library's; stream 0 (the
            # legacy default) maps to the library's own stream, which is blocking
            # with respect to it (include/tod.h tod_config.stream)
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream(device).cuda_stream or None
            except Exception:
                stream = None
        cfg = Config(device=device, format=FORMATS[fmt], kprime=kprime, flags=flags,
                     stream=stream, chunks=chunks, epilogue_split=split,
                     workspace_bytes=workspace_bytes)
        h = ctypes.c_void_p()
        st = self.lib.tod_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != TOD_OK:
            raise TodError(st, "tod_create(device=%d) failed" % device)
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.tod_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st):
        if st != TOD_OK:
            msg = self.lib.tod_last_message(self.h)
            raise TodError(st, msg.decode() if msg else "")

    def _alloc_knn(self, ref, q, k, want):
        o = {}
        o["idx"] = _empty_like_host_or_dev(ref, (q, k), np.int64) if "idx" in want else None
        o["dist"] = _empty_like_host_or_dev(ref, (q, k), np.float32) if "dist" in want else None
        o["dist64"] = _empty_like_host_or_dev(ref, (q, k), np.float64) if "dist64" in want else None
        o["score_kth"] = _empty_like_host_or_dev(ref, (q,), np.float32) if "score_kth" in want else None
        o["score_mean"] = _empty_like_host_or_dev(ref, (q,), np.float32) if "score_mean" in want else None
        o["kdist64"] = _empty_like_host_or_dev(ref, (q,), np.float64) if "kdist64" in want else None
        o["row_tier"] = _empty_like_host_or_dev(ref, (q,), np.int32) if "row_tier" in want else None
        ko = KnnOut(*[_ptr(o[f]) for f, _ in KnnOut._fields_])
        return o, ko

    ALL = ("idx", "dist", "dist64", "score_kth", "score_mean", "kdist64")

    def knn(self, X, k: int, q_begin: int = 0, q_count=None, want=ALL) -> KnnResult:
        """tod_knn: exact kNN self-join for rows [q_begin, q_begin+q_count) of X."""
        X = _as_f32_2d(X)
        n, d = X.shape
        if q_count is None:
            q_count = n - q_begin
        o, ko = self._alloc_knn(X, q_count, k, want)
        s = Stats()
        self._check(self.lib.tod_knn(self.h, _ptr(X), n, d, k, q_begin, q_count, ctypes.byref(ko),
                                     ctypes.byref(s)))
        return KnnResult(**o, stats=s.as_dict())

    def knn_query(self, Q, X, k: int, want=ALL) -> KnnResult:
        """tod_knn_query: kNN of rows of Q among rows of X (no exclusion)."""
        Q = _as_f32_2d(Q)
        X = _as_f32_2d(X)
        if Q.shape[1] != X.shape[1]:
            raise ValueError("dimension mismatch")
        o, ko = self._alloc_knn(X, Q.shape[0], k, want)
        s = Stats()
        self._check(self.lib.tod_knn_query(self.h, _ptr(Q), Q.shape[0], _ptr(X), X.shape[0],
                                           X.shape[1], k, ctypes.byref(ko), ctypes.byref(s)))
        return KnnResult(**o, stats=s.as_dict())

    def nwr(self, X, phi: float, q_begin: int = 0, q_count=None, lists: bool = True,
            capacity: int = 0):
        """tod_nwr: neighbours within range (D_ij <= phi, squared distance) of rows
        [q_begin, q_begin+q_count).  Returns (counts int64[q], row_ptr int64[q+1],
        cols int32[total] | None, stats).  With lists=True and no capacity given the
        call sizes cols from a counting call first (two library calls)."""
        X = _as_f32_2d(X)
        n, d = X.shape
        if q_count is None:
            q_count = n - q_begin
        counts = _empty_like_host_or_dev(X, (q_count,), np.int64)
        row_ptr = _empty_like_host_or_dev(X, (q_count + 1,), np.int64)
        total = ctypes.c_int64(0)
        s = Stats()
        if lists and capacity <= 0:
            self._check(self.lib.tod_nwr(self.h, _ptr(X), n, d, float(phi), q_begin, q_count,
                                         _ptr(counts), _ptr(row_ptr), None, 0,
                                         ctypes.byref(total), ctypes.byref(s)))
            capacity = max(1, int(total.value))
        cols = None
        if lists:
            cols = _empty_like_host_or_dev(X, (capacity,), np.int32)
        self._check(self.lib.tod_nwr(self.h, _ptr(X), n, d, float(phi), q_begin, q_count,
                                     _ptr(counts), _ptr(row_ptr), _ptr(cols),
                                     capacity if lists else 0, ctypes.byref(total),
                                     ctypes.byref(s)))
        if cols is not None:
            cols = cols[: int(total.value)]
        return counts, row_ptr, cols, s.as_dict()

    def abod(self, X, k: int, q_begin: int = 0, q_count=None, want_knn=()):
        """tod_abod: -Var over neighbour pairs of <a,b>/(|a|^2 |b|^2) (a, b = neighbour - row;
        Kriegel's weighted angle factor, reading A20); (score fp32[q], KnnResult|None, stats)."""
        X = _as_f32_2d(X)
        n, d = X.shape
        if q_count is None:
            q_count = n - q_begin
        score = _empty_like_host_or_dev(X, (q_count,), np.float32)
        o, ko = self._alloc_knn(X, q_count, k, want_knn)
        s = Stats()
        self._check(self.lib.tod_abod(self.h, _ptr(X), n, d, k, q_begin, q_count, _ptr(score),
                                      ctypes.byref(ko) if want_knn else None, ctypes.byref(s)))
        res = KnnResult(**o, stats=s.as_dict()) if want_knn else None
        return score, res, s.as_dict()

    def knn_classify(self, Q, X, labels, k: int):
        """tod_knn_classify: majority vote of the k nearest rows of X; int32[nq]."""
        Q = _as_f32_2d(Q)
        X = _as_f32_2d(X)
        if _is_torch(X):
            import torch
            labels = torch.as_tensor(labels, dtype=torch.int32, device=X.device).contiguous()
        else:
            labels = np.ascontiguousarray(labels, dtype=np.int32)
        pred = _empty_like_host_or_dev(Q, (Q.shape[0],), np.int32)
        s = Stats()
        self._check(self.lib.tod_knn_classify(self.h, _ptr(Q), Q.shape[0], _ptr(X), X.shape[0],
                                              X.shape[1], k, _ptr(labels), _ptr(pred),
                                              ctypes.byref(s)))
        return pred

    def lof(self, X, k: int, want_knn=()):
        """tod_lof: returns (lof fp32[n], lrd fp32[n], KnnResult|None, stats)."""
        X = _as_f32_2d(X)
        n, d = X.shape
        lof = _empty_like_host_or_dev(X, (n,), np.float32)
        lrd = _empty_like_host_or_dev(X, (n,), np.float32)
        o, ko = self._alloc_knn(X, n, k, want_knn)
        s = Stats()
        self._check(self.lib.tod_lof(self.h, _ptr(X), n, d, k, _ptr(lof), _ptr(lrd),
                                     ctypes.byref(ko) if want_knn else None, ctypes.byref(s)))
        res = KnnResult(**o, stats=s.as_dict()) if want_knn else None
        return lof, lrd, res, s.as_dict()

    def debug_mainpass(self, X):
        """tod_debug_mainpass (diagnostics, CUDA tensors): raw tensor-core
        accumulators of query rows [0, 128) against all rows, and the operands
        as multiplied.  Returns (w [128, n], a_ops [128, K], b_ops [n, K], kernel)."""
        import torch
        X = _as_f32_2d(X)
        n, d = X.shape
        K = ((d + 15) // 16) * 16
        K = (16 if d <= 16 else 32 if d <= 32 else 64 if d <= 64 else 128 if d <= 128
             else 256 if d <= 256 else 512) + 16
        w = torch.empty((128, n), dtype=torch.float32, device=X.device)
        a = torch.empty((128, K), dtype=torch.float32, device=X.device)
        b = torch.empty((n, K), dtype=torch.float32, device=X.device)
        k_out, mk = ctypes.c_int32(0), ctypes.c_int32(0)
        self._check(self.lib.tod_debug_mainpass(self.h, _ptr(X), n, d, _ptr(w), _ptr(a), _ptr(b),
                                                ctypes.byref(k_out), ctypes.byref(mk)))
        assert k_out.value == K
        return w, a, b, mk.value

    # ---------------------------------------------------------- sharded path
    def comm_init(self, rank: int, world: int, comm_id: bytes):
        """tod_comm_init: attach this rank's NCCL communicator (collective)."""
        buf = ctypes.create_string_buffer(bytes(comm_id), 128)
        self._check(self.lib.tod_comm_init(self.h, buf, rank, world))
        self.rank, self.world = rank, world

    def comm_init_loopback(self, world: int):
        """tod_comm_init_loopback (testing): `world` virtual ranks on this GPU."""
        self._check(self.lib.tod_comm_init_loopback(self.h, world))
        self.rank, self.world = 0, world

    def knn_sharded(self, X_local, n: int, row_offset: int, k: int, want=("idx", "dist64"),
                    gather_scores: bool = True):
        """tod_knn_sharded: kNN of this rank's rows; returns (KnnResult of the local
        rows, score_kth fp32[n] | None, score_mean fp32[n] | None) -- the scores of
        ALL rows, gathered."""
        X_local = _as_f32_2d(X_local)
        nl, d = X_local.shape
        o, ko = self._alloc_knn(X_local, nl, k, want)
        kth = _empty_like_host_or_dev(X_local, (n,), np.float32) if gather_scores else None
        mean = _empty_like_host_or_dev(X_local, (n,), np.float32) if gather_scores else None
        s = Stats()
        self._check(self.lib.tod_knn_sharded(self.h, _ptr(X_local), nl, row_offset, n, d, k,
                                             ctypes.byref(ko), _ptr(kth), _ptr(mean),
                                             ctypes.byref(s)))
        return KnnResult(**o, stats=s.as_dict()), kth, mean

    def lof_sharded(self, X_local, n: int, row_offset: int, k: int, want_knn=()):
        """tod_lof_sharded: returns (lof fp32[n], lrd fp32[n], KnnResult of the local
        rows | None, stats)."""
        X_local = _as_f32_2d(X_local)
        nl, d = X_local.shape
        lof = _empty_like_host_or_dev(X_local, (n,), np.float32)
        lrd = _empty_like_host_or_dev(X_local, (n,), np.float32)
        o, ko = self._alloc_knn(X_local, nl, k, want_knn)
        s = Stats()
        self._check(self.lib.tod_lof_sharded(self.h, _ptr(X_local), nl, row_offset, n, d, k,
                                             _ptr(lof), _ptr(lrd),
                                             ctypes.byref(ko) if want_knn else None,
                                             ctypes.byref(s)))
        res = KnnResult(**o, stats=s.as_dict()) if want_knn else None
        return lof, lrd, res, s.as_dict()

    def lof_lrd(self, n: int, k: int, idx, dist64, kdist64_all):
        q = idx.shape[0]
        out = _empty_like_host_or_dev(idx, (q,), np.float64)
        self._check(self.lib.tod_lof_lrd(self.h, n, k, q, _ptr(idx), _ptr(dist64),
                                         _ptr(kdist64_all), _ptr(out)))
        return out

    def lof_finish(self, n: int, k: int, q_begin: int, idx, lrd64_all):
        q = idx.shape[0]
        lof = _empty_like_host_or_dev(idx, (q,), np.float32)
        lrd = _empty_like_host_or_dev(idx, (q,), np.float32)
        self._check(self.lib.tod_lof_finish(self.h, n, k, q_begin, q, _ptr(idx), _ptr(lrd64_all),
                                            _ptr(lof), _ptr(lrd)))
        return lof, lrd
