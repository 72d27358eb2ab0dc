"""Thin Python binding of libsplit3.so (include/split3.h).

Argument marshalling only: tensors are passed as device pointers, torch's current
stream as the handle's stream and a torch uint8 tensor as the caller-owned
workspace.  Every step of the hot path runs in the library's CUDA kernels; there
is no CPU or PyTorch fallback — a missing library raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import _build

LIB_PATH = _build.LIB

OK = 0
ERR_INVALID_VALUE = 1
ERR_NOT_FINITE = 2
ERR_WORKSPACE = 3
ERR_CUDA = 4
ERR_ARCH = 5
ERR_NOT_IMPLEMENTED = 6

THREE_TERM = 0
FOUR_TERM = 1 << 0
CHECK_FINITE = 1 << 1
ONE_TERM = 1 << 2
BF16X3 = 1 << 3

# every symbol include/split3.h declares (checked by tests/test_capi.py)
EXPORTS = (
    "split3_sgemm_create", "split3_set_stream", "split3_sgemm_destroy",
    "split3_sgemm_workspace_size", "split3_sgemm_ex_workspace_size", "split3_sgemm_set_workspace", "split3_sgemm",
    "split3_sgemm_host_workspace_size", "split3_sgemm_host", "split3_last_bad_index", "split3_host_redo_count", "split3_host_last_layout",
    "split3_status_string", "split3_maxabs", "split3_split", "split3_gemm_planes",
    "split3_last_launch_count", "split3_last_path", "split3_timing_enable", "split3_timing_read",
    "split3_set_promotion", "split3_set_wave_sync", "split3_set_split_k", "split3_set_max_sms", "split3_set_schedule", "split3_set_fused_split", "split3_set_fused_split_a", "split3_set_fold",
    "split3_sgemm_ex", "split3_presplit", "split3_presplit_stored", "split3_split_bf16x3", "split3_debug_read", "split3_debug_fault", "split3_bias_act", "split3_relu_backward",
    "split3_softmax_xent", "split3_bias_grad", "split3_sgd_update",
)

class split3_matrix(ctypes.Structure):
    """ctypes mirror of include/split3.h's split3_matrix."""
    _fields_ = [("data", ctypes.c_void_p), ("ld", ctypes.c_int64), ("trans", ctypes.c_int),
                ("hi", ctypes.c_void_p), ("lo", ctypes.c_void_p), ("ldp", ctypes.c_int64),
                ("d_sexp", ctypes.c_void_p), ("stored", ctypes.c_int)]


class split3_host_layout(ctypes.Structure):
    """ctypes mirror of include/split3.h's split3_host_layout."""
    _fields_ = [("nblk", ctypes.c_int), ("npan", ctypes.c_int),
                ("blk_r0", ctypes.c_int64 * 32), ("blk_rows", ctypes.c_int64 * 32),
                ("pan_c0", ctypes.c_int64 * 4), ("pan_cols", ctypes.c_int64 * 4),
                ("A1", ctypes.c_void_p), ("A2", ctypes.c_void_p), ("ldpa", ctypes.c_int64),
                ("B1", ctypes.c_void_p), ("B2", ctypes.c_void_p), ("ldpb", ctypes.c_int64), ("b_mn", ctypes.c_int),
                ("d_sblk", ctypes.c_void_p), ("d_span", ctypes.c_void_p), ("d_redo", ctypes.c_void_p),
                ("d_sA", ctypes.c_void_p), ("d_sB", ctypes.c_void_p)]


class Planes:
    """A pre-split operand: FP16 planes (int16 tensors holding binary16 bits, padded leading
    dimension) and the device scale exponent.  From presplit(): role 0 = A operand (planes M x K),
    role 1 = B operand (planes N x K = op(B)^T), K-major.  From presplit_stored() (role None,
    stored=True): the plain split of the stored matrix, usable as A or B with either transpose."""

    def __init__(self, hi, lo, sexp, role, rows, cols, stored=False):
        self.hi, self.lo, self.sexp = hi, lo, sexp
        self.role, self.rows, self.cols = role, rows, cols   # op(X) (stored matrix if stored)
        self.stored = stored

    @property
    def shape(self):
        return (self.rows, self.cols)


_lib = None
_lock = threading.Lock()
_i64 = ctypes.c_int64
_p = ctypes.c_void_p


class Split3Error(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} ({status})")


class NotFiniteError(Split3Error):
    def __init__(self, status: int, what: str, index: int):
        self.index = index
        super().__init__(status, f"{what} (first non-finite index {index})")


def load() -> ctypes.CDLL:
    """Load libsplit3.so (raises if it was not built; never falls back)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        lib.split3_sgemm_create.argtypes = [ctypes.POINTER(_p), ctypes.c_int, _p]
        lib.split3_set_stream.argtypes = [_p, _p]
        lib.split3_sgemm_destroy.argtypes = [_p]
        lib.split3_sgemm_workspace_size.restype = ctypes.c_size_t
        lib.split3_sgemm_workspace_size.argtypes = [_i64, _i64, _i64, ctypes.c_uint32]
        lib.split3_sgemm_ex_workspace_size.restype = ctypes.c_size_t
        lib.split3_sgemm_ex_workspace_size.argtypes = [_i64, _i64, _i64, ctypes.c_uint32, ctypes.c_int, ctypes.c_int]
        lib.split3_sgemm_host_workspace_size.restype = ctypes.c_size_t
        lib.split3_sgemm_host_workspace_size.argtypes = [_i64, _i64, _i64, ctypes.c_uint32]
        lib.split3_sgemm_set_workspace.argtypes = [_p, _p, ctypes.c_size_t]
        lib.split3_sgemm.argtypes = [_p, _i64, _i64, _i64, _p, _i64, _p, _i64, _p, _i64, ctypes.c_uint32]
        lib.split3_sgemm_host.argtypes = [_p, _i64, _i64, _i64, _p, _p, _p, ctypes.c_uint32]
        lib.split3_last_bad_index.restype = _i64
        lib.split3_last_bad_index.argtypes = [_p]
        lib.split3_host_last_layout.argtypes = [_p, ctypes.POINTER(split3_host_layout)]
        lib.split3_host_redo_count.restype = _i64
        lib.split3_host_redo_count.argtypes = [_p]
        lib.split3_last_launch_count.argtypes = [_p]
        lib.split3_last_path.argtypes = [_p]
        lib.split3_timing_enable.argtypes = [_p, ctypes.c_int]
        lib.split3_set_promotion.argtypes = [_p, ctypes.c_int]
        lib.split3_set_wave_sync.argtypes = [_p, ctypes.c_int]
        lib.split3_set_split_k.argtypes = [_p, ctypes.c_int]
        lib.split3_set_max_sms.argtypes = [_p, ctypes.c_int]
        lib.split3_set_schedule.argtypes = [_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.split3_set_fused_split.argtypes = [_p, ctypes.c_int, _i64]
        lib.split3_set_fused_split_a.argtypes = [_p, ctypes.c_int, _i64]
        lib.split3_set_fold.argtypes = [_p, ctypes.c_int]
        lib.split3_sgemm_ex.argtypes = [_p, _i64, _i64, _i64, ctypes.POINTER(split3_matrix),
                                        ctypes.POINTER(split3_matrix), _p, _i64, ctypes.c_uint32]
        lib.split3_debug_read.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        lib.split3_debug_fault.argtypes = [ctypes.c_int]
        lib.split3_split_bf16x3.argtypes = [_p, _i64, _i64, _p, _i64, _p, _p, _p, _i64, ctypes.c_int]
        lib.split3_bias_act.argtypes = [_p, _i64, _i64, _p, _i64, _p, _p, _i64, ctypes.c_int]
        lib.split3_relu_backward.argtypes = [_p, _i64, _i64, _p, _p, _p]
        lib.split3_softmax_xent.argtypes = [_p, _i64, _i64, _p, _p, _p, _p, _p, _p]
        lib.split3_bias_grad.argtypes = [_p, _i64, _i64, _p, _p]
        lib.split3_sgd_update.argtypes = [_p, _i64, _p, _p, ctypes.c_float]
        lib.split3_presplit.argtypes = [_p, ctypes.c_int, _i64, _i64, _p, _i64, ctypes.c_int, _p, _p,
                                        _i64, _p]
        lib.split3_presplit_stored.argtypes = [_p, _i64, _i64, _p, _i64, _p, _p, _i64, _p]
        lib.split3_timing_read.argtypes = [_p, ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
        lib.split3_status_string.restype = ctypes.c_char_p
        lib.split3_status_string.argtypes = [ctypes.c_int]
        lib.split3_maxabs.argtypes = [_p, _i64, _i64, _p, _i64, _p, _p]
        lib.split3_split.argtypes = [_p, _i64, _i64, _p, _i64, _p, _p, _p, _i64, ctypes.c_int, _p]
        lib.split3_gemm_planes.argtypes = [_p, _i64, _i64, _i64, _p, _p, _i64, _p, _p, _p, _i64, _p,
                                           _p, _i64, ctypes.c_uint32]
        _lib = lib
        return lib


def debug_read(reset: bool = True):
    """The debug build's GEMM check record (code, detail, CTA, warp, count, ...); raises
    Split3Error(NOT_IMPLEMENTED) on a release library."""
    buf = (ctypes.c_uint64 * 8)()
    st = load().split3_debug_read(buf, int(reset))
    if st != OK:
        raise Split3Error(st, "split3_debug_read")
    return list(buf)


def debug_fault(fault: int):
    st = load().split3_debug_fault(int(fault))
    if st != OK:
        raise Split3Error(st, "split3_debug_fault")


def status_string(status: int) -> str:
    return load().split3_status_string(int(status)).decode()


def plane_ld(k: int) -> int:
    """Padded plane leading dimension (multiple of 8 elements), as the library uses."""
    return (k + 7) // 8 * 8


def _flags(four_term: bool, one_term: bool, check_finite: bool, bf16x3: bool = False) -> int:
    f = BF16X3 if bf16x3 else 0
    if four_term:
        f |= FOUR_TERM
    if one_term:
        f |= ONE_TERM
    if check_finite:
        f |= CHECK_FINITE
    return f


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


class _StreamState:
    """The library handle and workspace of one CUDA stream (include/split3.h: a handle is not
    thread-safe and serves one stream; its workspace and device counters are per call chain)."""

    __slots__ = ("h", "ws", "pinned", "captured")

    def __init__(self, h):
        self.h = h
        self.ws = None          # torch uint8 tensor attached as the workspace
        self.pinned = []        # retired workspaces a captured CUDA graph may still point into
        self.captured = False   # the current workspace was used under stream capture


class Handle:
    """split3 on one CUDA device.  Every call runs on torch's current stream; each stream gets its
    own library handle (device counters) and workspace, so calls on different streams never share
    scratch memory.  A workspace that a CUDA graph captured is never freed while the Handle lives
    (a later, larger call attaches a new one and keeps the old one alive for the graph's replays)."""

    def __init__(self, device=None):
        lib = load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", torch.device("cuda", device).index
                                   if not isinstance(device, int) else device)
        self._lib = lib
        self._states: dict[int, _StreamState] = {}
        self._settings: dict[str, tuple] = {}     # knob -> args, applied to every stream's handle
        self._closed = False
        self._state()                             # create the current stream's handle (errors here)

    def close(self):
        for stt in self._states.values():
            if stt.h:
                self._lib.split3_sgemm_destroy(stt.h)
                stt.h = _p()
        self._states = {}
        self._closed = True

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing ---------------------------------------------------------------
    def _state(self) -> _StreamState:
        if self._closed:
            raise RuntimeError("split3 Handle is closed")
        s = torch.cuda.current_stream(self.device).cuda_stream
        stt = self._states.get(s)
        if stt is None:
            hp = _p()
            st = self._lib.split3_sgemm_create(ctypes.byref(hp), self.device.index, _p(s))
            if st != OK:
                raise Split3Error(st, "split3_sgemm_create")
            stt = _StreamState(hp)
            for name, args in self._settings.items():
                st = getattr(self._lib, name)(hp, *args)
                if st != OK:
                    raise Split3Error(st, name)
            self._states[s] = stt
        return stt

    @property
    def _h(self):
        """the library handle of torch's current stream"""
        return self._state().h

    @property
    def _ws(self):
        return self._state().ws

    @_ws.setter
    def _ws(self, t):
        self._state().ws = t

    def _bind_stream(self):
        """Kept for the call sites: the handle of the current stream is created bound to it."""
        stt = self._state()
        if torch.cuda.is_current_stream_capturing():
            stt.captured = True
        return stt

    def _set(self, name: str, *args):
        """Apply a knob to every stream's handle, present and future."""
        self._settings[name] = args
        for stt in self._states.values():
            st = getattr(self._lib, name)(stt.h, *args)
            if st != OK:
                raise Split3Error(st, name)

    def _ensure_ws(self, nbytes: int):
        stt = self._state()
        if stt.ws is None or stt.ws.numel() < nbytes:
            if stt.ws is not None and (stt.captured or torch.cuda.is_current_stream_capturing()):
                stt.pinned.append(stt.ws)     # a captured graph may replay into it: keep it alive
            stt.captured = False
            # allocated on this stream: the caching allocator reuses a freed block only in this
            # stream's order, so a replaced (uncaptured) workspace is safe to drop
            stt.ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            st = self._lib.split3_sgemm_set_workspace(stt.h, stt.ws.data_ptr(), stt.ws.numel())
            if st != OK:
                raise Split3Error(st, "split3_sgemm_set_workspace")
        if torch.cuda.is_current_stream_capturing():
            stt.captured = True

    def workspace_size(self, M, N, K, flags=0) -> int:
        return int(self._lib.split3_sgemm_workspace_size(M, N, K, flags))

    def set_promotion(self, kblocks: int):
        """D_hi promotion period in 64-wide k-blocks (0 = library default)."""
        self._set("split3_set_promotion", int(kblocks))

    def set_wave_sync(self, enable: bool):
        self._set("split3_set_wave_sync", int(enable))

    def set_split_k(self, enable: bool):
        """Split-K tail on (default) or whole tiles only (deterministic per-element K order)."""
        self._set("split3_set_split_k", int(enable))

    def set_max_sms(self, sms: int):
        """Cap the SMs the GEMM occupies (0 = all; even)."""
        self._set("split3_set_max_sms", int(sms))

    def set_schedule(self, group_m: int = 0, l2_policy_a: int = 0, l2_policy_b: int = 0):
        self._set("split3_set_schedule", int(group_m), int(l2_policy_a), int(l2_policy_b))

    def set_fused_split(self, mode: int, max_m: int = 0):
        """Fused split of an fp32 B inside the GEMM (NEXT #2): 0 off, 1 auto (M <= max_m), 2 always."""
        self._set("split3_set_fused_split", int(mode), int(max_m))

    def set_fold(self, mode: int):
        """Folded accumulator (a k-block's 3 (4) products in one TMEM accumulator via scale-input-d):
        0 never, 1 4-term calls of >= 8192^3 multiply-adds (default), 2 every 4- and 3-term call."""
        self._set("split3_set_fold", int(mode))

    def set_fused_split_a(self, mode: int, max_n: int = 0):
        """Fused split of an fp32 A (NEXT #2) through C^T = B^T A^T: 0 off, 1 auto (N <= max_n and
        N < M), 2 always when eligible (before fused B)."""
        self._set("split3_set_fused_split_a", int(mode), int(max_n))

    def timing_enable(self, enable: bool = True):
        """CUDA-event timing of the split and GEMM phases of later calls (current stream's handle)."""
        self._lib.split3_timing_enable(self._h, int(enable))

    def timing_read(self):
        """(split_ms_total, gemm_ms_total, calls) since the last read (synchronises)."""
        s, g, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        st = self._lib.split3_timing_read(self._h, ctypes.byref(s), ctypes.byref(g), ctypes.byref(n))
        if st != OK:
            raise Split3Error(st, "split3_timing_read")
        return s.value, g.value, n.value

    def host_redo_count(self) -> int:
        """row blocks the host pipeline redid with the per-matrix scale"""
        return int(self._lib.split3_host_redo_count(self._h))

    def host_last_layout(self) -> split3_host_layout:
        """where the last sgemm_host call left its planes (device pointers into the workspace)"""
        out = split3_host_layout()
        self._chk(self._lib.split3_host_last_layout(self._h, ctypes.byref(out)), "split3_host_last_layout")
        return out

    def last_path(self) -> int:
        """SPLIT3_PATH_* bits of the last call: 1 fused B, 2 fused A, 8 one-launch front end,
        16 folded accumulator."""
        return int(self._lib.split3_last_path(self._h))

    def last_launch_count(self) -> int:
        return int(self._lib.split3_last_launch_count(self._h))

    # -- the whole method ---------------------------------------------------------
    def sgemm(self, A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None,
              four_term: bool = False, one_term: bool = False, check_finite: bool = False,
              bf16x3: bool = False):
        """C = A @ B (fp32, row-major; leading-dimension strides allowed)."""
        _check_mat(A, "A")
        _check_mat(B, "B")
        M, K = A.shape
        K2, N = B.shape
        if K != K2:
            raise ValueError(f"inner dimensions differ: {K} vs {K2}")
        if out is None:
            out = torch.empty((M, N), dtype=torch.float32, device=A.device)
        _check_mat(out, "C")
        flags = _flags(four_term, one_term, check_finite, bf16x3)
        self._ensure_ws(self.workspace_size(M, N, K, flags))
        self._bind_stream()
        st = self._lib.split3_sgemm(self._h, M, N, K, _ptr(A), _ld(A), _ptr(B), _ld(B),
                                    _ptr(out), _ld(out), flags)
        if st == ERR_NOT_FINITE:
            raise NotFiniteError(st, "split3_sgemm", int(self._lib.split3_last_bad_index(self._h)))
        if st != OK:
            raise Split3Error(st, "split3_sgemm")
        return out

    def presplit(self, X: torch.Tensor, role: int, trans: bool = False) -> Planes:
        """Split op(X) once (role 0: an A operand, role 1: a B operand) for reuse."""
        _check_mat(X, "X")
        rows, cols = (X.shape[1], X.shape[0]) if trans else (X.shape[0], X.shape[1])
        prow, pk = (rows, cols) if role == 0 else (cols, rows)
        ldp = plane_ld(pk)
        hi = torch.empty((prow, ldp), dtype=torch.int16, device=X.device)
        lo = torch.empty((prow, ldp), dtype=torch.int16, device=X.device)
        sexp = torch.zeros(1, dtype=torch.int32, device=X.device)
        self._bind_stream()
        st = self._lib.split3_presplit(self._h, int(role), rows, cols, _ptr(X), _ld(X), int(trans),
                                       _ptr(hi), _ptr(lo), ldp, _ptr(sexp))
        if st != OK:
            raise Split3Error(st, "split3_presplit")
        return Planes(hi, lo, sexp, role, rows, cols)

    def presplit_stored(self, X: torch.Tensor) -> Planes:
        """Split the stored matrix X (rows x cols) once, without a transpose; the planes serve
        sgemm_ex as A or B, with transA / transB as for the fp32 matrix."""
        _check_mat(X, "X")
        rows, cols = X.shape
        ldp = plane_ld(cols)
        hi = torch.empty((rows, ldp), dtype=torch.int16, device=X.device)
        lo = torch.empty((rows, ldp), dtype=torch.int16, device=X.device)
        sexp = torch.empty(1, dtype=torch.int32, device=X.device)    # written by the split
        self._bind_stream()
        st = self._lib.split3_presplit_stored(self._h, rows, cols, _ptr(X), _ld(X), _ptr(hi), _ptr(lo), ldp,
                                              _ptr(sexp))
        if st != OK:
            raise Split3Error(st, "split3_presplit_stored")
        return Planes(hi, lo, sexp, None, rows, cols, stored=True)

    def sgemm_ex(self, A, B, transA: bool = False, transB: bool = False, out=None,
                 four_term: bool = False, one_term: bool = False, check_finite: bool = False,
                 bf16x3: bool = False):
        """C = op(A) @ op(B); A / B are fp32 CUDA tensors or Planes from presplit()."""
        def desc(X, trans, role, name):
            if isinstance(X, Planes):
                if X.stored:
                    shp = (X.cols, X.rows) if trans else (X.rows, X.cols)
                    return split3_matrix(None, 0, int(trans), X.hi.data_ptr(), X.lo.data_ptr(), X.hi.stride(0),
                                         X.sexp.data_ptr(), 1), shp
                if X.role != role:
                    raise ValueError(f"{name}: planes were split for role {X.role}")
                return split3_matrix(None, 0, 0, X.hi.data_ptr(), X.lo.data_ptr(), X.hi.stride(0),
                                     X.sexp.data_ptr(), 0), X.shape
            _check_mat(X, name)
            shp = (X.shape[1], X.shape[0]) if trans else tuple(X.shape)
            return split3_matrix(X.data_ptr(), _ld(X), int(trans), None, None, 0, None, 0), shp

        da, (M, K) = desc(A, transA, 0, "A")
        db, (K2, N) = desc(B, transB, 1, "B")
        if K != K2:
            raise ValueError(f"inner dimensions differ: {K} vs {K2}")
        dev = A.hi.device if isinstance(A, Planes) else A.device
        if out is None:
            out = torch.empty((M, N), dtype=torch.float32, device=dev)
        _check_mat(out, "C")
        flags = _flags(four_term, one_term, check_finite, bf16x3)
        self._ensure_ws(int(self._lib.split3_sgemm_ex_workspace_size(
            M, N, K, flags, int(isinstance(A, Planes)), int(isinstance(B, Planes)))))
        self._bind_stream()
        st = self._lib.split3_sgemm_ex(self._h, M, N, K, ctypes.byref(da), ctypes.byref(db),
                                       _ptr(out), _ld(out), flags)
        if st == ERR_NOT_FINITE:
            raise NotFiniteError(st, "split3_sgemm_ex", int(self._lib.split3_last_bad_index(self._h)))
        if st != OK:
            raise Split3Error(st, "split3_sgemm_ex")
        return out

    # -- dense-network step helpers (NEXT #3) ------------------------------------------
    def _chk(self, st, what):
        if st != OK:
            raise Split3Error(st, what)

    def bias_act(self, Z, b, relu: bool, out=None):
        out = torch.empty_like(Z) if out is None else out
        self._bind_stream()
        self._chk(self._lib.split3_bias_act(self._h, Z.shape[0], Z.shape[1], _ptr(Z), _ld(Z), _ptr(b),
                                            _ptr(out), _ld(out), int(relu)), "split3_bias_act")
        return out

    def relu_backward(self, dH, H, out=None):
        out = torch.empty_like(dH) if out is None else out
        self._bind_stream()
        self._chk(self._lib.split3_relu_backward(self._h, dH.shape[0], dH.shape[1], _ptr(dH), _ptr(H),
                                                 _ptr(out)), "split3_relu_backward")
        return out

    def softmax_xent(self, L, labels=None, want_probs=True, want_grad=True):
        """(P, dL, loss) for logits L (M x N) and int32 labels; loss is a 0-d fp64 device tensor."""
        M, N = L.shape
        P = torch.empty_like(L) if want_probs else None
        dL = torch.empty_like(L) if (want_grad and labels is not None) else None
        loss = torch.zeros((), dtype=torch.float64, device=L.device) if labels is not None else None
        rows = torch.empty(M, dtype=torch.float64, device=L.device) if labels is not None else None
        self._bind_stream()
        self._chk(self._lib.split3_softmax_xent(self._h, M, N, _ptr(L), _ptr(labels), _ptr(P), _ptr(dL),
                                                _ptr(rows), _ptr(loss)), "split3_softmax_xent")
        if loss is not None:
            loss = loss / M
        return P, dL, loss

    def bias_grad(self, dZ, out=None):
        out = torch.empty(dZ.shape[1], dtype=torch.float32, device=dZ.device) if out is None else out
        self._bind_stream()
        self._chk(self._lib.split3_bias_grad(self._h, dZ.shape[0], dZ.shape[1], _ptr(dZ), _ptr(out)),
                  "split3_bias_grad")
        return out

    def sgd_update(self, w, g, lr: float):
        self._bind_stream()
        self._chk(self._lib.split3_sgd_update(self._h, w.numel(), _ptr(w), _ptr(g), float(lr)),
                  "split3_sgd_update")

    def sgemm_host(self, A, B, out=None, four_term=False, one_term=False):
        """C = A @ B with HOST (numpy / CPU torch) buffers: copies inside the C-ABI call."""
        import numpy as np

        A = np.ascontiguousarray(A, dtype=np.float32)
        B = np.ascontiguousarray(B, dtype=np.float32)
        M, K = A.shape
        K2, N = B.shape
        if K != K2:
            raise ValueError("inner dimensions differ")
        if out is None:
            out = np.empty((M, N), np.float32)
        flags = _flags(four_term, one_term, False)
        self._ensure_ws(int(self._lib.split3_sgemm_host_workspace_size(M, N, K, flags)))
        self._bind_stream()
        st = self._lib.split3_sgemm_host(self._h, M, N, K, A.ctypes.data, B.ctypes.data,
                                         out.ctypes.data, flags)
        if st != OK:
            raise Split3Error(st, "split3_sgemm_host")
        return out

    def sgemm_host_ptr(self, M, N, K, a_ptr, b_ptr, c_ptr, flags=0):
        """Raw-pointer variant of sgemm_host (pinned torch tensors in the bench)."""
        self._ensure_ws(int(self._lib.split3_sgemm_host_workspace_size(M, N, K, flags)))
        self._bind_stream()
        st = self._lib.split3_sgemm_host(self._h, M, N, K, a_ptr, b_ptr, c_ptr, flags)
        if st != OK:
            raise Split3Error(st, "split3_sgemm_host")

    # -- lower level --------------------------------------------------------------
    def maxabs(self, X: torch.Tensor, d_max: torch.Tensor, d_bad: torch.Tensor | None = None):
        """Fold max|X| over finite entries into d_max (float32[1], caller-initialised)."""
        _check_mat(X, "X")
        self._bind_stream()
        st = self._lib.split3_maxabs(self._h, X.shape[0], X.shape[1], _ptr(X), _ld(X),
                                     _ptr(d_max), _ptr(d_bad))
        if st != OK:
            raise Split3Error(st, "split3_maxabs")

    def split(self, X: torch.Tensor, d_max: torch.Tensor, transpose: bool = False,
              hi=None, lo=None, d_sexp=None):
        """Eq. A_1 planes of X (int16 tensors holding binary16 bits) with padded ld."""
        _check_mat(X, "X")
        rows, cols = X.shape
        prow, pcol = (cols, rows) if transpose else (rows, cols)
        ldp = plane_ld(pcol)
        if hi is None:
            hi = torch.empty((prow, ldp), dtype=torch.int16, device=X.device)
        if lo is None:
            lo = torch.empty((prow, ldp), dtype=torch.int16, device=X.device)
        if d_sexp is None:
            d_sexp = torch.zeros(1, dtype=torch.int32, device=X.device)
        self._bind_stream()
        st = self._lib.split3_split(self._h, rows, cols, _ptr(X), _ld(X), _ptr(d_max), _ptr(hi),
                                    _ptr(lo), hi.stride(0), int(transpose), _ptr(d_sexp))
        if st != OK:
            raise Split3Error(st, "split3_split")
        return hi, lo, d_sexp

    def split_bf16x3(self, X: torch.Tensor, transpose: bool = False):
        """bf16 x 3 planes (int16 tensors holding bfloat16 bits) of X, padded leading dimension."""
        _check_mat(X, "X")
        rows, cols = X.shape
        prow, pcol = (cols, rows) if transpose else (rows, cols)
        ldp = plane_ld(pcol)
        ps = [torch.empty((prow, ldp), dtype=torch.int16, device=X.device) for _ in range(3)]
        self._bind_stream()
        st = self._lib.split3_split_bf16x3(self._h, rows, cols, _ptr(X), _ld(X), *[_ptr(p) for p in ps], ldp,
                                           int(transpose))
        if st != OK:
            raise Split3Error(st, "split3_split_bf16x3")
        return ps

    def gemm_planes(self, M, N, K, A1, A2, d_sA, B1t, B2t, d_sB, out=None,
                    four_term=False, one_term=False):
        """C from planes: A1/A2 M x ldp, B1t/B2t N x ldp (K-major), device scale exponents."""
        if out is None:
            out = torch.empty((M, N), dtype=torch.float32, device=A1.device)
        flags = _flags(four_term, one_term, False)
        self._bind_stream()
        st = self._lib.split3_gemm_planes(self._h, M, N, K, _ptr(A1), _ptr(A2), A1.stride(0), _ptr(d_sA),
                                          _ptr(B1t), _ptr(B2t), B1t.stride(0), _ptr(d_sB),
                                          _ptr(out), _ld(out), flags)
        if st != OK:
            raise Split3Error(st, "split3_gemm_planes")
        return out


def _check_mat(t, name):
    if not isinstance(t, torch.Tensor) or t.dim() != 2:
        raise ValueError(f"{name} must be a 2-D torch tensor")
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be float32, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (use Handle.sgemm_host for host buffers)")
    if t.stride(1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        raise ValueError(f"{name} must be row-major with unit column stride")


def _ld(t) -> int:
    return max(t.stride(0), t.shape[1], 1) if t.shape[0] > 1 else max(t.shape[1], 1)


_handles: dict[int, Handle] = {}


def handle(device=None) -> Handle:
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    h = _handles.get(idx)
    if h is None:
        h = Handle(idx)
        _handles[idx] = h
    return h


def sgemm(A, B, out=None, four_term=False, one_term=False, check_finite=False, bf16x3=False):
    """C = A @ B emulated with FP16 tensor-core GEMMs (arXiv 2011.11188, Appendix A)."""
    return handle(A.device).sgemm(A, B, out=out, four_term=four_term, one_term=one_term,
                                  check_finite=check_finite, bf16x3=bf16x3)
