"""Thin Python binding of libsq (include/libsq.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this module
only turns torch tensors into device pointers and the current CUDA stream, and
raises on non-OK status.  There is no CPU fallback: if libsq.so is missing the
import of any entry point raises.

Names follow the C ABI (and the paper's notation):
  act_absmax(X)                        calibration max|X_j| (Eq. 6 input)
  smooth_scales(W, act_max, alpha)     Eq. 6 smoothing factors s
  quantize_pack_groupwise(W, s)        Eq. 5 fold + Eq. 1 INT4 quantize/pack
  w4a16_gemm(X, Wq, scales, zeros)     Eq. 3 W4A16 linear layer

Argument checks here (shape, dtype, device of caller-supplied outputs and vectors) only
protect the C ABI from out-of-bounds pointers; they do no arithmetic.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libsq.so")

SQ_OK, SQ_ERR_NULL, SQ_ERR_SHAPE, SQ_ERR_UNSUPPORTED, SQ_ERR_ALIGN, SQ_ERR_CUDA, SQ_ERR_WORKSPACE = range(7)
SQ_F16, SQ_BF16 = 0, 1
SQ_PATH_AUTO, SQ_PATH_DECODE, SQ_PATH_PREFILL = 0, 1, 2
SQ_OPT_PDL, SQ_OPT_DECODE_SCHEDULE, SQ_OPT_DECODE_GRID_LIMIT = 1, 3, 5
SQ_GEMM_WEIGHTS_STATIC = 1
SQ_ZEROS_U4 = 2
SQ_SCHED_AUTO, SQ_SCHED_STREAMK, SQ_SCHED_ROWBLOCK = 0, 1, 2
GROUP = 128

_lib = None


class SQError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libsq status {status}: {msg}")
        self.status = status


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsq.so not built ({LIB_PATH}); run `python -m paper_2312_03788_b200.build`")
    lib = ctypes.CDLL(LIB_PATH)
    c = ctypes
    vp, i64, i32, f64, sz = c.c_void_p, c.c_int64, c.c_int, c.c_double, c.c_size_t
    sig = {
        "sq_version": (i32, []),
        "sq_status_string": (c.c_char_p, [i32]),
        "sq_last_error": (c.c_char_p, []),
        "sq_decode_max_m": (i32, []),
        "sq_set_option": (i32, [i32, i32]),
        "sq_get_option": (i32, [i32]),
        "sq_act_absmax": (i32, [vp, i32, i64, i64, vp, i32, vp]),
        "sq_smooth_scales": (i32, [vp, i32, i64, i64, vp, f64, f64, vp, vp]),
        "sq_smooth_scales_wmax": (i32, [vp, vp, i64, f64, f64, vp, vp]),
        "sq_workspace_reset": (i32, [vp, sz, vp]),
        "sq_quantize_pack_groupwise": (i32, [vp, i32, vp, i64, i64, i32, vp, vp, vp, vp, vp]),
        "sq_quantize_pack_groupwise_ex": (i32, [vp, i32, vp, i64, i64, i32, vp, vp, vp, vp, c.c_uint, vp]),
        "sq_w4a16_gemm_workspace_bytes": (sz, [i64, i64, i64, i32]),
        "sq_w4a16_gemm": (i32, [vp, i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, sz, vp]),
        "sq_w4a16_gemm_path": (i32, [vp, i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, sz, i32, vp]),
        "sq_w4a16_gemm_ex": (i32, [vp, i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, sz, i32, c.c_uint, vp]),
        "sq_smooth_activations": (i32, [vp, i32, vp, i64, i64, vp, vp]),
        "sq_sq_diff_sum_workspace_bytes": (sz, []),
        "sq_fold_rows": (i32, [vp, i32, vp, i64, i64, vp, vp]),
        "sq_sq_diff_sum": (i32, [vp, vp, i32, i64, vp, vp, sz, vp]),
        "sq_allreduce_buffer_bytes": (sz, [i64, i32]),
        "sq_w4a16_gemm_allreduce": (i32, [vp, i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, sz, vp, i32, i32, i64,
                                          c.c_uint32, vp, c.c_uint, vp]),
        "sq_allreduce_oneshot": (i32, [vp, i32, vp, i64, i64, vp, i32, i32, c.c_uint32, vp, vp]),
        "sq_ipc_handle_bytes": (sz, []),
        "sq_ipc_get_handle": (i32, [vp, vp, c.POINTER(sz)]),
        "sq_ipc_open_handle": (i32, [vp, c.POINTER(vp)]),
        "sq_ipc_close": (i32, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


EXPORTED = (
    "sq_version", "sq_status_string", "sq_last_error", "sq_decode_max_m", "sq_set_option",
    "sq_get_option", "sq_act_absmax",
    "sq_smooth_scales", "sq_smooth_scales_wmax", "sq_quantize_pack_groupwise", "sq_quantize_pack_groupwise_ex",
    "sq_w4a16_gemm_workspace_bytes",
    "sq_workspace_reset", "sq_w4a16_gemm", "sq_w4a16_gemm_path", "sq_w4a16_gemm_ex", "sq_smooth_activations", "sq_sq_diff_sum_workspace_bytes",
    "sq_sq_diff_sum", "sq_fold_rows", "sq_allreduce_buffer_bytes", "sq_w4a16_gemm_allreduce", "sq_allreduce_oneshot", "sq_ipc_handle_bytes",
    "sq_ipc_get_handle", "sq_ipc_open_handle", "sq_ipc_close",
)


def lib():
    return _load()


def _check(st: int):
    if st != SQ_OK:
        L = _load()
        raise SQError(st, (L.sq_last_error() or b"").decode() or L.sq_status_string(st).decode())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float16:
        return SQ_F16
    if t.dtype == torch.bfloat16:
        return SQ_BF16
    raise TypeError(f"unsupported dtype {t.dtype} (need float16/bfloat16)")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libsq entry points take CUDA tensors (device pointers)")
        if t is not None and not t.is_contiguous():
            raise ValueError("libsq entry points take contiguous tensors")


def _check_out(out, shape, dtype, device, what="out"):
    """A caller-supplied output must match exactly: the C ABI cannot see tensor sizes."""
    if out is None:
        return
    if tuple(out.shape) != tuple(shape) or out.dtype != dtype or out.device != device:
        raise ValueError(f"{what}: need shape {tuple(shape)} {dtype} on {device}, got "
                         f"{tuple(out.shape)} {out.dtype} on {out.device}")


def _check_vec(v, K, what):
    """fp32[K] device vectors (s, act_max, w_max, d)."""
    if v is None:
        return
    if v.dtype != torch.float32 or v.numel() != K:
        raise ValueError(f"{what}: need float32[{K}], got {v.dtype}[{v.numel()}]")


def version() -> int:
    return _load().sq_version()


def decode_max_m() -> int:
    return _load().sq_decode_max_m()


def set_option(opt: int, value: int) -> None:
    """Process-wide launch option (SQ_OPT_PDL, SQ_OPT_DECODE_SCHEDULE; include/libsq.h)."""
    _check(_load().sq_set_option(int(opt), int(value)))


def get_option(opt: int) -> int:
    return int(_load().sq_get_option(int(opt)))


def act_absmax(X: torch.Tensor, out: torch.Tensor | None = None, accumulate: bool = False,
               stream=None) -> torch.Tensor:
    """act_max[k] = max_t |X[t][k]| (calibration statistic of Eq. 6)."""
    _need_cuda(X, out)
    T, K = X.shape
    _check_out(out, (K,), torch.float32, X.device)
    if out is None:
        out = torch.empty(K, dtype=torch.float32, device=X.device)
    _check(_load().sq_act_absmax(_ptr(X), _dtype_code(X), T, K, _ptr(out), int(accumulate), _stream(stream)))
    return out


def smooth_scales(W: torch.Tensor, act_max: torch.Tensor, alpha: float, eps: float = 1e-5,
                  out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Eq. 6 smoothing factors s[K] for the (possibly stacked) consumer weight W[N][K]."""
    _need_cuda(W, act_max, out)
    N, K = W.shape
    _check_vec(act_max, K, "act_max")
    _check_out(out, (K,), torch.float32, W.device)
    if out is None:
        out = torch.empty(K, dtype=torch.float32, device=W.device)
    _check(_load().sq_smooth_scales(_ptr(W), _dtype_code(W), N, K, _ptr(act_max), float(alpha),
                                    float(eps), _ptr(out), _stream(stream)))
    return out


def weight_absmax(W: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """w_max[k] = max_n |W[n][k]| (Eq. 6's weight maxima) -- the column abs-max kernel of
    sq_act_absmax applied to the [N][K] weight."""
    return act_absmax(W, out=out, stream=stream)


def smooth_scales_wmax(w_max: torch.Tensor, act_max: torch.Tensor, alpha: float, eps: float = 1e-5,
                       out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Eq. 6 from precomputed maxima (sq_smooth_scales_wmax): used by tensor-parallel
    shards after a MAX all-reduce of w_max, so every rank folds the same s."""
    _need_cuda(w_max, act_max, out)
    K = w_max.numel()
    _check_vec(w_max, K, "w_max")
    _check_vec(act_max, K, "act_max")
    _check_out(out, (K,), torch.float32, w_max.device)
    if out is None:
        out = torch.empty(K, dtype=torch.float32, device=w_max.device)
    _check(_load().sq_smooth_scales_wmax(_ptr(w_max), _ptr(act_max), K, float(alpha), float(eps), _ptr(out),
                                         _stream(stream)))
    return out


@dataclass
class QuantizedLinear:
    """W4 weight: codes [N][K/2] u8, scales [G][N] fp16 bits (int16 tensor), zeros [G][N]
    fp16 bits (int16) or, with zeros_u4, packed uint8 [G][N/2] (SQ_ZEROS_U4).

    static: the weights are final (inference).  GEMMs on this handle then pass
    SQ_GEMM_WEIGHTS_STATIC, letting the kernel stream its first weight stages before the
    previous kernel on the stream has finished.  A freshly quantized handle is not static
    until the caller says so (mark_static), because the quantize kernel that wrote it may
    still be running."""
    Wq: torch.Tensor
    scales: torch.Tensor
    zeros: torch.Tensor
    N: int
    K: int
    group: int = GROUP
    static: bool = False
    zeros_u4: bool = False

    def mark_static(self, static: bool = True) -> "QuantizedLinear":
        self.static = static
        return self

    @property
    def flags(self) -> int:
        return (SQ_GEMM_WEIGHTS_STATIC if self.static else 0) | (SQ_ZEROS_U4 if self.zeros_u4 else 0)

    def nbytes(self) -> int:
        return self.Wq.numel() + 2 * self.scales.numel() + self.zeros.numel() * self.zeros.element_size()


def quantize_pack_groupwise(W: torch.Tensor, s: torch.Tensor | None = None, group: int = GROUP,
                            nonfinite: torch.Tensor | None = None, stream=None,
                            zeros_u4: bool = False) -> QuantizedLinear:
    """Eq. 5 fold (W' = RN(W·s)) + Eq. 1 group-wise INT4 quantization and packing;
    zeros_u4: Z packed two per byte along n (SQ_ZEROS_U4, N % 32 == 0)."""
    _need_cuda(W, s, nonfinite)
    N, K = W.shape
    dev = W.device
    _check_vec(s, K, "s")
    if nonfinite is not None and (nonfinite.dtype != torch.int32 or nonfinite.numel() < 1):
        raise ValueError("nonfinite: need an int32 device counter")
    Wq = torch.empty((N, K // 2), dtype=torch.uint8, device=dev)
    scales = torch.empty((K // group, N), dtype=torch.int16, device=dev)
    if zeros_u4:
        zeros = torch.empty((K // group, N // 2), dtype=torch.uint8, device=dev)
    else:
        zeros = torch.empty((K // group, N), dtype=torch.int16, device=dev)
    _check(_load().sq_quantize_pack_groupwise_ex(_ptr(W), _dtype_code(W), _ptr(s), N, K, group, _ptr(Wq),
                                                 _ptr(scales), _ptr(zeros), _ptr(nonfinite),
                                                 SQ_ZEROS_U4 if zeros_u4 else 0, _stream(stream)))
    return QuantizedLinear(Wq, scales, zeros, N, K, group, zeros_u4=zeros_u4)


def w4a16_gemm_workspace_bytes(M: int, N: int, K: int, group: int = GROUP) -> int:
    return int(_load().sq_w4a16_gemm_workspace_bytes(M, N, K, group))


def workspace_reset(ws: torch.Tensor, stream=None) -> None:
    """Zero a GEMM workspace or all-reduce buffer on the stream (sq_workspace_reset)."""
    _need_cuda(ws)
    _check(_load().sq_workspace_reset(_ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


_WS: dict = {}


def default_workspace(device, nbytes: int) -> torch.Tensor:
    """A zero-filled per-device workspace, grown on demand (plumbing only: one
    workspace per device means GEMMs on one device must share a stream)."""
    key = torch.device(device).index if torch.device(device).index is not None else torch.cuda.current_device()
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def w4a16_gemm(X: torch.Tensor, q: QuantizedLinear, out: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None, path: int = SQ_PATH_AUTO,
               stream=None) -> torch.Tensor:
    """Eq. 3: Y[M][N] = X[M][K] · dequant(q)^T, fp32 accumulate, Y in X's dtype."""
    _need_cuda(X, out, workspace)
    M, K = X.shape
    if K != q.K:
        raise ValueError(f"K mismatch: X has {K}, weight has {q.K}")
    _check_out(out, (M, q.N), X.dtype, X.device)
    if out is None:
        out = torch.empty((M, q.N), dtype=X.dtype, device=X.device)
    if workspace is None:
        need = w4a16_gemm_workspace_bytes(M, q.N, K, q.group)
        if need:
            workspace = default_workspace(X.device, need)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(_load().sq_w4a16_gemm_ex(_ptr(X), _dtype_code(X), _ptr(q.Wq), _ptr(q.scales), _ptr(q.zeros),
                                    _ptr(out), M, q.N, K, q.group, _ptr(workspace), ws_bytes, int(path),
                                    q.flags, _stream(stream)))
    return out


def smooth_activations(X: torch.Tensor, s: torch.Tensor, out: torch.Tensor | None = None,
                       stream=None) -> torch.Tensor:
    """X̂ = RN(X / s) per input channel (activation side of Eq. 5); out may be X (in place)."""
    _need_cuda(X, s, out)
    M, K = X.shape
    _check_vec(s, K, "s")
    _check_out(out, (M, K), X.dtype, X.device)
    if out is None:
        out = torch.empty_like(X)
    _check(_load().sq_smooth_activations(_ptr(X), _dtype_code(X), _ptr(s), M, K, _ptr(out), _stream(stream)))
    return out


def sq_diff_sum(A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None,
                workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Σ (A - B)² in fp64 (the squared norm of Eq. 4), deterministic; returns a device
    float64 scalar tensor (no host sync)."""
    _need_cuda(A, B)
    if A.shape != B.shape or A.dtype != B.dtype:
        raise ValueError("sq_diff_sum: A and B need the same shape and dtype")
    L = _load()
    nb = L.sq_sq_diff_sum_workspace_bytes()
    if workspace is None:
        workspace = torch.empty(nb, dtype=torch.uint8, device=A.device)
    if out is None:
        out = torch.empty((), dtype=torch.float64, device=A.device)
    _check(L.sq_sq_diff_sum(_ptr(A), _ptr(B), _dtype_code(A), A.numel(), _ptr(out), _ptr(workspace),
                            workspace.numel() * workspace.element_size(), _stream(stream)))
    return out


def allreduce_buffer_bytes(n_max: int, world: int) -> int:
    return int(_load().sq_allreduce_buffer_bytes(int(n_max), int(world)))


def allreduce_oneshot(y_local: torch.Tensor, peers_dev: torch.Tensor, rank: int, world: int, epoch: int,
                      n_max: int, error_flag: torch.Tensor, out: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """One-shot all-reduce of the row-parallel partial y_local over peer memory
    (include/libsq.h sq_allreduce_oneshot).  peers_dev: int64 device tensor of the world
    symmetric-buffer addresses as mapped in this process."""
    _need_cuda(y_local, peers_dev, error_flag, out)
    _check_out(out, tuple(y_local.shape), y_local.dtype, y_local.device)
    if y_local.numel() > n_max:
        raise ValueError(f"allreduce: {y_local.numel()} elements > n_max {n_max}")
    if out is None:
        out = y_local
    _check(_load().sq_allreduce_oneshot(_ptr(y_local), _dtype_code(y_local), _ptr(out), y_local.numel(),
                                        int(n_max), _ptr(peers_dev), int(rank), int(world),
                                        ctypes.c_uint32(epoch & 0xFFFFFFFF), _ptr(error_flag), _stream(stream)))
    return out


def ipc_get_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(handle bytes, byte offset of t inside its cudaMalloc block)."""
    L = _load()
    buf = ctypes.create_string_buffer(L.sq_ipc_handle_bytes())
    off = ctypes.c_size_t(0)
    _check(L.sq_ipc_get_handle(_ptr(t), buf, ctypes.byref(off)))
    return buf.raw, int(off.value)


def ipc_open_handle(handle: bytes) -> int:
    """Map a peer's block; returns its base device address in this process."""
    p = ctypes.c_void_p()
    _check(_load().sq_ipc_open_handle(ctypes.create_string_buffer(handle, len(handle)), ctypes.byref(p)))
    return int(p.value)


def ipc_close(addr: int) -> None:
    _check(_load().sq_ipc_close(ctypes.c_void_p(addr)))


def w4a16_gemm_allreduce(X: torch.Tensor, q: QuantizedLinear, peers_dev: torch.Tensor, rank: int, world: int,
                         n_max: int, error_flag: torch.Tensor, epoch: int = 0, out: torch.Tensor | None = None,
                         workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Row-parallel W4A16 linear + all-reduce over peer memory: Y = sum over ranks of
    X_r · dequant(q_r)^T, identical on every rank (sq_w4a16_gemm_allreduce; one kernel for
    decode sizes)."""
    _need_cuda(X, out, workspace, peers_dev, error_flag)
    M, K = X.shape
    if K != q.K:
        raise ValueError(f"K mismatch: X has {K}, weight has {q.K}")
    _check_out(out, (M, q.N), X.dtype, X.device)
    if out is None:
        out = torch.empty((M, q.N), dtype=X.dtype, device=X.device)
    if workspace is None:
        need = w4a16_gemm_workspace_bytes(M, q.N, K, q.group)
        if need:
            workspace = default_workspace(X.device, need)
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(_load().sq_w4a16_gemm_allreduce(_ptr(X), _dtype_code(X), _ptr(q.Wq), _ptr(q.scales), _ptr(q.zeros),
                                           _ptr(out), M, q.N, K, q.group, _ptr(workspace), ws_bytes,
                                           _ptr(peers_dev), int(rank), int(world), int(n_max),
                                           ctypes.c_uint32(epoch & 0xFFFFFFFF), _ptr(error_flag), q.flags,
                                           _stream(stream)))
    return out


def fold_rows(W: torch.Tensor, d: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """W_out[n][k] = RN(W[n][k] / d[n]): fold the consumer's smoothing factors into the
    producer linear's output rows (Fig. 5); out may be W (in place)."""
    _need_cuda(W, d, out)
    N, K = W.shape
    _check_vec(d, N, "d")
    _check_out(out, (N, K), W.dtype, W.device)
    if out is None:
        out = torch.empty_like(W)
    _check(_load().sq_fold_rows(_ptr(W), _dtype_code(W), _ptr(d), N, K, _ptr(out), _stream(stream)))
    return out
