"""ctypes binding of the native library (`libparadiff_b200.so`, include/paradiff_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every solver entry point raises.  Device buffers are torch CUDA
tensors (torch is the allocator/stream plumbing); the C ABI sees raw device
pointers only.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import ConfigurationError, DeviceError, SolverError

LIB_PATH = Path(os.environ.get("PD_LIB") or Path(__file__).resolve().parent / "libparadiff_b200.so")

PD_OK, PD_ERR_CONFIG, PD_ERR_SOLVER, PD_ERR_CUDA = 0, 1, 2, 3

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_int = ctypes.c_int
_dbl = ctypes.c_double


class SolveReportC(ctypes.Structure):
    _fields_ = [("iterations", _i32), ("converged", _i32), ("diverged", _i32),
                ("hist_len", _i32)]


_SIGNATURES = {
    "pd_last_error": (ctypes.c_char_p, []),
    "pd_last_error_index": (_i64, []),
    "pd_version": (_int, []),
    "pd_launch_count": (ctypes.c_uint64, []),
    "pd_mg_level_precond": (_int, [_vp, _int, ctypes.POINTER(_vp)]),
    "pd_ctx_create": (_int, [_int, _vp, ctypes.POINTER(_vp)]),
    "pd_ctx_set_stream": (_int, [_vp, _vp]),
    "pd_ctx_destroy": (_int, [_vp]),
    "pd_csr_create": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _int, ctypes.POINTER(_vp)]),
    "pd_csr_set_values": (_int, [_vp, _vp, _vp, _int]),
    "pd_csr_spmv": (_int, [_vp, _vp, _vp, _vp, _int, _vp]),
    "pd_csr_destroy": (_int, [_vp]),
    "pd_ilu0_create": (_int, [_vp, _vp, _int, ctypes.POINTER(_vp)]),
    "pd_ilu0_refactor": (_int, [_vp, _vp]),
    "pd_ilu0_solve": (_int, [_vp, _vp, _vp, _vp]),
    "pd_ilu0_levels": (_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "pd_ilu0_set_wavefront": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, ctypes.POINTER(_int)]),
    "pd_ilu0_sweep_kind": (_int, [_vp, ctypes.POINTER(_int)]),
    "pd_ilu0_factor_values": (_int, [_vp, _vp, _vp, _i64]),
    "pd_csr_set_grid": (_int, [_vp, _vp, _i64, _int, _i64, ctypes.POINTER(_int)]),
    "pd_ilu0_destroy": (_int, [_vp]),
    "pd_dense_lu_create": (_int, [_vp, _vp, ctypes.POINTER(_vp)]),
    "pd_dense_lu_solve": (_int, [_vp, _vp, _vp, _vp]),
    "pd_dense_lu_destroy": (_int, [_vp]),
    "pd_gmres": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _int, _int,
                        ctypes.POINTER(SolveReportC), _vp, _int]),
    "pd_mg_create": (_int, [_vp, _int, _vp, _vp, _vp, _int, _int, _int, _int,
                            ctypes.POINTER(_vp)]),
    "pd_mg_level_matrix": (_int, [_vp, _int, ctypes.POINTER(_vp)]),
    "pd_mg_refactor": (_int, [_vp, _vp]),
    "pd_mg_vcycle": (_int, [_vp, _vp, _vp, _vp]),
    "pd_mg_solve": (_int, [_vp, _vp, _vp, _vp, _dbl, _dbl, _int, ctypes.POINTER(SolveReportC),
                           _vp, _int]),
    "pd_mg_destroy": (_int, [_vp]),
    "pd_pfast_create": (_int, [_vp, _int, _i64, _int, _dbl, _int, _i64, _dbl, _vp, _vp, _vp,
                               _int, _int, _int, _dbl, _dbl, ctypes.POINTER(_vp)]),
    "pd_pfast_residual": (_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pd_pfast_sweep": (_int, [_vp, _vp, _vp, _vp]),
    "pd_pfast_solve": (_int, [_vp, _vp, _vp, _vp, _dbl, _dbl, _int, ctypes.POINTER(SolveReportC),
                              _vp]),
    "pd_pfast_nl_residual": (_int, [_vp, _vp, _vp, _vp, _vp, _dbl, _int, _vp]),
    "pd_pfast_set_state": (_int, [_vp, _vp, _dbl, _int]),
    "pd_pfast_st_create": (_int, [_vp, _int, _int, _dbl, _int, _vp, _vp, _vp, _int, _vp, _vp, _vp,
                                  _vp, _vp, _vp, _vp, _vp, _int, _int, _int, _int, _dbl, _dbl,
                                  ctypes.POINTER(_vp)]),
    "pd_pfast_st_destroy": (_int, [_vp]),
    "pd_pfast_st_set_state": (_int, [_vp, _vp, _dbl, _int]),
    "pd_pfast_st_cycle": (_int, [_vp, _vp, _vp]),
    "pd_pfast_st_solve": (_int, [_vp, _vp, _vp, _dbl, _dbl, _int, ctypes.POINTER(SolveReportC),
                                 _vp]),
    "pd_pfast_st_level_plan": (_int, [_vp, _int, ctypes.POINTER(_vp)]),
    "pd_pfast_st_level_sweep": (_int, [_vp, _int, _vp, _vp, _vp]),
    "pd_pfast_st_level_restrict": (_int, [_vp, _int, _vp, _vp, _vp]),
    "pd_pfast_st_level_prolong": (_int, [_vp, _int, _vp]),
    "pd_pfast_st_level_last": (_int, [_vp, _int, _vp, _vp]),
    "pd_pfast_destroy": (_int, [_vp]),
    "pd_mg_set_fine_operator": (_int, [_vp, _vp]),
    "pd_mg_set_galerkin_intermediates": (_int, [_vp, _int, _vp]),
    "pd_mg_set_fine_values": (_int, [_vp, _vp]),
    "pd_jacobian_values": (_int, [_vp, _i64, _int, _i64, _dbl, _dbl, _int, _vp, _vp, _vp, _vp,
                                  _vp]),
    "pd_stop_create": (_int, [_vp, _i64, _int, _i64, _vp, _vp, _vp, _dbl, _vp, _vp,
                              ctypes.POINTER(_vp)]),
    "pd_stop_destroy": (_int, [_vp]),
    "pd_stop_apply": (_int, [_vp, _vp, _vp, _int, _vp, _vp]),
    "pd_stop_residual": (_int, [_vp, _vp, _vp, _vp, _dbl, _int]),
    "pd_st_residual_csr": (_int, [_vp, _vp, _vp, _dbl, _int, _vp, _vp, _vp, _vp]),
    "pd_reaction": (_int, [_vp, _int, _int, _vp, _vp, _i64]),
    "pd_axpy_to": (_int, [_vp, _vp, _vp, _vp, _dbl, _i64]),
    "pd_norm": (_int, [_vp, _vp, _i64, ctypes.POINTER(_dbl)]),
    "pd_dot": (_int, [_vp, _vp, _vp, _i64, ctypes.POINTER(_dbl)]),
    "pd_sdc_level_create": (_int, [_vp, _vp, _vp, _int, _vp, _vp, _vp, _dbl, _dbl, _int, _int,
                                   _int, _vp, _vp, _int, _i64, _dbl, ctypes.POINTER(_vp)]),
    "pd_sdc_level_destroy": (_int, [_vp]),
    "pd_sdc_sweep": (_int, [_vp, _vp, _vp, _vp, _int]),
    "pd_sdc_chain": (_int, [_vp, _vp, _vp, _vp, _int, _vp, _int]),
    "pd_sdc_residual": (_int, [_vp, _vp, _vp, _vp, _int, _vp]),
    "pd_sdc_coll_op": (_int, [_vp, _vp, _vp, _int]),
    "pd_sdc_errors": (_int, [_vp, ctypes.POINTER(_int)]),
    "pd_node_mix": (_int, [_vp, _vp, _vp, _int, _int, _int, _i64, _vp, _int]),
    "pd_csr_spmm": (_int, [_vp, _vp, _vp, _i64, _vp, _i64, _int, _int]),
    "pd_sub": (_int, [_vp, _vp, _vp, _vp, _i64]),
    "pd_spread": (_int, [_vp, _vp, _vp, _vp, _int, _int, _i64]),
    "pd_terminal": (_int, [_vp, _vp, _vp, _int, _int, _i64]),
    "pd_scale": (_int, [_vp, _vp, _vp, _dbl, _i64]),
    "pd_mode_product": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _int]),
    "pd_band_lu_create": (_int, [_vp, _vp, _int, _int, _vp, ctypes.POINTER(_vp)]),
    "pd_band_lu_solve": (_int, [_vp, _vp, _vp, _vp]),
    "pd_band_lu_destroy": (_int, [_vp]),
    "pd_gms_create": (_int, [_vp, _i64, _int, ctypes.POINTER(_vp)]),
    "pd_gms_destroy": (_int, [_vp]),
    "pd_gms_init": (_int, [_vp, _vp, _vp]),
    "pd_gms_begin": (_int, [_vp, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                            ctypes.POINTER(_vp)]),
    "pd_gms_dots": (_int, [_vp, ctypes.POINTER(_vp)]),
    "pd_gms_mgs_pass": (_int, [_vp, _int]),
    "pd_gms_end": (_int, [_vp, _int]),
    "pd_gms_apply": (_int, [_vp, _vp]),
    "pd_gms_error": (_int, [_vp, ctypes.POINTER(_int)]),
    "pd_dot_dev": (_int, [_vp, _vp, _vp, _i64, _vp]),
    "pd_gmres_callable": (_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _dbl,
                                 _dbl, _int, _int, ctypes.POINTER(SolveReportC), _vp, _int]),
}

APPLY_CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)

_lock = threading.Lock()
_LIB = None


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


def load_library(path: Path | None = None) -> ctypes.CDLL:
    """Load and type the native library (no GPU needed just to load it)."""
    global _LIB
    with _lock:
        if _LIB is not None and path is None:
            return _LIB
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"native library {p} not built; run `python -c 'import __graft_entry__ as g; "
                "g.build()'` (no CPU fallback exists)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _LIB = lib
        return lib


def check(status: int) -> None:
    if status == PD_OK:
        return
    lib = load_library()
    msg = (lib.pd_last_error() or b"").decode()
    if status == PD_ERR_CONFIG:
        raise ConfigurationError(msg)
    if status == PD_ERR_SOLVER:
        err = SolverError(msg)
        err.index = int(lib.pd_last_error_index())
        raise err
    raise DeviceError(msg)


def call(name: str, *args) -> None:
    check(getattr(load_library(), name)(*args))


# ------------------------------------------------------------------ device context
_torch = None


def torch_mod():
    global _torch
    if _torch is None:
        import torch

        _torch = torch
    return _torch


class Context:
    """One native context per CUDA device, bound to torch's current stream."""

    def __init__(self, device: int):
        torch = torch_mod()
        self.device = device
        self.torch_device = torch.device("cuda", device)
        self._stream = torch.cuda.current_stream(self.torch_device)
        h = _vp()
        call("pd_ctx_create", device, _vp(self._stream.cuda_stream), ctypes.byref(h))
        self.handle = h

    def sync_stream(self) -> None:
        """Rebind to torch's current stream (cheap; call before enqueueing)."""
        torch = torch_mod()
        s = torch.cuda.current_stream(self.torch_device)
        if s.cuda_stream != self._stream.cuda_stream:
            self._stream = s
            call("pd_ctx_set_stream", self.handle, _vp(s.cuda_stream))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                load_library().pd_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def require_cuda() -> None:
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: paradiff-b200 has no CPU fallback")


def context(device: int | None = None) -> Context:
    require_cuda()
    torch = torch_mod()
    if device is None:
        device = torch.cuda.current_device()
    ctx = _contexts.get(device)
    if ctx is None:
        load_library()
        ctx = Context(device)
        _contexts[device] = ctx
    ctx.sync_stream()
    return ctx


# ------------------------------------------------------------------ array helpers
def ptr(t) -> _vp:
    return _vp(t.data_ptr()) if t is not None else _vp()


# Large numpy vectors (a C2 space-time vector is 100 MB) cross the host/device
# boundary through a reusable pinned staging buffer in chunks: host threads copy
# chunk i between numpy and pinned memory while the DMA of its neighbours runs.
# A pageable torch copy runs at a few GB/s; the staged copy runs near the
# link's rate.  PD_STAGED_IO=0 turns it off.
_STAGE_MIN_BYTES = 1 << 23
_STAGE_CHUNK = 1 << 20  # doubles per chunk (8 MB)
_stage_lock = threading.Lock()
_stage_bufs: dict = {}  # (device index, direction) -> [pinned tensor, pending event or None]
_stage_pool = None


def _staging_enabled(nbytes: int) -> bool:
    return nbytes >= _STAGE_MIN_BYTES and os.environ.get("PD_STAGED_IO", "1") != "0"


def _pool():
    global _stage_pool
    if _stage_pool is None:
        from concurrent.futures import ThreadPoolExecutor

        _stage_pool = ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1)),
                                         thread_name_prefix="pd-stage")
    return _stage_pool


def _staging(ctx, direction: str, n: int):
    """The pinned buffer for (device, direction), at least n doubles; waits for
    the DMA that last used it."""
    torch = torch_mod()
    key = (ctx.device, direction)
    ent = _stage_bufs.get(key)
    if ent is None or ent[0].numel() < n:
        if ent is not None and ent[1] is not None:
            ent[1].synchronize()
        ent = [torch.empty(n, dtype=torch.float64, pin_memory=True), None]
        _stage_bufs[key] = ent
    elif ent[1] is not None:
        ent[1].synchronize()
        ent[1] = None
    return ent


def _chunks(n: int):
    return [(lo, min(n, lo + _STAGE_CHUNK)) for lo in range(0, n, _STAGE_CHUNK)]


def _h2d_staged(a: np.ndarray, ctx):
    torch = torch_mod()
    n = a.size
    out = torch.empty(n, dtype=torch.float64, device=ctx.torch_device)
    with _stage_lock:
        ent = _staging(ctx, "h2d", n)
        buf = ent[0]
        host = buf.numpy()
        parts = _chunks(n)
        futs = [_pool().submit(np.copyto, host[lo:hi], a[lo:hi]) for lo, hi in parts]
        for f, (lo, hi) in zip(futs, parts):
            f.result()
            out[lo:hi].copy_(buf[lo:hi], non_blocking=True)
        # complete on return, like a pageable copy: the caller may hand `out` to
        # work on any stream
        torch.cuda.current_stream(out.device).synchronize()
    return out


def _d2h_staged(t) -> np.ndarray:
    torch = torch_mod()
    n = t.numel()
    res = np.empty(n, dtype=np.float64)
    src = t.reshape(-1)
    with _stage_lock, torch.cuda.device(t.device):
        ent = _staging(context(t.device.index), "d2h", n)
        buf = ent[0]
        host = buf.numpy()
        parts = _chunks(n)
        evs = []
        for lo, hi in parts:
            buf[lo:hi].copy_(src[lo:hi], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            evs.append(ev)

        def drain(i):
            lo, hi = parts[i]
            evs[i].synchronize()
            np.copyto(res[lo:hi], host[lo:hi])

        for f in [_pool().submit(drain, i) for i in range(len(parts))]:
            f.result()
    return res.reshape(tuple(t.shape))


def to_device(x, ctx: Context | None = None):
    """numpy / torch -> contiguous float64 CUDA tensor on the context's device."""
    torch = torch_mod()
    ctx = ctx or context()
    if isinstance(x, torch.Tensor):
        t = x.to(device=ctx.torch_device, dtype=torch.float64)
        return t.contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if a.ndim == 1 and _staging_enabled(a.nbytes):
        return _h2d_staged(a, ctx)
    return torch.from_numpy(a).to(ctx.torch_device)


def to_host(t) -> np.ndarray:
    """CUDA tensor -> numpy (staged through pinned memory when large)."""
    if t.is_cuda and t.dtype == torch_mod().float64 and t.is_contiguous() and \
            _staging_enabled(t.numel() * 8):
        return _d2h_staged(t)
    return t.cpu().numpy()


def empty(n: int, ctx: Context | None = None):
    torch = torch_mod()
    ctx = ctx or context()
    return torch.empty(int(n), dtype=torch.float64, device=ctx.torch_device)


def zeros(n: int, ctx: Context | None = None):
    torch = torch_mod()
    ctx = ctx or context()
    return torch.zeros(int(n), dtype=torch.float64, device=ctx.torch_device)


def norm(x, ctx: Context | None = None) -> float:
    """||x||_2 of a CUDA tensor via the native deterministic reduction."""
    ctx = ctx or context()
    out = _dbl()
    call("pd_norm", ctx.handle, ptr(x), int(x.numel()), ctypes.byref(out))
    return float(out.value)


class _DeviceSpan:
    """A raw device pointer as a CUDA array (torch.as_tensor wraps it without a copy)."""

    def __init__(self, address: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(address), False), "version": 2}


def view(address, count: int, ctx: Context | None = None):
    """fp64 tensor view of `count` doubles at a device address owned by the library."""
    ctx = ctx or context()
    addr = address.value if hasattr(address, "value") else int(address)
    return torch_mod().as_tensor(_DeviceSpan(addr, count), device=ctx.torch_device)


def dot(x, y, ctx: Context | None = None) -> float:
    """x . y of two CUDA tensors via the native deterministic reduction."""
    ctx = ctx or context()
    out = _dbl()
    call("pd_dot", ctx.handle, ptr(x), ptr(y), int(x.numel()), ctypes.byref(out))
    return float(out.value)


def scale_into(y, x, s: float, ctx: Context | None = None):
    ctx = ctx or context()
    call("pd_scale", ctx.handle, ptr(y), ptr(x), float(s), int(x.numel()))
    return y


def is_tensor(x) -> bool:
    torch = torch_mod()
    return isinstance(x, torch.Tensor)


def like_input(result, template, out=None):
    """Hand a device result back in the caller's form: into `out` when given
    (e.g. a pinned host tensor: one DMA, no allocation); a tensor on the
    template's device for tensor inputs (host tensors come back on the host);
    numpy for numpy inputs."""
    if out is not None:
        out.copy_(result.view_as(out) if out.shape != result.shape else result)
        return out
    if is_tensor(template):
        return result if template.is_cuda else result.cpu()
    return to_host(result)
