"""B200-native Fast Haar Wavelet Transform (arXiv 1002.2184) — thin Python binding.

Every function here only marshals arguments (tensor -> device pointer, current CUDA stream ->
cudaStream_t, status -> exception) and calls the C ABI of ``libfhwt.so`` (include/fhwt.h),
whose sm_100a kernels do all of the arithmetic.  There is no CPU or PyTorch fallback: inputs
must be contiguous float32 CUDA tensors, and a missing library raises ``FhwtLibraryError``.

Names follow the C ABI: analyze_1d / synthesize_1d / analyze_2d / synthesize_2d, Plan1d / Plan2d
(plan handles), pack_ll_2d, roundtrip_2d_host / roundtrip_1d_host, band_offset_1d/2d.
"""
from __future__ import annotations

import ctypes
import os

__all__ = [
    "FhwtError", "FhwtLibraryError", "OddLength", "EmptySignal", "InvalidLevels", "InsufficientLength",
    "ShapeMismatch", "UnsupportedFilter", "Misaligned", "CudaError", "NoDevice", "InvalidArgument",
    "lib", "lib_path", "haar_filter_bank", "launch_count", "version",
    "analyze_1d", "synthesize_1d", "analyze_2d", "synthesize_2d", "Plan1d", "Plan2d",
    "pack_ll_2d", "pack_ll_2d_peers", "roundtrip_2d_host", "roundtrip_1d_host", "band_offset_1d", "band_offset_2d",
    "direct_workspace_bytes", "direct_analyze_1d", "direct_synthesize_1d", "direct_analyze_2d",
    "direct_synthesize_2d", "op_counts", "lowpass_2d_u8", "lowpass_2d_bf16",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# FHWT_LIB (A/B of two builds in the tuning sweeps) is honoured only with FHWT_TUNING=1, like the
# library's own FHWT_* knobs.
lib_path = ((os.environ.get("FHWT_LIB") if os.environ.get("FHWT_TUNING") == "1" else None)
            or os.path.join(_HERE, "libfhwt.so"))


class FhwtError(RuntimeError):
    status = -1


class FhwtLibraryError(FhwtError):
    pass


class InvalidArgument(FhwtError, ValueError):
    status = 1


class EmptySignal(FhwtError, ValueError):
    status = 2


class OddLength(FhwtError, ValueError):
    status = 3


class InvalidLevels(FhwtError, ValueError):
    status = 4


class InsufficientLength(FhwtError, ValueError):
    status = 5


class ShapeMismatch(FhwtError, ValueError):
    status = 6


LengthMismatch = DimensionMismatch = ShapeMismatch


class UnsupportedFilter(FhwtError, ValueError):
    status = 7


class Misaligned(FhwtError, ValueError):
    status = 8


class CudaError(FhwtError):
    status = 9


class NoDevice(FhwtError):
    status = 10


_BY_STATUS = {c.status: c for c in (InvalidArgument, EmptySignal, OddLength, InvalidLevels, InsufficientLength,
                                      ShapeMismatch, UnsupportedFilter, Misaligned, CudaError, NoDevice)}


class FilterBank(ctypes.Structure):
    """fhwt_filter_bank: the paper's problem statement (b0, b1, a0, a1, M) — PAPER.md:54, :88."""
    _fields_ = [("b0", ctypes.c_double * 2), ("b1", ctypes.c_double * 2), ("a0", ctypes.c_double * 2),
                ("a1", ctypes.c_double * 2), ("M", ctypes.c_int)]


_lib = None


def lib():
    """Load (building in-tree first if the sources are newer) libfhwt.so."""
    global _lib
    if _lib is not None:
        return _lib
    try:
        from . import _build
        if _build.stale():
            _build.build()
    except Exception as e:  # noqa: BLE001 - surface as a library error below if the .so is unusable
        if not os.path.exists(lib_path):
            raise FhwtLibraryError(f"libfhwt.so is missing and could not be built: {e}") from e
    if not os.path.exists(lib_path):
        raise FhwtLibraryError(f"{lib_path} not found; run `python -m paper_1002_2184_b200._build`")
    L = ctypes.CDLL(lib_path)
    i64, c_int, vp, st = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int
    sig = {
        "fhwt_haar_filter_bank": (st, [ctypes.POINTER(FilterBank)]),
        "fhwt_status_string": (ctypes.c_char_p, [st]),
        "fhwt_last_error_message": (ctypes.c_char_p, []),
        "fhwt_version": (c_int, []),
        "fhwt_launch_count": (ctypes.c_uint64, []),
        "fhwt_plan_1d": (st, [ctypes.POINTER(vp), i64, i64, c_int, ctypes.POINTER(FilterBank), c_int]),
        "fhwt_plan_2d": (st, [ctypes.POINTER(vp), i64, i64, i64, c_int, ctypes.POINTER(FilterBank), c_int]),
        "fhwt_plan_destroy": (st, [vp]),
        "fhwt_plan_workspace_bytes": (ctypes.c_size_t, [vp]),
        "fhwt_plan_analyze": (st, [vp, vp, vp, vp, vp]),
        "fhwt_plan_synthesize": (st, [vp, vp, vp, vp, vp]),
        "fhwt_analyze_1d": (st, [vp, vp, i64, i64, c_int, vp]),
        "fhwt_synthesize_1d": (st, [vp, vp, i64, i64, c_int, vp]),
        "fhwt_analyze_2d": (st, [vp, vp, i64, i64, i64, c_int, vp]),
        "fhwt_synthesize_2d": (st, [vp, vp, i64, i64, i64, c_int, vp]),
        "fhwt_band_offset_1d": (i64, [i64, c_int, c_int, ctypes.POINTER(i64)]),
        "fhwt_band_offset_2d": (i64, [i64, i64, c_int, c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "fhwt_pack_ll_2d": (st, [vp, vp, i64, i64, i64, c_int, vp]),
        "fhwt_plan_pack_ll_2d": (st, [vp, vp, vp, vp]),
        "fhwt_pack_ll_2d_peers": (st, [vp, vp, c_int, c_int, i64, i64, i64, c_int, vp]),
        "fhwt_workspace_bytes": (ctypes.c_size_t, [vp]),
        "fhwt_analyze": (st, [vp, vp, vp, vp, vp]),
        "fhwt_synthesize": (st, [vp, vp, vp, vp, vp]),
        "fhwt_roundtrip_2d_host": (st, [vp, vp, vp, i64, i64, i64, c_int, i64]),
        "fhwt_roundtrip_1d_host": (st, [vp, vp, vp, i64, i64, c_int, i64]),
        "fhwt_direct_workspace_bytes": (ctypes.c_size_t, [c_int, i64, i64, i64]),
        "fhwt_lowpass_workspace_bytes": (ctypes.c_size_t, [i64, i64, i64, c_int]),
        "fhwt_lowpass_2d_u8": (st, [vp, vp, i64, i64, i64, c_int, vp, vp]),
        "fhwt_lowpass_bf16_workspace_bytes": (ctypes.c_size_t, [i64, i64, i64, c_int]),
        "fhwt_lowpass_2d_bf16": (st, [vp, vp, i64, i64, i64, c_int, vp, vp]),
        "fhwt_direct_analyze_1d": (st, [vp, vp, i64, i64, c_int, vp, vp]),
        "fhwt_direct_synthesize_1d": (st, [vp, vp, i64, i64, c_int, vp, vp]),
        "fhwt_direct_analyze_2d": (st, [vp, vp, i64, i64, i64, c_int, vp, vp]),
        "fhwt_direct_synthesize_2d": (st, [vp, vp, i64, i64, i64, c_int, vp, vp]),
        "fhwt_op_counts": (st, [c_int, i64, i64, i64, c_int, c_int, c_int, ctypes.POINTER(ctypes.c_uint64),
                                ctypes.POINTER(ctypes.c_uint64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(status: int):
    if status == 0:
        return
    L = lib()
    msg = L.fhwt_last_error_message().decode(errors="replace")
    name = L.fhwt_status_string(status).decode()
    raise _BY_STATUS.get(status, FhwtError)(f"{name}: {msg}")


def version() -> int:
    return lib().fhwt_version()


def launch_count() -> int:
    """Number of kernels libfhwt.so has launched in this process."""
    return int(lib().fhwt_launch_count())


def haar_filter_bank() -> FilterBank:
    fb = FilterBank()
    _check(lib().fhwt_haar_filter_bank(ctypes.byref(fb)))
    return fb


# ------------------------------------------------------------------ tensor marshalling
# Per-call host cost matters for the latency-bound configs (c1, c3): the helpers below use
# torch's raw current-stream / current-device queries and plain attribute checks (a call costs
# ~2 us of Python on top of the C ABI call).
_torch = None


def _t():
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    return _torch


def _stream(stream, t=None):
    torch = _t()
    if stream is None:
        dev = t.get_device() if t is not None else torch._C._cuda_getDevice()
        return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(dev))
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_f32(t, what):
    torch = _t()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what} must be a torch.Tensor")
    if not t.is_cuda:
        raise InvalidArgument(f"{what} must be a CUDA tensor (this library has no CPU path)")
    if t.dtype is not torch.float32:
        raise InvalidArgument(f"{what} must be float32, got {t.dtype}")
    if not t.is_contiguous():
        raise InvalidArgument(f"{what} must be contiguous")
    return t.data_ptr()


def _out_like(x, out):
    if out is None:
        return _t().empty_like(x)
    if out.shape != x.shape:
        raise ShapeMismatch(f"out has shape {tuple(out.shape)}, expected {tuple(x.shape)}")
    if out.device != x.device:
        raise InvalidArgument(f"out is on {out.device}, input on {x.device}")
    return out


def _out_packed(out, numel, device, what):
    """A caller-supplied output the kernel fills with `numel` elements: check its size and device
    before the C ABI writes (an undersized buffer would be an out-of-bounds device write)."""
    if out.numel() != numel:
        raise ShapeMismatch(f"{what} has {out.numel()} elements, expected {numel}")
    if out.device != device:
        raise InvalidArgument(f"{what} is on {out.device}, expected {device}")
    return out


def _shape_1d(x):
    if x.dim() < 1:
        raise InvalidArgument("1-D transform needs at least one dimension")
    n = x.shape[-1]
    return n, (x.numel() // n if n else 0)


def _shape_2d(x):
    if x.dim() < 2:
        raise InvalidArgument("2-D transform needs at least two dimensions")
    h, w = x.shape[-2], x.shape[-1]
    return h, w, (x.numel() // (h * w) if h * w else 0)


class _NoGuard:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NO_GUARD = _NoGuard()


def _guard_device(x):
    """Context that makes x's device current for the call (a no-op when it already is)."""
    torch = _t()
    _dev_f32(x, "input")          # validate (CUDA, float32, contiguous) before touching the device
    dv = x.get_device()
    if dv == torch._C._cuda_getDevice():
        return _NO_GUARD
    return torch.cuda.device(dv)


def analyze_1d(d, levels: int, out=None, stream=None):
    """fhwt_analyze_1d: multi-level Fast Haar analysis along the last axis -> Mallat layout."""
    n, batch = _shape_1d(d)
    out = _out_like(d, out)
    with _guard_device(d):
        _check(lib().fhwt_analyze_1d(_dev_f32(d, "d"), _dev_f32(out, "coeffs"), n, batch, int(levels), _stream(stream, d)))
    return out


def synthesize_1d(coeffs, levels: int, out=None, stream=None):
    """fhwt_synthesize_1d: inverse of analyze_1d (perfect reconstruction)."""
    n, batch = _shape_1d(coeffs)
    out = _out_like(coeffs, out)
    with _guard_device(coeffs):
        _check(lib().fhwt_synthesize_1d(_dev_f32(coeffs, "coeffs"), _dev_f32(out, "d_R"), n, batch, int(levels),
                                        _stream(stream, coeffs)))
    return out


def analyze_2d(d, levels: int, out=None, stream=None):
    """fhwt_analyze_2d: separable multi-level Fast Haar analysis of [..., h, w] -> Mallat quadrants."""
    h, w, batch = _shape_2d(d)
    out = _out_like(d, out)
    with _guard_device(d):
        _check(lib().fhwt_analyze_2d(_dev_f32(d, "d"), _dev_f32(out, "coeffs"), h, w, batch, int(levels),
                                     _stream(stream, d)))
    return out


def synthesize_2d(coeffs, levels: int, out=None, stream=None):
    """fhwt_synthesize_2d: inverse of analyze_2d."""
    h, w, batch = _shape_2d(coeffs)
    out = _out_like(coeffs, out)
    with _guard_device(coeffs):
        _check(lib().fhwt_synthesize_2d(_dev_f32(coeffs, "coeffs"), _dev_f32(out, "d_R"), h, w, batch, int(levels),
                                        _stream(stream, coeffs)))
    return out


def _device(device) -> int:
    """Plan device argument: None = the device current at each call (-1), else a CUDA index."""
    if device is None:
        return -1
    if hasattr(device, "index"):   # torch.device
        if device.type != "cuda":
            raise InvalidArgument(f"plan device must be a CUDA device, got {device}")
        return -1 if device.index is None else int(device.index)
    return int(device)


class _Plan:
    _kind = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.fhwt_plan_destroy(h)
            self._h = None

    @property
    def workspace_bytes(self) -> int:
        return int(lib().fhwt_plan_workspace_bytes(self._h))

    def _ws(self, like, workspace, stream):
        import torch
        nb = self.workspace_bytes
        if nb == 0:
            return ctypes.c_void_p(0)
        if workspace is None:
            # one cached buffer per (device, stream): calls on different streams may run
            # concurrently and must not share the pass hand-off region
            key = (like.get_device(), stream.value)
            cache = self.__dict__.setdefault("_ws_cache", {})
            ws = cache.get(key)
            if ws is None:
                ws = torch.empty(nb, dtype=torch.uint8, device=like.device)
                cache[key] = ws
            workspace = ws
        if workspace.numel() * workspace.element_size() < nb or not workspace.is_cuda:
            raise InvalidArgument(f"workspace must be a CUDA buffer of >= {nb} bytes")
        return ctypes.c_void_p(workspace.data_ptr())

    def _check_shape(self, x):
        if tuple(x.shape[-self._kind:]) != self._tail or x.numel() != self._numel:
            raise ShapeMismatch(f"tensor shape {tuple(x.shape)} does not match the plan {self._tail} x {self.batch}")

    def analyze(self, d, out=None, workspace=None, stream=None):
        self._check_shape(d)
        out = _out_like(d, out)
        with _guard_device(d):
            st = _stream(stream, d)
            _check(lib().fhwt_plan_analyze(self._h, _dev_f32(d, "d"), _dev_f32(out, "coeffs"),
                                           self._ws(d, workspace, st), st))
        return out

    def synthesize(self, coeffs, out=None, workspace=None, stream=None):
        self._check_shape(coeffs)
        out = _out_like(coeffs, out)
        with _guard_device(coeffs):
            st = _stream(stream, coeffs)
            _check(lib().fhwt_plan_synthesize(self._h, _dev_f32(coeffs, "coeffs"), _dev_f32(out, "d_R"),
                                              self._ws(coeffs, workspace, st), st))
        return out


class Plan1d(_Plan):
    """fhwt_plan_1d handle: batch signals of n samples, `levels` levels, filter bank (default §II)."""
    _kind = 1

    def __init__(self, n: int, batch: int, levels: int, filter_bank: FilterBank | None = None,
                 device: int | None = None):
        h = ctypes.c_void_p()
        _check(lib().fhwt_plan_1d(ctypes.byref(h), int(n), int(batch), int(levels),
                                  ctypes.byref(filter_bank) if filter_bank is not None else None, _device(device)))
        self._h = h
        self.n, self.batch, self.levels = int(n), int(batch), int(levels)
        self._tail = (self.n,)
        self._numel = self.n * self.batch


class Plan2d(_Plan):
    """fhwt_plan_2d handle: batch images of h x w, `levels` separable levels."""
    _kind = 2

    def __init__(self, h: int, w: int, batch: int, levels: int, filter_bank: FilterBank | None = None,
                 device: int | None = None):
        hd = ctypes.c_void_p()
        _check(lib().fhwt_plan_2d(ctypes.byref(hd), int(h), int(w), int(batch), int(levels),
                                  ctypes.byref(filter_bank) if filter_bank is not None else None, _device(device)))
        self._h = hd
        self.h, self.w, self.batch, self.levels = int(h), int(w), int(batch), int(levels)
        self._tail = (self.h, self.w)
        self._numel = self.h * self.w * self.batch

    def pack_ll(self, coeffs, out=None, stream=None):
        """fhwt_plan_pack_ll_2d: the coarsest LL of every image, packed [batch][h >> L][w >> L]."""
        self._check_shape(coeffs)
        torch = _t()
        L = self.levels
        if out is None:
            out = torch.empty((self.batch, self.h >> L, self.w >> L), dtype=torch.float32, device=coeffs.device)
        _out_packed(out, self.batch * (self.h >> L) * (self.w >> L), coeffs.device, "ll")
        with _guard_device(coeffs):
            _check(lib().fhwt_plan_pack_ll_2d(self._h, _dev_f32(coeffs, "coeffs"), _dev_f32(out, "ll"),
                                              _stream(stream, coeffs)))
        return out


def pack_ll_2d_peers(coeffs, levels: int, peer_ptrs_dev: int, rank: int, npeers: int, stream=None):
    """fhwt_pack_ll_2d_peers: store this rank's packed LL_levels into every peer's gather buffer
    (peer_ptrs_dev: device address of an array of npeers peer device pointers)."""
    h, w, batch = _shape_2d(coeffs)
    with _guard_device(coeffs):
        _check(lib().fhwt_pack_ll_2d_peers(_dev_f32(coeffs, "coeffs"), ctypes.c_void_p(int(peer_ptrs_dev)), int(rank),
                                           int(npeers), h, w, batch, int(levels), _stream(stream, coeffs)))


def pack_ll_2d(coeffs, levels: int, out=None, stream=None):
    """fhwt_pack_ll_2d: contiguous copy of every image's coarsest LL band ([..., h>>L, w>>L])."""
    import torch
    h, w, batch = _shape_2d(coeffs)
    shape = tuple(coeffs.shape[:-2]) + (h >> levels, w >> levels)
    if out is None:
        out = torch.empty(shape, dtype=coeffs.dtype, device=coeffs.device)
    if levels >= 1:
        _out_packed(out, batch * (h >> levels) * (w >> levels), coeffs.device, "ll")
    with _guard_device(coeffs):
        _check(lib().fhwt_pack_ll_2d(_dev_f32(coeffs, "coeffs"), _dev_f32(out, "ll"), h, w, batch, int(levels),
                                     _stream(stream, coeffs)))
    return out


def _host_f32(t, what):
    import torch
    if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise InvalidArgument(f"{what} must be a contiguous float32 host tensor (pinned recommended)")
    return ctypes.c_void_p(t.data_ptr())


def _host_out(out, d, what):
    """Host outputs of the round trip: the C ABI writes d.numel() floats into them."""
    if out.shape != d.shape:
        raise ShapeMismatch(f"{what} has shape {tuple(out.shape)}, expected {tuple(d.shape)}")
    return out


def roundtrip_2d_host(d, levels: int, coeffs_out=None, out=None, chunk: int = 0):
    """fhwt_roundtrip_2d_host: DWT + IDWT of HOST images, streamed through the current device."""
    import torch
    h, w, batch = _shape_2d(d)
    if out is None:
        out = torch.empty_like(d, pin_memory=d.is_pinned())
    _host_out(out, d, "out")
    if coeffs_out is not None:
        _host_out(coeffs_out, d, "coeffs_out")
    _check(lib().fhwt_roundtrip_2d_host(_host_f32(d, "d"), _host_f32(coeffs_out, "coeffs") if coeffs_out is not None else None,
                                        _host_f32(out, "d_R"), h, w, batch, int(levels), int(chunk)))
    return out


def roundtrip_1d_host(d, levels: int, coeffs_out=None, out=None, chunk: int = 0):
    import torch
    n, batch = _shape_1d(d)
    if out is None:
        out = torch.empty_like(d, pin_memory=d.is_pinned())
    _host_out(out, d, "out")
    if coeffs_out is not None:
        _host_out(coeffs_out, d, "coeffs_out")
    _check(lib().fhwt_roundtrip_1d_host(_host_f32(d, "d"), _host_f32(coeffs_out, "coeffs") if coeffs_out is not None else None,
                                        _host_f32(out, "d_R"), n, batch, int(levels), int(chunk)))
    return out


def band_offset_1d(n: int, level: int, band: int):
    ln = ctypes.c_int64()
    off = lib().fhwt_band_offset_1d(int(n), int(level), int(band), ctypes.byref(ln))
    if off < 0:
        raise InvalidArgument(f"bad band query n={n} level={level} band={band}")
    return int(off), int(ln.value)


def band_offset_2d(h: int, w: int, level: int, band: int):
    r, c = ctypes.c_int64(), ctypes.c_int64()
    off = lib().fhwt_band_offset_2d(int(h), int(w), int(level), int(band), ctypes.byref(r), ctypes.byref(c))
    if off < 0:
        raise InvalidArgument(f"bad band query {h}x{w} level={level} band={band}")
    return int(off), int(r.value), int(c.value)



# ------------------------------------------------------------------ direct-form baseline (§8(f) f3)
def direct_workspace_bytes(dims: int, n_or_h: int, w: int, batch: int) -> int:
    return int(lib().fhwt_direct_workspace_bytes(int(dims), int(n_or_h), int(w), int(batch)))


def _direct_ws(x, dims, n_or_h, w, batch, workspace):
    import torch
    nb = direct_workspace_bytes(dims, n_or_h, w, batch)
    if workspace is None:
        workspace = torch.empty(max(nb, 1), dtype=torch.uint8, device=x.device)
    if not workspace.is_cuda or workspace.numel() * workspace.element_size() < nb:
        raise InvalidArgument(f"workspace must be a CUDA buffer of >= {nb} bytes")
    return ctypes.c_void_p(workspace.data_ptr())


def direct_analyze_1d(d, levels: int, out=None, workspace=None, stream=None):
    """fhwt_direct_analyze_1d: the paper's original structure (Fig. 2) on the GPU — baseline only."""
    n, batch = _shape_1d(d)
    out = _out_like(d, out)
    with _guard_device(d):
        _check(lib().fhwt_direct_analyze_1d(_dev_f32(d, "d"), _dev_f32(out, "coeffs"), n, batch, int(levels),
                                            _direct_ws(d, 1, n, 0, batch, workspace), _stream(stream, d)))
    return out


def direct_synthesize_1d(coeffs, levels: int, out=None, workspace=None, stream=None):
    """fhwt_direct_synthesize_1d: Fig. 5 (zero insertion + full-rate filters) — baseline only."""
    n, batch = _shape_1d(coeffs)
    out = _out_like(coeffs, out)
    with _guard_device(coeffs):
        _check(lib().fhwt_direct_synthesize_1d(_dev_f32(coeffs, "coeffs"), _dev_f32(out, "d_R"), n, batch,
                                               int(levels), _direct_ws(coeffs, 1, n, 0, batch, workspace),
                                               _stream(stream, coeffs)))
    return out


def direct_analyze_2d(d, levels: int, out=None, workspace=None, stream=None):
    h, w, batch = _shape_2d(d)
    out = _out_like(d, out)
    with _guard_device(d):
        _check(lib().fhwt_direct_analyze_2d(_dev_f32(d, "d"), _dev_f32(out, "coeffs"), h, w, batch, int(levels),
                                            _direct_ws(d, 2, h, w, batch, workspace), _stream(stream, d)))
    return out


def direct_synthesize_2d(coeffs, levels: int, out=None, workspace=None, stream=None):
    h, w, batch = _shape_2d(coeffs)
    out = _out_like(coeffs, out)
    with _guard_device(coeffs):
        _check(lib().fhwt_direct_synthesize_2d(_dev_f32(coeffs, "coeffs"), _dev_f32(out, "d_R"), h, w, batch,
                                               int(levels), _direct_ws(coeffs, 2, h, w, batch, workspace),
                                               _stream(stream, coeffs)))
    return out


_STRUCTURES = {"direct": 0, "fast": 1, "kernel": 2}


def op_counts(shape, levels: int, structure: str = "fast", synthesis: bool = False, batch: int = 1):
    """fhwt_op_counts: static (mul, add) counts of one transform; shape = (n,) or (h, w)."""
    m, a = ctypes.c_uint64(), ctypes.c_uint64()
    dims = len(shape)
    _check(lib().fhwt_op_counts(dims, int(shape[0]), int(shape[1]) if dims == 2 else 0, int(batch), int(levels),
                                _STRUCTURES[structure], int(bool(synthesis)), ctypes.byref(m), ctypes.byref(a)))
    return int(m.value), int(a.value)


# ------------------------------------------------------------------ LL-only lowpass (§8(f) f1)
def lowpass_2d_u8(d, levels: int, out=None, stream=None):
    """fhwt_lowpass_2d_u8: LL_levels of uint8 images [..., h, w] (the paper's Fig. 12 output), fp32."""
    import torch
    if not isinstance(d, torch.Tensor) or not d.is_cuda or d.dtype != torch.uint8 or not d.is_contiguous():
        raise InvalidArgument("d must be a contiguous uint8 CUDA tensor")
    h, w, batch = _shape_2d(d)
    shape = tuple(d.shape[:-2]) + (h >> levels, w >> levels)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=d.device)
    if levels >= 1:
        _out_packed(out, batch * (h >> levels) * (w >> levels), d.device, "ll")
    with torch.cuda.device(d.device):
        _check(lib().fhwt_lowpass_2d_u8(ctypes.c_void_p(d.data_ptr()), _dev_f32(out, "ll"), h, w, batch, int(levels),
                                        None, _stream(stream, d)))
    return out


def lowpass_2d_bf16(d, levels: int, out=None, stream=None):
    """fhwt_lowpass_2d_bf16: LL_levels of bfloat16 images [..., h, w] (w % 8 == 0), fp32 output; equal
    bitwise to analyze_2d(d.float(), levels)'s LL band."""
    import torch
    if not isinstance(d, torch.Tensor) or not d.is_cuda or d.dtype != torch.bfloat16 or not d.is_contiguous():
        raise InvalidArgument("d must be a contiguous bfloat16 CUDA tensor")
    h, w, batch = _shape_2d(d)
    shape = tuple(d.shape[:-2]) + (h >> levels, w >> levels)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=d.device)
    if levels >= 1:
        _out_packed(out, batch * (h >> levels) * (w >> levels), d.device, "ll")
    with torch.cuda.device(d.device):
        _check(lib().fhwt_lowpass_2d_bf16(ctypes.c_void_p(d.data_ptr()), _dev_f32(out, "ll"), h, w, batch,
                                          int(levels), None, _stream(stream, d)))
    return out
