"""ctypes binding of libddh.so (include/ddh.h) -- argument marshalling only.

Every step of the DDH-MBIR path runs in the CUDA kernels of libddh.so; this
module only checks tensor shapes/dtypes/devices and passes raw pointers.
There is no CPU fallback: if the library is missing or fails to load, every
entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DDH_LIB") or os.path.join(_HERE, "lib", "libddh.so")

DDH_F_NO_TIPTILT = 1
DDH_F_CALL_GRAPHS = 128  # multi-frame calls replayed from chunk graphs (include/ddh.h)
DDH_F_NO_ADAPTIVE_GRAPHS = 256  # never switch a long host-bound call to chunk graphs (include/ddh.h)

_STATUS = {0: "DDH_OK", 1: "DDH_E_INVAL", 2: "DDH_E_CUDA", 3: "DDH_E_NOMEM", 4: "DDH_E_STATE"}


class DdhParams(ctypes.Structure):
    """Mirror of ``ddh_params`` (include/ddh.h)."""

    _fields_ = [
        ("n", ctypes.c_int32),
        ("streams", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("aperture_diam", ctypes.c_float),
        ("aperture_mask", ctypes.POINTER(ctypes.c_uint8)),
        ("noise_var", ctypes.c_double),
        ("lam", ctypes.c_double),
        ("alpha", ctypes.c_double),
        ("n_k", ctypes.c_int32),
        ("r_min", ctypes.c_double),
        ("r_sigma", ctypes.c_double),
        ("r_T", ctypes.c_double),
        ("r_q", ctypes.c_double),
        ("phi_sigma", ctypes.c_double),
        ("icd_sweeps", ctypes.c_int32),
        ("boot_period", ctypes.c_int32),
        ("boot_alpha", ctypes.c_double),
        ("chunk_streams", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("lanes", ctypes.c_int32),
    ]


EXPORTS = [
    "ddh_default_params", "ddh_create", "ddh_destroy", "ddh_bootstrap", "ddh_step", "ddh_step_host", "ddh_step_host_async",
    "ddh_static", "ddh_get_state", "ddh_set_state", "ddh_strehl", "ddh_residual", "ddh_sync", "ddh_last_error",
    "ddh_kernel_launches", "ddh_frame_index", "ddh_test_fft2c", "ddh_test_estep", "ddh_test_ricd", "ddh_test_phiicd",
    "ddh_profile_enable", "ddh_profile_read", "ddh_kind_name",
    "ddh_synth_create", "ddh_synth_frames", "ddh_synth_reflectance", "ddh_synth_destroy",
]
KIND_COUNT = 17

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libddh.so (raises if it is missing: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libddh.so not built ({path}); run `python -m paper_2305_03284_b200.build`")
    lib = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    fp = ctypes.POINTER(ctypes.c_float)
    lib.ddh_default_params.argtypes = [ctypes.POINTER(DdhParams)]
    lib.ddh_create.argtypes = [ctypes.POINTER(DdhParams), vp, ctypes.POINTER(vp)]
    lib.ddh_destroy.argtypes = [vp]
    lib.ddh_bootstrap.argtypes = [vp, vp, i32, vp]
    lib.ddh_step.argtypes = [vp, vp, i32, vp, vp, vp]
    lib.ddh_step_host.argtypes = [vp, vp, i32, vp, vp, vp]
    lib.ddh_step_host_async.argtypes = [vp, vp, i32, vp, vp, vp]
    lib.ddh_static.argtypes = [vp, vp, i32, i32, vp, vp, vp]
    lib.ddh_get_state.argtypes = [vp, vp, vp, ctypes.POINTER(i64)]
    lib.ddh_set_state.argtypes = [vp, vp, vp, i64]
    lib.ddh_strehl.argtypes = [vp, vp, vp, i32, ctypes.POINTER(ctypes.c_double)]
    lib.ddh_residual.argtypes = [vp, vp, vp, i32, vp, vp, ctypes.POINTER(ctypes.c_double)]
    lib.ddh_sync.argtypes = [vp]
    lib.ddh_last_error.argtypes = [vp]
    lib.ddh_last_error.restype = ctypes.c_char_p
    lib.ddh_kernel_launches.argtypes = [vp]
    lib.ddh_kernel_launches.restype = ctypes.c_uint64
    lib.ddh_frame_index.argtypes = [vp]
    lib.ddh_frame_index.restype = i64
    lib.ddh_test_fft2c.argtypes = [vp, vp, vp, i32, i32]
    lib.ddh_test_estep.argtypes = [vp, vp, vp, i32, i32, vp, vp, vp]
    lib.ddh_test_ricd.argtypes = [vp, vp, vp, i32, vp]
    lib.ddh_test_phiicd.argtypes = [vp, vp, vp, vp, i32, vp]
    lib.ddh_profile_enable.argtypes = [vp, i32]
    lib.ddh_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
    lib.ddh_kind_name.argtypes = [i32]
    lib.ddh_kind_name.restype = ctypes.c_char_p
    dp = ctypes.POINTER(ctypes.c_double)
    lib.ddh_synth_create.argtypes = [i32, ctypes.c_float, i32, dp, dp, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_uint64, vp, ctypes.POINTER(vp)]
    lib.ddh_synth_frames.argtypes = [vp, i64, i32, vp, vp]
    lib.ddh_synth_reflectance.argtypes = [vp, vp]
    lib.ddh_synth_destroy.argtypes = [vp]
    for name in EXPORTS:
        if name not in ("ddh_last_error", "ddh_kernel_launches", "ddh_frame_index", "ddh_kind_name"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


class DDHError(RuntimeError):
    pass


def default_params() -> DdhParams:
    p = DdhParams()
    _check(load_library().ddh_default_params(ctypes.byref(p)), None)
    return p


def _check(code, ctx):
    if code != 0:
        msg = load_library().ddh_last_error(ctx).decode(errors="replace")
        raise DDHError(f"{_STATUS.get(code, code)}: {msg}")


def _ptr(t: Optional[torch.Tensor], dtype, shape, device, name, allow_none=True, host=False):
    if t is None:
        if not allow_none:
            raise ValueError(f"{name} is required")
        return None
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if host:
        if t.device.type != "cpu":
            raise ValueError(f"{name}: must be a host tensor")
    elif t.device != device:
        raise ValueError(f"{name}: must live on {device}")
    return ctypes.c_void_p(t.data_ptr())


class DDH:
    """One ``ddh_ctx``: S independent streams of N x N DH frames on one GPU.

    Parameters follow ``ddh_params``; ``stream`` is a torch.cuda.Stream
    (default: the current stream of ``device``)."""

    def __init__(self, n: int, streams: int = 1, device: int = 0, aperture_diam: float = None,
                 aperture_mask=None, stream: Optional[torch.cuda.Stream] = None, **kw):
        self.lib = load_library()
        p = default_params()
        p.n = n
        p.streams = streams
        p.device = device
        p.aperture_diam = float(n if aperture_diam is None else aperture_diam)
        self._mask_buf = None
        if aperture_mask is not None:
            import numpy as np
            m = np.ascontiguousarray(np.asarray(aperture_mask, dtype=np.uint8))
            if m.shape != (n, n):
                raise ValueError("aperture_mask must be N x N")
            self._mask_buf = m
            p.aperture_mask = m.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
            p.aperture_diam = 0.0
        alias = {"lambda": "lam"}
        for k, v in kw.items():
            k = alias.get(k, k)
            if not hasattr(p, k):
                raise TypeError(f"unknown parameter {k}")
            setattr(p, k, v)
        self.params = p
        self.n, self.S = n, streams
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        _check(self.lib.ddh_create(ctypes.byref(p), ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)), None)
        self.h = h

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            self.lib.ddh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _frames(self, T):
        return (T, self.S, self.n, self.n)

    # -- hot path
    def bootstrap(self, y0: torch.Tensor, k_b: int, status: Optional[torch.Tensor] = None):
        yp = _ptr(y0, torch.complex64, (self.S, self.n, self.n), self.device, "y0", allow_none=False)
        sp = _ptr(status, torch.uint8, (self.S,), self.device, "status")
        _check(self.lib.ddh_bootstrap(self.h, yp, int(k_b), sp), self.h)

    def step(self, y: torch.Tensor, phi_out=None, r_out=None, status=None):
        T = y.shape[0]
        yp = _ptr(y, torch.complex64, self._frames(T), self.device, "y", allow_none=False)
        pp = _ptr(phi_out, torch.float32, self._frames(T), self.device, "phi_out")
        rp = _ptr(r_out, torch.float32, self._frames(T), self.device, "r_out")
        sp = _ptr(status, torch.uint8, (T, self.S), self.device, "status")
        _check(self.lib.ddh_step(self.h, yp, T, pp, rp, sp), self.h)

    def step_host(self, y: torch.Tensor, phi_out=None, r_out=None, status=None, asynchronous=False):
        """ddh_step_host (synchronous) or ddh_step_host_async (then call sync()
        before reading the outputs or releasing any of the host buffers)."""
        T = y.shape[0]
        yp = _ptr(y, torch.complex64, self._frames(T), None, "y", allow_none=False, host=True)
        pp = _ptr(phi_out, torch.float32, self._frames(T), None, "phi_out", host=True)
        rp = _ptr(r_out, torch.float32, self._frames(T), None, "r_out", host=True)
        sp = _ptr(status, torch.uint8, (T, self.S), None, "status", host=True)
        fn = self.lib.ddh_step_host_async if asynchronous else self.lib.ddh_step_host
        _check(fn(self.h, yp, T, pp, rp, sp), self.h)

    def static(self, y: torch.Tensor, iters: int, phi_out=None, r_out=None, status=None):
        T = y.shape[0]
        yp = _ptr(y, torch.complex64, self._frames(T), self.device, "y", allow_none=False)
        pp = _ptr(phi_out, torch.float32, self._frames(T), self.device, "phi_out")
        rp = _ptr(r_out, torch.float32, self._frames(T), self.device, "r_out")
        sp = _ptr(status, torch.uint8, (T, self.S), self.device, "status")
        _check(self.lib.ddh_static(self.h, yp, T, int(iters), pp, rp, sp), self.h)

    # -- state
    def get_state(self):
        r = torch.empty((self.S, self.n, self.n), dtype=torch.float32, device=self.device)
        phi = torch.empty_like(r)
        fi = ctypes.c_int64()
        _check(self.lib.ddh_get_state(self.h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(phi.data_ptr()),
                                      ctypes.byref(fi)), self.h)
        return r, phi, fi.value

    def set_state(self, r: torch.Tensor, phi: torch.Tensor, frame_index: int = 0):
        shp = (self.S, self.n, self.n)
        rp = _ptr(r, torch.float32, shp, self.device, "r")
        pp = _ptr(phi, torch.float32, shp, self.device, "phi")
        _check(self.lib.ddh_set_state(self.h, rp, pp, int(frame_index)), self.h)

    def strehl(self, phi_hat: torch.Tensor, phi_true: torch.Tensor):
        B = phi_hat.shape[0]
        shp = (B, self.n, self.n)
        a = _ptr(phi_hat, torch.float32, shp, self.device, "phi_hat", allow_none=False)
        b = _ptr(phi_true, torch.float32, shp, self.device, "phi_true", allow_none=False)
        out = (ctypes.c_double * max(B, 1))()
        _check(self.lib.ddh_strehl(self.h, a, b, B, out), self.h)
        return [out[i] for i in range(B)]

    def residual(self, phi_hat: torch.Tensor, phi_true: torch.Tensor, want_psf: bool = True):
        """(residual phase, residual PSF or None, Strehl list) of B estimates
        (ddh_residual: P:273, 320; tip/tilt removed)."""
        B = phi_hat.shape[0]
        shp = (B, self.n, self.n)
        a = _ptr(phi_hat, torch.float32, shp, self.device, "phi_hat", allow_none=False)
        b = _ptr(phi_true, torch.float32, shp, self.device, "phi_true", allow_none=False)
        resid = torch.empty(shp, dtype=torch.float32, device=self.device)
        psf = torch.empty(shp, dtype=torch.float32, device=self.device) if want_psf else None
        out = (ctypes.c_double * max(B, 1))()
        _check(self.lib.ddh_residual(self.h, a, b, B, ctypes.c_void_p(resid.data_ptr()),
                                     ctypes.c_void_p(psf.data_ptr()) if psf is not None else None, out), self.h)
        return resid, psf, [out[i] for i in range(B)]

    def sync(self):
        _check(self.lib.ddh_sync(self.h), self.h)

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.ddh_kernel_launches(self.h))

    @property
    def frame_index(self) -> int:
        return int(self.lib.ddh_frame_index(self.h))

    # -- instrumentation
    def profile(self, enable: bool = True):
        _check(self.lib.ddh_profile_enable(self.h, int(enable)), self.h)

    def profile_read(self):
        """{kernel name: (total ms, launches)} accumulated since the last read."""
        ms = (ctypes.c_double * KIND_COUNT)()
        cnt = (ctypes.c_int64 * KIND_COUNT)()
        _check(self.lib.ddh_profile_read(self.h, ms, cnt), self.h)
        return {self.lib.ddh_kind_name(k).decode(): (ms[k], cnt[k]) for k in range(KIND_COUNT) if cnt[k]}

    # -- stage entry points (parity tests)
    def test_fft2c(self, x: torch.Tensor, inverse: bool = False) -> torch.Tensor:
        B = x.shape[0]
        xp = _ptr(x, torch.complex64, (B, self.n, self.n), self.device, "x", allow_none=False)
        out = torch.empty_like(x)
        _check(self.lib.ddh_test_fft2c(self.h, xp, ctypes.c_void_p(out.data_ptr()), B, int(inverse)), self.h)
        return out

    def test_estep(self, u: torch.Tensor, r_prev: torch.Tensor, warm: bool = True):
        """(r0, mu, q) of the E-step stage (Eq. 3 when warm) for B fields."""
        B = u.shape[0]
        shp = (B, self.n, self.n)
        up = _ptr(u, torch.complex64, shp, self.device, "u", allow_none=False)
        rp = _ptr(r_prev, torch.float32, shp, self.device, "r_prev", allow_none=False)
        r0 = torch.empty(shp, dtype=torch.float32, device=self.device)
        q = torch.empty_like(r0)
        mu = torch.empty(shp, dtype=torch.complex64, device=self.device)
        _check(self.lib.ddh_test_estep(self.h, up, rp, B, int(warm), ctypes.c_void_p(r0.data_ptr()),
                                       ctypes.c_void_p(mu.data_ptr()), ctypes.c_void_p(q.data_ptr())), self.h)
        return r0, mu, q

    def test_ricd(self, r_in: torch.Tensor, q: torch.Tensor) -> torch.Tensor:
        B = r_in.shape[0]
        shp = (B, self.n, self.n)
        a = _ptr(r_in, torch.float32, shp, self.device, "r_in", allow_none=False)
        b = _ptr(q, torch.float32, shp, self.device, "q", allow_none=False)
        out = torch.empty_like(r_in)
        _check(self.lib.ddh_test_ricd(self.h, a, b, B, ctypes.c_void_p(out.data_ptr())), self.h)
        return out

    def test_phiicd(self, phi_in: torch.Tensor, c: torch.Tensor, theta: torch.Tensor) -> torch.Tensor:
        B = phi_in.shape[0]
        shp = (B, self.n, self.n)
        a = _ptr(phi_in, torch.float32, shp, self.device, "phi_in", allow_none=False)
        b = _ptr(c, torch.float32, shp, self.device, "c", allow_none=False)
        t = _ptr(theta, torch.float32, shp, self.device, "theta", allow_none=False)
        out = torch.empty_like(phi_in)
        _check(self.lib.ddh_test_phiicd(self.h, a, b, t, B, ctypes.c_void_p(out.data_ptr())), self.h)
        return out


class DDHSynth:
    """On-device frame synthesiser (libddh ddh_synth_*): the
    BASELINE recipe with its own counter-based generator.  Input generation
    only.  d_r0: per-stream D/r0 (scalar or sequence); velocity: per-stream
    (rows, cols) px/frame (pair or sequence of pairs)."""

    def __init__(self, n: int, streams: int, d_r0, velocity, sigma_b: float, snr_db: float,
                 diam: float = None, seed: int = 20230504, device: int = 0):
        import numpy as np
        import torch
        self.lib = load_library()
        self.n, self.S = n, streams
        self.device = torch.device("cuda", device)
        self.stream = torch.cuda.current_stream(self.device)
        dr = np.broadcast_to(np.asarray(d_r0, np.float64), (streams,)).copy()
        v = np.broadcast_to(np.asarray(velocity, np.float64).reshape(-1, 2), (streams, 2)).copy()
        h = ctypes.c_void_p()
        dp = ctypes.POINTER(ctypes.c_double)
        st = self.lib.ddh_synth_create(int(n), float(n if diam is None else diam), int(streams),
                                       dr.ctypes.data_as(dp), v.ctypes.data_as(dp), float(sigma_b), float(snr_db),
                                       int(seed), ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        if st != 0:
            raise DDHError(f"ddh_synth_create failed with status {st}")
        self.h = h

    def frames(self, t0: int, T: int, want_phi: bool = True):
        import torch
        y = torch.empty((T, self.S, self.n, self.n), dtype=torch.complex64, device=self.device)
        phi = torch.empty((T, self.S, self.n, self.n), dtype=torch.float32, device=self.device) if want_phi else None
        st = self.lib.ddh_synth_frames(self.h, int(t0), int(T), ctypes.c_void_p(y.data_ptr()),
                                       ctypes.c_void_p(phi.data_ptr()) if phi is not None else None)
        if st != 0:
            raise DDHError(f"ddh_synth_frames failed with status {st}")
        return y, phi

    def reflectance(self):
        import torch
        r = torch.empty((self.S, self.n, self.n), dtype=torch.float32, device=self.device)
        st = self.lib.ddh_synth_reflectance(self.h, ctypes.c_void_p(r.data_ptr()))
        if st != 0:
            raise DDHError(f"ddh_synth_reflectance failed with status {st}")
        return r

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.ddh_synth_destroy(h)
            self.h = None
