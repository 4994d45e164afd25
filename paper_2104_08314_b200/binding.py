"""Thin ctypes binding of libspconv.so (include/spconv.h): argument marshalling only.

Every function has the C name and calls straight into the library; tensors are
torch CUDA tensors (device memory from PyTorch's allocator), the stream is
torch's current stream unless given.  There is no CPU fallback: importing this
module raises if the compiled sm_100a library is missing.
"""
from __future__ import annotations

import ctypes
import functools
import os
from dataclasses import dataclass, field

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPC_LIB_OVERRIDE") or os.path.join(_HERE, "libspconv.so")  # override: dev probes only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2104_08314_b200.build` "
                      "(nvcc, sm_100a); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

SPC_OK, SPC_EINVAL, SPC_EUNSUPPORTED, SPC_ECAPACITY, SPC_ECUDA, SPC_ECORRUPT = 0, -1, -2, -3, -4, -5
SPC_ALGO_IM2COL, SPC_ALGO_CPO, SPC_ALGO_CPS, SPC_ALGO_CSCC, SPC_ALGO_CPO_SA = 0, 1, 2, 3, 4
SPC_FAVOUR_TIME, SPC_FAVOUR_SPACE, SPC_BEST_OF_THREE = 0, 1, 2
SPC_NPC = -(2 ** 31)
SPC_NPF = -(2 ** 31) + 1
ALGO_NAMES = {0: "im2col", 1: "cpo", 2: "cps", 3: "cscc", 4: "cpo_sa"}


class SpcError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.spc_last_error().decode()
        super().__init__(f"{where} failed with status {status}: {msg}")
        self.status = status


class spc_conv_desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("N", "C", "H", "W", "K", "R", "S", "stride_h", "stride_w",
                 "pad_top", "pad_bottom", "pad_left", "pad_right")]


class spc_encoding(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("ptr_cap", ctypes.c_int64),
                ("da", ctypes.c_void_p), ("da_cap", ctypes.c_int64),
                ("in_", ctypes.c_void_p), ("in_cap", ctypes.c_int64),
                ("chan_ptr_off", ctypes.c_void_p), ("chan_nz_off", ctypes.c_void_p),
                ("chan_in_off", ctypes.c_void_p), ("lengths", ctypes.c_void_p),
                ("algo", ctypes.c_int32), ("geom", spc_conv_desc)]


_D = ctypes.POINTER(spc_conv_desc)
_E = ctypes.POINTER(spc_encoding)
_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_sigs = {
    "spc_encode_capacity": [_D, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                            ctypes.POINTER(_sz)],
    "spc_workspace_init": [_vp, _sz, _vp],
    "cpo_encode": [_D, _vp, _E, _vp, _sz, _vp],
    "cps_encode": [_D, _vp, _E, _vp, _sz, _vp],
    "spc_pack_weights": [_D, _vp, _vp, _vp],
    "sparse_conv_forward": [_D, _E, _vp, _vp, _i32, _vp, _sz, _vp],
    "im2col_conv_forward": [_D, _vp, _vp, _vp, _i32, _vp, _sz, _vp],
    "select_layer_algo": [_D, _vp, _i32, _vp, _i32, _i32, ctypes.POINTER(_i32),
                          ctypes.POINTER(ctypes.c_float), _vp, _sz, _vp],
    "spc_encoding_lengths": [_E, ctypes.POINTER(_i64), _vp],
    "spc_validate_encoding": [_D, _E, _vp, _sz, _vp],
    "spc_select_from_times": [ctypes.POINTER(ctypes.c_float), _i32, _i32, ctypes.POINTER(_i32)],
    "spc_output_dims": [_D, ctypes.POINTER(_i32), ctypes.POINTER(_i32)],
    "spc_cscc_capacity": [_D, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "spc_space_bound": [_D, _i32, ctypes.c_double, ctypes.POINTER(ctypes.c_double)],
    "spc_strided_capacity": [_D, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "cpo_encode_strided": [_D, _vp, _E, _vp, _sz, _vp],
    "sparse_conv_encode_forward": [_D, _E, _vp, _vp, _i32, _D, _E, _vp, _sz, _vp],
    "spc_cscc_q_bound": [_D, ctypes.POINTER(ctypes.c_double)],
    "spc_space_preselect": [_D, _i32, ctypes.c_double, ctypes.c_double, ctypes.POINTER(_i32)],
    "cscc_encode": [_D, _vp, _E, _vp],
    "cscc_conv_forward": [_D, _E, _vp, _vp, _i32, _vp],
}
for _n, _a in _sigs.items():
    getattr(_lib, _n).argtypes = _a
    getattr(_lib, _n).restype = ctypes.c_int
_lib.spc_set_im2col_gemm.argtypes = [ctypes.c_int]
_lib.spc_set_im2col_gemm.restype = ctypes.c_int
_lib.spc_get_im2col_gemm.argtypes = []
_lib.spc_get_im2col_gemm.restype = ctypes.c_int
_lib.spc_set_cps_inline.argtypes = [ctypes.c_int32]
_lib.spc_set_cps_inline.restype = ctypes.c_int
_lib.spc_get_cps_inline.argtypes = []
_lib.spc_get_cps_inline.restype = ctypes.c_int32
_lib.spc_im2col_engine.argtypes = [ctypes.c_void_p]
_lib.spc_last_conv_kernel.argtypes = []
_lib.spc_last_conv_kernel.restype = ctypes.c_int
_lib.spc_im2col_engine.restype = ctypes.c_int
_lib.spc_im2col_ws_bytes.argtypes = [ctypes.c_void_p]
_lib.spc_im2col_ws_bytes.restype = ctypes.c_size_t
_lib.spc_fused_ws_bytes.argtypes = [_D]
_lib.spc_fused_ws_bytes.restype = _sz
_lib.spc_select_ws_bytes.argtypes = [_D]
_lib.spc_select_ws_bytes.restype = _sz
_lib.spc_last_error.restype = ctypes.c_char_p
_lib.spc_version.restype = ctypes.c_char_p

EXPORTED = list(_sigs) + ["spc_fused_ws_bytes", "spc_select_ws_bytes", "spc_last_error", "spc_version", "spc_set_im2col_gemm",
                          "spc_get_im2col_gemm", "spc_im2col_engine", "spc_im2col_ws_bytes", "spc_last_conv_kernel",
                          "spc_set_cps_inline", "spc_get_cps_inline"]
SPC_GEMM_SIMT, SPC_GEMM_CUBLAS_FP32, SPC_GEMM_CUBLAS_BF16X9, SPC_GEMM_CUBLAS_TF32, SPC_GEMM_TC_3XTF32 = 0, 1, 2, 3, 4
SPC_GEMM_AUTO = 5
GEMM_NAMES = {0: "SIMT FP32 FFMA (this library, 128x128 tiles)", 1: "cuBLAS FP32 (CUBLAS_COMPUTE_32F)",
              2: "cuBLAS FP32 emulated by 3 bf16 terms on tensor cores (CUBLAS_COMPUTE_32F_EMULATED_16BFX9)",
              3: "cuBLAS TF32 tensor cores (CUBLAS_COMPUTE_32F_FAST_TF32, 1 term)",
              4: "tcgen05 3xTF32 (this library: fp32 from three TF32 products, TMEM accumulators)",
              5: "auto: tcgen05 3xTF32 for layers >= 2^28 MACs or >= 2^26 MACs over >= 20 tiles or CRS >= 2048 "
                 "(C*R*S % 4 == 0), cuBLAS FP32 otherwise"}


def spc_set_im2col_gemm(gemm: int) -> None:
    st = _lib.spc_set_im2col_gemm(int(gemm))
    if st != SPC_OK:
        raise SpcError(st, "spc_set_im2col_gemm")


def spc_get_im2col_gemm() -> int:
    return int(_lib.spc_get_im2col_gemm())


def spc_set_cps_inline(on: bool) -> None:
    st = _lib.spc_set_cps_inline(int(bool(on)))
    if st != SPC_OK:
        raise SpcError(st, "spc_set_cps_inline")


def spc_get_cps_inline() -> bool:
    return bool(_lib.spc_get_cps_inline())


def spc_im2col_ws_bytes(d: dict) -> int:
    """Recommended im2col workspace bytes for layer d under the current GEMM engine."""
    return int(_lib.spc_im2col_ws_bytes(ctypes.byref(make_desc(d))))


def alloc_im2col_workspace(d: dict, device="cuda") -> torch.Tensor:
    """fp32 workspace of spc_im2col_ws_bytes(d) bytes (lowered matrix + split weights)."""
    return torch.empty((spc_im2col_ws_bytes(d) + 3) // 4, dtype=torch.float32, device=device)


CONV_KERNELS = {3: "tile_conv_kernel (register-tiled)", 2: "ws_conv_kernel (warp-specialised)", 1: "strip_conv_kernel", 0: "sparse_conv_generic_kernel",
                -1: "none"}


def spc_last_conv_kernel() -> int:
    """Kernel of this thread's last sparse conv launch (CONV_KERNELS)."""
    return int(_lib.spc_last_conv_kernel())


def spc_im2col_engine(d: dict) -> int:
    """The GEMM engine im2col_conv_forward runs for layer d (AUTO and fallbacks resolved)."""
    return int(_lib.spc_im2col_engine(ctypes.byref(make_desc(d))))


def _check(rc: int, where: str):
    if rc != SPC_OK:
        raise SpcError(rc, where)


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    if not t.is_cuda:
        raise ValueError("tensors passed to libspconv must be CUDA tensors")
    return ctypes.c_void_p(t.data_ptr())


def make_desc(d: dict) -> spc_conv_desc:
    return spc_conv_desc(*(int(d[k]) for k in ("N", "C", "H", "W", "K", "R", "S", "stride_h", "stride_w",
                                               "pad_top", "pad_bottom", "pad_left", "pad_right")))


def spc_output_dims(d: dict) -> tuple[int, int]:
    """Output extents (Oh, Ow) the library uses for y (spc_output_dims)."""
    oh, ow = _i32(), _i32()
    _check(_lib.spc_output_dims(ctypes.byref(make_desc(d)), ctypes.byref(oh), ctypes.byref(ow)), "spc_output_dims")
    return oh.value, ow.value


out_hw = spc_output_dims


def spc_encode_capacity(d: dict) -> tuple[int, int, int, int]:
    p, a, i, w = _i64(), _i64(), _i64(), _sz()
    _check(_lib.spc_encode_capacity(ctypes.byref(make_desc(d)), ctypes.byref(p), ctypes.byref(a),
                                    ctypes.byref(i), ctypes.byref(w)), "spc_encode_capacity")
    return p.value, a.value, i.value, w.value


def spc_workspace_init(ws: torch.Tensor, stream=None):
    _check(_lib.spc_workspace_init(_ptr(ws), ws.numel() * ws.element_size(), _stream(stream)),
           "spc_workspace_init")


@dataclass
class Encoding:
    """Device buffers of one encoding (owned by PyTorch) + the C struct view."""
    ptr: torch.Tensor
    da: torch.Tensor
    inn: torch.Tensor
    chan_ptr_off: torch.Tensor
    chan_nz_off: torch.Tensor
    chan_in_off: torch.Tensor
    lengths: torch.Tensor
    c: spc_encoding = field(default_factory=spc_encoding)

    def __post_init__(self):
        self.c.ptr, self.c.ptr_cap = self.ptr.data_ptr(), self.ptr.numel()
        self.c.da, self.c.da_cap = self.da.data_ptr(), self.da.numel()
        self.c.in_, self.c.in_cap = self.inn.data_ptr(), self.inn.numel()
        self.c.chan_ptr_off = self.chan_ptr_off.data_ptr()
        self.c.chan_nz_off = self.chan_nz_off.data_ptr()
        self.c.chan_in_off = self.chan_in_off.data_ptr()
        self.c.lengths = self.lengths.data_ptr()

    @property
    def algo(self) -> int:
        return self.c.algo


def alloc_encoding(d: dict, device="cuda", caps: tuple[int, int, int] | None = None) -> Encoding:
    pc, dc, ic, _ = spc_encode_capacity(d)
    if caps is not None:
        pc, dc, ic = caps
    nc1 = d["N"] * d["C"] + 1
    return Encoding(
        ptr=torch.empty(max(pc, 1), dtype=torch.int32, device=device),
        da=torch.empty(max(dc, 1), dtype=torch.float32, device=device),
        inn=torch.empty(max(ic, 1), dtype=torch.int32, device=device),
        chan_ptr_off=torch.empty(nc1, dtype=torch.int64, device=device),
        chan_nz_off=torch.empty(nc1, dtype=torch.int64, device=device),
        chan_in_off=torch.empty(nc1, dtype=torch.int64, device=device),
        lengths=torch.zeros(4, dtype=torch.int64, device=device))


def alloc_workspace(d: dict, device="cuda") -> torch.Tensor:
    """Encoder / CPS workspace, zeroed once (spc_workspace_init)."""
    ws = torch.empty(spc_encode_capacity(d)[3], dtype=torch.uint8, device=device)
    spc_workspace_init(ws)
    return ws


def cpo_encode(d: dict, x: torch.Tensor, enc: Encoding, ws: torch.Tensor, stream=None):
    _check(_lib.cpo_encode(ctypes.byref(make_desc(d)), _ptr(x), ctypes.byref(enc.c), _ptr(ws), ws.numel(),
                           _stream(stream)), "cpo_encode")


def cps_encode(d: dict, x: torch.Tensor, enc: Encoding, ws: torch.Tensor, stream=None):
    _check(_lib.cps_encode(ctypes.byref(make_desc(d)), _ptr(x), ctypes.byref(enc.c), _ptr(ws), ws.numel(),
                           _stream(stream)), "cps_encode")


def spc_pack_weights(d: dict, w: torch.Tensor, w_packed: torch.Tensor, stream=None):
    _check(_lib.spc_pack_weights(ctypes.byref(make_desc(d)), _ptr(w), _ptr(w_packed), _stream(stream)),
           "spc_pack_weights")


def sparse_conv_forward(d: dict, enc: Encoding, w_packed: torch.Tensor, y: torch.Tensor, fuse_relu: bool = False,
                        ws: torch.Tensor | None = None, stream=None):
    _check(_lib.sparse_conv_forward(ctypes.byref(make_desc(d)), ctypes.byref(enc.c), _ptr(w_packed), _ptr(y),
                                    int(fuse_relu), _ptr(ws), 0 if ws is None else ws.numel(), _stream(stream)),
           "sparse_conv_forward")


def im2col_conv_forward(d: dict, x: torch.Tensor, w: torch.Tensor, y: torch.Tensor, fuse_relu: bool,
                        ws_lowered: torch.Tensor, stream=None):
    _check(_lib.im2col_conv_forward(ctypes.byref(make_desc(d)), _ptr(x), _ptr(w), _ptr(y), int(fuse_relu),
                                    _ptr(ws_lowered), ws_lowered.numel() * ws_lowered.element_size(),
                                    _stream(stream)), "im2col_conv_forward")


def spc_select_ws_bytes(d: dict) -> int:
    return int(_lib.spc_select_ws_bytes(ctypes.byref(make_desc(d))))


def select_layer_algo(d: dict, samples: torch.Tensor, M: int, w: torch.Tensor, mode: int, reps: int,
                      ws: torch.Tensor, stream=None) -> tuple[int, list[float]]:
    choice = _i32()
    times = (ctypes.c_float * 3)()
    _check(_lib.select_layer_algo(ctypes.byref(make_desc(d)), _ptr(samples), M, _ptr(w), mode, reps,
                                  ctypes.byref(choice), times, _ptr(ws), ws.numel(), _stream(stream)),
           "select_layer_algo")
    return choice.value, [times[0], times[1], times[2]]


def spc_select_from_times(times_ms, sparse_ok: bool, mode: int) -> int:
    """Replay of the selection rule on recorded {im2col, CPO, CPS} times (no GPU work)."""
    t = (ctypes.c_float * 3)(*[float(v) for v in times_ms])
    choice = _i32()
    _check(_lib.spc_select_from_times(t, int(bool(sparse_ok)), int(mode), ctypes.byref(choice)),
           "spc_select_from_times")
    return choice.value


def spc_validate_encoding(d: dict, enc: "Encoding", scratch: torch.Tensor, stream=None) -> None:
    """Debug validator: raises SpcError(SPC_ECORRUPT) for a malformed encoding."""
    _check(_lib.spc_validate_encoding(ctypes.byref(make_desc(d)), ctypes.byref(enc.c), _ptr(scratch),
                                      scratch.numel() * scratch.element_size(), _stream(stream)),
           "spc_validate_encoding")


def spc_encoding_lengths(enc: Encoding, stream=None) -> tuple[int, int, int]:
    out = (_i64 * 3)()
    _check(_lib.spc_encoding_lengths(ctypes.byref(enc.c), out, _stream(stream)), "spc_encoding_lengths")
    return out[0], out[1], out[2]


def spc_version() -> str:
    return _lib.spc_version().decode()


def spc_cscc_capacity(d: dict) -> tuple[int, int, int]:
    p, a, i = _i64(), _i64(), _i64()
    _check(_lib.spc_cscc_capacity(ctypes.byref(make_desc(d)), ctypes.byref(p), ctypes.byref(a), ctypes.byref(i)),
           "spc_cscc_capacity")
    return p.value, a.value, i.value


def alloc_cscc_encoding(d: dict, device="cuda", caps: tuple[int, int, int] | None = None) -> Encoding:
    pc, dc, ic = caps if caps is not None else spc_cscc_capacity(d)
    nc1 = d["N"] * d["C"] + 1
    return Encoding(
        ptr=torch.empty(max(pc, 1), dtype=torch.int32, device=device),
        da=torch.empty(max(dc, 1), dtype=torch.float32, device=device),
        inn=torch.empty(max(ic, 1), dtype=torch.int32, device=device),
        chan_ptr_off=torch.empty(nc1, dtype=torch.int64, device=device),
        chan_nz_off=torch.empty(nc1, dtype=torch.int64, device=device),
        chan_in_off=torch.empty(nc1, dtype=torch.int64, device=device),
        lengths=torch.zeros(4, dtype=torch.int64, device=device))


def cscc_encode(d: dict, x: torch.Tensor, enc: Encoding, stream=None):
    _check(_lib.cscc_encode(ctypes.byref(make_desc(d)), _ptr(x), ctypes.byref(enc.c), _stream(stream)), "cscc_encode")


def cscc_conv_forward(d: dict, enc: Encoding, w_packed: torch.Tensor, y: torch.Tensor, fuse_relu: bool = False,
                      stream=None):
    _check(_lib.cscc_conv_forward(ctypes.byref(make_desc(d)), ctypes.byref(enc.c), _ptr(w_packed), _ptr(y),
                                  int(fuse_relu), _stream(stream)), "cscc_conv_forward")


SPC_SPACE_VS_IM2COL, SPC_SPACE_VS_MEC, SPC_SPACE_VS_CSCC = 0, 1, 2


def spc_space_bound(d: dict, vs: int, rho_hat_bar: float = 0.0) -> float:
    out = ctypes.c_double()
    _check(_lib.spc_space_bound(ctypes.byref(make_desc(d)), int(vs), float(rho_hat_bar), ctypes.byref(out)),
           "spc_space_bound")
    return out.value


def spc_cscc_q_bound(d: dict) -> float:
    out = ctypes.c_double()
    _check(_lib.spc_cscc_q_bound(ctypes.byref(make_desc(d)), ctypes.byref(out)), "spc_cscc_q_bound")
    return out.value


def spc_space_preselect(d: dict, vs: int, rho_bar: float, rho_hat_bar: float = 0.0) -> int:
    out = _i32()
    _check(_lib.spc_space_preselect(ctypes.byref(make_desc(d)), int(vs), float(rho_bar), float(rho_hat_bar),
                                    ctypes.byref(out)), "spc_space_preselect")
    return out.value


def spc_strided_capacity(d: dict) -> tuple[int, int, int]:
    p, a, i = _i64(), _i64(), _i64()
    _check(_lib.spc_strided_capacity(ctypes.byref(make_desc(d)), ctypes.byref(p), ctypes.byref(a), ctypes.byref(i)),
           "spc_strided_capacity")
    return p.value, a.value, i.value


def alloc_strided_encoding(d: dict, device="cuda") -> Encoding:
    return alloc_cscc_encoding(d, device, caps=spc_strided_capacity(d))


def cpo_encode_strided(d: dict, x: torch.Tensor, enc: Encoding, ws: torch.Tensor | None = None, stream=None):
    _check(_lib.cpo_encode_strided(ctypes.byref(make_desc(d)), _ptr(x), ctypes.byref(enc.c),
                                   _ptr(ws) if ws is not None else None, ws.numel() if ws is not None else 0,
                                   _stream(stream)), "cpo_encode_strided")


def alloc_fused_workspace(d: dict, device="cuda") -> torch.Tensor:
    """Workspace of sparse_conv_encode_forward (conv workspace + output masks), zeroed once."""
    ws = torch.empty(int(_lib.spc_fused_ws_bytes(ctypes.byref(make_desc(d)))), dtype=torch.uint8, device=device)
    spc_workspace_init(ws)
    return ws


def sparse_conv_encode_forward(d: dict, enc: Encoding, w_packed: torch.Tensor, y: torch.Tensor, fuse_relu: bool,
                               next_d: dict, out: Encoding, ws: torch.Tensor, stream=None):
    _check(_lib.sparse_conv_encode_forward(ctypes.byref(make_desc(d)), ctypes.byref(enc.c), _ptr(w_packed), _ptr(y),
                                           int(fuse_relu), ctypes.byref(make_desc(next_d)), ctypes.byref(out.c),
                                           _ptr(ws), ws.numel(), _stream(stream)), "sparse_conv_encode_forward")


# ---- device routing: the C ABI launches on the CURRENT device, so every wrapper that
# passes tensors runs with the device of its first CUDA tensor (or encoding) made current.
def _device_of(args, kwargs):
    for a in (*args, *kwargs.values()):
        if isinstance(a, torch.Tensor) and a.is_cuda:
            return a.device
        if isinstance(a, Encoding) and a.ptr.is_cuda:
            return a.ptr.device
    return None


def _on_device(fn):
    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        dev = _device_of(args, kwargs)
        if dev is None or dev.index is None or dev.index == torch.cuda.current_device():
            return fn(*args, **kwargs)
        with torch.cuda.device(dev):
            return fn(*args, **kwargs)
    return wrapped


for _name in ("spc_workspace_init", "cpo_encode", "cps_encode", "spc_pack_weights", "sparse_conv_forward",
              "im2col_conv_forward", "select_layer_algo", "spc_validate_encoding", "spc_encoding_lengths",
              "cscc_encode", "cscc_conv_forward", "cpo_encode_strided", "sparse_conv_encode_forward"):
    globals()[_name] = _on_device(globals()[_name])
