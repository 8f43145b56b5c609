"""Thin ctypes binding over libmpb.so (include/mpb.h).

Argument marshalling only: every arithmetic step runs in the CUDA kernels of
``csrc/``.  PyTorch provides device memory and the current stream.  There is
no CPU fallback: importing this module without the built library, or calling
it without a CUDA device, raises.

Tensor conventions (all ``torch.int32`` holding uint32 bit patterns, on CUDA):
  * operand-major:  shape (count, L)          -- operand k's limbs contiguous
  * word-sliced:    shape (L // 4, count, 4)  -- the device layout of mpb.h
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPB_LIB") or os.path.join(_HERE, "libmpb.so")  # MPB_LIB: tuning builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the CUDA path)"
    )

_lib = ctypes.CDLL(LIB_PATH)
_vp, _sz, _i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
_SIGS = {
    "mpb_limbs": (_i, [_i]),
    "mpb_supported": (_i, [_i]),
    "mpb_layout_expand": (_i, [_vp, _vp, _sz, _i, _vp]),
    "mpb_layout_contract": (_i, [_vp, _vp, _sz, _i, _vp]),
    "mp_batch_mul": (_i, [_vp, _vp, _vp, _sz, _i, _i, _vp, _sz, _vp]),
    "mp_batch_sqr": (_i, [_vp, _vp, _sz, _i, _i, _vp, _sz, _vp]),
    "mp_batch_workspace": (_sz, [_sz, _i, _i]),
    "mont_batch_mul": (_i, [_vp, _vp, _vp, _vp, _vp, _sz, _i, _i, _vp, _sz, _vp]),
    "mont_batch_sqr": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _vp, _sz, _vp]),
    "mont_batch_redc": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _vp, _sz, _vp]),
    "mont_batch_workspace": (_sz, [_sz, _i]),
    "mont_batch_modexp_ct": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _sz, _i, _i, _i, _i, _vp, _sz, _vp]),
    "mont_batch_modexp_ct_workspace": (_sz, [_sz, _i, _i, _i]),
    "mont_batch_setup": (_i, [_vp, _vp, _vp, _sz, _i, _vp, _sz, _vp]),
    "mont_batch_setup_workspace": (_sz, [_sz, _i]),
    "mpb_modexp_host": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _i, _i, _vp]),
    "rsa_batch_crt_ct": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _i, _i, _i, _vp, _sz, _vp]),
    "rsa_batch_crt_workspace": (_sz, [_sz, _i, _i]),
    "mpb_last_error": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

MPB_OK, MPB_EINVAL, MPB_EUNSUPPORTED, MPB_ECUDA = 0, -1, -2, -3
REDC_FULL, REDC_TRUNCATED, REDC_CIOS = 0, 1, 2
ALGO_AUTO, ALGO_SCHOOLBOOK, ALGO_KARATSUBA, ALGO_KARATSUBA2, ALGO_RADIX52, ALGO_HYBRID = 0, 1, 2, 3, 4, 5


class MpbError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == MPB_OK:
        return
    msg = _lib.mpb_last_error().decode()
    if rc in (MPB_EINVAL, MPB_EUNSUPPORTED):
        raise ValueError(f"mpb error {rc}: {msg}")
    raise MpbError(f"mpb error {rc}: {msg}")


def limbs(bits: int) -> int:
    return _lib.mpb_limbs(bits)


def supported(bits: int) -> bool:
    return bool(_lib.mpb_supported(bits))


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if t.dtype != torch.int32:
        raise ValueError("expected torch.int32 (uint32 bit patterns)")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


def _sliced_shape(t: torch.Tensor) -> tuple[int, int]:
    if t.dim() != 3 or t.shape[2] != 4:
        raise ValueError("word-sliced tensors have shape (L//4, count, 4)")
    return 4 * t.shape[0], t.shape[1]


def _expect(t: torch.Tensor | None, L: int, count: int, name: str) -> None:
    """t must be word-sliced with exactly L limbs and `count` operands (the kernels index every
    array with the same L and count: a mismatch would read or write outside the allocation)."""
    if t is None:
        raise ValueError(f"{name} is required")
    shape = tuple(t.shape)
    if shape != (L // 4, count, 4):
        raise ValueError(f"{name}: expected word-sliced shape {(L // 4, count, 4)}, got {shape}")


def _limbs_for(bits: int, L: int, what: str = "operands") -> None:
    Lb = _lib.mpb_limbs(bits)
    if Lb <= 0:
        raise ValueError(f"bits must be positive (got {bits})")
    if Lb != L:
        raise ValueError(f"bits={bits} needs {Lb}-limb {what}, got {L} limbs")


def empty_sliced(L: int, count: int, device="cuda") -> torch.Tensor:
    return torch.empty((L // 4, count, 4), dtype=torch.int32, device=device)


def workspace(nbytes: int, device="cuda") -> torch.Tensor:
    return torch.empty((max(16, nbytes) + 15) // 16 * 4, dtype=torch.int32, device=device)


# ------------------------------------------------------------------- layout
def layout_expand(x: torch.Tensor) -> torch.Tensor:
    """operand-major (count, L) -> word-sliced (L//4, count, 4)  (the paper's `expand`)."""
    count, L = x.shape
    out = empty_sliced(L, count, x.device)
    _check(_lib.mpb_layout_expand(_ptr(x), _ptr(out), count, L, _stream()))
    return out


def layout_contract(y: torch.Tensor) -> torch.Tensor:
    """word-sliced (L//4, count, 4) -> operand-major (count, L)  (the paper's `contract`)."""
    L, count = _sliced_shape(y)
    out = torch.empty((count, L), dtype=torch.int32, device=y.device)
    _check(_lib.mpb_layout_contract(_ptr(y), _ptr(out), count, L, _stream()))
    return out


# --------------------------------------------------------------- products
def mp_workspace(count: int, bits: int, algo: int, device="cuda") -> torch.Tensor | None:
    n = _lib.mp_batch_workspace(count, bits, algo)
    return workspace(n, device) if n else None


def mp_batch_mul(a: torch.Tensor, b: torch.Tensor, bits: int, algo: int = ALGO_AUTO,
                 ws: torch.Tensor | None = None) -> torch.Tensor:
    L, count = _sliced_shape(a)
    _limbs_for(bits, L)
    _expect(b, L, count, "b")
    ws = ws if ws is not None else mp_workspace(count, bits, algo, a.device)
    c = empty_sliced(2 * L, count, a.device)
    _check(_lib.mp_batch_mul(_ptr(a), _ptr(b), _ptr(c), count, bits, algo, _ptr(ws),
                             0 if ws is None else ws.numel() * 4, _stream()))
    return c


def mp_batch_sqr(a: torch.Tensor, bits: int, algo: int = ALGO_AUTO, ws: torch.Tensor | None = None) -> torch.Tensor:
    L, count = _sliced_shape(a)
    _limbs_for(bits, L)
    ws = ws if ws is not None else mp_workspace(count, bits, algo, a.device)
    c = empty_sliced(2 * L, count, a.device)
    _check(_lib.mp_batch_sqr(_ptr(a), _ptr(c), count, bits, algo, _ptr(ws), 0 if ws is None else ws.numel() * 4,
                             _stream()))
    return c


def mont_workspace(count: int, bits: int, device="cuda") -> torch.Tensor:
    return workspace(_lib.mont_batch_workspace(count, bits), device)


def mont_batch_mul(a, b, N, Np, bits: int, redc: int = REDC_TRUNCATED, ws: torch.Tensor | None = None):
    L, count = _sliced_shape(a)
    _limbs_for(bits, L)
    for t, name in ((b, "b"), (N, "N"), (Np, "Np")):
        _expect(t, L, count, name)
    ws = ws if ws is not None else mont_workspace(count, bits, a.device)
    c = empty_sliced(L, count, a.device)
    _check(_lib.mont_batch_mul(_ptr(a), _ptr(b), _ptr(N), _ptr(Np), _ptr(c), count, bits, redc, _ptr(ws),
                               ws.numel() * 4, _stream()))
    return c


def mont_batch_sqr(a, N, Np, bits: int, redc: int = REDC_TRUNCATED, ws: torch.Tensor | None = None):
    L, count = _sliced_shape(a)
    _limbs_for(bits, L)
    for t, name in ((N, "N"), (Np, "Np")):
        _expect(t, L, count, name)
    ws = ws if ws is not None else mont_workspace(count, bits, a.device)
    c = empty_sliced(L, count, a.device)
    _check(_lib.mont_batch_sqr(_ptr(a), _ptr(N), _ptr(Np), _ptr(c), count, bits, redc, _ptr(ws), ws.numel() * 4,
                               _stream()))
    return c


def mont_batch_redc(T, N, Np, bits: int, redc: int = REDC_TRUNCATED, ws: torch.Tensor | None = None):
    L, count = _sliced_shape(N)
    _limbs_for(bits, L)
    _expect(Np, L, count, "Np")
    _expect(T, 2 * L, count, "T")
    ws = ws if ws is not None else mont_workspace(count, bits, N.device)
    c = empty_sliced(L, count, N.device)
    _check(_lib.mont_batch_redc(_ptr(T), _ptr(N), _ptr(Np), _ptr(c), count, bits, redc, _ptr(ws), ws.numel() * 4,
                                _stream()))
    return c


def mont_batch_setup(N: torch.Tensor, bits: int) -> tuple[torch.Tensor, torch.Tensor]:
    L, count = _sliced_shape(N)
    _limbs_for(bits, L)
    Np, R2 = empty_sliced(L, count, N.device), empty_sliced(L, count, N.device)
    ws = workspace(_lib.mont_batch_setup_workspace(count, bits), N.device)
    _check(_lib.mont_batch_setup(_ptr(N), _ptr(Np), _ptr(R2), count, bits, _ptr(ws), ws.numel() * 4, _stream()))
    return Np, R2


def modexp_workspace(count: int, bits: int, window: int, algo: int = ALGO_AUTO, device="cuda") -> torch.Tensor:
    return workspace(_lib.mont_batch_modexp_ct_workspace(count, bits, window, algo), device)


def mont_batch_modexp_ct(N, Np, R2, base, exp, bits: int, window: int = 5, redc: int = REDC_TRUNCATED,
                         algo: int = ALGO_AUTO, ws: torch.Tensor | None = None, out: torch.Tensor | None = None):
    L, count = _sliced_shape(N)
    _limbs_for(bits, L)
    for t, name in ((Np, "Np"), (R2, "R2"), (base, "base"), (exp, "exp")):
        _expect(t, L, count, name)
    ws = ws if ws is not None else modexp_workspace(count, bits, window, algo, N.device)
    if out is not None:
        _expect(out, L, count, "out")
    out = out if out is not None else empty_sliced(L, count, N.device)
    _check(_lib.mont_batch_modexp_ct(_ptr(N), _ptr(Np), _ptr(R2), _ptr(base), _ptr(exp), _ptr(out), count, bits,
                                     window, redc, algo, _ptr(ws), ws.numel() * 4, _stream()))
    return out


def rsa_workspace(count: int, bits: int, window: int, device="cuda") -> torch.Tensor:
    return workspace(_lib.rsa_batch_crt_workspace(count, bits, window), device)


def rsa_batch_crt_ct(c, p, q, dp, dq, qinv, bits: int, window: int = 5, redc: int = REDC_TRUNCATED,
                     ws: torch.Tensor | None = None, out: torch.Tensor | None = None):
    """m = c^d mod pq by CRT (word-sliced: c with L(bits) limbs, p/q/dp/dq/qinv with L(bits/2))."""
    L, count = _sliced_shape(c)
    _limbs_for(bits, L)
    Lh = _lib.mpb_limbs(bits // 2)
    for t, name in ((p, "p"), (q, "q"), (dp, "dp"), (dq, "dq"), (qinv, "qinv")):
        _expect(t, Lh, count, name)
    ws = ws if ws is not None else rsa_workspace(count, bits, window, c.device)
    if out is not None:
        _expect(out, L, count, "out")
    out = out if out is not None else empty_sliced(L, count, c.device)
    _check(_lib.rsa_batch_crt_ct(_ptr(c), _ptr(p), _ptr(q), _ptr(dp), _ptr(dq), _ptr(qinv), _ptr(out), count, bits,
                                 window, redc, _ptr(ws), ws.numel() * 4, _stream()))
    return out


def modexp_host(N: np.ndarray, base: np.ndarray, exp: np.ndarray, bits: int, window: int = 5,
                redc: int = REDC_TRUNCATED) -> np.ndarray:
    """End-to-end over host buffers (operand-major uint32 (count, L)); blocking."""
    N, base, exp = (np.ascontiguousarray(x, dtype=np.uint32) for x in (N, base, exp))
    if N.ndim != 2:
        raise ValueError("operand-major arrays have shape (count, L)")
    count, L = N.shape
    _limbs_for(bits, L)
    if base.shape != N.shape or exp.shape != N.shape:
        raise ValueError(f"N, base and exp must all have shape {N.shape}, got {base.shape} and {exp.shape}")
    out = np.empty_like(N)
    _check(_lib.mpb_modexp_host(N.ctypes.data, base.ctypes.data, exp.ctypes.data, out.ctypes.data, count, bits,
                                window, redc, _stream()))
    return out


def modexp_host_ptrs(N: int, base: int, exp: int, out: int, count: int, bits: int, window: int, redc: int,
                     stream: int) -> None:
    """mpb_modexp_host on raw host pointers (operand-major, count x mpb_limbs(bits) limbs each; the
    caller guarantees the sizes) and an explicit cudaStream_t handle (multi-device drivers)."""
    _check(_lib.mpb_modexp_host(N, base, exp, out, count, bits, window, redc, stream))


# ------------------------------------------------------- host <-> device
def to_device(x: np.ndarray, device="cuda") -> torch.Tensor:
    """operand-major uint32 numpy (count, L) -> word-sliced CUDA tensor."""
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).to(device)
    return layout_expand(t)


def to_host(y: torch.Tensor) -> np.ndarray:
    """word-sliced CUDA tensor -> operand-major uint32 numpy (count, L)."""
    return layout_contract(y).cpu().numpy().view(np.uint32)
