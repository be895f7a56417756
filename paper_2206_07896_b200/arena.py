"""DeviceArena — the reference's memory shim (arena.py:66-152) over B200 HBM.

Same surface and error behaviour as `blockfuse.arena`: integer handles from 1,
never reused; `alloc` zero-fills; out-of-range element access and dangling
handles raise `Trap("OutOfBounds")`; f32 stores round to single precision.
The storage is device memory owned by libbfgpu.so; host values are staged
through pinned memory on every call (host buffers are borrowed, not kept).
"""

from __future__ import annotations

import ctypes as C
import struct
import threading
from array import array
from typing import Iterable

import numpy as np

from . import _lib
from ._lib import BfError, check

_TYPECODE = {"i32": "i", "i64": "q", "f32": "f", "f64": "d"}
_NP = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64}
SCALAR_SIZE = {"i32": 4, "i64": 8, "f32": 4, "f64": 8}
TRACE_ALIGN = 64


class Trap(Exception):
    """Runtime fault inside a kernel; always trapped, never undefined behavior.

    Mirrors blockfuse.arena.Trap (arena.py:24-36)."""

    def __init__(self, kind: str, message: str, *, kernel: str = "?",
                 section: int = -1, tid: int = -1, span=None):
        self.kind = kind  # OutOfBounds | DivByZero | TypeFault | NonUniformTrip
        self.message = message
        self.kernel = kernel
        self.section = section
        self.tid = tid
        self.span = span
        super().__init__(f"[{kind}] {message} (kernel={kernel}, section={section}, "
                         f"tid={tid}, span={span})")


def wrap_int(value: int, ty: str) -> int:
    """i32/i64 two's-complement wrap (arena.py:39-41)."""
    bits = 32 if ty == "i32" else 64
    return (value + (1 << (bits - 1))) % (1 << bits) - (1 << (bits - 1))


class DeviceArena:
    """Handle-addressed buffers in the HBM of one B200 (arena.py:66-152)."""

    def __init__(self, device: int = 0):
        L = _lib.lib()
        self.device = device
        self._ptr = C.c_void_p()
        check(L.bf_arena_create(device, C.byref(self._ptr)))
        self._meta: dict[int, tuple[str, int]] = {}
        self._bases: dict[int, int] = {}
        self._next_base = 0
        # the reference's global atomic lock; device atomics need none, the
        # attribute stays for API compatibility (executor.py:190)
        self.atomic_lock = threading.Lock()

    # -- lifetime -------------------------------------------------------------
    def close(self) -> None:
        if self._ptr:
            _lib.lib().bf_arena_destroy(self._ptr)
            self._ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def native(self) -> C.c_void_p:
        return self._ptr

    # -- reference surface ------------------------------------------------------
    def alloc(self, scalar: str, length: int) -> int:
        if length < 0:
            raise ValueError(f"negative buffer length {length}")
        if scalar not in _lib.SCALARS:
            raise ValueError(f"unknown scalar type {scalar!r}")
        h = C.c_uint32()
        check(_lib.lib().bf_alloc(self._ptr, _lib.SCALARS[scalar], length, C.byref(h)))
        self._meta[h.value] = (scalar, length)
        nbytes = length * SCALAR_SIZE[scalar]
        self._bases[h.value] = self._next_base
        self._next_base += -(-max(nbytes, 1) // TRACE_ALIGN) * TRACE_ALIGN
        return h.value

    def free(self, handle: int) -> None:
        self._buf(handle)
        check(_lib.lib().bf_free(self._ptr, handle))
        del self._meta[handle]

    def view(self, handle: int, first: int, length: int) -> int:
        """A new handle aliasing elements [first, first + length) of `handle`
        (bf_view: no copy, 16 B-aligned offset); freed with free()."""
        scalar, _ = self._buf(handle)
        h = C.c_uint32()
        check(_lib.lib().bf_view(self._ptr, handle, first, length, C.byref(h)))
        self._meta[h.value] = (scalar, length)
        self._bases[h.value] = self._bases[handle] + first * SCALAR_SIZE[scalar]
        return h.value

    def _buf(self, handle: int) -> tuple[str, int]:
        m = self._meta.get(handle)
        if m is None:
            raise Trap("OutOfBounds", f"dangling buffer handle {handle}")
        return m

    def buffer(self, handle: int):
        return self._buf(handle)

    def scalar_type(self, handle: int) -> str:
        return self._buf(handle)[0]

    def length(self, handle: int) -> int:
        return self._buf(handle)[1]

    def base_address(self, handle: int) -> int:
        """Synthetic 64 B-aligned trace base (arena.py:21,80-82)."""
        self._buf(handle)
        return self._bases[handle]

    def device_ptr(self, handle: int) -> int:
        p = C.c_uint64()
        check(_lib.lib().bf_buffer_info(self._ptr, handle, None, None, C.byref(p)))
        return p.value

    def read(self, handle: int, index: int):
        scalar, length = self._buf(handle)
        if not 0 <= index < length:
            raise Trap("OutOfBounds", f"load index {index} out of range [0, {length})")
        raw = self._download(handle, SCALAR_SIZE[scalar], index * SCALAR_SIZE[scalar])
        return array(_TYPECODE[scalar], raw)[0]

    def write(self, handle: int, index: int, value) -> None:
        scalar, length = self._buf(handle)
        if not 0 <= index < length:
            raise Trap("OutOfBounds", f"store index {index} out of range [0, {length})")
        raw = array(_TYPECODE[scalar], [value]).tobytes()
        self._upload(handle, raw, index * SCALAR_SIZE[scalar])

    def to_list(self, handle: int) -> list:
        scalar, _ = self._buf(handle)
        return self.to_numpy(handle).tolist() if scalar in ("i32", "i64") else \
            array(_TYPECODE[scalar], self.to_bytes(handle)).tolist()

    def fill(self, handle: int, values: Iterable) -> None:
        """Store values[i] at i for i < length; extra values are ignored."""
        scalar, length = self._buf(handle)
        if isinstance(values, np.ndarray):
            data = np.ascontiguousarray(values[:length], dtype=_NP[scalar])
            raw = data.tobytes()
        else:
            buf = array(_TYPECODE[scalar])
            for i, v in enumerate(values):
                if i >= length:
                    break
                buf.append(v)
            raw = buf.tobytes()
        if raw:
            self._upload(handle, raw, 0)

    def to_bytes(self, handle: int) -> bytes:
        scalar, length = self._buf(handle)
        return self._download(handle, length * SCALAR_SIZE[scalar], 0)

    def from_bytes(self, handle: int, raw: bytes) -> None:
        scalar, length = self._buf(handle)
        expect = length * SCALAR_SIZE[scalar]
        if len(raw) != expect:
            raise ValueError(f"buffer file is {len(raw)} bytes, expected {expect}")
        if raw:
            self._upload(handle, raw, 0)

    # -- numpy helpers (not in the reference) -----------------------------------
    def to_numpy(self, handle: int) -> np.ndarray:
        scalar, length = self._buf(handle)
        out = np.empty(length, dtype=_NP[scalar])
        if length:
            check(_lib.lib().bf_download(self._ptr, handle, out.ctypes.data_as(C.c_void_p),
                                         out.nbytes, 0))
        return out

    def upload_numpy(self, handle: int, values: np.ndarray, offset_elems: int = 0) -> None:
        scalar, length = self._buf(handle)
        data = np.ascontiguousarray(values, dtype=_NP[scalar])
        if offset_elems < 0 or offset_elems + data.size > length:
            raise ValueError("upload range outside the buffer")
        if data.size:
            check(_lib.lib().bf_upload(self._ptr, handle, data.ctypes.data_as(C.c_void_p),
                                       data.nbytes, offset_elems * SCALAR_SIZE[scalar]))

    def download_into(self, handle: int, out: np.ndarray, offset_elems: int = 0) -> np.ndarray:
        scalar, length = self._buf(handle)
        if out.dtype != _NP[scalar] or not out.flags.c_contiguous:
            raise ValueError("destination must be a contiguous array of the buffer's type")
        if offset_elems < 0 or offset_elems + out.size > length:
            raise ValueError("download range outside the buffer")
        if out.size:
            check(_lib.lib().bf_download(self._ptr, handle, out.ctypes.data_as(C.c_void_p),
                                         out.nbytes, offset_elems * SCALAR_SIZE[scalar]))
        return out

    def fill_value(self, handle: int, value) -> None:
        """Set every element to `value` on the device (4-byte scalars)."""
        scalar, length = self._buf(handle)
        if SCALAR_SIZE[scalar] != 4:
            raise ValueError("fill_value supports 4-byte scalars")
        pat = struct.unpack("<I", struct.pack("<" + _TYPECODE[scalar], value))[0]
        check(_lib.lib().bf_fill32(self._ptr, handle, pat, 0, length * 4))

    def copy(self, dst: int, src: int) -> None:
        s_scalar, s_len = self._buf(src)
        d_scalar, d_len = self._buf(dst)
        if s_scalar != d_scalar or s_len != d_len:
            raise ValueError("copy needs buffers of the same type and length")
        check(_lib.lib().bf_copy(self._ptr, dst, 0, src, 0, s_len * SCALAR_SIZE[s_scalar]))

    def cuda_array(self, handle: int):
        """An object exposing __cuda_array_interface__ over the buffer, so
        torch.as_tensor(obj, device="cuda") aliases it without a copy."""
        scalar, length = self._buf(handle)
        ptr = self.device_ptr(handle)
        typestr = {"i32": "<i4", "i64": "<i8", "f32": "<f4", "f64": "<f8"}[scalar]

        class _View:
            __cuda_array_interface__ = {"shape": (length,), "typestr": typestr,
                                        "data": (ptr, False), "version": 2}
        return _View()

    # -- raw copies -------------------------------------------------------------
    def _upload(self, handle: int, raw: bytes, offset: int) -> None:
        try:
            check(_lib.lib().bf_upload(self._ptr, handle, raw, len(raw), offset))
        except BfError as e:
            if e.code == _lib.E_DANGLING:
                raise Trap("OutOfBounds", f"dangling buffer handle {handle}") from None
            raise

    def _download(self, handle: int, nbytes: int, offset: int) -> bytes:
        out = C.create_string_buffer(nbytes)
        try:
            check(_lib.lib().bf_download(self._ptr, handle, out, nbytes, offset))
        except BfError as e:
            if e.code == _lib.E_DANGLING:
                raise Trap("OutOfBounds", f"dangling buffer handle {handle}") from None
            raise
        return out.raw
