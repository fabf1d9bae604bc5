"""ctypes binding of the C ABI in include/flashsplat_b200.h.

The shared library is built in-tree (``csrc/Makefile`` ->
``_lib/libflashsplat_b200.so``) by ``__graft_entry__.build()``.  There is no
fallback: if the library or a CUDA device is missing every compute call
raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref
from pathlib import Path

import numpy as np

# FS_LIB=checked selects the bounds-checked build (csrc/Makefile ``checked``)
LIB_PATH = (Path(__file__).resolve().parent
            / ("_lib_checked" if os.environ.get("FS_LIB") == "checked" else "_lib")
            / "libflashsplat_b200.so")

FS_OK, FS_EINVAL, FS_ECUDA, FS_ENOMEM, FS_ELABEL = 0, 1, 2, 3, 4
MODE_BINARY, MODE_SCENE = 0, 1
# accumulator kinds (include/flashsplat_b200.h): float64 entries, or the
# deterministic fixed-point pair of uint64 words (schedule-independent sums)
ACC_F64, ACC_FIXED = 0, 1
ACC_DEFAULT = ACC_FIXED


def acc_entry_bytes(kind: int) -> int:
    return 16 if kind == ACC_FIXED else 8

# Every symbol include/flashsplat_b200.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "fs_last_error", "fs_version", "fs_create", "fs_destroy", "fs_device_count",
    "fs_device_alloc", "fs_device_free", "fs_memset_zero", "fs_copy_to_device",
    "fs_copy_to_host", "fs_synchronize", "fs_set_stream", "fs_host_alloc", "fs_host_free",
    "fs_host_pinned", "fs_set_timing", "fs_set_scene", "fs_set_scene_ply", "fs_copy_scene",
    "fs_project", "fs_bin", "fs_bin_splats",
    "fs_accumulate", "fs_accumulate_multi", "fs_finalize", "fs_reduce_finalize",
    "fs_enable_peer_access", "fs_finalize_multi", "fs_assign", "fs_member_counts", "fs_render",
    "fs_render_splats", "fs_render_mask", "fs_decode_mask_png",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library is not built or no sm_100 device is usable."""


class LabelRangeError(ValueError):
    """A mask label >= num_objects; `view` is the first offending view's position."""

    def __init__(self, msg: str, view: int):
        super().__init__(msg)
        self.view = view


class FsCamera(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("fx", ctypes.c_double), ("fy", ctypes.c_double),
        ("cx", ctypes.c_double), ("cy", ctypes.c_double),
        ("world_to_camera", ctypes.c_double * 16), ("near_clip", ctypes.c_double),
    ]


class FsProjectionStats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in
                ("n_input", "n_emitted", "n_behind", "n_degenerate", "n_offscreen")]


class FsAccumulateStats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in
                ("views", "view_pixels", "emitted", "instances", "tile_steps", "exact_evals",
                 "atomics", "retried_views", "launches", "label_error_view")] + [
                    (k, ctypes.c_double) for k in ("gpu_ms", "prep_ms", "bin_ms", "raster_ms")]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_lib_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load the library (once); raise NativeUnavailable if it is not built."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeUnavailable(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = ctypes.CDLL(str(LIB_PATH))
        P, I, I64, D, F = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double,
                           ctypes.c_float)
        sig = {
            "fs_last_error": ([], ctypes.c_char_p),
            "fs_version": ([], ctypes.c_char_p),
            "fs_create": ([I, I, ctypes.POINTER(P)], I),
            "fs_destroy": ([P], None),
            "fs_device_count": ([ctypes.POINTER(I)], I),
            "fs_device_alloc": ([P, ctypes.c_uint64, ctypes.POINTER(P)], I),
            "fs_device_free": ([P, P], I),
            "fs_memset_zero": ([P, P, ctypes.c_uint64], I),
            "fs_copy_to_device": ([P, P, P, ctypes.c_uint64], I),
            "fs_copy_to_host": ([P, P, P, ctypes.c_uint64], I),
            "fs_synchronize": ([P], I),
            "fs_set_stream": ([P, P], I),
            "fs_host_alloc": ([P, ctypes.c_uint64, ctypes.POINTER(P)], I),
            "fs_host_free": ([P, P], I),
            "fs_host_pinned": ([P, ctypes.c_uint64], I),
            "fs_set_timing": ([P, I], I),
            "fs_set_scene": ([P, I64, P, P, P, P], I),
            "fs_set_scene_ply": ([P, I64, P, I, P, P, P], I),
            "fs_copy_scene": ([P, P], I),
            "fs_project": ([P, P, P, P, P, P, P, P], I),
            "fs_bin": ([P, P, P, P, I64, ctypes.POINTER(I64)], I),
            "fs_bin_splats": ([P, I64, P, P, P, P, I, I, P, P, I64, ctypes.POINTER(I64)], I),
            "fs_accumulate": ([P, I, P, P, I, I, D, D, I, P, P], I),
            "fs_accumulate_multi": ([P, I, I, P, P, I, D, D, I, P, P, P], I),
            "fs_finalize": ([P, I, P, I64, I, P, I], I),
            "fs_reduce_finalize": ([P, I, P, I, I64, I64, I, I64, I64, P, I64, I], I),
            "fs_enable_peer_access": ([P, I], I),
            "fs_finalize_multi": ([P, I, I, P, I64, I, P, F, I, P], I),
            "fs_member_counts": ([P, P, I64, I, P], I),
            "fs_assign": ([P, P, I64, I, F, I, P, I], I),
            "fs_render": ([P, P, P, D, D, P, I, P, P, P], I),
            "fs_render_splats": ([P, I, I, I64, P, P, P, P, P, P, D, D, P, I, P, P, P], I),
            "fs_render_mask": ([P, P, P, I, D, D, D, P], I),
            "fs_decode_mask_png": ([P, I64, P, I64, ctypes.POINTER(I), ctypes.POINTER(I)], I),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def _check(rc: int) -> None:
    if rc == FS_OK:
        return
    msg = load().fs_last_error().decode(errors="replace")
    if rc == FS_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def device_count() -> int:
    c = ctypes.c_int(0)
    rc = load().fs_device_count(ctypes.byref(c))
    return c.value if rc == FS_OK else 0


def camera_struct(view) -> FsCamera:
    c = FsCamera()
    c.width, c.height = int(view.width), int(view.height)
    c.fx, c.fy, c.cx, c.cy = float(view.fx), float(view.fy), float(view.cx), float(view.cy)
    w = np.ascontiguousarray(view.world_to_camera, dtype=np.float64).reshape(16)
    ctypes.memmove(c.world_to_camera, w.ctypes.data, 16 * 8)
    c.near_clip = float(view.near_clip)
    return c


def _p(a) -> int:
    return None if a is None else a.ctypes.data


class DeviceBuffer:
    """A cudaMalloc'ed block owned by a Context (freed on release / GC)."""

    def __init__(self, ctx: "Context", nbytes: int):
        self.ctx = ctx
        self.nbytes = int(nbytes)
        ptr = ctypes.c_void_p()
        _check(load().fs_device_alloc(ctx.handle, self.nbytes, ctypes.byref(ptr)))
        self.ptr = ptr.value

    def zero(self) -> "DeviceBuffer":
        _check(load().fs_memset_zero(self.ctx.handle, self.ptr, self.nbytes))
        return self

    def to_host(self, out: np.ndarray) -> np.ndarray:
        assert out.nbytes <= self.nbytes
        _check(load().fs_copy_to_host(self.ctx.handle, _p(out), self.ptr, out.nbytes))
        return out

    def from_host(self, arr: np.ndarray) -> "DeviceBuffer":
        arr = np.ascontiguousarray(arr)
        assert arr.nbytes <= self.nbytes
        _check(load().fs_copy_to_device(self.ctx.handle, self.ptr, _p(arr), arr.nbytes))
        return self

    def release(self) -> None:
        if self.ptr and self.ctx.handle:
            load().fs_device_free(self.ctx.handle, self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class Context:
    """fs_context: one device, its streams, workspaces and the resident scene."""

    def __init__(self, device: int = 0, streams: int = 6):
        L = load()
        h = ctypes.c_void_p()
        rc = L.fs_create(int(device), int(streams), ctypes.byref(h))
        if rc != FS_OK:
            raise NativeUnavailable(L.fs_last_error().decode(errors="replace"))
        self.handle = h.value
        self.device = int(device)
        self._scene_key = None
        self.n = 0
        self.lock = threading.RLock()
        self._buffers: dict = {}
        self._pinned_pool: dict = {}
        self._pin_lock = threading.Lock()

    def set_timing(self, enable: bool) -> None:
        _check(load().fs_set_timing(self.handle, 1 if enable else 0))

    def set_stream(self, stream_handle: int) -> None:
        """Order the context's work after this CUDA stream (e.g. torch's current stream)."""
        _check(load().fs_set_stream(self.handle, int(stream_handle) or None))

    def close(self) -> None:
        for buf in getattr(self, "_buffers", {}).values():
            buf.release()
        self._buffers = {}
        if self.handle:
            for ptrs in getattr(self, "_pinned_pool", {}).values():
                for ptr in ptrs:
                    load().fs_host_free(self.handle, ptr)
            self._pinned_pool = {}
            load().fs_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- scene ---------------------------------------------------------------
    def set_scene(self, scene) -> None:
        if getattr(scene, "_ply_block", None) is not None:  # scene_io.PlyScene: raw records
            key = ("ply", id(scene), len(scene))
            if key != self._scene_key:
                self.set_scene_ply(scene)
                self._scene_key = key
                self._scene_ref = scene
            return
        key = (id(scene), len(scene), scene.means.ctypes.data, scene.rotations.ctypes.data,
               scene.scales.ctypes.data, scene.opacities.ctypes.data)
        if key == self._scene_key:
            return
        m = np.ascontiguousarray(scene.means, dtype=np.float64)
        q = np.ascontiguousarray(scene.rotations, dtype=np.float64)
        s = np.ascontiguousarray(scene.scales, dtype=np.float64)
        o = np.ascontiguousarray(scene.opacities, dtype=np.float64)
        _check(load().fs_set_scene(self.handle, len(scene), _p(m), _p(q), _p(s), _p(o)))
        self._scene_key = key
        self._scene_ref = scene  # keep the id() stable while cached
        self.n = len(scene)

    def copy_scene_from(self, src: "Context") -> None:
        """fs_copy_scene: take src's resident scene (device to device / NVLink)."""
        if src is self:
            return
        self._scene_key = None
        _check(load().fs_copy_scene(self.handle, src.handle))
        self._scene_key = src._scene_key
        self._scene_ref = getattr(src, "_scene_ref", None)
        self.n = src.n

    def set_scene_ply(self, scene, params: np.ndarray = None) -> np.ndarray:
        """fs_set_scene_ply: a PlyScene's float32 records -> the resident scene
        (activations + validation on the device).  Returns bad[4] (first
        offending vertex per check, -1 = none); raises nothing itself."""
        bad = np.full(4, -1, np.int64)
        offs = np.ascontiguousarray(scene._ply_offsets, dtype=np.int32)
        self._scene_key = None
        rc = load().fs_set_scene_ply(self.handle, len(scene), scene._ply_block.ctypes.data,
                                     int(scene._ply_stride), _p(offs), _p(bad), _p(params))
        if rc != FS_OK and not (bad >= 0).any():
            _check(rc)
        self.n = len(scene) if rc == FS_OK else 0
        return bad

    def set_arrays(self, means, quats, scales, opac) -> None:
        m = np.ascontiguousarray(means, dtype=np.float64).reshape(-1, 3)
        n = m.shape[0]
        q = np.ascontiguousarray(quats, dtype=np.float64).reshape(n, 4)
        s = np.ascontiguousarray(scales, dtype=np.float64).reshape(n, 3)
        o = np.ascontiguousarray(opac, dtype=np.float64).reshape(n)
        _check(load().fs_set_scene(self.handle, n, _p(m), _p(q), _p(s), _p(o)))
        self._scene_key = None
        self.n = n

    # -- stages --------------------------------------------------------------
    def project(self, view):
        n = self.n
        alive = np.zeros(n, np.uint8)
        mean2d = np.zeros((n, 2))
        conic = np.zeros((n, 3))
        depth = np.zeros(n)
        radius = np.zeros(n, np.int64)
        st = FsProjectionStats()
        cam = camera_struct(view)
        _check(load().fs_project(self.handle, ctypes.byref(cam), _p(alive), _p(mean2d),
                                 _p(conic), _p(depth), _p(radius), ctypes.byref(st)))
        stats = (st.n_input, st.n_emitted, st.n_behind, st.n_degenerate, st.n_offscreen)
        return alive.astype(bool), mean2d, conic, depth, radius, stats

    def render(self, view, member, alpha_floor: float, t_floor: float, channel=None):
        """fs_render over the resident scene: (value | None, alpha, depth)."""
        h, w = view.height, view.width
        # every pixel is written by the D2H copies: page-locked, uninitialised
        alpha = self.pinned_empty((h, w), np.float64)
        depth = self.pinned_empty((h, w), np.float64)
        channels, value, ch = 0, None, None
        if channel is not None:
            ch = np.ascontiguousarray(channel, dtype=np.float64)
            channels = 1 if ch.ndim == 1 else ch.shape[1]
            value = self.pinned_empty((h, w) if channels == 1 else (h, w, channels), np.float64)
        mem = None if member is None else np.ascontiguousarray(member, dtype=np.uint8)
        cam = camera_struct(view)
        _check(load().fs_render(self.handle, ctypes.byref(cam), _p(mem), float(alpha_floor),
                                float(t_floor), _p(ch), channels, _p(value), _p(alpha),
                                _p(depth)))
        return value, alpha, depth

    def render_mask(self, view, membership, tau: float, alpha_floor: float, t_floor: float):
        """fs_render_mask: H x W uint16 labels (membership: E x N)."""
        membership = np.ascontiguousarray(membership, dtype=np.uint8)
        labels = self.pinned_empty((view.height, view.width), np.uint16)
        cam = camera_struct(view)
        _check(load().fs_render_mask(self.handle, ctypes.byref(cam), _p(membership),
                                     int(membership.shape[0]), float(tau), float(alpha_floor),
                                     float(t_floor), _p(labels)))
        return labels

    def bin(self, view):
        cam = camera_struct(view)
        ntiles = ((view.width + 15) // 16) * ((view.height + 15) // 16)
        offs = np.zeros(ntiles + 1, np.int64)
        count = ctypes.c_int64(0)
        L = load()
        _check(L.fs_bin(self.handle, ctypes.byref(cam), _p(offs), None, 0, ctypes.byref(count)))
        items = np.zeros(max(count.value, 1), np.int64)
        _check(L.fs_bin(self.handle, ctypes.byref(cam), _p(offs), _p(items), items.size,
                        ctypes.byref(count)))
        return offs, items[:count.value]

    def accumulate(self, views, masks, num_objects: int, alpha_floor: float, t_floor: float,
                   acc_ptr: int, masks_on_device: bool = False, acc_kind: int = ACC_DEFAULT) -> dict:
        """Add every view's alpha*T mass into the N x E (Gaussian-major) device accumulator
        acc_ptr of kind ``acc_kind`` (ACC_F64 / ACC_FIXED)."""
        nv = len(views)
        cams = (FsCamera * max(nv, 1))(*[camera_struct(v) for v in views])
        if masks_on_device:
            ptrs = (ctypes.c_void_p * max(nv, 1))(*[int(m) for m in masks])
        else:
            keep = [np.ascontiguousarray(m, dtype=np.uint16) for m in masks]
            ptrs = (ctypes.c_void_p * max(nv, 1))(*[k.ctypes.data for k in keep])
        st = FsAccumulateStats()
        L = load()
        rc = L.fs_accumulate(self.handle, nv, ctypes.byref(cams), ctypes.byref(ptrs),
                             1 if masks_on_device else 0, int(num_objects), float(alpha_floor),
                             float(t_floor), int(acc_kind), acc_ptr, ctypes.byref(st))
        if rc == FS_ELABEL:
            raise LabelRangeError(L.fs_last_error().decode(errors="replace"),
                                  int(st.label_error_view))
        _check(rc)
        return st.as_dict()

    def acc_buffer(self, num_objects: int, n: int, acc_kind: int = ACC_DEFAULT,
                   role: str = "acc") -> "DeviceBuffer":
        """Grow-only N x E accumulator of kind ``acc_kind`` (not zeroed)."""
        return self.buffer(role, acc_entry_bytes(acc_kind) * int(num_objects) * max(int(n), 1))

    def buffer(self, role: str, nbytes: int) -> "DeviceBuffer":
        """Grow-only device scratch owned by the context, keyed by role."""
        buf = self._buffers.get(role)
        if buf is None or buf.ptr is None or buf.nbytes < nbytes:  # (re)allocate if released
            if buf is not None:
                buf.release()
            buf = DeviceBuffer(self, max(int(nbytes), 1))
            self._buffers[role] = buf
        return buf

    def finalize(self, acc_ptr: int, n: int, e: int, out_ptr: int = None,
                 out: np.ndarray = None, acc_kind: int = ACC_DEFAULT):
        """N x E accumulator -> E x N float32 (host ``out`` or device ``out_ptr``)."""
        if out is not None:
            _check(load().fs_finalize(self.handle, int(acc_kind), acc_ptr, n, e, _p(out), 0))
            return out
        _check(load().fs_finalize(self.handle, int(acc_kind), acc_ptr, n, e, out_ptr, 1))
        return None

    def reduce_finalize(self, parts, part_g0: int, n: int, e: int, g0: int, g1: int,
                        out_ptr: int, ld: int, out_on_device: bool = True,
                        acc_kind: int = ACC_DEFAULT) -> None:
        """Sum of accumulator parts over Gaussians [g0, g1) -> float32 E x (g1-g0) at out_ptr."""
        arr = (ctypes.c_void_p * len(parts))(*[int(p) for p in parts])
        _check(load().fs_reduce_finalize(self.handle, int(acc_kind), arr, len(parts), int(part_g0),
                                         int(n), int(e), int(g0), int(g1), out_ptr, int(ld),
                                         1 if out_on_device else 0))

    def member_counts(self, dev_ptr: int, n: int, rows: int) -> list:
        """Nonzero bytes per row of a rows x n uint8 device matrix (fs_member_counts)."""
        out = np.zeros(max(rows, 1), np.int64)
        _check(load().fs_member_counts(self.handle, dev_ptr, int(n), int(rows), _p(out)))
        return [int(x) for x in out[:rows]]

    def alloc(self, nbytes: int) -> DeviceBuffer:
        return DeviceBuffer(self, nbytes)

    def pinned_empty(self, shape, dtype) -> np.ndarray:
        """numpy array in page-locked host memory (device -> host copies at full
        DMA speed).  Blocks are pooled by size: when the array (or any view of
        it) is garbage-collected its block returns to the pool."""
        dtype = np.dtype(dtype)
        count = int(np.prod(shape)) if len(shape) else 1
        nbytes = max(count * dtype.itemsize, 1)
        with self._pin_lock:
            pool = self._pinned_pool.setdefault(nbytes, [])
            ptr = pool.pop() if pool else None
        if ptr is None:
            p = ctypes.c_void_p()
            _check(load().fs_host_alloc(self.handle, nbytes, ctypes.byref(p)))
            ptr = p.value
        holder = (ctypes.c_char * nbytes).from_address(ptr)
        weakref.finalize(holder, self._pinned_release, nbytes, ptr)
        return np.frombuffer(holder, dtype=dtype, count=count).reshape(shape)

    def _pinned_release(self, nbytes: int, ptr: int) -> None:
        with self._pin_lock:
            pool = self._pinned_pool.setdefault(nbytes, [])
            if len(pool) < 4 and self.handle:
                pool.append(ptr)
                return
        if self.handle:
            load().fs_host_free(self.handle, ptr)


def assign(values: np.ndarray, gamma: float, mode: int, ctx: Context = None,
           on_device_ptr: int = None, n: int = None, e: int = None, out_ptr: int = None):
    """fs_assign on host arrays (returns uint8) or on device pointers (in place).

    Host arrays go through the (default) context's cached device buffers,
    under the context lock.
    """
    L = load()
    if ctx is None:
        ctx = context()
    # fs_assign is reentrant (per-thread stream, stream-ordered scratch, no
    # context state): no lock, so service threads never wait on an accumulation
    if on_device_ptr is not None:
        _check(L.fs_assign(ctx.handle, on_device_ptr, int(n), int(e), float(gamma), int(mode),
                           out_ptr, 1))
        return None
    values = np.ascontiguousarray(values, dtype=np.float32)
    e, n = values.shape
    out = np.zeros(n if mode == MODE_BINARY else (e, n), np.uint8)
    _check(L.fs_assign(ctx.handle, _p(values), int(n), int(e), float(gamma), int(mode),
                       _p(out), 0))
    return out


_contexts: dict = {}
_ctx_lock = threading.Lock()


def default_device() -> int:
    env = os.environ.get("LOCAL_RANK")
    if env is not None and device_count() > 1:
        return int(env) % device_count()
    return 0


def context(device: int = None, slot: int = 0) -> Context:
    """Process-wide cached context per device (``slot`` > 0: further independent
    contexts on the same device, e.g. a device listed twice in ``devices=``)."""
    if device is None:
        device = default_device()
    key = (int(device), int(slot))
    with _ctx_lock:
        ctx = _contexts.get(key)
        if ctx is None:
            ctx = Context(key[0])
            _contexts[key] = ctx
        return ctx


def accumulate_multi(ctxs, views, masks, num_objects: int, alpha_floor: float, t_floor: float,
                     acc_ptrs, acc_kind: int = ACC_DEFAULT):
    """fs_accumulate_multi: one host thread per context, shared dynamic view queue.
    Returns (stats dict, per-view context index)."""
    nv = len(views)
    cams = (FsCamera * max(nv, 1))(*[camera_struct(v) for v in views])
    keep = [np.ascontiguousarray(m, dtype=np.uint16) for m in masks]
    ptrs = (ctypes.c_void_p * max(nv, 1))(*[k.ctypes.data for k in keep])
    handles = (ctypes.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
    accs = (ctypes.c_void_p * len(ctxs))(*[int(p) for p in acc_ptrs])
    owner = np.full(max(nv, 1), -1, np.int32)
    st = FsAccumulateStats()
    L = load()
    rc = L.fs_accumulate_multi(handles, len(ctxs), nv, ctypes.byref(cams), ctypes.byref(ptrs),
                               int(num_objects), float(alpha_floor), float(t_floor), int(acc_kind),
                               accs, _p(owner), ctypes.byref(st))
    if rc == FS_ELABEL:
        raise LabelRangeError(L.fs_last_error().decode(errors="replace"), int(st.label_error_view))
    _check(rc)
    return st.as_dict(), owner[:nv]


def finalize_multi(ctxs, acc_ptrs, n: int, e: int, out: np.ndarray, gamma: float = 0.0,
                   mode: int = -1, labels: np.ndarray = None, acc_kind: int = ACC_DEFAULT) -> None:
    """fs_finalize_multi: slice i of A reduced over all contexts' accumulators on context i
    (peer-memory loads), cast, optionally argmax'ed, copied into host ``out`` / ``labels``."""
    handles = (ctypes.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
    accs = (ctypes.c_void_p * len(ctxs))(*[int(p) for p in acc_ptrs])
    _check(load().fs_finalize_multi(handles, len(ctxs), int(acc_kind), accs, int(n), int(e),
                                    _p(out), float(gamma), int(mode), _p(labels)))


def bin_splats(mean2d, depth, radius, index, width: int, height: int, device: int = None):
    """fs_bin_splats: CSR tile lists (positions into the splat list)."""
    ctx = context(device)
    mean2d = np.ascontiguousarray(mean2d, dtype=np.float64).reshape(-1, 2)
    k = mean2d.shape[0]
    depth = np.ascontiguousarray(depth, dtype=np.float64).reshape(k)
    radius = np.ascontiguousarray(radius, dtype=np.int64).reshape(k)
    index = np.ascontiguousarray(index, dtype=np.int64).reshape(k)
    ntiles = ((width + 15) // 16) * ((height + 15) // 16)
    offs = np.zeros(ntiles + 1, np.int64)
    count = ctypes.c_int64(0)
    L = load()
    with ctx.lock:
        _check(L.fs_bin_splats(ctx.handle, k, _p(mean2d), _p(depth), _p(radius), _p(index),
                               int(width), int(height), _p(offs), None, 0, ctypes.byref(count)))
        items = np.zeros(max(count.value, 1), np.int64)
        _check(L.fs_bin_splats(ctx.handle, k, _p(mean2d), _p(depth), _p(radius), _p(index),
                               int(width), int(height), _p(offs), _p(items), items.size,
                               ctypes.byref(count)))
    return offs, items[:count.value]


def render_splats(width: int, height: int, mean2d, conic, depth, opacity, offsets, items,
                  alpha_floor: float, t_floor: float, channel=None, device: int = None):
    """fs_render_splats: composite a caller's binning -> (value | None, alpha, depth)."""
    ctx = context(device)
    mean2d = np.ascontiguousarray(mean2d, dtype=np.float64).reshape(-1, 2)
    k = mean2d.shape[0]
    conic = np.ascontiguousarray(conic, dtype=np.float64).reshape(k, 3)
    depth = np.ascontiguousarray(depth, dtype=np.float64).reshape(k)
    opacity = np.ascontiguousarray(opacity, dtype=np.float64).reshape(k)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    items = np.ascontiguousarray(items, dtype=np.int64)
    alpha = np.zeros((height, width))
    dep = np.zeros((height, width))
    channels, value, ch = 0, None, None
    if channel is not None:
        ch = np.ascontiguousarray(channel, dtype=np.float64)
        channels = 1 if ch.ndim == 1 else ch.shape[1]
        value = np.zeros((height, width) if channels == 1 else (height, width, channels))
    with ctx.lock:
        _check(load().fs_render_splats(ctx.handle, int(width), int(height), k, _p(mean2d),
                                       _p(conic), _p(depth), _p(opacity), _p(offsets), _p(items),
                                       float(alpha_floor), float(t_floor), _p(ch), channels,
                                       _p(value), _p(alpha), _p(dep)))
    return value, alpha, dep


def decode_mask_png(data: bytes):
    """fs_decode_mask_png: uint16 H x W labels, or None for PNG flavours the
    native decoder does not handle (caller falls back to Pillow)."""
    L = load()
    w, h = ctypes.c_int(0), ctypes.c_int(0)
    buf = ctypes.c_char_p(data)
    rc = L.fs_decode_mask_png(buf, len(data), None, 0, ctypes.byref(w), ctypes.byref(h))
    if rc != FS_OK:
        return None
    out = np.empty((h.value, w.value), np.uint16)
    rc = L.fs_decode_mask_png(buf, len(data), _p(out), out.size, ctypes.byref(w), ctypes.byref(h))
    return out if rc == FS_OK else None


def project(means, quats, scales, view, device: int = None):
    """Projection of an arbitrary (sub)set of Gaussians, for the stage API."""
    ctx = context(device)
    with ctx.lock:
        n = np.asarray(means).reshape(-1, 3).shape[0]
        ctx.set_arrays(means, quats, scales, np.ones(n))
        return ctx.project(view)
