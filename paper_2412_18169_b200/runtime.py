"""ctypes binding of the C-ABI data plane (include/kunserve_b200.h -> _kb.so).

This is the only path to the device: there is no host fallback.  Importing
this module without a built `_kb.so` raises immediately, and every call
checks the C status and re-raises the library's message.

Objects:
  Runtime     one GPU (CUDA primary context, peer access); creates pools.
  DevicePool  one instance's HBM: VMM slab pool + paged KV pool + block
              tables (the device side of memory.build_instance).
Free functions wrap the copy / append / attention entry points; tensors are
torch CUDA tensors passed by data_ptr (borrowed for the duration of the
call; the caller keeps them alive until its stream is synchronized).
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

from .core import ModelShape, ModelSpec

_HERE = os.path.dirname(os.path.abspath(__file__))
# KB_LIB_PATH: load a variant build of the same ABI (kernel A/B runs in tools/)
LIB_PATH = os.environ.get("KB_LIB_PATH") or os.path.join(_HERE, "_kb.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with "
                      "`python -m paper_2412_18169_b200.build` (no CPU fallback exists)")
_lib = C.CDLL(LIB_PATH)

KB_OK, KB_REFUSED = 0, 1
KB_KV_V_OVERFLOW, KB_KV_V_UNDERFLOW, KB_KV_NO_PAGE = 1, 2, 4


class ModelDesc(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("n_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("block_tokens", C.c_int32),
                ("slab_bytes", C.c_int64), ("page_bytes", C.c_int64)]


class PoolInfo(C.Structure):
    _fields_ = [("extent_pages", C.c_int64), ("live_pages", C.c_int64),
                ("slack_pages", C.c_int64), ("max_pages", C.c_int64),
                ("layers_mapped", C.c_int32), ("device", C.c_int32),
                ("weight_base", C.c_uint64), ("kv_base", C.c_uint64),
                ("block_table", C.c_uint64), ("npages", C.c_uint64),
                ("max_slots", C.c_int32), ("max_pages_per_seq", C.c_int32)]


class ExportDesc(C.Structure):
    _fields_ = [("model", ModelDesc), ("hbm_bytes", C.c_int64), ("head_bytes", C.c_int64),
                ("slack_pages", C.c_int64), ("device", C.c_int32), ("max_slots", C.c_int32),
                ("max_pages_per_seq", C.c_int32), ("n_handles", C.c_int32),
                ("bt_ipc", C.c_uint8 * 64), ("np_ipc", C.c_uint8 * 64)]


class Grow(C.Structure):
    _fields_ = [("slot", C.c_int32), ("layer_lo", C.c_int32), ("layer_hi", C.c_int32),
                ("add_pages", C.c_int32)]


class Move(C.Structure):
    _fields_ = [("src_slot", C.c_int32), ("dst_slot", C.c_int32), ("layer_lo", C.c_int32),
                ("layer_hi", C.c_int32), ("npages", C.c_int32), ("flat_lo", C.c_int32),
                ("flat_hi", C.c_int32), ("_pad", C.c_int32)]


_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_U = C.c_uint64
_S = C.c_size_t  # uintptr_t stream

_sigs = {
    "kb_last_error": (C.c_char_p, []),
    "kb_version": (C.c_int, []),
    "kb_init": (C.c_int, [C.c_int32, _I32P, C.c_int32]),
    "kb_vmm_granularity": (C.c_int, [C.c_int32, _I64P]),
    "kb_pool_create": (C.c_int, [C.c_int32, C.POINTER(ModelDesc), C.c_int64, C.c_int32,
                                 C.c_int32, C.c_int32, _I32P, C.c_int32, C.POINTER(_P)]),
    "kb_pool_destroy": (C.c_int, [_P]),
    "kb_pool_query": (C.c_int, [_P, C.POINTER(PoolInfo)]),
    "kb_pool_export": (C.c_int, [_P, C.POINTER(ExportDesc), _I32P, C.c_int32]),
    "kb_pool_import": (C.c_int, [C.c_int32, C.POINTER(ExportDesc), _I32P, C.c_int32,
                                 C.POINTER(_P)]),
    "kb_pool_view_refresh": (C.c_int, [_P, C.POINTER(C.c_uint8), C.c_int32]),
    "kb_pool_is_view": (C.c_int, [_P]),
    "kb_pool_stream_begin": (C.c_int, [_P, _S]),
    "kb_pool_stream_end": (C.c_int, [_P, _S]),
    "kb_pool_kv_status": (C.c_int, [_P, C.POINTER(C.c_uint32), C.c_int32]),
    "kb_drop_layers": (C.c_int, [_P, C.c_int32, C.c_int32, _I64P]),
    "kb_restore_begin": (C.c_int, [_P, C.c_int32, C.c_int32, _S, _I64P, _I64P]),
    "kb_restore_complete": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "kb_pool_last_moved": (C.c_int, [_P, _I64P]),
    "kb_weight_ptr": (C.c_uint64, [_P, C.c_int32]),
    "kb_pages_grow": (C.c_int, [_P, C.POINTER(Grow), C.c_int32, _S]),
    "kb_pages_release": (C.c_int, [_P, _I32P, C.c_int32, C.c_int32, C.c_int32, _S]),
    "kb_read_block_table": (C.c_int, [_P, C.c_int32, C.c_int32, _I32P, C.c_int32, _I32P]),
    "kb_read_bitmap": (C.c_int, [_P, C.POINTER(C.c_uint32), C.c_int64]),
    "kb_read_owner": (C.c_int, [_P, _I32P, C.c_int64]),
    "kb_pages_per_layer_count": (C.c_int64, [_P, C.c_int32, C.c_int32]),
    "kb_copy_pages": (C.c_int, [_P, _P, C.POINTER(Move), C.c_int32, _S]),
    "kb_copy_slabs": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int64, C.c_int64, _S]),
    "kb_copy_slabs_from_host": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int64,
                                          C.c_int64, _S]),
    "kb_copy_bytes": (C.c_int, [_U, _U, C.c_int64, _S]),
    "kb_copy_pages_host": (C.c_int, [_P, C.POINTER(Move), _P, C.c_int32, _S]),
    "kb_hash_segments": (C.c_int, [_U, C.c_int64, _U, C.c_int32, _U, _S]),
    "kb_add_rmsnorm": (C.c_int, [_U, _U, _U, _U, C.c_int32, C.c_int32, C.c_float, _S]),
    "kb_silu_mul": (C.c_int, [_U, _U, C.c_int32, C.c_int32, _S]),
    "kb_device_alloc": (C.c_int, [C.c_int32, C.c_int64, C.POINTER(C.c_uint64)]),
    "kb_device_free": (C.c_int, [_U]),
    "kb_ipc_mem_export": (C.c_int, [_U, C.POINTER(C.c_uint8)]),
    "kb_ipc_mem_import": (C.c_int, [C.c_int32, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)]),
    "kb_ipc_mem_close": (C.c_int, [_U]),
    "kb_kv_append": (C.c_int, [_P, C.c_int32, _U, _U, _U, _U, C.c_int32, C.c_int64, _S]),
    "kb_decode_workspace_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "kb_paged_decode": (C.c_int, [_P, C.c_int32, C.c_int32, _U, _U, _U, C.c_int32, C.c_int32,
                                  C.c_float, _U, _U, C.c_int64, C.c_int32, C.c_int32, _S]),
    "kb_prefill_workspace_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "kb_paged_prefill": (C.c_int, [_P, C.c_int32, C.c_int32, _U, _U, _U, _U, _U, C.c_int32,
                                   C.c_int32, C.c_float, _U, _U, C.c_int32, _S]),
}
for _name, (_res, _args) in _sigs.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_sigs)


class DeviceError(RuntimeError):
    pass


class Refused(ValueError):
    """Expected refusal (KB_REFUSED): out of pages / restore cannot vacate.
    A ValueError like the reference's "restore blocked" (memory.py:193-196)."""


# Kernel launches issued by this process through the library (the bench's
# `gpu_launches` claim): incremented by the wrappers that launch.
LAUNCHES = [0]
# Host -> device descriptor bytes this process passed through the C-ABI for
# device work (block-table grow requests, release slot lists, page-move
# lists): the per-step host input of the drop / exchange / restore path,
# which the library ships in kernel parameter space.  bench.py's e2e leg
# reports it per step.
H2D_BYTES = [0]


def _check(rc: int, launches: int = 0) -> None:
    if rc == KB_OK:
        LAUNCHES[0] += launches
        return
    msg = _lib.kb_last_error().decode()
    if rc == KB_REFUSED:
        raise Refused(msg)
    raise DeviceError(f"kb error {rc}: {msg}")


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _i32arr(vals: Sequence[int]):
    arr = (C.c_int32 * max(1, len(vals)))(*vals)
    return arr


class _CudaBuf:
    """Raw device range exposed to torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


def device_bytes(ptr: int, nbytes: int):
    """uint8 torch view of a device range owned by the library."""
    import torch
    return torch.as_tensor(_CudaBuf(ptr, nbytes), device="cuda")


class Runtime:
    """One GPU.  `peers` lists other devices every mapping must be accessible
    from (NVSwitch: all of them)."""

    def __init__(self, device: int = 0, peers: Sequence[int] = (), max_slots: int = 1024,
                 max_pages_per_seq: int = 1024, slack_pages: Optional[int] = None):
        self.device = device
        self.peers = list(peers)
        self.max_slots = max_slots
        self.max_pages_per_seq = max_pages_per_seq
        self.slack_pages = slack_pages
        _check(_lib.kb_init(device, _i32arr(self.peers), len(self.peers)))

    def granularity(self) -> int:
        g = C.c_int64()
        _check(_lib.kb_vmm_granularity(self.device, C.byref(g)))
        return g.value

    def create_pool(self, iid: int, model: ModelSpec, hbm_bytes: int,
                    shape: Optional[ModelShape] = None) -> "DevicePool":
        if shape is None:
            raise ValueError("device-backed instances need a ModelShape (page geometry)")
        return DevicePool(self, iid, model, hbm_bytes, shape)


class DevicePool:
    def __init__(self, rt: Runtime, iid: int, model: ModelSpec, hbm_bytes: int,
                 shape: ModelShape):
        if model.num_layers != shape.num_layers or \
                model.kv_bytes_per_token != shape.kv_bytes_per_token:
            raise ValueError("ModelSpec and ModelShape disagree")
        self.rt = rt
        self.iid = iid
        self.model = model
        self.shape = shape
        self.desc = ModelDesc(model.num_layers, shape.n_kv_heads, shape.head_dim,
                              shape.block_tokens, model.bytes_per_layer, shape.page_bytes)
        self.slack_pages = rt.slack_pages if rt.slack_pages is not None \
            else model.num_layers * 64
        h = _P()
        _check(_lib.kb_pool_create(rt.device, C.byref(self.desc), hbm_bytes, rt.max_slots,
                                   rt.max_pages_per_seq, self.slack_pages,
                                   _i32arr(rt.peers), len(rt.peers), C.byref(h)))
        self.h = h
        self.last_remap_ns = 0

    # -- lifecycle
    def close(self) -> None:
        if self.h:
            _lib.kb_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> PoolInfo:
        out = PoolInfo()
        _check(_lib.kb_pool_query(self.h, C.byref(out)))
        return out

    @property
    def page_bytes(self) -> int:
        return self.shape.page_bytes

    @property
    def slab_pages(self) -> int:
        return self.model.bytes_per_layer // self.shape.page_bytes

    # -- cross-process export (one process per GPU; see PeerPool)
    def export(self) -> tuple[bytes, list[int]]:
        """(descriptor bytes, file descriptors of the head segment and every
        layer slab).  The caller sends the fds to the peer (SCM_RIGHTS) and
        closes its copies."""
        desc = ExportDesc()
        n = 1 + self.model.num_layers
        fds = (C.c_int32 * n)()
        _check(_lib.kb_pool_export(self.h, C.byref(desc), fds, n))
        return bytes(desc), list(fds)

    # -- N1 / N3: drop and restore (memory.drop_layers / restore_layers)
    def drop_layers(self, lo: int, hi: int) -> int:
        ns = C.c_int64()
        _check(_lib.kb_drop_layers(self.h, lo, hi, C.byref(ns)))
        self.last_remap_ns = ns.value
        return ns.value

    def restore_begin(self, lo: int, hi: int, stream=None) -> None:
        """Asynchronous: the compaction is ordered on the device; its size
        is `last_moved_pages` (which waits for it)."""
        ns = C.c_int64()
        _check(_lib.kb_restore_begin(self.h, lo, hi, _stream(stream), None, C.byref(ns)))
        LAUNCHES[0] += 4  # plan + copy + fixup + mark
        self.last_remap_ns = ns.value

    @property
    def last_moved_pages(self) -> int:
        moved = C.c_int64()
        _check(_lib.kb_pool_last_moved(self.h, C.byref(moved)))
        return moved.value

    def restore_complete(self, lo: int, hi: int) -> None:
        _check(_lib.kb_restore_complete(self.h, lo, hi))

    # -- work the pool cannot see (CUDA graph replays)
    def stream_begin(self, stream=None) -> None:
        _check(_lib.kb_pool_stream_begin(self.h, _stream(stream)))

    def stream_end(self, stream=None) -> None:
        _check(_lib.kb_pool_stream_end(self.h, _stream(stream)))

    # -- fp16 V-cache range guard (kb_pool_kv_status)
    def kv_status(self, clear: bool = False) -> int:
        """KB_KV_V_* flags of every append that has completed (synchronize
        the appending stream first for an exact answer)."""
        f = C.c_uint32()
        _check(_lib.kb_pool_kv_status(self.h, C.byref(f), 1 if clear else 0))
        return f.value

    def check_kv_range(self, synchronize: bool = True) -> None:
        """Raise ValueError if any appended V value fell outside the fp16
        cache's exact range (|v| in [2^-14, 65504] or 0), or an append hit a
        position with no page; clears the flags."""
        if synchronize:
            import torch
            torch.cuda.synchronize(self.rt.device)
        f = self.kv_status(clear=True)
        if f & KB_KV_NO_PAGE:
            raise ValueError(f"pool {self.iid}: kv_append to a slot / position without a "
                             "page (outside the block table or never grown); the row was skipped")
        if f:
            what = []
            if f & KB_KV_V_OVERFLOW:
                what.append("|v| >= 65536 (inf in fp16)")
            if f & KB_KV_V_UNDERFLOW:
                what.append("0 < |v| < 2^-14 (fp16 subnormal)")
            raise ValueError(f"pool {self.iid}: V value out of the fp16 KV-cache range: "
                             + ", ".join(what))

    def weight_ptr(self, layer: int) -> int:
        return int(_lib.kb_weight_ptr(self.h, layer))

    def weight_bytes(self, layer: int):
        ptr = self.weight_ptr(layer)
        if not ptr:
            raise DeviceError(f"layer {layer} is not mapped on pool {self.iid}")
        return device_bytes(ptr, self.model.bytes_per_layer)

    def kv_bytes(self):
        """uint8 view of the whole KV VA (pages [0, max_pages)): head pages and
        every layer slab's alias, dropped or not."""
        inf = self.info()
        return device_bytes(inf.kv_base, inf.max_pages * self.page_bytes)

    # -- N2: block tables
    def grow(self, reqs: Sequence[tuple[int, int, int, int]], stream=None) -> bool:
        """reqs: (slot, layer_lo, layer_hi, add_pages).  False = out of pages."""
        if not reqs:
            return True
        arr = (Grow * len(reqs))(*[Grow(*r) for r in reqs])
        H2D_BYTES[0] += C.sizeof(arr)
        try:
            _check(_lib.kb_pages_grow(self.h, arr, len(reqs), _stream(stream)),
                   launches=-(-len(reqs) // 256))
        except Refused:
            return False
        return True

    def release(self, slots: Sequence[int], lo: int, hi: int, stream=None) -> None:
        if not slots:
            return
        H2D_BYTES[0] += 4 * len(slots)
        _check(_lib.kb_pages_release(self.h, _i32arr(slots), len(slots), lo, hi,
                                     _stream(stream)), launches=-(-len(slots) // 1024))

    def npages(self, slot: int, layer: int) -> int:
        return int(_lib.kb_pages_per_layer_count(self.h, slot, layer))

    def block_table(self, slot: int, layer: int) -> list[int]:
        cap = self.rt.max_pages_per_seq
        buf = (C.c_int32 * cap)()
        n = C.c_int32()
        _check(_lib.kb_read_block_table(self.h, slot, layer, buf, cap, C.byref(n)))
        return list(buf[:n.value])

    def bitmap(self, n_pages: Optional[int] = None):
        import numpy as np
        n_pages = n_pages or self.info().max_pages
        words = (n_pages + 31) // 32
        buf = (C.c_uint32 * words)()
        _check(_lib.kb_read_bitmap(self.h, buf, words))
        bits = np.unpackbits(np.frombuffer(bytes(buf), dtype=np.uint8), bitorder="little")
        return bits[:n_pages].astype(bool)

    def owners(self, n_pages: Optional[int] = None):
        import numpy as np
        n_pages = n_pages or self.info().max_pages
        buf = (C.c_int32 * n_pages)()
        _check(_lib.kb_read_owner(self.h, buf, n_pages))
        return np.frombuffer(bytes(buf), dtype=np.int32).copy()


class PeerPool:
    """Read-only view, in this process, of a pool another process owns
    (possibly on another GPU): its slabs and pages mapped into this process's
    VA from the owner's exported VMM handles, its block table and page
    counts opened through CUDA IPC.  Usable as the `src` of copy_pages /
    copy_slabs -- the pull travels over NVLink when the owner's GPU is a
    different one.  Every mutating call is the owner's job and the library
    refuses it on a view."""

    def __init__(self, rt: Runtime, iid: int, model: ModelSpec, shape: ModelShape,
                 desc: bytes, fds: Sequence[int]):
        d = ExportDesc.from_buffer_copy(desc)
        if d.model.num_layers != model.num_layers or d.model.page_bytes != shape.page_bytes:
            raise ValueError("exported pool disagrees with the model shape")
        self.rt = rt
        self.iid = iid
        self.model = model
        self.shape = shape
        self.owner_device = d.device
        h = _P()
        _check(_lib.kb_pool_import(rt.device, C.byref(d), _i32arr(list(fds)), len(fds),
                                   C.byref(h)))
        self.h = h
        self.last_remap_ns = 0

    def close(self) -> None:
        if self.h:
            _lib.kb_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def refresh(self, layers_held: Sequence[int]) -> None:
        """Re-read the owner's page counts (synchronizing) and take its layer
        states from the caller's mirror of the owner's segment table."""
        L = self.model.num_layers
        held = set(layers_held)
        arr = (C.c_uint8 * L)(*[1 if l in held else 0 for l in range(L)])
        _check(_lib.kb_pool_view_refresh(self.h, arr, L))

    def info(self) -> PoolInfo:
        out = PoolInfo()
        _check(_lib.kb_pool_query(self.h, C.byref(out)))
        return out

    @property
    def page_bytes(self) -> int:
        return self.shape.page_bytes

    def npages(self, slot: int, layer: int) -> int:
        return int(_lib.kb_pages_per_layer_count(self.h, slot, layer))

    def weight_bytes(self, layer: int):
        ptr = int(_lib.kb_weight_ptr(self.h, layer))
        if not ptr:
            raise DeviceError(f"layer {layer} is not held by pool {self.iid}'s owner")
        return device_bytes(ptr, self.model.bytes_per_layer)

    def kv_bytes(self):
        inf = self.info()
        return device_bytes(inf.kv_base, inf.max_pages * self.page_bytes)


def is_view(pool) -> bool:
    return bool(_lib.kb_pool_is_view(pool.h))


# -- N4 / N5 / N7 copies ------------------------------------------------------

def copy_pages(dst: DevicePool, src: DevicePool,
               moves: Sequence[tuple[int, int, int, int, int, int, int]], stream=None) -> None:
    """moves: (src_slot, dst_slot, layer_lo, layer_hi, npages, flat_lo, flat_hi)."""
    if not moves:
        return
    arr = (Move * len(moves))(*[Move(*m, 0) for m in moves])
    H2D_BYTES[0] += C.sizeof(arr)
    _check(_lib.kb_copy_pages(dst.h, src.h, arr, len(moves), _stream(stream)),
           launches=-(-len(moves) // 256))


def copy_slabs(dst: DevicePool, src: DevicePool, lo: int, hi: int, byte_lo: int,
               byte_hi: int, stream=None) -> None:
    H2D_BYTES[0] += 24  # (lo, hi, byte_lo, byte_hi)
    _check(_lib.kb_copy_slabs(dst.h, src.h, lo, hi, byte_lo, byte_hi, _stream(stream)),
           launches=1)


def copy_slabs_from_host(dst: DevicePool, host_ptr: int, lo: int, hi: int, byte_lo: int,
                         byte_hi: int, stream=None) -> None:
    _check(_lib.kb_copy_slabs_from_host(dst.h, C.c_void_p(host_ptr), lo, hi, byte_lo, byte_hi,
                                        _stream(stream)))


def copy_pages_host(pool: DevicePool, slot: int, layer_lo: int, layer_hi: int, npages: int,
                    host, to_host: bool, flat_lo: int = 0, flat_hi: Optional[int] = None,
                    stream=None) -> None:
    """Pages of `slot` (layers [lo, hi), npages each, flattened layer-major)
    to / from the pinned host tensor `host` (swap baseline)."""
    if flat_hi is None:
        flat_hi = (layer_hi - layer_lo) * npages
    if host.numel() * host.element_size() < flat_hi * pool.page_bytes:
        raise ValueError("host buffer too small for the pages")
    mv = Move(slot, slot, layer_lo, layer_hi, npages, flat_lo, flat_hi, 0)
    _check(_lib.kb_copy_pages_host(pool.h, C.byref(mv), C.c_void_p(host.data_ptr()),
                                   1 if to_host else 0, _stream(stream)), launches=1)


class IpcBuffer:
    """A device buffer shared across processes (CUDA IPC): the owner
    allocates and exports it, a peer imports it into its own VA."""

    def __init__(self, ptr: int, nbytes: int, owned: bool):
        self.ptr, self.nbytes, self.owned = ptr, nbytes, owned

    @classmethod
    def allocate(cls, device: int, nbytes: int) -> "IpcBuffer":
        p = C.c_uint64()
        _check(_lib.kb_device_alloc(device, nbytes, C.byref(p)))
        return cls(p.value, nbytes, True)

    def export(self) -> bytes:
        h = (C.c_uint8 * 64)()
        _check(_lib.kb_ipc_mem_export(self.ptr, h))
        return bytes(h)

    @classmethod
    def open(cls, device: int, handle: bytes, nbytes: int) -> "IpcBuffer":
        h = (C.c_uint8 * 64)(*handle)
        p = C.c_uint64()
        _check(_lib.kb_ipc_mem_import(device, h, C.byref(p)))
        return cls(p.value, nbytes, False)

    def tensor(self):
        return device_bytes(self.ptr, self.nbytes)

    def close(self) -> None:
        if self.ptr:
            _check(_lib.kb_device_free(self.ptr) if self.owned else _lib.kb_ipc_mem_close(self.ptr))
            self.ptr = 0


def hash_segments(base_ptr: int, seg_bytes: int, nseg: int, index=None, stream=None):
    """Position-sensitive 64-bit hash of nseg device segments (int64 torch
    tensor on the segments' device; see kb_hash_segments).  `index`: device
    int64 tensor of segment numbers (segment i at base + index[i] * seg_bytes),
    or None for 0..nseg-1."""
    import torch
    dev = index.device if index is not None else torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(max(nseg, 0), dtype=torch.int64, device=dev)
    if nseg <= 0:
        return out
    if index is not None and (index.dtype != torch.int64 or not index.is_contiguous()):
        index = index.to(torch.int64).contiguous()
    _check(_lib.kb_hash_segments(base_ptr, seg_bytes, 0 if index is None else index.data_ptr(), nseg,
                                 out.data_ptr(), _stream(stream)), launches=2)
    return out


def hash_tensor(t, seg_bytes: Optional[int] = None, stream=None):
    """hash_segments over a contiguous device tensor cut into seg_bytes
    segments (default: one segment)."""
    nbytes = t.numel() * t.element_size()
    seg = seg_bytes or nbytes
    if nbytes % seg:
        raise ValueError("tensor size is not a multiple of the segment size")
    import torch
    with torch.cuda.device(t.device):
        return hash_segments(t.data_ptr(), seg, nbytes // seg, stream=stream)


def add_rmsnorm(x, res, w, out, eps: float = 1e-5, stream=None) -> None:
    """x (+)= res in place (res None: no add); out = rmsnorm(x) * w (bf16 rows)."""
    _check(_lib.kb_add_rmsnorm(x.data_ptr(), 0 if res is None else res.data_ptr(), w.data_ptr(),
                               out.data_ptr(), x.shape[0], x.shape[1], eps, _stream(stream)),
           launches=1)


def silu_mul(gu, out, stream=None) -> None:
    """out = silu(gu[:, :F]) * gu[:, F:] (bf16)."""
    _check(_lib.kb_silu_mul(gu.data_ptr(), out.data_ptr(), gu.shape[0], out.shape[1],
                            _stream(stream)), launches=1)


def copy_bytes(dst_ptr: int, src_ptr: int, nbytes: int, stream=None) -> None:
    _check(_lib.kb_copy_bytes(dst_ptr, src_ptr, nbytes, _stream(stream)), launches=1)


# -- N8 attention -------------------------------------------------------------

def kv_append(pool: DevicePool, layer: int, k, v, slots, pos, stream=None) -> None:
    """k, v: [ntok, n_kv_heads, 128] bf16, rows contiguous or strided views of
    a wider row (e.g. the K / V blocks of a fused QKV output); slots/pos:
    int32 [ntok] (device)."""
    if k.stride()[1:] != (128, 1) or v.stride()[1:] != (128, 1) or k.stride(0) != v.stride(0):
        k, v = k.contiguous(), v.contiguous()
    _check(_lib.kb_kv_append(pool.h, layer, k.data_ptr(), v.data_ptr(), slots.data_ptr(),
                             pos.data_ptr(), k.shape[0], k.stride(0), _stream(stream)),
           launches=1)


def decode_workspace_bytes(nseq: int, n_q_heads: int, max_splits: int) -> int:
    return int(_lib.kb_decode_workspace_bytes(nseq, n_q_heads, max_splits))


DECODE_REUSE_PLAN = 1
DECODE_COMBINE = 2
DECODE_FUSE = 4


def paged_decode(pool: DevicePool, layer: int, q, slots, ctx_lens, max_ctx: int, out,
                 workspace, scale: float, max_splits: int = 16, reuse_plan: bool = False,
                 stream=None, combine: Optional[bool] = None) -> None:
    """q/out: [nseq, n_q_heads, 128] bf16; slots/ctx_lens int32 [nseq] (device).
    reuse_plan: the workspace already holds the plan for these ctx_lens and
    slots (a previous layer of the same decode step).  combine: None lets
    the library choose where the KV splits merge (inside the attention
    kernel for large batches, else a combine launch); True / False force the
    combine launch / the in-kernel merge."""
    flags = DECODE_REUSE_PLAN if reuse_plan else 0
    if combine is None:
        fused = q.shape[0] * pool.shape.n_kv_heads >= 4 * _sm_count(pool.rt.device)
    else:
        fused = not combine
        flags |= DECODE_COMBINE if combine else DECODE_FUSE
    _check(_lib.kb_paged_decode(pool.h, layer, q.shape[1], q.data_ptr(), slots.data_ptr(),
                                ctx_lens.data_ptr(), q.shape[0], max_ctx, scale,
                                out.data_ptr(), workspace.data_ptr(),
                                workspace.numel() * workspace.element_size(), max_splits, flags,
                                _stream(stream)),
           launches=(1 if reuse_plan else 2) + (0 if fused else 1))


def prefill_splits(nseq: int, n_q_heads: int, max_q_len: int, max_kv_len: int,
                   n_sm: int = 148) -> int:
    """KV splits for one prefill launch (1..8), keeping >= 16 key tiles per
    split.  Score = wave fill of the grid (one 256-row CTA per SM) x the
    share of a split's time spent streaming: each CTA pays a ramp worth
    ~6.5 key tiles (Q load, pipeline fill, O epilogue, partial write, its
    share of the combine launch), an unsplit CTA ~2 (no partials, no
    combine).  Fitted to the r4 B200 per-chunk sweep of config 4
    (tools/pf_split_sweep.py: 1 split up to 4k keys, 2 to ~13k, 3 to ~17k,
    4 beyond)."""
    units = nseq * -(-max_q_len // 256) * n_q_heads
    tiles = -(-max_kv_len // 128)

    def score(s: int) -> float:
        waves = units * s / (n_sm * -(-(units * s) // n_sm))
        per = tiles / s
        return waves * per / (per + (2.0 if s == 1 else 6.5))
    best, best_score = 1, score(1)
    for s in range(2, 9):
        if tiles < 16 * s:
            break
        sc = score(s)
        if sc > best_score:
            best, best_score = s, sc
    return best


def prefill_workspace_bytes(nseq: int, n_q_heads: int, max_q_len: int, kv_splits: int) -> int:
    return int(_lib.kb_prefill_workspace_bytes(nseq, n_q_heads, max_q_len, kv_splits))


def paged_prefill(pool: DevicePool, layer: int, q, slots, q_off, q_len, prefix, max_q_len: int,
                  out, scale: float, max_kv_len: Optional[int] = None,
                  kv_splits: Optional[int] = None, workspace=None, stream=None) -> None:
    """q/out: [total_q, n_q_heads, 128] bf16; per-sequence int32 vectors (device).
    max_kv_len (host-known longest prefix + chunk) enables KV splits chosen
    by prefill_splits; the workspace is cached on the pool when not given."""
    nseq, hq = slots.shape[0], q.shape[1]
    if kv_splits is None:
        kv_splits = 1 if max_kv_len is None else prefill_splits(
            nseq, hq, max_q_len, max_kv_len, _sm_count(pool.rt.device))
    ws_ptr = 0
    if kv_splits > 1:
        need = prefill_workspace_bytes(nseq, hq, max_q_len, kv_splits)
        if workspace is None:
            import torch
            ws = getattr(pool, "_prefill_ws", None)
            if ws is None or ws.numel() < need:
                ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{pool.rt.device}")
                pool._prefill_ws = ws
            workspace = ws
        elif workspace.numel() < need:
            raise ValueError(f"prefill workspace holds {workspace.numel()} < {need} bytes")
        ws_ptr = workspace.data_ptr()
    _check(_lib.kb_paged_prefill(pool.h, layer, hq, q.data_ptr(), slots.data_ptr(),
                                 q_off.data_ptr(), q_len.data_ptr(), prefix.data_ptr(),
                                 nseq, max_q_len, scale, out.data_ptr(), ws_ptr, kv_splits,
                                 _stream(stream)), launches=2 if kv_splits > 1 else 1)


_SMS: dict = {}


def _sm_count(device: int) -> int:
    if device not in _SMS:
        import torch
        _SMS[device] = torch.cuda.get_device_properties(device).multi_processor_count
    return _SMS[device]
