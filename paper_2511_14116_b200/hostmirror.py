"""Node-shared host state that outlives a failed rank, and the K7 copy
executor.

FailSafe recovers a lost GPU's state from host memory and from the
surviving peers (recovery.py:396-504).  In a one-process-per-GPU deployment
the host copies must not die with the process that wrote them, so they live
in named POSIX shared memory (``/dev/shm``) mapped by every rank of the node
and page-locked for the GPU (``fs_host_register``):

* :class:`KVMirror` -- one per rank: the K5 backup of the rank's KV pool
  (host slot == device page id, 8 KiB each) plus a small header with the
  rank's page map (item key (layer, head, request) -> block-table row) and
  the backed-up token watermark per item (``BackupState.backed``,
  recovery.py:143-191).  After the rank dies, the survivors open its mirror
  and restore the lost slices with K6 (``fs_pages_scatter``).
* :class:`WeightStore` -- one per node: the model's weights in a canonical
  per-piece layout (one piece per (layer, KV head) = the head's
  ``[Wq | Wk | Wv | Wo]``, one per (layer, FFN shard) = ``[Wg | Wu | Wd]``),
  the "host" the on-demand plan's ``pcie_host`` slices are loaded from
  (recovery.py:396-427).  Each rank publishes the pieces it owns at start-up.
* :class:`SegmentCopy` -- the K7 executor: builds ``fs_copy_seg`` lists
  (host -> device slices, peer -> device NVLink pulls, staging -> fused
  weight scatters) and runs each list as ONE ``fs_copy_segments`` launch.
"""

from __future__ import annotations

import ctypes as C
import mmap
import os

import numpy as np
import torch

from . import _native as N
from .core import SimulationError, ValidationError

SHM_DIR = "/dev/shm"
_ALIGN = 1 << 21


def _round_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


class SharedHostRegion:
    """``/dev/shm/<name>`` mapped into this process and page-locked for
    CUDA.  ``create=True`` makes a new region of ``nbytes`` (fails if it
    exists); otherwise an existing region is opened.  The region outlives
    the process until :meth:`unlink`."""

    def __init__(self, name: str, nbytes: int = 0, create: bool = False, register: bool = True):
        self.name = name
        self.path = os.path.join(SHM_DIR, name)
        flags = os.O_RDWR | ((os.O_CREAT | os.O_EXCL) if create else 0)
        fd = os.open(self.path, flags, 0o600)
        try:
            if create:
                # allocate every page now: page-locking a tmpfs range whose
                # pages are still holes fails (cudaErrorOperatingSystem) when
                # several processes race to fault them in
                os.posix_fallocate(fd, 0, nbytes)
            else:
                nbytes = os.fstat(fd).st_size
            self.nbytes = nbytes
            # an existing region is pre-faulted (MAP_POPULATE, ~20 GB/s): page-
            # locking then runs ~1.7x faster than faulting page by page
            flags = mmap.MAP_SHARED | (0 if create else getattr(mmap, "MAP_POPULATE", 0))
            self.mm = mmap.mmap(fd, nbytes, flags, mmap.PROT_READ | mmap.PROT_WRITE)
        finally:
            os.close(fd)
        self.host = torch.frombuffer(self.mm, dtype=torch.uint8)
        self.host_ptr = self.host.data_ptr()
        self.dev_ptr = None
        if register:
            p = C.c_void_p()
            N.check(N.lib.fs_host_register(C.c_void_p(self.host_ptr), nbytes, C.byref(p)),
                    "fs_host_register")
            self.dev_ptr = p.value

    def np(self, dtype, offset: int, count: int) -> np.ndarray:
        return np.frombuffer(self.mm, dtype=dtype, count=count, offset=offset)

    def close(self) -> None:
        if self.dev_ptr is not None:
            N.lib.fs_host_unregister(C.c_void_p(self.host_ptr))
            self.dev_ptr = None
        self.host = None
        try:
            self.mm.close()
        except BufferError:  # a numpy view still alive: leave it to the GC
            pass

    def unlink(self) -> None:
        try:
            os.unlink(self.path)
        except FileNotFoundError:
            pass

    @staticmethod
    def free_bytes() -> int:
        st = os.statvfs(SHM_DIR)
        return st.f_bavail * st.f_frsize


# ------------------------------------------------------------------ KV --
_MAGIC = 0x46534B56  # "FSKV"


class KVMirror:
    """Host mirror of one rank's KV pool + its page map (see module doc).

    Layout: int64 header[8] = (magic, n_items, pages_per_seq, n_pages,
    items_cap, generation, rank, 0); int32 keys[items_cap][3] (layer, head,
    request); int32 block_table[items_cap][pages_per_seq]; int32
    backed[items_cap]; then (2 MiB aligned) n_pages pages of 8 KiB.
    """

    def __init__(self, name: str, n_pages: int = 0, items_cap: int = 0, pages_per_seq: int = 0,
                 rank: int = -1, create: bool = False):
        if create:
            hdr = self._header_bytes(items_cap, pages_per_seq)
            nbytes = hdr + n_pages * N.PAGE_BYTES
            self.region = SharedHostRegion(name, nbytes, create=True)
            h = self.region.np(np.int64, 0, 8)
            h[:] = (_MAGIC, 0, pages_per_seq, n_pages, items_cap, 0, rank, 0)
        else:
            self.region = SharedHostRegion(name)
        h = self.region.np(np.int64, 0, 8)
        if int(h[0]) != _MAGIC:
            raise SimulationError(f"{name}: not a KV mirror")
        self.header = h
        self.pages_per_seq, self.n_pages, self.items_cap = int(h[2]), int(h[3]), int(h[4])
        self.rank = int(h[6])
        off = 64
        self.keys = self.region.np(np.int32, off, self.items_cap * 3).reshape(self.items_cap, 3)
        off += self.items_cap * 12
        self.bt = self.region.np(np.int32, off, self.items_cap * self.pages_per_seq).reshape(
            self.items_cap, self.pages_per_seq)
        off += self.items_cap * self.pages_per_seq * 4
        self.backed = self.region.np(np.int32, off, self.items_cap)
        self.page_base = self._header_bytes(self.items_cap, self.pages_per_seq)
        self.pages_dev_ptr = self.region.dev_ptr + self.page_base
        self.pages = self.region.host[self.page_base:].view(self.n_pages, N.PAGE_BYTES)

    @staticmethod
    def _header_bytes(items_cap: int, pages_per_seq: int) -> int:
        return _round_up(64 + items_cap * (3 + pages_per_seq + 1) * 4, _ALIGN)

    def publish_tables(self, keys: np.ndarray, block_table: np.ndarray) -> None:
        """Record the rank's page map (after every adoption)."""
        n = len(keys)
        if n > self.items_cap or block_table.shape[1] != self.pages_per_seq:
            raise ValidationError("page map larger than the mirror's header")
        self.keys[:n] = keys
        self.bt[:n] = block_table
        self.backed[:n] = 0
        self.header[1] = n
        self.header[5] += 1

    def set_backed(self, backed: np.ndarray) -> None:
        """Per-item tokens whose K/V are on the host (after the K5 copies
        that wrote them completed)."""
        self.backed[:len(backed)] = backed

    def tables(self):
        n = int(self.header[1])
        return self.keys[:n].copy(), self.bt[:n].copy(), self.backed[:n].copy()

    def close(self, unlink: bool = False) -> None:
        self.pages = None
        self.keys = self.bt = self.backed = self.header = None
        self.region.close()
        if unlink:
            self.region.unlink()


# ------------------------------------------------------------- weights --
class WeightLayout:
    """Canonical byte layout of the model's weights (bf16): per layer, the
    H head pieces then the S shard pieces.  Head piece = ``Wq [hid, qpk*hd]
    | Wk [hid, hd] | Wv [hid, hd] | Wo [qpk*hd, hid]`` =
    ``ModelSpec.attn_weight_bytes_per_head_layer`` (core.py); shard piece =
    ``Wg [hid, w] | Wu [hid, w] | Wd [w, hid]`` with w = ffn / shards, i.e.
    ``ffn_weight_bytes_per_layer / shards`` -- the byte units
    plan_weight_recovery splits (recovery.py:356-359)."""

    def __init__(self, model, num_shards: int):
        self.model = model
        hid, hd, qpk = model.hidden_dim, model.head_dim, model.q_heads_per_kv_head
        self.hid, self.hd, self.qpk = hid, hd, qpk
        self.S = num_shards
        self.w = model.ffn_intermediate_dim // num_shards
        self.H = model.num_kv_heads
        self.q_bytes = hid * qpk * hd * 2
        self.kv_bytes = hid * hd * 2
        self.head_bytes = 2 * self.q_bytes + 2 * self.kv_bytes
        self.shard_bytes = 3 * hid * self.w * 2
        self.layer_bytes = self.H * self.head_bytes + self.S * self.shard_bytes
        self.total = model.num_layers * self.layer_bytes

    def head_off(self, layer: int, head: int) -> int:
        return layer * self.layer_bytes + head * self.head_bytes

    def shard_off(self, layer: int, shard: int) -> int:
        return layer * self.layer_bytes + self.H * self.head_bytes + shard * self.shard_bytes


class WeightStore:
    """The node's host copy of the weights (:class:`WeightLayout`) in shared
    memory."""

    def __init__(self, name: str, layout: WeightLayout, create: bool = False,
                 register: bool = True):
        self.layout = layout
        self.region = SharedHostRegion(name, layout.total, create=create, register=register)
        if self.region.nbytes < layout.total:
            raise SimulationError(f"{name}: weight store smaller than the model")
        self.dev_ptr = self.region.dev_ptr

    def close(self, unlink: bool = False) -> None:
        self.region.close()
        if unlink:
            self.region.unlink()


class HostWeightStore:
    """Single-process weight store (pinned host memory, same layout and
    interface as :class:`WeightStore`) for the one-process emulation."""

    def __init__(self, layout: WeightLayout):
        self.layout = layout
        self.host = torch.empty(layout.total, dtype=torch.uint8, pin_memory=True)
        self.dev_ptr = self.host.data_ptr()  # pinned + UVA: device-addressable

    def close(self, unlink: bool = False) -> None:
        self.host = None


# --------------------------------------------------------------- copies --
_SEG = np.dtype([("src", np.uint64), ("dst", np.uint64), ("spitch", np.int64),
                 ("dpitch", np.int64), ("width", np.int64), ("height", np.int64)])
_CHUNK = 1 << 16  # a 1-row segment longer than this is split (warp-sized rows)


class SegmentCopy:
    """A list of 2-D copies executed as one ``fs_copy_segments`` launch."""

    def __init__(self):
        self.rows = []
        self.bytes = 0

    def add(self, dst: int, dpitch: int, src: int, spitch: int, width: int, height: int = 1):
        if width <= 0 or height <= 0:
            return
        self.bytes += width * height
        if height == 1 and width > _CHUNK:
            for a in range(0, width, _CHUNK):
                self.rows.append((src + a, dst + a, 0, 0, min(_CHUNK, width - a), 1))
            return
        self.rows.append((src, dst, spitch, dpitch, width, height))

    def add_bytes(self, dst: int, src: int, nbytes: int):
        self.add(dst, 0, src, 0, nbytes, 1)

    def run(self, device, stream=None, ctas: int = 0) -> None:
        if not self.rows:
            return
        segs = np.array(self.rows, dtype=_SEG)
        off = np.zeros(len(segs) + 1, dtype=np.int64)
        np.cumsum(segs["height"], out=off[1:])
        s = stream if stream is not None else torch.cuda.current_stream(device)
        d_segs = torch.from_numpy(segs.view(np.uint8).copy()).to(device, non_blocking=True)
        d_off = torch.from_numpy(off).to(device, non_blocking=True)
        N.check(N.lib.fs_copy_segments(C.c_void_p(d_segs.data_ptr()), C.c_void_p(d_off.data_ptr()),
                                       len(segs), ctas, C.c_void_p(s.cuda_stream)),
                "fs_copy_segments")
        d_segs.record_stream(s)
        d_off.record_stream(s)
