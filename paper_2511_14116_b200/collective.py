"""The exchange step over peer memory (fs_ar_residual).

``parallel_forward`` sums the per-rank attention / FFN partials in ascending
rank order and adds them to the residual stream (refexec.py:283-307).  On
B200s in one NVSwitch domain that exchange is ONE kernel per sub-layer: each
rank's projection GEMM writes its partial straight into a symmetric buffer
that every peer has mapped (CUDA IPC over NVLink), and ``fs_ar_residual``
signals the peers, waits for them, and does ``x += bf16(sum_r partial_r)``
reading the partials in rank order -- the reference's exact ordered sum,
bit-identical on every rank, with no NCCL launch and no separate residual
add.  Two buffers alternate between consecutive exchanges (the kernel's
flag protocol needs no second barrier then).  Large vectors on more than two
ranks use the kernel's two-shot form (each rank sums its 1/N slice, then
gathers the rounded slices), which reads 2(N-1)/N instead of N-1 vectors
over NVLink per rank and gives the same bits.
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _native as N
from .core import SimulationError, ValidationError


class _DeviceArray:
    """``__cuda_array_interface__`` view of raw device memory (uint16)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<u2", "data": (ptr, False),
                                         "version": 3, "strides": None}


class FusedExchange:
    """Two symmetric exchange buffers of this rank and their peer mappings.

    ``group``: the torch.distributed group of the alive ranks (any backend;
    used once to swap IPC handles) or a :class:`cluster.StoreControl` (the
    store-based control plane that survives a dead rank); ``max_elems``:
    largest partial (bf16 elements, e.g. batch x hidden).  All ranks must
    construct it together.
    """

    def __init__(self, group, max_elems: int, device=None, check: bool = True):
        self.device = torch.device(device if device is not None else "cuda")
        dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
        ctl = group if hasattr(group, "all_gather_object") else None
        self.rank = ctl.index if ctl else dist.get_rank(group)
        self.world = ctl.world if ctl else dist.get_world_size(group)
        if self.world > N.FS_AR_MAX_WORLD:
            raise ValidationError(f"fused exchange supports up to {N.FS_AR_MAX_WORLD} ranks")
        self.max_elems = int(max_elems) + (-int(max_elems)) % 8
        self.mode = 0  # fs_ar_residual_mode: automatic one-shot / two-shot
        self.nbytes = int(N.lib.fs_ar_buffer_bytes(self.max_elems))
        self.data_bytes = self.nbytes - 256
        self._own, self._opened = [], []
        self._ids = list(ctl.alive) if ctl else None  # global id per rank index
        handles = []
        for _ in range(2):
            p = C.c_void_p()
            N.check(N.lib.fs_ar_alloc(dev, self.nbytes, C.byref(p)), "fs_ar_alloc")
            self._own.append(p.value)
            h = (C.c_uint8 * 64)()
            N.check(N.lib.fs_ar_ipc_handle(C.c_void_p(p.value), h), "fs_ar_ipc_handle")
            handles.append(bytes(h))
        if ctl:
            every = ctl.all_gather_object(handles)
        else:
            every = [None] * self.world
            dist.all_gather_object(every, handles, group=group)
        self.peers = []
        for i in range(2):
            arr = (C.c_void_p * self.world)()
            for r in range(self.world):
                if r == self.rank:
                    arr[r] = self._own[i]
                    continue
                q = C.c_void_p()
                h = (C.c_uint8 * 64).from_buffer_copy(every[r][i])
                N.check(N.lib.fs_ar_ipc_open(h, C.byref(q)), "fs_ar_ipc_open")
                self._opened.append(q.value)
                arr[r] = q.value
            self.peers.append(arr)
        self._views = [torch.as_tensor(_DeviceArray(p, self.max_elems), device=self.device)
                       .view(torch.bfloat16) for p in self._own]
        if ctl:
            ctl.barrier()
        else:
            dist.barrier(group=group)
        if check:
            self._self_check()

    def shrink(self, ctl) -> None:
        """Re-form the exchange over the survivors ``ctl.alive`` (a
        :class:`cluster.StoreControl` of the next generation) WITHOUT new
        buffers: the dead ranks' mappings are closed, the survivors' buffers
        keep their IPC mappings and are re-indexed by the new rank order.
        Safe because every rank ran the same number of exchanges per buffer
        (lock-step steps): a flag slot's old value is at most the current
        use count, below the next use every waiter spins for."""
        if self._ids is None:
            raise ValidationError("shrink needs a FusedExchange built over a StoreControl")
        keep = set(ctl.alive)
        if not keep <= set(self._ids) or self._ids[self.rank] not in keep:
            raise ValidationError("shrink: the new world must be a subset containing this rank")
        torch.cuda.synchronize(self.device)
        for i in range(2):
            for r, g in enumerate(self._ids):
                if g not in keep and r != self.rank:
                    N.lib.fs_ar_ipc_close(C.c_void_p(self.peers[i][r]))
                    self._opened.remove(self.peers[i][r])
            arr = (C.c_void_p * len(ctl.alive))()
            for k, g in enumerate(ctl.alive):
                arr[k] = self.peers[i][self._ids.index(g)]
            self.peers[i] = arr
        self._ids = list(ctl.alive)
        self.rank, self.world = ctl.index, ctl.world

    def partial(self, i: int, shape) -> torch.Tensor:
        """This rank's partial buffer ``i`` (0/1) as a bf16 tensor of ``shape``
        -- the projection GEMM's ``out``."""
        n = 1
        for s in shape:
            n *= int(s)
        if n > self.max_elems:
            raise ValidationError("partial larger than the exchange buffer")
        return self._views[i][:n].view(*shape)

    def reduce_residual(self, i: int, x: torch.Tensor, mode: int = None) -> None:
        """``x += bf16(sum over ranks, in rank order, of partial_r)`` where
        partial_r is rank r's buffer ``i`` (its first ``x.numel()`` elements).
        ``mode``: 1 one-shot, 2 two-shot, 0 / None automatic (``self.mode``)."""
        if x.dtype != torch.bfloat16 or not x.is_contiguous() or x.numel() % 8:
            raise ValidationError("x must be contiguous bf16 with a multiple of 8 elements")
        st = torch.cuda.current_stream(self.device).cuda_stream
        N.check(N.lib.fs_ar_residual_mode(self.peers[i], self.rank, self.world, x.numel(),
                                          self.data_bytes, C.c_void_p(x.data_ptr()), 0,
                                          self.mode if mode is None else mode,
                                          C.c_void_p(st)), "fs_ar_residual")

    def _self_check(self) -> None:
        """Exchanges on each buffer, one-shot and two-shot, with rank-keyed
        data, checked against the ordered sum every rank can recompute."""
        n = min(self.max_elems, 4096)
        for i, mode in ((0, 1), (1, 1), (0, 2), (1, 2)):
            parts = [torch.randn(n, generator=torch.Generator().manual_seed(1000 * r + i))
                     .to(torch.bfloat16) for r in range(self.world)]
            self.partial(i, (n,)).copy_(parts[self.rank].to(self.device))
            x = torch.ones(n, dtype=torch.bfloat16, device=self.device)
            torch.cuda.current_stream(self.device).synchronize()
            self.reduce_residual(i, x, mode)
            total = torch.zeros(n)
            for p in parts:
                total += p.float()
            want = (torch.ones(n, dtype=torch.bfloat16).float() +
                    total.to(torch.bfloat16).float()).to(torch.bfloat16)
            if not torch.equal(x.cpu(), want):
                raise SimulationError(f"fused exchange self-check failed on rank {self.rank}")

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            N.lib.fs_ar_ipc_close(C.c_void_p(p))
        for p in self._own:
            N.lib.fs_ar_free(C.c_void_p(p))
        self._opened, self._own = [], []
