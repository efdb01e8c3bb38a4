"""Peer-mapped (and multicast) device memory for the fused allreduce + SGD.

The fused kernel (csrc/allreduce.cu, `wap_allreduce_sgd`) reads every rank's
gradient arena and writes every rank's variable arena directly over NVLink, so
each rank's arenas must be mapped into every other rank's address space. This
is plumbing on the CUDA driver's virtual-memory API (cuda-python bindings):

* each rank cuMemCreate's its physical memory (POSIX-fd shareable), maps it,
  and publishes (pid, fd) through the torch.distributed process group;
* the others pull the fd with pidfd_getfd(2), cuMemImportFromShareableHandle it,
  and cuMemMap it into their own VA space (NVLink P2P on an HGX node);
* NVLS mode also builds one multicast object per arena (cuMulticastCreate on
  rank 0, imported by the others, every device added, every rank's physical
  memory bound, and the multicast handle mapped): multimem.ld_reduce on it sums
  all ranks' copies in the switch, multimem.st writes all of them.

With world == 1 nothing is exported: the "peer" of rank 0 is itself, and a
one-device multicast object is still created and bound in NVLS mode (the path a
single GPU can exercise). Torch only sees the local arenas, wrapped zero-copy
as tensors through __cuda_array_interface__.
"""

from __future__ import annotations

import ctypes
import ctypes as C
import os

from . import _native as N
from .errors import EvalError

_PIDFD_GETFD = 438  # x86_64 / aarch64 syscall number


def _cu():
    from cuda.bindings import driver as cu

    return cu


def _ck(res, what):
    cu = _cu()
    err = res[0] if isinstance(res, tuple) else res
    if err != cu.CUresult.CUDA_SUCCESS:
        raise EvalError(f"{what} failed: {err}")
    if isinstance(res, tuple):
        return res[1] if len(res) == 2 else res[1:]
    return None


def _pidfd_getfd(pid: int, fd: int) -> int:
    libc = ctypes.CDLL(None, use_errno=True)
    pidfd = os.pidfd_open(pid)
    try:
        out = libc.syscall(_PIDFD_GETFD, pidfd, fd, 0)
        if out < 0:
            raise EvalError(f"pidfd_getfd({pid}, {fd}) failed: errno {ctypes.get_errno()}")
        return out
    finally:
        os.close(pidfd)


def multicast_supported(device: int = 0) -> tuple[bool, str]:
    """Can this box create an NVLS multicast object? (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED,
    then a one-device cuMulticastCreate: single-GPU boxes without an NVSwitch fabric
    report the attribute but refuse the object with CUDA_ERROR_INVALID_VALUE.)"""
    cu = _cu()
    _ck(cu.cuInit(0), "cuInit")
    dev = _ck(cu.cuDeviceGet(device), "cuDeviceGet")
    attr = _ck(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev),
               "multicast attribute")
    if not attr:
        return False, "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0"
    ctx = _ck(cu.cuDevicePrimaryCtxRetain(dev), "cuDevicePrimaryCtxRetain")
    _ck(cu.cuCtxSetCurrent(ctx), "cuCtxSetCurrent")
    mp = cu.CUmulticastObjectProp()
    mp.numDevices = 1
    mp.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    mp.size = 2 << 20
    res = cu.cuMulticastCreate(mp)
    if res[0] != cu.CUresult.CUDA_SUCCESS:
        return False, f"cuMulticastCreate: {res[0]}"
    cu.cuMemRelease(res[1])
    return True, ""


class _CudaArray:
    def __init__(self, ptr: int, nfloats: int):
        self.__cuda_array_interface__ = {"shape": (nfloats,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerArena:
    """`nbytes` of device memory per rank, mapped on every rank (and optionally
    multicast). `ptrs[q]` is rank q's copy in this process's address space."""

    def __init__(self, nbytes: int, rank: int, world: int, device: int, multicast: bool = False,
                 group=None):
        cu = _cu()
        _ck(cu.cuInit(0), "cuInit")
        self.cu = cu
        self.rank, self.world, self.device = rank, world, device
        self.dev = _ck(cu.cuDeviceGet(device), "cuDeviceGet")
        # the device's primary context: the one torch and the native library run in
        self._ctx = _ck(cu.cuDevicePrimaryCtxRetain(self.dev), "cuDevicePrimaryCtxRetain")
        _ck(cu.cuCtxSetCurrent(self._ctx), "cuCtxSetCurrent")
        prop = cu.CUmemAllocationProp()
        prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = device
        prop.requestedHandleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        gran = _ck(cu.cuMemGetAllocationGranularity(
            prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "granularity")
        self.mc_prop = None
        if multicast:
            mp = cu.CUmulticastObjectProp()
            mp.numDevices = world
            mp.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
            mp.size = max(int(nbytes), 1)
            mg = _ck(cu.cuMulticastGetGranularity(
                mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "mc granularity")
            gran = max(int(gran), int(mg))
            self.mc_prop = mp
        self.size = -(-max(int(nbytes), 1) // int(gran)) * int(gran)
        self.handle = _ck(cu.cuMemCreate(self.size, prop, 0), "cuMemCreate")
        self._maps: list[tuple[int, int]] = []
        self._imported = []
        local = self._map(self.handle)
        self.ptrs = [0] * world
        self.ptrs[rank] = local
        self._fds = []
        if world > 1:
            import torch.distributed as dist

            fd = _ck(cu.cuMemExportToShareableHandle(
                self.handle, cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "export")
            self._fds.append(int(fd))
            infos = [None] * world
            dist.all_gather_object(infos, (os.getpid(), int(fd)), group=group)
            for q, (pid, qfd) in enumerate(infos):
                if q == rank:
                    continue
                lfd = _pidfd_getfd(pid, qfd)
                try:
                    h = _ck(cu.cuMemImportFromShareableHandle(
                        lfd, cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), "import")
                finally:
                    os.close(lfd)
                self._imported.append(h)
                self.ptrs[q] = self._map(h)
            dist.barrier(group=group)  # every rank imported before exporters may close
        self.mc_ptr = 0
        if multicast:
            self._multicast(group)
        _ck(cu.cuMemsetD8(local, 0, self.size), "memset")
        _ck(cu.cuCtxSynchronize(), "sync")

    def _map(self, handle) -> int:
        cu = self.cu
        va = _ck(cu.cuMemAddressReserve(self.size, 0, 0, 0), "cuMemAddressReserve")
        _ck(cu.cuMemMap(va, self.size, 0, handle, 0), "cuMemMap")
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = self.device
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        _ck(cu.cuMemSetAccess(va, self.size, [acc], 1), "cuMemSetAccess")
        self._maps.append((int(va), self.size))
        return int(va)

    def _multicast(self, group) -> None:
        cu = self.cu
        self.mc_prop.size = self.size
        if self.rank == 0:
            mc = _ck(cu.cuMulticastCreate(self.mc_prop), "cuMulticastCreate")
        if self.world > 1:
            import torch.distributed as dist

            info = [None]
            if self.rank == 0:
                fd = _ck(cu.cuMemExportToShareableHandle(
                    mc, cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "mc export")
                self._fds.append(int(fd))
                info = [(os.getpid(), int(fd))]
            dist.broadcast_object_list(info, src=0, group=group)
            if self.rank != 0:
                lfd = _pidfd_getfd(*info[0])
                try:
                    mc = _ck(cu.cuMemImportFromShareableHandle(
                        lfd, cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), "mc import")
                finally:
                    os.close(lfd)
        _ck(cu.cuMulticastAddDevice(mc, self.dev), "cuMulticastAddDevice")
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier(group=group)  # all devices added before any bind
        _ck(cu.cuMulticastBindMem(mc, 0, self.handle, 0, self.size, 0), "cuMulticastBindMem")
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier(group=group)
        self.mc = mc
        self.mc_ptr = self._map(mc)

    def tensor(self, offset_bytes: int, nfloats: int):
        """Local copy as a torch float32 tensor view (zero-copy)."""
        import torch

        return torch.as_tensor(_CudaArray(self.ptrs[self.rank] + offset_bytes, nfloats),
                               device=torch.device("cuda", self.device))


class FusedAllReduce:
    """The gradient / variable arenas of one rank plus its wap_ar_group_t.

    mode: "p2p" (peer loads summed in ascending rank order: the reference's left
    fold, interp.py:115-119) or "nvls" (multimem.ld_reduce / multimem.st)."""

    def __init__(self, rank: int, world: int, device: int, mode: str = "p2p", group=None):
        if world > N.AR_MAX_RANKS:
            raise EvalError(f"fused allreduce supports up to {N.AR_MAX_RANKS} ranks, got {world}")
        if mode not in ("p2p", "nvls"):
            raise EvalError(f"unknown fused allreduce mode {mode!r}")
        self.rank, self.world, self.device, self.mode, self.group = rank, world, device, mode, group
        self.var = self.grad = self.flags = None

    def allocate(self, arena_floats: int):
        """(var tensor, grad tensor): this rank's arenas of `arena_floats` floats."""
        import torch

        nb = 4 * arena_floats
        mc = self.mode == "nvls"
        self.var = PeerArena(nb, self.rank, self.world, self.device, mc, self.group)
        self.grad = PeerArena(nb, self.rank, self.world, self.device, mc, self.group)
        self.flags = PeerArena(4 * N.AR_FLAG_WORDS, self.rank, self.world, self.device, False, self.group)
        dev = torch.device("cuda", self.device)
        self.counters = torch.zeros(2 * N.AR_SLOTS + 1, dtype=torch.int32, device=dev)
        g = N.wap_ar_group_t()
        g.world, g.rank, g.mode = self.world, self.rank, 1 if mc else 0
        for q in range(self.world):
            g.grad[q] = self.grad.ptrs[q]
            g.var[q] = self.var.ptrs[q]
            g.flags[q] = self.flags.ptrs[q]
        g.grad_mc = self.grad.mc_ptr or None
        g.var_mc = self.var.mc_ptr or None
        base = self.counters.data_ptr()
        g.epochs = base
        g.done = base + 4 * N.AR_SLOTS
        g.status = base + 8 * N.AR_SLOTS
        self.desc = g
        return self.var.tensor(0, arena_floats), self.grad.tensor(0, arena_floats)

    def launch(self, offset: int, n: int, lr: float, slot: int, stream_ptr: int, scale: float = 1.0) -> None:
        N.check(N.lib().wap_allreduce_sgd(C.byref(self.desc), offset, n, C.c_float(lr), C.c_float(scale), slot,
                                          stream_ptr), "wap_allreduce_sgd")

    def status(self) -> int:
        """Device error word: 1 if a barrier timed out (a peer never arrived)."""
        return int(self.counters[2 * N.AR_SLOTS].item())
