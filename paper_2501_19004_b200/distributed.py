"""Collectives of the sharded engine (lvn_louvain_sharded)
over torch.distributed.

One process per GPU, launched by torchrun. torch.distributed is the transport:
NCCL over NVLink / NVSwitch on the GPU box; gloo in the CPU tests (host
buffers) and in the single-GPU multi-rank test, where device buffers are
staged through host memory because two ranks cannot share a GPU under NCCL.

The engine calls ``allreduce`` / ``allgatherv`` from inside
lvn_louvain_sharded with its own stream idle; each call returns once the
result is in place (the torch stream is synchronised before returning).
A collective that raises is reported to the engine as a failure (non-zero
return), which makes lvn_louvain_sharded fail with LVN_CUDA on that rank.
"""

from __future__ import annotations

import ctypes as C
import traceback

import torch
import torch.distributed as dist

from . import _native as N

# element types of lvn_dtype; sums of u64 counters use int64 lanes (same bits)
_TORCH = {N.LVN_U8: (torch.uint8, 1), N.LVN_U32: (torch.int32, 4), N.LVN_U64: (torch.int64, 8),
          N.LVN_F64: (torch.float64, 8)}
_OPS = {N.LVN_SUM: dist.ReduceOp.SUM, N.LVN_MAX: dist.ReduceOp.MAX}


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class Collectives:
    """lvn_comm backed by a torch.distributed process group.

    location "cuda": the engine's buffers are device pointers on the current
    device (the product path). location "cpu": host pointers (CPU tests of
    the exchange protocol without a GPU).
    """

    def __init__(self, group=None, location: str = "cuda"):
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.backend = str(dist.get_backend(group))
        self.location = location
        self.stage = location == "cuda" and self.backend == "gloo"
        self.errors: list[str] = []
        self.calls = {"allreduce": 0, "allgatherv": 0, "alltoallv": 0}
        self.bytes = 0
        self._ar = N.ALLREDUCE_FN(self._allreduce)
        self._ag = N.ALLGATHERV_FN(self._allgatherv)
        self._aa = N.ALLTOALLV_FN(self._alltoallv)
        self.struct = N.lvn_comm(self.rank, self.size, None, self._ar, self._ag, self._aa)

    # -- views of engine buffers ------------------------------------------------------
    def _bytes(self, ptr: int, nbytes: int) -> torch.Tensor:
        if nbytes == 0:
            return torch.empty(0, dtype=torch.uint8, device=self.location)
        if self.location == "cuda":
            return torch.as_tensor(_CudaArray(ptr, nbytes), device="cuda")
        return torch.frombuffer((C.c_uint8 * nbytes).from_address(ptr), dtype=torch.uint8)

    def _sync(self):
        if self.location == "cuda":
            torch.cuda.current_stream().synchronize()

    # -- collectives ----------------------------------------------------------------
    def allreduce_tensor(self, t: torch.Tensor, op: int) -> None:
        if self.stage:
            h = t.cpu()
            dist.all_reduce(h, op=_OPS[op], group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=_OPS[op], group=self.group)

    def allgatherv_bytes(self, send: torch.Tensor, recv: torch.Tensor, counts: list[int]) -> None:
        mx = max(counts)
        if mx == 0:
            return
        dev = "cpu" if self.stage else send.device
        buf = torch.zeros(mx, dtype=torch.uint8, device=dev)
        buf[: counts[self.rank]].copy_(send[: counts[self.rank]])
        parts = [torch.empty(mx, dtype=torch.uint8, device=dev) for _ in range(self.size)]
        dist.all_gather(parts, buf, group=self.group)
        pos = 0
        for k, c in enumerate(counts):
            if c:
                recv[pos: pos + c].copy_(parts[k][:c])
            pos += c

    def alltoallv_bytes(self, send: torch.Tensor, scounts: list[int], recv: torch.Tensor,
                        rcounts: list[int]) -> None:
        if self.stage or send.device.type == "cpu":
            # gloo: all_to_all_single on host tensors
            s_h = send.cpu() if send.device.type != "cpu" else send
            r_h = torch.empty(sum(rcounts), dtype=torch.uint8)
            dist.all_to_all_single(r_h, s_h, output_split_sizes=rcounts, input_split_sizes=scounts,
                                   group=self.group)
            recv.copy_(r_h)
        else:
            dist.all_to_all_single(recv, send, output_split_sizes=rcounts, input_split_sizes=scounts,
                                   group=self.group)

    def _alltoallv(self, user, send, scounts, recv, rcounts) -> int:
        try:
            self.calls["alltoallv"] += 1
            sc = [int(scounts[k]) for k in range(self.size)]
            rc = [int(rcounts[k]) for k in range(self.size)]
            self.bytes += sum(sc)
            self.alltoallv_bytes(self._bytes(send, sum(sc)), sc, self._bytes(recv, sum(rc)), rc)
            self._sync()
            return 0
        except Exception:  # noqa: BLE001
            self.errors.append(traceback.format_exc())
            return 1

    def _allreduce(self, user, buf, count, dtype, op) -> int:
        try:
            self.calls["allreduce"] += 1
            tdt, size = _TORCH[dtype]
            nbytes = int(count) * size
            self.bytes += nbytes
            if nbytes:
                self.allreduce_tensor(self._bytes(buf, nbytes).view(tdt), op)
                self._sync()
            return 0
        except Exception:  # noqa: BLE001 - reported to the engine as a failed collective
            self.errors.append(traceback.format_exc())
            return 1

    def _allgatherv(self, user, send, recv, counts) -> int:
        try:
            self.calls["allgatherv"] += 1
            cs = [int(counts[k]) for k in range(self.size)]
            self.bytes += sum(cs)
            total = sum(cs)
            if total:
                # send may alias its own slot of recv: snapshot it first
                own = self._bytes(send, cs[self.rank]).clone() if cs[self.rank] else \
                    torch.empty(0, dtype=torch.uint8, device=self.location)
                self.allgatherv_bytes(own, self._bytes(recv, total), cs)
                self._sync()
            return 0
        except Exception:  # noqa: BLE001
            self.errors.append(traceback.format_exc())
            return 1


class NcclComm:
    """The library's own NCCL communicator (lvn_comm_nccl_create): collectives
    enqueued on the engine stream inside liblvn.so, no Python on the data path.
    torch.distributed only ships the NCCL unique id from rank 0 (any process
    group: the default one of torchrun)."""

    def __init__(self, group=None):
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        L = N.lib()
        uid = (C.c_ubyte * 128)()
        if self.rank == 0 and L.lvn_nccl_unique_id(uid) != 0:
            raise RuntimeError(N.last_error())
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
        ptr = C.POINTER(N.lvn_comm)()
        if L.lvn_comm_nccl_create(self.rank, self.size, uid, C.byref(ptr)) != 0:
            raise RuntimeError(N.last_error())
        self._ptr = ptr
        self.struct = ptr.contents
        self.errors: list[str] = []
        self.calls = {}

    def close(self) -> None:
        if self._ptr:
            N.lib().lvn_comm_destroy(self._ptr)
            self._ptr = None
            self.struct = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
