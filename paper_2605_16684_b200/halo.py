"""Face-trace halo exchange between partitions that live in different
processes (one process per GPU, torch.distributed for the plumbing).

Replaces the reference's in-process Transport<Real>::send / wait
(core/include/esdg/exchange.hpp:32-57, call sites solver.hpp:255,294): one
contiguous block of traces per peer per RHS, posted before the volume kernel
and awaited before the surface kernel, so the transfer overlaps the interior
work exactly like rhs_job's phase order (solver.hpp:248-317).

Backend agnostic: NCCL over NVLink with CUDA tensors that alias the shard's
send/receive buffers, gloo with CPU tensors in the world_size-2 CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class DeviceBuffer:
    """Zero-copy view of library-owned device memory for torch.as_tensor."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 2}


def device_tensor(ptr: int, count: int, dtype: torch.dtype, device: int) -> torch.Tensor:
    nbytes = count * torch.empty((), dtype=dtype).element_size()
    if count == 0 or ptr == 0:
        return torch.empty(0, dtype=dtype, device=f"cuda:{device}")
    raw = torch.as_tensor(DeviceBuffer(ptr, nbytes), device=f"cuda:{device}")
    return raw.view(dtype)


class HaloExchange:
    """peers: [(rank, offset, count)] in traces, identical for the send and the
    receive buffer (esdg_b200_rank_halo); trace_len = 5 * nq^2 values.

    With a backend that cannot move device memory (gloo) and CUDA buffers the
    blocks are staged through pinned host memory -- the reference's own
    "host-staging model" (exchange.hpp:20-22); over NCCL they move directly
    between the GPUs' buffers."""

    def __init__(self, peers, trace_len, send: torch.Tensor, recv: torch.Tensor, group=None):
        self.peers, self.trace_len = peers, trace_len
        self.send, self.recv, self.group = send, recv, group
        self.reqs = []
        self.exchanges = 0
        self.h_send = self.h_recv = None
        self.staged = send.is_cuda and dist.get_backend(group) == "gloo"
        if self.staged:
            self.h_send = torch.empty(send.shape, dtype=send.dtype, pin_memory=True)
            self.h_recv = torch.empty(recv.shape, dtype=recv.dtype, pin_memory=True)

    def begin(self):
        """Posts all sends/receives of this RHS; returns immediately."""
        src, dst = self.send, self.recv
        if self.staged:
            self.h_send.copy_(self.send, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            src, dst = self.h_send, self.h_recv
        ops = []
        for rank, off, cnt in self.peers:
            a, b = off * self.trace_len, (off + cnt) * self.trace_len
            ops.append(dist.P2POp(dist.irecv, dst[a:b], rank, self.group))
            ops.append(dist.P2POp(dist.isend, src[a:b], rank, self.group))
        self.reqs = dist.batch_isend_irecv(ops) if ops else []
        self.exchanges += 1

    def close(self):
        """Drops every tensor that references the solver's buffers or stream.
        Must run BEFORE the solver is destroyed: torch's pinned-memory
        allocator records an event on each stream a block was used on when the
        block is freed, and the solver's stream dies with the solver."""
        if self.send is not None and self.send.is_cuda:
            torch.cuda.synchronize()
        self.send = self.recv = None
        self.h_send = self.h_recv = None
        self.reqs = []

    def end(self):
        """Makes the current stream (CUDA) or the host (CPU) wait for them."""
        for r in self.reqs:
            r.wait()
        self.reqs = []
        if self.staged:
            self.recv.copy_(self.h_recv, non_blocking=True)


def make_exchange_callback(solver, device: int, group=None):
    """Builds the esdg_b200_exchange_fn for a one-partition-per-process
    GpuSolver: phase 0 posts the NCCL transfers on the solver's stream order,
    phase 1 makes that stream wait for the receives."""
    dtype = torch.float64 if solver.prec == 8 else torch.float32
    send_ptr, recv_ptr, _ = solver.halo_buffers()
    tl = 5 * solver.nq * solver.nq
    n = solver.n_ghost * tl
    ex = HaloExchange(solver.halo(), tl, device_tensor(send_ptr, n, dtype, device),
                      device_tensor(recv_ptr, n, dtype, device), group)
    ext = torch.cuda.ExternalStream(solver.stream, device=device)

    def callback(_user, phase, _stream):
        try:
            with torch.cuda.stream(ext):
                if phase == 0:
                    ex.begin()
                else:
                    ex.end()
            return 0
        except Exception as exc:  # never raise through the C ABI
            print(f"[esdg_b200] halo exchange failed: {exc!r}", flush=True)
            return 1

    return callback, ex
