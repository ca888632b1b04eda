"""Copy-engine exchanges over NVLink peer memory (torch symmetric memory).

The snapshot-partitioned epoch moves every exchanged frame as contiguous
[N/P rows x W] blocks (owner layout <-> vertex-major, `dist.py:176-228`).
Instead of NCCL all-to-all kernels -- which need SMs the persistent compute
kernels hold, and which can only start once a whole exchange is ready --
each block is *pushed* into the destination rank's receive buffer the moment
its producer kernel finishes: a `cudaMemcpyAsync` into the peer's mapping on
a side stream (the copy engines; no SMs), followed by a signal the consumer's
stream waits on just before the kernel that reads that block.  Every rank
allocates the same receive-buffer layout inside one symmetric allocation,
so a block's offset in the local buffer is its offset on every peer.
"""

from __future__ import annotations

import os

import torch

# a signal that does not arrive within this time traps the waiting kernel (a
# lost push or a rank that left the schedule); the engine reports it as
# ProtocolError instead of hanging (engine.Engine.finish)
TIMEOUT_MS = int(os.environ.get("DGNN_PEER_TIMEOUT_MS", "120000"))


class PeerExchange:
    def __init__(self, device, total_floats: int):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        group = dist.group.WORLD.group_name
        symm.enable_symm_mem_for_group(group)
        self.buf = symm.empty(int(total_floats), dtype=torch.float32, device=device)
        self.buf.zero_()
        self.hdl = symm.rendezvous(self.buf, group)
        self.stream = torch.cuda.Stream(device=device)
        self.used = 0
        self.bytes_pushed = 0
        self.max_channel = self.hdl.signal_pad_size // (4 * self.world) - 1

    def alloc(self, n: int) -> torch.Tensor:
        """A zeroed [n] fp32 view at the same offset on every rank."""
        n = int(n)
        n_al = (n + 63) // 64 * 64          # 256-byte aligned blocks
        if self.used + n_al > self.buf.numel():
            raise MemoryError("peer receive buffer exhausted")
        v = self.buf[self.used:self.used + n]
        self.used += n_al
        return v

    def _offset(self, view: torch.Tensor) -> int:
        return (view.data_ptr() - self.buf.data_ptr()) // 4

    def push(self, src: torch.Tensor, dst_view: torch.Tensor, dst_rank: int, channel: int) -> None:
        """Copy `src` into `dst_view`'s position on rank `dst_rank` once the
        work already enqueued on the current stream is done, then signal
        (`channel`) the destination.  Local destinations copy in stream order."""
        if dst_rank == self.rank:
            dst_view.copy_(src)
            return
        if channel > self.max_channel:
            raise ValueError("signal channel out of range")
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            peer = self.hdl.get_buffer(dst_rank, (src.numel(),), torch.float32, self._offset(dst_view))
            peer.copy_(src.view(-1), non_blocking=True)
            self.hdl.put_signal(dst_rank, channel)
        self.bytes_pushed += 4 * src.numel()

    def wait(self, src_rank: int, channel: int) -> None:
        """The current stream waits for `src_rank`'s push on `channel`."""
        if src_rank != self.rank:
            self.hdl.wait_signal(src_rank, channel, timeout_ms=TIMEOUT_MS)

    def drain(self) -> None:
        """The current stream waits for every push issued so far (before a
        pushed-from buffer is overwritten)."""
        torch.cuda.current_stream().wait_stream(self.stream)

    def barrier(self) -> None:
        """Stream-ordered barrier of all ranks (channel 0): nobody pushes into
        a buffer a peer may still be reading from the previous pass."""
        self.hdl.barrier(channel=0, timeout_ms=TIMEOUT_MS)
