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
        self.log = None            # a list: (start, end, bytes) of every push (bench NVLink roofline)

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
            if self.log is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
            peer.copy_(src.view(-1), non_blocking=True)
            if self.log is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(self.stream)
                self.log.append((e0, e1, 4 * src.numel()))
            self.hdl.put_signal(dst_rank, channel)
        self.bytes_pushed += 4 * src.numel()

    def nvlink_summary(self):
        """Pushes logged since `log` was set to a list: bytes, total copy-engine
        time (the copies are serialised on one stream) and the achieved rate
        while copying (synchronises)."""
        torch.cuda.synchronize()
        if not self.log:
            return None
        byts = sum(b for _, _, b in self.log)
        ms = sum(e0.elapsed_time(e1) for e0, e1, _ in self.log)
        return {"bytes": byts, "copy_ms": ms, "pushes": len(self.log),
                "achieved_gbs": byts / (ms / 1e3) / 1e9 if ms > 0 else None}

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


class HeadChain:
    """NVLink hand-off of chunk-boundary snapshots between the graph streams
    of neighbouring ranks (SURVEY §7 hard part 3, fix 2).

    In a block the ranks own consecutive chunks of timesteps, so the head
    A_{t0} of rank q's chunk directly follows the last snapshot A_{t0-1} of
    rank q-1's chunk (rank P-1 -> rank 0 across blocks).  Instead of
    shipping the head in full over PCIe, rank q-1 pushes its raw CSR of
    A_{t0-1} (rowptr + col, int32) into rank q's receive buffer with the copy
    engine and signals; rank q's graph stream waits for it, applies the
    1-step delta of t0 on top and acknowledges, which frees the buffer for
    the next hand-off.  Channels: DATA (q-1 -> q), ACK (q -> q-1).  A
    missing signal traps after TIMEOUT_MS (ProtocolError at the engine)."""

    DATA, ACK = 1, 2

    def __init__(self, device, n: int, cap_a: int):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        group = dist.group.WORLD.group_name
        symm.enable_symm_mem_for_group(group)
        self.n = int(n)
        self.buf = symm.empty(self.n + 1 + int(cap_a), dtype=torch.int32, device=device)
        self.hdl = symm.rendezvous(self.buf, group)
        self.sent = {}             # destination -> hand-offs so far
        self.bytes_pushed = 0

    def send(self, rowptr: torch.Tensor, col: torch.Tensor, nnz: int, dst: int, stream) -> None:
        """On `stream`: wait until `dst` released the previous hand-off, copy
        A's raw CSR into its receive buffer, signal."""
        n = self.n
        with torch.cuda.stream(stream):
            if self.sent.get(dst, 0):
                self.hdl.wait_signal(dst, self.ACK, timeout_ms=TIMEOUT_MS)
            peer = self.hdl.get_buffer(dst, (n + 1 + nnz,), torch.int32, 0)
            peer[:n + 1].copy_(rowptr[:n + 1], non_blocking=True)
            if nnz:
                peer[n + 1:n + 1 + nnz].copy_(col[:nnz], non_blocking=True)
            self.hdl.put_signal(dst, self.DATA)
        self.sent[dst] = self.sent.get(dst, 0) + 1
        self.bytes_pushed += 4 * (n + 1 + nnz)

    def recv_spec(self, src: int, nnz: int):
        """head_prev for Materializer.materialize: the local receive buffer,
        a wait for `src`'s DATA signal and the ACK once the head is rebuilt
        (both enqueued on the graph stream current at the call)."""
        n = self.n

        def wait():
            self.hdl.wait_signal(src, self.DATA, timeout_ms=TIMEOUT_MS)

        def done():
            self.hdl.put_signal(src, self.ACK)

        return self.buf[:n + 1], self.buf[n + 1:n + 1 + max(nnz, 1)], wait, done
