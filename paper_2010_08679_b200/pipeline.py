"""Overlapped host <-> device checkpoint pipeline for one rank.

The stall-window work of a checkpoint (K1 mark, K2 capture, K3 write) runs on
the compute stream; the next interval's lookups stream in (H2D) and the
previous checkpoint's payload streams out (D2H) on copy streams, so PCIe
transfers overlap the kernels (the paper's "background" write, engine.py:
347-411, with the quantization moved onto the GPU).

    pipe = CheckpointPipeline(checkpointer, idx_capacity)
    for host_idx in interval_lookups:          # pinned host tensors
        pipe.submit(host_idx, seg_off, seg_tables)
    payloads = pipe.drain()                    # [bytes, ...] with keep_outputs=True
"""

from __future__ import annotations

import torch

from . import _lib
from .sharded import ShardedCheckpointer
from .tracker import LookupStream


class CheckpointPipeline:
    """Double-buffered H2D -> compute -> D2H pipeline over a ShardedCheckpointer."""

    def __init__(self, ck: ShardedCheckpointer, idx_capacity: int, idx_dtype=torch.int32,
                 keep_outputs: bool = False):
        self.ck = ck
        dev = ck.device
        self.compute = torch.cuda.current_stream(dev)
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.idx = [torch.empty(idx_capacity, dtype=idx_dtype, device=dev) for _ in range(2)]
        self.payload = [ck.payload, torch.empty_like(ck.payload)]
        self.host_out = [torch.empty(ck.payload.numel(), dtype=torch.uint8, pin_memory=True)
                         for _ in range(2)]
        self.nbytes_host = torch.zeros(2, dtype=torch.int64, pin_memory=True)
        self.flags_host = torch.zeros(2, dtype=torch.int32, pin_memory=True)
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_done = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]
        self.k = 0
        self.pending = None  # (slot) whose D2H is not issued yet
        self.keep = keep_outputs
        self.outputs = []     # keep_outputs: every finished checkpoint's payload bytes
        self._retained = []   # (slot, nbytes) whose D2H is issued but not copied out yet
        self.h2d_bytes = 0
        self.d2h_bytes = 0

    def _issue_d2h(self, slot: int) -> None:
        self.ev_done[slot].synchronize()        # its counts are on the host now
        _lib.raise_flags(int(self.flags_host[slot]), "checkpoint")
        n = int(self.nbytes_host[slot])
        # this D2H rewrites host_out[slot]: copy a retained payload of the
        # slot's previous step out first
        self._collect(slot)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.ev_done[slot])
            self.host_out[slot][:n].copy_(self.payload[slot][:n], non_blocking=True)
            self.ev_out[slot].record(self.d2h)
        self.d2h_bytes += n
        if self.keep:
            self._retained.append((slot, n))

    def submit(self, host_idx, seg_off=None, seg_tables=None) -> None:
        """Queue one checkpoint interval whose lookups are in pinned host
        memory: a LookupStream (packed, mixed widths) or an index tensor split
        by seg_off."""
        s = self.k & 1
        packed = isinstance(host_idx, LookupStream)
        nbytes = host_idx.nbytes if packed else host_idx.numel() * host_idx.element_size()
        if self.idx[s].numel() * self.idx[s].element_size() < nbytes:
            raise ValueError("CheckpointPipeline: lookup stream larger than idx_capacity")
        # H2D: the slot's index buffer was last read by step k-2
        with torch.cuda.stream(self.h2d):
            if self.k >= 2:
                self.h2d.wait_event(self.ev_done[s])
            if packed:
                dev_in = host_idx.to(self.ck.device, out=self.idx[s].view(torch.uint8))
            else:
                n = host_idx.numel()
                self.idx[s][:n].copy_(host_idx, non_blocking=True)
                dev_in = self.idx[s][:n]
            self.ev_in[s].record(self.h2d)
        self.h2d_bytes += nbytes
        # compute: the slot's payload buffer must have left (D2H of step k-2)
        self.compute.wait_event(self.ev_in[s])
        if self.k >= 2:
            self.compute.wait_event(self.ev_out[s])
        self.ck.payload = self.payload[s]
        self.ck.step(dev_in, seg_off, seg_tables)
        self.nbytes_host[s:s + 1].copy_(self.ck.writer.sec_off[-1:], non_blocking=True)
        self.flags_host[s:s + 1].copy_(self.ck.writer.flags, non_blocking=True)
        self.ev_done[s].record(self.compute)
        # D2H of the previous step overlaps this step's kernels
        if self.pending is not None:
            self._issue_d2h(self.pending)
        self.pending = s
        self.k += 1

    def _collect(self, slot: int | None = None) -> None:
        """Copy retained payloads out of their pinned slots (all, or those of
        `slot`) once their D2H has completed, oldest first."""
        keep = []
        for s, n in self._retained:
            if slot is None or s == slot:
                self.ev_out[s].synchronize()
                self.outputs.append(bytes(self.host_out[s][:n].numpy()))
            else:
                keep.append((s, n))
        self._retained = keep

    def drain(self):
        """Issue the last D2H and wait for every transfer.  Returns every
        retained payload (keep_outputs=True) as bytes, in submission order,
        and clears the list."""
        if self.pending is not None:
            self._issue_d2h(self.pending)
            self.pending = None
        self.d2h.synchronize()
        self.compute.synchronize()
        self._collect()
        out, self.outputs = self.outputs, []
        return out


class TrainingCheckpointLoop:
    """Checkpoints overlapped with training (north star item 4): the payload
    of interval k is quantized, packed and copied to pinned host memory
    while interval k+1 trains.

    The reference runs its writer on a background job thread while the
    trainer continues (engine.py:229-233, 347-411; sim.py:329-352).  Here the
    stall is K2 + the dirty-row gather into a staging buffer on the compute
    stream (ShardedCheckpointer.checkpoint(staged_rows=...)); K3 then runs
    from the staged copy on a side stream, and a background thread waits for
    it and issues the pinned D2H on a copy stream -- the training steps never
    wait for either.  Payload slots are double-buffered; checkpoint() waits
    (on the host) only for the D2H of the checkpoint two intervals back
    before its slot is rewritten -- normally long complete.

        loop = TrainingCheckpointLoop(ck, staged_rows)
        for interval in ...:
            for batch in interval: train_step(...)   # marks ck.tracker
            loop.checkpoint()                        # returns the stall's end event
        payloads = loop.drain()                      # [bytes, ...] in order
    """

    def __init__(self, ck: ShardedCheckpointer, staged_rows: int, keep_outputs: bool = True,
                 on_payload=None):
        import queue
        import threading
        from ._device import device_of
        self.ck = ck
        self.staged_rows = int(staged_rows)
        dev = device_of(ck.device)
        self.device = dev
        self.copy = torch.cuda.Stream(dev)
        self.payload = [ck.payload, torch.empty_like(ck.payload)]
        self.host = [torch.empty(ck.payload.numel(), dtype=torch.uint8, pin_memory=True)
                     for _ in range(2)]
        self.meta = torch.zeros((2, 2), dtype=torch.int64, pin_memory=True)  # nbytes, flags
        self.ev_d2h = [torch.cuda.Event() for _ in range(2)]
        self.keep = keep_outputs
        self.on_payload = on_payload
        self.outputs, self.errors = [], []
        self.k = 0
        self.d2h_bytes = 0
        self._free = [threading.Event(), threading.Event()]  # the slot's D2H has completed
        for f in self._free:
            f.set()
        self._q = queue.Queue()
        self._t = threading.Thread(target=self._worker, daemon=True)
        self._t.start()

    def _worker(self) -> None:
        try:
            torch.cuda.set_device(self.device)
        except Exception as e:  # every checkpoint then reports it (no silent hang)
            self.errors.append(e)
        while True:
            item = self._q.get()
            if item is None:
                return
            s, ev = item
            try:
                ev.synchronize()  # K3 of this checkpoint (and its byte count) done
                n, fl = (int(v) for v in self.meta[s])
                _lib.raise_flags(fl, "checkpoint")
                with torch.cuda.stream(self.copy):
                    self.copy.wait_event(ev)
                    self.host[s][:n].copy_(self.payload[s][:n], non_blocking=True)
                    self.ev_d2h[s].record(self.copy)
                self.ev_d2h[s].synchronize()
                self.d2h_bytes += n
                out = bytes(self.host[s][:n].numpy()) if (self.keep or self.on_payload) else None
                if self.keep:
                    self.outputs.append(out)
                if self.on_payload is not None:
                    self.on_payload(out)
            except Exception as e:  # surfaced by drain()
                self.errors.append(e)
            finally:
                self._free[s].set()
                self._q.task_done()

    def checkpoint(self):
        """The interval ends: stall (capture + staging) on the current stream,
        then K3 and the D2H in the background.  Returns the event marking the
        end of the stall (training may update the tables after it)."""
        s = self.k & 1
        # the slot's previous payload (two checkpoints back) must have left:
        # normally long done, the host wait is then immediate
        self._free[s].wait()
        self._free[s].clear()
        try:
            self.ck.payload = self.payload[s]
            stall_end = self.ck.checkpoint(staged_rows=self.staged_rows)
            side = self.ck._side
            with torch.cuda.stream(side):
                self.meta[s, 0:1].copy_(self.ck.writer.sec_off[-1:], non_blocking=True)
                self.meta[s, 1:2].copy_(self.ck.writer.flags.to(torch.int64), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        except BaseException:
            self._free[s].set()  # nothing was queued for this slot
            raise
        self._q.put((s, ev))
        self.k += 1
        return stall_end

    def drain(self) -> list:
        """Wait for every queued checkpoint; raise the first error; return
        (and clear) the retained payloads in checkpoint order."""
        self._q.join()
        if self.errors:
            e, self.errors = self.errors[0], []
            raise e
        out, self.outputs = self.outputs, []
        return out

    def close(self) -> None:
        self.drain()
        self._q.put(None)
        self._t.join()
