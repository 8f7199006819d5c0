"""Row bands across GPUs: one process per GPU renders interleaved 8-row
blocks of every frame, gathered to the display rank (rank 0).

Pixels are independent (/root/reference/pkg/src/raytracer/renderer.py:14-15)
and the reference's output is the same for any worker count
(pkg/tests/test_renderer.py:229-238), so a frame is sharded by rows with no
exchange during the render.  Contiguous equal bands would be ~2.5x
imbalanced at 8 GPUs on the benchmark camera (the top 46% of rows are sky,
SURVEY.md §8e); round-robin 8-row blocks keep max/mean load within ~3%.

Three gathers:
  * `IpcFrame` (the device-resident path): rank 0 exports its device
    framebuffer through CUDA IPC and every rank's render kernel stores its
    rows straight into it over NVLink — the gather is fused into the render;
  * `ShmFrame` (the host-frame path): a page-locked host frame shared by the
    ranks of the node; every rank copies its own rows into it over its own
    PCIe link (rt_copy_partition_to_host), so the device-to-host traffic of a
    frame is spread over G links instead of funnelled through rank 0's;
  * `gather_bands` (collective fallback, and the CPU/gloo-testable path):
    compact rows per rank, `torch.distributed.gather` to rank 0, scatter into
    the frame.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native

BLOCK_ROWS = 8


def band_rows(height: int, part: int, n_parts: int, block_rows: int = BLOCK_ROWS) -> np.ndarray:
    """Frame rows rendered by partition `part`: (y // block_rows) % n_parts == part.
    Same mapping as the kernels' map_row (csrc/rt_device.cuh)."""
    if n_parts < 1 or not (0 <= part < n_parts) or block_rows < 1:
        raise ValueError("bad partition")
    y = np.arange(height)
    return y[(y // block_rows) % n_parts == part]


def band_row_counts(height: int, n_parts: int, block_rows: int = BLOCK_ROWS):
    return [len(band_rows(height, p, n_parts, block_rows)) for p in range(n_parts)]


def gather_bands(local_rows, frame, height, rank, world, block_rows=BLOCK_ROWS, group=None):
    """Gather each rank's compact rows [n_rows_r, W] into rank 0's `frame`
    [height, W] (torch tensors; CPU with gloo or CUDA with NCCL)."""
    import torch
    import torch.distributed as dist

    counts = band_row_counts(height, world, block_rows)
    width = local_rows.shape[1]
    pad = max(counts)
    send = torch.zeros((pad, width), dtype=local_rows.dtype, device=local_rows.device)
    send[: counts[rank]] = local_rows
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
    dist.gather(send, gather_list=bufs, dst=0, group=group)
    if rank == 0:
        for p in range(world):
            rows = torch.as_tensor(band_rows(height, p, world, block_rows), device=frame.device)
            frame.index_copy_(0, rows, bufs[p][: counts[p]])
    return frame if rank == 0 else None


def compact_rows(frame, part, n_parts, block_rows=BLOCK_ROWS):
    """The rows partition `part` renders, as a compact [n_rows, W] tensor."""
    import torch

    rows = torch.as_tensor(band_rows(frame.shape[0], part, n_parts, block_rows), device=frame.device)
    return frame.index_select(0, rows)


class IpcFrame:
    """Rank 0's device framebuffer, mapped into every rank's address space.

    `ptr` is where this rank's render kernel stores pixel (x, y) at
    ptr[y * width + x] — local memory on rank 0, NVLink peer memory elsewhere.
    `exchange` is a callable that broadcasts rank 0's 64-byte handle (e.g.
    torch.distributed.broadcast_object_list)."""

    def __init__(self, device: int, width: int, height: int, rank: int, exchange):
        self.lib = _native.load()
        self.rank = rank
        self.bytes = 4 * width * height
        self.owned = ctypes.c_void_p()
        self.ptr = None
        handle = (ctypes.c_uint8 * 64)()
        if rank == 0:
            _native.check(self.lib.rt_device_malloc(device, self.bytes, ctypes.byref(self.owned)), "rt_device_malloc")
            _native.check(self.lib.rt_ipc_get_handle(self.owned, handle), "rt_ipc_get_handle")
            self.ptr = self.owned
        blob = exchange(bytes(handle))
        if rank != 0:
            h = (ctypes.c_uint8 * 64).from_buffer_copy(blob)
            mapped = ctypes.c_void_p()
            _native.check(self.lib.rt_ipc_open(h, ctypes.byref(mapped)), "rt_ipc_open")
            self.ptr = mapped

    def close(self):
        if self.ptr is None:
            return
        if self.rank == 0:
            self.lib.rt_device_free(self.owned)
        else:
            self.lib.rt_ipc_close(self.ptr)
        self.ptr = None


class ShmFrame:
    """A host framebuffer shared by every rank of the node (POSIX shared
    memory), page-locked in each rank's process, uint32[width * height].

    `copy_rows(ctx, d_frame, part, n_parts)` copies this rank's rows of its
    device frame into it; after a barrier rank 0 holds the whole frame in
    `pixels`.  `exchange` broadcasts rank 0's segment name."""

    def __init__(self, ctx, width: int, height: int, rank: int, exchange):
        from multiprocessing import shared_memory

        self.width, self.height, self.rank = width, height, rank
        nbytes = 4 * width * height
        if rank == 0:
            self.shm = shared_memory.SharedMemory(create=True, size=nbytes)
            name = exchange(self.shm.name.encode()).decode()
        else:
            name = exchange(b"").decode()
            self.shm = shared_memory.SharedMemory(name=name)
            try:  # rank 0 owns (and unlinks) the segment; attached ranks must not
                from multiprocessing import resource_tracker

                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        self.pixels = np.ndarray((width * height,), dtype=np.uint32, buffer=self.shm.buf)
        self.ctx = ctx
        if not ctx.pin(self.pixels):
            raise _native.NativeError("could not page-lock the shared host frame")
        _native._PINS.hold(self.pixels)  # every rank copies into it: never evicted

    def copy_rows(self, d_frame, part: int, n_parts: int, stream=None, block_rows: int = BLOCK_ROWS):
        lib = _native.load()
        _native.check(lib.rt_copy_partition_to_host(self.ctx.handle, 0, _native.ptr(self.pixels), d_frame,
                                                    self.width, self.height, part, n_parts, block_rows, stream),
                      "rt_copy_partition_to_host")

    def close(self):
        if self.shm is None:
            return
        _native._PINS.release(self.pixels)
        self.ctx.unpin(self.pixels)
        self.pixels = None
        self.shm.close()
        if self.rank == 0:
            self.shm.unlink()
        self.shm = None


def torch_exchange(blob: bytes) -> bytes:
    """Broadcast rank 0's bytes to every rank with torch.distributed."""
    import torch.distributed as dist

    obj = [blob]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]
