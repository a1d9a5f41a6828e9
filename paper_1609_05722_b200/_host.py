"""Host <-> device transfers of the public API through cached pinned staging buffers.

Pageable copies go through the driver's own bounce buffers; staging through page-locked memory
that persists across calls makes the per-call H2D of the counts and D2H of the results plain DMA.
Staging buffers and their reuse events are per (thread, device): concurrent ``denoise`` callers
(benchmark.py:117-121 runs jobs in a thread pool) never share a buffer or wait on each other's
streams, and an event is only ever recorded on the device it was created for.
"""
from __future__ import annotations

import threading

import numpy as np

_tls = threading.local()


def _bufs() -> dict:
    d = getattr(_tls, "bufs", None)
    if d is None:
        d = _tls.bufs = {}
    return d


def _pinned(key, nbytes: int, device: int):
    """This thread's page-locked buffer for (key, device), grown to nbytes, and its reuse event."""
    import torch
    bufs = _bufs()
    ent = bufs.get((key, device))
    if ent is None or ent[0].numel() < nbytes:
        if ent is not None:
            ent[1].synchronize()  # the old buffer may still be the source of an in-flight copy
        with torch.cuda.device(device):
            ev = torch.cuda.Event()
        ent = (torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True), ev)
        bufs[(key, device)] = ent
    return ent


def upload(arr: np.ndarray):
    """numpy array -> CUDA tensor of the same dtype and shape (on the current device and stream)."""
    import torch
    arr = np.ascontiguousarray(arr)
    dev = torch.cuda.current_device()
    buf, ev = _pinned("up", arr.nbytes, dev)
    ev.synchronize()  # the previous upload from this buffer has been consumed
    host = buf[: arr.nbytes].numpy().view(arr.dtype).reshape(arr.shape)
    np.copyto(host, arr)
    out = torch.empty(arr.shape, dtype=torch.from_numpy(host[:0]).dtype, device=f"cuda:{dev}")
    out.copy_(torch.from_numpy(host), non_blocking=True)
    ev.record()
    return out


_DIRECT_MAX = 64 << 20  # results up to this size are returned in the page-locked memory they land in


def download(*tensors):
    """CUDA tensors -> numpy arrays (fresh, caller-owned), all transfers issued before one stream synchronise.

    Results up to 64 MiB are copied straight into page-locked blocks from torch's caching host allocator
    and returned as views that own them (no host-side copy; a block returns to the cache when its array
    is freed); larger ones go through this thread's staging buffers and a host copy."""
    import torch
    dev = torch.cuda.current_device()
    views = []
    for i, t in enumerate(tensors):
        t = t.contiguous()
        nbytes = t.numel() * t.element_size()
        if nbytes <= _DIRECT_MAX:
            host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            views.append((host, False))
        else:
            buf, _ = _pinned(("down", i), nbytes, dev)
            host = buf[:nbytes].view(t.dtype).view(t.shape)
            views.append((host, True))
        host.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return [h.numpy().copy() if staged else h.numpy() for h, staged in views]
