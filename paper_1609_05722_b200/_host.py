"""Host <-> device transfers of the public API through cached pinned staging buffers.

Pageable copies go through the driver's own bounce buffers; staging through page-locked memory
that persists across calls makes the per-call H2D of the counts and D2H of the results plain DMA.
One buffer per (direction, slot) grows to the largest request seen; an event guards reuse of an
upload buffer whose copy may still be in flight.
"""
from __future__ import annotations

import threading

import numpy as np

_lock = threading.Lock()
_bufs: dict = {}


def _pinned(key, nbytes: int):
    import torch
    ent = _bufs.get(key)
    if ent is None or ent[0].numel() < nbytes:
        ent = (torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
        _bufs[key] = ent
    return ent


def upload(arr: np.ndarray):
    """numpy array -> CUDA tensor of the same dtype and shape (on the current stream)."""
    import torch
    arr = np.ascontiguousarray(arr)
    with _lock:
        buf, ev = _pinned(("up", 0), arr.nbytes)
        ev.synchronize()  # the previous upload from this buffer has been consumed
        host = buf[: arr.nbytes].numpy().view(arr.dtype).reshape(arr.shape)
        np.copyto(host, arr)
        out = torch.empty(arr.shape, dtype=torch.from_numpy(host[:0]).dtype, device="cuda")
        out.copy_(torch.from_numpy(host), non_blocking=True)
        ev.record()
    return out


_DIRECT_MAX = 64 << 20  # results up to this size are returned in the page-locked memory they land in


def download(*tensors):
    """CUDA tensors -> numpy arrays (fresh, caller-owned), all transfers issued before one stream synchronise.

    Results up to 64 MiB are copied straight into page-locked blocks from torch's caching host allocator
    and returned as views that own them (no host-side copy; a block returns to the cache when its array
    is freed); larger ones go through the cached staging buffers and a host copy."""
    import torch
    outs = []
    with _lock:
        views = []
        for i, t in enumerate(tensors):
            t = t.contiguous()
            nbytes = t.numel() * t.element_size()
            if nbytes <= _DIRECT_MAX:
                host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                views.append((host, False))
            else:
                buf, _ = _pinned(("down", i), nbytes)
                host = buf[:nbytes].view(t.dtype).view(t.shape)
                views.append((host, True))
            host.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        for h, staged in views:
            outs.append(h.numpy().copy() if staged else h.numpy())
    return outs
