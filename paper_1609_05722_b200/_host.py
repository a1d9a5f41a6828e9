"""Host <-> device transfers of the public API through cached pinned staging buffers.

Pageable copies go through the driver's own bounce buffers; staging through page-locked memory
that persists across calls makes the per-call H2D of the counts and D2H of the results plain DMA.
Staging buffers and their reuse events are per (thread, device): concurrent ``denoise`` callers
(benchmark.py:117-121 runs jobs in a thread pool) never share a buffer or wait on each other's
streams, and an event is only ever recorded on the device it was created for.
"""
from __future__ import annotations

import os
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


def stage_counts(noisy: np.ndarray):
    """DenoiseRequest's count validation fused with the staging of the counts (as exact floats) in this thread's
    page-locked upload buffer: one native pass instead of a validation pass plus a host copy, and an H2D copy of
    4 bytes per pixel.  Returns (valid, token): token identifies the staged copy for `upload_staged` (None when
    nothing usable was staged: no CUDA device, or a count too large for an exact float)."""
    from . import _lib
    L = _lib.lib()
    try:
        import torch
        cuda = torch.cuda.is_available()
    except Exception:  # noqa: BLE001 -- validation must work without a usable torch / CUDA
        cuda = False
    if not cuda or noisy.size == 0:
        return (not (noisy.size and L.foe_counts_check(noisy.ctypes.data, noisy.size))), None
    dev = torch.cuda.current_device()
    buf, ev = _pinned("upf", noisy.size * 4, dev)
    ev.synchronize()  # the previous upload from this buffer has been consumed
    rc = L.foe_counts_check_stage(noisy.ctypes.data, noisy.size, buf.data_ptr())
    gen = _tls.stage_gen = getattr(_tls, "stage_gen", 0) + 1  # a later staging invalidates this one
    if rc == 1:
        return False, None
    return True, ((os.getpid(), threading.get_ident(), dev, gen) if rc == 0 else None)


def upload_staged(token, shape):
    """The float32 CUDA tensor of counts staged by `stage_counts`, or None if that copy is gone (another request
    was staged since, or this is another thread or device)."""
    import torch
    if token is None:
        return None
    pid, tid, dev, gen = token
    if pid != os.getpid() or tid != threading.get_ident() or dev != torch.cuda.current_device() or gen != getattr(_tls, "stage_gen", 0):
        return None
    n = int(np.prod(shape))
    buf, ev = _pinned("upf", n * 4, dev)
    out = torch.empty(tuple(shape), dtype=torch.float32, device=f"cuda:{dev}")
    out.copy_(buf[: n * 4].view(torch.float32).view(tuple(shape)), non_blocking=True)
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
