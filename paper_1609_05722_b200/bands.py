"""Row-band decomposition of one large image (BASELINE config 5) and batch sharding (config 4).

The reference runs one image in one process; there is no
distributed layer to mirror.  This module adds the two the north star asks for:

* ``shard_batch``: independent images split across ranks -- no collective on the
  data path (each image keeps its own solver state; ``denoise_batch`` per rank).
* ``solve_bands``: one image split into row bands along whole tile rows.  Per
  trial pass every band runs the fused kernel on its rows (+ a 2r halo), then
  the bands (1) all-gather their per-tile fp64 partials and (2) swap 2r boundary
  rows of the trial iterate and its gradient with their neighbours, and every
  band takes the same accept/reject decision from the same partials in the same
  order.  Any band count therefore reproduces the single-device solve bitwise.

Exchange backends: ``LocalExchange`` (all bands in this process, e.g. several
bands on one GPU to test the halo path) and ``DistExchange`` (one band per
rank over torch.distributed -- NCCL on B200s, gloo on CPU for the host-logic
tests).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .solver import BRANCH_CODES, SolverConfig, SolverTrace, NumericalFailure


class BandDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("B", "H", "W", "ty0", "ty1", "tiles_x", "tiles_y", "row0", "row1",
                                            "lrow0", "Hl", "halo")]


class BandBuffers(ctypes.Structure):
    _fields_ = [("partials", ctypes.c_void_p), ("partials_offset", ctypes.c_size_t),
                ("partials_count", ctypes.c_size_t), ("partials_total", ctypes.c_size_t),
                ("sendbuf", ctypes.c_void_p), ("recvbuf", ctypes.c_void_p), ("halo_count", ctypes.c_size_t),
                ("n_active", ctypes.c_void_p)]


def _bind():
    L = _lib.lib()
    if getattr(L, "_bands_bound", False):
        return L
    vp, i = ctypes.c_void_p, ctypes.c_int
    L.foe_tile_grid.argtypes = [i, i, i, ctypes.POINTER(i), ctypes.POINTER(i)]
    L.foe_band_geometry.argtypes = [i, i, i, i, i, i, ctypes.POINTER(BandDesc)]
    L.foe_band_describe.argtypes = [vp, i, i, i, i, i, ctypes.POINTER(BandDesc)]
    L.foe_band_workspace_size.argtypes = [vp, ctypes.POINTER(BandDesc), i]
    L.foe_band_workspace_size.restype = ctypes.c_size_t
    L.foe_band_buffers_get.argtypes = [vp, ctypes.POINTER(BandDesc), i, vp, ctypes.POINTER(BandBuffers)]
    L.foe_band_begin.argtypes = [vp, ctypes.POINTER(_lib.SolverCfgC), ctypes.POINTER(BandDesc), vp, vp, vp, vp, vp, i,
                                 vp, ctypes.c_size_t, vp]
    L.foe_band_trial.argtypes = [vp, ctypes.POINTER(_lib.SolverCfgC), ctypes.POINTER(BandDesc), i, vp,
                                 ctypes.c_size_t, vp]
    L.foe_band_commit.argtypes = [vp, ctypes.POINTER(_lib.SolverCfgC), ctypes.POINTER(BandDesc), i, i, vp,
                                  ctypes.c_size_t, vp]
    L.foe_band_final_pass.argtypes = L.foe_band_trial.argtypes
    L.foe_band_end.argtypes = [vp, ctypes.POINTER(BandDesc), i, vp, ctypes.c_size_t, vp, vp, vp, vp]
    L._bands_bound = True
    return L


def tile_grid(m: int, H: int, W: int) -> tuple[int, int]:
    tx, ty = ctypes.c_int(), ctypes.c_int()
    _lib.check(_bind().foe_tile_grid(m, H, W, ctypes.byref(tx), ctypes.byref(ty)), "foe_tile_grid")
    return tx.value, ty.value


def partition_tile_rows(tiles_y: int, n_bands: int) -> list[tuple[int, int]]:
    """Contiguous, balanced split of the global tile rows into n_bands bands."""
    if not 1 <= n_bands <= tiles_y:
        raise ValueError(f"cannot split {tiles_y} tile rows into {n_bands} bands")
    edges = [round(k * tiles_y / n_bands) for k in range(n_bands + 1)]
    return [(edges[k], edges[k + 1]) for k in range(n_bands)]


def band_geometry(m: int, B: int, H: int, W: int, ty0: int, ty1: int) -> BandDesc:
    d = BandDesc()
    _lib.check(_bind().foe_band_geometry(m, B, H, W, ty0, ty1, ctypes.byref(d)), "foe_band_geometry")
    return d


def shard_batch(n_images: int, rank: int, world: int) -> slice:
    """Contiguous shard of a batch for ``rank`` (config 4: no per-iteration collective)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = (n_images * rank) // world
    hi = (n_images * (rank + 1)) // world
    return slice(lo, hi)


class Band:
    """One row band of a B x H x W problem, resident on the current CUDA device."""

    def __init__(self, model, B, H, W, ty0, ty1, trace_cap, cfg: SolverConfig):
        import torch

        from .prior import device_bank
        self.L = _bind()
        self.bank = device_bank(model)
        self.cfg = cfg
        self.cfg_c = cfg.to_c()
        self.trace_cap = int(trace_cap)
        self.desc = BandDesc()
        _lib.check(self.L.foe_band_describe(self.bank.handle, B, H, W, ty0, ty1, ctypes.byref(self.desc)),
                   "foe_band_describe")
        d = self.desc
        self.ws_bytes = self.L.foe_band_workspace_size(self.bank.handle, ctypes.byref(d), self.trace_cap)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda")
        bufs = BandBuffers()
        _lib.check(self.L.foe_band_buffers_get(self.bank.handle, ctypes.byref(d), self.trace_cap, self.ws.data_ptr(),
                                               ctypes.byref(bufs)), "foe_band_buffers_get")
        base = self.ws.data_ptr()

        def view(ptr, count, dtype, itemsize):
            off = ptr - base
            return self.ws[off:off + count * itemsize].view(dtype)

        self.partials = view(bufs.partials, bufs.partials_total, torch.float64, 8)
        self.chunk = slice(bufs.partials_offset, bufs.partials_offset + bufs.partials_count)
        self.sendbuf = view(bufs.sendbuf, 2 * bufs.halo_count, torch.float32, 4).view(2, -1)
        self.recvbuf = view(bufs.recvbuf, 2 * bufs.halo_count, torch.float32, 4).view(2, -1)
        self.n_active = view(bufs.n_active, 1, torch.int32, 4)

    @property
    def rows(self):
        return self.desc.row0, self.desc.row1

    @property
    def local_rows(self):
        return self.desc.lrow0, self.desc.lrow0 + self.desc.Hl

    def _stream(self):
        import torch
        return torch.cuda.current_stream().cuda_stream

    def begin(self, u0_local, obs_local, lam, branch, max_iters):
        B = self.desc.B
        self._u0, self._obs = u0_local.contiguous(), obs_local.contiguous()
        self._lam = np.ascontiguousarray(np.broadcast_to(np.asarray(lam, np.float64), (B,)))
        br = [BRANCH_CODES[b] if isinstance(b, str) else int(b) for b in np.broadcast_to(np.asarray(branch), (B,))]
        self._br = np.ascontiguousarray(br, dtype=np.int32)
        self._it = np.ascontiguousarray(np.broadcast_to(np.asarray(max_iters, np.int32), (B,)))
        _lib.check(self.L.foe_band_begin(self.bank.handle, ctypes.byref(self.cfg_c), ctypes.byref(self.desc),
                                         self._u0.data_ptr(), self._obs.data_ptr(), self._lam.ctypes.data,
                                         self._br.ctypes.data, self._it.ctypes.data, self.trace_cap,
                                         self.ws.data_ptr(), self.ws_bytes, self._stream()), "foe_band_begin")

    def trial(self):
        _lib.check(self.L.foe_band_trial(self.bank.handle, ctypes.byref(self.cfg_c), ctypes.byref(self.desc),
                                         self.trace_cap, self.ws.data_ptr(), self.ws_bytes, self._stream()),
                   "foe_band_trial")

    def commit(self, init: bool):
        _lib.check(self.L.foe_band_commit(self.bank.handle, ctypes.byref(self.cfg_c), ctypes.byref(self.desc),
                                          self.trace_cap, int(init), self.ws.data_ptr(), self.ws_bytes,
                                          self._stream()), "foe_band_commit")

    def final_pass(self):
        """F at the final iterate (partials only; exchanged like a trial's, summed by end())."""
        _lib.check(self.L.foe_band_final_pass(self.bank.handle, ctypes.byref(self.cfg_c), ctypes.byref(self.desc),
                                              self.trace_cap, self.ws.data_ptr(), self.ws_bytes, self._stream()),
                   "foe_band_final_pass")

    def end(self):
        import torch
        d = self.desc
        u = torch.empty((d.B, d.row1 - d.row0, d.W), dtype=torch.float32, device="cuda")
        status = (_lib.ImageStatusC * d.B)()
        trace = np.zeros((d.B, self.trace_cap, 6))
        rc = self.L.foe_band_end(self.bank.handle, ctypes.byref(d), self.trace_cap, self.ws.data_ptr(), self.ws_bytes,
                                 u.data_ptr(), ctypes.cast(status, ctypes.c_void_p), trace.ctypes.data,
                                 self._stream())
        if rc not in (_lib.FOE_OK, _lib.FOE_E_NUMERICAL):
            _lib.check(rc, "foe_band_end")
        traces = [SolverTrace.from_rows(trace[b, :status[b].n_iters], status[b].n_trials) for b in range(d.B)]
        return u, traces, [status[b].status for b in range(d.B)], [status[b].failed_at for b in range(d.B)]


class LocalExchange:
    """All bands live in this process (one or several devices): exchange by device copies."""

    capturable = True  # stream-ordered device copies: a chunk of passes can be captured in a CUDA graph

    def __call__(self, bands):
        for p in bands:  # all-gather of the per-tile partials
            for q in bands:
                if q is not p:
                    p.partials[q.chunk].copy_(q.partials[q.chunk])
        for k, p in enumerate(bands):  # halo rows: dir 0 <- band above's dir 1, dir 1 <- band below's dir 0
            if k > 0:
                p.recvbuf[0].copy_(bands[k - 1].sendbuf[1])
            if k + 1 < len(bands):
                p.recvbuf[1].copy_(bands[k + 1].sendbuf[0])


class DistExchange:
    """One band per rank over torch.distributed: NCCL between B200s (device buffers); gloo (CPU tests, or
    several ranks sharing one GPU) stages the device buffers through host memory.  The gather buffers
    are allocated once and reused every pass.  The NCCL exchange is stream-ordered and can be captured
    with the passes in a CUDA graph (solve_bands(graph=True)); that is opt-in because no multi-GPU box
    was available to validate NCCL capture for this build, and the host-driven loop is the tested one."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self._bufs = {}

    capturable = False  # see the class note; solve_bands(graph=True) opts in for NCCL

    def _buf(self, name, n, dtype, device):
        import torch
        b = self._bufs.get(name)
        if b is None or b.numel() != n or b.dtype != dtype or b.device != device:
            b = self._bufs[name] = torch.zeros(n, dtype=dtype, device=device)
        return b

    def exchange_arrays(self, partials, chunk, chunk_sizes, sendbuf, recvbuf):
        """partials: full array (this rank's chunk filled); chunk_sizes: per-rank (offset, count)."""
        import torch
        dist = self.dist
        stage = self.backend == "gloo" and partials.is_cuda  # gloo moves host tensors only
        dev = torch.device("cpu") if stage else partials.device
        maxc = max(c for _, c in chunk_sizes)
        mine = self._buf("mine", maxc, partials.dtype, dev)
        mine[:chunk.stop - chunk.start].copy_(partials[chunk])
        gathered = self._buf("gather", maxc * self.world, partials.dtype, dev)
        dist.all_gather_into_tensor(gathered, mine, group=self.group)
        for r, (off, cnt) in enumerate(chunk_sizes):
            if r != self.rank:
                partials[off:off + cnt].copy_(gathered[r * maxc:r * maxc + cnt])
        if stage:
            send = self._buf("send", sendbuf.numel(), sendbuf.dtype, dev).view(sendbuf.shape)
            recv = self._buf("recv", recvbuf.numel(), recvbuf.dtype, dev).view(recvbuf.shape)
            send.copy_(sendbuf)
        else:
            send, recv = sendbuf, recvbuf
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, send[0], self._peer(self.rank - 1), self.group))
            ops.append(dist.P2POp(dist.irecv, recv[0], self._peer(self.rank - 1), self.group))
        if self.rank + 1 < self.world:
            ops.append(dist.P2POp(dist.isend, send[1], self._peer(self.rank + 1), self.group))
            ops.append(dist.P2POp(dist.irecv, recv[1], self._peer(self.rank + 1), self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if stage:
            recvbuf.copy_(recv)

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def __call__(self, bands):
        (band,) = bands
        self.exchange_arrays(band.partials, band.chunk, self.chunks, band.sendbuf, band.recvbuf)


def _one_pass(bands, exchange):
    for b in bands:
        b.trial()
    exchange(bands)
    for b in bands:
        b.commit(False)


def _pass_graph(bands, exchange, chunk):
    """A CUDA graph of `chunk` trial passes (trial -> exchange -> commit on every band), captured once per
    (band set, exchange) and replayed: no per-pass host orchestration.  Passes after an image is done are
    no-ops on the device (the pass, the exchange of unchanged buffers and the decision skip it)."""
    import torch
    key = (id(exchange), tuple(id(b) for b in bands), chunk)
    cache = bands[0].__dict__.setdefault("_graphs", {})
    g = cache.get(key)
    if g is None:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            for _ in range(chunk):
                _one_pass(bands, exchange)
        cache.clear()
        cache[key] = g
    return g


def solve_bands(bands, exchange, u0_locals, obs_locals, lam, branch, max_iters, poll: int = 8,
                raise_on_failure: bool = True, graph: bool | None = None):
    """Device-resident iPiano over row bands.  ``bands``: the bands this process drives (all of them
    for LocalExchange, its own one for DistExchange); ``u0_locals`` / ``obs_locals``: per band,
    (B, Hl, W) fp32 CUDA tensors holding rows [lrow0, lrow0 + Hl).  Returns per band (u_owned,
    traces, status, failed_at).

    With a capturable exchange (device copies, NCCL) the pass loop runs as replays of a CUDA graph of
    ``poll`` passes, the live-image count read once per replay; otherwise pass by pass from the host."""
    if isinstance(exchange, DistExchange):
        exchange.chunks = _all_chunks(bands[0], exchange)
    if graph is None:
        graph = bool(getattr(exchange, "capturable", False))
    if graph and isinstance(exchange, DistExchange) and exchange.backend != "nccl":
        raise ValueError("only device-side exchanges (LocalExchange, NCCL) can be captured in a CUDA graph")
    for b, u0, ob in zip(bands, u0_locals, obs_locals):
        b.begin(u0, ob, lam, branch, max_iters)
    exchange(bands)
    for b in bands:
        b.commit(True)
    n = 0
    cap = max(int(np.max(max_iters)) * 200 + 64, 64)
    if graph:
        g = _pass_graph(bands, exchange, poll)
    while True:
        if graph:
            g.replay()
            n += poll
        else:
            _one_pass(bands, exchange)
            n += 1
        if n % poll == 0 and int(bands[0].n_active.item()) == 0:
            break
        if n > cap:
            raise RuntimeError("band solve did not terminate")
    for b in bands:  # F(u_final) for the trace's F column (foe_solve's anchor, same partials and order)
        b.final_pass()
    exchange(bands)
    out = [b.end() for b in bands]
    if raise_on_failure:
        _u, traces, status, failed = out[0]
        for i, s in enumerate(status):
            if s == 1:
                raise NumericalFailure(f"non-finite smooth energy at iteration {failed[i]}", traces[i])
            if s == 2:
                raise NumericalFailure(f"backtracking stalled at iteration {failed[i]}", traces[i])
    return out


def _all_chunks(band, exchange):
    """(offset, count) of every rank's partials chunk, from the shared tile partition."""
    import torch
    t = torch.tensor([band.chunk.start, band.chunk.stop - band.chunk.start], dtype=torch.int64,
                     device=band.partials.device)
    out = [torch.zeros_like(t) for _ in range(exchange.world)]
    exchange.dist.all_gather(out, t, group=exchange.group)
    return [(int(x[0]), int(x[1])) for x in out]


def solve_image_bands(model, u0, obs, lam, branch, max_iters, n_bands: int, cfg: SolverConfig | None = None):
    """Split one (B,H,W) problem into ``n_bands`` row bands on the current device (LocalExchange) and
    reassemble the result -- the in-process form of the config-5 decomposition."""
    import torch
    cfg = cfg or SolverConfig()
    u0 = u0[None] if u0.dim() == 2 else u0
    obs = obs[None] if obs.dim() == 2 else obs
    B, H, W = u0.shape
    m = model.basis.size
    _, ty = tile_grid(m, H, W)
    cap = int(np.max(max_iters))
    bands = [Band(model, B, H, W, t0, t1, cap, cfg) for t0, t1 in partition_tile_rows(ty, n_bands)]
    u0l = [u0[:, b.local_rows[0]:b.local_rows[1]].contiguous() for b in bands]
    obl = [obs[:, b.local_rows[0]:b.local_rows[1]].contiguous() for b in bands]
    res = solve_bands(bands, LocalExchange(), u0l, obl, lam, branch, max_iters)
    u = torch.cat([r[0] for r in res], dim=1)
    return u, res[0][1], res[0][2]
