"""Streamed host <-> device transfer of eigenvector bases.

The reference keeps packs column-major (f32 on disk, memmapped) and streams
them in 64-column blocks (fastrw.py:38, 310-314, 380-382).  On the device the
basis is row-major f64, so every transfer is a transpose.  These
helpers move a basis in column blocks through two pinned staging buffers:
while block i is copied (DMA engine, side stream) and transposed (this
library's kernel, current stream), the host fills block i+1 (file read /
memmap page-in / array copy), so the host never holds a second full copy of
the basis and the file is read exactly once (the .rwpk checksum is updated
from the same staged bytes, packs.py).
"""

from __future__ import annotations

import ctypes as C
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .device import ptr, require_cuda, stream_handle

CHUNK_BYTES = 256 << 20     # staging block (two pinned + two device buffers of this size)


def _blocks(n: int, m: int, itemsize: int, chunk_bytes: int | None):
    chunk_bytes = CHUNK_BYTES if chunk_bytes is None else chunk_bytes
    cols = max(1, min(m, chunk_bytes // max(1, n * itemsize)))
    return [(c0, min(m, c0 + cols)) for c0 in range(0, m, cols)], cols


def upload_columns(V, ldv: int, n: int, m: int, dtype, fetch, *, on_block=None, chunk_bytes: int | None = None):
    """Fill V[:, :m] (device, row-major f64, ld ldv) from a column-major host
    source delivered block by block.

    ``fetch(c0, c1, out)`` writes columns c0..c1-1 into ``out`` (a numpy view
    of shape ((c1 - c0) * n,), dtype ``dtype``, column after column) — from a
    file (readinto), a memmap slice or an array.  ``on_block(out)`` sees the
    same staged bytes (e.g. a checksum).  Returns the bytes moved."""
    torch = require_cuda()
    dtype = np.dtype(dtype)
    if dtype == np.float32:
        tdt, fn = torch.float32, "swb_f32_colmajor_to_f64_rowmajor"
    elif dtype == np.float64:
        tdt, fn = torch.float64, "swb_f64_colmajor_to_f64_rowmajor"
    else:
        raise TypeError(f"unsupported basis dtype {dtype}")
    blocks, cols = _blocks(n, m, dtype.itemsize, chunk_bytes)
    size = cols * n
    nbuf = min(3, len(blocks))
    pinned = [torch.empty(size, dtype=tdt, pin_memory=True) for _ in range(nbuf)]
    stage = [torch.empty(size, dtype=tdt, device="cuda") for _ in range(nbuf)]
    host = [p.numpy() for p in pinned]
    copy_stream = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    h2d_done = [None] * nbuf
    tr_done = [None] * nbuf
    seen = [None] * nbuf
    st = stream_handle()
    moved = 0
    # on_block (the checksum) runs on one worker thread, in block order, beside
    # the next block's read and this block's DMA (ctypes / readinto drop the GIL)
    pool = ThreadPoolExecutor(1) if on_block is not None else None
    try:
        for i, (c0, c1) in enumerate(blocks):
            b = i % nbuf
            k = (c1 - c0) * n
            if h2d_done[b] is not None:
                h2d_done[b].synchronize()            # pinned[b]'s previous DMA finished
            if seen[b] is not None:
                seen[b].result()                     # ... and its checksum pass
            fetch(c0, c1, host[b][:k])
            if pool is not None:
                seen[b] = pool.submit(on_block, host[b][:k])
            _h2d_and_transpose(torch, copy_stream, cur, stage, pinned, b, k, tr_done, h2d_done, fn, n, c0, c1,
                               V, ldv, st)
            moved += k * dtype.itemsize
        for f in seen:
            if f is not None:
                f.result()
    finally:
        if pool is not None:
            pool.shutdown(wait=True)
    cur.synchronize()    # the pinned buffers are released on return
    return moved


def _h2d_and_transpose(torch, copy_stream, cur, stage, pinned, b, k, tr_done, h2d_done, fn, n, c0, c1, V, ldv, st):
    """Block b: pinned -> device stage (side stream), then the transpose into
    V[:, c0:c1] on the current stream."""
    with torch.cuda.stream(copy_stream):
        if tr_done[b] is not None:
            copy_stream.wait_event(tr_done[b])   # stage[b] consumed by its transpose
        stage[b][:k].copy_(pinned[b][:k], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(copy_stream)
        h2d_done[b] = ev
    cur.wait_event(ev)
    _lib.call(fn, ptr(stage[b]), n, c1 - c0, C.c_void_p(V.data_ptr() + 8 * c0), ldv, st)
    ev2 = torch.cuda.Event()
    ev2.record(cur)
    tr_done[b] = ev2


def download_columns_f32(V, ldv: int, n: int, m: int, col_map, sink, *, chunk_bytes: int | None = None):
    """Stream V[:, col(j)] (device row-major f64) to the host as f32
    column-major blocks: ``sink(block)`` receives each block (numpy f32,
    (c1 - c0) * n values, column after column) in column order — the .rwpk
    payload layout (fastrw.py:243).  ``col_map`` (device int32, m) or None."""
    torch = require_cuda()
    blocks, cols = _blocks(n, m, 4, chunk_bytes)
    size = cols * n
    nbuf = min(2, len(blocks))
    if col_map is None:
        col_map = torch.arange(m, dtype=torch.int32, device="cuda")
    pinned = [torch.empty(size, dtype=torch.float32, pin_memory=True) for _ in range(nbuf)]
    stage = [torch.empty(size, dtype=torch.float32, device="cuda") for _ in range(nbuf)]
    host = [p.numpy() for p in pinned]
    copy_stream = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    d2h_done = [None] * nbuf
    st = stream_handle()
    pending = []
    for i, (c0, c1) in enumerate(blocks):
        b = i % nbuf
        k = (c1 - c0) * n
        if d2h_done[b] is not None:              # hand the previous block in this buffer to the sink
            d2h_done[b].synchronize()
            pc0, pc1 = pending.pop(0)
            sink(host[b][:(pc1 - pc0) * n])
        _lib.call("swb_f64_rowmajor_to_f32_colmajor", ptr(V), n, ldv, c1 - c0, ptr(col_map[c0:c1]), ptr(stage[b]),
                  st)
        ev = torch.cuda.Event()
        ev.record(cur)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(ev)
            pinned[b][:k].copy_(stage[b][:k], non_blocking=True)
            ev2 = torch.cuda.Event()
            ev2.record(copy_stream)
            d2h_done[b] = ev2
        pending.append((c0, c1))
    for i in range(len(pending)):
        b = (len(blocks) - len(pending) + i) % nbuf
        d2h_done[b].synchronize()
        pc0, pc1 = pending[i]
        sink(host[b][:(pc1 - pc0) * n])
