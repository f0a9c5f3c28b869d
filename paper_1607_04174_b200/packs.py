"""`.rwpk` spectral packs straight to / from the GPU (reference
fastrw.py:228-325, format SPEC.md:318).

Layout: magic "RWPK", u32 version 1, u8 rank d, u64 dims[d], f64 spacing[d],
f64 beta, u32 m, u64 N, f64 values[m], f32 d_sqrt[N], f32 V column-major
N x m, u64 xxh64 of everything before it, 32-byte image hash.

load_pack verifies magic / size / checksum exactly like the reference (the
XXH64 runs natively in libspecwalk_b200.so instead of pure Python), uploads
the f32 block and transposes it on the GPU into the row-major f64 basis.
save_pack writes byte-identical files (reference test_fastrw.py:34-38).
"""

from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

from . import _lib
from .device import DevicePack, LatticeSpec, device_norm, ptr, require_cuda, round_up, stream_handle
from .errors import ChecksumMismatch, FormatError, IoError
from .types import PackProvenance

MAGIC = b"RWPK"
VERSION = 1
_CHUNK = 1 << 26


def xxh64_file(fh, nbytes: int) -> int:
    lib = _lib.load()
    st = C.create_string_buffer(lib.swb_xxh64_state_bytes())
    lib.swb_xxh64_init(st, 0)
    left = nbytes
    while left:
        chunk = fh.read(min(left, _CHUNK))
        if not chunk:
            raise FormatError("pack file truncated")
        lib.swb_xxh64_update(st, chunk, len(chunk))
        left -= len(chunk)
    return int(lib.swb_xxh64_digest(st))


def xxh64(data: bytes, seed: int = 0) -> int:
    lib = _lib.load()
    st = C.create_string_buffer(lib.swb_xxh64_state_bytes())
    lib.swb_xxh64_init(st, seed)
    lib.swb_xxh64_update(st, data, len(data))
    return int(lib.swb_xxh64_digest(st))


def _read_exact(fh, count, what):
    data = fh.read(count)
    if len(data) != count:
        raise FormatError(f"pack file truncated while reading {what}")
    return data


def load_pack(path, connectivity=None, weight_mode="abs", image=None) -> DevicePack:
    """fastrw.py:264-325 -> a GPU-resident pack (row-major f64 basis).

    One pass over the file: the header, eigenvalues and d_sqrt are read and
    hashed, then the f32 column-major eigenvector block streams through two
    pinned staging buffers into the device basis (transposed on the GPU,
    staging.upload_columns) while the same staged bytes feed the XXH64; the
    checksum is compared at the end (ChecksumMismatch, nothing returned).
    The host never holds the whole block (the reference streams 64-column
    blocks from a memmap, fastrw.py:310-314)."""
    from .staging import upload_columns
    try:
        fh = open(path, "rb", buffering=0)
    except OSError as exc:
        raise IoError(str(exc)) from exc
    lib = _lib.load()
    hs = C.create_string_buffer(lib.swb_xxh64_state_bytes())
    lib.swb_xxh64_init(hs, 0)

    def read(count, what):
        data = _read_exact(fh, count, what)
        lib.swb_xxh64_update(hs, data, len(data))
        return data

    with fh:
        if read(4, "magic") != MAGIC:
            raise FormatError(f"{path}: not a pack file (bad magic)")
        version = struct.unpack("<I", read(4, "version"))[0]
        if version != VERSION:
            raise FormatError(f"{path}: unsupported pack version {version}")
        d = struct.unpack("<B", read(1, "rank"))[0]
        if d not in (1, 2, 3):
            raise FormatError(f"{path}: bad dimensionality {d}")
        dims = np.frombuffer(read(8 * d, "dims"), dtype="<u8")
        spacing = np.frombuffer(read(8 * d, "spacing"), dtype="<f8")
        beta = struct.unpack("<d", read(8, "beta"))[0]
        m = struct.unpack("<I", read(4, "m"))[0]
        n = struct.unpack("<Q", read(8, "N"))[0]
        if int(np.prod(dims)) != n:
            raise FormatError(f"{path}: dims/N mismatch")
        q_offset = fh.tell() + 8 * m + 4 * n
        size = os.fstat(fh.fileno()).st_size
        expected = q_offset + 4 * n * m + 8 + 32
        if size != expected:
            raise FormatError(f"{path}: size {size} != expected {expected} bytes")
        values = np.frombuffer(read(8 * m, "eigenvalues"), dtype="<f8").astype(np.float64)
        d_sqrt = np.frombuffer(read(4 * n, "d_sqrt"), dtype="<f4").astype(np.float64)
        torch = require_cuda()
        ldv = round_up(max(m, 1), 8)
        V = torch.zeros((int(n), ldv), dtype=torch.float64, device="cuda")

        def fetch(c0, c1, out):
            mv = memoryview(out).cast("B")
            got = 0
            while got < mv.nbytes:
                k = fh.readinto(mv[got:])
                if not k:
                    raise FormatError("pack file truncated while reading eigenvectors")
                got += k

        def hash_block(out):
            lib.swb_xxh64_update(hs, out.ctypes.data_as(C.c_void_p), out.nbytes)

        upload_columns(V, ldv, int(n), int(m), np.float32, fetch, on_block=hash_block)
        digest = int(lib.swb_xxh64_digest(hs))
        stored = struct.unpack("<Q", _read_exact(fh, 8, "checksum"))[0]
        if digest != stored:
            raise ChecksumMismatch(f"{path}: checksum mismatch")
        image_hash = _read_exact(fh, 32, "image hash")
    dims_t = tuple(int(x) for x in dims)
    dsq = torch.from_numpy(d_sqrt).to("cuda")
    img_dev = None
    if image is not None:
        img_dev = torch.from_numpy(np.array(image.intensities, dtype=np.float64)).to("cuda")
    lattice = LatticeSpec.make(dims_t if len(dims_t) > 1 else dims_t + (1,), connectivity, weight_mode)
    return DevicePack(V, int(m), torch.from_numpy(values).to("cuda"), dsq, device_norm(dsq), dims_t,
                      tuple(float(s) for s in spacing), float(beta), PackProvenance(image_hash=image_hash),
                      lattice, image_dev=img_dev)


def save_pack(pack, path) -> None:
    """fastrw.py:228-254 from a GPU pack; byte-identical to the reference.

    The f32 column-major payload streams device -> pinned host blocks
    (staging.download_columns_f32, the refreshed pack's column order folded
    into the transpose) straight into the file and the XXH64, so the host
    holds one staging block, not the payload."""
    from .staging import download_columns_f32
    require_cuda()
    dims = tuple(int(x) for x in pack.dims)
    d = len(dims)
    m = int(pack.m)
    n = int(pack.n_vertices)
    header = b"".join([MAGIC, struct.pack("<I", VERSION), struct.pack("<B", d),
                       np.asarray(dims, dtype="<u8").tobytes(),
                       np.asarray(pack.spacing if pack.spacing else (1.0,) * d, dtype="<f8").tobytes(),
                       struct.pack("<d", float(pack.beta)), struct.pack("<I", m), struct.pack("<Q", n)])
    values = np.asarray(pack.values, dtype="<f8").tobytes()
    d_sqrt = np.asarray(pack.d_sqrt).astype("<f4", copy=False).tobytes()
    lib = _lib.load()
    st = C.create_string_buffer(lib.swb_xxh64_state_bytes())
    lib.swb_xxh64_init(st, 0)
    ihash = pack.provenance.image_hash if pack.provenance is not None else b"\0" * 32
    try:
        with open(path, "wb") as fh:
            for chunk in (header, values, d_sqrt):
                lib.swb_xxh64_update(st, chunk, len(chunk))
                fh.write(chunk)

            def sink(block):
                lib.swb_xxh64_update(st, block.ctypes.data_as(C.c_void_p), block.nbytes)
                fh.write(memoryview(block).cast("B"))

            download_columns_f32(pack.V, pack.ldv, n, m, pack.col_map, sink)
            fh.write(struct.pack("<Q", int(lib.swb_xxh64_digest(st))))
            fh.write(ihash)
    except OSError as exc:
        raise IoError(str(exc)) from exc
