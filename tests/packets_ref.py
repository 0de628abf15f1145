"""numpy restatement of the sparse packet exchange's record format (vr_packets_pack /
vr_packets_unpack in include/vr_capi.h) — test infrastructure: the CPU gloo tests run
the exchange plumbing with it and the GPU tests check the kernels against it."""
import numpy as np

INT_MAX = np.iinfo(np.int32).max


def pack(local, counts, region_lo, extra=None):
    """local [cnt, R, 8] float32, counts [cnt*R] -> (records [n, width] float32, n); records
    in segment order (the kernel's order is arbitrary)."""
    cnt, R, _ = local.shape
    segs = np.nonzero(np.asarray(counts).reshape(-1) > 0)[0]
    width = 9 if extra is None else 10
    rec = np.zeros((len(segs), width), dtype=np.float32)
    rec[:, 0] = (region_lo * R + segs).astype(np.int32).view(np.float32)
    rec[:, 1:9] = local.reshape(-1, 8)[segs]
    if extra is not None:
        rec[:, 9] = np.asarray(extra, dtype=np.float32).reshape(-1)[segs]
    return rec, len(segs)


def buffer(rec, cap):
    """One rank's send buffer [cap + 1, width]: row 0 = record count (int32 bits)."""
    out = np.zeros((cap + 1, rec.shape[1]), dtype=np.float32)
    out[0, 0] = np.array([len(rec)], dtype=np.int32).view(np.float32)[0]
    out[1:1 + len(rec)] = rec
    return out


def unpack(bufs, world, n_regions, R):
    """[world * (cap+1), width] -> (slab [K, R, 8], extra slab [K, R] or None)."""
    width = bufs.shape[1]
    rows = len(bufs) // world
    slab = np.zeros((n_regions * R, 8), dtype=np.float32)
    slab[:, 0] = 1.0
    slab[:, 7] = np.array([INT_MAX], dtype=np.int32).view(np.float32)[0]
    extra = np.ones(n_regions * R, dtype=np.float32) if width == 10 else None
    for rk in range(world):
        b = bufs[rk * rows:(rk + 1) * rows]
        n = int(b[0:1, 0].copy().view(np.int32)[0])
        rec = b[1:1 + n]
        idx = rec[:, 0].copy().view(np.int32).astype(np.int64)
        slab[idx] = rec[:, 1:9]
        if extra is not None:
            extra[idx] = rec[:, 9]
    return slab.reshape(n_regions, R, 8), None if extra is None else extra.reshape(n_regions, R)
