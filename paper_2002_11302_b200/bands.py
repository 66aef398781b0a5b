"""Row-band partitioning of C = A·B across GPUs.

C(r0:r1, :) = A(r0:r1, :) · B, so output row bands are independent. Rank r
of G takes the CSC row-slab of A for rows [cuts[r], cuts[r+1]) — cuts are
flop-balanced, from the per-row flop the reference's ``balanced_starts``
accumulates (pb_spgemm.cpp:58-82) — and all of B (broadcast once at setup).
No collective runs in the hot path; afterwards an all-gather of the G band
nnz values turns the band rowptrs into one global CSR, and concatenating the
bands in rank order *is* the global CSR.

This is the paper's thesis variant of partitioning A's rows per socket
(PAPER.md:913-914), applied per GPU.
"""
from __future__ import annotations

import numpy as np

from . import matrices as M


def plan_bands(a_csc: M.CscMatrix, b_csr: M.CsrMatrix, g: int) -> np.ndarray:
    """Flop-balanced row cuts (g+1 entries, cuts[0]=0, cuts[g]=nrows).
    Deterministic, so every rank computes the same cuts without talking."""
    if g < 1:
        raise ValueError("need at least one band")
    return M.band_cuts(M.row_flop(a_csc, b_csr), g)


def band_slab(a_csc: M.CscMatrix, cuts: np.ndarray, r: int) -> M.CscMatrix:
    """Rank r's CSC row-slab of A (rows renumbered from 0)."""
    return M.row_band(a_csc, int(cuts[r]), int(cuts[r + 1]))


def band_offsets(band_nnz) -> np.ndarray:
    """Exclusive prefix of the per-band nnz: where each band's entries start
    in the global colids/values arrays."""
    nz = np.asarray(band_nnz, dtype=np.uint64)
    off = np.zeros(nz.size + 1, dtype=np.uint64)
    np.cumsum(nz, out=off[1:])
    return off


def assemble(bands: list, cuts: np.ndarray, ncols: int) -> M.CsrMatrix:
    """Concatenate band CSRs (rows [cuts[r], cuts[r+1])) into the global CSR."""
    nrows = int(cuts[-1])
    off = band_offsets([b.nnz for b in bands])
    rowptr = np.zeros(nrows + 1, dtype=np.uint64)
    for r, b in enumerate(bands):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        if b.nrows != r1 - r0:
            raise ValueError(f"band {r} has {b.nrows} rows, expected {r1 - r0}")
        rowptr[r0:r1] = b.rowptr[:-1] + off[r]
    rowptr[nrows] = off[-1]
    colids = np.concatenate([b.colids for b in bands]) if bands else np.zeros(0, np.uint32)
    values = np.concatenate([b.values for b in bands]) if bands else np.zeros(0, np.float64)
    return M.CsrMatrix(nrows, ncols, rowptr, colids.astype(np.uint32, copy=False),
                       values.astype(np.float64, copy=False))


def gather_bands(band: M.CsrMatrix, cuts: np.ndarray, ncols: int, group=None, device=None):
    """Rank 0 assembles the global CSR from every rank's band with
    point-to-point tensor transfers (no pickling): an all-gather of the G
    band nnz values gives every band its entry offset, then each rank r > 0
    sends its rowptr / colids / values straight into rank 0's global arrays
    at those offsets. ``device`` = where the transfer tensors live (CPU for
    gloo; the rank's CUDA device for NCCL). Returns (offset of this band,
    global CSR on rank 0 else None)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = device or torch.device("cpu")
    nnz = torch.tensor([band.nnz], dtype=torch.int64, device=dev)
    all_nnz = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(all_nnz, nnz, group=group)
    off = band_offsets([int(t.item()) for t in all_nnz])
    t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x).view(dt)).to(dev)  # noqa: E731
    if rank != 0:
        # band-local rowptr shifted to global entry offsets on the sender
        rp = t(band.rowptr[:-1].astype(np.uint64) + off[rank], np.int64)
        for x in (rp, t(band.colids, np.int32), t(band.values, np.float64)):
            if x.numel():
                dist.send(x, 0, group=group)
        return int(off[rank]), None
    nrows = int(cuts[-1])
    rowptr = torch.empty(nrows + 1, dtype=torch.int64, device=dev)
    colids = torch.empty(int(off[-1]), dtype=torch.int32, device=dev)
    values = torch.empty(int(off[-1]), dtype=torch.float64, device=dev)
    rowptr[int(cuts[0]):int(cuts[1])] = t(band.rowptr[:-1], np.int64)
    colids[:band.nnz] = t(band.colids, np.int32)
    values[:band.nnz] = t(band.values, np.float64)
    for r in range(1, world):
        r0, r1 = int(cuts[r]), int(cuts[r + 1])
        e0, e1 = int(off[r]), int(off[r + 1])
        for x in (rowptr[r0:r1], colids[e0:e1], values[e0:e1]):
            if x.numel():
                buf = torch.empty_like(x)
                dist.recv(buf, r, group=group)
                x.copy_(buf)
    rowptr[nrows] = int(off[-1])
    full = M.CsrMatrix(nrows, ncols, rowptr.cpu().numpy().view(np.uint64),
                       colids.cpu().numpy().view(np.uint32), values.cpu().numpy())
    return 0, full


def distributed_multiply(a_csc: M.CscMatrix, b_csr: M.CsrMatrix, multiply_fn, group=None,
                         gather_to_root: bool = True, device=None):
    """Row-band C = A·B over a torch.distributed group.

    ``multiply_fn(a_slab_csc, b_csr) -> CsrMatrix`` computes one band (the GPU
    path on a B200 rank; any CPU stand-in in the gloo tests). Every rank
    returns (band CSR, global entry offset of the band, cuts); with
    ``gather_to_root`` rank 0 additionally returns the assembled global CSR
    (gather_bands: tensor point-to-point, no pickles).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cuts = plan_bands(a_csc, b_csr, world)
    band = multiply_fn(band_slab(a_csc, cuts, rank), b_csr)
    if gather_to_root:
        off, full = gather_bands(band, cuts, b_csr.ncols, group, device)
    else:
        import torch
        nnz = torch.tensor([band.nnz], dtype=torch.int64)
        all_nnz = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(all_nnz, nnz, group=group)
        off, full = int(band_offsets([int(x.item()) for x in all_nnz])[rank]), None
    return band, off, cuts, full
