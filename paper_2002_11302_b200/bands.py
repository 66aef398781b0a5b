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


def distributed_multiply(a_csc: M.CscMatrix, b_csr: M.CsrMatrix, multiply_fn, group=None,
                         gather_to_root: bool = True):
    """Row-band C = A·B over a torch.distributed group.

    ``multiply_fn(a_slab_csc, b_csr) -> CsrMatrix`` computes one band (the GPU
    path on a B200 rank; any CPU stand-in in the gloo tests). Every rank
    returns (band CSR, global entry offset of the band, cuts); with
    ``gather_to_root`` rank 0 additionally returns the assembled global CSR.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cuts = plan_bands(a_csc, b_csr, world)
    band = multiply_fn(band_slab(a_csc, cuts, rank), b_csr)
    nnz = torch.tensor([band.nnz], dtype=torch.int64)
    all_nnz = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(all_nnz, nnz, group=group)
    off = band_offsets([int(t.item()) for t in all_nnz])
    full = None
    if gather_to_root:
        objs = [None] * world if rank == 0 else None
        dist.gather_object((band.rowptr, band.colids, band.values), objs, dst=0, group=group)
        if rank == 0:
            bands = [M.CsrMatrix(int(cuts[r + 1] - cuts[r]), b_csr.ncols, *objs[r])
                     for r in range(world)]
            full = assemble(bands, cuts, b_csr.ncols)
    return band, int(off[rank]), cuts, full
