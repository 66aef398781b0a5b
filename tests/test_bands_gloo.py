"""Multi-GPU row-band partitioning, host side, on CPU with gloo (world 2).

Each rank takes its flop-balanced CSC row-slab of A, multiplies it by all of
B (here with the CPU oracle standing in for its GPU), exchanges band nnz with
an all-gather, and rank 0 assembles the global CSR — which must equal the
single-process product: rowptr/colids bit-exact, values within 1e-12 (the
reference's unstable in-bin radix sort orders duplicates by bin contents, so
a band's different bin layout may change the last bits).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2002_11302_b200 import bands, matrices as M

from helpers import assert_values_close


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_band(a_slab, b):
    r = oracle.multiply(a_slab, b, nbins=1)
    return M.CsrMatrix(a_slab.nrows, b.ncols, r.rowptr, r.colids, r.values)


def _worker(rank, world, port, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        csr = M.make_matrix(kind, 9, 8, seed=4)
        csc = M.csr_to_csc(csr)
        band, off, cuts, full = bands.distributed_multiply(csc, csr, _oracle_band)
        q.put((rank, off, band.nnz, cuts.tolist(),
               None if full is None else (full.rowptr, full.colids, full.values)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["er", "rmat"])
def test_two_rank_bands_equal_single_product(kind):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    csr = M.make_matrix(kind, 9, 8, seed=4)
    ref = oracle.multiply(M.csr_to_csc(csr), csr, nbins=1)
    # offsets: rank 1 starts where rank 0's entries end
    assert got[0][1] == 0 and got[1][1] == got[0][2]
    assert got[0][3] == got[1][3]  # both ranks computed the same cuts
    rowptr, colids, values = got[0][4]
    assert np.array_equal(rowptr, ref.rowptr)
    assert np.array_equal(colids, ref.colids)
    assert_values_close(values, ref.values)


def test_assemble_rejects_wrong_band_shape():
    csr = M.make_matrix("er", 6, 3, seed=1)
    cuts = np.array([0, 10, 64], dtype=np.uint32)
    b0 = M.CsrMatrix(9, 64, np.zeros(10, np.uint64), np.zeros(0, np.uint32), np.zeros(0))
    b1 = M.CsrMatrix(54, 64, np.zeros(55, np.uint64), np.zeros(0, np.uint32), np.zeros(0))
    with pytest.raises(ValueError):
        bands.assemble([b0, b1], cuts, csr.ncols)
