"""Row bands on the GPU: the multi-device host path, the
bounded-memory rounds with device-side cuts and slabs, the one-call
pbg_multiply_into, and the device-resident band API the benchmark times.

Every product is compared with the single-pass product (rowptr / colids
bit-exact, values within 1e-12: a band's bins differ from the full product's,
so duplicates may be summed in another order) or with the reference's own
band products (oracle/_ref).
"""
import ctypes
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2002_11302_b200 import api, bands, matrices as M

from helpers import assert_csr_matches, assert_values_close

pytestmark = pytest.mark.gpu


def gpu(a, b, **kw):
    return api.pb_multiply(a, b, api.PbConfig(device=0, **kw))


def _cases():
    out = []
    for kind, scale, ef, seed in (("er", 13, 8, 3), ("rmat", 12, 8, 9)):
        csr = M.make_matrix(kind, scale, ef, seed=seed)
        out.append((kind, M.csr_to_csc(csr), csr))
    return out


def _same(r, one):
    assert_csr_matches(r.c.rowptr, r.c.colids, r.c.values, one.c.rowptr, one.c.colids,
                       one.c.values)


@pytest.mark.parametrize("ngpus", [2, 3])
def test_multi_device_host_path_matches_single(ngpus):
    """cfg.ngpus > 1: one flop-balanced band per device (here wrapped onto
    the one GPU, one context per band), assembled in the caller's arrays."""
    for kind, a, b in _cases():
        one = gpu(a, b)
        r = gpu(a, b, ngpus=ngpus, wrap_devices=True)
        _same(r, one)
        assert r.report["ngpus"] == ngpus
        assert r.tuples_into_sort == one.sym.flop and r.merged_total == one.c.nnz
        assert r.sym.flop == one.sym.flop and r.sym.nbins == one.sym.nbins
        assert np.array_equal(r.sym.per_column_flop, one.sym.per_column_flop)
        assert np.array_equal(r.sym.per_bin_flop, one.sym.per_bin_flop)
        assert np.array_equal(r.sym.bin_row_starts, one.sym.bin_row_starts)
        # several devices and rounds on each
        rr = gpu(a, b, ngpus=ngpus, wrap_devices=True, max_round_tuples=max(one.sym.flop // 7, 1))
        _same(rr, one)
        assert rr.report["nrounds"] >= 2


def test_ngpus_above_device_count_is_an_error():
    import torch
    a, b = _cases()[0][1:]
    with pytest.raises(api.DeviceError):
        gpu(a, b, ngpus=torch.cuda.device_count() + 1)


@pytest.mark.parametrize("pinned", [False, True])
def test_multiply_into_caller_arrays(pinned):
    """pbg_multiply_into: C written straight into the caller's arrays, in
    rounds whose copies overlap the next round (forced by max_round_tuples)."""
    import torch
    for kind, a, b in _cases():
        one = gpu(a, b)
        k = one.c.nnz

        def arr(n, dt, tdt):
            if pinned:
                return torch.empty(n, dtype=tdt).pin_memory().numpy().view(dt)
            return np.empty(n, dt)
        for mrt in (0, max(one.sym.flop // 6, 1)):
            out = (arr(a.nrows + 1, np.uint64, torch.int64), arr(k + 5, np.uint32, torch.int32),
                   arr(k + 5, np.float64, torch.float64))
            r = api.pb_multiply(a, b, api.PbConfig(device=0, max_round_tuples=mrt), out=out)
            _same(r, one)
            if mrt:
                assert r.report["nrounds"] >= 6
        small = (np.empty(a.nrows + 1, np.uint64), np.empty(k // 2, np.uint32),
                 np.empty(k // 2, np.float64))
        with pytest.raises(api.DeviceError):
            api.pb_multiply(a, b, api.PbConfig(device=0, max_round_tuples=max(one.sym.flop // 4, 1)),
                            out=small)


def _upload(a, b):
    import torch
    dev = torch.device("cuda", 0)
    t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x).view(dt)).to(dev)  # noqa: E731
    A = (t(a.colptr, np.int64), t(a.rowids, np.int32), t(a.values, np.float64))
    B = (t(b.rowptr, np.int64), t(b.colids, np.int32), t(b.values, np.float64))
    return A, B


def _download(ctx, nrows, nnz, rows=None):
    """The context's product (or rows [r0, r1) of it) to host arrays."""
    rp, ci, va = ctx.result_pointers()
    cudart = ctypes.CDLL("libcudart.so.12")
    r0, r1 = rows or (0, nrows)
    rowptr = np.empty(r1 - r0 + 1, np.uint64)
    assert cudart.cudaMemcpy(ctypes.c_void_p(rowptr.ctypes.data), ctypes.c_void_p(rp + 8 * r0),
                             ctypes.c_size_t(rowptr.nbytes), 2) == 0
    lo, hi = int(rowptr[0]), int(rowptr[-1])
    colids = np.empty(hi - lo, np.uint32)
    values = np.empty(hi - lo, np.float64)
    if hi > lo:
        assert cudart.cudaMemcpy(ctypes.c_void_p(colids.ctypes.data), ctypes.c_void_p(ci + 4 * lo),
                                 ctypes.c_size_t(colids.nbytes), 2) == 0
        assert cudart.cudaMemcpy(ctypes.c_void_p(values.ctypes.data), ctypes.c_void_p(va + 8 * lo),
                                 ctypes.c_size_t(values.nbytes), 2) == 0
    return rowptr - lo, colids, values


def test_device_band_cuts_follow_the_host_rule_and_bands_assemble():
    for kind, a, b in _cases():
        A, B = _upload(a, b)
        ctx = api.DeviceContext(0)
        va = ctx.view(a.nrows, a.ncols, *A)
        vb = ctx.view(b.nrows, b.ncols, *B)
        rf = M.row_flop(a, b)
        one = gpu(a, b)
        nnz_full, _ = ctx.multiply(va, vb)
        full_ck = ctx.checksum()
        for g in (1, 2, 3, 7):
            cuts, flop = ctx.band_cuts(va, vb, g)
            assert flop == int(rf.sum())
            assert np.array_equal(cuts, M.band_cuts(rf, g))  # balanced_starts rule
            parts, ck = [], [0, 0, 0, 0.0]
            for r in range(g):
                r0, r1 = int(cuts[r]), int(cuts[r + 1])
                nnz, rep = ctx.multiply_band(va, vb, r0, r1)
                assert rep["flop"] == int(rf[r0:r1].sum())
                c = ctx.checksum(row_base=r0)
                ck = [ck[0] + c[0], (ck[1] + c[1]) % 2**64, (ck[2] + c[2]) % 2**64, ck[3] + c[3]]
                rp, ci, vv = _download(ctx, r1 - r0, nnz)
                parts.append(M.CsrMatrix(r1 - r0, b.ncols, rp, ci, vv))
            asm = bands.assemble(parts, cuts, b.ncols)
            assert_csr_matches(asm.rowptr, asm.colids, asm.values, one.c.rowptr, one.c.colids,
                               one.c.values)
            # checksums are sums: the bands add up to the whole product's
            assert ck[:3] == list(full_ck[:3]) and ck[0] == nnz_full
            assert abs(ck[3] - full_ck[3]) <= 1e-9 * abs(full_ck[3])


def test_device_row_slab_equals_host_row_band():
    """pbg_row_slab_device (selection bits, word scan, lookups, stable gather)
    against the host's row band, entry for entry: RMAT hub columns, an empty
    band, single rows, the whole matrix, nnz not a multiple of 32."""
    rng = np.random.default_rng(11)
    for kind, scale, ef in (("rmat", 12, 9), ("er", 10, 5)):
        csr = M.make_matrix(kind, scale, ef, seed=7)
        a = M.csr_to_csc(csr)
        A, _ = _upload(a, csr)
        ctx = api.DeviceContext(0)
        va = ctx.view(a.nrows, a.ncols, *A)
        n = a.nrows
        cuts = [(0, n), (0, 0), (n, n), (5, 6), (n - 1, n), (0, n // 3), (n // 3, n - 7)]
        cuts += [tuple(sorted(int(x) for x in rng.integers(0, n + 1, 2))) for _ in range(6)]
        for r0, r1 in cuts:
            (cp, ri, vv), _view = ctx.row_slab(va, r0, r1)
            ref = M.row_band(a, r0, r1)
            assert np.array_equal(cp.cpu().numpy().astype(np.uint64), ref.colptr), (kind, r0, r1)
            assert np.array_equal(ri.cpu().numpy().astype(np.uint32), ref.rowids), (kind, r0, r1)
            assert np.array_equal(vv.cpu().numpy(), ref.values), (kind, r0, r1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        csr = M.make_matrix("rmat", 12, 8, seed=9)
        csc = M.csr_to_csc(csr)
        A, B = _upload(csc, csr)
        ctx = api.DeviceContext(0)
        va = ctx.view(csc.nrows, csc.ncols, *A)
        vb = ctx.view(csr.nrows, csr.ncols, *B)
        cuts, _ = ctx.band_cuts(va, vb, world)  # every rank computes the same cuts
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        nnz, _ = ctx.multiply_band(va, vb, r0, r1)
        rp, ci, vv = _download(ctx, r1 - r0, nnz)
        band = M.CsrMatrix(r1 - r0, csr.ncols, rp, ci, vv)
        off, full = bands.gather_bands(band, cuts, csr.ncols)
        torch.cuda.synchronize()
        q.put((rank, off, None if full is None else (full.rowptr, full.colids, full.values)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_assemble_the_single_product():
    """The benchmark's N > 1 flow with the real GPU multiply: two ranks (gloo,
    both on cuda:0; their kernels never wait on each other), device-side
    cuts, one band each, tensor gather to rank 0."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, off, full = q.get(timeout=600)
        got[r] = (off, full)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    csr = M.make_matrix("rmat", 12, 8, seed=9)
    one = gpu(M.csr_to_csc(csr), csr)
    rp, ci, vv = got[0][1]
    assert_csr_matches(rp, ci, vv, one.c.rowptr, one.c.colids, one.c.values)
    assert got[1][0] == int(one.c.rowptr[int(bands.plan_bands(M.csr_to_csc(csr), csr, 2)[1])])


def _rounds_parity(cfg_name, rounds, window, nwin):
    """SURVEY.md §8c band parity on the path bench.py times for configs whose
    tuples exceed one GPU: the whole config in `rounds` flop-balanced bands
    cut and sliced on the device (ctx.band_cuts + multiply_band over the full
    A), and from every round windows of `window` rows — at least `nwin` in
    all, the heaviest row's window always among them — compared with the
    reference's product of the same rows."""
    a, b = M.make_config_gpu(cfg_name)
    A, B = _upload(a, b)
    ctx = api.DeviceContext(0)
    va = ctx.view(a.nrows, a.ncols, *A)
    vb = ctx.view(b.nrows, b.ncols, *B)
    rf = M.row_flop(a, b)
    heavy = int(np.argmax(rf))
    cuts, flop = ctx.band_cuts(va, vb, rounds)
    assert flop == int(rf.sum())
    impl = "reference" if oracle.ref_available() else "port"
    rng = np.random.default_rng(11)
    per_round = max(1, -(-nwin // rounds))
    checked = 0
    tot_nnz = 0
    for q in range(rounds):
        r0, r1 = int(cuts[q]), int(cuts[q + 1])
        if r0 == r1:
            continue
        nnz, rep = ctx.multiply_band(va, vb, r0, r1)
        tot_nnz += nnz
        assert rep["tuples_into_sort"] == int(rf[r0:r1].sum()) and rep["merged_total"] == nnz
        w = min(window, r1 - r0)
        starts = {int(x) for x in rng.integers(r0, r1 - w + 1, per_round)}
        if r0 <= heavy < r1:
            starts.add(min(max(r0, heavy - w // 2), r1 - w))
        for s in sorted(starts):
            rp, ci, vv = _download(ctx, r1 - r0, nnz, rows=(s - r0, s - r0 + w))
            slab = M.row_band(a, s, s + w)
            ref = oracle.multiply(slab, b, impl=impl, nthreads=0 if impl == "reference" else 1,
                                  stepwise=False)
            assert np.array_equal(rp, ref.rowptr)
            assert np.array_equal(ci, ref.colids)
            assert_values_close(vv, ref.values)
            checked += 1
    assert checked >= nwin
    return tot_nnz


@pytest.mark.slow
def test_config_C3_rounds_parity():
    nnz = _rounds_parity("C3", 7, 256, 10)
    assert nnz == 9709074530


@pytest.mark.slow
def test_config_C5b_rounds_parity_sampled():
    # C5b's 2.8e11 mults: 95 rounds at full size; a leading flop-balanced
    # eighth of the rows (the band rank 0 of 8 takes) in 12 rounds
    a, b = M.make_config_gpu("C5b")
    A, B = _upload(a, b)
    ctx = api.DeviceContext(0)
    va = ctx.view(a.nrows, a.ncols, *A)
    vb = ctx.view(b.nrows, b.ncols, *B)
    cuts8, _ = ctx.band_cuts(va, vb, 8)
    rf = M.row_flop(a, b)
    heavy = int(np.argmax(rf))
    band = next(i for i in range(8) if cuts8[i] <= heavy < cuts8[i + 1])
    r0, r1 = int(cuts8[band]), int(cuts8[band + 1])
    sub = M.band_cuts(rf[r0:r1], 12) + r0
    impl = "reference" if oracle.ref_available() else "port"
    rng = np.random.default_rng(13)
    checked = 0
    for q in range(12):
        s0, s1 = int(sub[q]), int(sub[q + 1])
        if s0 == s1:
            continue
        nnz, rep = ctx.multiply_band(va, vb, s0, s1)
        assert rep["tuples_into_sort"] == int(rf[s0:s1].sum())
        w = min(64, s1 - s0)
        starts = {int(rng.integers(s0, s1 - w + 1))}
        if s0 <= heavy < s1:
            starts.add(min(max(s0, heavy - w // 2), s1 - w))
        for s in sorted(starts):
            rp, ci, vv = _download(ctx, s1 - s0, nnz, rows=(s - s0, s - s0 + w))
            ref = oracle.multiply(M.row_band(a, s, s + w), b, impl=impl,
                                  nthreads=0 if impl == "reference" else 1, stepwise=False)
            assert np.array_equal(rp, ref.rowptr) and np.array_equal(ci, ref.colids)
            assert_values_close(vv, ref.values)
            checked += 1
    assert checked >= 12
