"""ctypes bindings of the in-tree native libraries.

``libpbg.so`` (the sm_100a PB-SpGEMM path behind include/pbg.h) and
``libpbg_host.so`` (host input preparation, include/pbg_host.h). Loading is
lazy and fails loudly: there is no CPU fallback for the product path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent

u32, u64, i32, f64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_double
P = C.POINTER
vp = C.c_void_p

# error codes (include/pbg.h)
PBG_OK = 0
PBG_ERR_DIM = 1
PBG_ERR_NBINS = 2
PBG_ERR_LBIN = 3
PBG_ERR_FLOP_OVERFLOW = 4
PBG_ERR_INTERNAL = 5
PBG_ERR_CUDA = 6
PBG_ERR_OOM = 7
PBG_ERR_NCCL = 8
PBG_ERR_ARG = 9
PBG_ERR_UNIMPLEMENTED = 10
PBG_ERR_NODEVICE = 11


class CsxView(C.Structure):
    _fields_ = [("nrows", u32), ("ncols", u32), ("nnz", u64),
                ("ptr", vp), ("idx", vp), ("val", vp)]


class Config(C.Structure):
    _fields_ = [("nbins", u32), ("lbin_bytes", u32), ("l2_bytes", u64),
                ("nthreads", i32), ("balanced_bins", i32), ("device", i32),
                ("bin_cap", u32), ("ngpus", i32), ("flags", u32), ("reserved", u64 * 4)]


PBG_FLAG_WRAP_DEVICES = 1


class Report(C.Structure):
    _fields_ = [("t_symbolic", f64), ("t_expand", f64), ("t_sort", f64),
                ("t_compress", f64), ("t_convert", f64), ("t_total", f64),
                ("t_h2d", f64), ("t_d2h", f64),
                ("flop", u64), ("nnz_c", u64), ("nnz_a", u64), ("nnz_b", u64),
                ("tuples_into_sort", u64), ("merged_total", u64),
                ("nbins", u32), ("gpu_bins", u32), ("heavy_bins", u32), ("bin_cap", u32),
                ("tuple_bytes", u64), ("sort_fallbacks", u64),
                ("expand_bands", u32), ("pad0", u32),
                ("t_count", f64), ("t_sortmerge_kernel", f64),
                ("ngpus", u32), ("nrounds", u32), ("t_device_max", f64), ("t_device_min", f64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


PBG_EXPORTS = {
    "pbg_last_error": (C.c_char_p, []),
    "pbg_default_config": (None, [P(Config)]),
    "pbg_device_available": (C.c_int, []),
    "pbg_multiply_begin": (C.c_int, [P(CsxView), P(CsxView), P(Config), P(vp), P(u64)]),
    "pbg_multiply_fetch": (C.c_int, [vp, vp, vp, vp, P(Report)]),
    "pbg_multiply_into": (C.c_int, [P(CsxView), P(CsxView), P(Config), vp, vp, vp, u64, P(u64),
                                    P(Report)]),
    "pbg_generate_begin": (C.c_int, [C.c_int, C.c_int, u32, u64, u64, C.c_int, P(Config), P(vp),
                                     P(u64)]),
    "pbg_hash_multiply_begin": (C.c_int, [P(CsxView), P(CsxView), P(Config), P(vp), P(u64)]),
    "pbg_coo_convert_begin": (C.c_int, [u32, u32, u64, vp, vp, vp, C.c_int, P(Config), P(vp),
                                        P(u64)]),
    "pbg_symbolic_fetch": (C.c_int, [vp, vp, vp, vp]),
    "pbg_release": (None, [vp]),
    "pbg_context_create": (C.c_int, [C.c_int, P(vp)]),
    "pbg_context_destroy": (None, [vp]),
    "pbg_multiply_device": (C.c_int, [vp, P(CsxView), P(CsxView), P(Config), vp, P(u64), P(Report)]),
    "pbg_context_result": (C.c_int, [vp, P(vp), P(vp), P(vp)]),
    "pbg_context_symbolic": (C.c_int, [vp, P(Config), vp, vp, vp]),
    "pbg_context_launches": (u32, [vp]),
    "pbg_band_cuts_device": (C.c_int, [vp, P(CsxView), P(CsxView), u32, u32, u32, vp, vp, P(u64)]),
    "pbg_row_slab_device": (C.c_int, [vp, P(CsxView), u32, u32, vp, vp, vp, vp, u64, P(u64)]),
    "pbg_multiply_device_band": (C.c_int, [vp, P(CsxView), P(CsxView), u32, u32, P(Config), vp,
                                           P(u64), P(Report)]),
    "pbg_context_checksum": (C.c_int, [vp, u64, vp, vp, P(f64)]),
    "pbg_context_workbins": (C.c_int, [vp, u64, vp, vp, vp, vp, vp]),
    "pbg_choose_nbins": (u32, [u64, u32, u64, u32]),
}

HOST_EXPORTS = {
    "pbgh_split_seed": (u64, [u64, u64]),
    "pbgh_gen_er": (C.c_int, [C.c_int, u32, u64, vp, vp]),
    "pbgh_gen_rmat": (C.c_int, [C.c_int, u32, u64, f64, f64, f64, vp, vp]),
    "pbgh_coo_to_csr": (C.c_int, [u32, u32, u64, vp, vp, vp, C.c_int, C.c_int, vp, vp, vp, P(u64)]),
    "pbgh_csr_to_csc": (C.c_int, [u32, u32, vp, vp, vp, vp, vp, vp]),
    "pbgh_csr_fill_values": (C.c_int, [u64, u32, vp, vp, vp]),
    "pbgh_stencil27": (C.c_int, [u32, u32, u32, vp, vp, vp, P(u64)]),
    "pbgh_csc_row_band": (C.c_int, [u32, u32, vp, vp, vp, u32, u32, vp, vp, vp, P(u64)]),
    "pbgh_row_flop": (C.c_int, [u32, u32, vp, vp, vp, vp]),
    "pbgh_band_cuts": (C.c_int, [u32, vp, u32, vp]),
    "pbgh_mm_open": (C.c_int, [C.c_char_p, P(vp), P(u32), P(u32), P(u64)]),
    "pbgh_mm_fetch": (C.c_int, [vp, vp, vp, vp]),
    "pbgh_mm_free": (None, [vp]),
    "pbgh_mm_write": (C.c_int, [C.c_char_p, u32, u32, u64, vp, vp, vp]),
    "pbgh_last_error": (C.c_char_p, []),
}

_libs: dict = {}


def _load(name: str, exports: dict):
    if name in _libs:
        return _libs[name]
    path = PKG / name
    if not path.exists():
        raise RuntimeError(
            f"native library {path} is missing — run `python -m paper_2002_11302_b200.build` "
            "(there is no CPU fallback for the GPU path)")
    lib = C.CDLL(str(path))
    for sym, (res, args) in exports.items():
        fn = getattr(lib, sym)
        fn.restype = res
        fn.argtypes = args
    _libs[name] = lib
    return lib


def pbg():
    """libpbg.so: the sm_100a PB-SpGEMM kernels behind the C-ABI
    (PBG_LIB=<name> selects an in-tree variant build, e.g. for A/B tuning)."""
    import os
    return _load(os.environ.get("PBG_LIB", "libpbg.so"), PBG_EXPORTS)


def host():
    """libpbg_host.so: host input preparation (generators, conversions)."""
    return _load("libpbg_host.so", HOST_EXPORTS)


def last_error() -> str:
    msg = pbg().pbg_last_error()
    return msg.decode() if msg else ""
