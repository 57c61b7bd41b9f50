"""ctypes binding of the C-ABI library ``libsamegibbs_b200.so``.

This is the whole Python<->CUDA boundary: plain pointers, sizes and a
``cudaStream_t`` (``torch.cuda.current_stream().cuda_stream``) go in, an
``sg_status`` comes out.  The structures mirror ``include/samegibbs_b200.h``
field for field.  There is no fallback: if the library is missing or the
machine has no CUDA device, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int32, c_int64, c_uint64, c_void_p
from pathlib import Path

from .errors import DeviceError

# SAMEGIBBS_LIB overrides the in-tree library (variant builds for kernel A/B runs)
LIB_PATH = Path(os.environ.get("SAMEGIBBS_LIB") or Path(__file__).resolve().parent / "libsamegibbs_b200.so")

SG_OK, SG_EINVAL, SG_ECUDA, SG_ECAPACITY = 0, 1, 2, 3
SG_ERR_ZERO_SUPPORT, SG_ERR_STATE_RANGE, SG_ERR_REJECT_OVERFLOW = 1, 2, 4
SG_RNG_FAST, SG_RNG_NUMPY, SG_RNG_INJECTED = 0, 1, 2
SG_ACC_MOVING, SG_ACC_EXPONENTIAL = 0, 1
SG_FINISH_PACKED_ONLY = 1
ABI_VERSION = 2  # include/samegibbs_b200.h SG_ABI_VERSION
SG_OBS_PREFETCH_ONLY = 0x100  # sg_joint_sweep obs_bits flag
TALLY_CHUNK_CELLS = 12288
REJ_SLACK = 64

NET_POINTERS = (
    "card", "group_start", "order", "par_start", "par_var", "par_stride", "par_slot",
    "mb_start", "mb_var", "mb_stride", "chl_start", "chl_var", "chl_vstride", "chl_slot",
    "chl_pstart", "chl_pslot", "chl_pstride", "cpt_off", "row_off", "tab_entries",
    "tab_start", "ptab_off", "ftab_off", "row_var",
)


NET_POINTERS_TAIL = ("joint_radix", "joint_cell", "var_desc", "fac_start", "fac_desc")


class SgNet(ctypes.Structure):
    _fields_ = [
        ("n", c_int32), ("num_groups", c_int32), ("max_card", c_int32), ("max_mb", c_int32),
        ("max_group", c_int32), ("direct_vars", c_int32),
        ("cells", c_int64), ("rows", c_int64), ("ptab_size", c_int64), ("ftab_size", c_int64),
        ("table_entries", c_int64),
    ] + [(name, c_void_p) for name in NET_POINTERS] + [("joint_size", c_int64)] + \
        [(name, c_void_p) for name in NET_POINTERS_TAIL] + \
        [("tally_chunks", c_int64), ("tally_chunk", c_void_p)] + \
        [("blob32", c_void_p), ("blob32_words", c_int64), ("blob64", c_void_p), ("blob64_words", c_int64)] + \
        [("bft_rows", c_int64), ("bft_start", c_void_p), ("bft_desc", c_void_p), ("bft_src", c_void_p),
         ("bft", c_void_p)]


class SgBatch(ctypes.Structure):
    _fields_ = [
        ("states", c_void_p), ("m", c_int32), ("cases", c_int32), ("pitch", c_int32),
        ("num_real", c_int32), ("case_base", c_int64), ("rank", c_void_p), ("ld_rank", c_int32),
        ("latent_permille", c_int32), ("nmiss", c_void_p),
    ]


SMALL_MAXV = 7
SMALL_MAXBITS = 7


class SgSmall(ctypes.Structure):
    _fields_ = [("n", c_int32), ("bits", c_int32), ("tab_words", c_int32), ("pad_", c_int32)] + \
        [(name, ctypes.c_int32 * SMALL_MAXV) for name in ("order", "off", "width")] + \
        [("mbmask", ctypes.c_uint32 * SMALL_MAXV)] + \
        [(name, ctypes.c_int32 * SMALL_MAXV) for name in ("card", "toff", "tstride")]


class SgJoint(ctypes.Structure):
    _fields_ = [("words", c_int32), ("header_words", c_int32), ("patterns", c_int32), ("max_b", c_int32)]


class SgFinish(ctypes.Structure):
    _fields_ = [
        ("acc_mode", c_int32), ("map_estimate", c_int32), ("decay", c_double),
        ("total", c_void_p), ("new_counts", c_void_p), ("prev_counts", c_void_p), ("alpha", c_void_p),
        ("key", c_uint64), ("key_dev", c_void_p), ("cpt", c_void_p), ("ptab", c_void_p), ("ftab", c_void_p),
        ("stab", c_void_p), ("clear_counts", c_void_p), ("key_table", c_void_p), ("key_index", c_void_p),
        ("kps", c_int32), ("flags", c_int32), ("key_current", c_void_p), ("vprob", c_void_p),
        ("cpt_host", c_void_p), ("check_obs", c_void_p), ("check_ld", c_int32), ("check_bits", c_int32),
        ("check_cases", c_int32), ("check_err", c_void_p),
    ]


_SIGNATURES = {
    "sg_abi_version": ([], c_int32),
    "sg_last_error": ([], ctypes.c_char_p),
    "sg_build_tables": ([POINTER(SgNet), c_void_p, c_void_p, c_void_p, c_void_p], c_int32),
    "sg_rank_latent": ([c_int32, c_void_p, c_int32, c_int32, c_void_p, c_int32, c_void_p, c_void_p,
                        c_void_p], c_int32),
    "sg_init_states": ([POINTER(SgNet), POINTER(SgBatch), c_void_p, c_int32, c_int32, c_uint64, c_void_p,
                        c_void_p, c_void_p, c_void_p], c_int32),
    "sg_sweep": ([POINTER(SgNet), POINTER(SgBatch), c_void_p, c_void_p, c_void_p, c_int32, c_uint64,
                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p], c_int32),
    "sg_tally": ([POINTER(SgNet), POINTER(SgBatch), c_void_p, c_void_p], c_int32),
    "sg_tally_weighted": ([POINTER(SgNet), POINTER(SgBatch), c_void_p, c_void_p, c_void_p], c_int32),
    "sg_accumulate": ([c_int32, c_void_p, c_void_p, c_void_p, c_double, c_int64, c_void_p], c_int32),
    "sg_accumulate_f64": ([c_int32, c_void_p, c_void_p, c_void_p, c_double, c_int64, c_void_p], c_int32),
    "sg_mean_cpts": ([POINTER(SgNet), c_void_p, c_void_p, c_void_p, c_void_p], c_int32),
    "sg_sample_cpts": ([POINTER(SgNet), c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, c_void_p], c_int32),
    "sg_forward_sample": ([POINTER(SgNet), c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64,
                           c_double, c_uint64, c_uint64, c_void_p], c_int32),
    "sg_check_range": ([POINTER(SgNet), c_void_p, c_int32, c_int32, c_void_p, c_void_p], c_int32),
    "sg_site_keys": ([c_void_p, ctypes.c_char_p, c_int32, c_int64, c_int32, c_void_p, c_void_p], c_int32),
    "sg_site_key_host": ([ctypes.c_char_p, c_int32, c_void_p], c_int32),
    "sg_predict_tally": ([c_void_p, c_int64, c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p],
                         c_int32),
    "sg_small_tables": ([POINTER(SgNet), POINTER(SgSmall), c_void_p, c_void_p, c_void_p], c_int32),
    "sg_small_prepare": ([POINTER(SgSmall), c_void_p, c_int32, c_int32, c_int32, c_int64, c_uint64, c_int32,
                          c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p], c_int32),
    "sg_small_sweep": ([POINTER(SgSmall), c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32,
                        c_int32, c_int64, c_uint64, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p,
                        c_int32, c_void_p, c_void_p], c_int32),
    "sg_joint_tables": ([POINTER(SgNet), POINTER(SgSmall), POINTER(SgJoint), c_void_p, c_void_p, c_void_p, c_void_p],
                        c_int32),
    "sg_step_tail_joint": ([POINTER(SgNet), POINTER(SgSmall), POINTER(SgFinish), POINTER(SgJoint), c_void_p,
                            c_void_p, c_void_p, c_void_p], c_int32),
    "sg_joint_prep_bytes": ([POINTER(SgSmall), POINTER(SgJoint), POINTER(ctypes.c_int64)], c_int32),
    "sg_joint_prep": ([POINTER(SgNet), POINTER(SgSmall), POINTER(SgJoint), c_void_p, c_void_p, c_void_p], c_int32),
    "sg_joint_smem": ([POINTER(SgSmall), POINTER(SgJoint), c_int32, POINTER(ctypes.c_int64)], c_int32),
    "sg_joint_sweep": ([POINTER(SgSmall), POINTER(SgJoint), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                        c_int32, c_int32, c_int32, c_int32, c_int64, c_uint64, c_void_p, c_void_p, c_int32,
                        c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p], c_int32),
    "sg_keys_advance": ([c_void_p, c_void_p, c_int32, c_void_p, c_void_p], c_int32),
    "sg_copy_async": ([c_void_p, c_void_p, c_int64, c_void_p], c_int32),
    "sg_copy2d_async": ([c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_void_p], c_int32),
    "sg_copy_small": ([c_void_p, c_void_p, c_int64, c_void_p], c_int32),
    "sg_event_create": ([POINTER(c_uint64)], c_int32),
    "sg_event_record": ([c_uint64, c_void_p], c_int32),
    "sg_event_elapsed": ([c_uint64, c_uint64, POINTER(ctypes.c_float)], c_int32),
    "sg_event_destroy": ([c_uint64], c_int32),
    "sg_noop": ([c_int32, c_int32, c_int32, c_void_p], c_int32),
    "sg_flush_l2": ([c_void_p, c_void_p, c_int64, ctypes.c_uint32, c_void_p], c_int32),
    "sg_np_uniforms": ([POINTER(SgBatch), c_void_p, c_int32, c_void_p, c_int64, c_void_p], c_int32),
    "sg_step_finish": ([POINTER(SgNet), c_void_p, POINTER(SgFinish), c_void_p], c_int32),
    "sg_unpack_nibbles": ([c_void_p, c_int64, c_void_p, c_int64, c_int32, c_int64, c_void_p], c_int32),
    "sg_unpack_crumbs": ([c_void_p, c_int64, c_void_p, c_int64, c_int32, c_int64, c_void_p], c_int32),
    "sg_small_import": ([POINTER(SgSmall), POINTER(SgBatch), c_void_p, c_void_p, c_int32, c_void_p], c_int32),
    "sg_small_export": ([POINTER(SgSmall), POINTER(SgBatch), c_void_p, c_void_p, c_void_p, c_int32, c_void_p],
                        c_int32),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load(path: Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the library; raises DeviceError when it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise DeviceError(
            f"CUDA library {p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.sg_abi_version() != ABI_VERSION:
        raise DeviceError("libsamegibbs_b200 ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


# Checked builds (-DSG_CHECKED, lib_checked.so): each translation unit with
# device-side index / protocol assertions exports sg_debug_checked_<tu>, which
# reports (and clears) the first failing source line of that unit.
CHECKED_LIB_PATH = Path(__file__).resolve().parent / "lib_checked.so"
CHECKED_UNITS = ("aux", "big", "small", "sweep")


def checked_lines(lib: ctypes.CDLL | None = None, probe: bool = False) -> dict[str, int]:
    """{unit: first failing SG_DCHECK line (0 = none)} of a checked build; clears
    the words.  ``probe`` first launches a kernel whose check fails on purpose."""
    lib = lib or load()
    out = {}
    for tu in CHECKED_UNITS:
        fn = getattr(lib, f"sg_debug_checked_{tu}", None)
        if fn is None:
            raise DeviceError(f"{LIB_PATH} is not a checked build (no sg_debug_checked_{tu})")
        fn.argtypes = [POINTER(ctypes.c_uint32), c_int32]
        fn.restype = c_int32
        line = ctypes.c_uint32(0)
        if fn(ctypes.byref(line), int(probe)) != SG_OK:
            raise DeviceError(f"sg_debug_checked_{tu} failed: {lib.sg_last_error().decode(errors='replace')}")
        out[tu] = int(line.value)
    return out


def check(status: int, what: str) -> None:
    if status != SG_OK:
        msg = load().sg_last_error().decode(errors="replace")
        raise DeviceError(f"{what} failed with status {status}: {msg}")


# kernels each entry point launches (for the bench's gpu_launches count)
KERNELS_PER_CALL = {
    "sg_build_tables": 1, "sg_rank_latent": 3, "sg_init_states": 1, "sg_sweep": 1, "sg_tally": 1,
    "sg_tally_weighted": 1, "sg_accumulate": 1, "sg_accumulate_f64": 1, "sg_mean_cpts": 1,
    "sg_sample_cpts": 1, "sg_forward_sample": 1, "sg_check_range": 1, "sg_np_uniforms": 1,
    "sg_small_tables": 1, "sg_small_prepare": 3, "sg_small_sweep": 1, "sg_small_import": 1, "sg_small_export": 1,
    "sg_joint_tables": 1, "sg_joint_sweep": 1, "sg_step_tail_joint": 1, "sg_joint_prep": 1, "sg_copy_small": 1, "sg_noop": 1,
    "sg_keys_advance": 1, "sg_copy2d_async": 1, "sg_step_finish": 1, "sg_site_keys": 1, "sg_predict_tally": 1, "sg_unpack_nibbles": 1, "sg_unpack_crumbs": 1,
}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    check(getattr(load(), name)(*args), name)
    launch_count += KERNELS_PER_CALL.get(name, 0)
