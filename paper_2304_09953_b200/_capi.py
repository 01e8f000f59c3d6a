"""ctypes binding of the C-ABI in ``include/vscreen_gpu/capi.h``.

The shared object ``libvscreen_gpu.so`` is built in-tree (``build.py``).
There is no fallback: if it is missing or fails to load, importing this
module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VSCREEN_GPU_LIB") or os.path.join(_HERE, "libvscreen_gpu.so")

# status codes (capi.h vs_status)
VS_OK = 0
VS_ERR_INVALID_ARGUMENT = -1
VS_ERR_ATOM_COUNT = -2
VS_ERR_EMPTY_BOUNDS = -3
VS_ERR_LENGTH = -4
VS_ERR_OUT_OF_RANGE = -5
VS_ERR_ITEM_TOO_LARGE = -6
VS_ERR_POCKET = -7
VS_ERR_PARSE = -8
VS_ERR_CAPACITY = -9
VS_ERR_CUDA = -10
VS_ERR_NO_DEVICE = -11
VS_ERR_STATE = -12
VS_ERR_DISCONNECTED = -13
VS_ERR_FORMAT = -14

P = C.POINTER


class vs_site(C.Structure):
    _fields_ = [("center", C.c_double * 3), ("weight", C.c_double), ("sigma", C.c_double),
                ("kind", C.c_int32), ("reserved", C.c_int32)]


class vs_pocket(C.Structure):
    _fields_ = [("sites", P(vs_site)), ("n_sites", C.c_int32), ("reserved", C.c_int32),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("clash_radius", C.c_double),
                ("clash_penalty", C.c_double)]


class vs_library(C.Structure):
    _fields_ = [("n_ligands", C.c_int32), ("reserved", C.c_int32),
                ("n_atoms", P(C.c_int32)), ("n_tors", P(C.c_int32)), ("rot_bonds", P(C.c_int32)),
                ("coords", P(C.c_double)), ("atom_class", P(C.c_int32)),
                ("axis_a", P(C.c_int32)), ("axis_b", P(C.c_int32)),
                ("moving_count", P(C.c_int32)), ("moving", P(C.c_int32)),
                ("seeds", P(C.c_uint64)), ("id_rank", P(C.c_uint32))]


class vs_size_class(C.Structure):
    _fields_ = [("atom_lo", C.c_int32), ("atom_hi", C.c_int32), ("rot_lo", C.c_int32),
                ("rot_hi", C.c_int32)]


class vs_dock_params(C.Structure):
    _fields_ = [("restarts", C.c_int32), ("rotations", C.c_int32), ("flex_angles", C.c_int32),
                ("flex_passes", C.c_int32), ("diversity_delta", C.c_double),
                ("keep_top", C.c_int32), ("write_all_poses", C.c_int32),
                ("min_score", C.c_double), ("rotation_seed", C.c_uint64), ("polish", C.c_int32),
                ("reserved", C.c_int32)]


class vs_pose(C.Structure):
    _fields_ = [("t", C.c_float * 3), ("q", C.c_float * 4), ("score", C.c_float),
                ("rescore", C.c_float), ("restart", C.c_int16), ("attempt", C.c_int16),
                ("rot", C.c_int16), ("reserved", C.c_int16)]


class vs_results(C.Structure):
    _fields_ = [("best", P(C.c_float)), ("n_kept", P(C.c_int32)), ("n_surv", P(C.c_int32)),
                ("surv", C.c_void_p), ("surv_tors", P(C.c_float)), ("all", C.c_void_p),
                ("all_tors", P(C.c_float)), ("keys", P(C.c_uint64))]


class vs_refined(C.Structure):
    _fields_ = [("n_poses", P(C.c_int32)), ("t", P(C.c_double)), ("q", P(C.c_double)),
                ("tors", P(C.c_double)), ("score", P(C.c_double)), ("restart", P(C.c_int32))]


class vs_ligand_buf(C.Structure):
    _fields_ = [("cap_atoms", C.c_int32), ("cap_bonds", C.c_int32), ("cap_tors", C.c_int32),
                ("cap_moving", C.c_int32), ("n_atoms", C.c_int32), ("n_bonds", C.c_int32),
                ("n_tors", C.c_int32), ("n_moving", C.c_int32), ("rot_bonds", C.c_int32),
                ("parse_kind", C.c_int32), ("parse_pos", C.c_int32),
                ("coords", P(C.c_double)), ("atom_class", P(C.c_int32)), ("elements", C.c_char_p),
                ("aromatic", P(C.c_uint8)), ("bonds", P(C.c_int32)), ("ring", P(C.c_uint8)),
                ("axis_a", P(C.c_int32)), ("axis_b", P(C.c_int32)),
                ("moving_count", P(C.c_int32)), ("moving", P(C.c_int32))]


# function table: name -> (restype, argtypes)
_SIGS = {
    "vs_create": (C.c_int, [C.c_int, P(C.c_void_p)]),
    "vs_destroy": (None, [C.c_void_p]),
    "vs_last_error": (C.c_char_p, [C.c_void_p]),
    "vs_device_info": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_int32), P(C.c_int32)]),
    "vs_set_pocket": (C.c_int, [C.c_void_p, P(vs_pocket), C.c_double, C.c_double]),
    "vs_grid_info": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_float), P(C.c_float)]),
    "vs_grid_fetch": (C.c_int, [C.c_void_p, P(C.c_float), P(C.c_float), P(C.c_float)]),
    "vs_upload_library": (C.c_int, [C.c_void_p, P(vs_library), P(vs_size_class), C.c_int32]),
    "vs_dock": (C.c_int, [C.c_void_p, P(vs_dock_params), C.c_void_p]),
    "vs_fetch_results": (C.c_int, [C.c_void_p, P(vs_results)]),
    "vs_dock_host": (C.c_int, [C.c_void_p, P(vs_library), P(vs_size_class), C.c_int32,
                               P(vs_dock_params), P(vs_results)]),
    "vs_dock_host_prefetch": (C.c_int, [C.c_void_p, P(vs_library), P(vs_library),
                                        P(vs_size_class), C.c_int32, P(vs_dock_params),
                                        P(vs_results)]),
    "vs_last_dock_ms": (C.c_double, [C.c_void_p]),
    "vs_launch_count": (C.c_uint64, [C.c_void_p]),
    "vs_last_phase_ms": (C.c_int, [C.c_void_p, P(C.c_double)]),
    "vs_last_stats": (C.c_int, [C.c_void_p, P(C.c_uint64)]),
    "vs_last_stats_ex": (C.c_int, [C.c_void_p, P(C.c_uint64), C.c_int32]),
    "vs_measure_peaks": (C.c_int, [C.c_void_p, P(C.c_double), P(C.c_double), P(C.c_double)]),
    "vs_measure_gather_peak": (C.c_int, [C.c_void_p, P(C.c_double)]),
    "vs_measure_gather_peak_ex": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_double)]),
    "vs_last_phase_ms_ex": (C.c_int, [C.c_void_p, P(C.c_double), C.c_int32]),
    "vs_topk": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_uint64)]),
    "vs_topk_device": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "vs_topk_merge_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                       C.c_void_p, C.c_void_p]),
    "vs_nccl_unique_id": (C.c_int, [P(C.c_uint8)]),
    "vs_comm_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, P(C.c_uint8)]),
    "vs_comm_attach": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vs_comm_destroy": (None, [C.c_void_p]),
    "vs_topk_allgather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "vs_start_draws": (C.c_int, [C.c_void_p, P(C.c_uint64), P(C.c_int32), C.c_int32, C.c_int32,
                                 C.c_int32, C.c_int32, P(C.c_float)]),
    "vs_topk_merge_host": (C.c_int, [P(C.c_uint64), C.c_int64, C.c_int32, P(C.c_uint64)]),
    "vs_key_score": (C.c_float, [C.c_uint64]),
    "vs_key_id_rank": (C.c_uint32, [C.c_uint64]),
    "vs_score_gradient": (C.c_int, [C.c_void_p, P(vs_library), C.c_int64, P(C.c_int32),
                                    P(C.c_double), P(C.c_double), P(C.c_double),
                                    P(C.c_double), P(C.c_double), P(C.c_double),
                                    P(C.c_double)]),
    "vs_rescore": (C.c_int, [C.c_void_p, P(vs_library), C.c_int64, P(C.c_int32), P(C.c_float),
                             P(C.c_float), P(C.c_float), P(C.c_float), P(C.c_float)]),
    "vs_rescore_checked": (C.c_int, [C.c_void_p, P(vs_library), C.c_int64, P(C.c_int32),
                                     P(C.c_float), P(C.c_float), P(C.c_float), C.c_int64,
                                     P(C.c_float), P(C.c_float)]),
    "vs_last_rescore_ms": (C.c_double, [C.c_void_p]),
    "vs_rescore_device": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vs_rescore_survivors": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vs_score64": (C.c_int, [C.c_void_p, P(vs_library), C.c_int64, P(C.c_int32), P(C.c_double),
                             P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double)]),
    "vs_dock_refined_host": (C.c_int, [C.c_void_p, P(vs_library), P(vs_size_class), C.c_int32,
                                       P(vs_dock_params), C.c_int32, P(vs_refined)]),
    "vs_ascend": (C.c_int, [C.c_void_p, P(vs_library), C.c_int64, P(C.c_int32), P(C.c_double),
                            P(C.c_double), P(C.c_double), C.c_int32, P(C.c_double),
                            P(C.c_int32)]),
    "vs_rng_u64": (C.c_int, [C.c_uint64, P(C.c_uint64), C.c_int32, C.c_int32, P(C.c_uint64)]),
    "vs_random_smiles": (C.c_int, [C.c_uint64, C.c_uint64, C.c_char_p, C.c_int32]),
    "vs_ligand_build": (C.c_int, [C.c_char_p, C.c_uint64, C.c_int32, P(vs_ligand_buf)]),
    "vs_libbuild_run": (C.c_int, [C.c_char_p, C.c_int32, P(C.c_uint64), C.c_int32, C.c_int32,
                                  P(C.c_void_p)]),
    "vs_libbuild_sizes": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_int64)]),
    "vs_libbuild_fetch": (C.c_int, [C.c_void_p] + [P(C.c_int32)] * 4 + [P(C.c_double)] +
                          [P(C.c_int32)] * 5),
    "vs_libbuild_free": (None, [C.c_void_p]),
    "vs_libbuild_relax": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "vs_libbuild_embed": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "vs_corpus_select": (C.c_int, [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_int32, C.c_int64, C.c_int32, P(C.c_int64)]),
    "vs_flexible_select": (C.c_int, [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_int64, P(C.c_int64), P(C.c_int32)]),
    "vs_libbuild_corpus": (C.c_int, [C.c_uint64, P(C.c_int64), C.c_int32, P(C.c_uint64),
                                     C.c_int32, C.c_int32, P(C.c_void_p)]),
    "vs_smzc_decompress": (C.c_int, [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, C.c_int32,
                                     C.c_void_p, C.c_int64, P(C.c_int64)]),
    "vs_codec_last_error": (C.c_char_p, []),
    "vs_host_alloc": (C.c_int, [C.c_int64, P(C.c_void_p)]),
    "vs_host_free": (C.c_int, [C.c_void_p]),
    "vs_smz1_check": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(C.c_int32)]),
    "vs_sha256": (C.c_int, [C.c_char_p, C.c_int64, C.c_char_p]),
    "vs_json_format_doubles": (C.c_int, [P(C.c_double), C.c_int64, C.c_char_p, C.c_int32]),
    "vs_default_classes": (C.c_int, [P(vs_size_class), C.c_int32]),
    "vs_size_class_of": (C.c_int, [C.c_int32, C.c_int32, P(vs_size_class), C.c_int32]),
    "vs_target_batch_size": (C.c_int, [P(vs_size_class), C.c_double, C.c_double, C.c_double,
                                       C.c_double, P(C.c_int64)]),
    "vs_simulate_throughput": (C.c_double, [C.c_int64, C.c_double, C.c_double]),
    "vs_bucket_replay": (C.c_int, [P(C.c_int32), P(C.c_int32), C.c_int32, P(vs_size_class),
                                   C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_double, P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                   P(C.c_int32)]),
    "vs_campaign_seeds": (C.c_int, [C.c_uint64, C.c_int32, P(C.c_int32), C.c_int32,
                                    P(C.c_uint64)]),
    "vs_filter_poses": (C.c_int, [P(C.c_double), C.c_int32, C.c_int64, C.c_double,
                                  P(C.c_int32)]),
    "vs_rank_ligands": (C.c_int, [C.c_char_p, P(C.c_double), C.c_int32, P(C.c_int32)]),
    "vs_id_ranks": (C.c_int, [C.c_char_p, C.c_int32, P(C.c_uint32)]),
}

EXPORTED = tuple(_SIGS)


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2304_09953_b200/build.py` "
            "(there is no CPU fallback for the dock-and-score path)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        if os.environ.get("VSCREEN_GPU_LIB") and not hasattr(lib, name):
            continue  # an older experiment variant (A/B timing) may predate this entry point
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def ptr(arr, ctype):
    """numpy array -> ctypes pointer (None passes through)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(P(ctype))
