"""ctypes mirror of include/djg_types.h, include/djg.h and include/djg_host.h.

The structs here are byte-for-byte the C structs; tests/test_abi.py checks
the field offsets against the compiled library. `load_library()` loads the
in-tree libdjg.so and raises if it is missing -- there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
# DJG_LIB_PATH: developer A/B override (tools/); default the in-tree build.
LIB_PATH = Path(os.environ.get("DJG_LIB_PATH") or PKG_DIR / "_build" / "libdjg.so")

DJG_T4, DJG_H8 = 0, 1
DJG_NH, DJG_TI, DJG_OT, DJG_MR, DJG_I57 = 0, 1, 2, 3, 4
DJG_ABORT, DJG_SKIP_AND_REPORT = 0, 1
DJG_FREE, DJG_FIXED, DJG_PRESCRIBED = 0, 1, 2
DJG_OK, DJG_E_INTERNAL, DJG_E_CONFIG, DJG_E_CUDA, DJG_E_INVERSION, DJG_E_DIVERGENCE, DJG_E_PEER = 0, 1, 2, 3, 4, 5, 6
DJG_FLAG_NO_GRAPH = 1
DJG_FLAG_SLABS = 2
DJG_FLAG_NO_DISCARD = 4
DJG_FLAG_COMPACT = 8
DJG_FLAG_DEVICE_PRECOMPUTE = 16
DJG_FLAG_FULL_RECORD = 32
DJG_FLAG_TLED = 64
DJG_FLAG_NO_PIPE = 128
DJG_FLAG_WINDOW = 256
DJG_FLAG_NO_FUSED = 512
DJG_FLAG_FUSED = 1024
DJG_PART_RCB, DJG_PART_METIS = 0, 1
DJG_PART_BOX = 2
PART_METHODS = {"rcb": DJG_PART_RCB, "metis": DJG_PART_METIS, "box": DJG_PART_BOX}

KIND_NAMES = {"T4": DJG_T4, "H8": DJG_H8}
MODEL_NAMES = {"NH": DJG_NH, "TI": DJG_TI, "OT": DJG_OT, "MR": DJG_MR, "I57": DJG_I57}


def npe_of(kind: int) -> int:
    return 4 if kind == DJG_T4 else 8


def const_count(kind: int, model: int) -> int:
    """Reals in the canonical hot-field record (include/djg.h)."""
    n = 23
    if model in (DJG_TI, DJG_OT):
        n += 12
    if model == DJG_OT:
        n += 12
    if model == DJG_MR:
        n += 57
    if model == DJG_I57:
        n += 114
    if kind == DJG_H8:
        n += 33
    return n


class djg_material_params(C.Structure):
    _fields_ = [
        ("model", C.c_int32), ("_pad", C.c_int32),
        ("mu", C.c_double), ("kappa", C.c_double), ("rho", C.c_double),
        ("eta_a", C.c_double), ("eta_b", C.c_double), ("c10", C.c_double), ("c01", C.c_double),
        ("fibre_a", C.c_double * 3), ("fibre_b", C.c_double * 3),
    ]


class djg_scenario_spec(C.Structure):
    _fields_ = [
        ("precision", C.c_int32), ("kind", C.c_int32),
        ("divisions", C.c_int32 * 3), ("_pad0", C.c_int32),
        ("extent", C.c_double * 3),
        ("num_nodes", C.c_int64), ("num_elements", C.c_int64),
        ("nodes", C.POINTER(C.c_double)), ("conn", C.POINTER(C.c_int32)),
        ("material", djg_material_params),
        ("c_hg", C.c_double),
        ("bc_mode", C.c_int32), ("fix_all_axes", C.c_int32),
        ("target", C.c_double), ("ramp_steps", C.c_int64),
        ("n_fixed", C.c_int64), ("fixed_node", C.POINTER(C.c_int32)), ("fixed_axis", C.POINTER(C.c_int32)),
        ("n_prescribed", C.c_int64), ("presc_node", C.POINTER(C.c_int32)), ("presc_axis", C.POINTER(C.c_int32)),
        ("presc_target", C.POINTER(C.c_double)), ("presc_t_total", C.POINTER(C.c_double)),
        ("dt", C.c_double), ("safety", C.c_double),
        ("alpha_mode", C.c_int32), ("policy", C.c_int32), ("alpha", C.c_double),
    ]


class djg_image_ptrs(C.Structure):
    _fields_ = [
        ("nodes", C.c_void_p), ("conn", C.c_void_p), ("csr_offsets", C.c_void_p), ("csr_elem", C.c_void_p),
        ("csr_local", C.c_void_p), ("consts", C.c_void_p), ("mass", C.c_void_p), ("c1", C.c_void_p),
        ("massless", C.c_void_p), ("dof_kind", C.c_void_p), ("dof_target", C.c_void_p), ("dof_t_total", C.c_void_p),
    ]


class djg_image_scalars(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int64), ("num_elements", C.c_int64), ("npe", C.c_int32), ("nconst", C.c_int32),
        ("dt", C.c_double), ("critical_dt", C.c_double), ("alpha", C.c_double), ("c2", C.c_double),
        ("c3", C.c_double), ("ramp_t_total", C.c_double), ("wave_speed", C.c_double),
    ]


class djg_report(C.Structure):
    _fields_ = [
        ("steps_done", C.c_int64), ("step", C.c_int64), ("first_inverted", C.c_int64),
        ("inverted_count", C.c_int64), ("inverted_steps", C.c_int64), ("fail_step", C.c_int64),
        ("diverged", C.c_int32), ("status", C.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class djg_assemble_stats(C.Structure):
    _fields_ = [("first_inverted", C.c_int64), ("inverted_count", C.c_int64)]


class djg_desc(C.Structure):
    _fields_ = [
        ("precision", C.c_int32), ("kind", C.c_int32), ("num_nodes", C.c_int64), ("num_elements", C.c_int64),
        ("conn", C.c_void_p), ("consts", C.c_void_p), ("nconst", C.c_int32), ("inversion_policy", C.c_int32),
        ("csr_offsets", C.c_void_p), ("csr_elem", C.c_void_p), ("csr_local", C.c_void_p),
        ("dof_kind", C.c_void_p), ("dof_target", C.c_void_p), ("dof_t_total", C.c_void_p),
        ("c1", C.c_void_p), ("massless", C.c_void_p),
        ("c2", C.c_double), ("c3", C.c_double), ("dt", C.c_double),
        ("material", djg_material_params), ("device", C.c_int32), ("flags", C.c_uint32),
        ("nodes", C.c_void_p), ("c_hg", C.c_double),
    ]


class djg_mesh_desc(C.Structure):
    _fields_ = [
        ("precision", C.c_int32), ("kind", C.c_int32), ("num_nodes", C.c_int64), ("num_elements", C.c_int64),
        ("nodes", C.c_void_p), ("conn", C.c_void_p), ("material", djg_material_params), ("c_hg", C.c_double),
        ("inversion_policy", C.c_int32), ("device", C.c_int32), ("flags", C.c_uint32), ("threads", C.c_int32),
    ]


class djg_step_desc(C.Structure):
    _fields_ = [
        ("node_mass", C.c_void_p), ("dof_kind", C.c_void_p), ("dof_target", C.c_void_p),
        ("dof_t_total", C.c_void_p), ("dt", C.c_double), ("alpha", C.c_double),
    ]


class djg_partition_info(C.Structure):
    _fields_ = [
        ("nparts", C.c_int32), ("part", C.c_int32), ("num_neighbors", C.c_int32), ("_pad", C.c_int32),
        ("num_nodes", C.c_int64), ("num_owned", C.c_int64), ("num_elements", C.c_int64),
        ("owned_elements", C.c_int64), ("send_total", C.c_int64), ("recv_total", C.c_int64),
        ("global_nodes", C.c_int64), ("global_elements", C.c_int64), ("interior_elements", C.c_int64),
    ]


class djg_engine_info(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int64), ("num_elements", C.c_int64), ("num_slots", C.c_int64),
        ("slot_capacity", C.c_int64), ("device_bytes", C.c_int64),
        ("npe", C.c_int32), ("nconst", C.c_int32), ("const_planes", C.c_int32), ("precision", C.c_int32),
        ("kernels_per_step", C.c_int32), ("sm_count", C.c_int32), ("slabs", C.c_int32),
        ("compact", C.c_int32), ("slab_elements", C.c_int64), ("formulation", C.c_int32), ("pipelined", C.c_int32),
        ("windowed", C.c_int32), ("window_tiles", C.c_int64), ("fused", C.c_int32), ("lattice", C.c_int32),
    ]


def ptr(a: np.ndarray | None):
    """void* of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:  # explicit check: `python -O` strips asserts
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(C.c_void_p)


def typed_ptr(a: np.ndarray | None, ctype):
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(C.POINTER(ctype))


_P = C.POINTER
# (name, restype, argtypes) of every function include/djg.h and include/djg_host.h declare.
EXPORTS = [
    ("djg_const_count", C.c_int32, [C.c_int32, C.c_int32]),
    ("djg_create", C.c_int, [_P(djg_desc), _P(C.c_void_p)]),
    ("djg_create_from_mesh", C.c_int, [_P(djg_mesh_desc), _P(C.c_void_p)]),
    ("djg_configure_step", C.c_int, [C.c_void_p, _P(djg_step_desc)]),
    ("djg_set_policy", C.c_int, [C.c_void_p, C.c_int32]),
    ("djg_destroy", None, [C.c_void_p]),
    ("djg_set_state", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    ("djg_set_external", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_get_state", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, _P(C.c_int64)]),
    ("djg_step", C.c_int, [C.c_void_p, C.c_int64, _P(djg_report)]),
    ("djg_step_async", C.c_int, [C.c_void_p, C.c_int64]),
    ("djg_sync", C.c_int, [C.c_void_p, _P(djg_report)]),
    ("djg_stream", C.c_void_p, [C.c_void_p]),
    ("djg_assemble", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, _P(djg_assemble_stats)]),
    ("djg_profile_steps", C.c_int, [C.c_void_p, C.c_int64, _P(C.c_float), _P(C.c_float), _P(C.c_float)]),
    ("djg_get_info", C.c_int, [C.c_void_p, _P(djg_engine_info)]),
    ("djg_get_slot_map", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_lump_mass", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_advance_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, _P(djg_report)]),
    ("djg_comm_unique_id", C.c_int, [C.c_void_p]),
    ("djg_set_interior", C.c_int, [C.c_void_p, C.c_int64]),
    ("djg_peer_export", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_peer_ipc_export", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_peer_ipc_open", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("djg_peer_setup", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_void_p, C.c_void_p]),
    ("djg_step_peer_local", C.c_int, [C.c_void_p]),
    ("djg_step_peer_agree", C.c_int, [C.c_void_p]),
    ("djg_step_interior", C.c_int, [C.c_void_p]),
    ("djg_step_boundary", C.c_int, [C.c_void_p]),
    ("djg_comm_init", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    ("djg_min_char_length", C.c_int, [C.c_void_p, _P(C.c_double)]),
    ("djg_get_consts", C.c_int64, [C.c_void_p, C.c_void_p]),
    ("djg_debug_cbrt", C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32]),
    ("djg_set_partition", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    ("djg_set_halo", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]),
    ("djg_set_counted_elements", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_halo_pack", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_halo_unpack", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_step_status", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_step_agree", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_partition_build", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, _P(C.c_void_p)]),
    ("djg_partition_build_method", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, _P(C.c_void_p)]),
    ("djg_partition_build_box", C.c_int, [_P(djg_scenario_spec), C.c_int32, C.c_int32, _P(C.c_void_p),
                                          _P(C.c_double)]),
    ("djg_partition_finish", C.c_int, [C.c_void_p, C.c_double]),
    ("djg_partition_free", None, [C.c_void_p]),
    ("djg_partition_get_info", C.c_int, [C.c_void_p, _P(djg_partition_info)]),
    ("djg_partition_desc", C.c_int, [C.c_void_p, C.c_int32, _P(djg_desc)]),
    ("djg_partition_image", C.c_int, [C.c_void_p, _P(djg_image_ptrs)]),
    ("djg_partition_halo", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("djg_partition_maps", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("djg_partition_owned_elements", C.c_int, [C.c_void_p, C.c_void_p]),
    ("djg_element_parts", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    ("djg_element_parts_method", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    ("djg_last_error", C.c_char_p, [C.c_void_p]),
    ("djg_status_string", C.c_char_p, [C.c_int32]),
    ("djg_create_error", C.c_char_p, []),
    ("djg_spec_default_box", None, [_P(djg_scenario_spec), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64]),
    ("djg_bench_material", None, [C.c_int32, _P(djg_material_params)]),
    ("djg_scenario_build", C.c_int, [_P(djg_scenario_spec), C.c_int32, _P(C.c_void_p)]),
    ("djg_scenario_free", None, [C.c_void_p]),
    ("djg_scenario_error", C.c_char_p, []),
    ("djg_scenario_scalars", C.c_int, [C.c_void_p, _P(djg_image_scalars)]),
    ("djg_scenario_image", C.c_int, [C.c_void_p, _P(djg_image_ptrs)]),
    ("djg_scenario_desc", C.c_int, [C.c_void_p, C.c_int32, _P(djg_desc)]),
]

_lib = None


def load_library(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load libdjg.so (the CUDA engine + host builder). Raises if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"libdjg.so not found at {p}: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, res, args in EXPORTS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
