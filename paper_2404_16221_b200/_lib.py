"""ctypes binding of the C-ABI library (include/vr_capi.h).

The library is built in-tree (``csrc/build.py`` -> ``libvolray_b200.so``).  There is
no CPU fallback: every hot-path call goes through this module, and loading fails
loudly when the shared object is missing or its struct layouts disagree with the
declarations below.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import (
    CapacityError,
    GradientOverflowError,
    NegativeLossError,
    NonFiniteInputError,
    OutOfBoundsError,
    VrError,
)

LIB_PATH = Path(__file__).resolve().parent / "libvolray_b200.so"
# VR_CHECKED=1: the checked build (device range checks, csrc/build.py --checked)
CHECKED_PATH = Path(__file__).resolve().parent / "libvolray_b200_checked.so"

VR_MAX_REGIONS = 32
VR_MAX_BLOBS = 32
VR_MAX_CHILDREN = 8
VR_MAX_LEVELS = 16
VR_PACKET_FLOATS = 8
VR_OUT_FIELDS = 7
VR_SUM_PARTIALS = 296  # vr_sum_f64 scratch (doubles)

VR_FLAG_NONFINITE = 1
VR_FLAG_NEG_LOSS = 2
VR_FLAG_OOB = 4
VR_FLAG_OVERFLOW = 8
VR_FLAG_TOO_MANY_SEGS = 16
VR_FLAG_GRAD_OVERFLOW = 32

VR_MLP_W1D = 0
VR_MLP_W2D = VR_MLP_W1D + 64 * 32
VR_MLP_W1C = VR_MLP_W2D + 16 * 64
VR_MLP_W2C = VR_MLP_W1C + 64 * 32
VR_MLP_W3C = VR_MLP_W2C + 64 * 64
VR_MLP_NPARAMS = VR_MLP_W3C + 16 * 64

D3 = C.c_double * 3


class VrTree(C.Structure):
    _fields_ = [
        ("root_mn", D3),
        ("root_mx", D3),
        ("leaf_mn", D3 * VR_MAX_REGIONS),
        ("leaf_mx", D3 * VR_MAX_REGIONS),
        ("node_plane", C.c_double * VR_MAX_REGIONS),
        ("node_axis", C.c_int32 * VR_MAX_REGIONS),
        ("node_low", C.c_int32 * VR_MAX_REGIONS),
        ("node_high", C.c_int32 * VR_MAX_REGIONS),
        ("n_leaves", C.c_int32),
        ("n_nodes", C.c_int32),
    ]


class VrBlob(C.Structure):
    _fields_ = [("center", D3), ("amplitude", C.c_double), ("scale", C.c_double), ("color", D3)]


class VrOccupancy(C.Structure):
    _fields_ = [("bits", C.c_void_p), ("res", C.c_int32), ("pad_", C.c_int32)]


class VrAnalyticField(C.Structure):
    _fields_ = [
        ("n_children", C.c_int32),
        ("n_blobs", C.c_int32),
        ("child_kind", C.c_int32 * VR_MAX_CHILDREN),
        ("child_blob_lo", C.c_int32 * VR_MAX_CHILDREN),
        ("child_blob_cnt", C.c_int32 * VR_MAX_CHILDREN),
        ("box_mn", D3 * VR_MAX_CHILDREN),
        ("box_mx", D3 * VR_MAX_CHILDREN),
        ("box_density", C.c_double * VR_MAX_CHILDREN),
        ("box_color", D3 * VR_MAX_CHILDREN),
        ("blobs", VrBlob * VR_MAX_BLOBS),
    ]


class VrVoxelDesc(C.Structure):
    _fields_ = [("box_mn", D3), ("box_mx", D3), ("res", C.c_int32 * 3), ("trilinear", C.c_int32)]


class VrHashGridDesc(C.Structure):
    _fields_ = [
        ("n_levels", C.c_int32),
        ("log2_T", C.c_int32),
        ("scale", C.c_float * VR_MAX_LEVELS),
        ("res", C.c_int32 * VR_MAX_LEVELS),
        ("dense", C.c_int32 * VR_MAX_LEVELS),
        ("offset", C.c_int64 * (VR_MAX_LEVELS + 1)),
        ("box_mn", D3),
        ("box_mx", D3),
    ]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
F32 = C.c_float
F64 = C.c_double

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES = {
    "vr_abi_version": [],
    "vr_tma_available": [],
    "vr_struct_sizes": [P],
    "vr_last_error": [],
    "vr_check_failures": [],
    "vr_device_sync": [],
    "vr_sample_count": [P, P, I64, I64, F64, I32, I32, P, P, P, P, P, P, P, P],
    "vr_scan_workspace_bytes": [I64],
    "vr_scan_offsets": [P, I64, P, P, C.c_size_t, P],
    "vr_sample_fill": [P, P, I64, I64, F64, I32, I32, P, P, P, P, P, I64, P, P, P],
    "vr_sample_stage_blocks": [I64],
    "vr_sample_stage": [P, P, I64, I64, F64, I32, I32, P, P, P, P, P, P, P, I64, P, P, P, P, P,
                        P],
    "vr_sample_compact": [I64, I32, P, P, P, P, P, P, P, P, P, I64, P, P],
    "vr_locate": [P, P, I64, P, P, P],
    "vr_field_analytic_fwd": [P, P, I64, P, P, P, I64, P, P],
    "vr_voxel_fwd": [P, P, P, P, I64, P, P, P, I64, P, P],
    "vr_voxel_bwd": [P, P, I64, P, P, P, I64, P, P, P],
    "vr_voxel_fwd_f64": [P, P, P, P, I64, P, P, P, I64, P, P, P],
    "vr_occupancy_points": [P, P, I32, C.c_uint32, P, P],
    "vr_occupancy_update": [P, I32, F32, F32, P, P, P],
    "vr_segment_aggregate_f64": [P, P, P, P, P, I64, P, P],
    "vr_compose_f64": [P, P, I32, I64, P, P, P],
    "vr_hash_fwd": [P, P, P, I64, P, P, P, I64, P, P, P],
    "vr_hash_bwd_workspace_bytes": [P],
    "vr_hash_bwd": [P, P, I64, P, P, P, I64, P, P, P, C.c_size_t, P],
    "vr_hash_indices": [P, P, I64, P, P, P, I64, P, P],
    "vr_hash_positions": [P, P, I64, P, P, P, I64, P, P],
    "vr_hash_lm_passes": [P],
    "vr_hash_fwd_lm": [P, P, P, I64, P, P],
    "vr_hash_bwd_lm": [P, P, I64, P, P, P, C.c_size_t, P],
    "vr_hash_scatter": [P, P, I64, P, P, P, C.c_size_t, I32, I32, P, P, P],
    "vr_mlp_fwd": [P, P, P, I64, P, I64, P, P],
    "vr_mlp_bwd": [P, P, P, I64, P, I64, P, P, P, P],
    "vr_mlp_fwd_tc": [P, P, P, I64, P, I64, P, P],
    "vr_mlp_bwd_tc": [P, P, P, I64, P, I64, P, P, P, P, P, I32, P, P, P],
    "vr_mlp_fwd_tc_density": [P, P, I64, P, P],
    "vr_mlp_bwd_tc_density": [P, P, P, I64, P, I64, P, P, P, P, P, I32, P, P, P],
    "vr_field_fwd_tc": [P, P, P, P, I64, P, P, P, I64, P, P, P],
    "vr_field_bwd_tc": [P, P, P, P, I64, P, P, P, I64, P, P, P, P, P, C.c_size_t, P, P, P, P, P],
    "vr_active_rows_workspace_bytes": [I64],
    "vr_active_rows": [P, I64, P, P, P, C.c_size_t, P],
    "vr_segment_fwd": [P, P, P, P, P, P, I64, I32, P, P, P, I64, P],
    "vr_segment_bwd": [P, P, P, P, P, I64, I32, P, P, P, P],
    "vr_segment_transmittance": [P, P, P, P, I64, I32, P, P],
    "vr_segment_permute": [P, P, P, I64, I32, P, P, I32, I32, P],
    "vr_packets_pack": [P, P, P, I64, I32, I32, P, I64, P, P, P],
    "vr_packets_unpack": [P, I32, I64, I32, I64, I32, P, P, P, P],
    "vr_global_fwd": [P, I32, I64, P, P, I32, P, P, P],
    "vr_global_fwd_records": [P, I32, P, I32, I64, P, P, I32, P, P, P],
    "vr_global_train_records": [P, I32, P, I32, I64, P, P, P, F32, I32, I32, P, P, P, P, P],
    "vr_packets_index": [P, I32, I64, I32, I64, I32, P, P, P],
    "vr_prefix_train_records": [P, P, I32, I64, I32, I32, P, P],
    "vr_global_train": [P, I32, I64, P, P, P, F32, I32, I32, P, P, P, P, P],
    "vr_prefix_train": [P, P, I32, I64, I32, I32, P, P],
    "vr_interlevel": [P, P, P, P, P, P, I64, I32, F32, F32, P, P, P],
    "vr_sum_f64": [P, I64, P, P, P],
    "vr_adam_step": [P, P, P, P, I64, F32, F32, F32, F32, I32, P, P],
    "vr_cast_f32_f16": [P, P, I64, P],
}
_RESTYPES = {"vr_last_error": C.c_char_p, "vr_scan_workspace_bytes": C.c_size_t,
             "vr_sample_stage_blocks": C.c_int64,
             "vr_hash_bwd_workspace_bytes": C.c_size_t,
             "vr_active_rows_workspace_bytes": C.c_size_t}

_LIB = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load (once) and type the C-ABI library; raises ImportError if absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    # VR_LIB_PATH: another build of the same ABI (A/B comparisons of kernel variants)
    p = Path(path) if path else Path(os.environ["VR_LIB_PATH"]) if os.environ.get(
        "VR_LIB_PATH") else (CHECKED_PATH if os.environ.get("VR_CHECKED") == "1" else LIB_PATH)
    if not p.exists():
        raise ImportError(
            f"volray B200 library not built: {p} is missing (run __graft_entry__.build() "
            "or python paper_2404_16221_b200/csrc/build.py). There is no CPU fallback."
        )
    lib = C.CDLL(str(p))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int)
    sizes = (C.c_int64 * 5)()
    lib.vr_struct_sizes(sizes)
    want = [C.sizeof(VrTree), C.sizeof(VrAnalyticField), C.sizeof(VrVoxelDesc),
            C.sizeof(VrHashGridDesc), C.sizeof(VrBlob)]
    if list(sizes) != want:
        raise ImportError(f"vr_capi.h struct layout mismatch: C {list(sizes)} vs ctypes {want}")
    _LIB = lib
    return lib


# Optional per-entry-point CUDA-event timer (bench.py's kernel roofline): an object with
# before(name, args) / after(name), both recording events on the current stream.
TIMER = None
# kernel launches per entry point (for bench.py's gpu_launches count)
# kernels per call where it is not one (checked against the ncu launch list of a c3 step;
# the hash-grid backward entry points add k_hash_rep_reduce for the replicated coarse
# level, vr_sample_stage adds k_sample_prefilter on a rank owning part of the regions)
LAUNCHES = {"vr_scan_offsets": 3, "vr_sum_f64": 2, "vr_field_bwd_tc": 2, "vr_hash_bwd": 2,
            "vr_hash_scatter": 2, "vr_hash_bwd_lm": 2, "vr_packets_pack": 2,
            "vr_packets_unpack": 2, "vr_active_rows": 3}
CALLS = {}
# kernels launched by the calls above
LAUNCHED = {}


def _launches(lib, name: str, args) -> int:
    return LAUNCHES.get(name, 1)


def call(name: str, *args) -> None:
    """Invoke an entry point and raise on a non-zero status."""
    lib = load()
    CALLS[name] = CALLS.get(name, 0) + 1
    LAUNCHED[name] = LAUNCHED.get(name, 0) + _launches(lib, name, args)
    if TIMER is not None:
        TIMER.before(name, args)
    rc = getattr(lib, name)(*args)
    if TIMER is not None:
        TIMER.after(name)
    if rc != 0:
        msg = lib.vr_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{name}: {msg}")
        raise VrError(f"{name} failed ({rc}): {msg}")


def raise_flags(flags: int, where: str = "") -> None:
    """Map device error bits to the reference's exception classes."""
    if not flags:
        return
    if flags & VR_FLAG_NONFINITE:
        raise NonFiniteInputError(f"non-finite segment aggregate {where}")
    if flags & VR_FLAG_NEG_LOSS:
        raise NegativeLossError(f"composed distortion below -1e-12 {where}")
    if flags & VR_FLAG_OOB:
        raise OutOfBoundsError(f"sample point outside the root box {where}")
    if flags & (VR_FLAG_OVERFLOW | VR_FLAG_TOO_MANY_SEGS):
        raise CapacityError(f"capacity overflow (flags={flags}) {where}")
    if flags & VR_FLAG_GRAD_OVERFLOW:
        raise GradientOverflowError(f"MLP gradient beyond the fp16 range {where}")
    raise VrError(f"device error flags {flags} {where}")


def ptr(t) -> int | None:
    """Device/host pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def addr(obj) -> int:
    """Host address of a ctypes struct/array (descriptor arguments)."""
    return C.addressof(obj)
