"""ctypes binding of libowb200.so (include/owb200.h) and device plumbing.

The library is the product: there is no CPU fallback.  Loading fails loudly
when the shared object is missing or no CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libowb200.so")

OW_OK, OW_ERR_INTERNAL, OW_ERR_INVALID, OW_ERR_PARSE, OW_ERR_CAPACITY = 0, 1, 2, 3, 4

_EXC = {
    OW_ERR_INTERNAL: errors.OctowallError,
    OW_ERR_INVALID: errors.InvalidParameterError,
    OW_ERR_PARSE: errors.GeometryParseError,
    OW_ERR_CAPACITY: errors.CapacityError,
}


class Grid(C.Structure):  # ow_grid
    _fields_ = [
        ("dim", C.c_int32),
        ("bins_per_axis", C.c_int32),
        ("dmin", C.c_double * 3),
        ("dmax", C.c_double * 3),
        ("min32", C.c_float * 3),
        ("len32", C.c_float * 3),
    ]


class ForestView(C.Structure):  # ow_forest (fields appended below: self-referential callback)
    pass


GROW_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(ForestView), C.c_int64)

ForestView._fields_ = [
    ("dim", C.c_int32),
    ("max_level", C.c_int32),
    ("root", C.c_int32 * 3),
    ("_pad", C.c_int32),
    ("dmin", C.c_double * 3),
    ("dext", C.c_double * 3),
    ("n_blocks", C.c_int64),
    ("capacity", C.c_int64),
    ("d_level", C.c_void_p),
    ("d_coord", C.c_void_p * 3),
    ("d_parent", C.c_void_p),
    ("d_first_child", C.c_void_p),
    ("d_marks", C.c_void_p),
    ("grow", GROW_FN),
    ("grow_user", C.c_void_p),
]


class FaceSummary(C.Structure):  # ow_face_summary
    _fields_ = [
        ("first_degenerate", C.c_int64),
        ("first_nonfinite", C.c_int64),
        ("bbox_min", C.c_float * 3),
        ("bbox_max", C.c_float * 3),
        ("abs_max", C.c_float),
        ("mean_extent", C.c_float),
    ]


MAX_PASSES = 26  # OW_MAX_PASSES
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                          C.POINTER(C.c_int64))


class NearWallParamsC(C.Structure):  # ow_nearwall_params
    _fields_ = [
        ("d_spec", C.c_float),
        ("n_levels", C.c_int32),
        ("d_spec64", C.c_double),
        ("reach", C.c_double),
        ("binned", C.c_int32),
        ("reuse_bins", C.c_int32),
        ("spacing", C.c_float),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("overlap_factor", C.c_int64),
        ("bin_fraction", C.c_int64),
        ("exchange", EXCHANGE_FN),
        ("exchange_user", C.c_void_p),
        ("comm", C.c_void_p),
    ]


class NearWallResultC(C.Structure):  # ow_nearwall_result
    _fields_ = [
        ("n_passes", C.c_int32),
        ("bins_built", C.c_int32),
        ("bin_entries", C.c_int64),
        ("marked_detected", C.c_int64 * MAX_PASSES),
        ("marked_refined", C.c_int64 * MAX_PASSES),
        ("n_split", C.c_int64 * MAX_PASSES),
        ("tests", C.c_int64 * MAX_PASSES),
        ("evaluated", C.c_int64 * MAX_PASSES),
        ("sphere_tests", C.c_int64 * MAX_PASSES),
        ("box_culls", C.c_int64 * MAX_PASSES),
        ("stage_ms", (C.c_float * 4) * MAX_PASSES),
    ]


ALLOC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_void_p))


class G2GParamsC(C.Structure):  # ow_g2g_params
    _fields_ = [
        ("nw", NearWallParamsC),
        ("lattice_q", C.c_int32),
        ("lattice_dirs", C.c_int8 * 81),
        ("alloc", ALLOC_FN),
        ("alloc_user", C.c_void_p),
        ("out_buf", C.c_void_p * 4),
        ("out_cap", C.c_int64 * 4),
        ("host_level", C.c_void_p),
        ("host_coord", C.c_void_p * 3),
        ("host_parent", C.c_void_p),
        ("host_first_child", C.c_void_p),
        ("host_marks", C.c_void_p),
        ("host_block_cap", C.c_int64),
        ("host_cells", C.c_void_p),
        ("host_q", C.c_void_p),
        ("host_row_cap", C.c_int64),
        ("host_rows", C.c_void_p),
        ("host_q_packed", C.c_void_p),
        ("host_link_cap", C.c_int64),
        ("copy_done", C.c_void_p),
        ("dev_rows", C.c_void_p),
        ("dev_q_packed", C.c_void_p),
        ("dev_row_cap", C.c_int64),
        ("dev_link_cap", C.c_int64),
        ("no_stage_times", C.c_int32),
    ]


class G2GResultC(C.Structure):  # ow_g2g_result
    _fields_ = [
        ("faces", FaceSummary),
        ("outside_domain", C.c_int32),
        ("finest_level", C.c_int32),
        ("nw", NearWallResultC),
        ("n_finest_leaves", C.c_int64),
        ("n_boundary", C.c_int64),
        ("lattice_stats", C.c_int64 * 3),
        ("host_copied", C.c_int32),
        ("reran", C.c_int32),
        ("n_links", C.c_int64),
        ("device_sized", C.c_int32),
        ("reserved", C.c_int32),
    ]


P = C.c_void_p
I32, I64, F32, F64 = C.c_int32, C.c_int64, C.c_float, C.c_double
PI64 = C.POINTER(C.c_int64)

# name -> argtypes (restype int unless listed in _RESTYPE)
_SIGS = {
    "ow_ctx_create": [C.c_int, C.POINTER(P)],
    "ow_ctx_destroy": [P],
    "ow_last_error": [],
    "ow_version": [],
    "ow_launch_count": [P],
    "ow_profile": [P, C.c_int],
    "ow_profile_read": [P, C.c_int, C.POINTER(C.c_double), PI64],
    "ow_stl_binary_to_soa": [P, P, I64, P, P],
    "ow_index_to_coords": [P, I32, P, P, I64, P, P],
    "ow_face_check": [P, I32, P, I64, C.POINTER(FaceSummary), P],
    "ow_fill_bins_count": [P, C.POINTER(Grid), P, I64, F32, P, PI64, PI64, P],
    "ow_fill_bins_emit": [P, C.POINTER(Grid), P, P, P, P],
    "ow_forest_leaves": [P, C.POINTER(ForestView), I32, P, PI64, P],
    "ow_forest_level_counts": [P, C.POINTER(ForestView), PI64, PI64, I32, P],
    "ow_forest_count_marks": [P, C.POINTER(ForestView), I32, I32, I32, PI64, P],
    "ow_forest_cell_centers": [P, C.POINTER(ForestView), P, I64, P, P],
    "ow_refine_marked": [P, C.POINTER(ForestView), I32, PI64, P],
    "ow_mark_near_wall": [P, C.POINTER(ForestView), P, I64, P, I64, I64, C.POINTER(Grid), P, P, P, I64, F32, F64,
                          PI64, PI64, PI64, P],
    "ow_propagate_marks": [P, C.POINTER(ForestView), P, I64, I32, P],
    "ow_forest_init_root": [P, C.POINTER(ForestView), P],
    "ow_geometry_to_grid": [P, P, P, I64, I64, C.POINTER(ForestView), C.POINTER(Grid), C.POINTER(G2GParamsC), P, I64,
                            P, P, C.POINTER(G2GResultC), P],
    "ow_geometry_to_grid_submit": [P, P, P, I64, I64, C.POINTER(ForestView), C.POINTER(Grid), C.POINTER(G2GParamsC),
                                   P, I64, P, P, C.POINTER(G2GResultC), P, PI64],
    "ow_geometry_to_grid_finish": [P, I64, P, I64, I64, C.POINTER(ForestView), C.POINTER(Grid), C.POINTER(G2GParamsC),
                                   P, I64, P, P, C.POINTER(G2GResultC), P],
    "ow_refine_near_wall": [P, C.POINTER(ForestView), P, I64, I64, C.POINTER(Grid), C.POINTER(NearWallParamsC), P,
                            I64, P, P, C.POINTER(NearWallResultC), P],
    "ow_cell_face_links_count": [P, C.POINTER(ForestView), P, I64, P, I64, I64, C.POINTER(Grid), P, P, P, F32, F64,
                                 I64, PI64, PI64, P],
    "ow_cell_face_links_emit": [P, P, P, P, P, P],
    "ow_lattice_links_count": [P, C.POINTER(ForestView), I32, P, I64, P, I64, I64, C.POINTER(Grid), P, I32, P, PI64, P],
    "ow_lattice_links_count_range": [P, C.POINTER(ForestView), I32, P, I64, I64, I64, P, I64, I64, C.POINTER(Grid), P,
                                     I32, P, PI64, P],
    "ow_lattice_links_emit": [P, P, P, P],
    "ow_lattice_links_emit_packed": [P, P, P, P, P, P],
    "ow_lattice_links_n_links": [P, PI64],
    "ow_lattice_stats": [P, PI64, P],
    "ow_lattice_tune": [P, C.c_int32, C.c_int32],
    "ow_set_device_pass": [P, C.c_int32],
    "ow_device_pass_stats": [P, PI64],
    "ow_near_pairs": [P, I32, P, P, P, I64, P, P],
    "ow_export_vtk": [P, C.POINTER(ForestView), C.c_char_p, C.c_char_p, P],
    "ow_referee_pairs": [P, I32, P, P, P, I64, P, P, P],
    "ow_parse_ascii_stl": [C.c_char_p, I64, P, I64, PI64, PI64],
    "ow_comm_create": [C.c_int, I32, I32, I64, C.POINTER(P), P],
    "ow_comm_open": [P, P],
    "ow_comm_destroy": [P],
    "ow_comm_status": [P, PI64],
    "ow_comm_allgather_u32": [P, P, P, I64, I64, I64, P],
}
_RESTYPE = {"ow_last_error": C.c_char_p, "ow_version": C.c_int, "ow_launch_count": C.c_int64}

_lib = None
_tls = threading.local()  # per host thread: {device index: ow_ctx}
_all_ctx = []             # every context made by this process (launch accounting)
_lock = threading.Lock()


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise errors.OctowallError(
                        f"{LIB_PATH} is missing: build it with paper_2502_16310_b200._build.build() "
                        "(there is no CPU fallback)")
                L = C.CDLL(LIB_PATH)
                for name, argt in _SIGS.items():
                    fn = getattr(L, name)
                    fn.argtypes = argt
                    fn.restype = _RESTYPE.get(name, C.c_int)
                _lib = L
    return _lib


def device():
    if not torch.cuda.is_available():
        raise errors.OctowallError("paper_2502_16310_b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def ctx():
    """The calling thread's ow_ctx on the current device (created lazily).

    A context carries two-phase state between calls (fill_bins count -> emit,
    lattice count -> emit, the pinned readback buffer, the copy stream), so
    it is never shared between host threads: one per (thread, device), which
    makes the entry points safe to call concurrently from several threads as
    the reference's pure functions are."""
    dev = device()
    key = dev.index
    per = getattr(_tls, "ctx", None)
    if per is None:
        per = _tls.ctx = {}
    c = per.get(key)
    if c is None:
        c = P()
        check(lib().ow_ctx_create(key, C.byref(c)))
        per[key] = c
        with _lock:
            _all_ctx.append(c)
    return c


def stream():
    return P(torch.cuda.current_stream().cuda_stream)


def check(status, exc_map=None):
    if status == OW_OK:
        return
    msg = lib().ow_last_error().decode("utf-8", "replace")
    cls = (exc_map or {}).get(status) or _EXC.get(status, errors.OctowallError)
    raise cls(msg)


def call(name, *args, exc_map=None):
    check(getattr(lib(), name)(*args), exc_map)


def ptr(t):
    return P(t.data_ptr()) if t is not None else P()


def launches():
    """Kernels launched by this process's contexts so far (bench instrumentation)."""
    with _lock:
        cs = list(_all_ctx)
    return sum(int(lib().ow_launch_count(c)) for c in cs)


PROF_IDS = {"mark": 0, "lattice": 1, "fill_bins": 2, "refine": 3, "propagate": 4, "links": 5, "stl": 6, "prep": 7,
            "lattice_sweep": 8}


def lattice_stats():
    """(candidate blocks, rows, intersection tests) of the last lattice call."""
    out = (C.c_int64 * 3)()
    call("ow_lattice_stats", ctx(), out, stream())
    return tuple(int(x) for x in out)


def set_device_pass(enable=True):
    """Device-sized fused passes on this thread's context (default on):
    ``False`` keeps ``GridPlan.run`` on the synchronous path."""
    call("ow_set_device_pass", ctx(), int(bool(enable)))


def device_pass_stats():
    """(device-sized passes, device-sized attempts that fell back) of this
    thread's context."""
    out = (C.c_int64 * 2)()
    call("ow_device_pass_stats", ctx(), out)
    return int(out[0]), int(out[1])


def profile(enable=True):
    call("ow_profile", ctx(), int(bool(enable)))


def profile_read():
    """{family: (total_ms, launches)} of the CUDA-event brackets since profile()."""
    out = {}
    for name, i in PROF_IDS.items():
        ms, n = C.c_double(0.0), C.c_int64(0)
        call("ow_profile_read", ctx(), i, C.byref(ms), C.byref(n))
        out[name] = (float(ms.value), int(n.value))
    return out


def device_numa_node(index=None):
    """NUMA node of the GPU's PCIe root (sysfs), or None when unknown."""
    index = torch.cuda.current_device() if index is None else index
    p = torch.cuda.get_device_properties(index)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    try:
        node = int(open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip())
    except (OSError, ValueError):
        return None
    return node if node >= 0 else None


def _cpulist(text):
    cpus = set()
    for part in text.strip().split(","):
        if part:
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
    return cpus


def bind_host_numa(index=None):
    """Pin this process's host threads to the CPUs of the GPU's NUMA node, so
    pinned staging buffers allocated afterwards are first-touched there and
    H2D / D2H copies do not cross the socket interconnect.  Call it before
    allocating pinned memory (once per rank, with the rank's device).  Returns
    the node, or None when the topology is unknown (nothing is changed)."""
    node = device_numa_node(index)
    if node is None:
        return None
    try:
        cpus = _cpulist(open(f"/sys/devices/system/node/node{node}/cpulist").read())
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return node
    except (OSError, AttributeError):
        pass
    return None
